#!/bin/bash
# One GPU call: ncu --set full of each hot kernel (one launch each, after warm-up) at c3
# with 262144 rays.  The plain command runs first and must exit 0 before any ncu pass.
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --rays 262144"
$CMD > gpurun_out/p_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/p_plain.log; exit 1; }
for ks in k_mlp_bwd_tc:9 k_hash_fwd:9 k_mlp_fwd_tc:9 k_segment_bwd_grp:3 k_segment_fwd_grp:3 k_sample:5; do
  k=${ks%%:*}; s=${ks##*:}
  timeout 600 ncu --set full --clock-control none --import-source on \
      -k regex:"$k" -s $s -c 1 -o gpurun_out/p_$k $CMD > gpurun_out/p_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
tail -3 gpurun_out/p_plain.log | cut -c1-300
