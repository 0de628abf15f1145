#!/bin/bash
# ncu --set full of the c4 level-major hash kernels (one launch each, reduced ray batch)
set -u
mkdir -p gpurun_out
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e --rays 1048576"
$CMD > gpurun_out/c4p_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/c4p_plain.log; exit 1; }
for ks in k_hash_bwd_lm:9 k_hash_fwd_lm:9; do
  k=${ks%%:*}; s=${ks##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c 1 \
      -o gpurun_out/c4p_$k $CMD > gpurun_out/c4p_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
