#!/bin/bash
# Steady-state (24 burn-in steps) ncu --set full captures of the c4 backward kernels after
# the sparse backward: one launch each of the NeRF scatter, the NeRF MLP backward and the
# proposal MLP backward (launch order per step: NeRF regions 0-7, then proposals 0-7), each
# only after the same command exited 0 without ncu.   prof_r2b.sh [regex:skip:name ...]
set -u
OUT=gpurun_out/r2b
mkdir -p $OUT
CMD="python bench.py --config c4 --sub none --steps 1 --warmup 1 --burnin 24 --batches 4 --no-cpu --no-e2e"
$CMD > $OUT/plain.json 2> $OUT/plain.err || { echo "plain run failed"; tail -5 $OUT/plain.err; exit 1; }
for e in ${@:-k_hash_bwd_lm:400:scatter_nerf k_hash_bwd_lm:408:scatter_prop k_mlp_bwd_tc:400:mlp_bwd_nerf k_mlp_bwd_tc:408:mlp_bwd_prop}; do
  IFS=: read -r k s n <<< "$e"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^$k" \
      -s $s -c 1 -o $OUT/$n $CMD > $OUT/ncu_$n.log 2>&1
  echo "$n rc=$?"
done
