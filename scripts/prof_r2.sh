#!/bin/bash
# Round-2 profiles of the c4 headline step at full size (4M rays, T = 2^22): the ncu
# launch list of one step, then --set full of one launch of each major kernel (the second
# step's region-0 instance), each only after the same command exited 0 without ncu.
#   bash scripts/prof_r2.sh [c4|c3|c5] [kernels...]
set -u
CFG=${1:-c4}
shift || true
OUT=gpurun_out/r2_$CFG
mkdir -p $OUT
CMD="python bench.py --config $CFG --sub none --steps 1 --warmup 1 --burnin 0 --batches 1 --no-cpu --no-e2e"
$CMD > $OUT/plain.json 2> $OUT/plain.err || { echo "plain run failed"; tail -5 $OUT/plain.err; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/launches.log 2>&1
echo "launch list rc=$?"
# kernel regex : launches of that name to skip (one step's worth)
if [ $CFG = c4 ]; then
  KS=${@:-"k_mlp_bwd_tc:16 k_hash_bwd_lm:2 k_hash_fwd_lm:8 k_hash_fwd:8 k_mlp_fwd_tc:16 k_segment_fwd_grp:1 k_segment_bwd_grp:1 k_interlevel:1 k_sample:2 k_hash_bwd:8"}
elif [ $CFG = c3 ]; then
  KS=${@:-"k_mlp_bwd_tc:8 k_hash_fwd:8 k_mlp_fwd_tc:8 k_segment_fwd_grp:1 k_segment_bwd_grp:1"}
else
  KS=${@:-"k_hash_fwd_lm:8 k_mlp_fwd_tc:8 k_segment_fwd_grp:1 k_hash_pos:8"}
fi
for ks in $KS; do
  k=${ks%%:*}; s=${ks##*:}
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^$k\$|^$k<" \
      --kernel-name-base function -s $s -c 1 -o $OUT/$k $CMD > $OUT/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
