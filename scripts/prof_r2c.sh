#!/bin/bash
# Round-2 evidence after the sparse backward / lane-serial K4 / scatter ILP changes, at the
# bench's steady state (24 burn-in + 1 warm-up steps, rotating batches): the ncu launch list
# of one c4 step, --set full captures of the major kernels of step 26 (region 0 instances;
# per step: 8 NeRF then 8 proposal launches of k_hash_fwd_lm / k_mlp_bwd_tc / k_hash_bwd_lm,
# 16 of k_rows_*), the active-row counts of that step, and c3 / c5 captures.  Each ncu
# command runs only after the same command exited 0 without ncu.  The reports are
# summarised on the box (scripts/ncu_summary.py, ncu_lines.py, ncu_bounds_r2c.py) and
# removed, so gpurun_out stays small.    prof_r2c.sh A|B
set -u
OUT=gpurun_out/r2c
mkdir -p $OUT
PART=${1:-A}
C4="python bench.py --config c4 --sub none --steps 1 --warmup 1 --burnin 24 --batches 4 --no-cpu --no-e2e"
C3="python bench.py --config c3 --sub none --steps 1 --warmup 1 --burnin 24 --batches 4 --no-cpu --no-e2e"
C5="python bench.py --config c5 --sub none --steps 1 --warmup 1 --batches 4 --no-cpu --no-e2e"
cap() {  # cap <out-name> <kernel-regex> <skip> <cmd...>
  local n=$1 k=$2 s=$3; shift 3
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c 1 \
      -o $OUT/$n "$@" > $OUT/ncu_$n.log 2>&1
  echo "$n rc=$?"
  python scripts/ncu_summary.py $OUT/$n.ncu-rep 12 > $OUT/$n.txt 2>&1
  python scripts/ncu_lines.py $OUT/$n.ncu-rep 25 > $OUT/${n}_lines.txt 2>&1
}
if [ $PART = A ]; then
  $C4 > $OUT/plain_c4.json 2> $OUT/plain_c4.err || { echo "plain run failed"; tail -5 $OUT/plain_c4.err; exit 1; }
  python scripts/rows_at_step.py c4 25 > $OUT/rows_c4.json 2> $OUT/rows_c4.err
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/c4_launches_all.csv $C4 > $OUT/launches.log 2>&1
  echo "launch list rc=$?"
  cap c4_k_hash_fwd_lm_nerf '^k_hash_fwd_lm' 400 $C4
  cap c4_k_hash_fwd_lm_prop '^k_hash_fwd_lm' 408 $C4
  cap c4_k_hash_bwd_lm_nerf '^k_hash_bwd_lm' 400 $C4
  cap c4_k_hash_bwd_lm_prop '^k_hash_bwd_lm' 408 $C4
  cap c4_k_mlp_bwd_tc_nerf '^k_mlp_bwd_tc' 400 $C4
  cap c4_k_mlp_bwd_tc_prop '^k_mlp_bwd_tc' 408 $C4
else
  $C4 > $OUT/plain_c4b.json 2> $OUT/plain_c4b.err || { echo "plain run failed"; exit 1; }
  cap c4_k_mlp_fwd_tc '^k_mlp_fwd_tc' 400 $C4
  cap c4_k_mlp_bwd_tc_nerf '^k_mlp_bwd_tc' 400 $C4
  cap c4_k_segment_fwd_ls '^k_segment_fwd_ls' 25 $C4
  cap c4_k_segment_bwd_ls '^k_segment_bwd_ls' 25 $C4
  cap c4_k_interlevel '^k_interlevel' 25 $C4
  cap c4_k_sample '^k_sample$|^k_sample<' 25 $C4
  $C3 > $OUT/plain_c3.json 2> $OUT/plain_c3.err && python scripts/rows_at_step.py c3 25 > $OUT/rows_c3.json 2> $OUT/rows_c3.err
  cap c3_k_mlp_bwd_tc '^k_mlp_bwd_tc' 200 $C3
  cap c3_k_hash_fwd '^k_hash_fwd$|^k_hash_fwd\(' 200 $C3
  $C5 > $OUT/plain_c5.json 2> $OUT/plain_c5.err
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/c5_launches_all.csv $C5 > $OUT/launches_c5.log 2>&1
  cap c5_k_hash_fwd_lm '^k_hash_fwd_lm' 40 $C5
  cap c5_k_mlp_fwd_tc '^k_mlp_fwd_tc' 40 $C5
fi
# raw metrics for profiles/kernel_bounds.json, then drop the reports
mkdir -p $OUT/raw
for r in $OUT/*.ncu-rep; do
  ncu -i $r --page raw --csv > $OUT/raw/$(basename $r .ncu-rep).csv 2>/dev/null
done
rm -f $OUT/*.ncu-rep
du -sh gpurun_out
