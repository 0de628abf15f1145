#!/bin/bash
# Final round-2 evidence refresh after the interlevel / position-pass changes: the c4 launch
# list of one steady-state step and --set full captures of k_interlevel and k_hash_pos
# (summarised on the box; reports removed).
set -u
OUT=gpurun_out/r2d
mkdir -p $OUT
C4="python bench.py --config c4 --sub none --steps 1 --warmup 1 --burnin 24 --batches 4 --no-cpu --no-e2e"
$C4 > $OUT/plain_c4.json 2> $OUT/plain_c4.err || { echo "plain run failed"; exit 1; }
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/c4_launches_all.csv $C4 > $OUT/launches.log 2>&1
echo "launch list rc=$?"
cap() {
  local n=$1 k=$2 s=$3; shift 3
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c 1 \
      -o $OUT/$n "$@" > $OUT/ncu_$n.log 2>&1
  echo "$n rc=$?"
  python scripts/ncu_summary.py $OUT/$n.ncu-rep 12 > $OUT/$n.txt 2>&1
  python scripts/ncu_lines.py $OUT/$n.ncu-rep 25 > $OUT/${n}_lines.txt 2>&1
  rm -f $OUT/$n.ncu-rep
}
cap c4_k_interlevel '^k_interlevel' 25 $C4
cap c4_k_hash_pos '^k_hash_pos' 200 $C4
cap c4_k_segment_fwd_ls '^k_segment_fwd_ls' 25 $C4
du -sh gpurun_out
