#!/bin/bash
# After the ReLU-in-conversion epilogue: --set full captures of the MLP forward at the
# bench's steady state (c4 step 26 region 0, c5), and the c4 / c5 launch lists of one step.
# Reports summarised on the box and removed (as prof_r2c.sh).
set -u
OUT=gpurun_out/r2e
mkdir -p $OUT
C4="python bench.py --config c4 --sub none --steps 1 --warmup 1 --burnin 24 --batches 4 --no-cpu --no-e2e"
C5="python bench.py --config c5 --sub none --steps 1 --warmup 1 --batches 4 --no-cpu --no-e2e"
cap() {  # cap <out-name> <kernel-regex> <skip> <cmd...>
  local n=$1 k=$2 s=$3; shift 3
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c 1 \
      -o $OUT/$n "$@" > $OUT/ncu_$n.log 2>&1
  echo "$n rc=$?"
  python scripts/ncu_summary.py $OUT/$n.ncu-rep 12 > $OUT/$n.txt 2>&1
  python scripts/ncu_lines.py $OUT/$n.ncu-rep 25 > $OUT/${n}_lines.txt 2>&1
}
$C4 > $OUT/plain_c4.json 2> $OUT/plain_c4.err || { echo "plain c4 failed"; tail -5 $OUT/plain_c4.err; exit 1; }
$C5 > $OUT/plain_c5.json 2> $OUT/plain_c5.err || { echo "plain c5 failed"; exit 1; }
cap c4_k_mlp_fwd_tc '^k_mlp_fwd_tc' 400 $C4
cap c5_k_mlp_fwd_tc '^k_mlp_fwd_tc' 40 $C5
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/c4_launches_all.csv $C4 > $OUT/launches_c4.log 2>&1
echo "c4 launch list rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/c5_launches_all.csv $C5 > $OUT/launches_c5.log 2>&1
echo "c5 launch list rc=$?"
rm -f $OUT/*.ncu-rep
du -sh gpurun_out
