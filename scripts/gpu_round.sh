#!/bin/bash
# One GPU call: tests, smoke, benches, ncu launch list + full capture of the hot kernels.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/r_tests.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r_bench_c3.log 2>&1
timeout 900 python bench.py --config c4 --steps 5 > gpurun_out/r_bench_c4.log 2>&1
timeout 600 python bench.py --config c5 > gpurun_out/r_bench_c5.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/r_bench_ref.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/r_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
      --log-file gpurun_out/r_launches.csv $CMD > gpurun_out/r_ncu_launch.log 2>&1
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --rays 262144"
$CMD2 > gpurun_out/r_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on \
      -k regex:"k_hash_fwd|k_mlp_bwd_tc|k_mlp_fwd_tc|k_segment_bwd_grp|k_sample" -s 40 -c 6 \
      -o gpurun_out/r_prof $CMD2 > gpurun_out/r_ncu_full.log 2>&1
cat gpurun_out/r_tests.log gpurun_out/r_smoke.log
for f in r_bench_c3 r_bench_c4 r_bench_c5 r_bench_ref; do echo "== $f"; tail -1 gpurun_out/$f.log | cut -c1-400; done
tail -2 gpurun_out/r_ncu_full.log
