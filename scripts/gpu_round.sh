#!/bin/bash
# One GPU call: tests, smoke, benches (c3 default, c4, c5, reference arm), ncu launch
# list of the default bench and --set full captures of the hot kernels.
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
bash scripts/prof_one.sh k_mlp_bwd_tc 9 r_mlp_bwd_fused > /dev/null 2>&1
bash scripts/prof_one.sh k_hash_fwd 9 r_hash_fwd > /dev/null 2>&1
bash scripts/prof_one.sh "^k_sample$" 1 r_sample_stage > /dev/null 2>&1
bash scripts/prof_one.sh k_sample_compact 1 r_sample_compact > /dev/null 2>&1
cat gpurun_out/r_tests.log gpurun_out/r_smoke.log
for f in r_bench_c3 r_bench_c4 r_bench_c5 r_bench_ref; do echo "== $f"; tail -1 gpurun_out/$f.log | cut -c1-400; done
ls gpurun_out/r_*.ncu-rep
