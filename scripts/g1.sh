set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/g1_tests.log 2>&1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/g1_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/g1_bench.log 2>&1
tail -25 gpurun_out/g1_tests.log; tail -2 gpurun_out/g1_smoke.log; tail -1 gpurun_out/g1_bench.log | cut -c1-1500
