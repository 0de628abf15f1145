set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/g11_tests.log 2>&1
tail -3 gpurun_out/g11_tests.log
timeout 900 python -m pytest "tests/test_gpu_configs.py" -q -s -m gpu 2>&1 | grep "per-sample\|passed\|failed" | cut -c1-180
timeout 900 python bench.py --sub "" --no-cpu --no-e2e > gpurun_out/g11_bench.log 2>&1
tail -1 gpurun_out/g11_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])
for k,v in d['kernels'].items(): print('  ', k, round(v['ms_per_step'],2))"
