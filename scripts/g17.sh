set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hand_cases.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py "tests/test_gpu_configs.py::test_c1_matches_oracle" -q -x -m gpu > gpurun_out/g17_tests.log 2>&1
tail -2 gpurun_out/g17_tests.log
timeout 900 python bench.py --sub "" --no-cpu --no-e2e > gpurun_out/g17_bench.log 2>&1
tail -1 gpurun_out/g17_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])
for k,v in d['kernels'].items(): print('  ', k, round(v['ms_per_step'],2))"
