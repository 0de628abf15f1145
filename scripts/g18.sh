set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py tests/test_gpu_hand_cases.py "tests/test_gpu_configs.py::test_c1_matches_oracle" tests/test_gpu_checked.py -q -x -m gpu > gpurun_out/g18_tests.log 2>&1
tail -2 gpurun_out/g18_tests.log
for i in 1 2; do
timeout 900 python bench.py --sub "" --no-cpu --no-e2e > gpurun_out/g18_bench.log 2>&1
tail -1 gpurun_out/g18_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])
for k,v in d['kernels'].items():
  if v['ms_per_step'] > 2: print('  ', k, round(v['ms_per_step'],2))"
done
