set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hand_cases.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py "tests/test_gpu_configs.py::test_c1_matches_oracle" -q -x -m gpu > gpurun_out/g23_tests.log 2>&1
tail -2 gpurun_out/g23_tests.log
timeout 300 python scripts/k4_tma_check.py 2>&1 | tail -3
for V in 1 0; do
VR_K4_TMA=$V timeout 900 python bench.py --sub "" --no-cpu --no-e2e --steps 5 > gpurun_out/g23_bench.log 2>&1
tail -1 gpurun_out/g23_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('tma=$V', d['value'], d['ms_per_step'])
for k,v in d['kernels'].items():
  if 'segment' in k: print('  ', k, round(v['ms_per_step'],2))"
done
