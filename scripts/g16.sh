set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py "tests/test_gpu_configs.py::test_c1_matches_oracle" -q -x -m gpu > gpurun_out/g16_tests.log 2>&1
tail -2 gpurun_out/g16_tests.log
VR_OVERLAP_BWD=0 timeout 900 python bench.py --sub "" --no-cpu --no-e2e > gpurun_out/g16_bench0.log 2>&1
tail -1 gpurun_out/g16_bench0.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])
for k,v in d['kernels'].items():
  if 'bwd' in k or 'scatter' in k or 'rows' in k: print('  ', k, round(v['ms_per_step'],2))"
timeout 900 python bench.py --sub "" --no-cpu --no-e2e > gpurun_out/g16_bench.log 2>&1
tail -1 gpurun_out/g16_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
