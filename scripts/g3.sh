set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sparse_bwd.py -q -x -m gpu > gpurun_out/g3_tests.log 2>&1
tail -3 gpurun_out/g3_tests.log
timeout 900 python bench.py --sub "" --no-cpu > gpurun_out/g3_bench.log 2>&1
tail -1 gpurun_out/g3_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['step_ms_trend'])
for k,v in d['kernels'].items(): print(k, round(v['ms_per_step'],2))"
timeout 300 python scripts/active_frac.py c4 2>&1 | tail -3
timeout 300 python scripts/active_frac.py c3 2>&1 | tail -3
