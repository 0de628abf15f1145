set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py -q -x -m gpu > gpurun_out/g14_tests.log 2>&1
tail -2 gpurun_out/g14_tests.log
for V in 1 0; do
VR_OVERLAP_BWD=$V timeout 900 python bench.py --sub "" --no-cpu --no-e2e > gpurun_out/g14_bench_$V.log 2>&1
tail -1 gpurun_out/g14_bench_$V.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ovl $V', d['value'], d['ms_per_step'])
for k,v in d['kernels'].items():
  if 'bwd' in k or 'scatter' in k or 'rows' in k: print('  ', k, round(v['ms_per_step'],2))"
done
