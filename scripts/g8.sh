set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k interlevel -q -x -m gpu > gpurun_out/g8_tests.log 2>&1
tail -3 gpurun_out/g8_tests.log
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_configs.py -q -x -m gpu > gpurun_out/g8_tests2.log 2>&1
tail -3 gpurun_out/g8_tests2.log
timeout 900 python bench.py --sub "" --no-cpu --no-e2e > gpurun_out/g8_bench.log 2>&1
tail -1 gpurun_out/g8_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])
for k,v in d['kernels'].items(): print('  ', k, round(v['ms_per_step'],2))"
