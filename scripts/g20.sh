set -u
for cfg in "VR_SC_MINB=1" "VR_SC_MINB=4"; do
env $cfg timeout 900 python bench.py --sub "" --no-cpu --no-e2e --steps 5 > gpurun_out/g20_bench.log 2>&1
tail -1 gpurun_out/g20_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['ms_per_step'])
for k,v in d['kernels'].items():
  if 'scatter' in k or 'bwd' in k: print('  ', k, round(v['ms_per_step'],2))"
VR_OVERLAP_BWD=0 env $cfg timeout 900 python bench.py --sub "" --no-cpu --no-e2e --steps 5 > gpurun_out/g20_bench.log 2>&1
tail -1 gpurun_out/g20_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('serial $cfg', d['value'], d['ms_per_step'])
for k,v in d['kernels'].items():
  if 'scatter' in k or 'bwd' in k: print('  ', k, round(v['ms_per_step'],2))"
done
