set -u
mkdir -p gpurun_out
for cfg in "VR_IL_MINB=1 VR_K4_MINB=2" "VR_IL_MINB=3 VR_K4_MINB=3" "VR_IL_MINB=4 VR_K4_MINB=2"; do
env $cfg timeout 900 python bench.py --sub "" --no-cpu --no-e2e --steps 5 > gpurun_out/g19_bench.log 2>&1
tail -1 gpurun_out/g19_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['ms_per_step'])
for k,v in d['kernels'].items():
  if 'segment' in k or 'interlevel' in k: print('  ', k, round(v['ms_per_step'],2))"
done
