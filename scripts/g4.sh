set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/g4_bench.log 2>&1
tail -1 gpurun_out/g4_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['step_ms_trend'], d['active_rows'], d['e2e']['value'])
print(json.dumps(d['roofline'])[:600])
for k,v in d['sub_results'].items(): print(k, v['value'], v['ms_per_step'], v.get('active_rows'), json.dumps(v.get('roofline'))[:300])"
VR_OVERLAP_FWD=1 timeout 900 python bench.py --sub "" --no-cpu --no-e2e > gpurun_out/g4_ovl.log 2>&1
tail -1 gpurun_out/g4_ovl.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('overlap fwd', d['value'], d['ms_per_step'])"
CMD="python bench.py --sub none --steps 1 --warmup 1 --burnin 24 --batches 4 --no-cpu --no-e2e"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g4_launches.csv $CMD > gpurun_out/g4_ncu.log 2>&1
echo ncu rc=$?
