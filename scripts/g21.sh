set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/g21_tests.log 2>&1
tail -3 gpurun_out/g21_tests.log
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/g21_bench.log 2>&1
tail -1 gpurun_out/g21_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['step_ms_trend'], d['active_rows'], d['e2e']['value'], d['clocks'], d['gpu_launches'])
print(json.dumps(d['roofline'])[:700])
for k,v in d['kernels'].items(): print('  ', k, round(v['ms_per_step'],2))
for k,v in d['sub_results'].items(): print(k, v['value'], v['ms_per_step'], v['e2e']['value'] if v.get('e2e') else None)
print(json.dumps(d['cpu_baseline']))"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g21_ref.log 2>&1
tail -1 gpurun_out/g21_ref.log | cut -c1-400
