set -u
mkdir -p gpurun_out
for W in grp ls; do
VR_K4_WALK=$W timeout 900 python -m pytest "tests/test_gpu_configs.py::test_c1_matches_oracle" "tests/test_gpu_configs.py::test_c2_two_processes_match_single_process_oracle_and_c1" -q -s -m gpu > gpurun_out/g9_$W.log 2>&1
echo "== $W"; grep "per-sample\|passed\|failed" gpurun_out/g9_$W.log | cut -c1-200
done
for W in grp ls; do
VR_K4_WALK=$W timeout 900 python bench.py --sub "" --no-cpu --no-e2e --steps 5 > gpurun_out/g9_bench_$W.log 2>&1
tail -1 gpurun_out/g9_bench_$W.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$W', d['value'], d['ms_per_step'])
for k,v in d['kernels'].items():
  if 'segment' in k or 'interlevel' in k: print('  ', k, round(v['ms_per_step'],2))"
done
