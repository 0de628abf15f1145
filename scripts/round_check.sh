#!/bin/bash
# Round-end check on one GPU: the whole -m gpu suite, smoke(), the default bench line (c4
# headline with c3 / c5 sub-results, e2e, CPU baseline) and the reference arm.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/rc_tests.log 2>&1
tail -3 gpurun_out/rc_tests.log
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/rc_bench.log 2>&1
tail -1 gpurun_out/rc_bench.log > gpurun_out/rc_bench.json
python - <<'PY'
import json
d = json.load(open("gpurun_out/rc_bench.json"))
print(d["value"], d["ms_per_step"], d["step_ms_trend"], d["e2e"]["value"], d["clocks"], d["gpu_launches"])
print(json.dumps(d["roofline"])[:300])
for k, v in d["sub_results"].items():
    print(k, v["value"], v["ms_per_step"], (v.get("e2e") or {}).get("value"))
print(json.dumps(d["cpu_baseline"])[:200])
PY
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/rc_ref.log 2>&1
tail -1 gpurun_out/rc_ref.log | cut -c1-300
