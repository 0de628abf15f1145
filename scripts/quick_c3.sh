#!/bin/bash
# c3 bench only (kernel breakdown)
set -u
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/qc3.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/qc3.log").read().strip().splitlines()[-1])
print("ms", round(d["ms_per_step"], 2), {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items() if v["ms_per_step"] > 0.3})
PY
