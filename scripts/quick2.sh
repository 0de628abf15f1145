#!/bin/bash
# quick GPU check: sampler + render parity, then c3 bench
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
timeout 600 python bench.py --no-cpu > gpurun_out/q_bench.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/q_bench.log").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"] if d.get("e2e") else None)
print({k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items()})
PY
