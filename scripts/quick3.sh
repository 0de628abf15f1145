#!/bin/bash
# GPU check: full parity suite, c3 + c4 benches
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
summ() { python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "value", round(d["value"]), "ms", round(d["ms_per_step"], 2), "e2e", round(d["e2e"]["value"]) if d.get("e2e") else None,
      "roof", {k: d["roofline"][k] for k in ("kernel", "achieved", "frac")} if d.get("roofline") else None)
print({k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items() if v["ms_per_step"] > 0.3})
PY
}
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/q3_c3.log 2>&1; summ gpurun_out/q3_c3.log
timeout 900 python bench.py --config c4 --steps 3 --no-cpu --no-e2e > gpurun_out/q3_c4.log 2>&1; summ gpurun_out/q3_c4.log
