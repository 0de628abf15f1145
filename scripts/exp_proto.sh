#!/bin/bash
set -u
summ() { python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "value", round(d["value"]), "ms", round(d["ms_per_step"], 2), d["exchange"], {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items() if v["ms_per_step"] > 0.5})
PY
}
timeout 600 python bench.py --protocol sample --no-cpu --no-e2e > gpurun_out/pr_c3.log 2>&1; summ gpurun_out/pr_c3.log
timeout 600 python bench.py --config c5 --protocol sample --no-cpu --no-e2e > gpurun_out/pr_c5.log 2>&1; summ gpurun_out/pr_c5.log
