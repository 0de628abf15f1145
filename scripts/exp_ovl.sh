#!/bin/bash
set -u
summ() { python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "ms", round(d["ms_per_step"], 2), {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items() if v["ms_per_step"] > 1})
PY
}
for b in 0 296 592; do
VR_SCATTER_BLOCKS=$b timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/ov_$b.log 2>&1; summ gpurun_out/ov_$b.log
done
