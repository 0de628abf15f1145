#!/bin/bash
# field-backward decomposition: fused / unfused (tc).  (The fused kernel without its
# scatter was measured with a since-removed debug switch: 21.0 ms at c3.)
set -u
mkdir -p gpurun_out
summ() { python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k = d["kernels"]
print(sys.argv[1], "ms", round(d["ms_per_step"], 2), {n: round(v["ms_per_step"], 2) for n, v in k.items() if v["ms_per_step"] > 1})
PY
}
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/e_fused.log 2>&1; summ gpurun_out/e_fused.log
VR_BENCH_MLP_IMPL=tc timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/e_tc.log 2>&1; summ gpurun_out/e_tc.log
