#!/bin/bash
set -u
summ() { python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "ms", round(d["ms_per_step"], 2), {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items() if v["ms_per_step"] > 1})
PY
}
VR_BENCH_HASH_ORDER=level timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/eo_c3_level.log 2>&1; summ gpurun_out/eo_c3_level.log
VR_BENCH_HASH_ORDER=sample VR_BENCH_MLP_IMPL=tc timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/eo_c3_tc.log 2>&1; summ gpurun_out/eo_c3_tc.log
VR_BENCH_HASH_ORDER=sample timeout 900 python bench.py --config c4 --steps 3 --no-cpu --no-e2e > gpurun_out/eo_c4_sample.log 2>&1; summ gpurun_out/eo_c4_sample.log
