#!/bin/bash
# A/B of two builds on the bench workloads: bash scripts/ab_bench.sh <old.so> [kernel-substring]
# (VR_LIB_PATH=<old.so> vs the in-tree build; c5 and c4 without sub-results, CPU leg or e2e).
set -u
OLD=$1; PAT=${2:-mlp}
mkdir -p gpurun_out
for c in c5 c4; do for L in "$OLD" paper_2404_16221_b200/libvolray_b200.so; do
  out=gpurun_out/ab_${c}_$(basename "$L").json
  VR_LIB_PATH=$L timeout 600 python bench.py --config $c --sub none --no-cpu --no-e2e 2>/dev/null | tail -1 > "$out"
  python - "$out" "$c" "$(basename "$L")" "$PAT" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print(sys.argv[2], sys.argv[3], round(d["ms_per_step"], 2),
      {k: round(v["ms_per_step"], 3) for k, v in d["kernels"].items() if sys.argv[4] in k})
PY
done; done
