"""kernel_bounds.json entries from the prof_r2c.sh captures (steady-state c4 / c3 / c5).

Sample counts per captured launch: the dense kernels process a whole region (the region's
samples in plain_<cfg>.json's config... taken from rows_<cfg>.json's n), the sparse
backward kernels the region's active rows (rows_<cfg>.json's count).  Writes
profiles/kernel_bounds.json and prints one line per kernel."""
import csv
import io
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
D = ROOT / "gpurun_out" / "r2c"
out_path = ROOT / "profiles" / "kernel_bounds.json"
doc = json.loads(out_path.read_text()) if out_path.exists() else {}
keys = {"t": "gpu__time_duration.sum", "dr": "dram__bytes_read.sum", "dw": "dram__bytes_write.sum",
        "rq_rd": "lts__t_requests_srcunit_tex_op_read.sum",
        "rq_red": "lts__t_requests_srcunit_tex_op_red.sum",
        "rq_wr": "lts__t_requests_srcunit_tex_op_write.sum",
        "lts": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "tc": "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "l1": "l1tex__throughput.avg.pct_of_peak_sustained_active"}
scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "request": 1, "%": 1, "": 1,
         "Krequest": 1e3, "Mrequest": 1e6, "Grequest": 1e9}


def metrics(name):
    """The --page raw CSV prof_r2c.sh exported on the box (the reports are not kept)."""
    raw = (D / "raw" / f"{name}.csv").read_text()
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    m = {}
    for k, name in keys.items():
        if name in h:
            i = h.index(name)
            m[k] = float(v[i].replace(",", "")) * scale.get(u[i], 1.0)
    return m


def rows_of(cfg):
    p = D / f"rows_{cfg}.json"
    return json.loads(p.read_text()) if p.exists() else None


# name -> (config, C-ABI entry point, which count, bound text)
#   count: ("n", field) = the region's samples, ("rows", field) = its active rows
SPEC = {
    "c4_k_hash_fwd_lm_nerf": ("c4", "vr_hash_fwd_lm", ("n", "nerf"), None),
    "c4_k_hash_bwd_lm_nerf": ("c4", "vr_hash_scatter", ("rows", "nerf"), None),
    "c4_k_mlp_bwd_tc_nerf": ("c4", "vr_mlp_bwd_tc", ("rows", "nerf"), None),
    "c4_k_mlp_bwd_tc_prop": ("c4", "vr_mlp_bwd_tc_density", ("rows", "proposal"), None),
    "c4_k_mlp_fwd_tc": ("c4", "vr_mlp_fwd_tc", ("n", "nerf"), None),
    "c4_k_segment_fwd_ls": ("c4", "vr_segment_fwd", ("all", None), None),
    "c4_k_segment_bwd_ls": ("c4", "vr_segment_bwd", ("all", None), None),
    "c3_k_mlp_bwd_tc": ("c3", "vr_field_bwd_tc", ("rows", "nerf"), None),
    "c3_k_hash_fwd": ("c3", "vr_hash_fwd", ("n", "nerf"), None),
    "c5_k_hash_fwd_lm": ("c5", "vr_hash_fwd_lm", ("plain", None), None),
    "c5_k_mlp_fwd_tc": ("c5", "vr_mlp_fwd_tc", ("plain", None), None),
}
bounds = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
for name, (cfg, entry, (what, field), _) in SPEC.items():
    if not (D / "raw" / f"{name}.csv").exists():
        print("missing", name)
        continue
    rc = rows_of(cfg)
    if what in ("n", "rows"):
        cnt, n = rc[field][0]
        units = cnt if what == "rows" else n
    elif what == "all":
        units = sum(n for _, n in rc["nerf"])
    else:  # render: region 0's samples from the plain run (samples per step / regions)
        pj = json.loads((D / f"plain_{cfg}.json").read_text().strip().splitlines()[-1])
        units = pj["config"]["samples_per_step"] / pj["config"]["regions"]
    m = metrics(name)
    t = m["t"]
    ev = {"dram_bytes_per_sample": (m["dr"] + m["dw"]) / units,
          "bound": bounds.get(name, "see summary"), "ncu_ms": t * 1e3,
          "lts_pct": m.get("lts"), "dram_pct": m.get("dram_pct"), "l1_pct": m.get("l1"),
          "tensor_pipe_pct": m.get("tc"),
          "l2_read_requests_per_sample": m.get("rq_rd", 0) / units,
          "l2_red_requests_per_sample": m.get("rq_red", 0) / units,
          "l2_requests_per_s": (m.get("rq_rd", 0) + m.get("rq_red", 0) + m.get("rq_wr", 0)) / t,
          "samples": int(units),
          "source": f"profiles/r2/steady/{name}.txt (ncu --set full, one launch at the bench's steady "
                    f"state, {int(units)} {'active rows' if what == 'rows' else 'samples'})"}
    doc.setdefault(cfg, {})[entry] = ev
    print(name, entry, json.dumps({k: (round(v, 3) if isinstance(v, float) else v)
                                   for k, v in ev.items() if k != "source"}))
out_path.write_text(json.dumps(doc, indent=1))
