"""Per-kernel evidence for bench.py's rooflines from ncu --set full captures.

    python scripts/ncu_bounds.py <config> <n_samples_of_the_profiled_launch> <kernel>=<entry>:<bound> ...

Reads gpurun_out/r2_<config>/<kernel>.ncu-rep, prints and merges into
profiles/kernel_bounds.json: DRAM bytes per sample, the L2 request counts per sample (reads
and REDs from the SM side), the kernel time, and the bound the capture shows."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
cfg, n = sys.argv[1], float(sys.argv[2])
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
for arg in sys.argv[3:]:
    kern, rest = arg.split("=", 1)
    entry, bound = rest.split(":", 1)
    rep = Path(kern) if kern.endswith(".ncu-rep") else ROOT / "gpurun_out" / f"r2_{cfg}" / f"{kern}.ncu-rep"
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    m = {}
    for k, name in keys.items():
        if name in h:
            i = h.index(name)
            m[k] = float(v[i].replace(",", "")) * scale.get(u[i], 1.0)
    t = m["t"]
    ev = {"dram_bytes_per_sample": (m["dr"] + m["dw"]) / n, "bound": bound,
          "ncu_ms": t * 1e3, "lts_pct": m.get("lts"), "dram_pct": m.get("dram_pct"),
          "l1_pct": m.get("l1"), "tensor_pipe_pct": m.get("tc"),
          "l2_read_requests_per_sample": m.get("rq_rd", 0) / n,
          "l2_red_requests_per_sample": m.get("rq_red", 0) / n,
          "l2_requests_per_s": (m.get("rq_rd", 0) + m.get("rq_red", 0) + m.get("rq_wr", 0)) / t,
          "source": f"profiles/r2/{cfg}_{kern}.txt (ncu --set full, one launch, {int(n)} samples)"}
    doc.setdefault(cfg, {})[entry] = ev
    print(cfg, entry, json.dumps(ev))
out_path.write_text(json.dumps(doc, indent=1))
