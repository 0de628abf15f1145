"""Per-source-line warp-stall samples of an ncu report (needs -lineinfo + --import-source)."""
import csv
import io
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
fname = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 5 and r[0] != "Line No" and r[2] == "-":
        try:
            v = int(r[4])
        except ValueError:
            continue
        if v:
            res.append((v, fname, r[0], r[1].strip()))
tot = sum(v for v, *_ in res) or 1
for v, f, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{v / tot * 100:5.1f}% {f}:{ln}  {src[:100]}")
