"""The launches of the last step in an ncu launch list (gpu__time_duration.sum CSV): the last
run of launches from one K1 launch (`k_sample<`) to the next that has at least 20 launches
(the bench's trailing K1-only sampling pass is skipped), as
`Kernel Name,gpu__time_duration.sum (ns)`.
    python scripts/last_step.py <launches_all.csv> > <one_step.csv>"""
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
body = rows[1:]
ks = [i for i, r in enumerate(body) if r[ik].startswith("void vr::k_sample<")] + [len(body)]
start, end = [(a, b) for a, b in zip(ks, ks[1:]) if b - a >= 20][-1]
print("Kernel Name,gpu__time_duration.sum (ns)")
scale = {"ns": 1, "nsecond": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}
for r in body[start:end]:
    print(f'"{r[ik].split("(")[0]}",{int(float(r[iv].replace(",", "")) * scale.get(r[iu], 1))}')
