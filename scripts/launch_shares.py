"""Share of each kernel in an ncu launch list (gpu__time_duration.sum CSV)."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    c = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        name = r[ik].split("(")[0].replace("void ", "")
        c[name][0] += 1
        c[name][1] += float(r[iv].replace(",", "")) / 1e6
    tot = sum(v[1] for v in c.values())
    print(f"{path}: {sum(v[0] for v in c.values())} launches, {tot:.1f} ms (serialised, cold)")
    for k, v in sorted(c.items(), key=lambda x: -x[1][1])[:16]:
        print(f"  {k:44s} {v[0]:5d} {v[1]:9.2f} ms {100 * v[1] / tot:5.1f} %")
