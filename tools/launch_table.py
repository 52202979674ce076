"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list.
Usage: python tools/launch_table.py launches.csv [--seq]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
agg = collections.defaultdict(lambda: [0, 0.0, []])
seq = []
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    us = float(r[vi].replace(",", "")) * scale[r[ui]]
    name = r[ki].split("(")[0].replace("dfs::<unnamed>::", "").replace("void ", "")[-48:]
    agg[name][0] += 1
    agg[name][1] += us
    agg[name][2].append(us)
    seq.append((name, us))
tot = sum(v[1] for v in agg.values())
print(f"{'total':>10s} {tot/1e3:9.3f} ms")
for k, (c, t, xs) in sorted(agg.items(), key=lambda x: -x[1][1]):
    xs = sorted(xs)
    print(f"{t/1e3:9.3f} ms {100*t/tot:5.1f}% n={c:4d} med={xs[len(xs)//2]:9.1f}us max={xs[-1]:9.1f}us  {k}")
if "--seq" in sys.argv:
    for name, us in seq:
        print(f"{us:10.1f} {name}")
