"""Aggregate ncu warp-stall samples by CUDA source line (needs -lineinfo).
Usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
wi = h.index("Warp Stall Sampling (All Samples)")
ls = h.index("stall_long_sb") if "stall_long_sb" in h else None
src = {}
agg = {}
cur = None
for r in rows[hi + 1:]:
    if not r:
        continue
    if r[0] and r[0].isdigit():  # a CUDA line row: Line No, Source, then its aggregated metrics
        cur = int(r[0])
        src[cur] = r[1]
        try:
            agg[cur] = (int(r[wi] or 0), int(r[ls] or 0) if ls is not None else 0)
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values()) or 1
for ln, (v, lsb) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * v / tot:5.1f}% (long_sb {100 * lsb / tot:4.1f}%) L{ln:<5d} {src[ln].strip()[:90]}")
