"""Per-CUDA-line executed warp instructions of an ncu report (needs -lineinfo).
Usage: python tools/ncu_instr_lines.py report.ncu-rep [top]"""
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
ie = h.index("Instructions Executed")
agg, src = {}, {}
for r in rows[hi + 1:]:
    if r and r[0] and r[0].isdigit():
        try:
            agg[int(r[0])] = int(r[ie] or 0)
            src[int(r[0])] = r[1]
        except ValueError:
            pass
tot = sum(agg.values()) or 1
print(f"total warp instructions {tot:,}")
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}% {v:>14,} L{ln:<5d} {src[ln].strip()[:90]}")
