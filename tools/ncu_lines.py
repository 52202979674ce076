"""Per-CUDA-source-line stall samples of an ncu report (needs -lineinfo).
Usage: python tools/ncu_lines.py report.ncu-rep [top] [kernel-id]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    args += ["--print-kernel-base", "function", "-k", sys.argv[3]]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
wi = hdr.index("Warp Stall Sampling (All Samples)")
lines = [(r[0], r[1], int(r[wi])) for r in rows if r and r[0].isdigit() and r[wi].isdigit()]
tot = sum(x[2] for x in lines) or 1
for ln, src, w in sorted(lines, key=lambda x: -x[2])[:top]:
    print(f"{100 * w / tot:5.1f}%  L{ln:>5s}  {src.strip()[:100]}")

ii = hdr.index("Instructions Executed")
lines2 = [(r[0], r[1], int(r[ii])) for r in rows if r and r[0].isdigit() and r[ii].isdigit()]
tot2 = sum(x[2] for x in lines2) or 1
print("\n# top lines by warp instructions executed")
for ln, src, w in sorted(lines2, key=lambda x: -x[2])[:top]:
    print(f"{100 * w / tot2:5.1f}%  L{ln:>5s}  {src.strip()[:100]}")
