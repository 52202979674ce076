"""Summarise an ncu report: key metrics + top stall sites (SASS, with CUDA line).
Usage: python tools/ncu_summary.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Executed Ipc Active", "Achieved Active Warps Per SM", "Avg. Active Threads Per Warp",
        "Registers Per Thread", "Grid Size", "Issued Instructions", "Warp Cycles Per Issued Instruction",
        "Compute (SM) Throughput", "Branch Efficiency", "Eligible Warps Per Scheduler"]


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "details", "--csv"]))))
    h = rows[0]
    ki, mi, ui, vi = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                      h.index("Metric Value"))
    ii = h.index("ID")
    for r in rows[1:]:
        if r[mi] in KEYS:
            print(f"[{r[ii]}] {r[ki][:30]:30s} {r[mi]:40s} {r[vi]:>14s} {r[ui]}")
    raw = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    hh = raw[0]
    for want in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        if want in hh:
            j = hh.index(want)
            print(want, [r[j] for r in raw[2:]], raw[1][j])
    src = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "source", "--csv",
                                            "--print-source", "sass"]))))
    hs = src[1]
    si, wi = hs.index("Source"), hs.index("Warp Stall Sampling (All Samples)")
    data = [r for r in src[2:] if len(r) > wi and r[wi].isdigit()]
    tot = sum(int(r[wi]) for r in data) or 1
    order = sorted(range(len(data)), key=lambda k: -int(data[k][wi]))[:top]
    for k in order:
        prev = data[k - 1][si].strip() if k else ""
        print(f"{int(data[k][wi]) / tot * 100:5.1f}%  {data[k][si].strip()[:58]:58s} | {prev[:48]}")


if __name__ == "__main__":
    main()
