"""Aggregate an `ncu -i X.ncu-rep --page source --print-source cuda,sass --csv`
export by CUDA source line: warp-stall samples and warp instructions.

    ncu -i rep --page source --print-source cuda,sass --csv > x.csv
    python tools/ncu_cuda_lines.py x.csv [N]
"""
import collections
import csv
import sys

N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_file = "?"
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
tot_s = tot_i = 0.0
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        ins = float(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    key = (cur_file, r[0])
    a = agg[key]
    a[0] += s
    a[1] += ins
    a[2] = r[1][:80]
    tot_s += s
    tot_i += ins
print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.0f}")
for (f, ln), (s, ins, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:N]:
    print(f"{f}:{ln:>5s} samp {100*s/max(tot_s,1):5.1f}% inst {100*ins/max(tot_i,1):5.1f}%  {src.strip()}")
