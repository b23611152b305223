"""Summarise an `ncu --page source --csv` export: top instructions by warp
stall samples with their dominant stall reasons.

    python tools/ncu_src_top.py gpurun_out/src_k_find.csv [N]
"""
import csv
import sys

path = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
# first row: kernel name; second: header
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
data = []
for r in rows[hi + 1:]:
    if r and r[0] == "Address":
        break  # the export repeats per launch: keep the first one
    if len(r) == len(hdr):
        data.append(r)
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[si] or 0) for r in data)
tot_by = {hdr[i]: sum(float(r[i] or 0) for r in data) for i in stall_cols}
print(f"total samples {tot:.0f}")
print("by reason:", ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in sorted(tot_by.items(), key=lambda x: -x[1])[:8]))
data.sort(key=lambda r: -float(r[si] or 0))
for r in data[:N]:
    s = float(r[si] or 0)
    reasons = sorted(((hdr[i][6:], float(r[i] or 0)) for i in stall_cols), key=lambda x: -x[1])[:3]
    print(f"{r[0]:>6s} {100*s/tot:5.1f}%  {r[1][:70]:70s} " + " ".join(f"{k}:{v:.0f}" for k, v in reasons))
