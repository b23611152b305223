"""One line per kernel from an `ncu --page raw --csv` export: duration, DRAM
bytes, DRAM/SM throughput, occupancy, registers.

    python tools/ncu_raw_summary.py gpurun_out/x_raw.csv
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
want = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rdMB"),
        ("dram__bytes_write.sum", "wrMB"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"), ("launch__registers_per_thread", "regs"),
        ("launch__grid_size", "grid"), ("lts__t_sector_hit_rate.pct", "L2hit%")]
idx = [(hdr.index(k), lab) for k, lab in want if k in hdr]
units = rows[1]
print(" | ".join(f"{lab}" for _, lab in idx))
for r in rows[2:]:
    out = []
    for i, lab in idx:
        v = r[i]
        if lab == "kernel":
            v = v.split("(")[0].replace("void ", "")[:40]
        elif units[i] == "Gbyte":
            v = f"{float(v) * 1000:.1f}"
        elif units[i] == "Kbyte":
            v = f"{float(v) / 1000:.3f}"
        elif units[i] == "ms":
            v = f"{float(v) * 1000:.1f}"
        out.append(v)
    print(" | ".join(out))
