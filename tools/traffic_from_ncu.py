"""DRAM bytes per launch of bench.py's roofline candidates from two
`ncu --page raw --csv` exports of tools/prof_c2.py (lambda 0.5 and 1.0):
dram__bytes_read.sum + dram__bytes_write.sum, the bench's lambdas
0.5 / 0.75 / 1.0 averaged as (2 x lambda0.5 + lambda1.0) / 3 (lambda 0.75
inserts are 99.9 % free-slot inserts like lambda 0.5).

    python tools/traffic_from_ncu.py raw_0.5.csv raw_1.0.csv > profiles/traffic.json
"""
import csv
import json
import sys


def per_kernel(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    ki, rd, wr = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = {}
    for r in rows[2:]:
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0].replace("hkv::", "")
        b = float(r[rd]) * scale[units[rd]] + float(r[wr]) * scale[units[wr]]
        out.setdefault(name, []).append(b)
    return {k: sum(v) / len(v) for k, v in out.items()}


a, b = per_kernel(sys.argv[1]), per_kernel(sys.argv[2])
avg = lambda k: (2 * a.get(k, 0) + b.get(k, 0)) / 3
res = {
    "k_meta_tps": int(avg("k_meta_tps")),
    "find:k_find+k_find_gather": int(avg("k_find_fused") + avg("k_find_gather")),
    "k_values_write": int(avg("k_values_write")),
    "_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch from ncu --set full (tools/capture_r02.sh: "
             "tools/prof_c2.py at lambda 0.5 and 1.0, 1M-key batches, 2^27 slots, dim 64); bench lambdas averaged as "
             "(2 x lambda0.5 + lambda1.0)/3",
    "per_lambda": {"0.5": {k: int(v) for k, v in a.items()}, "1.0": {k: int(v) for k, v in b.items()}},
}
print(json.dumps(res, indent=1))
