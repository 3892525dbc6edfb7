"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of
`ncu --set full` captures -> profiles/<round>/traffic.json, keyed by the
kernel names bench.py's per-kernel profile uses.

usage: python tools/ncu_traffic.py out.json name=report.ncu-rep [...]
"""
import csv
import io
import json
import subprocess
import sys


def dram_bytes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        tot += float(vals[i].replace(",", "")) * scale[units[i]]
    t = hdr.index("gpu__time_duration.sum")
    return tot, float(vals[t].replace(",", "")), units[t]


res = {}
for arg in sys.argv[2:]:
    name, rep = arg.split("=", 1)
    b, t, tu = dram_bytes(rep)
    res[name] = {"dram_bytes_per_launch": b, "ncu_time": t, "ncu_time_unit": tu, "report": rep.rsplit("/", 1)[-1]}
json.dump(res, open(sys.argv[1], "w"), indent=1)
print(json.dumps(res, indent=1))
