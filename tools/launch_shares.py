"""Per-kernel share of device time from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file launches.csv <cmd>`).

usage: python tools/launch_shares.py launches.csv
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[1:]:
    if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[iu], 1.0)
    name = r[ik].split("(")[0].replace("unnamed>::", "").replace("void ", "")
    tot[name] += v * scale
    cnt[name] += 1
s = sum(tot.values())
print(f"| kernel | launches | total ms (ncu, serialised, cold) | share |\n|---|---|---|---|")
for k, v in tot.most_common():
    print(f"| {k} | {cnt[k]} | {v:.2f} | {v / s:.1%} |")
print(f"| **total** | {sum(cnt.values())} | {s:.2f} | 100% |")
