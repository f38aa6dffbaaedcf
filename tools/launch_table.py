"""Per-kernel totals of the second half (last step) of an ncu launch-list CSV:
time, and (when the CSV has them) DRAM read+write bytes and achieved GB/s.

    python tools/launch_table.py launches.csv [first_id]
"""
import csv
import re
import sys
from collections import defaultdict

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}

rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
ki, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
recs = defaultdict(lambda: {"us": 0.0, "bytes": 0.0})
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    d = recs[int(r[ii])]
    d["name"] = re.sub(r"\(.*", "", re.sub(r"\(CUtensorMap.*", "", r[ki])).replace("void ", "").replace(
        "(anonymous namespace)::", "").replace("unnamed>::", "")
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        d["us"] = v * UNIT.get(r[ui], 1)
    elif r[mi].startswith("dram__bytes"):
        d["bytes"] += v * BYTES.get(r[ui], 1)
ids = sorted(recs)
last = ids[len(ids) // 2:] if len(sys.argv) < 3 else ids[int(sys.argv[2]):]
tot, cnt, byt = defaultdict(float), defaultdict(int), defaultdict(float)
for i in last:
    tot[recs[i]["name"]] += recs[i]["us"]
    byt[recs[i]["name"]] += recs[i]["bytes"]
    cnt[recs[i]["name"]] += 1
allt = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    gbs = byt[k] / (v * 1e-6) / 1e9 if v else 0.0
    print(f"{v:9.1f} us {100 * v / allt:5.1f}% n={cnt[k]:3d} avg {v / cnt[k]:7.1f} us "
          f"{byt[k] / cnt[k] / 1e6:8.1f} MB/launch {gbs:7.0f} GB/s  {k[:60]}")
print(f"total {allt:.1f} us")
