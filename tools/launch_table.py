"""Per-kernel totals of the second half (last step) of an ncu launch-list CSV."""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
ki, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
recs = defaultdict(dict)
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    d = recs[int(r[ii])]
    d["name"] = re.sub(r"\(.*", "", re.sub(r"\(CUtensorMap.*", "", r[ki])).replace("void ", "").replace(
        "(anonymous namespace)::", "").replace("unnamed>::", "")
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        d["us"] = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1)
ids = sorted(recs)
last = ids[len(ids) // 2:] if len(sys.argv) < 3 else ids[int(sys.argv[2]):]
tot, cnt = defaultdict(float), defaultdict(int)
for i in last:
    tot[recs[i]["name"]] += recs[i]["us"]
    cnt[recs[i]["name"]] += 1
allt = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:9.1f} us {100 * v / allt:5.1f}% n={cnt[k]:3d} avg {v / cnt[k]:7.1f} {k[:70]}")
print(f"total {allt:.1f} us")
