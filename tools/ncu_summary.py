"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import re
import sys
from collections import defaultdict


def main(path, skip_launches=0):
    rows = list(csv.reader(open(path)))
    hdr = None
    for i, r in enumerate(rows):
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = i
            break
    h = rows[hdr]
    ki, vi, ui, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr + 1:]:
        if len(r) <= vi or int(r[ii]) < skip_launches:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        name = re.sub(r"\(.*", "", r[ki])
        name = re.sub(r"<.*", "", name) if "gemm_tc_kernel" not in name else r[ki][:80]
        tot[name] += ns
        cnt[name] += 1
    all_ns = sum(tot.values())
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v / 1e6:10.3f} ms {100 * v / all_ns:6.2f}%  n={cnt[k]:5d}  {k}")
    print(f"total {all_ns / 1e6:.3f} ms over {sum(cnt.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
