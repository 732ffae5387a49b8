"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name:
    python tools/launch_summary2.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    only = sys.argv[2] if len(sys.argv) > 2 else None  # regex on the kernel name
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ix["Kernel Name"]])[:70]
        if only and not re.search(only, r[ix["Kernel Name"]]):
            continue
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        v *= {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"total {T:.2f} ms over {sum(cnt.values())} launches")
    for k, v in sorted(tot.items(), key=lambda z: -z[1]):
        print(f"{v:10.3f} ms {100 * v / T:5.1f}%  x{cnt[k]:5d}  {k}")


if __name__ == "__main__":
    main()
