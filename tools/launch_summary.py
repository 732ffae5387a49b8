"""Summarise an ncu launch list (gpu__time_duration.sum CSV) by kernel name:
count, total and share of the step.  Usage: python tools/launch_summary.py launches.csv [--last N]"""
import csv
import re
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = re.sub(r"\(.*", "", name)
        short = re.sub(r"^void ", "", short)
        rows.append((short[:90], float(r["Metric Value"]) / 1e3))
    if "--last" in sys.argv:
        rows = rows[-int(sys.argv[sys.argv.index("--last") + 1]):]
    agg = OrderedDict()
    for n, t in rows:
        c, s = agg.get(n, (0, 0.0))
        agg[n] = (c + 1, s + t)
    tot = sum(t for _, t in rows)
    print(f"{'kernel':92s} {'launches':>8s} {'total_us':>10s} {'share':>7s}")
    for n, (c, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:92s} {c:8d} {s:10.1f} {100 * s / tot:6.1f}%")
    print(f"{'TOTAL':92s} {len(rows):8d} {tot:10.1f}")


if __name__ == "__main__":
    main()
