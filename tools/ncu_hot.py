"""Hot SASS instructions of a `ncu --page source --csv` export (per-instruction
rows): top-N by warp-stall samples, with instruction counts.
    ncu -i rep --page source --csv --kernel-name regex:K --launch-count 1 > x.csv
    python tools/ncu_hot.py x.csv [N]"""
import csv
import sys


def main():
    path = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    with open(path) as f:
        lines = f.readlines()
    rows = list(csv.reader(lines[1:]))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    data = []
    tot_s = tot_i = 0
    for r in rows[1:]:
        if len(r) < len(hdr) or r[0] == "Address":
            continue
        try:
            float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ins = float(r[ix["Instructions Executed"]] or 0)
        tot_s += s
        tot_i += ins
        data.append((s, ins, r[ix["Address"]], r[ix["Source"]]))
    print(f"total stall samples {tot_s:.0f}, warp instructions {tot_i:.0f}")
    for s, ins, a, src in sorted(data, key=lambda x: -x[0])[:n]:
        print(f"{s:7.0f} {100 * s / max(tot_s, 1):5.1f}% {ins:8.0f}  {a}  {src[:90]}")


if __name__ == "__main__":
    main()
