"""Modelled strong-scaling efficiency E_P = T_1 / (P T_P) of the 1D
column-block-cyclic schedule from MEASURED one-GPU per-phase
times (a bench.py JSON line) -- NOT a scaling measurement (this run has one
GPU).  Per phase at P ranks:
  sketch, S5 trailing, S6 sample update     / P          (column-local work)
  S2 sample QRCP                             x 1          (replicated on every rank)
  S4 panel QR                                x 1          (the panel's owner)
  S3 swaps                                   x 1 (+ exchanges below)
  exchanges per panel (fixed size): integer-sum reduce of the packed pivot
  columns (m bb 8 B), broadcasts of V (m' bb 8 B) and of the displaced slot
  columns (m bb 8 B), allgather of the updated sample (l_pad n'' 8 B), each at
  BW bytes/s plus LAT s; the initial sample allgather (l_pad n 8 B).
    python tools/scaling_model.py profiles/r02_v3_bench_C5.json [P] [BW_GBs] [LAT_us]
"""
import json
import sys


def model(line, P, bw=700e9, lat=20e-6):
    c = line["config"]
    m, n, k, b, p = c["m"], c["n"], c["k"], c["b"], c["p"]
    lpad = (b + p + 7) // 8 * 8
    ph = line["phases_ms_per_step"]
    t1 = line["ms_per_step"]
    div = (ph["sketch_ms"] + ph["trailing_ms"] + ph["sample_update_ms"]) / P
    rep = ph["sample_qrcp_ms"] + ph["panel_ms"] + ph["swap_ms"] + ph["omega_ms"]
    comm = (lpad * n * 8) / bw + lat
    for i in range(0, k, b):
        bb = min(b, k - i)
        mp, npp = m - i, n - i - bb
        comm += (m * bb * 8 + mp * bb * 8 + m * bb * 8 + lpad * npp * 8) / bw + 4 * lat
    rest = max(0.0, t1 - (ph["sketch_ms"] + ph["trailing_ms"] + ph["sample_update_ms"] + rep))
    tp = div + rep + comm * 1e3 + rest
    return t1, tp, t1 / (P * tp), dict(column_local=div, serial=rep, comm=comm * 1e3, other=rest)


def main():
    line = json.load(open(sys.argv[1]))
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    bw = float(sys.argv[3]) * 1e9 if len(sys.argv) > 3 else 700e9
    lat = float(sys.argv[4]) * 1e-6 if len(sys.argv) > 4 else 20e-6
    for q in sorted({2, 4, P}):
        t1, tp, e, parts = model(line, q, bw, lat)
        print(f"{line['config']['workload']} P={q}: T1 {t1:.1f} ms, T_P {tp:.1f} ms, E_P {e:.2f}  "
              + ", ".join(f"{k} {v:.1f} ms" for k, v in parts.items()))


if __name__ == "__main__":
    main()
