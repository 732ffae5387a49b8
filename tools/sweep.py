"""Grid-size sweep of the latency-bound kernels + per-step phase traces.

    RQRCP_TRACE=1 python tools/sweep.py --config C2 [--sq 16,32,64,148] [--pn 16,32,64,148]

Prints the per-phase times (CUDA events inside the library) of one warm
factorization per setting.  Diagnostic tool; not part of the product path."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--sq", default="")
    ap.add_argument("--pn", default="")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--var", action="append", default=[], help="ENVNAME=v1,v2,... (one run per value)")
    args = ap.parse_args()
    import torch

    import inputs
    import paper_1804_05138_b200 as rq
    c = inputs.CONFIGS[args.config]
    m, n, k, b, p, seed = c["m"], c["n"], c["k"], c["b"], c["p"], c["seed"]
    A0 = inputs.make(c["kind"], m, n, seed, device="cuda")
    A = A0.t().clone().t()
    ctx = rq.RQRCP(max_m=m, max_n=n, max_b=b, max_p=p)

    def run(label):
        best = None
        for _ in range(args.reps):
            A.copy_(A0)
            ctx.factor(A, k, b, p, seed=seed)
            torch.cuda.synchronize()
            t = ctx.timings()
            if best is None or t["total_ms"] < best["total_ms"]:
                best = t
        keys = ["total_ms", "sketch_ms", "sample_qrcp_ms", "swap_ms", "panel_ms", "trailing_ms", "sample_update_ms"]
        print(label, " ".join(f"{kk[:-3]}={best[kk]:.3f}" for kk in keys),
              f"hh_panels={best['panels_householder']}/{best['panels']}", flush=True)

    run("default")
    for s in [x for x in args.sq.split(",") if x]:
        os.environ["RQRCP_SQ_GRID"] = s
        run(f"sq_grid={s}")
    os.environ.pop("RQRCP_SQ_GRID", None)
    for s in [x for x in args.pn.split(",") if x]:
        os.environ["RQRCP_PN_GRID"] = s
        run(f"pn_grid={s}")
    os.environ.pop("RQRCP_PN_GRID", None)
    for spec in args.var:
        name, vals = spec.split("=", 1)
        for v in vals.split(","):
            os.environ[name] = v
            run(f"{name}={v}")
        os.environ.pop(name, None)
    ctx.close()


if __name__ == "__main__":
    main()
