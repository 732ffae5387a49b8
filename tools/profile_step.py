"""One warm factorization of a config, for ncu / compute-sanitizer runs.

    python tools/profile_step.py [--config C2] [--reps 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--warm", type=int, default=1)
    args = ap.parse_args()
    import torch

    import inputs
    import paper_1804_05138_b200 as rq
    c = inputs.CONFIGS[args.config]
    m, n, k, b, p, seed = c["m"], c["n"], c["k"], c["b"], c["p"], c["seed"]
    A0 = inputs.make(c["kind"], m, n, seed, device="cuda")
    A = A0.t().clone().t()
    ctx = rq.RQRCP(max_m=m, max_n=n, max_b=b, max_p=p)
    for _ in range(args.warm + args.reps):
        A.copy_(A0)
        jpvt, tau, rank = ctx.factor(A, k, b, p, seed=seed)
    torch.cuda.synchronize()
    print("rank", rank, ctx.timings())
    ctx.close()


if __name__ == "__main__":
    main()
