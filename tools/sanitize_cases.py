"""Small factorizations covering every launch path, for compute-sanitizer
(memcheck / racecheck / synccheck): the cluster and register-grid sample
QRCPs, the cluster and grid panel kernels, the three schedules, Eq. (5), the
CholeskyQR2 panel, and a 2-rank loopback group.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [--quick]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    import inputs
    import paper_1804_05138_b200 as rq
    quick = "--quick" in sys.argv
    cases = [
        ("C1", "svd_exp", 512, 512, 64, 32, 8, {}),
        ("cluster74", "iid", 1500, 1200, 192, 64, 10, {}),
        ("reg74", "iid", 700, 4700, 128, 64, 10, {}),
        ("reg144_gridpanel", "graded", 1500, 900, 256, 128, 16, {}),
        ("sched0", "iid", 900, 800, 128, 64, 10, {"schedule": 0}),
        ("sched2", "iid", 900, 800, 128, 64, 10, {"schedule": 2}),
        ("gridsq", "iid", 600, 500, 64, 32, 8, {"sq_cluster": 0, "sq_reg": 0}),
        ("cqr", "graded", 900, 700, 128, 64, 10, {"panel": 1}),
    ]
    if quick:
        cases = cases[:3]
    for name, kind, m, n, k, b, p, opts in cases:
        A = inputs.make(kind, m, n, 3, rank=64, device="cuda")
        ctx = rq.RQRCP(max_m=m, max_n=n, max_b=b, max_p=p)
        for kk, v in opts.items():
            ctx.set_option(kk, v)
        jp, tau, rank = ctx.factor(A, k, b, p, seed=5)
        torch.cuda.synchronize()
        ctx.close()
        print(name, "rank", rank, flush=True)
    if not quick:
        ctx = rq.RQRCP(max_m=700, max_n=600, max_b=64, max_p=10)
        ctx.set_update_rule(2)
        A = inputs.make("iid", 700, 600, 4, device="cuda")
        ctx.factor(A, 128, 64, 10, seed=1)
        torch.cuda.synchronize()
        ctx.close()
        print("eq5 ok", flush=True)
        g = rq.LoopbackGroup(2, max_m=600, max_n=500, max_b=32, max_p=8)
        A = inputs.make("iid", 600, 500, 6).numpy()
        cols = [rq.shard_columns(500, 32, 2, r) for r in range(2)]
        shards = [inputs.fortran(torch.as_tensor(np.asarray(A[:, c]))).cuda() for c in cols]
        jp, ta, rk, codes = g.factor(shards, 500, 96, 32, 8, seed=2)
        g.close()
        print("loopback P=2 codes", codes, flush=True)


if __name__ == "__main__":
    main()
