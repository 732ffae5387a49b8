"""The multi-GPU driver (1D column-block-cyclic layout) run
on ONE B200 through the in-process loopback transport
(rqrcp_create_loopback_group): P contexts, one host thread each, the same
collectives as NCCL (pivot-column integer-sum reduce to the panel owner,
owner broadcasts of V / tau / R11 / state and of the displaced slot columns,
sample allgathers) as host rendezvous + device copies -- no kernel waits on
another rank's kernel.

(i) Bitwise P-invariance (SURVEY.md §8(c)(v), §8(e) "Determinism across P"):
jpvt, tau and every entry of the factored matrix for P = 2, 3 equal the P = 1
run bit for bit, for each schedule; (ii) parity of the P-rank result with the
CPU oracle (test_gpu_parity.compare)."""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu

CASES = [
    # name, kind, m, n, k, b, p, seed
    ("ragged", "iid", 700, 523, 100, 32, 8, 11),
    ("tall", "svd_poly", 1500, 700, 200, 64, 10, 12),
    ("b128", "graded", 900, 1100, 256, 128, 16, 17),
    ("odd", "iid", 333, 301, 77, 13, 3, 18),
    ("lowrank", "lowrank", 1024, 1024, 160, 64, 10, 14),
]


def run_group(A, k, b, p, seed, P, opts=None):
    import paper_1804_05138_b200 as rq
    m, n = A.shape
    g = rq.LoopbackGroup(P, max_m=m, max_n=n, max_b=max(b, 8), max_p=max(p, 1))
    try:
        for kk, v in (opts or {}).items():
            g.set_option(kk, v)
        cols = [rq.shard_columns(n, b, P, r) for r in range(P)]
        shards = [inputs.fortran(torch.as_tensor(np.asarray(A[:, c]))).cuda() for c in cols]
        jp, ta, rk, codes = g.factor(shards, n, k, b, p, seed=seed)
        assert all(c in (0, rq.RQRCP_W_RANK_DEFICIENT) for c in codes), (codes, [g.last_error(r) for r in range(P)])
        F = np.zeros((m, n))
        for r in range(P):
            F[:, cols[r]] = shards[r].cpu().numpy()
        jps = [j.cpu().numpy() for j in jp]
        tas = [t.cpu().numpy() for t in ta]
        for r in range(1, P):
            assert np.array_equal(jps[r], jps[0]) and np.array_equal(tas[r], tas[0]) and rk[r] == rk[0]
        return dict(A=F, jpvt=jps[0], tau=tas[0], rank=rk[0])
    finally:
        g.close()


def run_single(A, k, b, p, seed, opts=None):
    import paper_1804_05138_b200 as rq
    m, n = A.shape
    ctx = rq.RQRCP(max_m=m, max_n=n, max_b=max(b, 8), max_p=max(p, 1))
    try:
        for kk, v in (opts or {}).items():
            ctx.set_option(kk, v)
        Ad = inputs.fortran(torch.as_tensor(np.asarray(A))).cuda()
        jpvt, tau, rank = ctx.factor(Ad, k, b, p, seed=seed)
        torch.cuda.synchronize()
        return dict(A=Ad.cpu().numpy(), jpvt=jpvt.cpu().numpy(), tau=tau.cpu().numpy(), rank=rank)
    finally:
        ctx.close()


def assert_bitwise(g, s):
    assert g["rank"] == s["rank"]
    assert np.array_equal(g["jpvt"], s["jpvt"])
    assert np.array_equal(g["tau"], s["tau"])
    assert np.array_equal(g["A"], s["A"])


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", CASES, ids=[c[0] for c in CASES])
def test_p_invariance_bitwise(P, name, kind, m, n, k, b, p, seed):
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    s = run_single(A, k, b, p, seed)
    g = run_group(A, k, b, p, seed, P)
    assert_bitwise(g, s)


@pytest.mark.parametrize("schedule", [0, 1, 2])
def test_p_invariance_schedules(schedule):
    A = inputs.make("iid", 800, 900, 31).numpy()
    s = run_single(A, 192, 64, 10, 31, opts=dict(schedule=schedule))
    g = run_group(A, 192, 64, 10, 31, 2, opts=dict(schedule=schedule))
    assert_bitwise(g, s)


def test_multirank_oracle_parity():
    from test_gpu_parity import compare
    A = inputs.make("graded", 900, 1100, 17).numpy()
    o = oracle.rqrcp(A, 256, 128, 16, seed=17)
    g = run_group(A, 256, 128, 16, 17, 4)
    compare(A, g, o, 256)


def test_multirank_rank_deficient():
    """The sample-norm stop and the R11-diagonal state travel with the panel
    broadcast: every rank stops at the same rank."""
    rng = np.random.default_rng(42)
    A = rng.standard_normal((120, 25)) @ rng.standard_normal((25, 100))
    o = oracle.rqrcp(A, 60, 16, 8, seed=1)
    g = run_group(A, 60, 16, 8, 1, 2)
    assert g["rank"] == o["rank"] == 25
    assert np.array_equal(g["jpvt"], o["jpvt"])


def test_p_invariance_tournament():
    """Tournament pivoting (replicated over the ranks' copies of the sample)
    keeps the bitwise P-invariance."""
    A = inputs.make("graded", 900, 1100, 17).numpy()
    s = run_single(A, 256, 64, 10, 17, opts=dict(tournament=4))
    g = run_group(A, 256, 64, 10, 17, 2, opts=dict(tournament=4))
    assert_bitwise(g, s)
