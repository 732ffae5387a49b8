"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Acceptance (BASELINE.json north_star): identical pivot sequences; |diag R|
within 1e-10 relative; ||A Pi - Q1 [R11 R12]||_F/||A||_F (and ||R22||_F/||A||_F)
within 1e-12 of the oracle's.  Inputs are seeded synthetic matrices from
inputs/ with the recipes of BASELINE.json's configs, at sizes the oracle
finishes in seconds (several GEMM / sample-QRCP / panel tiles and ragged tails).
"""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu

DIAG_RTOL = 1e-10
RES_ATOL = 1e-12


@pytest.fixture(scope="module")
def ctx():
    """Default context: grid-wide (cooperative) sample-QRCP / panel kernels."""
    import paper_1804_05138_b200 as rq
    c = rq.RQRCP(max_m=5000, max_n=5000, max_b=128, max_p=32)
    yield c
    c.close()


def to_dev(A):
    return inputs.fortran(torch.as_tensor(np.asarray(A))).cuda()


def gpu_factor(ctx, A, k, b, p, seed, **kw):
    Ad = to_dev(A)
    jpvt, tau, rank = ctx.factor(Ad, k, b, p, seed=seed, **kw)
    torch.cuda.synchronize()
    return dict(A=Ad.cpu().numpy(), jpvt=jpvt.cpu().numpy(), tau=tau.cpu().numpy(), rank=rank)


def full_R(F, k):
    R = F.copy()
    for j in range(k):
        R[j + 1:, j] = 0.0
    return R


def trunc_residual(A, res, k, probes=None):
    """||A Pi - Q1 [R11 R12]||_F / ||A||_F (exact when probes is None)."""
    Api = A[:, res["jpvt"]]
    Rt = np.triu(res["A"][:k, :])
    Rfull = np.zeros_like(res["A"])
    Rfull[:k] = Rt
    if probes is None:
        return np.linalg.norm(Api - oracle.apply_q(res["A"], res["tau"][:k], Rfull)) / np.linalg.norm(A)
    X = probes
    return (np.linalg.norm(Api @ X - oracle.apply_q(res["A"], res["tau"][:k], Rfull @ X))
            / np.linalg.norm(A @ X))


def compare(A, g, o, k, probes=None):
    assert g["rank"] == o["rank"] == k
    # identical pivot sequences (the whole permutation: same transpositions)
    if not np.array_equal(g["jpvt"], o["jpvt"]):
        bad = int(np.nonzero(g["jpvt"] != o["jpvt"])[0][0])
        pytest.fail(f"pivots differ first at {bad}; oracle gap there {o['gaps'][min(bad, k - 1)]:.3e}")
    dg = np.abs(np.diag(g["A"])[:k])
    do = np.abs(np.diag(o["A"])[:k])
    assert np.max(np.abs(dg - do) / do) <= DIAG_RTOL
    nA = np.linalg.norm(A)
    r22g = np.linalg.norm(full_R(g["A"], k)[k:, k:]) / nA
    r22o = np.linalg.norm(full_R(o["A"], k)[k:, k:]) / nA
    assert abs(r22g - r22o) <= RES_ATOL
    rg = trunc_residual(A, g, k, probes)
    ro = trunc_residual(A, o, k, probes)
    assert abs(rg - ro) <= RES_ATOL
    return rg


CASES = [
    # name, kind, m, n, k, b, p, seed
    ("C1", "svd_exp", 512, 512, 64, 32, 8, 1001),
    ("ragged", "iid", 700, 523, 100, 32, 8, 11),
    ("tall", "svd_poly", 1500, 700, 200, 64, 10, 12),
    ("wide", "graded", 600, 1900, 130, 32, 5, 13),
    ("lowrank", "lowrank", 1024, 1024, 160, 64, 10, 14),
    ("b1p0", "iid", 40, 30, 5, 1, 0, 15),
    ("kfull", "iid", 256, 256, 256, 32, 8, 16),
    ("b128", "graded", 900, 1100, 256, 128, 16, 17),
    ("odd", "iid", 333, 301, 77, 13, 3, 18),
]


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", CASES, ids=[c[0] for c in CASES])
def test_factor_parity(ctx, name, kind, m, n, k, b, p, seed):
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    g = gpu_factor(ctx, A, k, b, p, seed)
    compare(A, g, o, k)


def test_C2_full_size(ctx):
    """configs[1] (the bench workload) at its full size: 4096^2, k=512, b=64, p=10."""
    c = inputs.CONFIGS["C2"]
    A = inputs.config_matrix("C2").numpy()
    o = oracle.rqrcp(A, c["k"], c["b"], c["p"], seed=c["seed"])
    g = gpu_factor(ctx, A, c["k"], c["b"], c["p"], c["seed"])
    X = np.random.default_rng(0).standard_normal((c["n"], 8))
    compare(A, g, o, c["k"], probes=X)


def test_philox_words_bitwise(ctx):
    rng = np.random.default_rng(1)
    ctr = rng.integers(0, 2 ** 32, size=(257, 4), dtype=np.uint64)
    key = (0x12345678, 0x9ABCDEF0)
    got = ctx.philox_words(torch.tensor(ctr.astype(np.int64)).cuda(), key).cpu().numpy()
    for i in range(ctr.shape[0]):
        assert tuple(int(x) for x in got[i]) == oracle.philox4x32_10(ctr[i], key)


def test_omega_normals(ctx):
    """Device Philox + Box-Muller vs the oracle's: a few ulp (libm differences)."""
    out = inputs.fortran(torch.empty(37, 61, dtype=torch.float64)).cuda()
    ctx.fill_gaussian(out, 4242, 0, row0=3, col0=100)
    ref = oracle.normal(4242, 0, 37, 61, row0=3, col0=100)
    got = out.cpu().numpy()
    assert np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3)) < 16 * np.finfo(float).eps


def test_omega_out_matches_oracle(ctx):
    A = inputs.iid(5, 300, 200).numpy()
    om = torch.empty(40 * 300, dtype=torch.float64, device="cuda")
    gpu_factor(ctx, A, 40, 32, 8, 77, omega_out=om)
    got = om.cpu().numpy().reshape(300, 40).T
    ref = oracle.omega(77, 40, 300)
    assert np.max(np.abs(got - ref)) < 1e-14


def test_omega_in(ctx):
    """Injected Omega (testing hook) = the oracle's explicit-Omega mode."""
    A = inputs.iid(6, 400, 350).numpy()
    om = np.random.default_rng(3).standard_normal((24, 400))
    o = oracle.rqrcp(A, 60, 16, 8, omega=om)
    g = gpu_factor(ctx, A, 60, 16, 8, 0, omega=torch.tensor(om.ravel(order="F")).cuda())
    compare(A, g, o, 60)


def test_deterministic(ctx):
    A = inputs.iid(7, 800, 700).numpy()
    g1 = gpu_factor(ctx, A, 128, 64, 10, 3)
    g2 = gpu_factor(ctx, A, 128, 64, 10, 3)
    assert np.array_equal(g1["A"], g2["A"]) and np.array_equal(g1["jpvt"], g2["jpvt"])


def test_rank_deficient(ctx):
    rng = np.random.default_rng(42)
    A = rng.standard_normal((120, 25)) @ rng.standard_normal((25, 100))
    o = oracle.rqrcp(A, 60, 16, 8, seed=1)
    g = gpu_factor(ctx, A, 60, 16, 8, 1)
    assert g["rank"] == o["rank"] == 25
    assert np.array_equal(g["jpvt"], o["jpvt"])
    assert np.all(g["tau"][25:] == 0.0)


def test_zero_matrix(ctx):
    g = gpu_factor(ctx, np.zeros((50, 40)), 10, 4, 2, 1)
    assert g["rank"] == 0 and np.array_equal(g["jpvt"], np.arange(40))


def test_nonfinite(ctx):
    import paper_1804_05138_b200 as rq
    A = np.ones((64, 48))
    A[5, 7] = np.nan
    with pytest.raises(rq.RqrcpError) as e:
        gpu_factor(ctx, A, 8, 4, 2, 1)
    assert e.value.code == rq.RQRCP_E_NONFINITE


def test_argument_errors(ctx):
    import ctypes

    import paper_1804_05138_b200 as rq
    L = rq.lib()
    A = torch.zeros(10, 8, dtype=torch.float64, device="cuda").t().contiguous().t()
    jp = torch.zeros(8, dtype=torch.int64, device="cuda")
    ta = torch.zeros(8, dtype=torch.float64, device="cuda")
    r = ctypes.c_int64()
    h = ctx._h
    call = lambda *a: L.rqrcp_factor(*a)
    assert call(None, A.data_ptr(), 10, 10, 8, 4, 2, 2, 0, jp.data_ptr(), ta.data_ptr(), ctypes.byref(r)) == -1
    assert call(h, None, 10, 10, 8, 4, 2, 2, 0, jp.data_ptr(), ta.data_ptr(), ctypes.byref(r)) == -2
    assert call(h, A.data_ptr(), 9, 10, 8, 4, 2, 2, 0, jp.data_ptr(), ta.data_ptr(), ctypes.byref(r)) == -3
    assert call(h, A.data_ptr(), 10, 0, 8, 4, 2, 2, 0, jp.data_ptr(), ta.data_ptr(), ctypes.byref(r)) == -4
    assert call(h, A.data_ptr(), 10, 10, 0, 4, 2, 2, 0, jp.data_ptr(), ta.data_ptr(), ctypes.byref(r)) == -5
    assert call(h, A.data_ptr(), 10, 10, 8, 9, 2, 2, 0, jp.data_ptr(), ta.data_ptr(), ctypes.byref(r)) == -6
    assert call(h, A.data_ptr(), 10, 10, 8, 4, 0, 2, 0, jp.data_ptr(), ta.data_ptr(), ctypes.byref(r)) == -7
    assert call(h, A.data_ptr(), 10, 10, 8, 4, 4, 7, 0, jp.data_ptr(), ta.data_ptr(), ctypes.byref(r)) == -8
    assert call(h, A.data_ptr(), 10, 10, 8, 4, 2, 2, 0, None, ta.data_ptr(), ctypes.byref(r)) == -10
    assert call(h, A.data_ptr(), 10, 10, 8, 4, 2, 2, 0, jp.data_ptr(), None, ctypes.byref(r)) == -11
    assert call(h, A.data_ptr(), 10, 10, 8, 4, 2, 2, 0, jp.data_ptr(), ta.data_ptr(), None) == -12
    big = L.rqrcp_factor(h, A.data_ptr(), 6000, 6000, 8, 4, 2, 2, 0, jp.data_ptr(), ta.data_ptr(), ctypes.byref(r))
    assert big == rq.RQRCP_E_WORKSPACE


def test_factor_host_equals_device(ctx):
    A = inputs.iid(8, 640, 512).numpy()
    g = gpu_factor(ctx, A, 96, 32, 8, 5)
    Ah = inputs.fortran(torch.as_tensor(A)).pin_memory()
    jp, ta, rank = ctx.factor_host(Ah, 96, 32, 8, seed=5)
    assert rank == 96
    assert np.array_equal(Ah.numpy(), g["A"])
    assert np.array_equal(jp.numpy(), g["jpvt"])


# ---- launch-shape variants of the sample QRCP (threads per column, spill) ----
# RQRCP_SQ_GRID caps the cooperative grid (fewer CTAs -> more columns per CTA,
# fewer threads per column) and RQRCP_SQ_NSM caps the columns a CTA keeps in
# shared memory (the rest go through the transposed L2 spill buffer).
SQ_VARIANTS = [("148", None), ("2", "0"), ("7", "5"), ("33", None), ("1", "40")]
SQ_CASES = [c for c in CASES if c[0] in ("ragged", "odd", "b128", "b1p0", "lowrank")]


@pytest.mark.parametrize("grid,nsm", SQ_VARIANTS, ids=[f"g{g}-nsm{n}" for g, n in SQ_VARIANTS])
@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", SQ_CASES, ids=[c[0] for c in SQ_CASES])
def test_sample_qrcp_launch_variants(ctx, grid, nsm, name, kind, m, n, k, b, p, seed):
    import os
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    os.environ["RQRCP_SQ_GRID"] = grid
    os.environ["RQRCP_SQ_CLUSTER"] = "0"
    os.environ["RQRCP_SQ_REG"] = "0"
    if nsm is not None:
        os.environ["RQRCP_SQ_NSM"] = nsm
    try:
        g = gpu_factor(ctx, A, k, b, p, seed)
    finally:
        for v in ("RQRCP_SQ_GRID", "RQRCP_SQ_NSM", "RQRCP_SQ_CLUSTER", "RQRCP_SQ_REG"):
            os.environ.pop(v, None)
    compare(A, g, o, k)


# ---- the register-resident grid sample QRCP (sample_qrcp_reg.cuh) ----------
# RQRCP_SQ_CLUSTER=0 takes the one-cluster kernel out, so every sample with
# l in {40, 74, 144} runs on the grid of 1 + ceil(n'/256) CTAs; the wide cases
# span several column CTAs with a ragged last one.
REG_CASES = [c for c in CASES if c[0] in ("C1", "ragged", "tall", "lowrank", "kfull", "b128")] + [
    ("reg_wide74", "iid", 800, 1900, 192, 64, 10, 21),
    ("reg_wide144", "graded", 900, 2100, 256, 128, 16, 22),
    ("reg_lowrank144", "lowrank", 700, 1300, 300, 128, 16, 23),
]


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", REG_CASES, ids=[c[0] for c in REG_CASES])
def test_sample_qrcp_register_grid(ctx, name, kind, m, n, k, b, p, seed):
    import os
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    os.environ["RQRCP_SQ_CLUSTER"] = "0"
    try:
        g = gpu_factor(ctx, A, k, b, p, seed)
    finally:
        os.environ.pop("RQRCP_SQ_CLUSTER", None)
    compare(A, g, o, k)


# ---- panel kernels: the register-resident cluster kernel (panel_cl.cuh) is the
# default when bb <= 64 and m' fits one cluster (256 rows per CTA at bb <= 64,
# 512 at bb <= 32, <= 16 CTAs); RQRCP_PN_CLUSTER=0 forces the cooperative grid
# kernel (panel.cuh) everywhere.  Both are checked against the oracle.
PN_CASES = [c for c in CASES if c[0] in ("C1", "ragged", "tall", "wide", "odd", "kfull", "b1p0")] + [
    ("pncl_tall32", "iid", 5000, 300, 96, 32, 8, 24),   # 10 CTAs of 512 rows, ragged last
    ("pncl_4096", "lowrank", 4096, 700, 192, 64, 10, 25),  # 16 CTAs of 256 rows
]


@pytest.mark.parametrize("variant", ["cluster2", "cluster1", "grid"])
@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", PN_CASES, ids=[c[0] for c in PN_CASES])
def test_panel_kernels(ctx, variant, name, kind, m, n, k, b, p, seed):
    """cluster2: two columns x 32 rows per thread (bb in (32, 64]); cluster1: one
    column x 64 rows per thread; grid: the cooperative grid kernel."""
    import os
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    os.environ["RQRCP_PN_CLUSTER"] = "0" if variant == "grid" else "1"
    os.environ["RQRCP_PN_CPT"] = "1" if variant == "cluster1" else "2"
    try:
        g = gpu_factor(ctx, A, k, b, p, seed)
    finally:
        os.environ.pop("RQRCP_PN_CLUSTER", None)
        os.environ.pop("RQRCP_PN_CPT", None)
    compare(A, g, o, k)


# ---- the bulk trailing update overlapped with the next sample QRCP (default
# when that runs on one cluster, P = 1, Eq. (4)) vs the serial schedule.
OVL_CASES = [c for c in CASES if c[0] in ("C1", "ragged", "tall", "lowrank", "kfull")] + [
    # n' > 4096: the next sample QRCP runs on the register grid, the bulk update
    # with dynamically claimed tiles beside it
    ("ovl_grid74", "iid", 700, 4700, 192, 64, 10, 28),
]


@pytest.mark.parametrize("overlap", ["1", "0"])
@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", OVL_CASES, ids=[c[0] for c in OVL_CASES])
def test_overlap_schedule(ctx, overlap, name, kind, m, n, k, b, p, seed):
    import os
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    os.environ["RQRCP_OVERLAP"] = overlap
    try:
        g = gpu_factor(ctx, A, k, b, p, seed)
    finally:
        os.environ.pop("RQRCP_OVERLAP", None)
    compare(A, g, o, k)


def test_overlap_grid_bitwise_equal_serial(ctx):
    """The dynamically scheduled bulk update (grid sample QRCP) gives the same bits."""
    import os
    A = inputs.make("graded", 800, 4800, 29).numpy()
    outs = []
    for ov in ("1", "0"):
        os.environ["RQRCP_OVERLAP"] = ov
        try:
            outs.append(gpu_factor(ctx, A, 256, 64, 10, 29))
        finally:
            os.environ.pop("RQRCP_OVERLAP", None)
    assert np.array_equal(outs[0]["jpvt"], outs[1]["jpvt"])
    assert np.array_equal(outs[0]["A"], outs[1]["A"])


def test_overlap_bitwise_equal_serial(ctx):
    """Overlapping changes the schedule, not the arithmetic: bitwise equal outputs."""
    import os
    c = inputs.CONFIGS["C2"]
    A = inputs.config_matrix("C2").numpy()
    outs = []
    for ov in ("1", "0"):
        os.environ["RQRCP_OVERLAP"] = ov
        try:
            outs.append(gpu_factor(ctx, A, c["k"], c["b"], c["p"], c["seed"]))
        finally:
            os.environ.pop("RQRCP_OVERLAP", None)
    assert np.array_equal(outs[0]["jpvt"], outs[1]["jpvt"])
    assert np.array_equal(outs[0]["tau"], outs[1]["tau"])
    assert np.array_equal(outs[0]["A"], outs[1]["A"])


# ---- updating formula 2 (Eq. (5)) on the GPU: SURVEY.md §8(f) N2 ----
EQ5_CASES = [c for c in CASES if c[0] in ("C1", "ragged", "tall", "lowrank", "b128", "odd")]


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", EQ5_CASES, ids=[c[0] for c in EQ5_CASES])
def test_eq5_update_parity(ctx, name, kind, m, n, k, b, p, seed):
    """GPU Eq. (5) vs the oracle's Eq. (5) mode: identical pivots, |diag R| and
    residuals within the acceptance tolerances."""
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed, update_rule=2)
    ctx.set_update_rule(2)
    try:
        g = gpu_factor(ctx, A, k, b, p, seed)
    finally:
        ctx.set_update_rule(1)
    compare(A, g, o, k)


def test_eq4_eq5_identical_permutations_gpu(ctx):
    """the two updating formulas give the same permutation (C2 shape
    scaled down, iid: the pivot-choice stress case)."""
    A = inputs.iid(31, 1024, 1024).numpy()
    g4 = gpu_factor(ctx, A, 256, 64, 10, 31)
    ctx.set_update_rule(2)
    try:
        g5 = gpu_factor(ctx, A, 256, 64, 10, 31)
    finally:
        ctx.set_update_rule(1)
    assert np.array_equal(g4["jpvt"], g5["jpvt"])
    d4 = np.abs(np.diag(g4["A"])[:256])
    d5 = np.abs(np.diag(g5["A"])[:256])
    assert np.max(np.abs(d4 - d5) / d4) <= DIAG_RTOL


# ---- SRQR verification (Alg. 3 first half): SURVEY.md §8(f) N1 ----
SRQR_CASES = [
    ("C1", "svd_exp", 512, 512, 64, 32, 8, 1001),
    ("ragged", "iid", 700, 523, 100, 32, 8, 11),
    ("lowrank", "lowrank", 1024, 1024, 160, 64, 10, 14),
    ("b128", "graded", 900, 1100, 256, 128, 16, 17),
]


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", SRQR_CASES, ids=[c[0] for c in SRQR_CASES])
def test_srqr_verify_parity(ctx, name, kind, m, n, k, b, p, seed):
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.srqr_verify(A, k, b, p, seed=seed, d=8)
    Ad = to_dev(A)
    jpvt, tau, rank, diag = ctx.srqr_verify(Ad, k, b, p, seed=seed, d=8)
    torch.cuda.synchronize()
    assert rank == k
    assert diag["pivot"] == o["pivot"]
    assert np.array_equal(jpvt.cpu().numpy(), o["res"]["jpvt"])
    assert diag["alpha"] == pytest.approx(o["alpha"], rel=1e-10)
    assert diag["g1"] == pytest.approx(o["g1"], rel=1e-10)
    assert diag["g2_est"] == pytest.approx(o["g2_est"], rel=1e-9)
    assert diag["tau_bound"] == pytest.approx(o["tau_bound"], rel=1e-9)
    F = Ad.cpu().numpy()
    dg, do = np.abs(np.diag(F)[:k]), np.abs(np.diag(o["res"]["A"])[:k])
    assert np.max(np.abs(dg - do) / do) <= DIAG_RTOL


def test_srqr_verify_errors(ctx):
    import paper_1804_05138_b200 as rq
    A = to_dev(inputs.iid(3, 64, 48).numpy())
    with pytest.raises(rq.RqrcpError):
        ctx.srqr_verify(A, 48, 16, 4, d=8)     # k = min(m, n): nothing to verify
    with pytest.raises(rq.RqrcpError):
        ctx.srqr_verify(A, 16, 8, 4, d=0)      # d out of range


# ---- the CholeskyQR2 + Householder-reconstruction panel (cqr.cuh; the "TSQR
#      for the panel" future work of P:775) ----
CQR_CASES = [c for c in CASES if c[0] in ("C1", "ragged", "tall", "wide", "lowrank", "b128", "odd")]


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", CQR_CASES, ids=[c[0] for c in CQR_CASES])
def test_cqr_panel_parity(ctx, name, kind, m, n, k, b, p, seed):
    """RQRCP_PANEL=cqr: every well-conditioned panel goes through CholeskyQR2 +
    reconstruction (checked through the panels_householder counter) and the
    result meets the same acceptance as the column-by-column panel."""
    import os
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    os.environ["RQRCP_PANEL"] = "cqr"
    try:
        g = gpu_factor(ctx, A, k, b, p, seed)
        t = ctx.timings()
    finally:
        os.environ.pop("RQRCP_PANEL", None)
    compare(A, g, o, k)
    assert t["panels_householder"] < t["panels"]  # the CholeskyQR2 path factored panels


def test_cqr_guard_falls_back(ctx):
    """A rank-stopped panel (rank 40 < k = 64, b = 32: the second panel stops
    at bb_eff = 8, reading R-G12) fails the CholeskyQR2 guard and is factored
    by the column-by-column kernel; the result matches the oracle's."""
    import os
    rng = np.random.default_rng(5)
    A = rng.standard_normal((300, 40)) @ rng.standard_normal((40, 260))
    o = oracle.rqrcp(A, 64, 32, 8, seed=3, check=False)
    os.environ["RQRCP_PANEL"] = "cqr"
    try:
        Ad = to_dev(A)
        jpvt, tau, rank = ctx.factor(Ad, 64, 32, 8, seed=3)
        torch.cuda.synchronize()
        t = ctx.timings()
    finally:
        os.environ.pop("RQRCP_PANEL", None)
    assert rank == o["rank"] == 40
    assert t["panels_householder"] >= 1
    assert np.array_equal(jpvt.cpu().numpy()[:40], o["jpvt"][:40])
    dg, do = np.abs(np.diag(Ad.cpu().numpy())[:40]), np.abs(np.diag(o["A"])[:40])
    assert np.max(np.abs(dg - do) / do) <= DIAG_RTOL


def test_update_kernels_agree(ctx):
    """b = 128 (K = 128: the TMA-epilogue update kernel) vs the same
    factorization with the panels shifted by one row (odd offsets: the
    register-epilogue / cp.async kernels) -- both against the oracle."""
    A = inputs.make("iid", 1200, 1000, 33).numpy()
    o = oracle.rqrcp(A, 256, 128, 16, seed=33)
    g = gpu_factor(ctx, A, 256, 128, 16, 33)
    compare(A, g, o, 256)


# ---- low-rank outputs: SURVEY.md §8(f) N4 ----
LR_CASES = [c for c in CASES if c[0] in ("C1", "ragged", "tall", "wide", "b128", "odd")]


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", LR_CASES, ids=[c[0] for c in LR_CASES])
def test_lowrank_outputs(ctx, name, kind, m, n, k, b, p, seed):
    """Q1 against the oracle's reflectors applied to [I; 0] (P:120 'Q = H1 H2
    ... Hk'), Q1^T Q1 = I, Q1 [R11 R12] = A Pi truncated; CX
    coefficients against the definition X = C^+ A (least squares) and
    ||A - C X||_F = ||R22||_F."""
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    Ad = to_dev(A)
    jpvt, tau, rank = ctx.factor(Ad, k, b, p, seed=seed)
    torch.cuda.synchronize()
    assert np.array_equal(jpvt.cpu().numpy(), o["jpvt"])
    Q1 = ctx.form_q1(Ad, k, b, tau)
    X = ctx.cx(Ad, k, jpvt)
    torch.cuda.synchronize()
    Q1h, Xh = Q1.cpu().numpy(), X.cpu().numpy()
    E = np.zeros((m, k))
    E[:k, :k] = np.eye(k)
    Q1o = oracle.apply_q(o["A"], o["tau"], E)
    assert np.max(np.abs(Q1h - Q1o)) <= 1e-10
    assert np.linalg.norm(Q1h.T @ Q1h - np.eye(k)) <= 1e-12 * k
    F = Ad.cpu().numpy()
    Rt = np.triu(F[:k, :])
    jp = jpvt.cpu().numpy()
    assert np.linalg.norm(A[:, jp][:, :k] - Q1h @ Rt[:, :k]) <= 1e-12 * np.linalg.norm(A)
    C = A[:, jp[:k]]
    Xref = np.linalg.lstsq(C, A, rcond=None)[0]
    assert np.linalg.norm(Xh - Xref) <= 1e-8 * np.linalg.norm(Xref)
    r22 = np.linalg.norm(F[k:, k:])
    assert abs(np.linalg.norm(A - C @ Xh) - r22) <= 1e-10 * np.linalg.norm(A)
