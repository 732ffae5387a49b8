"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Acceptance (BASELINE.json north_star): identical pivot sequences; |diag R|
within 1e-10 relative; ||A Pi - Q1 [R11 R12]||_F/||A||_F (and ||R22||_F/||A||_F)
within 1e-12 of the oracle's.  On top of that every case compares, ELEMENT BY
ELEMENT (both sides use the dlarfg convention of reading R-G7, so no sign
fixing): [R11 R12] to 1e-10 max|R|, tau to 1e-10, the Householder vectors V
to 1e-10, and the full reconstruction A Pi = Q [R11 R12; 0 R22] to 1e-13.
Tolerances: the two sides sum in different orders, so entries differ by
O(kappa eps ||R||) (<= 1e-15 on these inputs); 1e-10 sits
five orders above that and five below an R12 that is wrong by 1e-6 relative.
Inputs are seeded synthetic matrices from inputs/ with the recipes of
BASELINE.json's configs, at sizes the oracle finishes in seconds (several
GEMM / sample-QRCP / panel tiles and ragged tails).
"""
import contextlib

import numpy as np
import pytest
import torch

import inputs
import oracle
from gpu_helpers import check_trace_panels

pytestmark = pytest.mark.gpu

DIAG_RTOL = 1e-10
RES_ATOL = 1e-12
ELEM_RTOL = 1e-10
RECON_TOL = 1e-13

DEFAULT_OPTS = dict(schedule=-1, panel=2, upd_kernel=2, pn_blocked=1, tournament=0, gemm_ws=1, pn_cluster=1, pn_cpt=2, pn_grid=0, pn_rows=128, la_panel_ctas=48,
                    sq_cluster=1, sq_reg=1, sq_grid=0, sq_nsm=-1, sq_hstride=8, sq_poll=3, cqr_rg=1, host_out=0, sq_wide=1, sq_smtop=1, sq_spec=0)


@pytest.fixture(scope="module")
def ctx():
    import paper_1804_05138_b200 as rq
    c = rq.RQRCP(max_m=5000, max_n=5000, max_b=128, max_p=32)
    yield c
    c.close()


@contextlib.contextmanager
def options(ctx, **kv):
    """Launch-path options for the duration of a block (create-time config of
    the context; restored to the defaults afterwards)."""
    for k, v in kv.items():
        ctx.set_option(k, v)
    try:
        yield
    finally:
        for k in kv:
            ctx.set_option(k, DEFAULT_OPTS[k])


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


def reflectors(F, k):
    """V (m x k): unit lower trapezoidal Householder vectors of the factored matrix."""
    m = F.shape[0]
    V = np.zeros((m, k))
    for j in range(k):
        V[j, j] = 1.0
        V[j + 1:, j] = F[j + 1:, j]
    return V


def q_apply(F, tau, C):
    """Q C with Q = H_1 ... H_k from the LAPACK-layout reflectors of F,
    by LAPACK dormqr (a library routine; the same layout as dgeqrf's)."""
    from scipy.linalg import lapack
    k = len(tau)
    if k == 0:
        return np.array(C, dtype=np.float64)
    a = np.asfortranarray(F[:, :k])
    c = np.asfortranarray(C, dtype=np.float64)
    lw = lapack.dormqr("L", "N", a, tau, c, -1)[1]
    out, _, info = lapack.dormqr("L", "N", a, tau, c, int(lw[0]) if np.ndim(lw) else int(lw), overwrite_c=0)
    assert info == 0
    return out


def trunc_residual(A, res, k, probes=None):
    """||A Pi - Q1 [R11 R12]||_F / ||A||_F (exact when probes is None)."""
    Api = A[:, res["jpvt"]]
    Rt = np.triu(res["A"][:k, :])
    Rfull = np.zeros_like(res["A"])
    Rfull[:k] = Rt
    if probes is None:
        return np.linalg.norm(Api - q_apply(res["A"], res["tau"][:k], Rfull)) / np.linalg.norm(A)
    X = probes
    return np.linalg.norm(Api @ X - q_apply(res["A"], res["tau"][:k], Rfull @ X)) / np.linalg.norm(A @ X)


def reconstruction_error(A, res, k):
    """||A Pi - Q [R11 R12; 0 R22]||_F / ||A||_F from the GPU's own outputs."""
    R = full_R(res["A"], k)
    return np.linalg.norm(A[:, res["jpvt"]] - q_apply(res["A"], res["tau"][:k], R)) / np.linalg.norm(A)


def compare(A, g, o, k, probes=None, rank=None):
    k_eff = k if rank is None else rank
    assert g["rank"] == o["rank"] == k_eff
    # identical pivot sequences (the whole permutation: same transpositions)
    if not np.array_equal(g["jpvt"], o["jpvt"]):
        bad = int(np.nonzero(g["jpvt"] != o["jpvt"])[0][0])
        pytest.fail(f"pivots differ first at {bad}; oracle gap there {o['gaps'][min(bad, k - 1)]:.3e}")
    kk = k_eff
    dg = np.abs(np.diag(g["A"])[:kk])
    do = np.abs(np.diag(o["A"])[:kk])
    assert np.max(np.abs(dg - do) / do, initial=0.0) <= DIAG_RTOL
    # element-wise [R11 R12], tau, V (reading R-G7: same convention on both sides)
    Rg, Ro = np.triu(g["A"][:kk, :]), np.triu(o["A"][:kk, :])
    rmax = np.max(np.abs(Ro), initial=1.0)
    assert np.max(np.abs(Rg - Ro), initial=0.0) <= ELEM_RTOL * rmax, "R11/R12 differ element-wise"
    assert np.max(np.abs(g["tau"][:kk] - o["tau"][:kk]), initial=0.0) <= ELEM_RTOL, "tau differs"
    Vg, Vo = reflectors(g["A"], kk), reflectors(o["A"], kk)
    assert np.max(np.abs(Vg - Vo), initial=0.0) <= ELEM_RTOL * max(1.0, np.max(np.abs(Vo), initial=0.0)), "V differs"
    if kk < k:
        assert np.all(g["tau"][kk:k] == 0.0)
    nA = np.linalg.norm(A)
    r22g = np.linalg.norm(full_R(g["A"], kk)[kk:, kk:]) / nA
    r22o = np.linalg.norm(full_R(o["A"], kk)[kk:, kk:]) / nA
    assert abs(r22g - r22o) <= RES_ATOL
    rg = trunc_residual(A, g, kk, probes)
    ro = trunc_residual(A, o, kk, probes)
    assert abs(rg - ro) <= RES_ATOL
    if probes is None:
        assert reconstruction_error(A, g, kk) <= RECON_TOL
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
    """configs[1] at its full size: 4096^2, k=512, b=64, p=10, element-wise."""
    c = inputs.CONFIGS["C2"]
    A = inputs.config_matrix("C2").numpy()
    o = oracle.rqrcp(A, c["k"], c["b"], c["p"], seed=c["seed"])
    g = gpu_factor(ctx, A, c["k"], c["b"], c["p"], c["seed"])
    compare(A, g, o, c["k"])


# ---- the per-panel trace (rqrcp_factor_ex) against the
#      oracle's panel callback: pivots, R-hat after S2 and the
#      updated sample after S6 (Eq. (4)) element by element ------
def trace_compare(ctx, A, k, b, p, seed, update_rule=1, opts=None):
    m, n = A.shape
    l = b + p
    npan = (k + b - 1) // b
    tr = ctx.make_trace(n, b, p, 0, npan)
    Ad = to_dev(A)
    if update_rule == 2:
        ctx.set_update_rule(2)
    try:
        with options(ctx, **(opts or {})):
            jpvt, tau, rank = ctx.factor(Ad, k, b, p, seed=seed, trace=tr)
    finally:
        ctx.set_update_rule(1)
    torch.cuda.synchronize()
    assert tr.recorded == npan
    panels = []
    o = oracle.rqrcp(A, k, b, p, seed=seed, update_rule=update_rule,
                     callback=lambda i, bb, l_, mp, np_, Rh, Bn, Oc, On, Af: panels.append((i, bb, Rh, Bn)))
    assert len(panels) == npan
    jp = jpvt.cpu().numpy()
    assert np.array_equal(jp, o["jpvt"])
    check_trace_panels(tr, panels, o["jpvt"])
    return panels


TRACE_CASES = [c for c in CASES if c[0] in ("C1", "ragged", "tall", "lowrank", "b128", "odd")]


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", TRACE_CASES, ids=[c[0] for c in TRACE_CASES])
def test_trace_per_panel(ctx, name, kind, m, n, k, b, p, seed):
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    trace_compare(ctx, A, k, b, p, seed)


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", TRACE_CASES[:4], ids=[c[0] for c in TRACE_CASES[:4]])
def test_trace_per_panel_eq5(ctx, name, kind, m, n, k, b, p, seed):
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    trace_compare(ctx, A, k, b, p, seed, update_rule=2)


def test_trace_window_and_C2(ctx):
    """A recording window (panels 2..4 of C2 at full size)."""
    c = inputs.CONFIGS["C2"]
    A = inputs.config_matrix("C2").numpy()
    m, n, k, b, p = c["m"], c["n"], c["k"], c["b"], c["p"]
    tr = ctx.make_trace(n, b, p, 2, 3)
    Ad = to_dev(A)
    ctx.factor(Ad, k, b, p, seed=c["seed"], trace=tr)
    torch.cuda.synchronize()
    assert tr.recorded == 3
    panels = []
    o = oracle.rqrcp(A, 5 * b, b, p, seed=c["seed"], invariant=True,
                     callback=lambda i, bb, l_, mp, np_, Rh, Bn, Oc, On, Af: panels.append((i, bb, Rh, Bn)))
    # the window records panels 2..4 (trace slots 0..2)
    check_trace_panels(tr, panels, o["jpvt"], first=2, last=5)


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


def test_duplicate_columns_tie_rule(ctx):
    """Exact ties of the squared sample norms go to the LOWEST current position
    (reading R-G5): every column appears twice, so each first pick is a
    bitwise tie between two identical sample columns."""
    rng = np.random.default_rng(8)
    X = rng.standard_normal((300, 60)) * np.exp(-np.arange(60) / 10.0)
    A = np.repeat(X, 2, axis=1)  # columns 2c and 2c+1 identical
    o = oracle.rqrcp(A, 32, 8, 4, seed=9, check=False)
    g = gpu_factor(ctx, A, 32, 8, 4, 9)
    assert g["rank"] == o["rank"]
    r = o["rank"]
    assert np.array_equal(g["jpvt"][:r], o["jpvt"][:r])
    # the first pivot is the even (lower) member of its identical pair
    assert o["jpvt"][0] % 2 == 0


def test_rank_deficient(ctx):
    rng = np.random.default_rng(42)
    A = rng.standard_normal((120, 25)) @ rng.standard_normal((25, 100))
    o = oracle.rqrcp(A, 60, 16, 8, seed=1)
    g = gpu_factor(ctx, A, 60, 16, 8, 1)
    assert g["rank"] == o["rank"] == 25
    assert np.array_equal(g["jpvt"], o["jpvt"])
    assert np.all(g["tau"][25:] == 0.0)


def r11_stop_problem():
    """A panel whose R11 diagonal collapses while its sample norms stay large:
    column 5 of A is 1e-15 e_5 but Omega amplifies row 5 by 1e17, so the sample
    QRCP picks it second (its sample norm ~ 270 vs ~ 600 for the 200-scaled
    column 0 and ~ 3 for the rest); |R(1,1)| = 1e-15 <
    1e3 eps ||panel||_F (reading R-G12b) stops the factorization at rank 1."""
    m, n, b, p = 40, 30, 8, 2
    A = np.zeros((m, n))
    for j in range(n):
        A[j, j] = 1.0
    A[5, 5] = 1e-15
    A[:, 0] *= 200.0
    Om = np.random.default_rng(11).standard_normal((b + p, m))
    Om[:, 5] *= 1e17
    return A, Om, b, p


def test_r11_diagonal_rank_stop(ctx):
    A, Om, b, p = r11_stop_problem()
    o = oracle.rqrcp(A, 16, b, p, omega=Om, check=False)
    assert o["rank"] == 1 and o["jpvt"][1] == 5
    g = gpu_factor(ctx, A, 16, b, p, 0, omega=torch.tensor(Om.ravel(order="F")).cuda())
    assert g["rank"] == 1
    assert np.array_equal(g["jpvt"][:2], o["jpvt"][:2])
    assert np.all(g["tau"][1:] == 0.0)
    assert abs(abs(g["A"][0, 0]) - abs(o["A"][0, 0])) <= 1e-12 * abs(o["A"][0, 0])


def test_r11_stop_blocked_panel(ctx):
    """The R11-diagonal stop inside the 2nd / 4th 32-column sub-panel of a
    b = 128 blocked grid panel.  A = diag(0.8^j) except a 1e-16 entry in column
    `col`, whose Omega column is amplified so that its sample norm sits between
    those of columns col-1 and col: the sample QRCP picks it at step col, where
    |R(col,col)| = 1e-16 stops the factorization at rank col (oracle pin); the
    GPU agrees on rank, pivots and R rows."""
    for col in (40, 100):
        m, n, b, p = 600, 400, 128, 16
        rng = np.random.default_rng(col)
        A = np.zeros((m, n))
        A[np.arange(n), np.arange(n)] = 0.8 ** np.arange(n)
        A[col, col] = 1e-16
        Om = rng.standard_normal((b + p, m))
        Om[:, col] *= 0.8 ** (col - 0.5) * 1e16
        o = oracle.rqrcp(A, 256, b, p, omega=Om, check=False)
        assert o["rank"] == col
        with options(ctx, pn_cluster=0, pn_blocked=2):
            g = gpu_factor(ctx, A, 256, b, p, 0, omega=torch.tensor(Om.ravel(order="F")).cuda())
        assert g["rank"] == col
        assert np.array_equal(g["jpvt"][:col + 1], o["jpvt"][:col + 1])
        assert np.max(np.abs(np.triu(g["A"][:col]) - np.triu(o["A"][:col]))) <= 1e-10 * np.max(np.abs(o["A"][:col]))
        assert np.all(g["tau"][col:] == 0.0)


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
    assert L.rqrcp_set_option(h, b"no_such_option", 1) == -2
    assert L.rqrcp_set_option(h, b"schedule", 7) == -3


def test_binding_validation(ctx):
    """The binding rejects overlapping views and wrong output vectors."""
    A = torch.zeros(64, 48, dtype=torch.float64, device="cuda").t().contiguous().t()
    with pytest.raises(ValueError):
        ctx.factor(A[:, :1].expand(64, 8), 4, 2, 2)
    with pytest.raises(TypeError):
        ctx.factor(A, 4, 2, 2, jpvt=torch.zeros(48, dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        ctx.factor(A, 4, 2, 2, tau=torch.zeros(2, dtype=torch.float64, device="cuda"))


def test_factor_host_equals_device(ctx):
    A = inputs.iid(8, 640, 512).numpy()
    g = gpu_factor(ctx, A, 96, 32, 8, 5)
    Ah = inputs.fortran(torch.as_tensor(A)).pin_memory()
    jp, ta, rank = ctx.factor_host(Ah, 96, 32, 8, seed=5)
    assert rank == 96
    assert np.array_equal(Ah.numpy(), g["A"])
    assert np.array_equal(jp.numpy(), g["jpvt"])


def test_factor_host_streams_chunks(ctx):
    """The end-to-end path streams A in by 2048-column chunks (each chunk's
    sketch as it lands) and the finished panels out during the factorization:
    bitwise the device-path result, also in place (A_out = A_in)."""
    A = inputs.iid(9, 400, 4700).numpy()
    g = gpu_factor(ctx, A, 128, 32, 8, 6)
    Ah = inputs.fortran(torch.as_tensor(A)).pin_memory()
    Ao = inputs.fortran(torch.zeros_like(torch.as_tensor(A))).pin_memory()
    jp, ta, rank = ctx.factor_host(Ah, 128, 32, 8, seed=6, out=Ao)
    assert rank == 128
    assert np.array_equal(Ao.numpy(), g["A"]) and np.array_equal(jp.numpy(), g["jpvt"])
    jp2, ta2, rank2 = ctx.factor_host(Ah, 128, 32, 8, seed=6)  # in place
    assert np.array_equal(Ah.numpy(), g["A"])


def test_factor_host_factors_only(ctx):
    """Option host_out = 1: the host receives the partial factorization's
    outputs only -- columns 0..k-1 full height (V, R11) and rows
    0..k-1 of the trailing columns (R12), bitwise the device result; the R22
    block of the output buffer is left untouched."""
    A = inputs.iid(10, 500, 3000).numpy()
    k = 96
    g = gpu_factor(ctx, A, k, 32, 8, 7)
    Ah = inputs.fortran(torch.as_tensor(A)).pin_memory()
    Ao = inputs.fortran(torch.full(A.shape, 7.25, dtype=torch.float64)).pin_memory()
    ctx.set_option("host_out", 1)
    try:
        jp, ta, rank = ctx.factor_host(Ah, k, 32, 8, seed=7, out=Ao)
    finally:
        ctx.set_option("host_out", 0)
    o = Ao.numpy()
    assert rank == k
    assert np.array_equal(o[:, :k], g["A"][:, :k])
    assert np.array_equal(o[:k, k:], g["A"][:k, k:])
    assert np.all(o[k:, k:] == 7.25)
    assert np.array_equal(jp.numpy(), g["jpvt"]) and np.array_equal(ta.numpy(), g["tau"][:k])


# ---- launch-shape variants of the sample QRCP (threads per column, spill) ----
# sq_grid caps the cooperative grid (fewer CTAs -> more columns per CTA, fewer
# threads per column) and sq_nsm caps the columns a CTA keeps in shared memory
# (the rest go through the transposed L2 spill buffer).
SQ_VARIANTS = [(148, -1), (2, 0), (7, 5), (33, -1), (1, 40)]
SQ_CASES = [c for c in CASES if c[0] in ("ragged", "odd", "b128", "b1p0", "lowrank")]


@pytest.mark.parametrize("grid,nsm", SQ_VARIANTS, ids=[f"g{g}-nsm{n}" for g, n in SQ_VARIANTS])
@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", SQ_CASES, ids=[c[0] for c in SQ_CASES])
def test_sample_qrcp_launch_variants(ctx, grid, nsm, name, kind, m, n, k, b, p, seed):
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    with options(ctx, sq_grid=grid, sq_cluster=0, sq_reg=0, sq_nsm=nsm):
        g = gpu_factor(ctx, A, k, b, p, seed)
    compare(A, g, o, k)


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", SQ_CASES[:3], ids=[c[0] for c in SQ_CASES[:3]])
def test_sample_qrcp_exchange_modes_bitwise(ctx, name, kind, m, n, k, b, p, seed):
    """Grid sample QRCP: the tagged-unit exchange (sq_poll 3, no fences) and
    the release / acquire header exchange (0, 1) move the same candidates and
    columns: same bits."""
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    outs = []
    for pm in (0, 1, 3):
        with options(ctx, sq_grid=7, sq_cluster=0, sq_reg=0, sq_nsm=5, sq_poll=pm):
            outs.append(gpu_factor(ctx, A, k, b, p, seed))
    for o in outs[:2]:
        for key in ("A", "jpvt", "tau"):
            assert np.array_equal(o[key], outs[2][key])


# ---- the register-resident grid sample QRCP (sample_qrcp_reg.cuh) ----------
REG_CASES = [c for c in CASES if c[0] in ("C1", "ragged", "tall", "lowrank", "kfull", "b128")] + [
    ("reg_wide74", "iid", 800, 1900, 192, 64, 10, 21),
    ("reg_wide144", "graded", 900, 2100, 256, 128, 16, 22),
    ("reg_lowrank144", "lowrank", 700, 1300, 300, 128, 16, 23),
]


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", REG_CASES, ids=[c[0] for c in REG_CASES])
def test_sample_qrcp_register_grid(ctx, name, kind, m, n, k, b, p, seed):
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    with options(ctx, sq_cluster=0):
        g = gpu_factor(ctx, A, k, b, p, seed)
    compare(A, g, o, k)


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", REG_CASES[:3] + REG_CASES[-3:],
                         ids=[c[0] for c in REG_CASES[:3] + REG_CASES[-3:]])
def test_sample_qrcp_register_grid_all_sms_bitwise(ctx, name, kind, m, n, k, b, p, seed):
    """sq_wide = 2 spreads the sample over every SM (fewer columns per CTA, the
    launch bench.py takes for wide samples); the per-column arithmetic and the
    tie rule do not depend on the partition: bitwise the fewest-CTA launch."""
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    with options(ctx, sq_cluster=0, sq_wide=0):
        g0 = gpu_factor(ctx, A, k, b, p, seed)
    with options(ctx, sq_cluster=0, sq_wide=2):
        g2 = gpu_factor(ctx, A, k, b, p, seed)
    with options(ctx, sq_cluster=0, sq_reg=2, sq_wide=2):
        g3 = gpu_factor(ctx, A, k, b, p, seed)
    with options(ctx, sq_cluster=0, sq_reg=2, sq_wide=0):
        g4 = gpu_factor(ctx, A, k, b, p, seed)
    for key in ("A", "jpvt", "tau"):
        assert np.array_equal(g0[key], g2[key]), key
        assert np.array_equal(g3[key], g4[key]), key


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", REG_CASES[-2:], ids=[c[0] for c in REG_CASES[-2:]])
@pytest.mark.parametrize("sq_reg", [1, 2])
def test_sample_qrcp_register_grid_row_layouts(ctx, name, kind, m, n, k, b, p, seed, sq_reg):
    """Both row layouts of the l = 144 register grids (shared-memory rows above
    the register rows -- the default -- and below them) match the oracle; they
    sum the rows in a different grouping, so only the pivots are bitwise equal."""
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    gs = []
    for smt in (0, 1):
        with options(ctx, sq_cluster=0, sq_reg=sq_reg, sq_smtop=smt):
            g = gpu_factor(ctx, A, k, b, p, seed)
        compare(A, g, o, k)
        gs.append(g)
    assert np.array_equal(gs[0]["jpvt"], gs[1]["jpvt"])


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", REG_CASES[:2] + REG_CASES[-2:],
                         ids=[c[0] for c in REG_CASES[:2] + REG_CASES[-2:]])
@pytest.mark.parametrize("sq_reg", [1, 2])
def test_sample_qrcp_register_grid_speculative_exchange_bitwise(ctx, name, kind, m, n, k, b, p, seed, sq_reg):
    """The speculative column fetch of the register grids' exchange (sq_spec = 1)
    picks the same winner and reflector as fetching after every header: bitwise."""
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    gs = []
    for spec in (0, 1):
        with options(ctx, sq_cluster=0, sq_reg=sq_reg, sq_wide=2, sq_spec=spec):
            gs.append(gpu_factor(ctx, A, k, b, p, seed))
    for key in ("A", "jpvt", "tau"):
        assert np.array_equal(gs[0][key], gs[1][key]), key


# the 512-thread register grid with the top 60 rows in global memory
# (sample_qrcp_reg2.cuh, l = 144: the C5 sample); sq_reg = 2 selects it at
# oracle-feasible widths, including samples narrower than one CTA per SM
REG2_CASES = [("reg2_wide144", "graded", 900, 2100, 256, 128, 16, 22),
              ("reg2_lowrank144", "lowrank", 700, 1300, 300, 128, 16, 23),
              ("reg2_iid_ragged", "iid", 650, 4997, 384, 128, 16, 24),
              ("reg2_kfull", "iid", 400, 600, 400, 128, 16, 25)]


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", REG2_CASES, ids=[c[0] for c in REG2_CASES])
def test_sample_qrcp_register_grid_top_rows_global(ctx, name, kind, m, n, k, b, p, seed):
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    with options(ctx, sq_cluster=0, sq_reg=2):
        g = gpu_factor(ctx, A, k, b, p, seed)
    compare(A, g, o, k)


# ---- panel kernels: the register-resident cluster kernel (panel_cl.cuh) and
# the cooperative grid kernel (panel.cuh); pn_rows = 8 forces the grid
# kernel's rows-beyond-shared-memory (L2) path at an oracle-feasible size.
PN_CASES = [c for c in CASES if c[0] in ("C1", "ragged", "tall", "wide", "odd", "kfull", "b1p0")] + [
    ("pncl_tall32", "iid", 5000, 300, 96, 32, 8, 24),
    ("pncl_4096", "lowrank", 4096, 700, 192, 64, 10, 25),
]
PN_VARIANTS = {"cluster2": dict(pn_cluster=1, pn_cpt=2), "cluster1": dict(pn_cluster=1, pn_cpt=1),
               "grid": dict(pn_cluster=0, pn_blocked=0), "gridblocked": dict(pn_cluster=0, pn_blocked=2)}


@pytest.mark.parametrize("variant", list(PN_VARIANTS))
@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", PN_CASES, ids=[c[0] for c in PN_CASES])
def test_panel_kernels(ctx, variant, name, kind, m, n, k, b, p, seed):
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    with options(ctx, **PN_VARIANTS[variant]):
        g = gpu_factor(ctx, A, k, b, p, seed)
    compare(A, g, o, k)


@pytest.mark.parametrize("rows,grid", [(8, 4), (16, 2), (1, 1)])
def test_panel_grid_l2_rows(ctx, rows, grid):
    """Grid panel kernel with more rows per CTA than shared memory holds
    (PN_MAXROWS staging, rows >= nsm via L2): b = 128 panels of 3000 rows on
    1-4 CTAs put ~750-3000 rows per CTA, ~200 of them in shared memory."""
    A = inputs.make("graded", 3000, 700, 41).numpy()
    o = oracle.rqrcp(A, 256, 128, 16, seed=41)
    for blocked in (0, 2):
        with options(ctx, pn_cluster=0, pn_rows=rows, pn_grid=grid, pn_blocked=blocked):
            g = gpu_factor(ctx, A, 256, 128, 16, 41)
        compare(A, g, o, 256)


# ---- schedules: serial, bulk update beside the next sample QRCP, bulk update
# beside the next panel QR (look-ahead): the same arithmetic, bitwise -------
SCHED_CASES = [c for c in CASES if c[0] in ("C1", "ragged", "tall", "lowrank", "kfull", "b128", "odd")] + [
    ("grid74", "iid", 700, 4700, 192, 64, 10, 28),    # register-grid sample QRCP
    ("gridpanel", "graded", 4500, 900, 256, 128, 16, 29),  # grid panel kernel (b = 128)
]


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", SCHED_CASES, ids=[c[0] for c in SCHED_CASES])
def test_schedules_bitwise_and_parity(ctx, name, kind, m, n, k, b, p, seed):
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    outs = []
    for s in (0, 1, 2):
        with options(ctx, schedule=s):
            outs.append(gpu_factor(ctx, A, k, b, p, seed))
    compare(A, outs[2], o, k)
    for g in outs[:2]:
        assert np.array_equal(g["jpvt"], outs[2]["jpvt"])
        assert np.array_equal(g["tau"], outs[2]["tau"])
        assert np.array_equal(g["A"], outs[2]["A"])


@pytest.mark.parametrize("uk", [0, 1])
@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", [c for c in SCHED_CASES if c[0] in ("tall", "b128", "gridpanel")],
                         ids=["tall", "b128", "gridpanel"])
def test_update_kernels_bitwise(ctx, uk, name, kind, m, n, k, b, p, seed):
    """The update GEMM variants (CTA-wide TMA epilogue / warp-specialised
    with per-warp epilogues) compute every element the same way: same bits."""
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    ref = gpu_factor(ctx, A, k, b, p, seed)
    with options(ctx, upd_kernel=uk):
        g = gpu_factor(ctx, A, k, b, p, seed)
    assert np.array_equal(g["A"], ref["A"]) and np.array_equal(g["jpvt"], ref["jpvt"])


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", [c for c in SCHED_CASES if c[0] in ("tall", "b128", "grid74")],
                         ids=["tall", "b128", "grid74"])
def test_skinny_gemm_kernels_bitwise(ctx, name, kind, m, n, k, b, p, seed):
    """The sketch / W = V^T A22 GEMM: warp-specialised vs CTA-barrier ring
    kernels -- same tiles, same K slices, same bits."""
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    ref = gpu_factor(ctx, A, k, b, p, seed)
    with options(ctx, gemm_ws=0):
        g = gpu_factor(ctx, A, k, b, p, seed)
    assert np.array_equal(g["A"], ref["A"]) and np.array_equal(g["jpvt"], ref["jpvt"])


def test_schedules_bitwise_C2(ctx):
    c = inputs.CONFIGS["C2"]
    A = inputs.config_matrix("C2").numpy()
    outs = []
    for s in (0, 1, 2):
        with options(ctx, schedule=s):
            outs.append(gpu_factor(ctx, A, c["k"], c["b"], c["p"], c["seed"]))
    for g in outs[1:]:
        assert np.array_equal(g["jpvt"], outs[0]["jpvt"])
        assert np.array_equal(g["A"], outs[0]["A"])


# ---- updating formula 2 (Eq. (5)) on the GPU: SURVEY.md §8(f) N2 ----
EQ5_CASES = [c for c in CASES if c[0] in ("C1", "ragged", "tall", "lowrank", "b128", "odd")]


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", EQ5_CASES, ids=[c[0] for c in EQ5_CASES])
def test_eq5_update_parity(ctx, name, kind, m, n, k, b, p, seed):
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed, update_rule=2)
    ctx.set_update_rule(2)
    try:
        g = gpu_factor(ctx, A, k, b, p, seed)
    finally:
        ctx.set_update_rule(1)
    compare(A, g, o, k)


def test_eq4_eq5_identical_permutations_gpu(ctx):
    """the two updating formulas give the same permutation."""
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


@pytest.mark.parametrize("rg", [1, 0], ids=["regs", "smem"])
@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", CQR_CASES, ids=[c[0] for c in CQR_CASES])
def test_cqr_panel_parity(ctx, name, kind, m, n, k, b, p, seed, rg):
    """panel=1: every well-conditioned panel goes through CholeskyQR2 +
    reconstruction (checked through the panels_householder counter); the
    result meets the same acceptance.  R, V, tau come from a different
    algorithm here, so they are compared to 1e-10 like everything else.
    rg: the one-CTA factorizations in registers (cqr_rg.cuh) or in shared
    memory (cqr.cuh)."""
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    with options(ctx, panel=1, cqr_rg=rg):
        g = gpu_factor(ctx, A, k, b, p, seed)
        t = ctx.timings()
    compare(A, g, o, k)
    assert t["panels_householder"] < t["panels"]


def test_cqr_tall_in_place_products_deterministic():
    """Tall panels through the CholeskyQR2 path (the default from 8192 rows): the
    512-thread row product writes V2 over its own input (two warps per row tile),
    which needs every fragment load of a round before the round's stores -- a race
    there shows as run-to-run differences and a broken reconstruction.  Three runs
    bitwise equal, and A Pi = Q R to 1e-13 (probe)."""
    import paper_1804_05138_b200 as rq
    m, n, k, b, p = 40000, 640, 384, 128, 16
    A = inputs.make("graded", m, n, 31).numpy()
    c = rq.RQRCP(max_m=m, max_n=n, max_b=b, max_p=p)
    outs = []
    for _ in range(3):
        Ad = to_dev(A)
        jpvt, tau, rank = c.factor(Ad, k, b, p, seed=31)
        torch.cuda.synchronize()
        outs.append((Ad.cpu().numpy(), jpvt.cpu().numpy(), tau.cpu().numpy()))
    t = c.timings()
    c.close()
    assert t["panels_householder"] < t["panels"]  # the CholeskyQR2 path ran
    for o in outs[1:]:
        assert all(np.array_equal(x, y) for x, y in zip(outs[0], o))
    F, jp, ta = outs[0]
    rng = np.random.default_rng(3)
    X = rng.standard_normal((n, 2))
    R = np.triu(F[:k, :])
    RX = np.zeros((m, 2))
    RX[:k] = R @ X
    RX[k:] = (F[:, k:] @ X[k:])[k:]
    Xp = np.zeros_like(X)
    Xp[jp] = X
    Y = RX.copy()
    for j in range(k - 1, -1, -1):
        v = F[j:, j].copy()
        v[0] = 1.0
        Y[j:] -= ta[j] * np.outer(v, v @ Y[j:])
    err = np.linalg.norm(A @ Xp - Y) / (np.linalg.norm(A) * np.linalg.norm(X))
    assert err <= 1e-13, err


def test_cqr_default_crosses_row_threshold():
    """Default panel option 2: CholeskyQR2 while the panel has >= 8192 rows, the
    column-by-column kernels below -- one factorization crossing the threshold
    (m = 8300, b = 128: panel 0 via CholeskyQR2, panels 1.. via Householder)
    matches the oracle like any other case."""
    import paper_1804_05138_b200 as rq
    m, n, k, b, p, seed = 8300, 600, 384, 128, 16, 41
    A = inputs.make("iid", m, n, seed).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    c = rq.RQRCP(max_m=m, max_n=n, max_b=b, max_p=p)
    g = gpu_factor(c, A, k, b, p, seed)
    t = c.timings()
    c.close()
    compare(A, g, o, k)
    assert 0 < t["panels_householder"] < t["panels"]


def test_cqr_guard_falls_back(ctx):
    """A rank-stopped panel fails the CholeskyQR2 guard and is factored by the
    column-by-column kernel; the result matches the oracle's."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((300, 40)) @ rng.standard_normal((40, 260))
    o = oracle.rqrcp(A, 64, 32, 8, seed=3, check=False)
    with options(ctx, panel=1):
        Ad = to_dev(A)
        jpvt, tau, rank = ctx.factor(Ad, 64, 32, 8, seed=3)
        torch.cuda.synchronize()
        t = ctx.timings()
    assert rank == o["rank"] == 40
    assert t["panels_householder"] >= 1
    assert np.array_equal(jpvt.cpu().numpy()[:40], o["jpvt"][:40])
    dg, do = np.abs(np.diag(Ad.cpu().numpy())[:40]), np.abs(np.diag(o["A"])[:40])
    assert np.max(np.abs(dg - do) / do) <= DIAG_RTOL


def test_r11_stop_cqr_declines(ctx):
    """With the CholeskyQR2 panel the R11-diagonal stop is still taken (the
    guard declines a panel with a diagonal below the threshold)."""
    A, Om, b, p = r11_stop_problem()
    with options(ctx, panel=1):
        g = gpu_factor(ctx, A, 16, b, p, 0, omega=torch.tensor(Om.ravel(order="F")).cuda())
    assert g["rank"] == 1


# ---- low-rank outputs: SURVEY.md §8(f) N4 ----
LR_CASES = [c for c in CASES if c[0] in ("C1", "ragged", "tall", "wide", "b128", "odd")]


@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", LR_CASES, ids=[c[0] for c in LR_CASES])
def test_lowrank_outputs(ctx, name, kind, m, n, k, b, p, seed):
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


# ---- tournament pivoting on the sample (reading R-TP): the GPU
#      variant (sample QRCP kernels on column groups + merges) vs the oracle's
TP_CASES = [c for c in CASES if c[0] in ("C1", "ragged", "tall", "lowrank", "b128", "odd", "wide")]


@pytest.mark.parametrize("groups", [2, 3, 8])
@pytest.mark.parametrize("name,kind,m,n,k,b,p,seed", TP_CASES, ids=[c[0] for c in TP_CASES])
def test_tournament_parity(ctx, groups, name, kind, m, n, k, b, p, seed):
    A = inputs.make(kind, m, n, seed, rank=64).numpy()
    o = oracle.rqrcp(A, k, b, p, seed=seed, tournament=groups)
    with options(ctx, tournament=groups):
        g = gpu_factor(ctx, A, k, b, p, seed)
    compare(A, g, o, k)


def test_tournament_trace_and_C2(ctx):
    """C2 at full size with 8 groups, with the per-panel trace (R-hat after the
    tournament, B_next after Eq. (4)) against the oracle's callback."""
    c = inputs.CONFIGS["C2"]
    A = inputs.config_matrix("C2").numpy()
    m, n, k, b, p = c["m"], c["n"], c["k"], c["b"], c["p"]
    tr = ctx.make_trace(n, b, p, 0, k // b)
    Ad = to_dev(A)
    with options(ctx, tournament=8):
        jpvt, tau, rank = ctx.factor(Ad, k, b, p, seed=c["seed"], trace=tr)
    torch.cuda.synchronize()
    panels = []
    o = oracle.rqrcp(A, k, b, p, seed=c["seed"], tournament=8,
                     callback=lambda i, bb, l_, mp, np_, Rh, Bn, Oc, On, Af: panels.append((i, bb, Rh, Bn)))
    assert np.array_equal(jpvt.cpu().numpy(), o["jpvt"])
    check_trace_panels(tr, panels, o["jpvt"])
    g = dict(A=Ad.cpu().numpy(), jpvt=jpvt.cpu().numpy(), tau=tau.cpu().numpy(), rank=rank)
    compare(A, g, o, k)


def test_tournament_rank_deficient(ctx):
    rng = np.random.default_rng(42)
    A = rng.standard_normal((120, 25)) @ rng.standard_normal((25, 100))
    o = oracle.rqrcp(A, 60, 16, 8, seed=1, tournament=4)
    with options(ctx, tournament=4):
        g = gpu_factor(ctx, A, 60, 16, 8, 1)
    assert g["rank"] == o["rank"] == 25
    assert np.array_equal(g["jpvt"][:25], o["jpvt"][:25])
