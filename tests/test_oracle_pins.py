"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test names the passage (P:line of PAPER.md, S:line of SPEC.md) or the
DESIGN.md reading it checks.  None of them compares the oracle with itself:
the pins are paper-printed values (tests/golden/), closed forms, special
cases that reduce to LAPACK dgeqp3 (scipy) or to a brute-force definition,
and invariants of the exact-arithmetic method.
"""
import math

import numpy as np
import pytest
import scipy.linalg as sl

import inputs
import oracle

EPS = np.finfo(np.float64).eps


def brute_force_qrcp_pivots(A, k):
    """Greedy column selection by definition: at each step the
    column whose component orthogonal to the chosen columns has the largest
    norm; residual norms recomputed from scratch via a library QR."""
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[1]
    chosen = []
    for _ in range(k):
        if chosen:
            Q, _ = np.linalg.qr(A[:, chosen])
            Res = A - Q @ (Q.T @ A)
        else:
            Res = A
        norms = np.linalg.norm(Res, axis=0)
        norms[chosen] = -1.0
        chosen.append(int(np.argmax(norms)))
    return np.array(chosen)


def full_R(res, k):
    """R = [R11 R12; 0 R22]: the factored matrix with reflectors removed."""
    R = res["A"].copy()
    for j in range(k):
        R[j + 1:, j] = 0.0
    return R


def graded_matrix(rng, m, n, ratio):
    d = ratio ** (-np.arange(n, dtype=np.float64))
    rng.shuffle(d)
    return rng.standard_normal((m, n)) * d, d


# ----------------------------------------------------------------------------
# Generator (reading G8): Philox4x32-10 + Box-Muller
# ----------------------------------------------------------------------------
def test_philox_known_answers(golden):
    """Published Philox4x32-10 known answers (tests/golden/philox4x32_10_kat.txt)."""
    import torch
    for row in golden("philox4x32_10_kat.txt"):
        v = [int(x, 16) for x in row]
        ctr, key, out = v[0:4], v[4:6], tuple(v[6:10])
        assert oracle.philox4x32_10(ctr, key) == out
        t = [torch.tensor(x, dtype=torch.int64) for x in ctr]
        assert tuple(int(x) for x in inputs.philox4x32_10(*t, key[0], key[1])) == out


def test_normal_distribution():
    """Omega must be i.i.d. N(0,1): moments and Kolmogorov-Smirnov."""
    from scipy import stats
    z = oracle.normal(1234, 0, 400, 500).ravel()
    assert abs(z.mean()) < 5.0 / math.sqrt(z.size)
    assert abs(z.var() - 1.0) < 5.0 * math.sqrt(2.0 / z.size)
    assert stats.kstest(z, "norm").pvalue > 1e-3
    # neighbouring rows (the Box-Muller pair) are uncorrelated
    Z = oracle.normal(99, 0, 2, 100000)
    assert abs(np.corrcoef(Z[0], Z[1])[0, 1]) < 5.0 / math.sqrt(1e5)


def test_normal_two_implementations_agree():
    """oracle (C) and inputs (torch) implement the same map: integer words
    bitwise, normals to a few ulp (libm log/sin/cos are not correctly rounded)."""
    a = oracle.normal(77, 3, 37, 29, row0=5, col0=11)
    b = inputs.gaussian(77, 3, 37, 29, row0=5, col0=11).numpy()
    assert np.max(np.abs(a - b) / np.maximum(np.abs(a), 1e-300)) < 8 * EPS


def test_normal_partition_invariant():
    full = oracle.normal(5, 0, 40, 64)
    part = oracle.normal(5, 0, 21, 17, row0=7, col0=30)
    assert np.array_equal(full[7:28, 30:47], part)


# ----------------------------------------------------------------------------
# O1 sketch
# ----------------------------------------------------------------------------
def test_sketch_closed_forms():
    """A = I -> B = Omega exactly; A = 0 -> B = 0."""
    om = oracle.omega(3, 12, 40)
    assert np.array_equal(oracle.sketch(om, np.eye(40)), om)
    assert np.array_equal(oracle.sketch(om, np.zeros((40, 7))), np.zeros((12, 7)))
    rng = np.random.default_rng(0)
    A = rng.standard_normal((40, 9))
    ref = om @ A  # library GEMM
    assert np.max(np.abs(oracle.sketch(om, A) - ref)) < 1e-13 * np.max(np.abs(ref))


# ----------------------------------------------------------------------------
# O3 sample QRCP = Alg. 1 on the sample
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(6))
def test_sample_qrcp_brute_force(seed):
    """Businger-Golub pivots equal the brute-force definition."""
    rng = np.random.default_rng(seed)
    l, nn, bb = 12, 30, 8
    B = rng.standard_normal((l, nn)) * rng.uniform(0.2, 3.0, nn)
    res = oracle.sample_qrcp(B, bb)
    assert res["steps"] == bb
    assert np.array_equal(res["perm"][:bb], brute_force_qrcp_pivots(B, bb))
    # R-hat: abs(diag) non-increasing, Q^T B Pi reproduced by a library QR
    d = np.abs(np.diag(res["R"][:bb, :bb]))
    assert np.all(d[:-1] >= d[1:] * (1 - 1e-12))
    _, Rl = np.linalg.qr(B[:, res["perm"]])
    assert np.allclose(np.abs(np.diag(Rl))[:bb], d, rtol=1e-13)
    # upper triangle rows of R-hat vs library R up to row signs
    s = np.sign(np.diag(Rl)[:bb]) * np.sign(np.diag(res["R"])[:bb])
    assert np.allclose(res["R"][:bb, :], Rl[:bb, :] * s[:, None], atol=1e-13 * np.abs(Rl).max())


def test_sample_qrcp_example_diag():
    """diag(5,4,3,2,1) padded to 8x5 -> first three pivots are the
    three largest columns (deterministic QRCP on the sample itself)."""
    A = np.zeros((8, 5))
    A[:5, :5] = np.diag([5.0, 4, 3, 2, 1])
    res = oracle.sample_qrcp(A, 3)
    assert list(res["perm"][:3]) == [0, 1, 2]
    assert np.allclose(np.abs(np.diag(res["R"][:3, :3])), [5, 4, 3])


# ----------------------------------------------------------------------------
# Whole oracle, QRCP mode (Omega = I or Haar, l = m): reduces to LAPACK dgeqp3
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("m,n,k,b,seed", [(60, 60, 24, 8, 0), (70, 50, 29, 8, 1), (45, 80, 45, 16, 2),
                                          (64, 64, 64, 5, 3)])
def test_omega_identity_equals_dgeqp3(m, n, k, b, seed):
    rng = np.random.default_rng(seed)
    A, _ = graded_matrix(rng, m, n, 2.0 ** (1.0 / 3.0))
    res = oracle.rqrcp(A, k, b, m - b, omega=np.eye(m))
    _, R2, P = sl.qr(A, pivoting=True)
    assert res["rank"] == k
    assert np.array_equal(res["jpvt"][:k], P[:k])
    dR = np.abs(np.diag(full_R(res, k)))[:k]
    assert np.max(np.abs(dR - np.abs(np.diag(R2))[:k]) / np.abs(np.diag(R2))[:k]) < 1e-13


def test_omega_haar_equals_dgeqp3():
    rng = np.random.default_rng(7)
    m = n = 60
    A, _ = graded_matrix(rng, m, n, 1.3)
    H = inputs.haar(11, 1, m).numpy()
    res = oracle.rqrcp(A, 24, 8, m - 8, omega=H)
    _, _, P = sl.qr(A, pivoting=True)
    assert np.array_equal(res["jpvt"][:24], P[:24])


def test_qrcp_dominance_lemma():
    """Lemma: |r_ii| >= ||R(i:m, j)|| for j > i, exact for QRCP
    (Omega = I mode), 1e-10 relative slack."""
    rng = np.random.default_rng(3)
    m, n, k, b = 50, 40, 30, 8
    A = rng.standard_normal((m, n))
    res = oracle.rqrcp(A, k, b, m - b, omega=np.eye(m))
    R = full_R(res, k)
    for i in range(k):
        tail = np.linalg.norm(R[i:, i + 1:], axis=0)
        assert np.all(abs(R[i, i]) >= tail * (1 - 1e-10))


# ----------------------------------------------------------------------------
# Paper-printed values: Kahan matrix, Tables I and II
# ----------------------------------------------------------------------------
# Printed values have 4 significant digits; "agree" = within half a unit of
# the 4th digit plus rounding of the print (5e-4 relative).
def _kahan(n):
    return inputs.kahan(n).numpy()


def test_kahan_table1_qrcp_column(golden):
    """QRCP = RQRCP with Omega = I: no interchanges on Kahan and the
    residuals of Table I's QRCP column to 4 digits."""
    for n, k, _, qrcp in golden("kahan_table1.txt"):
        n, k = int(n), int(k)
        K = _kahan(n)
        res = oracle.rqrcp(K, k, 64, n - 64, omega=np.eye(n))
        assert np.array_equal(res["jpvt"], np.arange(n))
        r = abs(res["A"][n - 1, n - 1]) / np.linalg.norm(K)
        assert abs(r - float(qrcp)) <= 5e-4 * float(qrcp), (n, r, qrcp)


def _left_out_closed_form(K, j):
    """k = n-1 leaves a 1x1 R22: |R22| = dist(col j, span(others)) = 1/||e_j^T K^-1||."""
    Kinv = sl.solve_triangular(K, np.eye(K.shape[0]))
    return 1.0 / np.linalg.norm(Kinv[j, :])


def test_kahan_table1_rqrcp_column(golden):
    """Table I "SRQR" column = the hot path itself, RQRCP with
    b = 64, p = 10, whenever it leaves out column 0;
    for every seed |R22| equals the closed form of the left-out column."""
    for n, k, srqr, _ in golden("kahan_table1.txt"):
        n, k = int(n), int(k)
        K = _kahan(n)
        hits = 0
        for seed in range(4):
            res = oracle.rqrcp(K, k, 64, 10, seed=seed)
            j = int(res["jpvt"][n - 1])
            r22 = abs(res["A"][n - 1, n - 1])
            cf = _left_out_closed_form(K, j)
            assert abs(r22 - cf) <= 1e-8 * cf, (n, seed, r22, cf)
            if j == 0:
                hits += 1
                r = r22 / np.linalg.norm(K)
                assert abs(r - float(srqr)) <= 5e-4 * float(srqr), (n, r, srqr)
        assert hits >= 1


def test_kahan_table2(golden):
    """Table II: sigma_j(R11)/sigma_j(A) at n = 192, k = 191."""
    n, k = 192, 191
    K = _kahan(n)
    sA = np.linalg.svd(K, compute_uv=False)
    qr = oracle.rqrcp(K, k, 64, n - 64, omega=np.eye(n))
    rq = oracle.rqrcp(K, k, 64, 10, seed=0)
    s_qr = np.linalg.svd(np.triu(qr["A"][:k, :k]), compute_uv=False)
    s_rq = np.linalg.svd(np.triu(rq["A"][:k, :k]), compute_uv=False)
    for j, srqr, qrcp in golden("kahan_table2.txt"):
        j = int(j)
        ratio_rq = s_rq[j - 1] / sA[j - 1]
        assert abs(ratio_rq - float(srqr)) < 5e-4, (j, ratio_rq)
        ratio_qr = s_qr[j - 1] / sA[j - 1]
        if j < 191:
            assert abs(ratio_qr - float(qrcp)) <= 1e-4, (j, ratio_qr)
        else:
            assert ratio_qr <= 1e-10


def test_oversampling_bound(golden):
    """Theorem 2 with the printed example p >= 508."""
    for n, k, e, d, p in golden("oversampling.txt"):
        assert oracle.min_oversampling(int(n), int(k), float(e), float(d)) == int(p)
    assert oracle.min_oversampling(1000, 200, 0.5, 0.1) <= oracle.min_oversampling(1000, 200, 0.5, 0.05)


# ----------------------------------------------------------------------------
# Gaussian Omega, tiny well-separated matrices
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("orthogonal", [False, True])
def test_well_separated_equals_qrcp(orthogonal):
    """Column norms in ratio 10: RQRCP with Gaussian Omega picks the QRCP
    pivots (dgeqp3 and brute force) for every seed; for orthogonal columns
    |R11| = diag(d sorted descending) in closed form."""
    m, n, k, b, p = 40, 30, 12, 4, 4
    for seed in range(25):
        rng = np.random.default_rng(100 + seed)
        d = 10.0 ** (-rng.permutation(n).astype(np.float64))
        if orthogonal:
            U, _ = np.linalg.qr(rng.standard_normal((m, n)))
            A = U * d
        else:
            A = rng.standard_normal((m, n)) * d
        res = oracle.rqrcp(A, k, b, p, seed=seed)
        _, _, P = sl.qr(A, pivoting=True)
        assert np.array_equal(res["jpvt"][:k], P[:k])
        assert np.array_equal(res["jpvt"][:k], brute_force_qrcp_pivots(A, k))
        if orthogonal:
            R11 = np.triu(res["A"][:k, :k])
            ds = np.sort(d)[::-1][:k]
            assert np.allclose(np.abs(np.diag(R11)), ds, rtol=1e-14, atol=0)
            off = R11 - np.diag(np.diag(R11))
            assert np.all(np.abs(off) <= 1e-14 * ds[:, None] + 1e-15 * ds[0])


# ----------------------------------------------------------------------------
# Panel + trailing update: reconstruction, orthogonality, library R
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("m,n,k,b,p", [(120, 90, 40, 16, 8), (90, 150, 50, 12, 5), (200, 200, 64, 32, 8)])
def test_reconstruction_and_orthogonality(m, n, k, b, p):
    rng = np.random.default_rng(m + n)
    A = rng.standard_normal((m, n)) * np.exp(-np.arange(n) / 30.0)
    res = oracle.rqrcp(A, k, b, p, seed=5)
    Api = A[:, res["jpvt"]]
    R = full_R(res, k)
    QR = oracle.apply_q(res["A"], res["tau"], R)
    assert np.linalg.norm(Api - QR) <= 100 * EPS * np.linalg.norm(A)
    Q = oracle.apply_q(res["A"], res["tau"], np.eye(m))
    assert np.linalg.norm(Q.T @ Q - np.eye(m)) <= 10 * m * EPS
    # R11/R12 = Householder QR of A Pi up to row signs (library routine)
    _, Rl = np.linalg.qr(Api[:, :k], mode="complete")
    Ql, _ = np.linalg.qr(Api[:, :k], mode="complete")
    R12l = Ql.T @ Api[:, k:]
    sgn = np.sign(np.diag(Rl)[:k]) * np.sign(np.diag(R)[:k])
    top = np.hstack([Rl[:k, :k], R12l[:k]]) * sgn[:, None]
    assert np.max(np.abs(R[:k] - top)) <= 1e-13 * np.abs(R[:k]).max()
    # truncated residual two ways: ||R22||_F vs ||A Pi - Q1 [R11 R12]||_F
    Rt = R.copy()
    Rt[k:, :] = 0.0
    r1 = np.linalg.norm(R[k:, k:]) / np.linalg.norm(A)
    r2 = np.linalg.norm(Api - oracle.apply_q(res["A"], res["tau"], Rt)) / np.linalg.norm(A)
    assert abs(r1 - r2) <= 1e-12


def test_exact_rank_recovery():
    """300x300 rank-40 product of Gaussians, k=40, b=32, p=10."""
    rng = np.random.default_rng(41)
    A = rng.standard_normal((300, 40)) @ rng.standard_normal((40, 300))
    res = oracle.rqrcp(A, 40, 32, 10, seed=2)
    assert np.linalg.norm(full_R(res, 40)[40:, 40:]) / np.linalg.norm(A) <= 1e-10


def test_rank_deficient_stops(tmp_path):
    """Reading G12: early stop with the achieved rank."""
    rng = np.random.default_rng(42)
    A = rng.standard_normal((120, 25)) @ rng.standard_normal((25, 100))
    res = oracle.rqrcp(A, 60, 16, 8, seed=1)
    assert res["rank"] == 25
    assert np.all(res["tau"][25:] == 0.0)
    assert sorted(res["jpvt"]) == list(range(100))
    z = oracle.rqrcp(np.zeros((30, 20)), 5, 4, 2, seed=1)
    assert z["rank"] == 0 and np.array_equal(z["jpvt"], np.arange(20))


def test_errors():
    A = np.ones((10, 8))
    A[3, 2] = np.nan
    assert oracle.rqrcp(A, 4, 2, 2, check=False)["status"] == 4
    B = np.ones((10, 8))
    assert oracle.rqrcp(B, 0, 2, 2, check=False)["status"] == -6
    assert oracle.rqrcp(B, 9, 2, 2, check=False)["status"] == -6
    assert oracle.rqrcp(B, 4, 0, 2, check=False)["status"] == -7
    assert oracle.rqrcp(B, 4, 4, 7, check=False)["status"] == -8
    assert oracle.rqrcp(B, 4, 4, -1, check=False)["status"] == -8


# ----------------------------------------------------------------------------
# Sample update
# ----------------------------------------------------------------------------
def _collect(A, k, b, p, seed, rule):
    snaps = []

    def cb(i, bb, l, mp, np_, Rhat, Bnext, OmCur, OmNew, Aa):
        snaps.append(dict(i=i, bb=bb, Rhat=Rhat, Bnext=Bnext, OmCur=OmCur, OmNew=OmNew, A=Aa))
    res = oracle.rqrcp(A, k, b, p, seed=seed, update_rule=rule, invariant=True, callback=cb)
    return res, snaps


@pytest.mark.parametrize("kind", ["decay", "lowrank"])
def test_fresh_sketch_invariant(kind):
    """The updated sample is a fresh sketch of the trailing matrix with the
    transformed Gaussian: B_next = Omega-hat_2 R22 (Eq. (4)
    = Omega-hat_2 R22); Omega-hat block upper triangular.
    Error normalised by the inputs of the formula (DESIGN.md R-G17)."""
    rng = np.random.default_rng(9)
    m = n = 160
    if kind == "decay":
        A = rng.standard_normal((m, n)) * np.exp(-np.arange(n) / 20.0)
    else:
        A = rng.standard_normal((m, 48)) @ rng.standard_normal((48, n)) / 7.0 + 1e-6 * rng.standard_normal((m, n))
    k, b, p = 48, 16, 8
    res, snaps = _collect(A, k, b, p, 3, 1)
    assert len(snaps) == 3
    for s in snaps:
        i, bb = s["i"], s["bb"]
        R22 = s["A"][i + bb:, i + bb:]
        R12 = s["A"][i:i + bb, i + bb:]
        Om2 = s["OmNew"][:, bb:]
        Om11 = s["OmNew"][:bb, :bb]
        pred = Om2 @ R22
        scale = (np.linalg.norm(s["Rhat"][:bb, bb:]) + np.linalg.norm(s["Rhat"][bb:, bb:])
                 + np.linalg.norm(Om11 @ R12))
        assert np.linalg.norm(s["Bnext"] - pred) <= 1e-12 * scale
        # Omega-hat_21 = 0
        assert np.linalg.norm(s["OmNew"][bb:, :bb]) <= 1e-13 * np.linalg.norm(s["OmNew"])
        # the sample entering this panel is OmegaCur times the trailing matrix
        # of the previous panel's output (checked on the first panel: B = Omega A)
    s0 = snaps[0]
    B0 = oracle.sketch(s0["OmCur"], A)
    assert np.linalg.norm(B0 - s0["OmCur"] @ A) <= 1e-13 * np.linalg.norm(B0)


@pytest.mark.parametrize("seed", range(8))
def test_formula4_formula5_identical_permutations(seed):
    """Eq. (4) and Eq. (5) produce identical permutations; residuals
    equal to 1e-10 relative; sample column norms agree (ST-1)."""
    rng = np.random.default_rng(seed)
    m, n = int(rng.integers(80, 200)), int(rng.integers(80, 200))
    A = rng.standard_normal((m, n)) * np.exp(-np.arange(n) / rng.uniform(10, 60))
    k, b, p = 40, 8, 6
    r1, s1 = _collect(A, k, b, p, seed, 1)
    r2, s2 = _collect(A, k, b, p, seed, 2)
    assert np.array_equal(r1["jpvt"], r2["jpvt"])
    e1 = np.linalg.norm(full_R(r1, k)[k:, k:])
    e2 = np.linalg.norm(full_R(r2, k)[k:, k:])
    assert abs(e1 - e2) <= 1e-10 * e1
    for a, c in zip(s1, s2):
        if a["Bnext"] is None:
            continue
        n1 = np.linalg.norm(a["Bnext"], axis=0)
        n2 = np.linalg.norm(c["Bnext"], axis=0)
        assert np.max(np.abs(n1 - n2) / n1) <= 1e-11


# ----------------------------------------------------------------------------
# Prefix property, singular-value bounds, determinism
# ----------------------------------------------------------------------------
def test_prefix_property():
    """RQRCP to k' (b | k') = first k' pivots and R rows of RQRCP to k
    (Omega does not depend on k): bitwise."""
    rng = np.random.default_rng(4)
    A = rng.standard_normal((150, 130)) * np.exp(-np.arange(130) / 25.0)
    a = oracle.rqrcp(A, 16, 8, 5, seed=8)
    c = oracle.rqrcp(A, 48, 8, 5, seed=8)
    assert np.array_equal(a["jpvt"][:16], c["jpvt"][:16])
    pa = np.argsort(a["jpvt"])
    pc = np.argsort(c["jpvt"])
    Ra, Rc = full_R(a, 16), full_R(c, 48)
    for col in range(130):
        assert np.array_equal(Ra[:16, pa[col]], Rc[:16, pc[col]])
    assert np.array_equal(a["tau"], c["tau"][:16])


def test_singular_value_bounds():
    """Interlacing and Eq. (6) with sigma(A) known by
    construction (C1 recipe at 256^2)."""
    m = n = 256
    k = 48
    j = np.arange(1, n + 1)
    sig = np.exp(-j / 20.0)
    A = inputs.svd_matrix(31, m, n, __import__("torch").tensor(sig)).numpy()
    res = oracle.rqrcp(A, k, 16, 8, seed=31)
    R = full_R(res, k)
    s11 = np.linalg.svd(R[:k, :k], compute_uv=False)
    st = np.linalg.svd(R[:k, :], compute_uv=False)
    r22 = np.linalg.norm(R[k:, k:], 2)
    sA = np.linalg.svd(A, compute_uv=False)  # = sig up to rounding
    assert np.allclose(sA[:k + 1], sig[:k + 1], rtol=1e-10)
    assert np.all(s11 <= st * (1 + 1e-12))
    assert np.all(st <= sA[:k] * (1 + 1e-12))
    assert r22 >= sA[k] * (1 - 1e-12)
    assert np.all(sA[:k] ** 2 <= (st ** 2 + r22 ** 2) * (1 + 1e-12))


def test_thread_count_independence():
    """bitwise identical results for any worker count."""
    rng = np.random.default_rng(12)
    A = rng.standard_normal((140, 120))
    prev = oracle.set_threads(1)
    try:
        a = oracle.rqrcp(A, 40, 16, 6, seed=3)
        oracle.set_threads(max(prev, 3))
        c = oracle.rqrcp(A, 40, 16, 6, seed=3)
    finally:
        oracle.set_threads(prev)
    assert np.array_equal(a["A"], c["A"]) and np.array_equal(a["jpvt"], c["jpvt"])
    assert np.array_equal(a["tau"], c["tau"])


def test_gaussian_omega_matches_explicit():
    """Passing the drawn Omega explicitly gives bitwise the same factorization
    (the generator is the only source of randomness)."""
    rng = np.random.default_rng(13)
    A = rng.standard_normal((70, 60))
    a = oracle.rqrcp(A, 20, 8, 4, seed=21)
    c = oracle.rqrcp(A, 20, 8, 4, omega=oracle.omega(21, 12, 70))
    assert np.array_equal(a["A"], c["A"])


# ----------------------------------------------------------------------------
# SRQR verification (Alg. 3 first half)
# ----------------------------------------------------------------------------
def _orth_cols(seed, m, n, ratio):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    d = ratio ** (-np.arange(n, dtype=np.float64))
    rng.shuffle(d)
    return U * d, np.sort(d)[::-1]


@pytest.mark.parametrize("seed", range(4))
def test_srqr_qrcp_mode_g1_is_one(seed):
    """for QRCP |alpha| is the largest trailing column norm, so g1 = 1.
    Omega = I_m makes Alg. 2 a QRCP (SURVEY ST-2); separated norms."""
    A, _ = graded_matrix(np.random.default_rng(seed), 60, 45, 1.7)
    m = A.shape[0]
    o = oracle.srqr_verify(A, 14, 7, m - 7, seed=seed, omega=np.eye(m))
    assert o["g1"] == 1.0


@pytest.mark.parametrize("omega_identity", [True, False])
def test_srqr_orthogonal_columns_closed_form(omega_identity):
    """Orthonormal columns scaled by well-separated d: R-hat = diag(d_1..d_{k+1})
    up to signs, |alpha| = d_{k+1}, so g1 = 1 and g2 = |alpha| max 1/d_i = 1."""
    A, ds = _orth_cols(3, 70, 50, 10.0 ** 0.5)
    m, k, b = 70, 15, 5
    p = m - b if omega_identity else 6
    o = oracle.srqr_verify(A, k, b, p, seed=2, omega=np.eye(m) if omega_identity else None)
    assert o["g1"] == pytest.approx(1.0, abs=1e-12)
    assert o["g2_exact"] == pytest.approx(1.0, rel=1e-10)
    assert o["alpha"] == pytest.approx(ds[k], rel=1e-12)


def test_srqr_kahan_pathology():
    """g2 'can be exceptionally large for contrived pathological
    matrices' -- the Kahan matrix under QRCP (identity pivots, Table I) -- and
    stays below the QRCP bound g2 <= 2^l; RQRCP's random pivots give a
    modest g2 on the same matrix (Table I 'SRQR' residuals)."""
    n = 96
    K = inputs.kahan(n).numpy()
    oq = oracle.srqr_verify(K, n - 1, 64, n - 64, seed=1, omega=np.eye(n))
    assert oq["g2_exact"] > 1e6
    assert oq["g2_exact"] <= 2.0 ** n
    for seed in range(3):
        orr = oracle.srqr_verify(K, n - 1, 64, 10, seed=seed)
        assert orr["g2_exact"] < 10.0


def test_srqr_estimator_statistics():
    """The d-row Gaussian estimate of g2 against the exact value:
    within a factor 3 in >= 95% of 60 seeds (d = 8)."""
    A = inputs.make("svd_exp", 120, 90, 4).numpy()
    ok = 0
    for seed in range(60):
        o = oracle.srqr_verify(A, 20, 10, 6, seed=seed, d=8)
        r = o["g2_est"] / o["g2_exact"]
        ok += (1.0 / 3.0 <= r <= 3.0)
    assert ok >= 57


@pytest.mark.parametrize("seed", range(3))
def test_srqr_tau_caps(seed):
    """Eqs. (9)-(12) with exact quantities: tau = g1 g2 (||R22||_2/||R22||_{1,2})
    (||R-hat^{-T}||_{1,2}^{-1}/sigma_{l+1}(A)) <= g1 g2 sqrt((l+1)(n-l)) and
    tau-hat <= g1 g2 sqrt(l (n-l)), l = k."""
    A = inputs.make("svd_exp", 100, 80, 10 + seed).numpy()
    k = 16
    o = oracle.srqr_verify(A, k, 8, 6, seed=seed)
    F = o["res"]["A"]
    m, n = F.shape
    R22 = F[k:, k:]
    c12 = np.max(np.linalg.norm(R22, axis=0))
    s22 = np.linalg.norm(R22, 2)
    sA = np.linalg.svd(A, compute_uv=False)
    g1, g2 = o["g1"], o["g2_exact"]
    rinv_12 = g2 / o["alpha"]   # ||R-hat^{-T}||_{1,2}
    tau = g1 * g2 * (s22 / c12) * (1.0 / rinv_12) / sA[k]
    assert s22 == pytest.approx(tau * sA[k], rel=1e-12)          # Eq. (9) as an identity
    assert tau <= g1 * g2 * np.sqrt((k + 1) * (n - k)) * (1 + 1e-12)  # Eq. (10)
    R11 = np.triu(F[:k, :k])
    r11inv_12 = np.max(np.linalg.norm(np.linalg.inv(R11), axis=1))  # ||R11^{-T}||_{1,2}
    Rt = np.triu(F[:k, :])
    s_l = np.linalg.svd(Rt, compute_uv=False)[k - 1]
    tau_hat = g1 * g2 * (s22 / c12) * (1.0 / r11inv_12) / s_l
    assert tau_hat <= g1 * g2 * np.sqrt(k * (n - k)) * (1 + 1e-12)  # Eq. (12)


# ----------------------------------------------------------------------------
# R11-diagonal rank stop (reading R-G12b) and the tie rule (R-G5)
# ----------------------------------------------------------------------------
def test_r11_diagonal_stop_closed_form():
    """Column 5 of A is 1e-15 e_5 but Omega amplifies row 5 by 1e17: the sample
    QRCP picks it as the second pivot; |R(1,1)| = 1e-15 is below
    1e3 eps ||panel||_F (~ 4.4e-11 here), so the factorization stops at rank 1
    with tau = 0 from there on, R(0,0) = +200 (dlarfg on 200 e_0: x(1:) = 0
    gives tau = 0 and beta = alpha, reading R-G7), and the untouched column 5
    still holds its input value below the stop."""
    m, n, b, p = 40, 30, 8, 2
    A = np.zeros((m, n))
    for j in range(n):
        A[j, j] = 1.0
    A[5, 5] = 1e-15
    A[:, 0] *= 200.0
    Om = np.random.default_rng(11).standard_normal((b + p, m))
    Om[:, 5] *= 1e17
    o = oracle.rqrcp(A, 16, b, p, omega=Om, check=False)
    assert o["status"] == 0
    assert o["rank"] == 1
    assert o["jpvt"][0] == 0 and o["jpvt"][1] == 5
    assert o["A"][0, 0] == 200.0
    assert np.all(o["tau"] == 0.0)
    assert o["A"][5, 1] == 1e-15  # column 5 (now at position 1) untouched: H_0 = I on it


def test_r11_stop_not_triggered_on_full_rank():
    """Well-conditioned inputs never trip the R11-diagonal stop."""
    A = inputs.iid(3, 200, 150).numpy()
    o = oracle.rqrcp(A, 100, 16, 8, seed=2)
    assert o["rank"] == 100


def test_tie_rule_lowest_position():
    """Bitwise-identical columns tie in the squared sample norms; the lowest
    current position wins (reading R-G5).  Every column is duplicated, so
    the pivots are the even (first) members of the pairs."""
    rng = np.random.default_rng(8)
    X = rng.standard_normal((300, 60)) * np.exp(-np.arange(60) / 10.0)
    A = np.repeat(X, 2, axis=1)
    o = oracle.rqrcp(A, 16, 8, 4, seed=9, check=False)
    assert np.all(o["jpvt"][:16] % 2 == 0)
    q = oracle.sample_qrcp(np.repeat(np.eye(4)[:, :2] * [2.0, 1.0], 2, axis=1), 1)
    assert q["piv"][0] == 0  # columns 0 and 1 identical: position 0 wins


def test_householder_convention_matches_lapack():
    """Reading R-G7 pinned to LAPACK: with the oracle's pivots, the oracle's
    V, tau and R equal dgeqrf on A Pi (same dlarfg convention) to rounding."""
    from scipy.linalg import lapack
    A = inputs.iid(12, 120, 90).numpy()
    o = oracle.rqrcp(A, 90, 16, 8, seed=4)
    Api = np.asfortranarray(A[:, o["jpvt"]])
    qr, tau, work, info = lapack.dgeqrf(Api)
    assert info == 0
    F = o["A"]
    assert np.max(np.abs(np.triu(F[:90]) - np.triu(qr[:90]))) <= 1e-12 * np.max(np.abs(qr))
    assert np.max(np.abs(o["tau"] - tau[:90])) <= 1e-12
    assert np.max(np.abs(np.tril(F[:, :90], -1) - np.tril(qr[:, :90], -1))) <= 1e-12


# ----------------------------------------------------------------------------
# Tournament pivoting on the sample (reading R-TP): the oracle variant
# ----------------------------------------------------------------------------
def brute_force_tournament(B, i, b, groups, bb):
    """The tournament of reading R-TP from its definition, with the
    brute-force greedy selector (norms recomputed from scratch by a library
    QR each step, brute_force_qrcp_pivots): groups by the block-cyclic layout,
    local selections, pairwise merges up the tree (left list, then right list)."""
    n = B.shape[1]
    cand = []
    for g in range(groups):
        idx = [c for c in range(n) if ((i + c) // b) % groups == g]
        sel = brute_force_qrcp_pivots(B[:, idx], min(bb, len(idx))) if idx else []
        cand.append([idx[s] for s in sel])
    span = 1
    while span < groups:
        for g in range(0, groups - span, 2 * span):
            u = cand[g] + cand[g + span]
            sel = brute_force_qrcp_pivots(B[:, u], min(bb, len(u))) if u else []
            cand[g] = [u[s] for s in sel]
        span *= 2
    return cand[0]


def test_tournament_one_group_is_alg1():
    """One group: the tournament is Alg. 1 itself -- bitwise the same factorization."""
    A = inputs.make("iid", 300, 280, 3).numpy()
    o0 = oracle.rqrcp(A, 96, 32, 8, seed=4)
    o1 = oracle.rqrcp(A, 96, 32, 8, seed=4, tournament=1)
    assert np.array_equal(o0["A"], o1["A"]) and np.array_equal(o0["jpvt"], o1["jpvt"])


@pytest.mark.parametrize("groups", [2, 3, 4, 7])
def test_tournament_matches_brute_force(groups):
    """The oracle's tournament (per panel, on the sample it sees) equals the
    brute-force tournament of the definition on the same sample, for tiny
    generic inputs (distinct residual norms); two panels."""
    for seed in range(6):
        rng = np.random.default_rng(700 + 10 * groups + seed)
        m, n, b, p = 48, 40, 6, 4
        A = rng.standard_normal((m, n)) * np.exp(-rng.permutation(n) / 8.0)
        samples = []
        res = oracle.rqrcp(A, 2 * b, b, p, seed=seed, tournament=groups, invariant=True,
                           callback=lambda i, bb, l_, mp, np_, Rh, Bn, Oc, On, Af: samples.append((i, bb, Bn)))
        # panel 0 works on the initial sample Omega A
        B0 = oracle.sketch(oracle.omega(seed, b + p, m), A)
        assert list(res["jpvt"][:b]) == brute_force_tournament(B0, 0, b, groups, b)
        # panel 1 works on panel 0's updated sample, positions relative to column b
        # of A Pi after panel 0 (whose order the one-panel run gives)
        one = oracle.rqrcp(A, b, b, p, seed=seed, tournament=groups)
        sel1 = brute_force_tournament(samples[0][2], b, b, groups, b)
        assert list(res["jpvt"][b:2 * b]) == [int(one["jpvt"][b + c]) for c in sel1]


@pytest.mark.parametrize("groups", [2, 3, 4, 8])
def test_tournament_separated_equals_qrcp(groups):
    """Orthogonal columns with norms in ratio 10 (ST-9): every local and merged
    selection keeps the largest columns, so the tournament gives the QRCP
    (dgeqp3) pivots and |R11| = diag(d sorted descending)."""
    m, n, k, b, p = 60, 48, 16, 4, 4
    for seed in range(10):
        rng = np.random.default_rng(300 + seed)
        d = 10.0 ** (-rng.permutation(n).astype(np.float64) / 2.0)
        U, _ = np.linalg.qr(rng.standard_normal((m, n)))
        A = U * d
        res = oracle.rqrcp(A, k, b, p, seed=seed, tournament=groups)
        _, _, P = sl.qr(A, pivoting=True)
        assert np.array_equal(res["jpvt"][:k], P[:k])
        assert np.allclose(np.abs(np.diag(res["A"])[:k]), np.sort(d)[::-1][:k], rtol=1e-13, atol=0)


@pytest.mark.parametrize("groups", [2, 4])
def test_tournament_invariants(groups):
    """Whatever the pivots, Alg. 2's algebra holds: A Pi = Q R to 100 eps,
    Q orthogonal, R-hat = the QR of the sample in the chosen order (up to row
    signs), and the fresh-sketch invariant of Eq. (4)."""
    rng = np.random.default_rng(77)
    m, n, k, b, p = 140, 120, 48, 16, 8
    A = rng.standard_normal((m, n)) * np.exp(-np.arange(n) / 25.0)
    snaps = []
    res = oracle.rqrcp(A, k, b, p, seed=6, tournament=groups, invariant=True,
                       callback=lambda i, bb, l_, mp, np_, Rh, Bn, Oc, On, Af:
                       snaps.append(dict(i=i, bb=bb, Rhat=Rh, Bnext=Bn, OmCur=Oc, OmNew=On, A=Af)))
    Api = A[:, res["jpvt"]]
    R = full_R(res, k)
    assert np.linalg.norm(Api - oracle.apply_q(res["A"], res["tau"], R)) <= 100 * EPS * np.linalg.norm(A)
    Q = oracle.apply_q(res["A"], res["tau"], np.eye(m))
    assert np.linalg.norm(Q.T @ Q - np.eye(m)) <= 10 * m * EPS
    # panel 0: R-hat11 = the R factor of the initial sample's chosen columns
    B0 = oracle.sketch(oracle.omega(6, b + p, m), A)
    Rl = np.linalg.qr(B0[:, res["jpvt"][:b]])[1]
    assert np.max(np.abs(np.abs(snaps[0]["Rhat"][:b, :b]) - np.abs(Rl))) <= 1e-12 * np.abs(Rl).max()
    for s in snaps:
        i, bb = s["i"], s["bb"]
        R22 = s["A"][i + bb:, i + bb:]
        R12 = s["A"][i:i + bb, i + bb:]
        pred = s["OmNew"][:, bb:] @ R22
        scale = (np.linalg.norm(s["Rhat"][:bb, bb:]) + np.linalg.norm(s["Rhat"][bb:, bb:])
                 + np.linalg.norm(s["OmNew"][:bb, :bb] @ R12))
        if s["Bnext"] is not None:
            assert np.linalg.norm(s["Bnext"] - pred) <= 1e-12 * scale
