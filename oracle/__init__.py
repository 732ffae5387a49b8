"""CPU oracle for the RQRCP hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(paper_1804_05138_b200/) never imports it and shares no code with it.

Thin ctypes wrapper over oracle/rqrcp_oracle.c (plain unblocked C, fp64,
OpenMP only across independent columns).  See that file's header for the
passages of PAPER.md each step follows.  Parity status per function is listed
in DESIGN.md ("Oracle pins"); every function exported here is pinned by a
``-m "not gpu"`` test in tests/test_oracle_*.py.

Helper formulas of the paper that are not part of Alg. 2 itself
(Theorem 2's oversampling bound) are also here, written from the paper.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rqrcp_oracle.c")
_LIB_PATH = os.path.join(_HERE, "librqrcp_oracle.so")
_lib = None
_lock = threading.Lock()

ORACLE_INVARIANT = 1


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2, OpenMP, no FMA contraction)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared",
                               "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


PANEL_CB = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                            ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            i64, dp, vp = ctypes.c_int64, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p
            L.oracle_philox4x32_10.argtypes = [ctypes.POINTER(ctypes.c_uint32)] * 3
            L.oracle_normal_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint32, i64, i64, i64, i64, dp, i64]
            L.oracle_sketch.argtypes = [i64, i64, i64, dp, i64, dp, i64, dp, i64]
            L.oracle_sample_qrcp.argtypes = [i64, i64, i64, dp, i64, ctypes.POINTER(i64), dp, ctypes.c_double, dp]
            L.oracle_sample_qrcp.restype = i64
            L.oracle_rqrcp.argtypes = [i64, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, vp,
                                       ctypes.c_int, ctypes.c_int, dp, i64, ctypes.POINTER(i64), dp,
                                       ctypes.POINTER(i64), vp, PANEL_CB, vp]
            L.oracle_rqrcp.restype = ctypes.c_int
            L.oracle_rqrcp_tp.argtypes = [i64, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, vp,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, i64, ctypes.POINTER(i64), dp,
                                          ctypes.POINTER(i64), vp, PANEL_CB, vp]
            L.oracle_rqrcp_tp.restype = ctypes.c_int
            L.oracle_set_threads.argtypes = [ctypes.c_int]
            L.oracle_set_threads.restype = ctypes.c_int
            _lib = L
    return _lib


def set_threads(n: int) -> int:
    """Set the oracle's OpenMP thread count; returns the previous one."""
    return int(lib().oracle_set_threads(int(n)))


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64f(a) -> np.ndarray:
    """Column-major float64 copy (accepts numpy or torch)."""
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.array(a, dtype=np.float64, order="F", copy=True)


def philox4x32_10(ctr, key):
    c = (ctypes.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (ctypes.c_uint32 * 4)()
    lib().oracle_philox4x32_10(c, k, o)
    return tuple(int(x) for x in o)


def normal(seed: int, stream: int, rows: int, cols: int, row0: int = 0, col0: int = 0) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float64, order="F")
    lib().oracle_normal_fill(seed, stream, row0, rows, col0, cols, _dp(out), max(rows, 1))
    return out


def omega(seed: int, l: int, m: int) -> np.ndarray:
    """The l x m sketch Omega the oracle draws (stream 0), as in Alg. 2 P:143."""
    return normal(seed, 0, l, m)


def sketch(Omega, A) -> np.ndarray:
    Om, A = _f64f(Omega), _f64f(A)
    l, m = Om.shape
    m2, n = A.shape
    assert m == m2
    B = np.empty((l, n), dtype=np.float64, order="F")
    lib().oracle_sketch(l, m, n, _dp(Om), max(l, 1), _dp(A), max(m, 1), _dp(B), max(l, 1))
    return B


def sample_qrcp(B, bb: int, stop_tol2: float = 0.0):
    """bb steps of Businger-Golub QRCP (Alg. 1) on B; returns dict with
    'R' (transformed B, reflectors zeroed), 'piv' (transpositions),
    'perm' (resulting column order), 'tau', 'steps', 'gaps'."""
    Bw = _f64f(B)
    l, nn = Bw.shape
    piv = np.zeros(max(bb, 1), dtype=np.int64)
    tauh = np.zeros(max(bb, 1), dtype=np.float64)
    gaps = np.zeros(max(bb, 1), dtype=np.float64)
    steps = lib().oracle_sample_qrcp(l, nn, bb, _dp(Bw), max(l, 1),
                                     piv.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dp(tauh),
                                     stop_tol2, _dp(gaps))
    perm = np.arange(nn)
    for j in range(max(steps, 0)):
        s = piv[j]
        perm[j], perm[s] = perm[s], perm[j]
    R = Bw.copy(order="F")
    for j in range(max(steps, 0)):
        R[j + 1:, j] = 0.0
    return dict(R=R, V=Bw, piv=piv[:max(steps, 0)], perm=perm, tau=tauh[:max(steps, 0)], steps=steps,
                gaps=gaps[:max(steps, 0)])


class OracleError(RuntimeError):
    pass


def rqrcp(A, k: int, b: int, p: int, seed: int = 0, omega=None, update_rule: int = 1,
          invariant: bool = False, callback=None, check: bool = True, tournament: int = 0):
    """Alg. 2 on a copy of A.  Returns dict(A=factored (LAPACK layout),
    jpvt, tau, rank, gaps, status).

    callback(i, bb, l, mp, np_, Rhat, Bnext, OmegaCur, OmegaNew, A) receives
    numpy copies per panel (tests only; see rqrcp_oracle.c).
    tournament = G > 1: the pivots of each panel from tournament pivoting on
    the sample over G block-cyclic column groups (rqrcp_oracle.c)."""
    Af = _f64f(A)
    m, n = Af.shape
    l = b + p
    om = None
    if omega is not None:
        om = _f64f(omega)
        assert om.shape == (l, m), (om.shape, l, m)
    jpvt = np.zeros(n, dtype=np.int64)
    tau = np.zeros(max(k, 1), dtype=np.float64)
    rank = ctypes.c_int64(0)
    gaps = np.ones(max(k, 1), dtype=np.float64)

    def _cb(user, i, bb, l_, mp, np_, Rhat, Bnext, OmCur, OmNew, Aptr, lda):
        def arr(ptr, r, c, ld):
            if not ptr or r * c == 0:
                return None
            buf = (ctypes.c_double * (ld * (c - 1) + r)).from_address(ptr)
            a = np.frombuffer(buf, dtype=np.float64, count=ld * (c - 1) + r)
            return np.lib.stride_tricks.as_strided(a, shape=(r, c), strides=(8, 8 * ld)).copy(order="F")
        callback(int(i), int(bb), int(l_), int(mp), int(np_), arr(Rhat, l_, np_, l_),
                 arr(Bnext, l_, np_ - bb, l_), arr(OmCur, l_, mp, l_), arr(OmNew, l_, mp, l_),
                 arr(Aptr, m, n, lda))

    cbp = PANEL_CB(_cb) if callback is not None else PANEL_CB()
    flags = ORACLE_INVARIANT if invariant else 0
    st = lib().oracle_rqrcp_tp(m, n, k, b, p, seed, om.ctypes.data if om is not None else None, update_rule, flags,
                               int(tournament), _dp(Af), max(m, 1), jpvt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                               _dp(tau), ctypes.byref(rank), gaps.ctypes.data, cbp, None)
    if check and st != 0:
        raise OracleError(f"oracle_rqrcp returned {st}")
    return dict(A=Af, jpvt=jpvt, tau=tau[:k], rank=int(rank.value), gaps=gaps[:k], status=st)


# ---------------------------------------------------------------------------
# Post-processing helpers written from the definitions (not from the C code)
# ---------------------------------------------------------------------------
def apply_q(Af: np.ndarray, tau: np.ndarray, X: np.ndarray, transpose: bool = False) -> np.ndarray:
    """Q X (or Q^T X) with Q = H_1 ... H_k from the LAPACK-layout reflectors
    ("Q = H1 H2 ... Hk")."""
    m = Af.shape[0]
    k = len(tau)
    Y = np.array(X, dtype=np.float64, copy=True)
    order = range(k) if transpose else range(k - 1, -1, -1)
    for j in order:
        v = np.zeros(m)
        v[j] = 1.0
        v[j + 1:] = Af[j + 1:, j]
        Y -= tau[j] * np.outer(v, v @ Y)
    return Y


def r_factor(Af: np.ndarray, k: int) -> np.ndarray:
    """[R11 R12] (k x n): upper trapezoid of the top k rows."""
    return np.triu(Af[:k, :])


def min_oversampling(n: int, k: int, eps: float, delta: float) -> int:
    """Theorem 2: p >= ceil(4/(eps^2 - eps^3) log(2nk/Delta)) - 1,
    natural log (reading G16)."""
    if not (0 < eps < 1 and 0 < delta < 1):
        raise ValueError("eps, delta must lie in (0,1)")
    return int(math.ceil(4.0 / (eps ** 2 - eps ** 3) * math.log(2.0 * n * k / delta))) - 1


# ---------------------------------------------------------------------------
# SRQR verification (Alg. 3, first half)
# ---------------------------------------------------------------------------
SRQR_STREAM = 7  # Philox stream of the d x (l+1) Gaussian of the g2 estimate


def srqr_verify(A, k: int, b: int, p: int, seed: int = 0, d: int = 8, omega=None, update_rule: int = 1):
    """Alg. 3's verification on top of Alg. 2 run to rank k (the paper's l):

    * the sample after the LAST panel's update (reading G9: kept here) gives
      r_i = ||B(:, i)||^2 / (b + p) for the trailing columns;
    * iota = argmax r_i (lowest position on ties, reading G5); columns k and
      k + iota of A and Pi are swapped;
    * one QR step on A(k:m, k:n): |alpha| = ||A(k:m, k)||;
    * g1 = ||R22||_{1,2} / |alpha| (Eq. 8), R22 = A(k:m, k:n);
    * R-hat = [[R11, a], [0, alpha]] and
      g2 ~= |alpha| / sqrt(d) ||Omega_d R-hat^{-T}||_{1,2} with Omega_d a
      d x (k+1) N(0,1) matrix, formed by d triangular solves;
      also the exact g2 = |alpha| ||R-hat^{-T}||_{1,2} (Eq. 8);
    * the tau caps of Eqs. (10) and (12): g1 g2 sqrt((l+1)(n-l)) and
      g1 g2 sqrt(l(n-l)), with l = k.
    Returns a dict (the factorization after the swap under 'res')."""
    import scipy.linalg as sla
    state = {}

    def cb(i, bb, l_, mp, np_, Rhat, Bnext, OmCur, OmNew, Af):
        state["Bnext"] = Bnext

    res = rqrcp(A, k, b, p, seed=seed, omega=omega, update_rule=update_rule, invariant=True, callback=cb)
    F = res["A"]
    jpvt = res["jpvt"]
    m, n = F.shape
    out = dict(res=res, k=k, d=d)
    if k >= n or k >= m or state.get("Bnext") is None:
        out.update(g1=0.0, g2_est=0.0, g2_exact=0.0, alpha=0.0, pivot=-1, tau_bound=0.0, tau_hat_bound=0.0)
        return out
    B = state["Bnext"]                   # l x (n - k): the sample of R22
    r = np.zeros(B.shape[1])
    for c in range(B.shape[1]):          # ascending sums of squares
        s = 0.0
        for t in range(B.shape[0]):
            s += B[t, c] * B[t, c]
        r[c] = s / (b + p)
    iota = int(np.argmax(r))             # first (lowest) index on exact ties
    if iota != 0:
        F[:, [k, k + iota]] = F[:, [k + iota, k]]
        jpvt[[k, k + iota]] = jpvt[[k + iota, k]]
    colnorm = np.sqrt(np.sum(F[k:, k:] ** 2, axis=0))
    alpha = float(colnorm[0])
    g1 = float(np.max(colnorm) / alpha) if alpha > 0 else float("inf")
    Rh = np.zeros((k + 1, k + 1))
    Rh[:k, :k] = np.triu(F[:k, :k])
    Rh[:k, k] = F[:k, k]
    Rh[k, k] = alpha
    Od = normal(seed, SRQR_STREAM, d, k + 1)
    Y = sla.solve_triangular(Rh, Od.T, lower=False)      # R-hat^{-1} Omega_d^T = (Omega_d R-hat^{-T})^T
    g2_est = alpha / math.sqrt(d) * float(np.max(np.sqrt(np.sum(Y * Y, axis=1))))
    Rinv = sla.solve_triangular(Rh, np.eye(k + 1), lower=False)
    g2_exact = alpha * float(np.max(np.sqrt(np.sum(Rinv * Rinv, axis=1))))  # max column norm of R-hat^{-T}
    out.update(g1=g1, g2_est=g2_est, g2_exact=g2_exact, alpha=alpha, pivot=iota,
               tau_bound=g1 * g2_est * math.sqrt((k + 1) * (n - k)),
               tau_hat_bound=g1 * g2_est * math.sqrt(k * (n - k)))
    return out
