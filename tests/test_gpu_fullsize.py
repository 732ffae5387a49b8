"""Parity at BASELINE.json's full sizes (C3, C4, C5), in the launch
configuration bench.py times (default context and schedule), against the CPU
oracle:

* C3 (16384^2, k = 1024): the FULL oracle run -- identical pivots, |diag R|,
  [R11 R12], tau and V element by element, residuals (as test_gpu_parity), and
  the per-panel trace of all 16 panels (R-hat after S2, the Eq. (4) sample
  after S6) against the oracle's panel callback;
* C4 (32768^2, k = 8192) and C5 (65536^2, k = 4096): the PREFIX oracle to
  k' = 512 = 4 panels at both (the prefix property, pinned for the
  oracle in test_oracle_pins.py::test_prefix_property: the first k' pivots
  and R rows do not depend on k): identical first k' pivots, R rows 0..k'-1
  element-wise matched by column id (later swaps only permute columns),
  tau / V of the first k' columns, and the per-panel trace of those panels;
* C3 again with the column-by-column Householder panel (option panel = 0;
  the default from 8192 rows is CholeskyQR2 + reconstruction);
* at any size, probes: with R = [R11 R12; 0 R22] from the factored matrix,
  ||A Pi x - Q (R x)|| / (||A||_F ||x||) <= 1e-13 and ||Q^T Q x - x|| / ||x||
  <= 1e-13 for Gaussian x (SURVEY.md §8(c) C4/C5 plan).
"""
import os

import numpy as np
import pytest
import torch

import inputs
import oracle
from gpu_helpers import check_trace_panels

pytestmark = pytest.mark.gpu

ELEM_RTOL = 1e-10


def _apply_q(F, tau, X, transpose=False):
    """Q X (or Q^T X), Q = H_0 ... H_{k-1}, reflectors from the factored matrix."""
    k = len(tau)
    Y = X.copy()
    order = range(k) if transpose else range(k - 1, -1, -1)
    for j in order:
        t = tau[j]
        if t == 0.0:
            continue
        v = F[j:, j].copy()
        v[0] = 1.0
        Y[j:] -= t * np.outer(v, v @ Y[j:])
    return Y


def _run(name, prefix_panels=None, nprobe=4, opts=None):
    import paper_1804_05138_b200 as rq
    c = inputs.CONFIGS[name]
    m, n, k, b, p, seed = c["m"], c["n"], c["k"], c["b"], c["p"], c["seed"]
    npan_all = (k + b - 1) // b
    npan = npan_all if prefix_panels is None else min(npan_all, prefix_panels)
    kp = min(k, npan * b)
    Ad = inputs.config_matrix(name, device="cuda")
    A = Ad.cpu().numpy()  # host copy of the input (not from the CUDA path)
    ctx = rq.RQRCP(max_m=m, max_n=n, max_b=b, max_p=p)
    for kk, vv in (opts or {}).items():
        ctx.set_option(kk, vv)
    tr = ctx.make_trace(n, b, p, 0, npan)
    jpvt, tau, rank = ctx.factor(Ad, k, b, p, seed=seed, trace=tr)
    torch.cuda.synchronize()
    ctx.close()
    F = Ad.cpu().numpy()
    jp = jpvt.cpu().numpy()
    ta = tau.cpu().numpy()
    del Ad
    torch.cuda.empty_cache()
    assert rank == k
    assert np.array_equal(np.sort(jp), np.arange(n))
    # ---- probes (any size) ----
    rng = np.random.default_rng(7)
    X = rng.standard_normal((n, nprobe))
    R = np.triu(F[:k, :])
    RX = np.zeros((m, nprobe))
    RX[:k] = R @ X
    RX[k:] = (F[:, k:] @ X[k:])[k:]
    del R
    Xp = np.zeros_like(X)
    Xp[jp] = X
    lhs = A @ Xp
    err = np.linalg.norm(lhs - _apply_q(F, ta, RX)) / (np.linalg.norm(A) * np.linalg.norm(X))
    assert err <= 1e-13, err
    Y = rng.standard_normal((m, nprobe))
    err2 = np.linalg.norm(_apply_q(F, ta, _apply_q(F, ta, Y, transpose=True)) - Y) / np.linalg.norm(Y)
    assert err2 <= 1e-13, err2
    r22 = np.linalg.norm(F[k:, k:]) / np.linalg.norm(A)
    # ---- oracle (full or prefix) ----
    panels = []
    o = oracle.rqrcp(A, kp, b, p, seed=seed, invariant=True,
                     callback=lambda i, bb, l_, mp, np_, Rh, Bn, Oc, On, Af: panels.append((i, bb, Rh, Bn)))
    del A
    assert np.array_equal(jp[:kp], o["jpvt"][:kp]), "pivots differ"
    Fo = o["A"]
    dg = np.abs(np.diag(F)[:kp])
    do = np.abs(np.diag(Fo)[:kp])
    assert np.max(np.abs(dg - do) / do) <= 1e-10
    # R rows 0..kp-1 matched by original column id (later panels only permute columns)
    pos_g = np.empty(n, dtype=np.int64)
    pos_g[jp] = np.arange(n)
    pos_o = np.empty(n, dtype=np.int64)
    pos_o[o["jpvt"]] = np.arange(n)
    Rg = np.triu(F[:kp, :])[:, pos_g]
    Ro = np.triu(Fo[:kp, :])[:, pos_o]
    assert np.max(np.abs(Rg - Ro)) <= ELEM_RTOL * np.max(np.abs(Ro)), "R rows differ"
    del Rg, Ro
    assert np.max(np.abs(ta[:kp] - o["tau"][:kp])) <= ELEM_RTOL
    Vg = np.tril(F[:, :kp], -1)
    Vo = np.tril(Fo[:, :kp], -1)
    assert np.max(np.abs(Vg - Vo)) <= ELEM_RTOL
    del Vg, Vo, F, Fo
    check_trace_panels(tr, panels, o["jpvt"], k=k)
    return r22


def test_C3_full_size():
    r = _run("C3")
    assert 0.0 < r < 1e-3  # low rank (1024 = k) plus 1e-6 noise: residual at the noise level


def test_C3_full_size_householder_panel():
    """The default panel at C3-C5 is CholeskyQR2 + reconstruction (panel = 2:
    from 8192 rows); the column-by-column Householder grid panel gets the same
    full-size check."""
    r = _run("C3", opts={"panel": 0})
    assert 0.0 < r < 1e-3


def test_C4_full_size():
    r = _run("C4", prefix_panels=int(os.environ.get("RQRCP_TEST_C4_PANELS", "4")))
    assert 0.0 < r < 0.1


def test_C5_full_size():
    r = _run("C5", prefix_panels=int(os.environ.get("RQRCP_TEST_C5_PANELS", "4")), nprobe=2)
    assert 0.0 < r < 1.0
