"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (default context, grid kernels), on outputs the oracle can compute:

* prefix: the oracle run to k' = 2b (two panels) must give exactly the first k'
  pivots and the same |diag R| rows as the GPU run to the full k (the prefix
  property, pinned for the oracle in test_oracle_pins.py::test_prefix_property;
  Omega does not depend on k);
* probes (properties that hold at any size): with R = [R11 R12; 0 R22] from
  the factored matrix, ||A Pi x - Q (R x)|| / (||A||_F ||x||) <= 1e-13 and
  ||Q^T Q x - x|| / ||x|| <= 1e-13 for Gaussian x (SURVEY.md §8(c) C4/C5 plan);
* jpvt is a permutation; the achieved rank is k.
"""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu


def _apply_q(F, tau, X, transpose=False):
    """Q X (or Q^T X), Q = H_0 ... H_{k-1}, reflectors from the factored matrix."""
    m = F.shape[0]
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


def _run(name, kprefix_panels=2, nprobe=4):
    import paper_1804_05138_b200 as rq
    c = inputs.CONFIGS[name]
    m, n, k, b, p, seed = c["m"], c["n"], c["k"], c["b"], c["p"], c["seed"]
    Ad = inputs.config_matrix(name, device="cuda")
    A = Ad.cpu().numpy()  # host copy of the input (not from the CUDA path)
    ctx = rq.RQRCP(max_m=m, max_n=n, max_b=b, max_p=p)
    jpvt, tau, rank = ctx.factor(Ad, k, b, p, seed=seed)
    torch.cuda.synchronize()
    ctx.close()
    F = Ad.cpu().numpy()
    jp = jpvt.cpu().numpy()
    ta = tau.cpu().numpy()
    del Ad
    torch.cuda.empty_cache()
    assert rank == k
    assert np.array_equal(np.sort(jp), np.arange(n))
    # ---- prefix oracle ----
    kp = min(k, kprefix_panels * b)
    o = oracle.rqrcp(A, kp, b, p, seed=seed)
    assert np.array_equal(jp[:kp], o["jpvt"][:kp]), "prefix pivots differ"
    dg = np.abs(np.diag(F)[:kp])
    do = np.abs(np.diag(o["A"])[:kp])
    assert np.max(np.abs(dg - do) / do) <= 1e-10
    # ---- probes ----
    rng = np.random.default_rng(7)
    X = rng.standard_normal((n, nprobe))
    R = np.triu(F[:k, :])  # top k rows: [R11 R12]
    RX = np.zeros((m, nprobe))
    RX[:k] = R @ X
    RX[k:] = (F[:, k:] @ X[k:])[k:]  # R22 block (trailing by-product); no strided copy
    Xp = np.zeros_like(X)
    Xp[jp] = X  # A Pi X = A (Pi X) without materialising A Pi
    lhs = A @ Xp
    err = np.linalg.norm(lhs - _apply_q(F, ta, RX)) / (np.linalg.norm(A) * np.linalg.norm(X))
    assert err <= 1e-13, err
    Y = rng.standard_normal((m, nprobe))
    err2 = np.linalg.norm(_apply_q(F, ta, _apply_q(F, ta, Y, transpose=True)) - Y) / np.linalg.norm(Y)
    assert err2 <= 1e-13, err2
    return np.linalg.norm(F[k:, k:]) / np.linalg.norm(A)


def test_C3_full_size():
    r = _run("C3")
    assert 0.0 < r < 1e-3  # low rank (1024 = k) plus 1e-6 noise: residual at the noise level


def test_C4_full_size():
    r = _run("C4", kprefix_panels=1)
    assert 0.0 < r < 0.1


@pytest.mark.slow
def test_C5_full_size():
    r = _run("C5", kprefix_panels=1, nprobe=2)
    assert 0.0 < r < 1.0
