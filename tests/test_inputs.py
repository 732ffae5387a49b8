"""Input generators (inputs/): recipes of BASELINE.json's configs."""
import math

import numpy as np
import torch

import inputs


def test_fortran_layout():
    a = inputs.iid(1, 7, 5)
    assert a.shape == (7, 5) and a.stride() == (1, 7)


def test_haar_orthogonal():
    q = inputs.haar(3, 1, 64).numpy()
    assert np.linalg.norm(q.T @ q - np.eye(64)) < 1e-13


def test_svd_matrix_spectrum():
    j = torch.arange(1, 97, dtype=torch.float64)
    sig = torch.exp(-j / 20.0)
    a = inputs.svd_matrix(5, 96, 96, sig).numpy()
    s = np.linalg.svd(a, compute_uv=False)
    assert np.allclose(s[:40], sig.numpy()[:40], rtol=1e-11)


def test_low_rank_plus_noise():
    a = inputs.low_rank_plus_noise(2, 200, 150, 20).numpy()
    s = np.linalg.svd(a, compute_uv=False)
    assert s[19] > 1e-2 and s[20] < 1e-4


def test_graded_columns():
    a = inputs.graded(4, 300, 100).numpy()
    c = np.linalg.norm(a, axis=0)
    ratio = c[-1] / c[0]
    assert 10 ** (-6 * 99 / 100) / 3 < ratio < 3 * 10 ** (-6 * 99 / 100)


def test_kahan_definition():
    k = inputs.kahan(3).numpy()
    s = math.sqrt(0.9998 - 0.285 ** 2)
    assert np.allclose(k[0], [1, -0.285, -0.285])
    assert np.allclose(k[1], [0, s, -0.285 * s])
    assert np.allclose(k[2], [0, 0, s * s])


def test_configs_listed():
    assert set(inputs.CONFIGS) == {"C1", "C2", "C3", "C4", "C5"}
    c = inputs.CONFIGS["C2"]
    assert (c["m"], c["n"], c["k"], c["b"], c["p"]) == (4096, 4096, 512, 64, 10)
