"""Seeded synthetic input generators (shared by tests, bench.py and smoke()).

This module holds NONE of the method's arithmetic: it only produces the input
matrices A of the five BASELINE.json configs (and small test matrices of the
same recipes).  It is the single module that both the CUDA path's callers and
the oracle's callers draw inputs from; the Gaussian sketch Omega that RQRCP
itself draws (Alg. 2) is NOT generated here - the library
(kernel K1) and the oracle (oracle/rqrcp_oracle.c) each implement the same
counter-based generator independently.

Generator mapping: element (r, c) of a generated matrix
comes from Philox4x32-10 (Salmon et al., SC'11) with key = (seed lo, seed hi)
and counter = (c mod 2^32, floor(r/2), stream, c >> 32).  Words (w0, w1) give
u1 = (((w0 << 32) | w1) >> 11 + 1/2) * 2^-53, (w2, w3) give u2; Box-Muller
gives z0 = sqrt(-2 ln u1) cos(2 pi u2) for even r and z1 = ... sin(...) for
odd r.  Streams: 0 = Omega (inside the library), 1 = G_U, 2 = G_V, 3 = X,
4 = Y, 5 = E, 6 = iid A.

Implementation: plain torch integer ops (int64 tensors holding uint32 words),
so the same code runs on CPU tensors (tests) and CUDA tensors (bench-size
inputs, which would take minutes to build on the host).  Matrices are returned
as "Fortran-ordered" torch tensors: shape (rows, cols), stride (1, rows), i.e.
column-major storage, the layout the C ABI takes.
"""
from __future__ import annotations

import math

import torch

PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF

STREAM_OMEGA = 0
STREAM_GU = 1
STREAM_GV = 2
STREAM_X = 3
STREAM_Y = 4
STREAM_E = 5
STREAM_IID = 6


def _mulhilo(a: torch.Tensor, m: int):
    # a < 2^32, m < 2^32: the product fits in 64 bits; int64 multiply wraps
    # two's-complement, so masking recovers the exact unsigned halves.
    prod = a * m
    return (prod >> 32) & MASK32, prod & MASK32


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Philox4x32-10 on int64 tensors of uint32 words (broadcastable)."""
    x0, x1, x2, x3 = c0, c1, c2, c3
    for r in range(10):
        if r:
            k0 = (k0 + PHILOX_W0) & MASK32
            k1 = (k1 + PHILOX_W1) & MASK32
        hi0, lo0 = _mulhilo(x0, PHILOX_M0)
        hi1, lo1 = _mulhilo(x2, PHILOX_M1)
        x0, x1, x2, x3 = hi1 ^ x1 ^ k0, lo1, hi0 ^ x3 ^ k1, lo0
    return x0, x1, x2, x3


def _u53(hi: torch.Tensor, lo: torch.Tensor) -> torch.Tensor:
    # ((hi << 32) | lo) >> 11 without leaving int64's positive range
    a = (hi << 21) | (lo >> 11)
    return (a.to(torch.float64) + 0.5) * (2.0 ** -53)


def gaussian(seed: int, stream: int, rows: int, cols: int, row0: int = 0, col0: int = 0,
             device="cpu") -> torch.Tensor:
    """Rows [row0, row0+rows) x cols [col0, col0+cols) of the N(0,1) matrix
    (seed, stream); returned column-major (stride (1, rows))."""
    dev = torch.device(device)
    k0, k1 = seed & MASK32, (seed >> 32) & MASK32
    r = torch.arange(row0, row0 + rows, device=dev, dtype=torch.int64)
    c = torch.arange(col0, col0 + cols, device=dev, dtype=torch.int64)
    out = torch.empty((cols, rows), dtype=torch.float64, device=dev)
    # chunk over columns to bound temporaries (C4/C5 are 1e9 elements)
    chunk = max(1, (1 << 24) // max(rows, 1))
    rpair = (r >> 1).view(1, -1)
    odd = (r & 1).view(1, -1).bool()
    for j0 in range(0, cols, chunk):
        cc = c[j0:j0 + chunk].view(-1, 1)
        w0, w1, w2, w3 = philox4x32_10(cc & MASK32, rpair, torch.full_like(cc, stream),
                                       cc >> 32, k0, k1)
        u1 = _u53(w0, w1)
        u2 = _u53(w2, w3)
        rho = torch.sqrt(-2.0 * torch.log(u1))
        ang = (2.0 * math.pi) * u2
        out[j0:j0 + chunk] = torch.where(odd, rho * torch.sin(ang), rho * torch.cos(ang))
    return out.t()


def fortran(t: torch.Tensor) -> torch.Tensor:
    """Column-major copy of a 2-D tensor."""
    return t.t().contiguous().t()


def haar(seed: int, stream: int, n: int, device="cpu") -> torch.Tensor:
    """Haar-orthogonal n x n: Q of a Gaussian QR, columns times sign(diag R)
    (Mezzadri's correction)."""
    g = gaussian(seed, stream, n, n, device=device)
    q, r = torch.linalg.qr(g)
    d = torch.sign(torch.diagonal(r))
    d[d == 0] = 1.0
    return fortran(q * d.view(1, -1))


def svd_matrix(seed: int, m: int, n: int, sigma: torch.Tensor, device="cpu") -> torch.Tensor:
    """A = U diag(sigma) V^T with U, V the first min(m, n) columns of Haar
    m x m / n x n orthogonal matrices (streams 1, 2)."""
    r = min(m, n)
    u = haar(seed, STREAM_GU, m, device=device)[:, :r]
    v = haar(seed, STREAM_GV, n, device=device)[:, :r]
    return fortran((u * sigma[:r].to(device).view(1, -1)) @ v.t())


def iid(seed: int, m: int, n: int, device="cpu") -> torch.Tensor:
    return gaussian(seed, STREAM_IID, m, n, device=device)


def low_rank_plus_noise(seed: int, m: int, n: int, rank: int, noise: float = 1e-6,
                        device="cpu") -> torch.Tensor:
    x = gaussian(seed, STREAM_X, m, rank, device=device) / math.sqrt(rank)
    y = gaussian(seed, STREAM_Y, n, rank, device=device) / math.sqrt(rank)
    e = gaussian(seed, STREAM_E, m, n, device=device)
    a = x @ y.t()
    a = fortran(a)
    a.add_(e, alpha=noise)
    return a


def graded(seed: int, m: int, n: int, decades: float = 6.0, device="cpu") -> torch.Tensor:
    a = gaussian(seed, STREAM_IID, m, n, device=device)
    j = torch.arange(n, dtype=torch.float64, device=a.device)
    a.mul_(torch.pow(10.0, -decades * j / n).view(1, -1))
    return a


def kahan(n: int, c: float = 0.285, s2c2: float = 0.9998) -> torch.Tensor:
    """Kahan matrix K = diag(s^(i-1)) (I - c * strict-upper-ones) (
    s^2 + c^2 = 0.9998 per DESIGN.md reading R-G13, the paper prints 0.9999)."""
    s = math.sqrt(s2c2 - c * c)
    k = torch.eye(n, dtype=torch.float64) - c * torch.triu(torch.ones(n, n, dtype=torch.float64), 1)
    k = torch.pow(torch.tensor(s, dtype=torch.float64), torch.arange(n, dtype=torch.float64)).view(-1, 1) * k
    return fortran(k)


# --------------------------------------------------------------------------
# BASELINE.json configs (SURVEY.md §8(d) "Configs")
# --------------------------------------------------------------------------
CONFIGS = {
    "C1": dict(m=512, n=512, k=64, b=32, p=8, seed=1001, kind="svd_exp"),
    "C2": dict(m=4096, n=4096, k=512, b=64, p=10, seed=1002, kind="iid"),
    "C3": dict(m=16384, n=16384, k=1024, b=64, p=10, seed=1003, kind="lowrank"),
    "C4": dict(m=32768, n=32768, k=8192, b=128, p=16, seed=1004, kind="svd_poly"),
    "C5": dict(m=65536, n=65536, k=4096, b=128, p=16, seed=1005, kind="graded"),
}


def make(kind: str, m: int, n: int, seed: int, device="cpu", rank: int = 1024) -> torch.Tensor:
    """Input A (column-major fp64) for a recipe; any (m, n) for test shapes."""
    if kind == "svd_exp":
        j = torch.arange(1, min(m, n) + 1, dtype=torch.float64)
        return svd_matrix(seed, m, n, torch.exp(-j / 20.0), device=device)
    if kind == "svd_poly":
        j = torch.arange(1, min(m, n) + 1, dtype=torch.float64)
        return svd_matrix(seed, m, n, 1.0 / j, device=device)
    if kind == "iid":
        return iid(seed, m, n, device=device)
    if kind == "lowrank":
        return low_rank_plus_noise(seed, m, n, rank, device=device)
    if kind == "graded":
        return graded(seed, m, n, device=device)
    raise ValueError(kind)


def config_matrix(name: str, device="cpu") -> torch.Tensor:
    c = CONFIGS[name]
    return make(c["kind"], c["m"], c["n"], c["seed"], device=device)
