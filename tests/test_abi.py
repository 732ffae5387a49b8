"""The C-ABI library loads and exports every symbol include/rqrcp.h declares
(no compute calls: runs without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            src = open(os.path.join(ROOT, "include", fn)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names |= set(re.findall(r"\b(rqrcp_[a-z_0-9]+)\s*\(", src))
    return sorted(names)


@pytest.fixture(scope="module")
def lib():
    from paper_1804_05138_b200 import build
    build.build()
    return ctypes.CDLL(build.LIB)


def test_header_declares_the_north_star_api():
    syms = declared_symbols()
    for s in ("rqrcp_create", "rqrcp_factor", "rqrcp_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_names_match_header():
    import paper_1804_05138_b200 as rq
    assert sorted(rq.EXPORTED) == declared_symbols()


def test_flops_counts(lib):
    """rqrcp_flops (host-only) against the closed forms of SURVEY.md §8(d)."""
    import paper_1804_05138_b200 as rq
    f = rq.rqrcp_flops(4096, 4096, 512, 64, 10)
    assert f["sketch"] == 2 * 74 * 4096 * 4096
    qr = sum(4.0 * (4096 - j) * (4096 - j) for j in range(512))
    assert abs(f["qr"] - qr) <= 1e-12 * qr
    assert abs(f["total"] - 3.332e10) / 3.332e10 < 2e-3
    c5 = rq.rqrcp_flops(65536, 65536, 4096, 128, 16)
    assert abs(c5["total"] - 6.7451e13) / 6.7451e13 < 2e-3


def test_no_gpu_raises_loudly():
    import torch

    import paper_1804_05138_b200 as rq
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        rq.RQRCP(64, 64)
