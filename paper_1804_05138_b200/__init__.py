"""B200-native randomized QR with column pivoting (RQRCP) -- Python binding.

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of librqrcp.so (built in-tree by ``build.py``) behind the C ABI in
include/rqrcp.h.  PyTorch supplies device memory, streams and (for the
multi-GPU layout) process groups.  There is NO CPU fallback: if the library
is missing or no CUDA device is present, the calls raise.

Matrices are column-major fp64: a torch tensor of shape (m, n) with stride
(1, lda), e.g. ``A = torch.empty(n, m, dtype=torch.float64, device='cuda').t()``.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "librqrcp.so")

RQRCP_OK = 0
RQRCP_E_CUDA = 1
RQRCP_E_NCCL = 2
RQRCP_E_WORKSPACE = 3
RQRCP_E_NONFINITE = 4
RQRCP_E_UNSUPPORTED = 5
RQRCP_W_RANK_DEFICIENT = 16


class RqrcpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"rqrcp error {code}: {msg}")
        self.code = code


class RqrcpConfig(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("nranks", ctypes.c_int),
                ("rank", ctypes.c_int), ("nccl_uid", ctypes.c_uint8 * 128), ("max_m", ctypes.c_int64),
                ("max_n", ctypes.c_int64), ("max_b", ctypes.c_int), ("max_p", ctypes.c_int)]


class RqrcpTimings(ctypes.Structure):
    _fields_ = [("total_ms", ctypes.c_double), ("omega_ms", ctypes.c_double), ("sketch_ms", ctypes.c_double),
                ("sample_qrcp_ms", ctypes.c_double), ("swap_ms", ctypes.c_double), ("panel_ms", ctypes.c_double),
                ("trailing_ms", ctypes.c_double), ("sample_update_ms", ctypes.c_double),
                ("comm_ms", ctypes.c_double), ("panels", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("panels_householder", ctypes.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def lib():
    """Load librqrcp.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        i64, vp, ip = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        L.rqrcp_create.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(RqrcpConfig)]
        L.rqrcp_factor.argtypes = [vp, vp, i64, i64, i64, i64, ip, ip, ctypes.c_uint64, vp, vp,
                                   ctypes.POINTER(i64)]
        L.rqrcp_factor_ex.argtypes = L.rqrcp_factor.argtypes + [vp, vp, vp]
        L.rqrcp_factor_host.argtypes = [vp, vp, i64, i64, i64, i64, ip, ip, ctypes.c_uint64, vp, vp, vp,
                                        ctypes.POINTER(i64)]
        L.rqrcp_fill_gaussian.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint32, i64, i64, i64, i64, vp, i64]
        L.rqrcp_philox_words.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_uint32), vp, i64]
        L.rqrcp_flops.argtypes = [i64, i64, i64, ip, ip, ctypes.POINTER(ctypes.c_double)]
        L.rqrcp_get_timings.argtypes = [vp, ctypes.POINTER(RqrcpTimings)]
        L.rqrcp_set_timing.argtypes = [vp, ip]
        L.rqrcp_set_update_rule.argtypes = [vp, ip]
        L.rqrcp_form_q1.argtypes = [vp, vp, i64, i64, i64, i64, ip, vp, vp, i64]
        L.rqrcp_cx.argtypes = [vp, vp, i64, i64, i64, i64, vp, vp, i64]
        L.rqrcp_srqr_verify.argtypes = [vp, vp, i64, i64, i64, i64, ip, ip, ctypes.c_uint64, ip, vp, vp,
                                        ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_double)]
        L.rqrcp_destroy.argtypes = [vp]
        L.rqrcp_last_error.argtypes = [vp]
        L.rqrcp_last_error.restype = ctypes.c_char_p
        L.rqrcp_version.restype = ctypes.c_char_p
        L.rqrcp_shard_columns.argtypes = [i64, ip, ip, ip]
        L.rqrcp_shard_columns.restype = i64
        L.rqrcp_shard_global_index.argtypes = [i64, ip, ip, ip]
        L.rqrcp_shard_global_index.restype = i64
        L.rqrcp_nccl_unique_id.argtypes = [ctypes.POINTER(ctypes.c_uint8)]
        _lib = L
    return _lib


EXPORTED = ["rqrcp_create", "rqrcp_factor", "rqrcp_factor_host", "rqrcp_factor_ex", "rqrcp_fill_gaussian",
            "rqrcp_philox_words", "rqrcp_flops", "rqrcp_get_timings", "rqrcp_set_timing", "rqrcp_set_update_rule", "rqrcp_srqr_verify",
            "rqrcp_form_q1", "rqrcp_cx", "rqrcp_destroy",
            "rqrcp_last_error", "rqrcp_version", "rqrcp_shard_columns", "rqrcp_shard_global_index",
            "rqrcp_nccl_unique_id"]


def shard_columns(n, b, nranks, rank):
    """Global column indices held by `rank` in the 1D column-block-cyclic
    layout (block = b), in local order (host-side, from the C library)."""
    L = lib()
    nloc = L.rqrcp_shard_columns(n, b, nranks, rank)
    if nloc < 0:
        raise ValueError("invalid layout arguments")
    return [int(L.rqrcp_shard_global_index(q, b, nranks, rank)) for q in range(nloc)]


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (create on rank 0, broadcast to the others)."""
    buf = (ctypes.c_uint8 * 128)()
    rc = lib().rqrcp_nccl_unique_id(buf)
    if rc:
        raise RqrcpError(rc, "ncclGetUniqueId failed (libnccl.so.2 missing?)")
    return bytes(buf)


def rqrcp_flops(m, n, k, b, p):
    out = (ctypes.c_double * 4)()
    rc = lib().rqrcp_flops(m, n, k, b, p, out)
    if rc:
        raise RqrcpError(rc, "invalid argument")
    return dict(sketch=out[0], qr=out[1], sample_qrcp=out[2], sample_update=out[3], total=sum(out))


def _check_colmajor(A):
    import torch
    if not isinstance(A, torch.Tensor) or A.dtype != torch.float64 or A.dim() != 2:
        raise TypeError("A must be a 2-D float64 torch tensor")
    m, n = A.shape
    if A.stride(0) != 1 and m > 1:
        raise ValueError("A must be column-major (stride(0) == 1)")
    lda = A.stride(1) if n > 1 else max(m, 1)
    return m, n, max(lda, m, 1)


class RQRCP:
    """One context (workspace + stream) per device: rqrcp_create/_destroy."""

    def __init__(self, max_m, max_n, max_b=128, max_p=16, device=None, stream=None, nranks=1, rank=0,
                 nccl_uid=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("RQRCP needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        cfg = RqrcpConfig()
        cfg.device = self.device.index
        cfg.stream = ctypes.c_void_p(stream.cuda_stream)
        cfg.nranks = nranks
        cfg.rank = rank
        if nccl_uid is not None:
            for i, v in enumerate(bytes(nccl_uid)[:128]):
                cfg.nccl_uid[i] = v
        cfg.max_m, cfg.max_n, cfg.max_b, cfg.max_p = max_m, max_n, max_b, max_p
        self.nranks, self.rank = nranks, rank
        h = ctypes.c_void_p()
        rc = lib().rqrcp_create(ctypes.byref(h), ctypes.byref(cfg))
        if rc:
            raise RqrcpError(rc, "rqrcp_create failed")
        self._h = h

    def _err(self, rc):
        msg = lib().rqrcp_last_error(self._h)
        return RqrcpError(rc, msg.decode() if msg else "")

    def factor(self, A, k, b, p, seed=0, jpvt=None, tau=None, omega=None, omega_out=None, gaps=None,
               allow_rank_deficient=True, n=None):
        """Factor A in place (Alg. 2).  Returns (jpvt, tau, rank).

        Multi-GPU (nranks > 1): A is this rank's shard (shard_columns(n, b,
        nranks, rank)) and n the global column count."""
        import torch
        m, n_loc, lda = _check_colmajor(A)
        n = n_loc if n is None else n
        if jpvt is None:
            jpvt = torch.empty(n, dtype=torch.int64, device=A.device)
        if tau is None:
            tau = torch.empty(max(k, 1), dtype=torch.float64, device=A.device)
        rank = ctypes.c_int64(0)
        if omega is None and omega_out is None and gaps is None:
            rc = lib().rqrcp_factor(self._h, A.data_ptr(), lda, m, n, k, b, p, seed, jpvt.data_ptr(),
                                    tau.data_ptr(), ctypes.byref(rank))
        else:
            rc = lib().rqrcp_factor_ex(self._h, A.data_ptr(), lda, m, n, k, b, p, seed, jpvt.data_ptr(),
                                       tau.data_ptr(), ctypes.byref(rank),
                                       omega.data_ptr() if omega is not None else None,
                                       omega_out.data_ptr() if omega_out is not None else None,
                                       gaps.data_ptr() if gaps is not None else None)
        if rc and not (rc == RQRCP_W_RANK_DEFICIENT and allow_rank_deficient):
            raise self._err(rc)
        return jpvt, tau[:k], int(rank.value)

    def factor_raw(self, A_ptr, lda, m, n, k, b, p, seed, jpvt_ptr, tau_ptr):
        """Unchecked pointer call (bench inner loop); returns (code, rank)."""
        rank = ctypes.c_int64(0)
        rc = lib().rqrcp_factor(self._h, A_ptr, lda, m, n, k, b, p, seed, jpvt_ptr, tau_ptr, ctypes.byref(rank))
        return rc, int(rank.value)

    def factor_host(self, A_host, k, b, p, seed=0, out=None, jpvt=None, tau=None):
        """End-to-end path with HOST (ideally pinned) column-major buffers."""
        import torch
        m, n, lda = _check_colmajor(A_host)
        if out is None:
            out = A_host
        if jpvt is None:
            jpvt = torch.empty(n, dtype=torch.int64, pin_memory=True)
        if tau is None:
            tau = torch.empty(max(k, 1), dtype=torch.float64, pin_memory=True)
        rank = ctypes.c_int64(0)
        rc = lib().rqrcp_factor_host(self._h, A_host.data_ptr(), lda, m, n, k, b, p, seed, out.data_ptr(),
                                     jpvt.data_ptr(), tau.data_ptr(), ctypes.byref(rank))
        if rc and rc != RQRCP_W_RANK_DEFICIENT:
            raise self._err(rc)
        return jpvt, tau[:k], int(rank.value)

    def fill_gaussian(self, out, seed, stream, row0=0, col0=0):
        m, n, ld = _check_colmajor(out)
        rc = lib().rqrcp_fill_gaussian(self._h, seed, stream, m, n, row0, col0, out.data_ptr(), ld)
        if rc:
            raise self._err(rc)
        return out

    def philox_words(self, ctr, key):
        """ctr: int32/uint32-valued CUDA tensor (count, 4); returns (count, 4) words as int64."""
        import torch
        c = ctr.to(torch.int64).to(torch.int32).contiguous()
        out = torch.empty_like(c)
        k = (ctypes.c_uint32 * 2)(int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF)
        rc = lib().rqrcp_philox_words(self._h, c.data_ptr(), k, out.data_ptr(), c.shape[0])
        if rc:
            raise self._err(rc)
        return out.to(torch.int64) & 0xFFFFFFFF

    def timings(self):
        t = RqrcpTimings()
        lib().rqrcp_get_timings(self._h, ctypes.byref(t))
        return t.as_dict()

    def srqr_verify(self, A, k, b, p, seed=0, d=8, jpvt=None, tau=None):
        """RQRCP to rank k + the SRQR verification of Alg. 3, see
        rqrcp_srqr_verify in include/rqrcp.h.  A is factored in place (with the
        (k+1)-th pivot swapped to position k).  Returns (jpvt, tau, rank, diag)
        with diag = dict(g1, g2_est, alpha, tau_bound, tau_hat_bound, pivot)."""
        import torch
        m, n, lda = _check_colmajor(A)
        if jpvt is None:
            jpvt = torch.empty(n, dtype=torch.int64, device=A.device)
        if tau is None:
            tau = torch.empty(max(k, 1), dtype=torch.float64, device=A.device)
        rank = ctypes.c_int64(0)
        out = (ctypes.c_double * 6)()
        rc = lib().rqrcp_srqr_verify(self._h, A.data_ptr(), lda, m, n, k, b, p, seed, d, jpvt.data_ptr(),
                                     tau.data_ptr(), ctypes.byref(rank), out)
        if rc:
            raise self._err(rc)
        names = ("g1", "g2_est", "alpha", "tau_bound", "tau_hat_bound", "pivot")
        diag = {nm: float(v) for nm, v in zip(names, out)}
        diag["pivot"] = int(diag["pivot"])
        return jpvt, tau[:k], int(rank.value), diag

    def form_q1(self, A, k, b, tau, Q1=None):
        """Q1 = first k columns of Q = H_1...H_k from a factored A."""
        import torch
        m, n, lda = _check_colmajor(A)
        if Q1 is None:
            Q1 = torch.empty(k, m, dtype=torch.float64, device=A.device).t()
        _, _, ldq = _check_colmajor(Q1)
        rc = lib().rqrcp_form_q1(self._h, A.data_ptr(), lda, m, n, k, b, tau.data_ptr(), Q1.data_ptr(), ldq)
        if rc:
            raise self._err(rc)
        return Q1

    def cx(self, A, k, jpvt, X=None):
        """CX coefficients X = C^+ A, C = A Pi(:, :k), from a factored A."""
        import torch
        m, n, lda = _check_colmajor(A)
        if X is None:
            X = torch.empty(n, k, dtype=torch.float64, device=A.device).t()
        _, _, ldx = _check_colmajor(X)
        rc = lib().rqrcp_cx(self._h, A.data_ptr(), lda, m, n, k, jpvt.data_ptr(), X.data_ptr(), ldx)
        if rc:
            raise self._err(rc)
        return X

    def set_update_rule(self, rule: int):
        """1: Eq. (4) (default), 2: Eq. (5) -- see rqrcp_set_update_rule in include/rqrcp.h."""
        rc = lib().rqrcp_set_update_rule(self._h, int(rule))
        if rc:
            raise ValueError(f"update rule must be 1 or 2 (rc {rc})")

    def set_timing(self, enabled: bool):
        lib().rqrcp_set_timing(self._h, 1 if enabled else 0)

    def close(self):
        if getattr(self, "_h", None):
            lib().rqrcp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def version() -> str:
    return lib().rqrcp_version().decode()
