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


class RqrcpTrace(ctypes.Structure):
    _fields_ = [("first_panel", ctypes.c_int64), ("npanels", ctypes.c_int64), ("pivots", ctypes.c_void_p),
                ("rhat", ctypes.c_void_p), ("bnext", ctypes.c_void_p), ("recorded", ctypes.c_int64)]


_lib = None


def _nccl_hint():
    """Point the library at the NCCL torch uses (the nvidia-nccl wheel), unless
    RQRCP_NCCL_LIB is set; the library dlopen()s it for nranks > 1 only."""
    if os.environ.get("RQRCP_NCCL_LIB"):
        return
    try:
        import nvidia.nccl
        for d in list(getattr(nvidia.nccl, "__path__", [])):
            cand = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["RQRCP_NCCL_LIB"] = cand
                return
    except Exception:
        pass


def lib():
    """Load librqrcp.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        _nccl_hint()
        L = ctypes.CDLL(LIB_PATH)
        i64, vp, ip = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        L.rqrcp_create.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(RqrcpConfig)]
        L.rqrcp_factor.argtypes = [vp, vp, i64, i64, i64, i64, ip, ip, ctypes.c_uint64, vp, vp,
                                   ctypes.POINTER(i64)]
        L.rqrcp_factor_ex.argtypes = L.rqrcp_factor.argtypes + [vp, vp, ctypes.POINTER(RqrcpTrace)]
        L.rqrcp_set_option.argtypes = [vp, ctypes.c_char_p, i64]
        L.rqrcp_create_loopback_group.argtypes = [ctypes.POINTER(vp), ip, ctypes.POINTER(RqrcpConfig)]
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
            "rqrcp_set_option", "rqrcp_create_loopback_group",
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
    if n > 1 and lda < max(m, 1):
        # an expanded (stride-0) or overlapping view would be read and written
        # out of bounds by the library
        raise ValueError(f"column stride {lda} < rows {m}: overlapping or expanded view")
    return m, n, max(lda, 1)


def _check_vec(name, t, dtype, count, device):
    """Validate a caller-supplied output vector (dtype, length, device)."""
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != dtype:
        raise TypeError(f"{name} must be a {dtype} torch tensor")
    if t.dim() != 1 or t.numel() < count or (t.numel() > 1 and t.stride(0) != 1):
        raise ValueError(f"{name} must be a contiguous 1-D tensor with >= {count} elements")
    if t.device != device:
        raise ValueError(f"{name} is on {t.device}, the context runs on {device}")


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

    def last_error(self):
        msg = lib().rqrcp_last_error(self._h)
        return msg.decode() if msg else ""

    def _err(self, rc):
        msg = lib().rqrcp_last_error(self._h)
        return RqrcpError(rc, msg.decode() if msg else "")

    def factor(self, A, k, b, p, seed=0, jpvt=None, tau=None, omega=None, omega_out=None, trace=None,
               allow_rank_deficient=True, n=None):
        """Factor A in place (Alg. 2).  Returns (jpvt, tau, rank).

        Multi-GPU (nranks > 1): A is this rank's shard (shard_columns(n, b,
        nranks, rank)) and n the global column count.  trace: a Trace (see
        make_trace) filled per panel (testing hook of rqrcp_factor_ex)."""
        import torch
        m, n_loc, lda = _check_colmajor(A)
        if A.device != self.device:
            raise ValueError(f"A is on {A.device}, the context runs on {self.device}")
        n = n_loc if n is None else n
        if jpvt is None:
            jpvt = torch.empty(n, dtype=torch.int64, device=A.device)
        if tau is None:
            tau = torch.empty(max(k, 1), dtype=torch.float64, device=A.device)
        _check_vec("jpvt", jpvt, torch.int64, n, self.device)
        _check_vec("tau", tau, torch.float64, max(k, 1), self.device)
        self._order_after_caller()
        rank = ctypes.c_int64(0)
        if omega is None and omega_out is None and trace is None:
            rc = lib().rqrcp_factor(self._h, A.data_ptr(), lda, m, n, k, b, p, seed, jpvt.data_ptr(),
                                    tau.data_ptr(), ctypes.byref(rank))
        else:
            rc = lib().rqrcp_factor_ex(self._h, A.data_ptr(), lda, m, n, k, b, p, seed, jpvt.data_ptr(),
                                       tau.data_ptr(), ctypes.byref(rank),
                                       omega.data_ptr() if omega is not None else None,
                                       omega_out.data_ptr() if omega_out is not None else None,
                                       ctypes.byref(trace.c) if trace is not None else None)
            if trace is not None:
                trace.recorded = int(trace.c.recorded)
        if rc and not (rc == RQRCP_W_RANK_DEFICIENT and allow_rank_deficient):
            raise self._err(rc)
        return jpvt, tau[:k], int(rank.value)

    def _order_after_caller(self):
        """The context runs on the stream it was created with (include/rqrcp.h);
        work the caller queued on its CURRENT stream (e.g. filling A) must be
        complete before the library reads it: make the context stream wait."""
        import torch
        cur = torch.cuda.current_stream(self.device)
        if cur.cuda_stream != self.stream.cuda_stream:
            self.stream.wait_stream(cur)

    def set_option(self, name, value):
        """Launch-path option (rqrcp_set_option; testing / diagnosis)."""
        rc = lib().rqrcp_set_option(self._h, name.encode(), int(value))
        if rc:
            raise ValueError(f"rqrcp_set_option({name!r}, {value}) failed: {rc}")

    def make_trace(self, n, b, p, first_panel=0, npanels=1, device=None):
        return Trace(n, b, p, first_panel, npanels, device or self.device)

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
        self._order_after_caller()
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
        self._order_after_caller()
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
        self._order_after_caller()
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


class Trace:
    """Device buffers of the per-panel trace (rqrcp_trace): pivots
    (npanels x b), rhat / bnext (npanels blocks of l x n, ld l)."""

    def __init__(self, n, b, p, first_panel, npanels, device):
        import torch
        l = b + p
        self.n, self.b, self.l = n, b, l
        self.first_panel, self.npanels = first_panel, npanels
        self.pivots = torch.full((npanels * b,), -1, dtype=torch.int64, device=device)
        self.rhat = torch.zeros(npanels * l * n, dtype=torch.float64, device=device)
        self.bnext = torch.zeros(npanels * l * n, dtype=torch.float64, device=device)
        self.c = RqrcpTrace(first_panel, npanels, self.pivots.data_ptr(), self.rhat.data_ptr(),
                            self.bnext.data_ptr(), 0)
        self.recorded = 0

    def panel(self, t, bb, i):
        """(pivots[bb], rhat l x (n - i), bnext l x (n - i - bb)) of panel t as numpy."""
        q = t - self.first_panel
        l, n = self.l, self.n
        piv = self.pivots[q * self.b:q * self.b + bb].cpu().numpy()
        rh = self.rhat[q * l * n:q * l * n + l * (n - i)].cpu().numpy().reshape(n - i, l).T
        nb = n - i - bb
        bn = self.bnext[q * l * n:q * l * n + l * nb].cpu().numpy().reshape(nb, l).T
        return piv, rh, bn


class LoopbackGroup:
    """P contexts on ONE device forming an in-process group
    (rqrcp_create_loopback_group, testing API): runs the multi-rank driver
    logic -- block-cyclic shards, pivot-column reduce, panel broadcast,
    displaced-column broadcast, sample allgather -- with host-rendezvous
    collectives, one host thread per rank."""

    def __init__(self, nranks, max_m, max_n, max_b=128, max_p=16, device=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("LoopbackGroup needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.nranks = nranks
        cfg = RqrcpConfig()
        cfg.device = self.device.index
        cfg.max_m, cfg.max_n, cfg.max_b, cfg.max_p = max_m, max_n, max_b, max_p
        arr = (ctypes.c_void_p * nranks)()
        rc = lib().rqrcp_create_loopback_group(arr, nranks, ctypes.byref(cfg))
        if rc:
            raise RqrcpError(rc, "rqrcp_create_loopback_group failed")
        self._h = [ctypes.c_void_p(arr[r]) for r in range(nranks)]

    def set_option(self, name, value):
        for h in self._h:
            rc = lib().rqrcp_set_option(h, name.encode(), int(value))
            if rc:
                raise ValueError(f"rqrcp_set_option({name!r}) failed: {rc}")

    def factor(self, shards, n, k, b, p, seed=0):
        """shards[r]: rank r's column-major m x n_loc device tensor (factored in
        place).  Returns (jpvt list, tau list, rank list, codes)."""
        import threading

        import torch
        P = self.nranks
        jp = [torch.empty(n, dtype=torch.int64, device=self.device) for _ in range(P)]
        ta = [torch.empty(max(k, 1), dtype=torch.float64, device=self.device) for _ in range(P)]
        rk = [ctypes.c_int64(0) for _ in range(P)]
        codes = [None] * P
        torch.cuda.synchronize(self.device)

        def work(r):
            m, n_loc, lda = _check_colmajor(shards[r])
            codes[r] = lib().rqrcp_factor(self._h[r], shards[r].data_ptr(), lda, m, n, k, b, p, seed,
                                          jp[r].data_ptr(), ta[r].data_ptr(), ctypes.byref(rk[r]))

        th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize(self.device)
        return jp, [t[:k] for t in ta], [int(x.value) for x in rk], codes

    def last_error(self, r):
        msg = lib().rqrcp_last_error(self._h[r])
        return msg.decode() if msg else ""

    def close(self):
        for h in getattr(self, "_h", []):
            lib().rqrcp_destroy(h)
        self._h = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def version() -> str:
    return lib().rqrcp_version().decode()
