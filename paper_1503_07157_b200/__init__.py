"""B200-native blocked randomized QB factorization (Martinsson & Voronin, arXiv 1503.07157).

Thin Python binding over the C ABI in include/qb.h (libqb.so, built in-tree for sm_100a by
``python -m paper_1503_07157_b200.build``).  This module only marshals arguments: every
arithmetic step of the factorization runs in the library's CUDA kernels.  There is no CPU
fallback — if libqb.so is missing or no B200 is visible, calls raise.

Function names mirror the C entry points: qb_create, qb_factor, qb_stats, qb_omega, qb_orth,
qb_destroy, qb_status_string, qb_last_error, qb_kernel_launches.  ``factor()`` is a
convenience wrapper for torch CUDA tensors (torch supplies device memory only).
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QB_LIB_PATH") or os.path.join(_HERE, "libqb.so")  # override: experiments only

QB_OK = 0
QB_NOT_CONVERGED = 1
QB_ERR_INVALID_ARG = 2
QB_ERR_OOM = 3
QB_ERR_CUDA = 4
QB_ERR_NCCL = 5
QB_ERR_ORTH_BREAKDOWN = 6
QB_ERR_UNSUPPORTED = 7

QB_F64 = 0
QB_F32 = 1

QB_SHARD_COLS = 0
QB_SHARD_ROWS = 1
QB_COMM_NCCL = 0
QB_COMM_LOOPBACK = 1
QB_LOOPBACK_MAX_RANKS = 8

QB_OVERWRITE_A = 1
QB_NO_REPROJ = 2
QB_SKIP_POWER_ORTH = 4
QB_FORCE_GENERAL = 8


class QBError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_status_name(status)}: {msg}")
        self.status = status


class BlockStats(ctypes.Structure):
    _fields_ = [("ell", ctypes.c_int64), ("w", ctypes.c_int64), ("r2", ctypes.c_double),
                ("ei", ctypes.c_double), ("ms", ctypes.c_double), ("ms_sketch", ctypes.c_double),
                ("ms_bmat", ctypes.c_double), ("ms_down", ctypes.c_double), ("fallback", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("ms_orth", ctypes.c_double), ("ms_orth_z", ctypes.c_double),
                ("ms_reproj", ctypes.c_double), ("ms_power", ctypes.c_double), ("kappa_r", ctypes.c_double)]


class QBDist(ctypes.Structure):
    """qb_dist (include/qb.h)."""
    _fields_ = [("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("shard", ctypes.c_int), ("comm", ctypes.c_int),
                ("nccl_id", ctypes.c_void_p), ("loopback", ctypes.c_void_p), ("offset", ctypes.c_int64),
                ("global_", ctypes.c_int64)]


_lib = None


def lib():
    """The loaded libqb.so (raises loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1503_07157_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        c_ctx = ctypes.c_void_p
        i64, u64, dbl, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        P = ctypes.POINTER
        L.qb_create.argtypes = [P(c_ctx), ctypes.c_int, ctypes.c_int, vp]
        L.qb_create_dist.argtypes = [P(c_ctx), ctypes.c_int, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, vp,
                                     i64, i64]
        L.qb_create_dist_rows.argtypes = [P(c_ctx), ctypes.c_int, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, vp,
                                          i64, i64]
        L.qb_nccl_unique_id.argtypes = [vp]
        L.qb_create_sharded.argtypes = [P(c_ctx), ctypes.c_int, ctypes.c_int, vp, P(QBDist)]
        L.qb_loopback_create.argtypes = [P(vp), ctypes.c_int]
        L.qb_loopback_destroy.argtypes = [vp]
        L.qb_loopback_destroy.restype = None
        L.qb_factor.argtypes = [c_ctx, vp, i64, i64, i64, dbl, i64, ctypes.c_int, u64, i64, ctypes.c_uint,
                                P(i64), P(vp), P(i64), P(vp), P(i64), P(dbl)]
        L.qb_factor_host.argtypes = [c_ctx, vp, i64, i64, i64, dbl, i64, ctypes.c_int, u64, i64, P(i64), vp, i64,
                                     vp, i64, i64, P(dbl)]
        L.qb_gemm.argtypes = [c_ctx, ctypes.c_int, ctypes.c_int, i64, i64, i64, vp, i64, vp, i64, vp, i64,
                              ctypes.c_int, P(dbl)]
        L.qb_chol_rinv.argtypes = [c_ctx, vp, i64, i64, i64, vp, i64, P(ctypes.c_int)]
        L.qb_stats.argtypes = [c_ctx, vp, i64, P(i64)]
        L.qb_omega.argtypes = [c_ctx, u64, i64, i64, i64, i64, vp, i64]
        L.qb_orth.argtypes = [c_ctx, vp, i64, i64, i64]
        L.rqb_svd.argtypes = [c_ctx, dbl, i64, P(i64), P(vp), P(i64), P(vp), P(vp), P(i64)]
        L.qb_svd_sweeps.argtypes = [c_ctx]
        L.qb_svd_sweeps.restype = ctypes.c_int
        L.qb_pivoted_qr.argtypes = [c_ctx, vp, P(vp), P(i64), P(vp), P(i64)]
        L.qb_fixed_rank.argtypes = [c_ctx, vp, i64, i64, i64, i64, ctypes.c_int, u64, ctypes.c_uint, P(vp), P(i64),
                                    P(vp), P(i64), P(dbl)]
        L.qb_kernel_launches.argtypes = [c_ctx]
        L.qb_kernel_launches.restype = i64
        L.qb_destroy.argtypes = [c_ctx]
        L.qb_destroy.restype = None
        L.qb_status_string.argtypes = [ctypes.c_int]
        L.qb_status_string.restype = ctypes.c_char_p
        L.qb_last_error.argtypes = [c_ctx]
        L.qb_last_error.restype = ctypes.c_char_p
        for f in ("qb_create", "qb_create_dist", "qb_create_dist_rows", "qb_create_sharded", "qb_loopback_create", "qb_nccl_unique_id", "qb_factor", "qb_factor_host", "qb_gemm", "qb_chol_rinv", "qb_stats", "qb_omega",
                  "qb_orth", "rqb_svd", "qb_fixed_rank", "qb_pivoted_qr"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _status_name(s):
    try:
        return lib().qb_status_string(int(s)).decode()
    except Exception:  # pragma: no cover
        return f"status {s}"


def qb_status_string(s):
    return lib().qb_status_string(int(s)).decode()


def qb_last_error(ctx):
    return lib().qb_last_error(ctx).decode()


def _check(ctx, s, ok=(QB_OK,)):
    if s not in ok:
        raise QBError(s, qb_last_error(ctx) if ctx else "")
    return s


def qb_create(device=0, dtype=QB_F64, stream=None):
    ctx = ctypes.c_void_p()
    s = lib().qb_create(ctypes.byref(ctx), int(device), int(dtype), stream)
    if s != QB_OK:
        msg = qb_last_error(ctx) if ctx.value else ""
        if ctx.value:
            lib().qb_destroy(ctx)
        raise QBError(s, msg)
    return ctx


def qb_nccl_unique_id():
    """128-byte ncclUniqueId (bytes) for qb_create_dist; rank 0 creates it, all ranks share it."""
    buf = ctypes.create_string_buffer(128)
    s = lib().qb_nccl_unique_id(buf)
    if s != QB_OK:
        raise QBError(s, "qb_nccl_unique_id failed (is libnccl.so.2 loadable?)")
    return buf.raw


def qb_create_dist(device, rank, nranks, unique_id, col_offset, n_global, dtype=QB_F64, stream=None, rows=False):
    """Column-sharded context (rows=False: col_offset / n_global) or row-sharded context
    (rows=True: the same two arguments are row_offset / m_global)."""
    ctx = ctypes.c_void_p()
    uid = ctypes.create_string_buffer(bytes(unique_id), 128)
    fn = lib().qb_create_dist_rows if rows else lib().qb_create_dist
    s = fn(ctypes.byref(ctx), int(device), int(dtype), stream, int(rank), int(nranks), uid, int(col_offset),
           int(n_global))
    if s != QB_OK:
        msg = qb_last_error(ctx) if ctx.value else ""
        if ctx.value:
            lib().qb_destroy(ctx)
        raise QBError(s, msg)
    return ctx


def qb_create_sharded(device, rank, nranks, shard, offset, global_, dtype=QB_F64, stream=None, unique_id=None,
                      loopback=None):
    """Sharded context from a qb_dist descriptor: shard QB_SHARD_COLS / QB_SHARD_ROWS; NCCL
    (unique_id, 128 bytes) or an in-process loopback group (loopback = qb_loopback_create())."""
    d = QBDist()
    d.rank, d.nranks, d.shard = int(rank), int(nranks), int(shard)
    uid = None
    if loopback is not None:
        d.comm = QB_COMM_LOOPBACK
        d.loopback = loopback.value if isinstance(loopback, ctypes.c_void_p) else loopback
    else:
        d.comm = QB_COMM_NCCL
        uid = ctypes.create_string_buffer(bytes(unique_id), 128)
        d.nccl_id = ctypes.cast(uid, ctypes.c_void_p)
    d.offset, d.global_ = int(offset), int(global_)
    ctx = ctypes.c_void_p()
    s = lib().qb_create_sharded(ctypes.byref(ctx), int(device), int(dtype), stream, ctypes.byref(d))
    if s != QB_OK:
        msg = qb_last_error(ctx) if ctx.value else ""
        if ctx.value:
            lib().qb_destroy(ctx)
        raise QBError(s, msg)
    return ctx


def qb_loopback_create(nranks):
    """An in-process loopback group of nranks ranks (one GPU, one host thread per rank)."""
    g = ctypes.c_void_p()
    s = lib().qb_loopback_create(ctypes.byref(g), int(nranks))
    if s != QB_OK:
        raise QBError(s, f"qb_loopback_create({nranks})")
    return g


def qb_loopback_destroy(group):
    if group is not None and group.value:
        lib().qb_loopback_destroy(group)


def qb_destroy(ctx):
    if ctx is not None and ctx.value:
        lib().qb_destroy(ctx)


def qb_kernel_launches(ctx):
    return int(lib().qb_kernel_launches(ctx))


def qb_factor(ctx, A_ptr, m, n, lda, eps, b, q=0, seed=1, kmax=0, flags=0):
    """Raw call: returns dict(status, k, Q, ldq, B, ldb, resid) with device pointers."""
    k = ctypes.c_int64()
    Q = ctypes.c_void_p()
    ldq = ctypes.c_int64()
    B = ctypes.c_void_p()
    ldb = ctypes.c_int64()
    resid = ctypes.c_double()
    s = lib().qb_factor(ctx, ctypes.c_void_p(A_ptr), m, n, lda, float(eps), b, q, seed, kmax, flags,
                        ctypes.byref(k), ctypes.byref(Q), ctypes.byref(ldq), ctypes.byref(B), ctypes.byref(ldb),
                        ctypes.byref(resid))
    _check(ctx, s, ok=(QB_OK, QB_NOT_CONVERGED))
    return dict(status=s, k=k.value, Q=Q.value, ldq=ldq.value, B=B.value, ldb=ldb.value, resid=resid.value)


def qb_fixed_rank(ctx, A_ptr, m, n, lda, l, P=0, seed=1, flags=0, want_resid=True):
    """Raw call of the fixed-rank schemes randQB / randQB_p (see include/qb.h).
    Returns dict(Q, ldq, B, ldb, resid) with device pointers (resid None unless requested)."""
    Q, B = ctypes.c_void_p(), ctypes.c_void_p()
    ldq, ldb = ctypes.c_int64(), ctypes.c_int64()
    resid = ctypes.c_double()
    _check(ctx, lib().qb_fixed_rank(ctx, ctypes.c_void_p(A_ptr), m, n, lda, l, P, seed, flags, ctypes.byref(Q),
                                    ctypes.byref(ldq), ctypes.byref(B), ctypes.byref(ldb),
                                    ctypes.byref(resid) if want_resid else None))
    return dict(Q=Q.value, ldq=ldq.value, B=B.value, ldb=ldb.value, resid=resid.value if want_resid else None)


def qb_factor_host(ctx, A_host_ptr, m, n, lda, eps, b, q, seed, kmax, Q_host_ptr, ldq, B_host_ptr, ldb, kcap):
    """End-to-end call with host buffers (see include/qb.h).  Returns dict(status, k, resid)."""
    k = ctypes.c_int64()
    resid = ctypes.c_double()
    s = lib().qb_factor_host(ctx, ctypes.c_void_p(A_host_ptr), m, n, lda, float(eps), b, q, seed, kmax,
                             ctypes.byref(k), ctypes.c_void_p(Q_host_ptr), ldq, ctypes.c_void_p(B_host_ptr), ldb,
                             kcap, ctypes.byref(resid))
    _check(ctx, s, ok=(QB_OK, QB_NOT_CONVERGED))
    return dict(status=s, k=k.value, resid=resid.value)


def qb_stats(ctx):
    n = ctypes.c_int64()
    _check(ctx, lib().qb_stats(ctx, None, 0, ctypes.byref(n)))
    arr = (BlockStats * max(n.value, 1))()
    _check(ctx, lib().qb_stats(ctx, ctypes.cast(arr, ctypes.c_void_p), n.value, ctypes.byref(n)))
    return [dict(ell=a.ell, w=a.w, r2=a.r2, ei=a.ei, ms=a.ms, ms_sketch=a.ms_sketch, ms_bmat=a.ms_bmat,
                 ms_down=a.ms_down, fallback=a.fallback, ms_orth=a.ms_orth, ms_orth_z=a.ms_orth_z,
                 ms_reproj=a.ms_reproj, ms_power=a.ms_power, kappa_r=a.kappa_r) for a in arr[:n.value]]


def rqb_svd(ctx, kkeep=0, eps=0.0):
    """QB -> partial SVD of the context's last factorization (see include/qb.h).
    Returns dict(kk, U, ldu, S, V, ldv) of device pointers (context-owned); kk = the rank kept."""
    U, S, V = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    ldu, ldv, kk = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(ctx, lib().rqb_svd(ctx, float(eps), int(kkeep), ctypes.byref(kk), ctypes.byref(U), ctypes.byref(ldu),
                              ctypes.byref(S), ctypes.byref(V), ctypes.byref(ldv)))
    return dict(kk=kk.value, U=U.value or 0, ldu=ldu.value, S=S.value or 0, V=V.value or 0, ldv=ldv.value)


def qb_svd_sweeps(ctx):
    return int(lib().qb_svd_sweeps(ctx))


def qb_pivoted_qr(ctx, n):
    """QB -> partial pivoted QR of the context's last factorization (see include/qb.h).
    Returns dict(perm (numpy int64, n), Qh, ldqh, R, ldr) with device pointers."""
    import numpy as np
    perm = np.empty(n, dtype=np.int64)
    Qh, R = ctypes.c_void_p(), ctypes.c_void_p()
    ldq, ldr = ctypes.c_int64(), ctypes.c_int64()
    _check(ctx, lib().qb_pivoted_qr(ctx, ctypes.c_void_p(perm.ctypes.data), ctypes.byref(Qh), ctypes.byref(ldq),
                                    ctypes.byref(R), ctypes.byref(ldr)))
    return dict(perm=perm, Qh=Qh.value or 0, ldqh=ldq.value, R=R.value or 0, ldr=ldr.value)


def qb_omega(ctx, seed, row0, row1, col0, w, out_ptr, ldo):
    _check(ctx, lib().qb_omega(ctx, seed, row0, row1, col0, w, ctypes.c_void_p(out_ptr), ldo))


def qb_gemm(ctx, layout, epi, M, N, K, A_ptr, lda, B_ptr, ldb, C_ptr, ldc, split=True, want_sumsq=False):
    """Test hook over the library GEMM (see include/qb.h).  Returns ||.||_F^2 or None."""
    ss = ctypes.c_double()
    _check(ctx, lib().qb_gemm(ctx, layout, epi, M, N, K, ctypes.c_void_p(A_ptr), lda, ctypes.c_void_p(B_ptr), ldb,
                              ctypes.c_void_p(C_ptr), ldc, 1 if split else 0,
                              ctypes.byref(ss) if want_sumsq else None))
    return ss.value if want_sumsq else None


def qb_chol_rinv(ctx, G_ptr, ldg, w, m_rows, R_ptr, ldr):
    """Test hook: R^-1 (row-major) of the Cholesky factor of a Gram matrix.  Returns shifted flag."""
    sh = ctypes.c_int()
    _check(ctx, lib().qb_chol_rinv(ctx, ctypes.c_void_p(G_ptr), ldg, w, m_rows, ctypes.c_void_p(R_ptr), ldr,
                                   ctypes.byref(sh)))
    return sh.value


def qb_orth(ctx, X_ptr, m, w, ldx):
    _check(ctx, lib().qb_orth(ctx, ctypes.c_void_p(X_ptr), m, w, ldx))


# ------------------------------------------------------------------ torch convenience layer
class _CAI:
    """Expose a device pointer as a strided array to torch (no copy)."""

    def __init__(self, ptr, shape, strides_bytes, typestr="<f8"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "strides": tuple(strides_bytes),
                                         "typestr": typestr, "data": (int(ptr), False), "version": 3}


def view_colmajor(ptr, rows, cols, ld, typestr="<f8"):
    import torch
    es = 8 if typestr.endswith("8") else 4
    return torch.as_tensor(_CAI(ptr, (rows, cols), (es, es * ld), typestr), device="cuda")


def view_rowmajor(ptr, rows, cols, ld, typestr="<f8"):
    import torch
    es = 8 if typestr.endswith("8") else 4
    return torch.as_tensor(_CAI(ptr, (rows, cols), (es * ld, es), typestr), device="cuda")


class QB:
    """Owns one context (on torch's current stream of `device` unless `stream` is given).
    ``factor(A, eps, b, q, seed)`` with A a CUDA float64 tensor whose columns are contiguous
    (``A.stride(0) == 1``)."""

    def __init__(self, device=0, dtype=QB_F64, stream=None, dist=None):
        """dist: None, dict(rank, nranks, unique_id, col_offset, n_global) for a column-sharded
        context, or dict(shard="rows", rank, nranks, unique_id, row_offset, m_global) for a
        row-sharded one (see paper_1503_07157_b200.dist); with loopback=<qb_loopback_create()>
        instead of unique_id the ranks are in-process contexts on one GPU (one host thread each)."""
        # Default to torch's current stream on `device` so that the library's kernels are
        # stream-ordered after the torch work that produced their inputs.
        if stream is None:
            import torch
            h = torch.cuda.current_stream(device).cuda_stream
            stream = ctypes.c_void_p(h if h else 1)   # 0 (torch's default) -> cudaStreamLegacy
        if dist is None:
            self.ctx = qb_create(device, dtype, stream)
        elif dist.get("loopback") is not None:
            rows = dist.get("shard", "cols") == "rows"
            self.ctx = qb_create_sharded(device, dist["rank"], dist["nranks"],
                                         QB_SHARD_ROWS if rows else QB_SHARD_COLS,
                                         dist["row_offset"] if rows else dist["col_offset"],
                                         dist["m_global"] if rows else dist["n_global"], dtype, stream,
                                         loopback=dist["loopback"])
        else:
            if dist.get("shard", "cols") == "rows":
                self.ctx = qb_create_dist(device, dist["rank"], dist["nranks"], dist["unique_id"], dist["row_offset"],
                                          dist["m_global"], dtype, stream, rows=True)
            else:
                self.ctx = qb_create_dist(device, dist["rank"], dist["nranks"], dist["unique_id"],
                                          dist["col_offset"], dist["n_global"], dtype, stream)

    def close(self):
        qb_destroy(self.ctx)
        self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def factor(self, A, eps, b, q=0, seed=1, kmax=0, overwrite=False, copy_out=True, flags=0):
        import torch
        assert A.is_cuda and A.dtype in (torch.float64, torch.float32) and A.dim() == 2 and (A.stride(0) == 1 or A.numel() == 0)
        m, n = A.shape
        r = qb_factor(self.ctx, A.data_ptr(), m, n, max(A.stride(1) if n > 1 else m, 1), eps, b, q, seed, kmax,
                      (QB_OVERWRITE_A if overwrite else 0) | flags)
        k = r["k"]
        ts = "<f8" if A.dtype == torch.float64 else "<f4"
        Q = view_colmajor(r["Q"], m, k, r["ldq"], ts) if k > 0 else torch.zeros(m, 0, dtype=A.dtype, device=A.device)
        B = view_rowmajor(r["B"], k, n, r["ldb"], ts) if k > 0 else torch.zeros(0, n, dtype=A.dtype, device=A.device)
        if copy_out:
            Q, B = Q.clone(), B.clone()
        self._last = (m, n, k, A.dtype)
        return dict(status=r["status"], k=k, Q=Q, B=B, resid=r["resid"], stats=qb_stats(self.ctx))

    def fixed_rank(self, A, l, P=0, seed=1, overwrite=False, flags=0, want_resid=True, copy_out=True):
        """randQB (P = 0, Fig. 1) / randQB_p (Fig. 3): Q (m x l), B (l x n) for a fixed rank l."""
        import torch
        assert A.is_cuda and A.dtype in (torch.float64, torch.float32) and A.dim() == 2 and A.stride(0) == 1
        m, n = A.shape
        r = qb_fixed_rank(self.ctx, A.data_ptr(), m, n, A.stride(1) if n > 1 else m, l, P, seed,
                          (QB_OVERWRITE_A if overwrite else 0) | flags, want_resid)
        ts = "<f8" if A.dtype == torch.float64 else "<f4"
        Q = view_colmajor(r["Q"], m, l, r["ldq"], ts)
        B = view_rowmajor(r["B"], l, n, r["ldb"], ts)
        if copy_out:
            Q, B = Q.clone(), B.clone()
        self._last = (m, n, l, A.dtype)
        return dict(Q=Q, B=B, resid=r["resid"])

    def pivoted_qr(self, copy_out=True):
        """A P ~ Qh R from the last ``factor`` / ``fixed_rank``: returns
        dict(perm, Qh (m x k), R (k x n upper trapezoidal)); column j of A P is column perm[j] of A."""
        import torch
        if getattr(self, "_last", None) is None:
            qb_pivoted_qr(self.ctx, 0)  # raises QBError: no factorization yet
        m, n, k, dt = self._last
        r = qb_pivoted_qr(self.ctx, n)
        ts = "<f8" if dt == torch.float64 else "<f4"
        if k == 0:
            return dict(perm=r["perm"], Qh=torch.zeros(m, 0, dtype=dt, device="cuda"),
                        R=torch.zeros(0, n, dtype=dt, device="cuda"))
        Qh = view_colmajor(r["Qh"], m, k, r["ldqh"], ts)
        R = view_rowmajor(r["R"], k, n, r["ldr"], ts)
        if copy_out:
            Qh, R = Qh.clone(), R.clone()
        return dict(perm=r["perm"], Qh=Qh, R=R)

    def svd(self, kkeep=0, eps=0.0, copy_out=True):
        """Partial SVD A ~ U diag(S) V^T from the last ``factor`` (rqb_svd):
        U m x k', S k', V n x k' with k' from kkeep and / or the tail rule with eps (include/qb.h)."""
        import torch
        r = rqb_svd(self.ctx, kkeep, eps)  # raises QBError without a prior factorization
        m, n, k, dt = self._last
        kk = r["kk"] if k > 0 else 0
        ts = "<f8" if dt == torch.float64 else "<f4"
        if kk == 0:
            z = lambda *s: torch.zeros(*s, dtype=dt, device="cuda")  # noqa: E731
            return dict(U=z(m, 0), S=z(0), V=z(n, 0), kk=0)
        U = view_colmajor(r["U"], m, kk, r["ldu"], ts)
        S = view_colmajor(r["S"], kk, 1, kk, ts)[:, 0]
        V = view_colmajor(r["V"], n, kk, r["ldv"], ts)
        if copy_out:
            U, S, V = U.clone(), S.clone(), V.clone()
        return dict(U=U, S=S, V=V, kk=kk)

    def launches(self):
        return qb_kernel_launches(self.ctx)
