"""paper_2209_04626_b200 -- B200-native mixed-precision one-sided Jacobi SVD.

Thin ctypes binding over the C-ABI of libmpjsvd.so (include/mpjsvd.h).  The
binding only marshals arguments: every step of the SVD runs in the library's
sm_100a kernels.  torch is used for device memory and streams only.  There
is no CPU fallback: if libmpjsvd.so cannot be loaded, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmpjsvd.so")

OK = 0
WARN_NOT_CONVERGED = 1
PATH_FORCE_MIXED = 0
PATH_FORCE_FP64 = 2
STAGES = ("qr_tall", "qrp", "lq", "gates", "fp32", "lift", "fp64", "assemble")


class MpjsvdError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        msg = f"mpjsvd error {code}: {strerror(code)}"
        if code == -4:
            msg += f" [{last_cuda_error()}]"
        if what:
            msg = f"{what}: {msg}"
        super().__init__(msg)


class Options(C.Structure):
    _fields_ = [("num_gpus", C.c_int32), ("device_id", C.c_int32), ("block_cols", C.c_int32),
                ("tol_mult32", C.c_double), ("tol_mult64", C.c_double), ("inner_tol_div", C.c_int32),
                ("max_sweeps32", C.c_int32), ("max_sweeps64", C.c_int32), ("max_inner", C.c_int32),
                ("path", C.c_int32), ("x_from_lq", C.c_int32), ("compute_gates", C.c_int32),
                ("stream", C.c_void_p), ("virtual_shards", C.c_int32), ("split_rows", C.c_int32),
                ("fp32_tensor_cores", C.c_int32), ("pdl_overlap", C.c_int32),
                ("mp_rrqr", C.c_int32), ("max_inner32", C.c_int32), ("switch_u", C.c_int32),
                ("tol_orth", C.c_double), ("tol_alg", C.c_double), ("tol_cond_mult", C.c_double),
                ("cond_d_min", C.c_double), ("tail_frac", C.c_double), ("tail_cut_log2", C.c_int32),
                ("gram_tma", C.c_int32), ("gram_kt", C.c_int32), ("gram_variant", C.c_int32),
                ("update_tpc", C.c_int32), ("skip_unchanged", C.c_int32), ("qr_panel_mode", C.c_int32),
                ("diag_timing", C.c_int32), ("refine_v", C.c_int32), ("update_variant", C.c_int32),
                ("qrp_panel_stages", C.c_int32), ("gram_pdl", C.c_int32), ("l2_order", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("path_taken", C.c_int32), ("sweeps32", C.c_int32), ("sweeps64", C.c_int32),
                ("converged", C.c_int32), ("stage_ms", C.c_double * 8), ("total_ms", C.c_double),
                ("orth_measure", C.c_double), ("tail_fraction", C.c_double),
                ("cond_estimate", C.c_double), ("final_off32", C.c_double), ("final_off64", C.c_double),
                ("off_trace32", C.c_double * 32), ("off_trace64", C.c_double * 32),
                ("upd_trace32", C.c_int32 * 32), ("upd_trace64", C.c_int32 * 32),
                ("kernel_launches", C.c_int64),
                ("inner_max_trace32", C.c_int32 * 32), ("inner_max_trace64", C.c_int32 * 32),
                ("inner_sum_trace32", C.c_int32 * 32), ("inner_sum_trace64", C.c_int32 * 32),
                ("skip_trace32", C.c_int32 * 32), ("skip_trace64", C.c_int32 * 32),
                ("cond_scaled", C.c_double), ("cond_d", C.c_double), ("v_sweeps64", C.c_int32)]

    def as_dict(self) -> dict:
        s32, s64 = self.sweeps32, self.sweeps64
        return {
            "path_taken": self.path_taken, "sweeps32": s32, "sweeps64": s64,
            "converged": bool(self.converged),
            "stage_ms": dict(zip(STAGES, list(self.stage_ms))), "total_ms": self.total_ms,
            "orth_measure": self.orth_measure, "tail_fraction": self.tail_fraction,
            "cond_estimate": self.cond_estimate, "final_off32": self.final_off32,
            "cond_scaled": self.cond_scaled, "cond_d": self.cond_d, "v_sweeps64": self.v_sweeps64,
            "final_off64": self.final_off64,
            "off_trace32": list(self.off_trace32[:min(s32, 32)]),
            "off_trace64": list(self.off_trace64[:min(s64, 32)]),
            "upd_trace32": list(self.upd_trace32[:min(s32, 32)]),
            "upd_trace64": list(self.upd_trace64[:min(s64, 32)]),
            "kernel_launches": int(self.kernel_launches),
            "inner_max_trace32": list(self.inner_max_trace32[:min(s32, 32)]),
            "inner_max_trace64": list(self.inner_max_trace64[:min(s64, 32)]),
            "inner_sum_trace32": list(self.inner_sum_trace32[:min(s32, 32)]),
            "inner_sum_trace64": list(self.inner_sum_trace64[:min(s64, 32)]),
            "skip_trace32": list(self.skip_trace32[:min(s32, 32)]),
            "skip_trace64": list(self.skip_trace64[:min(s64, 32)]),
        }


_lock = threading.Lock()
_lib = None

EXPORTS = [
    "mpjsvd_default_options", "mpjsvd_create", "mpjsvd_factor", "mpjsvd_destroy", "mpjsvd_strerror",
    "mpjsvd_last_cuda_error", "mpjsvd_version", "mpjsvd_block_jacobi_f64", "mpjsvd_block_jacobi_f32",
    "mpjsvd_inner_solve", "mpjsvd_qr", "mpjsvd_lift", "mpjsvd_switch_u", "mpjsvd_qrsvd32", "mpjsvd_apply_q", "mpjsvd_gemm_f64",
    "mpjsvd_set_profiling", "mpjsvd_get_profile", "mpjsvd_comm_unique_id", "mpjsvd_comm_init",
    "mpjsvd_comm_info", "mpjsvd_plan_create", "mpjsvd_plan_info", "mpjsvd_plan_pairs", "mpjsvd_plan_advance",
    "mpjsvd_plan_locate", "mpjsvd_plan_destroy",
]
COMM_ID_BYTES = 128


def lib():
    """Load libmpjsvd.so (raises if it is missing: there is no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2209_04626_b200.build` "
                              "(nvcc, sm_100a). No CPU fallback exists.")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.mpjsvd_default_options.argtypes = [C.POINTER(Options)]
        L.mpjsvd_create.argtypes = [C.POINTER(vp), C.POINTER(Options)]
        L.mpjsvd_factor.argtypes = [vp, vp, i64, i64, i64, vp, i64, vp, vp, i64, C.POINTER(Stats)]
        L.mpjsvd_destroy.argtypes = [vp]
        L.mpjsvd_strerror.argtypes = [C.c_int]
        L.mpjsvd_strerror.restype = C.c_char_p
        L.mpjsvd_last_cuda_error.restype = C.c_char_p
        L.mpjsvd_block_jacobi_f64.argtypes = [vp, vp, i64, i64, i64, vp, i64, i64, dbl, dbl, i32,
                                              C.POINTER(i32), C.POINTER(Stats)]
        L.mpjsvd_block_jacobi_f32.argtypes = [vp, vp, i64, i64, i64, vp, i64, i64, C.c_float,
                                              C.c_float, i32, i32, C.POINTER(i32), C.POINTER(Stats)]
        L.mpjsvd_inner_solve.argtypes = [vp, i32, vp, vp, i32, i32, dbl, i32, vp]
        L.mpjsvd_qr.argtypes = [vp, vp, i64, i64, i64, vp, vp, i32]
        L.mpjsvd_lift.argtypes = [vp, vp, i64, i64, vp, i64]
        L.mpjsvd_switch_u.argtypes = [vp, vp, i64, i64, vp, i64, vp, i64, i32]
        L.mpjsvd_apply_q.argtypes = [vp, vp, i64, i64, i64, vp, vp, i64, i64]
        L.mpjsvd_qrsvd32.argtypes = [vp, vp, i64, i64, vp, i64, vp]
        L.mpjsvd_gemm_f64.argtypes = [vp, i32, i32, i64, i64, i64, dbl, vp, i64, vp, i64, dbl, vp, i64]
        L.mpjsvd_set_profiling.argtypes = [vp, i32]
        L.mpjsvd_get_profile.argtypes = [vp, i32, C.c_char_p, i32, C.POINTER(dbl), C.POINTER(i64)]
        L.mpjsvd_comm_unique_id.argtypes = [vp]
        L.mpjsvd_comm_init.argtypes = [vp, i32, i32, vp]
        L.mpjsvd_comm_info.argtypes = [vp, C.POINTER(i32), C.POINTER(i32)]
        L.mpjsvd_plan_create.argtypes = [C.POINTER(vp), i32, i32]
        L.mpjsvd_plan_info.argtypes = [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]
        L.mpjsvd_plan_pairs.argtypes = [vp, i32, vp]
        L.mpjsvd_plan_advance.argtypes = [vp, vp, i32]
        L.mpjsvd_plan_locate.argtypes = [vp, i32, C.POINTER(i32), C.POINTER(i32)]
        L.mpjsvd_plan_destroy.argtypes = [vp]
        _lib = L
        return L


def strerror(code: int) -> str:
    return lib().mpjsvd_strerror(code).decode()


def last_cuda_error() -> str:
    return lib().mpjsvd_last_cuda_error().decode()


def _check(rc: int, what: str = "", allow_warn: bool = True) -> int:
    if rc < 0 or (rc > 0 and not allow_warn):
        raise MpjsvdError(rc, what)
    return rc


def default_options(**kw) -> Options:
    o = Options()
    lib().mpjsvd_default_options(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


class Handle:
    """Owns an mpjsvd handle (device workspaces, stream, events)."""

    def __init__(self, stream=None, **opts):
        o = default_options(**opts)
        if stream is not None:
            o.stream = C.c_void_p(int(stream))
        self._h = C.c_void_p()
        _check(lib().mpjsvd_create(C.byref(self._h), C.byref(o)), "mpjsvd_create")
        self.options = o

    def close(self):
        if self._h:
            lib().mpjsvd_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def ptr(self):
        return self._h

    def comm_init(self, rank: int, world: int, uid: bytes):
        """Attach an NCCL communicator (multi-GPU, one process per GPU).  uid
        is comm_unique_id() of rank 0, distributed by the caller."""
        if len(uid) != COMM_ID_BYTES:
            raise ValueError("unique id must be 128 bytes")
        buf = C.create_string_buffer(uid, COMM_ID_BYTES)
        _check(lib().mpjsvd_comm_init(self._h, rank, world, buf), "mpjsvd_comm_init")

    def comm_info(self):
        r, w = C.c_int32(), C.c_int32()
        _check(lib().mpjsvd_comm_info(self._h, C.byref(r), C.byref(w)))
        return r.value, w.value

    def comm_init_torch(self, group=None):
        """comm_init over an initialised torch.distributed group (rank 0's
        NCCL unique id is broadcast with broadcast_object_list)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        self.comm_init(rank, world, obj[0])

    def set_profiling(self, on: bool = True):
        _check(lib().mpjsvd_set_profiling(self._h, int(on)), "mpjsvd_set_profiling")

    def profile(self) -> dict:
        """{kernel name: (summed device ms, launches)} since set_profiling(True)."""
        L = lib()
        n = L.mpjsvd_get_profile(self._h, -1, None, 0, None, None)
        out = {}
        for i in range(max(n, 0)):
            buf = C.create_string_buffer(64)
            ms = C.c_double()
            cnt = C.c_int64()
            L.mpjsvd_get_profile(self._h, i, buf, 64, C.byref(ms), C.byref(cnt))
            out[buf.value.decode()] = (ms.value, cnt.value)
        return out


def comm_unique_id() -> bytes:
    """NCCL unique id (rank 0) for Handle.comm_init."""
    buf = C.create_string_buffer(COMM_ID_BYTES)
    _check(lib().mpjsvd_comm_unique_id(buf), "mpjsvd_comm_unique_id")
    return buf.raw


class ShardPlan:
    """The library's host-side shard plan (include/mpjsvd.h mpjsvd_plan_*):
    the round-robin schedule over `world` ranks and the block moves of every
    round.  Host only (no GPU)."""

    def __init__(self, nblk: int, world: int):
        self._p = C.c_void_p()
        _check(lib().mpjsvd_plan_create(C.byref(self._p), nblk, world), "mpjsvd_plan_create")
        M, k, nb = C.c_int32(), C.c_int32(), C.c_int32()
        lib().mpjsvd_plan_info(self._p, C.byref(M), C.byref(k), C.byref(nb))
        self.nblk, self.world, self.M, self.k, self.nbuf = nblk, world, M.value, k.value, nb.value

    def pairs(self, rank: int):
        """[(buf0, buf1, blk0, blk1)] of the rank's k local pairs this round."""
        out = (C.c_int32 * (4 * self.k))()
        _check(lib().mpjsvd_plan_pairs(self._p, rank, out), "mpjsvd_plan_pairs")
        return [tuple(out[4 * t:4 * t + 4]) for t in range(self.k)]

    def advance(self):
        """Apply one round's shift; [(blk, src_rank, src_buf, dst_rank, dst_buf)]."""
        cap = 4 * self.world + 8
        out = (C.c_int32 * (5 * cap))()
        cnt = lib().mpjsvd_plan_advance(self._p, out, cap)
        _check(cnt, "mpjsvd_plan_advance")
        assert cnt <= cap
        return [tuple(out[5 * i:5 * i + 5]) for i in range(cnt)]

    def locate(self, blk: int):
        r, b = C.c_int32(), C.c_int32()
        _check(lib().mpjsvd_plan_locate(self._p, blk, C.byref(r), C.byref(b)), "mpjsvd_plan_locate")
        return r.value, b.value

    def __del__(self):
        try:
            if self._p:
                lib().mpjsvd_plan_destroy(self._p)
                self._p = C.c_void_p()
        except Exception:
            pass


def _col_major(t):
    """(rows, cols) torch tensor -> column-major fp64 storage (stride (1, ld))."""
    import torch
    if t.dtype != torch.float64:
        raise TypeError("mpjsvd expects float64")
    if t.dim() != 2:
        raise ValueError("expected a matrix")
    if t.stride(0) == 1 and t.stride(1) >= max(1, t.shape[0]):
        return t, t.stride(1)
    ct = t.t().contiguous().t()
    return ct, max(1, ct.stride(1))


def empty_col_major(rows: int, cols: int, dtype, device):
    import torch
    return torch.empty((cols, rows), dtype=dtype, device=device).t()


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p()


def mpjsvd_factor(handle: Handle, A, U, S, V, m: int, n: int, lda: int, ldu: int, ldv: int):
    """Raw C-ABI call on pointers (device tensors or host tensors; None for
    the non-root ranks of a multi-GPU handle).  Returns (rc, stats)."""
    st = Stats()
    rc = lib().mpjsvd_factor(handle.ptr, _ptr(A), m, n, lda, _ptr(U), ldu, _ptr(S), _ptr(V), ldv, C.byref(st))
    return rc, st


def factor(A, handle: Handle | None = None, **opts):
    """SVD of the m x n (m >= n) float64 tensor A (device or host).

    Returns (U m x n, S n, V n x n, stats dict) on A's device; U and V are
    column-major views.  Raises MpjsvdError on errors; a non-converged fp64
    stage is reported in stats['converged'] (return code 1).
    """
    import torch
    own = handle is None
    if own:
        if A.is_cuda:
            # bind the handle to A's device and that device's current stream (not the current device's)
            opts.setdefault("device_id", A.device.index)
            stream = torch.cuda.current_stream(A.device).cuda_stream
        else:
            stream = None
        handle = Handle(stream=stream, **opts)
    try:
        Ac, lda = _col_major(A)
        m, n = Ac.shape
        dev = Ac.device
        U = empty_col_major(m, n, torch.float64, dev)
        V = empty_col_major(n, n, torch.float64, dev)
        S = torch.empty(n, dtype=torch.float64, device=dev)
        rc, st = mpjsvd_factor(handle, Ac, U, S, V, m, n, lda, max(1, m), max(1, n))
        _check(rc, "mpjsvd_factor")
        d = st.as_dict()
        d["rc"] = rc
        return U, S, V, d
    finally:
        if own:
            handle.close()


def block_jacobi(X, V=None, tol: float = 0.0, tol_in: float = 0.0, max_sweeps: int = 30,
                 stagnation: bool = False, handle: Handle | None = None, **opts):
    """Step-level: block round-robin Jacobi (fp64 or fp32 by X.dtype) in place
    on device tensors X (m x n) and V (nv x n).  Returns (sweeps, stats)."""
    import torch
    own = handle is None
    if own:
        handle = Handle(stream=torch.cuda.current_stream().cuda_stream, **opts)
    try:
        m, n = X.shape
        assert X.stride(0) == 1 and (V is None or V.stride(0) == 1)
        sw = C.c_int32(0)
        st = Stats()
        vptr = C.c_void_p(V.data_ptr()) if V is not None else C.c_void_p()
        nv = V.shape[0] if V is not None else 0
        ldv = V.stride(1) if V is not None else 1
        if X.dtype == torch.float64:
            rc = lib().mpjsvd_block_jacobi_f64(handle.ptr, C.c_void_p(X.data_ptr()), m, n, X.stride(1), vptr, nv,
                                               ldv, tol, tol_in, max_sweeps, C.byref(sw), C.byref(st))
        else:
            rc = lib().mpjsvd_block_jacobi_f32(handle.ptr, C.c_void_p(X.data_ptr()), m, n, X.stride(1), vptr, nv,
                                               ldv, tol, tol_in, max_sweeps, int(stagnation), C.byref(sw),
                                               C.byref(st))
        _check(rc, "mpjsvd_block_jacobi")
        return sw.value, st.as_dict()
    finally:
        if own:
            handle.close()


def inner_solve(G, tol_in: float, max_inner: int = 30, handle: Handle | None = None):
    """Step-level: batched 2b x 2b inner solve on device tensor G (count, w, w).
    Returns (G_out, E, rotations)."""
    import torch
    own = handle is None
    if own:
        handle = Handle(stream=torch.cuda.current_stream().cuda_stream)
    try:
        G = G.clone().contiguous()
        count, w, _ = G.shape
        E = torch.zeros_like(G)
        rot = (C.c_int32 * count)()
        rc = lib().mpjsvd_inner_solve(handle.ptr, int(G.dtype == torch.float64), C.c_void_p(G.data_ptr()),
                                      C.c_void_p(E.data_ptr()), w, count, tol_in, max_inner, rot)
        _check(rc, "mpjsvd_inner_solve")
        # kernel wrote column-major w x w blocks: transpose back to (row, col)
        return G.transpose(1, 2), E.transpose(1, 2), list(rot)
    finally:
        if own:
            handle.close()


def qr(A, pivot: int = 1, handle: Handle | None = None, **opts):
    """Step-level: Householder QR on a copy of a device fp64 tensor.
    pivot = 1: column-pivoted (lazy cooperative kernel of the path), 2: the
    unblocked pivoted kernel, 0: blocked unpivoted QR.  Returns (packed, tau, perm)."""
    import torch
    own = handle is None
    if own:
        handle = Handle(stream=torch.cuda.current_stream().cuda_stream, **opts)
    try:
        Ac, lda = _col_major(A.clone())
        m, n = Ac.shape
        tau = torch.empty(n, dtype=torch.float64, device=Ac.device)
        perm = torch.empty(n, dtype=torch.int32, device=Ac.device)
        rc = lib().mpjsvd_qr(handle.ptr, C.c_void_p(Ac.data_ptr()), m, n, lda, C.c_void_p(tau.data_ptr()),
                             C.c_void_p(perm.data_ptr()), int(pivot))
        _check(rc, "mpjsvd_qr")
        return Ac, tau, perm
    finally:
        if own:
            handle.close()


def lift(V32, handle: Handle | None = None):
    """Step-level: Q = qr(fl64(V32)) by CholeskyQR on device."""
    import torch
    own = handle is None
    if own:
        handle = Handle(stream=torch.cuda.current_stream().cuda_stream)
    try:
        n = V32.shape[0]
        Vc = V32.t().contiguous().t()
        Q = empty_col_major(n, n, torch.float64, V32.device)
        rc = lib().mpjsvd_lift(handle.ptr, C.c_void_p(Vc.data_ptr()), n, Vc.stride(1), C.c_void_p(Q.data_ptr()),
                               Q.stride(1))
        _check(rc, "mpjsvd_lift")
        return Q
    finally:
        if own:
            handle.close()


def switch_u(X, Ulow, x_lower: bool = True, handle: Handle | None = None):
    """Step-level: U-route switch Q = qr(X^T Ulow) on device."""
    import torch
    own = handle is None
    if own:
        handle = Handle(stream=torch.cuda.current_stream().cuda_stream)
    try:
        n = X.shape[0]
        Xc = X.t().contiguous().t()
        Uc = Ulow.t().contiguous().t()
        Q = empty_col_major(n, n, torch.float64, X.device)
        rc = lib().mpjsvd_switch_u(handle.ptr, C.c_void_p(Xc.data_ptr()), n, Xc.stride(1),
                                   C.c_void_p(Uc.data_ptr()), Uc.stride(1), C.c_void_p(Q.data_ptr()), Q.stride(1),
                                   int(x_lower))
        _check(rc, "mpjsvd_switch_u")
        return Q
    finally:
        if own:
            handle.close()


def qrsvd32(X32, handle: Handle | None = None):
    """Step-level: the fp32 QR SVD of the AUTO branch (U only; reading c-24) of a device fp32 n x n tensor.
    Returns (U fp64 n x n column-major, S fp32 descending)."""
    import torch
    own = handle is None
    if own:
        handle = Handle(stream=torch.cuda.current_stream().cuda_stream)
    try:
        n = X32.shape[0]
        Xc = X32.t().contiguous().t()
        U = empty_col_major(n, n, torch.float64, X32.device)
        S = torch.empty(n, dtype=torch.float32, device=X32.device)
        rc = lib().mpjsvd_qrsvd32(handle.ptr, C.c_void_p(Xc.data_ptr()), n, Xc.stride(1), C.c_void_p(U.data_ptr()),
                                  U.stride(1), C.c_void_p(S.data_ptr()))
        _check(rc, "mpjsvd_qrsvd32")
        return U, S
    finally:
        if own:
            handle.close()


def apply_q(packed, tau, Cmat, handle: Handle | None = None):
    """Step-level: C <- Q C with Q = H_0 ... H_{k-1} packed as returned by qr()."""
    import torch
    own = handle is None
    if own:
        handle = Handle(stream=torch.cuda.current_stream().cuda_stream)
    try:
        Pc, ldp = _col_major(packed)
        Cc, ldc = _col_major(Cmat.clone())
        m = Pc.shape[0]
        rc = lib().mpjsvd_apply_q(handle.ptr, C.c_void_p(Pc.data_ptr()), m, tau.numel(), ldp,
                                  C.c_void_p(tau.data_ptr()), C.c_void_p(Cc.data_ptr()), ldc, Cc.shape[1])
        _check(rc, "mpjsvd_apply_q")
        return Cc
    finally:
        if own:
            handle.close()


def gemm(transa: bool, transb: bool, A, B, alpha: float = 1.0, handle: Handle | None = None):
    """Step-level: alpha op(A) op(B) with the library's fp64 GEMM."""
    import torch
    own = handle is None
    if own:
        handle = Handle(stream=torch.cuda.current_stream().cuda_stream)
    try:
        Ac, lda = _col_major(A)
        Bc, ldb = _col_major(B)
        M = Ac.shape[1] if transa else Ac.shape[0]
        K = Ac.shape[0] if transa else Ac.shape[1]
        N = Bc.shape[0] if transb else Bc.shape[1]
        Cm = empty_col_major(M, N, torch.float64, A.device)
        rc = lib().mpjsvd_gemm_f64(handle.ptr, int(transa), int(transb), M, N, K, alpha, C.c_void_p(Ac.data_ptr()),
                                   lda, C.c_void_p(Bc.data_ptr()), ldb, 0.0, C.c_void_p(Cm.data_ptr()),
                                   max(1, M))
        _check(rc, "mpjsvd_gemm_f64")
        return Cm
    finally:
        if own:
            handle.close()
