"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the mixed-precision
one-sided Jacobi SVD (arXiv 2209.04626).

Only tests/, __graft_entry__.smoke() and bench.py's `cpu_baseline` leg (and
`bench.py --impl reference`) may import this package.  The product path
(paper_2209_04626_b200) never does; the two share no code.

O-MIX (`mixed_svd`) follows Algorithm 3 step by step in
plain C (omix.c); O-CYC (`cyclic_svd`) is the textbook Algorithm 1
 in fp64 with the row-cyclic order of eq. (2.1), run on
X = L from a LAPACK (scipy) QRP + LQ.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRCS = ["omix.c", "ocyc.c", "qrsvd.c"]
_DEPS = _SRCS + ["bj_impl.inc", "oracle.h"]
_lock = threading.Lock()
_lib = None

U64 = 2.0 ** -53
U32 = 2.0 ** -24


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc -O2 -ffp-contract=off -fopenmp (c-14)."""
    newest = max(os.path.getmtime(os.path.join(_HERE, f)) for f in _DEPS)
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= newest:
        return _SO
    tmp = _SO + f".{os.getpid()}.tmp"
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
           "-std=c11", "-o", tmp] + [os.path.join(_HERE, s) for s in _SRCS] + ["-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, _SO)
    return _SO


class Opts(C.Structure):
    _fields_ = [("b", C.c_int32), ("tol_mult32", C.c_double), ("tol_mult64", C.c_double),
                ("inner_tol_div", C.c_int32), ("max_sweeps32", C.c_int32),
                ("max_sweeps64", C.c_int32), ("max_inner", C.c_int32), ("path", C.c_int32),
                ("x_from_lq", C.c_int32), ("nthreads", C.c_int32), ("mp_rrqr", C.c_int32),
                ("max_inner32", C.c_int32), ("switch_u", C.c_int32),
                ("tol_orth", C.c_double), ("tol_alg", C.c_double), ("tol_cond_mult", C.c_double),
                ("cond_d_min", C.c_double), ("tail_frac", C.c_double), ("tail_cut_log2", C.c_int32),
                ("refine_v", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("sweeps32", C.c_int32), ("sweeps64", C.c_int32), ("converged", C.c_int32),
                ("path_taken", C.c_int32), ("orth_measure", C.c_double),
                ("tail_fraction", C.c_double), ("cond_estimate", C.c_double),
                ("final_off32", C.c_double), ("final_off64", C.c_double),
                ("off_trace32", C.c_double * 64), ("off_trace64", C.c_double * 64),
                ("upd_trace32", C.c_int32 * 64), ("upd_trace64", C.c_int32 * 64),
                ("perm", C.c_int32 * 1), ("cond_scaled", C.c_double), ("cond_d", C.c_double),
                ("v_sweeps64", C.c_int32)]

    def as_dict(self) -> dict:
        s32, s64 = self.sweeps32, self.sweeps64
        return {
            "sweeps32": s32, "sweeps64": s64, "converged": bool(self.converged),
            "orth_measure": self.orth_measure, "tail_fraction": self.tail_fraction,
            "cond_estimate": self.cond_estimate, "final_off32": self.final_off32,
            "path_taken": self.path_taken, "cond_scaled": self.cond_scaled, "cond_d": self.cond_d,
            "v_sweeps64": self.v_sweeps64,
            "final_off64": self.final_off64,
            "off_trace32": list(self.off_trace32[:min(s32, 64)]),
            "off_trace64": list(self.off_trace64[:min(s64, 64)]),
            "upd_trace32": list(self.upd_trace32[:min(s32, 64)]),
            "upd_trace64": list(self.upd_trace64[:min(s64, 64)]),
        }


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            dp = C.POINTER(C.c_double)
            fp = C.POINTER(C.c_float)
            ip = C.POINTER(C.c_int32)
            i64 = C.c_int64
            L.om_default_opts.argtypes = [C.POINTER(Opts)]
            L.om_house.argtypes = [dp, i64]
            L.om_house.restype = C.c_double
            L.om_qr.argtypes = [dp, i64, i64, i64, dp]
            L.om_qrp.argtypes = [dp, i64, i64, i64, ip, dp]
            L.om_qrp_f32.argtypes = [fp, i64, i64, i64, ip, fp]
            L.om_mprrqr.argtypes = [dp, i64, i64, i64, ip, dp]
            L.om_apply_q.argtypes = [dp, i64, i64, i64, dp, dp, i64, i64]
            L.om_inner_solve_f64.argtypes = [dp, C.c_int32, C.c_double, C.c_int32, dp, ip]
            L.om_inner_solve_f64.restype = C.c_int64
            L.om_inner_solve_f32.argtypes = [fp, C.c_int32, C.c_float, C.c_int32, fp, ip]
            L.om_inner_solve_f32.restype = C.c_int64
            L.om_block_jacobi_f64.argtypes = [dp, i64, i64, i64, dp, i64, i64, C.c_int32, C.c_double,
                                              C.c_double, C.c_int32, C.c_int32, dp, ip, C.c_int32]
            L.om_block_jacobi_f64.restype = C.c_int32
            L.om_block_jacobi_f32.argtypes = [fp, i64, i64, i64, fp, i64, i64, C.c_int32, C.c_float,
                                              C.c_float, C.c_int32, C.c_int32, C.c_int32, dp, ip,
                                              C.c_int32]
            L.om_block_jacobi_f32.restype = C.c_int32
            L.om_lift.argtypes = [fp, i64, i64, dp, i64]
            L.om_switch_u.argtypes = [dp, i64, i64, dp, i64, dp, i64]
            L.om_mixed_svd.argtypes = [dp, i64, i64, i64, C.POINTER(Opts), dp, i64, dp, dp, i64,
                                       C.POINTER(Stats)]
            L.om_gate_orth.argtypes = [dp, i64, i64, fp]
            L.om_gate_orth.restype = C.c_double
            L.om_gate_tail.argtypes = [dp, i64, i64, C.c_int32]
            L.om_gate_tail.restype = C.c_double
            L.om_gate_cond_scaled.argtypes = [dp, i64, i64, dp]
            L.om_gate_cond_scaled.restype = C.c_double
            L.om_gate_cond_d.argtypes = [dp, i64]
            L.om_gate_cond_d.restype = C.c_double
            L.oc_cyclic_jacobi.argtypes = [dp, i64, i64, i64, dp, i64, C.c_double, C.c_int32,
                                           C.POINTER(C.c_int64)]
            L.oc_cyclic_jacobi.restype = C.c_int32
            L.om_qrsvd32.argtypes = [fp, i64, i64, dp, i64, fp]
            _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def default_opts(**kw) -> Opts:
    o = Opts()
    lib().om_default_opts(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def tol(n: int, mult: float = 4.0, u: float = U64) -> float:
    """eps_tol = mult * sqrt(n) * u (reading c-1)."""
    return mult * np.sqrt(n) * u


# ---------------------------------------------------------------- wrappers
def house(x: np.ndarray):
    x = np.array(x, dtype=np.float64)
    t = lib().om_house(_dp(x), x.size)
    return x, t


def qr(a: np.ndarray):
    """Unpivoted Householder QR in place (returns packed factor, tau)."""
    a = np.array(a, dtype=np.float64, order="F")
    m, n = a.shape
    tau = np.zeros(n)
    rc = lib().om_qr(_dp(a), m, n, m, _dp(tau))
    return a, tau, rc


def qrp(a: np.ndarray):
    a = np.array(a, dtype=np.float64, order="F")
    m, n = a.shape
    tau = np.zeros(n)
    perm = np.zeros(n, dtype=np.int32)
    rc = lib().om_qrp(_dp(a), m, n, m, _ip(perm), _dp(tau))
    return a, perm, tau, rc


def qrp_f32(a: np.ndarray):
    """Businger-Golub QRP entirely in fp32 (Alg. 4 line 2)."""
    a = np.array(a, dtype=np.float32, order="F")
    m, n = a.shape
    tau = np.zeros(n, dtype=np.float32)
    perm = np.zeros(n, dtype=np.int32)
    rc = lib().om_qrp_f32(_fp(a), m, n, m, _ip(perm), _fp(tau))
    return a, perm, tau, rc


def mprrqr(a: np.ndarray):
    """Mixed-precision RRQR (Alg. 4): packed R / reflectors of A P, perm, tau."""
    a = np.array(a, dtype=np.float64, order="F")
    m, n = a.shape
    tau = np.zeros(n)
    perm = np.zeros(n, dtype=np.int32)
    rc = lib().om_mprrqr(_dp(a), m, n, m, _ip(perm), _dp(tau))
    return a, perm, tau, rc


def apply_q(packed: np.ndarray, tau: np.ndarray, c: np.ndarray) -> np.ndarray:
    packed = np.asfortranarray(packed, dtype=np.float64)
    c = np.array(c, dtype=np.float64, order="F")
    m = packed.shape[0]
    k = tau.size
    lib().om_apply_q(_dp(packed), m, k, m, _dp(np.ascontiguousarray(tau)), _dp(c), m, c.shape[1])
    return c


def form_q(packed: np.ndarray, tau: np.ndarray, ncols: int | None = None) -> np.ndarray:
    m = packed.shape[0]
    ncols = packed.shape[1] if ncols is None else ncols
    e = np.zeros((m, ncols), order="F")
    e[np.arange(ncols), np.arange(ncols)] = 1.0
    return apply_q(packed, tau, e)


def inner_solve(g: np.ndarray, tol_in: float, max_inner: int = 30, dtype=np.float64):
    g = np.array(g, dtype=dtype, order="F")
    w = g.shape[0]
    e = np.zeros((w, w), dtype=dtype, order="F")
    isw = np.zeros(1, dtype=np.int32)
    if dtype == np.float64:
        nrot = lib().om_inner_solve_f64(_dp(g), w, tol_in, max_inner, _dp(e), _ip(isw))
    else:
        nrot = lib().om_inner_solve_f32(_fp(g), w, tol_in, max_inner, _fp(e), _ip(isw))
    return g, e, int(nrot), int(isw[0])


def block_jacobi(x: np.ndarray, v: np.ndarray | None, b: int, tol_: float, tol_in: float,
                 max_sweeps: int = 30, max_inner: int = 30, stagnation: bool = False,
                 nthreads: int = 0, dtype=np.float64):
    x = np.array(x, dtype=dtype, order="F")
    m, n = x.shape
    if v is not None:
        v = np.array(v, dtype=dtype, order="F")
    offs = np.zeros(64)
    upds = np.zeros(64, dtype=np.int32)
    nv = 0 if v is None else v.shape[0]
    if dtype == np.float64:
        vp = _dp(v) if v is not None else C.POINTER(C.c_double)()
        sw = lib().om_block_jacobi_f64(_dp(x), m, n, m, vp, nv, max(nv, 1), b, tol_, tol_in,
                                       max_sweeps, max_inner, _dp(offs), _ip(upds), nthreads)
    else:
        vp = _fp(v) if v is not None else C.POINTER(C.c_float)()
        sw = lib().om_block_jacobi_f32(_fp(x), m, n, m, vp, nv, max(nv, 1), b, tol_, tol_in,
                                       max_sweeps, max_inner, int(stagnation), _dp(offs),
                                       _ip(upds), nthreads)
    k = min(abs(sw), 64)
    return x, v, int(sw), offs[:k].copy(), upds[:k].copy()


def lift(v32: np.ndarray) -> tuple[np.ndarray, int]:
    v32 = np.asfortranarray(v32, dtype=np.float32)
    n = v32.shape[0]
    q = np.zeros((n, n), order="F")
    rc = lib().om_lift(_fp(v32), n, n, _dp(q), n)
    return q, rc


def switch_u(x: np.ndarray, ulow: np.ndarray) -> tuple[np.ndarray, int]:
    """U-route switch: Q of the Householder QR of X^T Ulow."""
    x = np.asfortranarray(x, dtype=np.float64)
    ulow = np.asfortranarray(ulow, dtype=np.float64)
    n = x.shape[0]
    q = np.zeros((n, n), order="F")
    rc = lib().om_switch_u(_dp(x), n, n, _dp(ulow), n, _dp(q), n)
    return q, rc


def gate_orth(x: np.ndarray) -> float:
    """orth = ||X_t^T X_t - I||_max in fp32 (om_gate_orth)."""
    x = np.asfortranarray(x, dtype=np.float64)
    n = x.shape[0]
    work = np.zeros(n * n, dtype=np.float32)
    return float(lib().om_gate_orth(_dp(x), n, n, _fp(work)))


def gate_tail(x: np.ndarray, cut_log2: int = -60) -> float:
    x = np.asfortranarray(x, dtype=np.float64)
    return float(lib().om_gate_tail(_dp(x), x.shape[0], x.shape[0], cut_log2))


def gate_cond_scaled(r: np.ndarray, c: np.ndarray) -> float:
    """kappa_1(R diag(1/c)) of the upper triangle of r (om_gate_cond_scaled)."""
    r = np.asfortranarray(r, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    return float(lib().om_gate_cond_scaled(_dp(r), r.shape[0], r.shape[0], _dp(c)))


def gate_cond_d(cn: np.ndarray) -> float:
    cn = np.ascontiguousarray(cn, dtype=np.float64)
    return float(lib().om_gate_cond_d(_dp(cn), cn.size))


def qrsvd32(x32: np.ndarray):
    """The fp32 QR SVD of the AUTO branch (qrsvd.c, reading c-24): (U fp64 n x n, sigma fp32, rc)."""
    x32 = np.asfortranarray(x32, dtype=np.float32)
    n = x32.shape[0]
    u = np.zeros((n, n), order="F")
    s = np.zeros(n, dtype=np.float32)
    rc = lib().om_qrsvd32(_fp(x32), n, n, _dp(u), n, _fp(s))
    return u, s, rc


def mixed_svd(a: np.ndarray, **opts):
    """O-MIX: returns (U, S, V, stats_dict, rc)."""
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    o = default_opts(**opts)
    u = np.zeros((m, n), order="F")
    s = np.zeros(n)
    v = np.zeros((n, n), order="F")
    st = Stats()
    rc = lib().om_mixed_svd(_dp(a), m, n, m, C.byref(o), _dp(u), m, _dp(s), _dp(v), n, C.byref(st))
    return u, s, v, st.as_dict(), int(rc)


def cyclic_jacobi(x: np.ndarray, tol_: float, max_sweeps: int = 60, v: np.ndarray | None = None):
    x = np.array(x, dtype=np.float64, order="F")
    m, n = x.shape
    v = np.eye(n, order="F") if v is None else np.array(v, dtype=np.float64, order="F")
    nrot = C.c_int64(0)
    sw = lib().oc_cyclic_jacobi(_dp(x), m, n, m, _dp(v), n, tol_, max_sweeps, C.byref(nrot))
    return x, v, int(sw), int(nrot.value)


def cyclic_svd(a: np.ndarray, precondition: bool = True, mult: float = 4.0, max_sweeps: int = 60):
    """O-CYC: textbook Alg. 1 (fp64, eq. (2.1) order).  With `precondition`
    it runs on X = L from a LAPACK QRP (scipy dgeqp3) + LQ,
    else directly on A.  Returns (U, S, V, sweeps)."""
    import scipy.linalg as sl
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if precondition:
        q1, r, piv = sl.qr(a, mode="economic", pivoting=True)
        q2t, lt = np.linalg.qr(r.T)          # R^T = Q2t L^T  ->  R = L Q2t^T
        x = lt.T
        x, vx, sw, _ = cyclic_jacobi(x, tol(n, mult), max_sweeps)
        s = np.linalg.norm(x, axis=0)
        order = np.argsort(-s, kind="stable")
        s = s[order]
        ux = x[:, order] / s
        vx = vx[:, order]
        u = q1 @ ux
        v = np.zeros((n, n))
        v[piv, :] = q2t @ vx
        return u, s, v, sw
    x, vx, sw, _ = cyclic_jacobi(a, tol(n, mult), max_sweeps)
    s = np.linalg.norm(x, axis=0)
    order = np.argsort(-s, kind="stable")
    return x[:, order] / s[order], s[order], vx[:, order], sw
