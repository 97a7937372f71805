"""Seeded synthetic test matrices shared by the oracle tests, the GPU parity
tests and bench.py.

This module holds NO arithmetic of the method (no QR preconditioning, no
Jacobi, no lift).  It only builds inputs A = Q1 * diag(sigma) * Q2^T with the
shapes and value distributions of the paper's workloads (PAPER.md:840-898,
sec. 5.1: A = B*D with B = W1*Sigma*W2*W3) as fixed by BASELINE.json's five
configs (SURVEY.md sec. 8(d) gives the seeds and draw order used here).

Every generator is deterministic given its arguments (numpy PCG64
default_rng).  Matrices are returned column-major (Fortran order) float64.
"""
from __future__ import annotations

import hashlib
import os

import numpy as np

try:
    from threadpoolctl import threadpool_limits
except ImportError:  # pragma: no cover
    threadpool_limits = None

# OpenBLAS partitions the QR / GEMM work of the Haar constructions by thread count, and the
# partition changes the rounding: the same seeds give different bits with 8 and 16 BLAS
# threads (measured: this container vs the GPU box).  Every construction therefore runs with
# exactly BLAS_THREADS threads, so that the inputs -- and the digests stored in the oracle
# goldens -- are bit-identical on every host.
BLAS_THREADS = 8
GEN_VERSION = "g2"      # cache key: bump when the bits of a construction change


def _pinned(fn):
    def wrapped(*a, **k):
        if threadpool_limits is None:
            return fn(*a, **k)
        with threadpool_limits(limits=BLAS_THREADS, user_api="blas"):
            return fn(*a, **k)
    wrapped.__name__ = fn.__name__
    wrapped.__doc__ = fn.__doc__
    return wrapped

__all__ = [
    "haar", "geom", "config_matrix", "CONFIGS", "planted_sigma",
    "exact_sigma_matrix", "graded_matrix", "sylvester_hadamard", "digest",
]


@_pinned
def haar(rows: int, cols: int, seed: int) -> np.ndarray:
    """Haar-distributed orthonormal columns: economy QR of a seeded N(0,1)
    matrix with the R diagonal sign folded into Q."""
    g = np.random.default_rng(seed).standard_normal((rows, cols))
    q, r = np.linalg.qr(g)
    return q * np.sign(np.diag(r))


def geom(n: int, lo: float) -> np.ndarray:
    """sigma_i = lo^((i-1)/(n-1)), geometric from 1 down to lo."""
    if n == 1:
        return np.ones(1)
    return lo ** (np.arange(n) / (n - 1))


# config name -> (m, n, description)  -- BASELINE.json "configs"[0..4]
CONFIGS = {
    "C1": (256, 256, "Haar, sigma geometric 1 -> 1e-4 (kappa 1e4)"),
    "C2": (1024, 1024, "column-graded B*D, sigma geometric 1 -> 1e-3, D = 10^U[-6,6]"),
    "C3": (4096, 4096, "Haar, log10 sigma ~ U[-10,0] iid sorted descending"),
    "C4": (16384, 2048, "tall Q1(16384x2048)*diag(geom 1e-6)*Q2^T, columns * 10^U[-3,3]"),
    "C5": (8192, 8192, "Haar, sigma geometric 1 -> 1e-8"),
}


def planted_sigma(name: str, n: int | None = None) -> np.ndarray | None:
    """The sigma planted in the B factor of a config (before column grading),
    descending.  For C1/C3/C5 it is sigma(A) up to construction rounding."""
    m0, n0, _ = CONFIGS[name]
    n = n0 if n is None else n
    if name == "C1":
        return geom(n, 1e-4)
    if name == "C2":
        return geom(n, 1e-3)
    if name == "C3":
        s = 10.0 ** np.random.default_rng(3003).uniform(-10, 0, n)
        return np.sort(s)[::-1].copy()
    if name == "C4":
        return geom(n, 1e-6)
    if name == "C5":
        return geom(n, 1e-8)
    raise KeyError(name)


@_pinned
def config_matrix(name: str, n: int | None = None, m: int | None = None) -> np.ndarray:
    """Build config `name` (C1..C5, SURVEY.md sec. 8(d) pseudo-code).

    `n` / `m` override the size (same recipe, smaller shape) for parity tests
    that must finish on the CPU oracle in seconds.  For C4 the default aspect
    ratio m = 8n is kept when only n is given.
    """
    m0, n0, _ = CONFIGS[name]
    n = n0 if n is None else int(n)
    if name == "C4":
        m = (8 * n if m is None else int(m))
    else:
        m = n if m is None else int(m)
    if name == "C1":
        a = (haar(m, n, 1001) * geom(n, 1e-4)) @ haar(n, n, 1002).T
    elif name == "C2":
        b = (haar(m, n, 2001) * geom(n, 1e-3)) @ haar(n, n, 2002).T
        a = b * 10.0 ** np.random.default_rng(2003).uniform(-6, 6, n)
    elif name == "C3":
        a = (haar(m, n, 3001) * planted_sigma("C3", n)) @ haar(n, n, 3002).T
    elif name == "C4":
        b = (haar(m, n, 4001) * geom(n, 1e-6)) @ haar(n, n, 4002).T
        a = b * 10.0 ** np.random.default_rng(4003).uniform(-3, 3, n)
    elif name == "C5":
        a = (haar(m, n, 5001) * geom(n, 1e-8)) @ haar(n, n, 5002).T
    else:
        raise KeyError(name)
    return np.asfortranarray(a)


def sylvester_hadamard(n: int) -> np.ndarray:
    """Sylvester-Hadamard matrix of order n = 2^k (entries +-1)."""
    if n < 1 or n & (n - 1):
        raise ValueError("n must be a power of two")
    h = np.ones((1, 1))
    while h.shape[0] < n:
        h = np.block([[h, h], [h, -h]])
    return h


@_pinned
def exact_sigma_matrix(n: int, seed: int | None = None, emax: int = 13):
    """Pin P2: A = (1/n) (S1 P1 H) diag(sigma) (S2 P2 H)^T.

    H is Sylvester-Hadamard, S random signs, P random row permutations, and
    sigma_i = (1 + k_i/1024) * 2^-e_i with k_i in [0,1024), e_i =
    floor(emax (i-1)/(n-1)) (emax = 13 -> kappa ~ 1.6e4).  Every sigma_i is a
    multiple of 2^-(10+emax) below 2, so
    every entry of A and every partial sum of the product needs at most
    log2(2n) + 10 + emax <= 53 bits: A is exact in fp64 under any summation order and
    sigma(A) = sigma exactly (columns of S P H / sqrt(n) are orthonormal).
    Returns (A column-major, sigma descending).
    """
    k = int(np.log2(n))
    if 2 ** k != n:
        raise ValueError("n must be a power of two")
    rng = np.random.default_rng(9000 + k if seed is None else seed)
    kk = rng.integers(0, 1024, n)
    ee = np.floor(float(emax) * np.arange(n) / max(n - 1, 1)).astype(int)
    sigma = np.sort((1.0 + kk / 1024.0) * 2.0 ** (-ee))[::-1].copy()
    h = sylvester_hadamard(n)
    m1 = (rng.choice([-1.0, 1.0], n)[:, None] * h[rng.permutation(n)])
    m2 = (rng.choice([-1.0, 1.0], n)[:, None] * h[rng.permutation(n)])
    a = ((m1 * sigma) @ m2.T) / n
    return np.asfortranarray(a), sigma


def graded_matrix(n: int, span_exp: int, seed: int = 7):
    """Pin P4: A = B * diag(2^d_j), B from the exact-sigma construction of
    order n with a mild spectrum (emax = 7, kappa(B) <= 256), d_j uniform
    integers in [-span, span].  Column grading by powers of two is exact."""
    rng = np.random.default_rng(seed)
    b, _ = exact_sigma_matrix(n, seed=seed + 1, emax=7)
    d = rng.integers(-span_exp, span_exp + 1, n)
    return np.asfortranarray(b * 2.0 ** d), d


def digest(a: np.ndarray) -> str:
    """Content hash of a matrix (shape + column-major bytes)."""
    h = hashlib.sha256()
    h.update(str(a.shape).encode())
    h.update(np.asfortranarray(a).tobytes(order="F"))
    return h.hexdigest()[:16]


def cached_config(name: str, n: int | None = None, cache_dir: str | None = None) -> np.ndarray:
    """config_matrix with an optional on-disk .npy cache (speed only; the
    matrix is regenerated whenever the cache file is missing)."""
    cache_dir = cache_dir or os.environ.get("MPJSVD_CACHE", "/tmp/mpjsvd_cache")
    m0, n0, _ = CONFIGS[name]
    key = f"{name}_{n0 if n is None else n}_{GEN_VERSION}.npy"
    path = os.path.join(cache_dir, key)
    try:
        return np.load(path, mmap_mode=None)
    except Exception:
        pass
    a = config_matrix(name, n)
    try:
        os.makedirs(cache_dir, exist_ok=True)
        tmp = path[:-4] + f".{os.getpid()}.tmp.npy"
        np.save(tmp, a)
        os.replace(tmp, path)
    except Exception:
        pass
    return a
