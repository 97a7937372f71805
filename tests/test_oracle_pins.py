"""Pins for the CPU oracle (oracle/), run without a GPU.

Each test checks the oracle against something other than itself: a closed
form, an exact construction, brute force in high precision, a LAPACK routine
standing in for a textbook special case, or a mathematical invariant.  A
plausible slip in the oracle (a dropped term, wrong sign, transposed operand,
wrong index) fails at least one of them; DESIGN.md lists which pin covers
which step.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import testmat

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))
U = 2.0 ** -53


def orth(q):
    return np.abs(q.T @ q - np.eye(q.shape[1])).max()


def tiered_tol(sigma_ref, kappa):
    """max(1e-12, 1e3 u min(kappa, sigma_1/sigma_i))."""
    return np.maximum(1e-12, 1e3 * U * np.minimum(kappa, sigma_ref[0] / sigma_ref))


# ---------------------------------------------------------------- P1 closed forms
def test_golden_ratio_2x2():
    g = GOLD["golden_ratio_2x2"]
    a = np.array(g["A_rowmajor"], order="F")
    u, s, v, st, rc = oracle.mixed_svd(a)
    assert rc == 0
    np.testing.assert_allclose(s, g["sigma"], rtol=2e-16 * 4, atol=0)
    assert np.linalg.norm(a - (u * s) @ v.T) < 4e-16 * 4


def test_rotation_closed_form():
    """G = [[a, c], [c, b]] with a=1, b=2, c=0.5: one rotation, t = tan(pi/8)."""
    g = GOLD["rotation_a1_b2_c05"]
    G = np.array([[g["a"], g["c"]], [g["c"], g["b"]]])
    gout, e, nrot, isw = oracle.inner_solve(G, 1e-15)
    assert nrot == 1
    J = np.eye(2) + e
    np.testing.assert_allclose(J, [[g["cs"], g["sn"]], [-g["sn"], g["cs"]]], rtol=0, atol=2e-16)
    # diagonal = eigenvalues (3 -+ sqrt 2)/2 of G, off-diagonal exactly 0
    np.testing.assert_allclose(np.diag(gout), [(3 - np.sqrt(2)) / 2, (3 + np.sqrt(2)) / 2], rtol=4e-16)
    assert gout[0, 1] == 0.0 and gout[1, 0] == 0.0


def test_rotation_closed_form_fp32():
    g = GOLD["rotation_a1_b2_c05"]
    G = np.array([[g["a"], g["c"]], [g["c"], g["b"]]], dtype=np.float32)
    gout, e, nrot, isw = oracle.inner_solve(G, 1e-6, dtype=np.float32)
    J = np.eye(2) + e.astype(np.float64)
    np.testing.assert_allclose(J, [[g["cs"], g["sn"]], [-g["sn"], g["cs"]]], rtol=0, atol=2e-7)


def test_symmetric_case_45_degrees():
    """a = b, c > 0: zeta = 0, t = 1, cs = sn = 1/sqrt2 (SPEC.md jacobi example)."""
    G = np.array([[2.0, 0.5], [0.5, 2.0]])
    gout, e, nrot, _ = oracle.inner_solve(G, 1e-15)
    np.testing.assert_allclose(np.eye(2) + e, np.array([[1, 1], [-1, 1]]) / np.sqrt(2), atol=2e-16)
    np.testing.assert_allclose(np.diag(gout), [1.5, 2.5], rtol=2e-16)


@pytest.mark.parametrize("b", [1, 4, 32])
def test_identity_one_sweep(b):
    g = GOLD["identity_one_sweep"]
    x = np.eye(40)
    xo, vo, sw, offs, upds = oracle.block_jacobi(x, np.eye(40), b, oracle.tol(40), oracle.tol(40) / 8)
    assert sw == g["sweeps"] and upds.sum() == g["rotations"]
    assert np.array_equal(xo, np.eye(40))


def test_householder_maps_to_positive_multiple_of_e1():
    rng = np.random.default_rng(1)
    for x0 in ([3.0, 4.0], [-3.0, 4.0], [5.0, 0.0], [-5.0, 0.0], rng.standard_normal(17), -np.abs(rng.standard_normal(9))):
        x0 = np.asarray(x0, dtype=float)
        out, tau = oracle.house(x0)
        v = np.concatenate([[1.0], out[1:]])
        H = np.eye(x0.size) - tau * np.outer(v, v)
        assert orth(H) < 8 * U
        hx = H @ x0
        assert out[0] >= 0
        np.testing.assert_allclose(hx[0], np.linalg.norm(x0), rtol=4 * U)
        np.testing.assert_allclose(out[0], np.linalg.norm(x0), rtol=4 * U)
        assert np.abs(hx[1:]).max() <= 8 * U * np.linalg.norm(x0)
    out, tau = oracle.house(np.array([3.0, 4.0]))
    assert out[0] == 5.0


# ---------------------------------------------------------------- QR building blocks
def test_qr_against_lapack_and_invariants():
    rng = np.random.default_rng(2)
    a = rng.standard_normal((50, 20))
    packed, tau, rc = oracle.qr(a)
    assert rc == 0
    r = np.triu(packed[:20, :])
    q = oracle.form_q(packed, tau, 20)
    assert orth(q) < 1e-14
    assert np.abs(q @ r - a).max() < 1e-14
    assert np.all(np.diag(r) >= 0)
    r_lapack = np.linalg.qr(a, mode="r")
    np.testing.assert_allclose(np.abs(r), np.abs(r_lapack), atol=1e-13)


def test_qrp_against_lapack_dgeqp3():
    import scipy.linalg as sl
    rng = np.random.default_rng(3)
    a = rng.standard_normal((60, 60)) * 10.0 ** rng.uniform(-3, 3, 60)
    packed, perm, tau, rc = oracle.qrp(a)
    _, r_l, piv = sl.qr(a, pivoting=True)
    assert np.array_equal(perm, piv)       # same Businger-Golub pivot sequence
    r = np.triu(packed)
    np.testing.assert_allclose(np.abs(r), np.abs(r_l), rtol=1e-12, atol=1e-12 * np.abs(r_l).max())
    q = oracle.form_q(packed, tau)
    assert np.abs(q @ r - a[:, perm]).max() < 1e-13 * np.abs(a).max()
    d = np.diag(r)
    assert np.all(d >= 0) and np.all(d[:-1] >= d[1:] * (1 - 1e-12))
    # RRQR property: R_kk >= ||R(k:j, j)|| for j > k
    for k in range(59):
        assert d[k] >= np.linalg.norm(r[k:, k + 1:], axis=0).max() * (1 - 1e-12)


@pytest.mark.parametrize("m,n", [(60, 60), (120, 45)])
def test_qrp_f32_against_lapack_sgeqp3(m, n):
    """Alg. 4 line 2: the fp32 QRP is LAPACK's single-precision
    Businger-Golub QRP -- same pivot sequence as sgeqp3, |R| within fp32 rounding."""
    import scipy.linalg.lapack as la
    rng = np.random.default_rng(m + n)
    a = (rng.standard_normal((m, n)) * 10.0 ** rng.uniform(-3, 3, n)).astype(np.float32)
    packed, perm, tau, rc = oracle.qrp_f32(a)
    qr_l, jpvt, tau_l, *_, info = la.sgeqp3(np.asfortranarray(a))
    assert rc == 0 and info == 0
    assert np.array_equal(perm, jpvt - 1)
    r, r_l = np.triu(packed[:n]), np.triu(qr_l[:n])
    np.testing.assert_allclose(np.abs(r), np.abs(r_l), rtol=0, atol=2e-5 * np.abs(r_l).max())


def test_mprrqr_is_qr_of_permuted_matrix():
    """Alg. 4: P from the fp32 QRP of lower(A) (power-of-two
    scaled, c-9), then the fp64 QR of A P: R equals LAPACK dgeqrf of A P, the
    factorisation reproduces A P to fp64 accuracy, and R is rank revealing up to
    the fp32 pivoting (diagonal non-increasing within a u32-sized slack)."""
    import scipy.linalg as sl
    rng = np.random.default_rng(4)
    n = 80
    a = rng.standard_normal((n, n)) * 10.0 ** rng.uniform(-3, 3, n)
    packed, perm, tau, rc = oracle.mprrqr(a)
    assert rc == 0
    _, perm32, _, _ = oracle.qrp_f32((a * 2.0 ** -np.frexp(np.abs(a).max())[1]).astype(np.float32))
    assert np.array_equal(perm, perm32)
    r = np.triu(packed)
    r_l = sl.qr(a[:, perm], mode="r")[0]
    np.testing.assert_allclose(np.abs(r), np.abs(r_l), rtol=1e-12, atol=1e-12 * np.abs(r_l).max())
    q = oracle.form_q(packed, tau)
    assert np.abs(q @ r - a[:, perm]).max() < 1e-13 * np.abs(a).max()
    d = np.diag(r)
    assert np.all(d >= 0) and np.all(d[:-1] >= d[1:] * (1 - 1e-5))
    # the fp32 pivots agree with the fp64 QRP's wherever the latter's choice is not a near tie
    _, perm64, _, _ = oracle.qrp(a)
    assert np.mean(perm == perm64) > 0.9


def test_qrp_ties_lowest_index():
    a = np.asfortranarray(np.eye(6) * 2.0)
    packed, perm, tau, rc = oracle.qrp(a)
    assert list(perm) == list(range(6))


def test_rank_deficient_and_invalid():
    a = testmat.config_matrix("C1", 16)
    a[:, 5] = 0.0
    assert oracle.mixed_svd(a)[4] == -3
    b = testmat.config_matrix("C1", 16)
    b[3, 3] = np.nan
    assert oracle.mixed_svd(b)[4] == -2
    assert oracle.mixed_svd(np.ones((4, 6)))[4] == -1


# ---------------------------------------------------------------- inner solve
@pytest.mark.parametrize("w", [2, 7, 64])
def test_inner_solve_diagonalises(w):
    rng = np.random.default_rng(w)
    b = rng.standard_normal((3 * w, w)) * 10.0 ** rng.uniform(-2, 2, w)
    G0 = b.T @ b
    tol_in = oracle.tol(3 * w) / 8
    g, e, nrot, isw = oracle.inner_solve(G0, tol_in)
    J = np.eye(w) + e
    assert orth(J) < 50 * U * w ** 0.5
    D = J.T @ G0 @ J
    dd = np.sqrt(np.diag(D))
    off = np.abs(D - np.diag(np.diag(D))) / np.outer(dd, dd)
    assert off.max() < 20 * tol_in
    # LAPACK dsyevd is absolutely (not relatively) accurate: Weyl-type bound
    lam = np.linalg.eigvalsh(G0)
    assert np.abs(np.sort(np.diag(g)) - lam).max() <= 64 * w * U * lam[-1]


# ---------------------------------------------------------------- block Jacobi
@pytest.mark.parametrize("n,b", [(96, 16), (100, 16), (7, 4), (50, 64), (33, 1)])
def test_block_jacobi_orthogonalises(n, b):
    rng = np.random.default_rng(n + b)
    x0 = rng.standard_normal((n, n))
    tol_ = oracle.tol(n)
    x, v, sw, offs, upds = oracle.block_jacobi(x0, np.eye(n), b, tol_, tol_ / 8, max_sweeps=40)
    assert sw > 0
    nrm = np.linalg.norm(x, axis=0)
    c = np.abs(x.T @ x) / np.outer(nrm, nrm)
    np.fill_diagonal(c, 0)
    assert c.max() <= 4 * tol_
    assert orth(v) < 16 * n * U
    assert np.abs(x0 @ v - x).max() < 1e-13 * np.abs(x0).max() * n ** 0.5
    np.testing.assert_allclose(np.sort(nrm)[::-1], np.linalg.svd(x0, compute_uv=False), rtol=1e-12)
    assert upds[-1] == 0


def test_block_jacobi_f32_stage():
    rng = np.random.default_rng(5)
    n = 64
    x0 = rng.standard_normal((n, n)).astype(np.float32)
    tol_ = np.float32(4 * np.sqrt(n) * 2.0 ** -24)
    x, v, sw, offs, upds = oracle.block_jacobi(x0, np.eye(n, dtype=np.float32), 8, tol_, tol_ / 8,
                                               stagnation=True, dtype=np.float32)
    assert sw > 0
    assert orth(v.astype(np.float64)) < 1e-5
    s = np.sort(np.linalg.norm(x.astype(np.float64), axis=0))[::-1]
    np.testing.assert_allclose(s, np.linalg.svd(x0.astype(np.float64), compute_uv=False), rtol=1e-5)


# ---------------------------------------------------------------- lift (switch repair)
def test_lift_repairs_orthogonality():
    """orth(fl64(V32)) ~ u_low while orth(Q) <= 1e-14; Q^T V is
    upper triangular with positive diagonal (V = Q R_v)."""
    import scipy.linalg as sl
    a = testmat.config_matrix("C1", 128)
    _, r, _ = sl.qr(a, pivoting=True)
    x = np.linalg.qr(r.T)[1].T
    e = np.frexp(np.abs(x).max())[1]
    x32 = np.ldexp(x, -e).astype(np.float32)
    t32 = np.float32(4 * np.sqrt(128) * 2.0 ** -24)
    _, v32, sw, _, _ = oracle.block_jacobi(x32, np.eye(128, dtype=np.float32), 32, t32, t32 / 8,
                                           stagnation=True, dtype=np.float32)
    o32 = orth(v32.astype(np.float64))
    assert 1e-8 <= o32 <= 1e-4
    q, rc = oracle.lift(v32)
    assert rc == 0 and orth(q) < 1e-14
    rv = q.T @ v32.astype(np.float64)
    assert np.abs(np.tril(rv, -1)).max() < 1e-14
    assert np.all(np.diag(rv) > 0)
    assert np.abs(q - v32).max() < 1e-4


# ---------------------------------------------------------------- U-route switch
def _exact_factors(n, emax=13, seed=None):
    """A = U diag(sigma) V^T with U, V = S P H / sqrt(n) exactly representable (n = 4^k)."""
    k = int(np.log2(n))
    rng = np.random.default_rng(9000 + k if seed is None else seed)
    kk = rng.integers(0, 1024, n)
    ee = np.floor(float(emax) * np.arange(n) / max(n - 1, 1)).astype(int)
    sigma = np.sort((1.0 + kk / 1024.0) * 2.0 ** (-ee))[::-1].copy()
    h = testmat.sylvester_hadamard(n)
    r = np.sqrt(n)
    uu = rng.choice([-1.0, 1.0], n)[:, None] * h[rng.permutation(n)] / r
    vv = rng.choice([-1.0, 1.0], n)[:, None] * h[rng.permutation(n)] / r
    a = (uu * sigma) @ vv.T
    return np.asfortranarray(a), uu, sigma, vv


@pytest.mark.parametrize("n", [16, 64, 256])
def test_switch_u_recovers_v_exactly_known(n):
    """with U_low = U_X, qr(X^T U_X) gives Q = V_X "in exact arithmetic"
    (X^T U_X = V_X Sigma, R2 = Sigma > 0 so no sign flips).  U, V are exactly representable
    (entries +-2^-k), so Q must equal V to rounding; a transposed operand (X U) or a wrong
    reflector sign fails this."""
    a, uu, sigma, vv = _exact_factors(n)
    q, rc = oracle.switch_u(a, uu)
    assert rc == 0
    assert np.abs(q - vv).max() < 50 * n * U
    assert orth(q) < 20 * n * U


def test_switch_u_column_scaling_bitwise():
    """Householder QR is invariant to power-of-two column scaling (reflector vectors and tau are
    scale-free), so Q(X, U_low 2^D) == Q(X, U_low) bitwise: the normalisation of U_low cannot
    change the switch."""
    a = testmat.config_matrix("C1", 64)
    rng = np.random.default_rng(3)
    ul = np.linalg.qr(rng.standard_normal((64, 64)))[0]
    q1, _ = oracle.switch_u(a, ul)
    q2, _ = oracle.switch_u(a, ul * 2.0 ** rng.integers(-30, 30, 64))
    assert np.array_equal(q1, q2)


def test_switch_u_is_qr_of_xtu_against_lapack():
    """Q R2 = X^T U_low: the same Q as LAPACK dgeqrf/dorgqr after fixing diag(R2) >= 0 (c-13), and
    Q^T (X^T U_low) upper triangular with a non-negative diagonal."""
    import scipy.linalg as sl
    rng = np.random.default_rng(5)
    a = np.asfortranarray(rng.standard_normal((96, 96)))      # kappa(X^T U) ~ 1e2..1e3: Q fixed to ~u kappa
    ul = np.linalg.qr(rng.standard_normal((96, 96)))[0]
    q, rc = oracle.switch_u(a, ul)
    z = a.T @ ul
    ql, rl = sl.qr(z)
    ql = ql * np.sign(np.diag(rl))
    assert rc == 0 and np.abs(q - ql).max() < 1e-12
    r2 = q.T @ z
    assert np.abs(np.tril(r2, -1)).max() < 1e-12 * np.abs(z).max()
    assert np.all(np.diag(r2) >= 0)


@pytest.mark.parametrize("route", [0, 1])
def test_routes_agree_on_structural_bounds(route):
    """Both precision switches (V-route c-11 / U-route PAPER.md:563-573) give a valid SVD with
    "typically three" refinement sweeps."""
    a = testmat.config_matrix("C5", 256)
    u, s, v, st, rc = oracle.mixed_svd(a, switch_u=route)
    assert rc == 0 and orth(u) <= 1e-13 and orth(v) <= 1e-13
    assert np.linalg.norm(a - (u * s) @ v.T) / np.linalg.norm(a) <= 1e-13
    assert st["sweeps64"] <= GOLD["refinement_sweeps"]["max_with_slack"]
    sr = oracle.mixed_svd(a, switch_u=1 - route)[1]
    assert np.abs(s - sr).max() / s[0] <= 8 * np.sqrt(256) * U


# ---------------------------------------------------------------- P2 exact sigma
@pytest.mark.parametrize("n", [16, 64, 256])
@pytest.mark.parametrize("route", [0, 1])
def test_exact_sigma(n, route):
    a, sigma = testmat.exact_sigma_matrix(n)
    u, s, v, st, rc = oracle.mixed_svd(a, switch_u=route)
    assert rc == 0
    rel = np.abs(s - sigma) / sigma
    assert np.all(rel <= tiered_tol(sigma, sigma[0] / sigma[-1]))
    assert rel.max() < 1e-12
    assert orth(u) < 1e-13 and orth(v) < 1e-13


# ---------------------------------------------------------------- P3 brute force n <= 8
@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_brute_force_small(n):
    import mpmath
    mpmath.mp.dps = 50
    rng = np.random.default_rng(100 + n)
    a = rng.standard_normal((n, n)) * 10.0 ** rng.uniform(-1, 1, n)
    fa = [[Fraction(float(a[i, j])) for j in range(n)] for i in range(n)]
    ata = [[sum(fa[k][i] * fa[k][j] for k in range(n)) for j in range(n)] for i in range(n)]
    M = mpmath.matrix([[mpmath.mpf(ata[i][j].numerator) / ata[i][j].denominator for j in range(n)]
                       for i in range(n)])
    ev = mpmath.eigsy(M, eigvals_only=True)
    ref = np.array(sorted([float(mpmath.sqrt(x)) for x in ev], reverse=True))
    u, s, v, st, rc = oracle.mixed_svd(np.asfortranarray(a))
    assert rc == 0
    kappa = ref[0] / ref[-1]
    assert np.all(np.abs(s - ref) / ref <= np.maximum(64 * n * U, 64 * U * kappa))


# ---------------------------------------------------------------- P4 high relative accuracy
@pytest.mark.parametrize("n,span", [(16, 20), (32, 20), (32, 40)])
def test_high_relative_accuracy_graded(n, span):
    import mpmath
    mpmath.mp.dps = 80
    a, d = testmat.graded_matrix(n, span)
    M = mpmath.matrix(a.tolist())
    ref = np.array(sorted([float(x) for x in mpmath.svd_r(M, compute_uv=False)], reverse=True))
    u, s, v, st, rc = oracle.mixed_svd(a)
    assert rc == 0
    assert ref[0] / ref[-1] > 1e10
    assert np.max(np.abs(s - ref) / ref) < 1e-13


# ---------------------------------------------------------------- P5 invariances
def test_power_of_two_scaling_bitwise():
    a = testmat.config_matrix("C2", 64)
    u1, s1, v1, _, _ = oracle.mixed_svd(a)
    u2, s2, v2, _, _ = oracle.mixed_svd(np.asfortranarray(a * 2.0 ** 37))
    assert np.array_equal(s2, s1 * 2.0 ** 37)
    assert np.array_equal(u1, u2) and np.array_equal(v1, v2)


def test_column_permutation_invariance():
    a = testmat.config_matrix("C1", 64)
    pi = np.random.default_rng(9).permutation(64)
    u1, s1, v1, _, _ = oracle.mixed_svd(a)
    u2, s2, v2, _, _ = oracle.mixed_svd(np.asfortranarray(a[:, pi]))
    assert np.array_equal(s1, s2)
    assert np.array_equal(u1, u2)
    assert np.array_equal(v1[pi, :], v2)


def test_thread_count_independence():
    a = testmat.config_matrix("C1", 128)
    r1 = oracle.mixed_svd(a, nthreads=1)
    r4 = oracle.mixed_svd(a, nthreads=4)
    for x, y in zip(r1[:3], r4[:3]):
        assert np.array_equal(x, y)


# ---------------------------------------------------------------- P6/P7 structure, sweeps
@pytest.mark.parametrize("name,n", [("C1", 256), ("C2", 256), ("C3", 256), ("C4", 128), ("C5", 256)])
def test_structural_bounds_and_sweeps(name, n):
    a = testmat.config_matrix(name, n)
    m = a.shape[0]
    u, s, v, st, rc = oracle.mixed_svd(a)
    assert rc == 0
    assert orth(u) <= 1e-13 and orth(v) <= 1e-13
    res = np.linalg.norm(a - (u * s) @ v.T) / np.linalg.norm(a)
    assert res <= 1e-13
    # columnwise backward error (preconditioned Jacobi, sec. 4)
    colres = np.linalg.norm(a - (u * s) @ v.T, axis=0) / np.linalg.norm(a, axis=0)
    assert colres.max() <= 200 * n * U
    assert np.all(s[:-1] >= s[1:]) and np.all(s > 0)
    # "typically three sweeps"; +1 slack
    assert st["sweeps64"] <= GOLD["refinement_sweeps"]["max_with_slack"]
    assert st["upd_trace64"][-1] == 0
    assert st["sweeps32"] >= 2


def test_force_fp64_path_agrees():
    a = testmat.config_matrix("C1", 128)
    u1, s1, v1, st1, _ = oracle.mixed_svd(a)
    u2, s2, v2, st2, _ = oracle.mixed_svd(a, path=2)
    assert st2["sweeps32"] == 0 and st2["sweeps64"] > st1["sweeps64"]
    assert np.max(np.abs(s1 - s2) / s2) < 1e-12


def test_x_from_r_ablation_agrees():
    a = testmat.config_matrix("C1", 96)
    s1 = oracle.mixed_svd(a)[1]
    s2 = oracle.mixed_svd(a, x_from_lq=0)[1]
    assert np.max(np.abs(s1 - s2) / s2) < 1e-12


# ---------------------------------------------------------------- P8 / P9 cross-checks
def _dgejsv_sigma(a):
    from scipy.linalg import lapack
    sva, _, _, wo, _, info = lapack.dgejsv(a, joba=0, jobu=3, jobv=3)
    assert info == 0
    return np.sort(sva * wo[0] / wo[1])[::-1]


@pytest.mark.parametrize("name,n,kappa_s", [("C1", 256, 1e4), ("C2", 512, 1e3), ("C5", 256, 1e8)])
def test_against_dgejsv(name, n, kappa_s):
    a = testmat.config_matrix(name, n)
    s = oracle.mixed_svd(a)[1]
    sj = _dgejsv_sigma(a)
    assert np.all(np.abs(s - sj) / sj <= tiered_tol(sj, kappa_s))


def test_graded_vs_dgejsv_paper_scale():
    """max relative difference vs DGEJSV 4.7879e-14 on
    1024^2 graded test matrices; C2 (kappa_s ~ 1e3, columns graded 1e12) at
    n = 512 must land on the same scale."""
    a = testmat.config_matrix("C2", 512)
    s = oracle.mixed_svd(a)[1]
    sj = _dgejsv_sigma(a)
    assert np.max(np.abs(s - sj) / sj) < 10 * GOLD["mixed_vs_dgejsv_max_rel"]["value"]


@pytest.mark.parametrize("name,n", [("C1", 128), ("C2", 128), ("C4", 64)])
def test_omix_vs_ocyc(name, n):
    a = testmat.config_matrix(name, n)
    u1, s1, v1, st, _ = oracle.mixed_svd(a)
    u2, s2, v2, sw = oracle.cyclic_svd(a)
    assert sw > 0
    assert np.all(np.abs(s1 - s2) / s2 <= tiered_tol(s2, 1e4))
    # singular vectors agree up to sign where sigma is well separated
    gap = np.minimum(np.abs(np.diff(s2, prepend=np.inf)), np.abs(np.diff(s2, append=-np.inf))) / s2
    ok = gap > 1e-3
    dots = np.abs(np.sum(v1 * v2, axis=0))
    assert np.all(np.abs(dots[ok] - 1) < 1e-9)


def test_ocyc_unpreconditioned_textbook():
    """O-CYC directly on A (no preconditioning) against the exact sigma."""
    a, sigma = testmat.exact_sigma_matrix(32)
    u, s, v, sw = oracle.cyclic_svd(a, precondition=False)
    assert sw > 0
    assert np.max(np.abs(s - sigma) / sigma) < 1e-12
    assert orth(v) < 1e-14


# ---------------------------------------------------------------- P2b planted sigma
@pytest.mark.parametrize("name", ["C1", "C5"])
def test_planted_sigma_construction_bound(name):
    n = 256
    a = testmat.config_matrix(name, n)
    s = oracle.mixed_svd(a)[1]
    planted = testmat.planted_sigma(name, n)
    assert np.abs(s - planted).max() <= 8 * np.sqrt(n) * U * planted[0]


# ---------------------------------------------------------------- AUTO gates
def auto_cases(n=64):
    """Inputs that trigger each branch of the AUTO path (reading c-15)."""
    rng = np.random.default_rng(21)
    q = testmat.haar(n, n, 2101)
    cases = {}
    # cond gate: orthogonal columns (scaled cond(R) = 1) with norms spanning 1e20 (cond(D) > 1e15)
    d = 10.0 ** np.linspace(0, 20, n)
    cases["cond"] = (np.asfortranarray(q * d), {}, 3, np.sort(d)[::-1])
    # tail gate: half of the columns scaled by 2^-70 (below 2^-60 max after preconditioning)
    b = rng.standard_normal((n, n))
    cases["tail"] = (np.asfortranarray(b * np.where(np.arange(n) < n // 2, 1.0, 2.0 ** -70)), {}, 4, None)
    # orth gate: orthogonal columns, mild grading (cond(D) = 1e3 < 1e15): X is diagonal after QRP + LQ
    d2 = 10.0 ** np.linspace(0, 3, n)
    cases["orth"] = (np.asfortranarray(q * d2), {}, 5, np.sort(d2)[::-1])
    # Jacobi (orth > tol_orth, tol_alg = inf) and the QR SVD branch (orth > tol_alg = 1e-3)
    c1 = testmat.config_matrix("C1", n)
    cases["jacobi"] = (c1, {}, 0, None)
    cases["qrsvd"] = (c1, {"tol_alg": 1e-3}, 6, None)
    return cases


@pytest.mark.parametrize("case", ["cond", "tail", "orth", "jacobi", "qrsvd"])
def test_auto_gates_take_the_papers_branch(case):
    """Alg. 3's gates in order (cond, tail, orth, then Jacobi vs QR SVD by tol_alg): each input takes its
    branch, the result is a valid SVD, and where sigma is known exactly (columns orthogonal: sigma = column
    norms) it is reached to high relative accuracy."""
    a, kw, taken, sig = auto_cases()[case]
    n = a.shape[1]
    u, s, v, st, rc = oracle.mixed_svd(a, path=1, **kw)
    assert rc == 0 and st["path_taken"] == taken, (st["path_taken"], taken)
    assert orth(u) <= 1e-13 and orth(v) <= 1e-13
    assert np.linalg.norm(a - (u * s) @ v.T) / np.linalg.norm(a) <= 1e-13
    if sig is not None:
        assert np.max(np.abs(s - sig) / sig) <= 1e-13
    else:
        # third opinion: LAPACK dgejsv (high relative accuracy on column-graded inputs, F6)
        sj = _dgejsv_sigma(a)
        kap = np.linalg.cond(a / np.linalg.norm(a, axis=0))
        assert np.all(np.abs(s - sj) / sj <= tiered_tol(sj, kap))
    if taken in (3, 4, 5):
        assert st["sweeps32"] == 0
    assert st["sweeps64"] <= GOLD["refinement_sweeps"]["max_with_slack"] or taken in (3, 4, 5)


def test_auto_qrsvd_branch_matches_jacobi_branch_sigma():
    """Both low-precision solvers only seed the fp64 refinement: the final sigma of
    the QR-SVD branch equals the Jacobi branch's to the refinement's accuracy."""
    a = testmat.config_matrix("C2", 128)
    s_j = oracle.mixed_svd(a, path=1)[1]
    _, s_q, _, st, rc = oracle.mixed_svd(a, path=1, tol_alg=1e-3)
    assert rc == 0 and st["path_taken"] == 6
    assert np.max(np.abs(s_q - s_j) / s_j) <= 1e-12


# ---------------------------------------------------------------- gate measures
def _hadamard_cols(n, seed):
    """P H D: Sylvester-Hadamard (n = 4^k, so H/sqrt(n) is exact), random row permutation and power-of-two
    column scales.  Columns exactly orthogonal in any arithmetic; X X^T != I (transposition shows)."""
    rng = np.random.default_rng(seed)
    h = testmat.sylvester_hadamard(n)[rng.permutation(n)]
    return np.asfortranarray(h * 2.0 ** rng.integers(-20, 20, n)), rng


@pytest.mark.parametrize("n", [4, 16, 64])
def test_gate_orth_exactly_orthogonal_columns_is_zero(n):
    """Exactly orthogonal dyadic columns: X_t = P H / sqrt(n) is exact in fp32, so ||X_t^T X_t - I||_max = 0
    exactly (a missing normalisation, a transposed product X X^T, or a wrong norm fails)."""
    x, _ = _hadamard_cols(n, n)
    assert oracle.gate_orth(x) == 0.0
    # rows scaled unevenly: columns no longer orthogonal, the measure sees it (X X^T is still diagonal-free)
    y = x * np.linspace(1.0, 2.0, n)[:, None]
    assert oracle.gate_orth(y) > 1e-3


def test_gate_orth_closed_forms():
    """Closed forms in the paper's lower precision ("one matrix-matrix multiplication in
    the lower precision"):
      X = [[3, 0], [4, 5]] (columns (3,4), (0,5)): X_t = ((3/5, 4/5), (0, 1)) in fp32, off-diagonal
        fl32(4/5) * 1 = fl32(0.8); the diagonal of column 1 is fl32(0.6)^2 + fl32(0.8)^2 rounded -> orth =
        fl32(0.8) exactly;
      X = [[1, -2^-12], [2^-12, 1]]: both norms round to 1 in fp32, the columns are exactly orthogonal,
        and 1 + 2^-24 rounds to 1 in an fp32 accumulation: orth = 0 (an fp64-accumulated Gram gives 2^-24)."""
    x = np.array([[3.0, 0.0], [4.0, 5.0]], order="F")
    assert oracle.gate_orth(x) == float(np.float32(0.8))
    e = 2.0 ** -12
    y = np.array([[1.0, -e], [e, 1.0]], order="F")
    assert oracle.gate_orth(y) == 0.0


def test_gate_orth_scaling_invariance_and_error_bound():
    """Power-of-two column scaling is exact through fl32 and the normalisation: bitwise invariance.  For a
    random X the fp32 measure is within the fp32 GEMM bound of the exact value of the same definition."""
    rng = np.random.default_rng(5)
    n = 48
    x = np.asfortranarray(rng.standard_normal((n, n)))
    s = 2.0 ** rng.integers(-30, 30, n)
    assert oracle.gate_orth(x) == oracle.gate_orth(np.asfortranarray(x * s))
    x32 = x.astype(np.float32).astype(np.float64)
    xt = x32 / np.linalg.norm(x32, axis=0)
    exact = np.abs(xt.T @ xt - np.eye(n)).max()
    assert abs(oracle.gate_orth(x) - exact) <= 2 * n * 2.0 ** -24


def test_gate_tail_counts_small_columns():
    """Tail fraction: columns strictly below 2^cut max are counted; a column exactly at
    the cut is not."""
    n = 12
    x, _ = _hadamard_cols(16, 3)
    x = np.asfortranarray(x[:n, :n] * 0 + np.eye(n))
    scales = np.array([1.0, 0.5, 2.0 ** -60, 2.0 ** -61, 2.0 ** -70, 1.0, 1.0, 2.0 ** -80, 1.0, 1.0, 1.0, 1.0])
    x = np.asfortranarray(x * scales)
    assert oracle.gate_tail(x, -60) == 3.0 / n
    assert oracle.gate_tail(x, -10) == 4.0 / n
    assert oracle.gate_tail(x, -100) == 0.0


def test_gate_cond_scaled_closed_forms_and_lapack():
    """cond_R of the column-scaled R (Alg. 3 l.423; reading c-15) = kappa_1(R diag(1/c)):
      R = diag(d), c = |d|: R_s = I -> 1 exactly (any grading of D is removed);
      R = [[1, t], [0, 1]], c = (1, sqrt(1+t^2)): ||R_s||_1 = (|t|+1)/sqrt(1+t^2) or 1, R_s^-1 =
        [[1, -t], [0, sqrt(1+t^2)]] -> closed form below;
      a random upper-triangular R with its true column norms: numpy.linalg.cond(R_s, 1) (LAPACK)."""
    d = 2.0 ** np.arange(-20, 20, 4)
    assert oracle.gate_cond_scaled(np.diag(d), np.abs(d)) == 1.0
    t = 3.0
    r = np.array([[1.0, t], [0.0, 1.0]], order="F")
    c = np.array([1.0, np.sqrt(1 + t * t)])
    nrm = max(1.0, (abs(t) + 1) / np.sqrt(1 + t * t))
    inv = max(1.0, abs(t) + np.sqrt(1 + t * t))
    assert abs(oracle.gate_cond_scaled(r, c) - nrm * inv) <= 4 * U * nrm * inv
    rng = np.random.default_rng(9)
    n = 40
    r = np.triu(rng.standard_normal((n, n))) + 4 * np.eye(n)
    r = np.asfortranarray(r * 10.0 ** rng.uniform(-6, 6, n))
    c = np.linalg.norm(r, axis=0)
    ref = np.linalg.cond(r / c, 1)
    assert abs(oracle.gate_cond_scaled(r, c) - ref) <= 1e-12 * ref
    # only the upper triangle is read (reflectors may sit below the diagonal)
    junk = np.asfortranarray(r + np.tril(rng.standard_normal((n, n)), -1))
    assert oracle.gate_cond_scaled(junk, c) == oracle.gate_cond_scaled(r, c)


def test_gate_cond_d_closed_form():
    """cond(D) of A = B D (Alg. 3 l.423-424): max/min column norm."""
    assert oracle.gate_cond_d(np.array([2.0, 8.0, 0.5, 1.0])) == 16.0
    assert oracle.gate_cond_d(np.array([3.0, 3.0])) == 1.0


def test_gate_measures_in_mixed_svd_are_the_gate_functions():
    """mixed_svd's reported measures are those of its own X = L / R (AUTO): orthogonal columns with a
    known grading give cond_d = the grading's span, cond_scaled = 1 to rounding, orth ~ 0."""
    n = 64
    q = testmat.haar(n, n, 77)
    d = 10.0 ** np.linspace(0, 8, n)
    u, s, v, st, rc = oracle.mixed_svd(np.asfortranarray(q * d), path=1)
    assert abs(st["cond_d"] / 1e8 - 1) <= 1e-12
    assert abs(st["cond_scaled"] - 1.0) <= 1e-10
    assert st["orth_measure"] <= 1e-6


# ---------------------------------------------------------------- sec. 3.4 V formation
@pytest.mark.parametrize("n", [64, 256])
def test_refine_v_exact_sigma_and_one_sweep(n):
    """refine_v = 1 (reading c-23): refinement without V, V_X = qr(X^T U_X), one accumulating refinement.
    Exact-sigma input: sigma exact within the tiered bound, U and V orthogonal, small residual, and the
    accumulating refinement "always converges in one sweep": one sweep with rotations at
    most, plus the check sweep."""
    a, sigma = testmat.exact_sigma_matrix(n)
    u, s, v, st, rc = oracle.mixed_svd(a, refine_v=1)
    assert rc == 0
    rel = np.abs(s - sigma) / sigma
    assert rel.max() < 1e-12
    assert orth(u) < 1e-13 and orth(v) < 1e-13
    assert np.linalg.norm(a - (u * s) @ v.T) / np.linalg.norm(a) < 1e-13
    assert 1 <= st["v_sweeps64"] <= 2
    assert st["sweeps64"] > st["v_sweeps64"]


@pytest.mark.parametrize("name,n", [("C1", 128), ("C2", 128), ("C3", 256), ("C5", 256)])
def test_refine_v_matches_accumulating_refinement(name, n):
    """Both V handlings are the same SVD: sigma agree to the refinement's accuracy (tiered bound vs the
    column-scaled condition number), both U/V orthogonal, and the accumulating stage needs <= 2 sweeps."""
    a = testmat.config_matrix(name, n)
    u0, s0, v0, st0, rc0 = oracle.mixed_svd(a)
    u1, s1, v1, st1, rc1 = oracle.mixed_svd(a, refine_v=1)
    assert rc0 == 0 and rc1 == 0
    kap = np.linalg.cond(a / np.linalg.norm(a, axis=0))
    assert np.all(np.abs(s1 - s0) / s0 <= tiered_tol(s0, kap))
    assert orth(u1) < 1e-13 and orth(v1) < 1e-13
    assert np.linalg.norm(a - (u1 * s1) @ v1.T) / np.linalg.norm(a) < 1e-13
    assert st1["v_sweeps64"] <= 2 and st0["v_sweeps64"] == st0["sweeps64"]


def test_refine_v_high_relative_accuracy():
    """Column-graded input (sigma spanning ~1e12) through refine_v = 1 against 80-digit mpmath (pin P4)."""
    import mpmath
    mpmath.mp.dps = 80
    a, _ = testmat.graded_matrix(32, 20)
    s = oracle.mixed_svd(a, refine_v=1)[1]
    ref = np.array(sorted((float(x) for x in mpmath.svd_r(mpmath.matrix(a.tolist()), compute_uv=False)),
                          reverse=True))
    assert np.max(np.abs(s - ref) / ref) < 1e-13


# ---------------------------------------------------------------- fp32 QR SVD
U32 = 2.0 ** -24


@pytest.mark.parametrize("n", [16, 64, 256])
def test_qrsvd32_exact_sigma_within_fp32_bound(n):
    """The lower-precision QR SVD (qrsvd.c, reading c-24) of fl32(A) for the exact-sigma construction:
    |sigma_i - sigma_i(A)| <= n u32 sigma_1 (input rounding + backward error of bidiagonalisation and QR
    iteration, Weyl), U orthogonal to the fp32 level, and U^T X has orthogonal rows of norms sigma."""
    a, sigma = testmat.exact_sigma_matrix(n)
    x = a.astype(np.float32)
    u, s, rc = oracle.qrsvd32(x)
    assert rc == 0
    assert np.all(np.diff(s.astype(np.float64)) <= 0)
    assert np.abs(s - sigma).max() <= n * U32 * sigma[0]
    assert orth(u) <= 4 * n * U32
    g = u.T @ x.astype(np.float64)
    gg = g @ g.T
    assert np.abs(gg - np.diag(np.diag(gg))).max() <= 8 * n * U32 * sigma[0] ** 2
    assert np.abs(np.sqrt(np.diag(gg)) - s).max() <= n * U32 * sigma[0]


def test_qrsvd32_closed_forms():
    """Diagonal input (signs, distinct magnitudes): no rotation survives, sigma = sorted |d| exactly and |U| is
    the sorting permutation; [[1, 1], [0, 1]]: sigma = (phi, 1/phi) to fp32 accuracy; an exact zero on the
    bidiagonal's diagonal is rank deficient (rc = -3, reading c-18)."""
    d = np.array([0.5, -2.0, 0.25, 1.0, -0.125], dtype=np.float32)
    u, s, rc = oracle.qrsvd32(np.diag(d))
    assert rc == 0
    order = np.argsort(-np.abs(d), kind="stable")
    assert np.array_equal(s, np.abs(d)[order])
    assert np.array_equal(np.abs(u), np.eye(5)[:, order])
    u, s, rc = oracle.qrsvd32(np.array([[1.0, 1.0], [0.0, 1.0]], dtype=np.float32))
    phi = (1 + np.sqrt(5)) / 2
    assert rc == 0 and abs(s[0] - phi) <= 4 * U32 * phi and abs(s[1] - 1 / phi) <= 4 * U32 * phi
    z = np.asfortranarray(np.random.default_rng(3).standard_normal((6, 6)).astype(np.float32))
    z[:, 2] = 0.0
    u, s, rc = oracle.qrsvd32(z)
    # singular input: either an exact zero on B's diagonal (rc -3) or a computed sigma_min at rounding level
    assert rc == -3 or (rc == 0 and s[-1] <= 6 * U32 * s[0])
    z[:, 0] = 0.0
    z[0, :] = 0.0     # first column zero: the first reflector is the identity and d_0 = 0 exactly
    assert oracle.qrsvd32(z)[2] == -3


def test_qrsvd32_vs_lapack_sgesvd():
    """Third opinion: LAPACK sgesvd (the routine the paper's x86 code calls for this branch)
    on the C1 recipe: sigma within the fp32 bound, left singular vectors equal up to sign where the sigma are
    well separated."""
    import scipy.linalg as sl
    n = 128
    x = testmat.config_matrix("C1", n).astype(np.float32)
    u, s, rc = oracle.qrsvd32(x)
    ul, sl_, _ = sl.svd(x, lapack_driver="gesvd")
    assert rc == 0
    assert np.abs(s - sl_).max() <= n * U32 * sl_[0]
    gap = np.minimum(np.r_[np.inf, -np.diff(sl_)], np.r_[-np.diff(sl_), np.inf]) / sl_[0]
    ok = gap > 1e-3
    dots = np.abs(np.sum(u * ul.astype(np.float64), axis=0))
    assert np.all(dots[ok] >= 1 - 1e-3)


# ---------------------------------------------------------------- fp32-stage exits (reading c-10)
def _one_pair_matrix(theta):
    """64 x 64 identity with column 40 += theta column 3: two blocks of b = 32, one pair per sweep; the pair
    metric is theta / sqrt(1 + theta^2) exactly as constructed (dyadic theta, exact in fp32)."""
    x = np.eye(64, dtype=np.float32)
    x[3, 40] = np.float32(theta)
    return np.asfortranarray(x)


def test_fp32_near_convergence_exit():
    """m = 64: eps_tol32 = 4 sqrt(64) 2^-24 = 2^-19 exactly.  A pair metric of 1.5 eps_tol rotates (> eps_tol)
    and then ends the stage (<= 2 eps_tol, the near-convergence exit): 1 sweep, converged.  At 3 eps_tol there is
    no exit after sweep 1 and the check sweep finds nothing: 2 sweeps.  Without the exit (fp64 rule,
    stagnation = False) 1.5 eps_tol also takes 2 sweeps."""
    tol = np.float32(2.0 ** -19)
    assert tol == np.float32(4 * np.sqrt(64) * 2.0 ** -24)
    for theta, stag, expect in ((1.5 * 2.0 ** -19, True, 1), (3 * 2.0 ** -19, True, 2), (1.5 * 2.0 ** -19, False, 2)):
        x = _one_pair_matrix(theta)
        xo, _, sw, offs, upd = oracle.block_jacobi(x, None, 32, tol, tol / 8, max_sweeps=20, max_inner=1,
                                                   stagnation=stag, dtype=np.float32)
        assert sw == expect, (theta, stag, sw, offs, upd)
        assert upd[0] == 1
        assert abs(offs[0] - theta / np.sqrt(1 + theta * theta)) <= 1e-6 * theta


def test_fp32_stagnation_exit_rule():
    """An unreachable tolerance (1e-20) in fp32: the stage stops by the stagnation exit (reading c-10) at the
    first sweep k >= 3 whose max metric is <= 1e-4 and > 1/4 of the previous sweep's, reports convergence,
    and no earlier sweep met that condition."""
    a = testmat.config_matrix("C1", 96)
    x = np.asfortranarray(np.linalg.qr(a.T)[1].T).astype(np.float32)
    xo, _, sw, offs, upd = oracle.block_jacobi(x, None, 32, np.float32(1e-20), np.float32(1e-21), max_sweeps=20,
                                               max_inner=1, stagnation=True, dtype=np.float32)
    assert sw > 0
    k = sw
    assert k >= 3 and offs[k - 1] <= 1e-4 and offs[k - 1] > 0.25 * offs[k - 2]
    for j in range(3, k):
        assert not (offs[j - 1] <= 1e-4 and offs[j - 1] > 0.25 * offs[j - 2])
    assert np.all(upd[:k] > 0)
