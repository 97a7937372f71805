"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs.  Run on a B200 via gpurun:  pytest -m gpu tests/

Tolerances:
  sigma: rel <= 1e-12 when kappa_s <= 1e4, else the tiered
         max(1e-12, 1e3 u min(kappa_s, sigma_1/sigma_i));
  ||U^T U - I||_max, ||V^T V - I||_max <= 1e-13;  ||A - U S V^T||_F/||A||_F <= 1e-13;
  sweeps32 / sweeps64 within +-1 of the oracle.
"""
import numpy as np
import pytest

import oracle
import testmat

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
U64 = 2.0 ** -53


@pytest.fixture(scope="module")
def mp():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2209_04626_b200 as m
    m.lib()
    return m


def dev(a, dtype=torch.float64):
    return torch.from_numpy(np.asfortranarray(a)).to(dtype).cuda().t().contiguous().t()


def host(t):
    return t.detach().cpu().numpy()


def orth(q):
    return np.abs(q.T @ q - np.eye(q.shape[1])).max()


# tiered sigma bound max(1e-12, C u min(kappa_s, sigma_1/sigma_i)) (SURVEY.md 8(c) proposed C = 1e3); the
# achieved ratios recorded on B200 (MPJSVD_RECORD_DIR) are <= 35 at reduced sizes and 98 at full-size C5,
# so C = 250 keeps a 2.5x margin (SURVEY F5 saw 48-281 between correct implementations)
C_TIER = 250.0


def tiered(sref, kappa):
    return np.maximum(1e-12, C_TIER * U64 * np.minimum(kappa, sref[0] / sref))


def record_ratio(got, sref, kappa):
    """Achieved max |dsigma_i| / (sigma_i u min(kappa_s, sigma_1/sigma_i)) of a tiered comparison, appended to
    $MPJSVD_RECORD_DIR/tiered_ratios.jsonl (how much of the 1e3 constant a test uses)."""
    import json
    import os
    d = os.environ.get("MPJSVD_RECORD_DIR")
    if not d:
        return
    got, sref = np.asarray(got, dtype=np.float64), np.asarray(sref, dtype=np.float64)
    r = np.abs(got - sref) / sref / (U64 * np.minimum(kappa, sref[0] / sref))
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "tiered_ratios.jsonl"), "a") as f:
        f.write(json.dumps({"test": os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], "n": int(sref.size),
                            "kappa": float(kappa), "max_ratio": float(r.max()),
                            "max_rel": float((np.abs(got - sref) / sref).max())}) + "\n")


def kappa_s(a):
    d = np.linalg.norm(a, axis=0)
    s = np.linalg.svd(a / d, compute_uv=False)
    return s[0] / s[-1]


# ------------------------------------------------------------------- kernels
def test_gemm_matches_plain_reference(mp):
    rng = np.random.default_rng(0)
    for (M, N, K, ta, tb) in [(130, 70, 33, 0, 0), (64, 64, 64, 1, 0), (100, 37, 211, 0, 1), (5, 200, 129, 1, 1)]:
        A = rng.standard_normal((K, M) if ta else (M, K))
        B = rng.standard_normal((N, K) if tb else (K, N))
        C = host(mp.gemm(bool(ta), bool(tb), dev(A), dev(B)))
        ref = (A.T if ta else A) @ (B.T if tb else B)
        assert np.abs(C - ref).max() <= 4 * K * U64 * (np.abs(A).max() * np.abs(B).max() * K)


@pytest.mark.parametrize("w,dtype", [(64, np.float64), (37, np.float64), (64, np.float32), (16, np.float32)])
def test_inner_solve_vs_oracle(mp, w, dtype):
    rng = np.random.default_rng(w)
    count = 5
    Gs, tol_in = [], (oracle.tol(4096) if dtype == np.float64 else 4 * 64 * 2.0 ** -24) / 8
    for c in range(count):
        b = rng.standard_normal((2 * w, w)) * 10.0 ** rng.uniform(-1, 1, w)
        Gs.append((b.T @ b).astype(dtype))
    Gd = torch.from_numpy(np.stack(Gs)).cuda()
    Go, Eo, rot = mp.inner_solve(Gd, tol_in)
    Go, Eo = host(Go), host(Eo)
    for c in range(count):
        g_ref, e_ref, nrot, isw = oracle.inner_solve(Gs[c], tol_in, dtype=dtype)
        J = np.eye(w) + Eo[c].astype(np.float64)
        eps = 2.0 ** -53 if dtype == np.float64 else 2.0 ** -24
        assert orth(J) < 100 * eps * w
        # diagonalised: off-diagonal of J^T G J below the inner threshold scale
        D = J.T @ Gs[c].astype(np.float64) @ J
        dd = np.sqrt(np.diag(D))
        off = np.abs(D - np.diag(np.diag(D))) / np.outer(dd, dd)
        assert off.max() < 50 * tol_in + 100 * eps
        # same eigenvalues as the oracle's solve (relative, SDD matrices)
        np.testing.assert_allclose(np.sort(np.diag(Go[c])), np.sort(np.diag(g_ref)),
                                   rtol=1e3 * eps, atol=1e3 * eps * np.abs(np.diag(g_ref)).max())
        assert abs(rot[c] - nrot) <= max(3, 0.02 * nrot)


@pytest.mark.parametrize("n,b,m", [(256, 32, 256), (100, 16, 100), (96, 8, 130), (33, 32, 40), (512, 32, 512)])
def test_block_jacobi_f64_vs_oracle(mp, n, b, m):
    rng = np.random.default_rng(n * 7 + b)
    a = testmat.config_matrix("C1", max(n, m))[:m, :n].copy()
    # start from a nearly orthogonal Y like the refinement stage sees it
    q, _ = np.linalg.qr(a)
    x0 = np.asfortranarray(q[:, :n] * np.geomspace(1, 1e-6, n) + 1e-7 * rng.standard_normal((m, n)))
    t = oracle.tol(m)
    xo, vo, sw_o, offs_o, upd_o = oracle.block_jacobi(x0, np.eye(n), b, t, t / 8)
    X, V = dev(x0), dev(np.eye(n))
    sw, st = mp.block_jacobi(X, V, t, t / 8, 30, block_cols=b)
    X, V = host(X), host(V)
    assert sw > 0 and sw_o > 0 and abs(sw - sw_o) <= 1
    s_gpu = np.sort(np.linalg.norm(X, axis=0))[::-1]
    s_or = np.sort(np.linalg.norm(xo, axis=0))[::-1]
    assert np.max(np.abs(s_gpu - s_or) / s_or) < 1e-12
    assert orth(V) < 1e-13
    assert np.abs(x0 @ V - X).max() < 1e-13 * np.abs(x0).max()


@pytest.mark.parametrize("n,b", [(256, 32), (130, 16)])
def test_block_jacobi_f32_vs_oracle(mp, n, b):
    a = testmat.config_matrix("C1", n)
    x0 = np.asfortranarray(np.linalg.qr(a.T)[1].T).astype(np.float32)
    t = np.float32(4 * np.sqrt(n) * 2.0 ** -24)
    xo, vo, sw_o, _, _ = oracle.block_jacobi(x0, np.eye(n, dtype=np.float32), b, t, t / 8,
                                             stagnation=True, dtype=np.float32)
    X, V = dev(x0, torch.float32), dev(np.eye(n), torch.float32)
    sw, st = mp.block_jacobi(X, V, float(t), float(t / 8), 20, stagnation=True, block_cols=b)
    X, V = host(X).astype(np.float64), host(V).astype(np.float64)
    assert abs(abs(sw) - abs(sw_o)) <= 1
    s_gpu = np.sort(np.linalg.norm(X, axis=0))[::-1]
    s_or = np.sort(np.linalg.norm(xo.astype(np.float64), axis=0))[::-1]
    assert np.max(np.abs(s_gpu - s_or) / s_or) < 1e-4
    assert orth(V) < 1e-4


@pytest.mark.parametrize("m,n,pivot", [(300, 300, 1), (257, 100, 1), (1000, 77, 0), (64, 64, 0), (300, 300, 2),
                                       (700, 700, 1), (2100, 700, 0), (300, 300, 3), (700, 700, 3), (257, 100, 3)])
def test_qr_vs_oracle(mp, m, n, pivot):
    """pivot 1: lazy (xLAQPS-style) cooperative QRP; pivot 2: the unblocked
    cooperative kernel; pivot 0: blocked Householder QR; pivot 3: the path's
    mixed-precision RRQR (Alg. 4: fp32 lazy QRP pivots, fp64 blocked QR of A P)
    against the oracle's om_mprrqr."""
    rng = np.random.default_rng(m + n)
    a = np.asfortranarray(rng.standard_normal((m, n)) * 10.0 ** rng.uniform(-2, 2, n))
    packed, tau, perm = mp.qr(dev(a), pivot=pivot)
    packed, tau, perm = host(packed), host(tau), host(perm)
    if pivot == 3:
        p_o, perm_o, tau_o, _ = oracle.mprrqr(a)
    elif pivot:
        p_o, perm_o, tau_o, _ = oracle.qrp(a)
    else:
        p_o, tau_o, _ = oracle.qr(a)
        perm_o = np.arange(n)
    assert np.array_equal(perm, perm_o)
    r, r_o = np.triu(packed[:n]), np.triu(p_o[:n])
    assert np.abs(r - r_o).max() <= 1e-12 * np.abs(r_o).max()
    assert np.abs(tau - tau_o).max() <= 1e-12
    q = oracle.form_q(packed, tau, n)
    assert orth(q) < 1e-13
    assert np.abs(q @ r - a[:, perm]).max() <= 1e-13 * np.abs(a).max()


@pytest.mark.parametrize("m,n", [(8192, 600), (4200, 1200), (2100, 1500)])
def test_qrp_row_instantiations_vs_oracle(mp, m, n):
    """The lazy QRP kernel is instantiated by row count (rows per thread RPT = 16 for 4097..8192 rows: C5's
    8192 x 8192 A1; RPT = 8 for 2049..4096: C3) and deals ~n/148 columns to each CTA.  At those row counts,
    with several columns per CTA, the pivot sequence is identical to the oracle's Businger-Golub QRP and R,
    tau agree to 1e-12."""
    rng = np.random.default_rng(m * 3 + n)
    a = np.asfortranarray(rng.standard_normal((m, n)) * 10.0 ** rng.uniform(-2, 2, n))
    packed, tau, perm = mp.qr(dev(a), pivot=1)
    packed, tau, perm = host(packed), host(tau), host(perm)
    p_o, perm_o, tau_o, _ = oracle.qrp(a)
    assert np.array_equal(perm, perm_o)
    r, r_o = np.triu(packed[:n]), np.triu(p_o[:n])
    assert np.abs(r - r_o).max() <= 1e-12 * np.abs(r_o).max()
    assert np.abs(tau - tau_o).max() <= 1e-12


@pytest.mark.parametrize("m,n,kt,with_v", [(6144, 256, 0, False), (6144, 256, 0, True), (8192, 128, 0, False),
                                           (512, 256, 32, False), (1000, 192, 32, True), (7000, 128, 64, False)])
def test_block_jacobi_f32_gram_variants_vs_oracle(mp, m, n, kt, with_v):
    """fp32 block Jacobi through the TMA Gram variant the C5 path runs (32-row stages at 4 CTAs/SM, chosen
    for >= 6144 rows; forced with gram_kt = 32 at small sizes, 64 forced at large) and the TMA-fed update
    (U-route: no V), with the path's one inner sweep per pair (max_inner32 = 1, reading c-5), against the
    oracle's plain fp32 block Jacobi: sweeps +-1, sigma (column norms) within the TF32x3 stage's accuracy,
    orthogonality of the normalised columns at the fp32 tolerance."""
    rng = np.random.default_rng(m + 17 * n)
    a = (testmat.haar(m, n, 11 + n) * np.geomspace(1.0, 1e-3, n)) @ testmat.haar(n, n, 12 + n).T
    x0 = np.asfortranarray(a).astype(np.float32)
    t = np.float32(4 * np.sqrt(m) * 2.0 ** -24)
    v0 = np.eye(n, dtype=np.float32) if with_v else None
    xo, vo, sw_o, _, _ = oracle.block_jacobi(x0, v0, 32, t, t / 8, max_sweeps=20, max_inner=1,
                                             stagnation=True, dtype=np.float32)
    X = dev(x0, torch.float32)
    V = dev(np.eye(n), torch.float32) if with_v else None
    sw, st = mp.block_jacobi(X, V, float(t), float(t / 8), 20, stagnation=True, max_inner=1, gram_kt=kt)
    X = host(X).astype(np.float64)
    assert abs(abs(sw) - abs(sw_o)) <= 1, (sw, sw_o)
    s_gpu = np.sort(np.linalg.norm(X, axis=0))[::-1]
    s_or = np.sort(np.linalg.norm(xo.astype(np.float64), axis=0))[::-1]
    # two fp32-stage roundings (plain fp32 vs TF32x3 products, ~2^-21 each): absolute errors ~ u sigma_1
    assert np.all(np.abs(s_gpu - s_or) / s_or <= 1e-4 + 2e-6 * s_or[0] / s_or)
    xn = X / np.linalg.norm(X, axis=0)
    assert np.abs(xn.T @ xn - np.eye(n)).max() < 1e-4
    if with_v:
        # V-route accumulation on TF32x3 products (~2^-21 each, reading c-20: 8x the fp32 unit) over ~14
        # sweeps: the oracle's plain fp32 V reaches ~2e-5, the tensor-core stage ~2e-4; V must still map X0 to X
        v = host(V).astype(np.float64)
        assert orth(v) < 1e-3
        assert np.abs(x0.astype(np.float64) @ v - X).max() <= 1e-3 * np.abs(X).max()
    del rng


@pytest.mark.parametrize("mode", [1, 2, 0])
def test_blocked_qr_panel_modes(mp, mode):
    """Blocked Householder QR with its three panel schedules: the cooperative (grid-barrier) panel kernel,
    the flag-chained panel kernel, and the chained kernel with look-ahead (panel p+1 factored on a side stream
    beside panel p's trailing update).  Several 128-column panels, a ragged last panel, tall and square; the
    whole mixed-precision SVD (LQ and U-route switch both run the blocked QR) against the oracle."""
    # odd panel widths (a CTA with one column), a 1-column panel, and > 8192 rows (one column per CTA)
    for m, n in ((1000, 300), (700, 700), (2100, 520), (1000, 301), (600, 257), (9000, 131)):
        rng = np.random.default_rng(m * n)
        a = np.asfortranarray(rng.standard_normal((m, n)) * 10.0 ** rng.uniform(-2, 2, n))
        packed, tau, _ = mp.qr(dev(a), pivot=0, qr_panel_mode=mode)
        packed, tau = host(packed), host(tau)
        p_o, tau_o, _ = oracle.qr(a)
        r, r_o = np.triu(packed[:n]), np.triu(p_o[:n])
        assert np.abs(r - r_o).max() <= 1e-12 * np.abs(r_o).max()
        assert np.abs(tau - tau_o).max() <= 1e-12
        q = oracle.form_q(packed, tau, n)
        assert orth(q) < 1e-13
        assert np.abs(q @ r - a).max() <= 1e-13 * np.abs(a).max()
    a = testmat.config_matrix("C3", 512)
    U, S, V, st = mp.factor(dev(a), qr_panel_mode=mode)
    check_svd(a, host(U), host(S), host(V))
    uo, so, vo, sto, rc = oracle.mixed_svd(a)
    record_ratio(host(S), so, kappa_s(a))
    assert np.all(np.abs(host(S) - so) / so <= tiered(so, kappa_s(a)))
    assert abs(st["sweeps32"] - sto["sweeps32"]) <= 1 and abs(st["sweeps64"] - sto["sweeps64"]) <= 1


@pytest.mark.parametrize("name,n", [("C1", 200), ("C3", 512), ("C2", 352), ("orthcols", 300)])
def test_gate_orth_measure_vs_oracle(mp, name, n):
    """The orth gate measure ||X_t^T X_t - I||_max (fp32; k_gate_orth, 128 x 128 tiles, ragged
    n) against the oracle's plain fp32 triple loop: equal up to fp32 summation order."""
    if name == "orthcols":
        a = np.asfortranarray(testmat.haar(n, n, 5) * 10.0 ** np.linspace(0, -12, n))
    else:
        a = testmat.config_matrix(name, n)
    st = mp.factor(dev(a))[3]
    sto = oracle.mixed_svd(a)[3]
    assert abs(st["orth_measure"] - sto["orth_measure"]) <= 1e-5 + 1e-3 * sto["orth_measure"]


def test_qrp_recompute_path(mp):
    """Strongly decaying partial norms (sigma 1 -> 1e-14) force the partial-norm
    recomputation (xLAQP2 rule) on many columns: pivots and R must still match."""
    n = 400
    a = np.asfortranarray((testmat.haar(n, n, 11) * testmat.geom(n, 1e-14)) @ testmat.haar(n, n, 12).T)
    packed, tau, perm = mp.qr(dev(a), pivot=1)
    packed, tau, perm = host(packed), host(tau), host(perm)
    p_o, perm_o, tau_o, _ = oracle.qrp(a)
    r, r_o = np.triu(packed), np.triu(p_o)
    d, d_o = np.diag(r), np.diag(r_o)
    # QR is normwise backward stable: R_kk agree to ~u ||A|| absolutely; pivots are
    # identical while the diagonal is well above that level
    assert np.abs(d - d_o).max() <= 64 * n * U64 * d_o[0]
    ok = d_o > 1e-8 * d_o[0]
    kmax = int(np.argmin(ok)) if not ok.all() else n
    assert kmax > 100
    assert np.array_equal(perm[:kmax], perm_o[:kmax])
    q = oracle.form_q(packed, tau)
    assert orth(q) < 1e-13
    assert np.abs(q @ r - a[:, perm]).max() <= 1e-13 * np.abs(a).max()


def test_apply_q_vs_oracle(mp):
    rng = np.random.default_rng(4)
    m, n = 500, 140
    a = rng.standard_normal((m, n))
    p_o, tau_o, _ = oracle.qr(a)
    c = rng.standard_normal((m, 90))
    ref = oracle.apply_q(p_o, tau_o, c)
    out = host(mp.apply_q(dev(p_o), torch.from_numpy(tau_o).cuda(), dev(c)))
    assert np.abs(out - ref).max() < 1e-13 * np.abs(c).max() * 10


def test_lift_vs_oracle(mp):
    n = 200
    a = testmat.config_matrix("C1", n)
    x = np.linalg.qr(a.T)[1].T
    x32 = x.astype(np.float32)
    t = np.float32(4 * np.sqrt(n) * 2.0 ** -24)
    _, v32, _, _, _ = oracle.block_jacobi(x32, np.eye(n, dtype=np.float32), 32, t, t / 8, stagnation=True,
                                          dtype=np.float32)
    q_ref, rc = oracle.lift(v32)
    q = host(mp.lift(torch.from_numpy(v32).cuda()))
    assert orth(q) < 1e-14
    assert np.abs(q - q_ref).max() < 1e-13


@pytest.mark.parametrize("n,x_lower", [(200, True), (200, False), (97, True)])
def test_switch_u_vs_oracle(mp, n, x_lower):
    """U-route switch Q = qr(X^T U_low) on X = L and U_low from the fp32 stage,
    GPU against the oracle's step; with x_lower the GEMM skips the zero triangle of X^T."""
    a = testmat.config_matrix("C1", n)
    x = np.asfortranarray(np.linalg.qr(a.T)[1].T)
    e = np.frexp(np.abs(x).max())[1]
    x32 = np.ldexp(x, -e).astype(np.float32)
    t = np.float32(4 * np.sqrt(n) * 2.0 ** -24)
    x32, _, _, _, _ = oracle.block_jacobi(x32, None, 32, t, t / 8, stagnation=True, dtype=np.float32)
    s32 = np.linalg.norm(x32.astype(np.float64), axis=0)
    order = np.argsort(-s32, kind="stable")
    ul = np.asfortranarray(x32[:, order].astype(np.float64) / s32[order])
    q_ref, rc = oracle.switch_u(x, ul)
    q = host(mp.switch_u(dev(x), dev(ul), x_lower=x_lower))
    assert rc == 0 and orth(q) < 1e-14
    assert np.abs(q - q_ref).max() < 1e-11, np.abs(q - q_ref).max()
    y = x @ q        # columns orthogonal to the level of u_low
    g = y.T @ y
    d = np.sqrt(np.diag(g))
    assert np.abs(g / d[:, None] / d[None, :] - np.eye(n)).max() < 1e-4


def test_switch_u_exact_factors(mp):
    """Q = V_X exactly in exact arithmetic: exactly representable U, V."""
    n = 256
    rng = np.random.default_rng(11)
    h = testmat.sylvester_hadamard(n) / 16.0
    uu = rng.choice([-1.0, 1.0], n)[:, None] * h[rng.permutation(n)]
    vv = rng.choice([-1.0, 1.0], n)[:, None] * h[rng.permutation(n)]
    sigma = np.sort((1.0 + rng.integers(0, 1024, n) / 1024.0) * 2.0 ** -np.floor(13 * np.arange(n) / (n - 1)))[::-1]
    a = (uu * sigma) @ vv.T
    q = host(mp.switch_u(dev(a), dev(uu), x_lower=False))
    assert np.abs(q - vv).max() < 50 * n * U64


# ------------------------------------------------------------------- end to end
def check_svd(a, U, S, V, tol_orth=1e-13, tol_res=1e-13):
    assert np.all(S[:-1] >= S[1:]) and np.all(S > 0)
    assert orth(U) <= tol_orth, orth(U)
    assert orth(V) <= tol_orth, orth(V)
    res = np.linalg.norm(a - (U * S) @ V.T) / np.linalg.norm(a)
    assert res <= tol_res, res


@pytest.mark.parametrize("route", [1, 0])
@pytest.mark.parametrize("name,n,kappa", [("C1", 256, 1e4), ("C2", 1024, 1e3), ("C3", 512, None),
                                          ("C4", 256, None), ("C5", 512, None)])
def test_factor_vs_oracle(mp, name, n, kappa, route):
    """route 1: U-route switch (default); 0: V-route (reading c-11)."""
    a = testmat.config_matrix(name, n)
    U, S, V, st = mp.factor(dev(a), switch_u=route)
    U, S, V = host(U), host(S), host(V)
    uo, so, vo, sto, rc = oracle.mixed_svd(a, switch_u=route)
    assert rc == 0 and st["rc"] == 0
    check_svd(a, U, S, V)
    k = kappa if kappa is not None else kappa_s(a)
    rel = np.abs(S - so) / so
    record_ratio(S, so, k)
    if k <= 1e4:
        assert rel.max() <= 1e-12, rel.max()
    assert np.all(rel <= tiered(so, k))
    assert abs(st["sweeps32"] - sto["sweeps32"]) <= 1, (st["sweeps32"], sto["sweeps32"])
    assert abs(st["sweeps64"] - sto["sweeps64"]) <= 1, (st["sweeps64"], sto["sweeps64"])
    # singular vectors agree with the oracle up to sign where sigma is well separated
    gap = np.minimum(np.abs(np.diff(so, prepend=np.inf)), np.abs(np.diff(so, append=-np.inf))) / so
    ok = gap > 1e-6
    assert np.all(np.abs(np.abs(np.sum(V * vo, axis=0))[ok] - 1) < 1e-8)


@pytest.mark.parametrize("m,n", [(100, 100), (257, 257), (77, 33), (1000, 77), (2, 2), (40, 3)])
def test_factor_ragged_shapes(mp, m, n):
    rng = np.random.default_rng(m * n)
    a = np.asfortranarray(rng.standard_normal((m, n)) * 10.0 ** rng.uniform(-2, 2, n))
    U, S, V, st = mp.factor(dev(a))
    U, S, V = host(U), host(S), host(V)
    check_svd(a, U, S, V)
    so = oracle.mixed_svd(a)[1]
    record_ratio(S, so, kappa_s(a))
    assert np.all(np.abs(S - so) / so <= tiered(so, kappa_s(a)))


def test_exact_sigma(mp):
    for n in (256, 1024):
        a, sigma = testmat.exact_sigma_matrix(n)
        U, S, V, st = mp.factor(dev(a))
        rel = np.abs(host(S) - sigma) / sigma
        assert np.all(rel <= tiered(sigma, sigma[0] / sigma[-1]))
        check_svd(a, host(U), host(S), host(V))


def test_graded_high_relative_accuracy(mp):
    import mpmath
    mpmath.mp.dps = 80
    a, _ = testmat.graded_matrix(32, 40)
    ref = np.array(sorted([float(x) for x in mpmath.svd_r(mpmath.matrix(a.tolist()), compute_uv=False)],
                          reverse=True))
    U, S, V, st = mp.factor(dev(a))
    assert np.max(np.abs(host(S) - ref) / ref) < 1e-13


def test_host_pointers_e2e_equal_device_path(mp):
    a = testmat.config_matrix("C1", 128)
    U1, S1, V1, _ = mp.factor(dev(a))
    At = torch.from_numpy(a.T.copy()).t()          # host, column-major
    U2, S2, V2, st = mp.factor(At)
    assert not U2.is_cuda
    assert np.array_equal(host(S1), S2.numpy())
    assert np.array_equal(host(U1), U2.numpy()) and np.array_equal(host(V1), V2.numpy())


def test_deterministic(mp):
    a = testmat.config_matrix("C2", 256)
    r1 = mp.factor(dev(a))
    r2 = mp.factor(dev(a))
    for x, y in zip(r1[:3], r2[:3]):
        assert torch.equal(x, y)


def test_power_of_two_scaling_bitwise(mp):
    a = testmat.config_matrix("C2", 128)
    S1 = host(mp.factor(dev(a))[1])
    S2 = host(mp.factor(dev(a * 2.0 ** -40))[1])
    assert np.array_equal(S2, S1 * 2.0 ** -40)


def test_force_fp64_path(mp):
    a = testmat.config_matrix("C1", 256)
    U, S, V, st = mp.factor(dev(a), path=2)
    so = oracle.mixed_svd(a, path=2)
    assert st["sweeps32"] == 0 and abs(st["sweeps64"] - so[3]["sweeps64"]) <= 1
    check_svd(a, host(U), host(S), host(V))


def test_errors(mp):
    a = testmat.config_matrix("C1", 64)
    bad = a.copy()
    bad[5, 7] = np.nan
    with pytest.raises(mp.MpjsvdError) as e:
        mp.factor(dev(bad))
    assert e.value.code == -2
    z = a.copy()
    z[:, 3] = 0.0
    with pytest.raises(mp.MpjsvdError) as e:
        mp.factor(dev(z))
    assert e.value.code == -3
    with pytest.raises(mp.MpjsvdError) as e:
        mp.factor(dev(np.ones((4, 8))))
    assert e.value.code == -1
    # not converged: soft warning, outputs filled
    U, S, V, st = mp.factor(dev(a), max_sweeps64=1)
    assert st["rc"] == 1 and not st["converged"]


@pytest.mark.parametrize("kind", ["nan_row", "nan_cols", "inf_col", "all_nan"])
def test_nonfinite_inputs_fail_cleanly(mp, kind):
    """a NaN/Inf input must return MPJSVD_ERR_NONFINITE before the QRP (whose argmax has no
    finite candidate) -- a whole NaN row, several NaN columns, an Inf column, all NaN -- on the square and the
    tall path and with mp_rrqr; the same handle then factors a valid matrix correctly (no context damage)."""
    a = testmat.config_matrix("C1", 256)
    bad = a.copy()
    if kind == "nan_row":
        bad[17, :] = np.nan
    elif kind == "nan_cols":
        bad[:, [3, 100, 255]] = np.nan
    elif kind == "inf_col":
        bad[:, 9] = np.inf
    else:
        bad[:] = np.nan
    h = mp.Handle(stream=torch.cuda.current_stream().cuda_stream)
    for arr, kw in ((bad, {}), (np.vstack([bad, bad]), {}), (bad, {"mp_rrqr": 1})):
        hh = mp.Handle(stream=torch.cuda.current_stream().cuda_stream, **kw) if kw else h
        with pytest.raises(mp.MpjsvdError) as e:
            mp.factor(dev(np.asfortranarray(arr)), handle=hh)
        assert e.value.code == -2
    U, S, V, st = mp.factor(dev(a), handle=h)
    check_svd(a, host(U), host(S), host(V))
    torch.cuda.synchronize()


@pytest.mark.parametrize("name,n", [("C3", 512), ("C2", 384), ("C4", 256)])
def test_factor_mixed_precision_rrqr_vs_oracle(mp, name, n):
    """The mixed-precision RRQR preconditioning (Alg. 4;
    option mp_rrqr = 1) end to end against the oracle run with the same option."""
    a = testmat.config_matrix(name, n)
    U, S, V, st = mp.factor(dev(a), mp_rrqr=1)
    U, S, V = host(U), host(S), host(V)
    uo, so, vo, sto, rc = oracle.mixed_svd(a, mp_rrqr=1)
    assert rc == 0 and st["rc"] == 0
    check_svd(a, U, S, V)
    record_ratio(S, so, kappa_s(a))
    assert np.all(np.abs(S - so) / so <= tiered(so, kappa_s(a)))
    assert abs(st["sweeps32"] - sto["sweeps32"]) <= 1
    assert abs(st["sweeps64"] - sto["sweeps64"]) <= 1


def test_gram_tma_equals_cp_async_gram(mp):
    """The TMA-fed fp32 Gram (k_pair_gram_tma) lands the same operand layout and issues the same MMA
    sequence as the cp.async Gram: with the same row slabs (split_rows = 128) the whole SVD is bitwise
    equal; the default (automatic) slabs stay within the parity bar."""
    a = testmat.config_matrix("C3", 512)
    res = {}
    for tma in (2, 1, 0):
        U, S, V, st = mp.factor(dev(a), split_rows=128, gram_tma=tma)
        res[tma] = (host(U), host(S), host(V), st["sweeps32"], st["sweeps64"])
    for x, y, z in zip(res[2], res[1], res[0]):
        assert np.array_equal(np.asarray(x), np.asarray(y))
        assert np.array_equal(np.asarray(x), np.asarray(z))
    # ragged n (last block narrower) and an odd block count (bye pairs) through the TMA Gram
    for n in (200, 352):
        b = testmat.config_matrix("C1", n)
        U, S, V, st = mp.factor(dev(b))
        check_svd(b, host(U), host(S), host(V))
        so = oracle.mixed_svd(b)[1]
        assert np.max(np.abs(host(S) - so) / so) <= 1e-12


@pytest.mark.parametrize("name,n,extra", [("C1", 256, {}), ("C3", 512, {"virtual_shards": 2}),
                                          ("C2", 384, {"max_sweeps64": 30})])
def test_skip_unchanged_pairs_is_exact(mp, name, n, extra):
    """Skipping the Gram and solve of a pair whose blocks did not rotate since its previous evaluation
    (one sweep earlier) is exact: outputs and sweep counts are bitwise those of evaluating every pair."""
    a = testmat.config_matrix(name, n)
    res = {}
    for sk in (1, 0):
        U, S, V, st = mp.factor(dev(a), skip_unchanged=sk, **extra)
        res[sk] = (host(U), host(S), host(V), st)
    for x, y in zip(res[1][:3], res[0][:3]):
        assert np.array_equal(x, y)
    s1, s0 = res[1][3], res[0][3]
    for k in ("sweeps32", "sweeps64", "upd_trace32", "upd_trace64", "off_trace32", "off_trace64"):
        assert s1[k] == s0[k], k
    assert sum(s0["skip_trace32"]) == 0 and sum(s0["skip_trace64"]) == 0
    # the final check sweep follows a sweep with few rotations: some pairs are skipped
    assert sum(s1["skip_trace32"]) + sum(s1["skip_trace64"]) > 0


@pytest.mark.parametrize("case", ["cond", "tail", "orth", "jacobi", "qrsvd"])
def test_auto_path_vs_oracle(mp, case):
    """AUTO (reading c-15): the GPU takes the oracle's branch on inputs built
    to trigger each gate (tests/test_oracle_pins.py auto_cases) and matches its sigma; the fp32 QR-SVD
    branch (cuSOLVER sgesvd on the GPU, LAPACK sgesvd in the oracle) only seeds the fp64 refinement."""
    import test_oracle_pins as pins
    a, kw, taken, sig = pins.auto_cases()[case]
    U, S, V, st = mp.factor(dev(a), path=1, **kw)
    U, S, V = host(U), host(S), host(V)
    uo, so, vo, sto, rc = oracle.mixed_svd(a, path=1, **kw)
    assert rc == 0 and st["rc"] == 0
    assert st["path_taken"] == sto["path_taken"] == taken, (st["path_taken"], sto["path_taken"], taken)
    check_svd(a, U, S, V)
    kap = kappa_s(a)
    record_ratio(S, so, kap)
    assert np.all(np.abs(S - so) / so <= tiered(so, kap))
    if sig is not None:
        assert np.max(np.abs(S - sig) / sig) <= 1e-13
    assert abs(st["sweeps64"] - sto["sweeps64"]) <= 1
    np.testing.assert_allclose(st["cond_scaled"], sto["cond_scaled"], rtol=1e-6)
    np.testing.assert_allclose(st["cond_d"], sto["cond_d"], rtol=1e-12)


@pytest.mark.parametrize("name,n", [("C2", 384), ("C3", 512), ("C4", 256), ("C5", 320)])
def test_gate_measures_vs_oracle(mp, name, n):
    """All AUTO gate quantities (reading c-15) on the config recipes: the column-
    scaled kappa_1(R_s) (GPU: triangular solve on DMMA GEMMs + column reductions; oracle: back substitution),
    cond(D), the orth measure and the tail fraction equal the oracle's up to rounding order; same branch."""
    a = testmat.config_matrix(name, n)
    st = mp.factor(dev(a), path=1)[3]
    sto = oracle.mixed_svd(a, path=1)[3]
    assert st["path_taken"] == sto["path_taken"]
    assert abs(st["cond_scaled"] - sto["cond_scaled"]) <= 1e-9 * sto["cond_scaled"] * max(1.0, 1e-4 * sto["cond_scaled"])
    assert abs(st["cond_d"] - sto["cond_d"]) <= 1e-12 * sto["cond_d"]
    assert abs(st["orth_measure"] - sto["orth_measure"]) <= 1e-5 + 1e-3 * sto["orth_measure"]
    assert st["tail_fraction"] == sto["tail_fraction"]


@pytest.mark.parametrize("name,n,extra", [("C1", 256, {}), ("C2", 512, {}), ("C3", 512, {}), ("C5", 640, {}),
                                          ("C4", 256, {}), ("C3", 512, {"virtual_shards": 4}),
                                          ("C5", 384, {"path": 2})])
def test_refine_v_vs_oracle(mp, name, n, extra):
    """Sec. 3.4 V formation (refine_v = 1; reading c-23): refinement without V, V_X =
    qr(X^T U_X), one accumulating refinement -- against the oracle's same steps: valid SVD, sigma within the
    tiered bound, both fp64 stages' sweep counts +-1, and the accumulating stage converges within 2 sweeps
    ("always converges in one sweep" + the check sweep).  Also through the sharded engine and the fp64-only
    path."""
    a = testmat.config_matrix(name, n)
    U, S, V, st = mp.factor(dev(a), refine_v=1, **extra)
    U, S, V = host(U), host(S), host(V)
    oo = {"path": extra["path"]} if "path" in extra else {}
    uo, so, vo, sto, rc = oracle.mixed_svd(a, refine_v=1, **oo)
    assert rc == 0 and st["rc"] == 0
    check_svd(a, U, S, V)
    record_ratio(S, so, kappa_s(a))
    assert np.all(np.abs(S - so) / so <= tiered(so, kappa_s(a)))
    assert 1 <= st["v_sweeps64"] <= 2 and 1 <= sto["v_sweeps64"] <= 2
    assert abs((st["sweeps64"] - st["v_sweeps64"]) - (sto["sweeps64"] - sto["v_sweeps64"])) <= 1
    assert abs(st["sweeps32"] - sto["sweeps32"]) <= 1


@pytest.mark.parametrize("opts,oopts", [
    ({"fp32_tensor_cores": 0}, {}),
    ({"pdl_overlap": 0}, {}),
    ({"pdl_overlap": 0, "switch_u": 0}, {"switch_u": 0}),
    ({"block_cols": 16}, {"b": 16}),
    ({"x_from_lq": 0}, {"x_from_lq": 0}),
    ({"max_inner32": 2}, {"max_inner32": 2}),
    ({"l2_order": 1}, {}),
    ({"l2_order": 1, "switch_u": 0}, {"switch_u": 0}),
])
def test_option_paths_vs_oracle(mp, opts, oopts):
    """Non-default implementation paths (FFMA fp32 stage, serial solve/update, V-route without overlap,
    b = 16 (SIMT kernels), X = R, two fp32 inner sweeps, the L2-aware traversal: interleaved Gram row
    tiles and the bottom-up tile-group-major update) against the oracle run with the same
    algorithmic options: valid SVD, tiered sigma bound, sweeps +-1."""
    a = testmat.config_matrix("C3", 384)
    U, S, V, st = mp.factor(dev(a), **opts)
    U, S, V = host(U), host(S), host(V)
    uo, so, vo, sto, rc = oracle.mixed_svd(a, **oopts)
    assert rc == 0 and st["rc"] == 0
    check_svd(a, U, S, V)
    record_ratio(S, so, kappa_s(a))
    assert np.all(np.abs(S - so) / so <= tiered(so, kappa_s(a)))
    assert abs(st["sweeps64"] - sto["sweeps64"]) <= 1
    if not opts.get("x_from_lq", 1) == 0:
        assert abs(st["sweeps32"] - sto["sweeps32"]) <= 1

@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(200, 200), (352, 352), (1000, 77), (6144, 256)])
def test_l2_order_ragged_vs_oracle(mp, m, n):
    """l2_order = 1 (interleaved Gram row tiles, bottom-up group-major update) on ragged block widths, odd block
    counts (bye pairs), a tall input and the 32-row-stage Gram's row count: sigma against the oracle within the
    parity bar, valid SVD, and the same sweep counts as the default traversal (the two differ in rounding only)."""
    a = testmat.config_matrix("C1", n) if m == n else testmat.config_matrix("C4", n, m=m)
    r0 = mp.factor(dev(a))
    r1 = mp.factor(dev(a), l2_order=1)
    U, S, V = host(r1[0]), host(r1[1]), host(r1[2])
    check_svd(a, U, S, V)
    so = oracle.mixed_svd(a)[1]
    if m == n:
        assert np.max(np.abs(S - so) / so) <= 1e-12
    else:
        assert np.all(np.abs(S - so) / so <= tiered(so, kappa_s(a)))
    assert abs(r1[3]["sweeps32"] - r0[3]["sweeps32"]) <= 1 and abs(r1[3]["sweeps64"] - r0[3]["sweeps64"]) <= 1


@pytest.mark.parametrize("name,n", [("exact", 64), ("C1", 256), ("C3", 500), ("C2", 384), ("C5", 1000)])
def test_qrsvd32_vs_oracle(mp, name, n):
    """The hand-written fp32 QR SVD of the AUTO branch (k_bidiag32 cooperative bidiagonalisation, k_bdqr32
    implicit-shift QR, k_rot_apply fp64 accumulation, WY application; reading c-24) against the oracle's
    plain-C steps (oracle/qrsvd.c): sigma within twice the fp32 bound n u32 sigma_1, U orthogonal to the
    fp32 level, U^T X with orthogonal rows, and left singular vectors equal up to sign where sigma is well
    separated."""
    U32 = 2.0 ** -24
    if name == "exact":
        a, _ = testmat.exact_sigma_matrix(n)
    else:
        a = testmat.config_matrix(name, n)
        a = np.asfortranarray(np.linalg.qr(a.T)[1].T)     # X = L like the path (lower triangular)
    x = np.asfortranarray((a / np.abs(a).max()).astype(np.float32))
    U, S = mp.qrsvd32(dev(x, torch.float32))
    U, S = host(U), host(S).astype(np.float64)
    uo, so, rc = oracle.qrsvd32(x)
    so = so.astype(np.float64)
    assert rc == 0
    assert np.all(np.diff(S) <= 0)
    assert np.abs(S - so).max() <= 2 * n * U32 * so[0]
    assert orth(U) <= 4 * n * U32
    g = U.T @ x.astype(np.float64)
    gg = g @ g.T
    assert np.abs(gg - np.diag(np.diag(gg))).max() <= 8 * n * U32 * so[0] ** 2
    gap = np.minimum(np.r_[np.inf, -np.diff(so)], np.r_[-np.diff(so), np.inf]) / so[0]
    ok = gap > 1e-3
    dots = np.abs(np.sum(U * uo, axis=0))
    assert np.all(dots[ok] >= 1 - 1e-3)


def test_auto_qrsvd_branch_larger_vs_oracle(mp):
    """AUTO with tol_alg = 1e-3 (every C-config input then takes the QR SVD branch, F2): end to end against
    the oracle's same branch at n = 512 -- valid SVD, tiered sigma, fp64 sweeps +-1."""
    a = testmat.config_matrix("C3", 512)
    U, S, V, st = mp.factor(dev(a), path=1, tol_alg=1e-3)
    U, S, V = host(U), host(S), host(V)
    uo, so, vo, sto, rc = oracle.mixed_svd(a, path=1, tol_alg=1e-3)
    assert rc == 0 and st["rc"] == 0
    assert st["path_taken"] == sto["path_taken"] == 6
    check_svd(a, U, S, V)
    record_ratio(S, so, kappa_s(a))
    assert np.all(np.abs(S - so) / so <= tiered(so, kappa_s(a)))
    assert abs(st["sweeps64"] - sto["sweeps64"]) <= 1


@pytest.mark.parametrize("variant,kt", [(8, 0), (9, 0), (8, 32), (9, 32), (10, 0), (11, 0), (10, 32), (16, 0), (17, 0),
                                        (18, 0), (19, 0), (20, 0), (21, 0), (22, 0), (23, 0), (24, 0), (25, 0), (26, 0)])
def test_gram_tma_warp_specialised_bitwise(mp, variant, kt):
    """Gram kernel variants with the same MMA sequence as k_pair_gram_tma: 8 / 9 warp-specialised (producer +
    MMA lane, lo-part warps, per-stage mbarriers instead of a CTA barrier per tile), 10 / 11 the 128-byte-
    swizzled operand layout fed by 2-D TMA boxes (3 / 4 stages), 16 / 17 its warp-specialised form, 18 / 19 the
    same with the A operand [H ; L] in tensor memory (8 / 6 stages of raw columns only): the whole SVD is bitwise
    equal when the row slabs are the same (split_rows fixed)."""
    a = testmat.config_matrix("C3", 512)
    r0 = mp.factor(dev(a), split_rows=128, gram_kt=kt)
    r1 = mp.factor(dev(a), split_rows=128, gram_kt=kt, gram_variant=variant)
    for x, y in zip(r0[:3], r1[:3]):
        assert torch.equal(x, y)
    assert r0[3]["sweeps32"] == r1[3]["sweeps32"] and r0[3]["sweeps64"] == r1[3]["sweeps64"]


@pytest.mark.parametrize("extra", [{}, {"switch_u": 0}, {"virtual_shards": 2}])
def test_update_a_in_tmem_bitwise(mp, extra):
    """The fp32 update with its A operand (W hi / lo) in tensor memory (update_variant = 1, tcgen05.mma
    A-from-TMEM, double buffered) computes the same products in the same order as the shared-memory-A update:
    the whole SVD is bitwise equal (U-route TMA tiles, V-route cp.async tiles with V, sharded engine)."""
    a = testmat.config_matrix("C3", 512)
    r0 = mp.factor(dev(a), update_variant=0, **extra)
    for v in (1,):
        r1 = mp.factor(dev(a), update_variant=v, **extra)
        for x, y in zip(r0[:3], r1[:3]):
            assert torch.equal(x, y)
        assert r0[3]["sweeps32"] == r1[3]["sweeps32"] and r0[3]["sweeps64"] == r1[3]["sweeps64"]


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,pivot", [(8192, 600, 1), (2100, 700, 1), (700, 700, 1), (257, 100, 1), (4200, 900, 3)])
def test_qrp_panel_ring_bitwise(mp, m, n, pivot):
    """The lazy QRP's end-of-panel update through the per-thread cp.async ring (qrp_panel_stages = -1 auto,
    2, 3) performs the same fused multiply-adds in the same order as the register path (0): packed factors,
    tau and pivots are bitwise equal, including the fp32 QRP of Alg. 4 (pivot 3)."""
    rng = np.random.default_rng(m * 7 + n)
    a = np.asfortranarray(rng.standard_normal((m, n)) * 10.0 ** rng.uniform(-2, 2, n))
    ref = mp.qr(dev(a), pivot=pivot, qrp_panel_stages=0)
    for st in (-1, 2, 3):
        out = mp.qr(dev(a), pivot=pivot, qrp_panel_stages=st)
        for x, y in zip(ref, out):
            assert torch.equal(x, y), st


@pytest.mark.parametrize("name,n,extra", [("C3", 512, {}), ("C5", 640, {"virtual_shards": 2}), ("C1", 300, {}),
                                          ("C2", 256, {"refine_v": 1}), ("C3", 384, {"skip_unchanged": 0})])
def test_gram_pdl_bitwise(mp, name, n, extra):
    """The Jacobi rounds with the solve launched as a programmatic dependent of the Gram (gram_pdl = 1: per-pair
    counters, a pair's solve starts when its row-slab partials are in) compute exactly what the serialised
    rounds (0) compute: the whole SVD is bitwise equal (fp32 tcgen05 Gram, fp64 DMMA Gram, ragged widths,
    exact skip on and off, the sharded engine)."""
    a = testmat.config_matrix(name, n)
    r0 = mp.factor(dev(a), gram_pdl=0, **extra)
    r1 = mp.factor(dev(a), gram_pdl=1, **extra)
    for x, y in zip(r0[:3], r1[:3]):
        assert torch.equal(x, y)
    assert r0[3]["sweeps32"] == r1[3]["sweeps32"] and r0[3]["sweeps64"] == r1[3]["sweeps64"]
