"""GPU parity at BASELINE.json's full sizes (C3 4096^2, C4 16384x2048,
C5 8192^2) and the exact-sigma construction at n = 4096, in the launch
configuration bench.py times (default options, one handle, device-resident
input).

At these sizes the oracle cannot run inside the test, so the checks are
  * properties that hold at any size: ||U^T U - I||_max, ||V^T V - I||_max
    <= 1e-13, ||A - U S V^T||_F / ||A||_F <= 1e-13, sigma descending > 0;
  * sigma against a truth that does not come from the CUDA path: the exact
    sigma of the Hadamard-dyadic construction, and the planted sigma of the
    Haar constructions within their construction bound 8 sqrt(n) u sigma_1
    (SURVEY.md 8(c) P2b);
  * sigma element by element (tiered tolerance, the achieved ratio is
    recorded) and sweep counts within +-1 against the oracle's full-size run
    stored in tests/golden/omix_<cfg>.json (written by
    tests/golden/make_golden.py, which calls only oracle/).  The regenerated
    input must have the golden's digest (testmat pins the BLAS thread count
    so that the bits are host-independent); a mismatch fails.
"""
import json
import os

import numpy as np
import pytest

import testmat

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
U64 = 2.0 ** -53
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def mp():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2209_04626_b200 as m
    return m


@pytest.fixture(scope="module")
def handle(mp):
    return mp.Handle(stream=torch.cuda.current_stream().cuda_stream)


def run(mp, handle, a):
    A = torch.from_numpy(np.ascontiguousarray(a.T)).t().cuda()
    U, S, V, st = mp.factor(A, handle=handle)
    return A, U, S, V, st


def check_props(A, U, S, V):
    n = S.numel()
    eye = torch.eye(n, dtype=torch.float64, device=A.device)
    orth_u = float((U.T @ U - eye).abs().max())
    orth_v = float((V.T @ V - eye).abs().max())
    res = float(torch.linalg.norm(A - (U * S) @ V.T) / torch.linalg.norm(A))
    s = S.cpu().numpy()
    assert np.all(s[:-1] >= s[1:]) and np.all(s > 0)
    assert orth_u <= 1e-13, orth_u
    assert orth_v <= 1e-13, orth_v
    assert res <= 1e-13, res
    return s


def golden(name):
    p = os.path.join(GOLD, f"omix_{name}.json")
    assert os.path.exists(p), f"missing oracle golden {p} (tests/golden/make_golden.py {name})"
    return json.load(open(p))


# tiered sigma bound: |dsigma_i|/sigma_i <= max(1e-12, C u min(kappa_s, sigma_1/sigma_i)).
# Achieved on B200 against the full-size goldens: C3 35, C4 22, C5 98 (recorded with MPJSVD_RECORD_DIR); the
# survey's proposal 1e3 is tightened to 250 (2.5x margin over the worst observed).
C_TIER = 250.0


def kappa_bound(sref, kappa, c=C_TIER):
    return np.maximum(1e-12, c * U64 * np.minimum(kappa, sref[0] / sref))


def kappa_s_gpu(A):
    """kappa_2 of the column-scaled input (reading c-16), by torch's SVD on the GPU (harness only)."""
    As = A / torch.linalg.norm(A, dim=0)
    sv = torch.linalg.svdvals(As)
    return float(sv[0] / sv[-1])


def record(name, payload):
    d = os.environ.get("MPJSVD_RECORD_DIR")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, f"fullsize_{name}.json"), "w") as f:
            json.dump(payload, f, indent=1)


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_fullsize_config(mp, handle, name):
    """Full-size parity against the oracle's own full-size run (tests/golden/omix_<name>.json):
    the regenerated input must be bit-identical to the oracle's (digest), sigma element by
    element within the tiered bound, sweeps +-1, plus the size-independent invariants."""
    g = golden(name)
    a = testmat.cached_config(name)
    assert g["digest"] == testmat.digest(a), (
        f"{name}: input digest {testmat.digest(a)} != golden {g['digest']} -- the generator no longer "
        "reproduces the oracle's input bits (testmat.BLAS_THREADS / GEN_VERSION)")
    A, U, S, V, st = run(mp, handle, a)
    s = check_props(A, U, S, V)
    n = a.shape[1]
    if name in ("C3", "C5"):
        planted = testmat.planted_sigma(name)
        assert np.abs(s - planted).max() <= 8 * np.sqrt(n) * U64 * planted[0]
    so = np.array(g["sigma"])
    kap = kappa_s_gpu(A)
    rel = np.abs(s - so) / so
    ratio = rel / (U64 * np.minimum(kap, so[0] / so))
    record(name, {"kappa_s": kap, "max_rel": float(rel.max()), "max_ratio": float(ratio.max()),
                  "argmax_ratio": int(ratio.argmax()), "sweeps": [st["sweeps32"], st["sweeps64"]],
                  "oracle_sweeps": [g["stats"]["sweeps32"], g["stats"]["sweeps64"]]})
    assert np.all(rel <= kappa_bound(so, kap)), (float(ratio.max()), int(ratio.argmax()))
    assert abs(st["sweeps32"] - g["stats"]["sweeps32"]) <= 1, (st["sweeps32"], g["stats"]["sweeps32"])
    assert abs(st["sweeps64"] - g["stats"]["sweeps64"]) <= 1, (st["sweeps64"], g["stats"]["sweeps64"])
    assert st["sweeps64"] <= 4       # "typically three sweeps" + 1


def test_fullsize_exact_sigma(mp, handle):
    a, sigma = testmat.exact_sigma_matrix(4096)
    A, U, S, V, st = run(mp, handle, a)
    s = check_props(A, U, S, V)
    assert np.all(np.abs(s - sigma) / sigma <= kappa_bound(sigma, sigma[0] / sigma[-1]))
    assert np.max(np.abs(s - sigma) / sigma) <= 1e-11



def test_size_limits(mp):
    """The largest sizes the library accepts run in the full-size tests above (C5: n = 8192, the column-pivoted
    QR's limit; C4: m = 16384 rows).  One more column, or one more row, is refused with MPJSVD_ERR_NOT_SUPPORTED
    before any work (no partial run, no device fault), and the handle stays usable."""
    h = mp.Handle(stream=torch.cuda.current_stream().cuda_stream)
    for m, n in [(8193, 8193), (16385, 64)]:
        A = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
        with pytest.raises(mp.MpjsvdError) as e:
            mp.factor(A, handle=h)
        assert e.value.code == -7
    a = testmat.config_matrix("C1", 64)
    U, S, V, st = mp.factor(torch.from_numpy(np.ascontiguousarray(a.T)).t().cuda(), handle=h)
    assert st["rc"] == 0
    h.close()
