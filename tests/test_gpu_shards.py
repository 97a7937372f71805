"""GPU: the sharded (multi-GPU) Jacobi engine, emulated on one B200.

mpjsvd_options.virtual_shards = G runs the engine of SURVEY.md 8(e) with G
shards on one device: shard buffers (2k+2 column slabs per rank), the block
exchange after every round as device copies between the shards' buffers,
and one kernel over all shards' pairs (the guide's rule for fewer GPUs than
ranks).  Only the transport differs from the NCCL path (ncclSend/ncclRecv
instead of cudaMemcpyAsync; the plan and the move list are the same code, and
the plan's exchange logic is tested over gloo in tests/test_shard_plan.py).

  * N_b a multiple of 2G: the schedule is the one-GPU schedule, so U, S, V and
    the sweep traces are bitwise identical to G = 1 (SURVEY.md 8(e)
    "Determinism");
  * N_b padded to a multiple of 2G: a different valid schedule; parity with
    the oracle within the tiered tolerance and sweeps +-1;
  * the step-level block Jacobi entry through the shards vs the oracle.
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


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("name,n,b", [("C1", 256, 8), ("C5", 512, 16), ("C2", 512, 32)])
def test_virtual_shards_bitwise_equal_one_gpu(mp, G, name, n, b):
    a = testmat.config_matrix(name, n)
    nblk = -(-n // b)
    assert (nblk + (nblk & 1)) % (2 * G) == 0
    U1, S1, V1, st1 = mp.factor(dev(a), block_cols=b)
    Ug, Sg, Vg, stg = mp.factor(dev(a), block_cols=b, virtual_shards=G)
    assert torch.equal(S1, Sg) and torch.equal(U1, Ug) and torch.equal(V1, Vg)
    for key in ("sweeps32", "sweeps64", "upd_trace32", "upd_trace64", "off_trace32", "off_trace64"):
        assert st1[key] == stg[key], key


@pytest.mark.parametrize("G,name,n,b", [(4, "C1", 200, 16), (8, "C5", 300, 8), (2, "C3", 333, 32),
                                        (8, "C2", 96, 32)])
def test_virtual_shards_padded_schedule_vs_oracle(mp, G, name, n, b):
    a = testmat.config_matrix(name, n)
    U, S, V, st = mp.factor(dev(a), block_cols=b, virtual_shards=G)
    U, S, V = host(U), host(S), host(V)
    uo, so, vo, sto, rc = oracle.mixed_svd(a, b=b)
    assert st["rc"] == 0
    d = np.linalg.norm(a, axis=0)
    s = np.linalg.svd(a / d, compute_uv=False)
    k = s[0] / s[-1]
    assert np.all(np.abs(S - so) / so <= tiered(so, k))
    assert orth(U) <= 1e-13 and orth(V) <= 1e-13
    assert np.linalg.norm(a - (U * S) @ V.T) / np.linalg.norm(a) <= 1e-13
    assert abs(st["sweeps32"] - sto["sweeps32"]) <= 1
    assert abs(st["sweeps64"] - sto["sweeps64"]) <= 1


@pytest.mark.parametrize("G", [2, 4])
def test_virtual_shards_block_jacobi_f64_vs_oracle(mp, G):
    rng = np.random.default_rng(11)
    m, n, b = 300, 128, 16
    x = rng.standard_normal((m, n)) * 10.0 ** rng.uniform(-3, 3, n)
    tol = 4 * np.sqrt(m) * U64
    X = dev(x)
    V = dev(np.eye(n))
    h = mp.Handle(stream=torch.cuda.current_stream().cuda_stream, block_cols=b, virtual_shards=G)
    sw, st = mp.block_jacobi(X, V, tol=tol, tol_in=tol / 8, max_sweeps=30, handle=h)
    X1 = dev(x)
    V1 = dev(np.eye(n))
    h1 = mp.Handle(stream=torch.cuda.current_stream().cuda_stream, block_cols=b)
    sw1, st1 = mp.block_jacobi(X1, V1, tol=tol, tol_in=tol / 8, max_sweeps=30, handle=h1)
    assert sw == sw1 and torch.equal(X, X1) and torch.equal(V, V1)     # N_b = 8: same schedule
    xs, vs = host(X), host(V)
    assert np.abs(xs - x @ vs).max() <= 1e-12 * np.abs(x).max() * np.sqrt(n)
    s = np.sort(np.linalg.norm(xs, axis=0))[::-1]
    sref = np.linalg.svd(x, compute_uv=False)
    assert np.max(np.abs(s - sref) / sref) <= 1e-10
    xo, vo, sw_o, _, _ = oracle.block_jacobi(x, np.eye(n), b, tol, tol / 8, max_sweeps=30)
    assert abs(sw - sw_o) <= 1


def test_nccl_communicator_world1_equals_plain(mp):
    """The NCCL code path of mpjsvd_factor (header agreement all-reduce, status
    broadcasts, matrix broadcasts, per-sweep counter all-reduces) on a
    one-rank communicator: bitwise equal to the handle without one.  (More
    ranks need more GPUs: the exchange itself is covered by the virtual
    shards above and by the gloo test of the plan.)"""
    a = testmat.config_matrix("C1", 256)
    U1, S1, V1, st1 = mp.factor(dev(a))
    h = mp.Handle(stream=torch.cuda.current_stream().cuda_stream)
    try:
        uid = mp.comm_unique_id()
    except mp.MpjsvdError as e:
        pytest.skip(f"NCCL unavailable: {e}")
    h.comm_init(0, 1, uid)
    assert h.comm_info() == (0, 1)
    U2, S2, V2, st2 = mp.factor(dev(a), handle=h)
    assert torch.equal(S1, S2) and torch.equal(U1, U2) and torch.equal(V1, V2)
    assert st1["sweeps64"] == st2["sweeps64"]


@pytest.mark.parametrize("n", [256, 1000])
def test_fp32_tensor_core_stage_vs_simt_and_oracle(mp, n):
    """The fp32 stage on tcgen05 TF32 (hi/lo split, reading c-20) against the
    FFMA path and the oracle: same sweeps +-1, and the final SVD within the
    parity bar either way."""
    a = testmat.config_matrix("C5", n)
    U1, S1, V1, st1 = mp.factor(dev(a), fp32_tensor_cores=1)
    U0, S0, V0, st0 = mp.factor(dev(a), fp32_tensor_cores=0)
    uo, so, vo, sto, rc = oracle.mixed_svd(a)
    for (U, S, V, st) in ((U1, S1, V1, st1), (U0, S0, V0, st0)):
        U, S, V = host(U), host(S), host(V)
        assert orth(U) <= 1e-13 and orth(V) <= 1e-13
        assert np.linalg.norm(a - (U * S) @ V.T) / np.linalg.norm(a) <= 1e-13
        k = so[0] / so[-1]
        assert np.all(np.abs(S - so) / so <= tiered(so, k))
        assert abs(st["sweeps32"] - sto["sweeps32"]) <= 1
        assert abs(st["sweeps64"] - sto["sweeps64"]) <= 1
