"""bench.py's roofline accounting (DESIGN.md sec. 8 "Algorithmic work per unit") against the closed forms,
on a synthetic stats record: Gram bytes n w s per evaluated pair (pairs skipped as unchanged excluded), update
bytes 2 n w s per updated pair and matrix (X; V only when the stage accumulates it), QRP 8 n^3 / 3 bytes."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


STATS = {"sweeps32": 2, "upd_trace32": [10, 3], "skip_trace32": [0, 2],
         "sweeps64": 2, "upd_trace64": [28, 0], "skip_trace64": [0, 5]}


def test_accounting_closed_forms():
    bench = _bench()
    n, b = 256, 32                      # 8 blocks: 4 pairs per round, 7 rounds per sweep, w = 64
    w = 2 * b
    work = bench.algorithmic_work([STATS], n, b)
    assert work["bytes"]["pair_gram_f32"] == (2 * 7 * 4 - 2) * n * w * 4
    assert work["bytes"]["pair_gram_f64"] == (2 * 7 * 4 - 5) * n * w * 8
    assert work["flops"]["pair_gram_f32"] == (2 * 7 * 4 - 2) * n * w * (w + 1)
    # U-route fp32 stage: X only; fp64 refinement: X and V
    assert work["bytes"]["pair_update_f32"] == 13 * 2 * n * w * 4
    assert work["bytes"]["pair_update_f64"] == (28 + 28) * 2 * n * w * 8
    assert work["flops"]["pair_update_f64"] == (28 + 28) * 2 * n * w * w
    assert work["bytes"]["qrp_coop"] == 8 * n ** 3 / 3
    assert work["bound"]["pair_gram_f32"] == "hbm" and work["bound"]["qrp_coop"] == "hbm"


def test_accounting_v_route_and_refine_v():
    bench = _bench()
    n, b, w = 256, 32, 64
    # V-route fp32 stage: V32 updated with X
    work = bench.algorithmic_work([STATS], n, b, v32=True)
    assert work["bytes"]["pair_update_f32"] == (13 + 13) * 2 * n * w * 4
    # sec. 3.4 V formation: only the last v_sweeps64 sweeps accumulate V
    st = dict(STATS, upd_trace64=[28, 4], v_sweeps64=1)
    work = bench.algorithmic_work([st], n, b)
    assert work["bytes"]["pair_update_f64"] == ((28 + 4) + 4) * 2 * n * w * 8   # X: both sweeps, V: the last


def test_roofline_entry_units():
    bench = _bench()
    work = bench.algorithmic_work([STATS], 256, 32)
    peaks = {"measured": {"hbm_gbs": 6000.0}, "micro": {"dmma_tflops": 36.0}}
    r = bench.roofline_for("qrp_coop", 10.0, 1, work, peaks, 256, 32)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] == 6000.0
    assert abs(r["achieved"] - 8 * 256 ** 3 / 3 / 0.010 / 1e9) < 1e-9
    assert abs(r["frac"] - r["achieved"] / 6000.0) < 1e-12
    r64 = bench.roofline_for("pair_update_f64", 1.0, 1, work, peaks, 256, 32)
    assert r64["bound"] == "tensor" and r64["unit"] == "TFLOP/s" and r64["peak"] == 36.0
