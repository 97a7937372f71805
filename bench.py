#!/usr/bin/env python
"""bench.py -- time-to-SVD of the B200 mixed-precision Jacobi SVD (C-ABI path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl mpjsvd|reference]

A step is one full fp64 SVD A = U S V^T (mpjsvd_factor: QRP + LQ
preconditioning, fp32 block Jacobi computing U_low, U-route precision switch,
fp64 block Jacobi refinement, assembly) of BASELINE.json's config on inputs
resident in HBM.  Metric (BASELINE.json): "fp64 SVD time at n=4096 and 8192
(1/2/4/8 B200); sweep HBM GB/s vs peak" -> value = seconds per SVD at n = 8192
(C5, lower is better); the n = 4096 config (C3) is timed in the same run under
"also".

Timing: W warm-up steps, then K steps between CUDA events on the handle's
stream with a 512 MiB L2 flush before each step and no per-kernel
instrumentation (value); a separate pass of min(K, 5) steps with per-launch
events feeds "kernels", "roofline" and "jacobi_roofline" ("profiled"); "e2e"
times the same C-ABI call on pinned host buffers (H2D of A and D2H of U, S, V
inside the timed region).  nvidia-smi clocks are sampled during the timed steps.

Rank 0 prints ONE JSON line.  Multi-GPU: `--gpus N` (N > 1) re-launches itself
under torch.distributed.run with N ranks when WORLD_SIZE is unset; one SVD of
the config per step, sharded over the N GPUs: rank 0 holds A
and the outputs and runs preconditioning / switch / assembly, both Jacobi
stages run column-block sharded with the per-round block exchange over NCCL
(ncclSend/ncclRecv inside libmpjsvd.so).  Total work is fixed as N grows
("scaling": "strong"); the timed region is bracketed by barrier +
synchronize and the max over ranks is reported.

--impl reference times the oracle O-MIX (the only reference of this tier) on
the host cores on a bounded sample (the config's recipe at n = 1024, scaled by
the n^3 work ratio); --impl reference --full CFG runs O-MIX once on the full
config (minutes) to calibrate that extrapolation (profiles/cpu_oracle_full_*).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 SVD time at n=4096 and 8192 (1/2/4/8 B200); sweep HBM GB/s vs peak"
SAMPLE_N = 2048          # largest oracle sample size for the CPU baseline
SAMPLE_BUDGET_S = 150.0  # host seconds a whole --impl reference run may spend on its samples


def sample_n_for(runs: int, cores: int) -> int:
    """Largest sample size (<= SAMPLE_N) whose O-MIX run, repeated `runs` times, fits SAMPLE_BUDGET_S.
    Cost model from the measured 1024^2 C5-recipe run (2.73 s on 16 cores of the GPU box host) scaled by n^3
    and by the core count; the sample is what is measured, the model only picks its size."""
    for n in (2048, 1792, 1536, 1280, 1024, 768, 512):
        est = 2.73 * (n / 1024.0) ** 3 * 16.0 / max(1, cores)
        if n <= SAMPLE_N and est * max(1, runs) <= SAMPLE_BUDGET_S:
            return n
    return 512


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("MPJSVD_BENCH_CONFIG", "C5"))
    ap.add_argument("--impl", default="mpjsvd", choices=["mpjsvd", "reference"])
    ap.add_argument("--block-cols", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-profile", action="store_true", help="skip the separate per-kernel profiled pass")
    ap.add_argument("--also", default="C3", help="comma list of extra configs timed in the same run "
                                                  "(reported under 'also'; '' for none)")
    ap.add_argument("--full", default="", help="--impl reference: time O-MIX once on this FULL config "
                                                  "(minutes) and print the measurement (profiles/cpu_oracle_full_*)")
    ap.add_argument("--dist-check", action="store_true",
                    help="launcher check: init the process group (gloo without CUDA), print rank/world, exit")
    ap.add_argument("--verbose", action="store_true")
    return ap.parse_args()


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` (N > 1) started as a plain process: re-exec the same command line under
    torch.distributed.run with N ranks on this node (rendezvous on 127.0.0.1); rank 0's JSON line is
    the only stdout line the ranks print."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_check(args):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    if world > 1:
        dist.init_process_group(backend)
        t = torch.tensor([rank + 1], dtype=torch.int64)
        if backend == "nccl":
            torch.cuda.set_device(local)
            t = t.cuda()
        dist.all_reduce(t)
        total = int(t.item())
        dist.destroy_process_group()
    else:
        total = 1
    if rank == 0:
        print(json.dumps({"dist_check": True, "world": world, "gpus_arg": args.gpus, "rank_sum": total,
                          "backend": backend}), flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------- CPU oracle
def oracle_sample(config: str, n_full: int, m_full: int, runs: int = 1):
    """Time O-MIX (oracle/, as it stands, all host threads) on the config's
    recipe at the largest sample size whose `runs` repetitions fit the host
    budget (sample_n_for) and scale by the flop ratio to the full size."""
    import oracle
    import testmat
    import numpy as np
    cores = len(os.sched_getaffinity(0))
    n_s = min(sample_n_for(runs, cores), n_full)
    a = testmat.config_matrix(config, n_s)
    t0 = time.perf_counter()
    _, s, _, st, rc = oracle.mixed_svd(a, nthreads=cores)
    dt = time.perf_counter() - t0
    m_s = a.shape[0]
    # O-MIX cost ~ (2 m n^2 [tall QR] + c n^3): scale both terms by the size ratio
    scale = (n_full / n_s) ** 3 if m_full == n_full else (m_full * n_full ** 2) / (m_s * n_s ** 2)
    return {
        "value": dt * scale, "unit": "s", "cores": cores, "kind": "oracle", "cpu": cpu_model(),
        "sample": (f"O-MIX mixed_svd on the {config} recipe at {m_s}x{n_s} (same seeds), {dt:.2f} s "
                   f"measured, scaled x{scale:.0f} by the n^3 flop ratio to {m_full}x{n_full}; "
                   f"sweeps32={st['sweeps32']} sweeps64={st['sweeps64']}"),
        "sample_seconds": dt,
    }


def run_reference(args):
    """--impl reference: the oracle (the only reference in this tier) timed on
    the host cores; each step a bounded sample (see oracle_sample)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import testmat
    if args.full:
        import oracle
        m_f, n_f, _ = testmat.CONFIGS[args.full]
        a = testmat.cached_config(args.full)
        cores = len(os.sched_getaffinity(0))
        t0 = time.perf_counter()
        _, s, _, st, rc = oracle.mixed_svd(a, nthreads=cores)
        dt = time.perf_counter() - t0
        ex = oracle_sample(args.full, n_f, m_f)
        print(json.dumps({"config": args.full, "m": m_f, "n": n_f, "seconds": dt, "cores": cores, "cpu": cpu_model(),
                          "rc": rc, "sweeps32": st["sweeps32"], "sweeps64": st["sweeps64"],
                          "digest": testmat.digest(a), "extrapolated_seconds": ex["value"],
                          "extrapolation_sample": ex["sample"], "measured_over_extrapolated": dt / ex["value"],
                          "what": "O-MIX (oracle/, as it stands) on the full config, all host cores"}), flush=True)
        return
    m_full, n_full, _ = testmat.CONFIGS[args.config]
    vals = []
    last = None
    for i in range(args.warmup + args.steps):
        cb = oracle_sample(args.config, n_full, m_full, runs=args.warmup + args.steps)
        if i >= args.warmup:
            vals.append(cb["value"])
            last = cb
    v = statistics.median(vals)
    cb = dict(last)
    cb["value"] = v
    cb.pop("sample_seconds", None)
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
        "config": {"workload": args.config, "m": m_full, "n": n_full},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            return None
        rows = [[c.strip() for c in l.split(",")] for l in out.strip().splitlines() if l.strip()]
        rows = [r for r in rows if len(r) == len(self.FIELDS)]
        if not rows:
            return None
        sm = []
        for r in rows:
            try:
                sm.append(float(r[0]))
            except ValueError:
                pass
        load = [x for x in sm if x > 500] or sm
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[3:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        try:
            mx = float(rows[0][1])
        except ValueError:
            mx = None
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(rows)}


# ----------------------------------------------------------------- peaks
def load_peaks():
    peaks = {}
    try:
        peaks["measured"] = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        peaks["measured"] = None
    try:
        peaks["micro"] = json.load(open(os.path.join(ROOT, "profiles", "peaks.json")))
    except Exception:
        peaks["micro"] = None
    return peaks


def roofline_for(kernel: str, ms_total: float, launches: int, work: dict, peaks: dict, n: int, b: int):
    """Roofline entry of one kernel from its algorithmic work (DESIGN.md sec. 8
    "Algorithmic work per unit"), its summed CUDA-event time over the timed
    steps and the measured peaks (MEASURED_PEAKS.json copy bandwidth;
    profiles/peaks.json DFMA/DMMA/FFMA microbenchmarks)."""
    hbm = (peaks["measured"] or {}).get("hbm_gbs") or 6650.0
    hbm_src = "MEASURED_PEAKS.json hbm_gbs (copy)" if (peaks["measured"] or {}).get("hbm_gbs") else "fallback 6.65 TB/s"
    micro = peaks["micro"] or {}
    sec = ms_total / 1e3
    flops = work["flops"].get(kernel)
    byts = work["bytes"].get(kernel)
    base = {"kernel": kernel, "launches": launches, "avg_launch_us": ms_total * 1e3 / max(launches, 1),
            "traffic": work.get("traffic", {}).get(kernel)}
    if byts is not None:
        base["algorithmic_bytes_per_launch"] = byts / max(launches, 1)
        base["hbm_gbs_achieved"] = byts / sec / 1e9
        base["hbm_frac"] = byts / sec / 1e9 / hbm
    if flops is not None:
        base["algorithmic_flops_per_launch"] = flops / max(launches, 1)
    bound = work["bound"].get(kernel)
    if bound == "hbm" and byts is not None:
        ach = byts / sec / 1e9
        base.update({"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                     "peak_source": hbm_src})
    elif bound == "alu64" and flops is not None:
        ach = flops / sec / 1e12
        peak = micro.get("dmma_tflops") or micro.get("dfma_tflops") or (148 * 64 * 2 * 1.965e9 / 1e12)
        # FP64 DMMA (mma.sync m8n8k4 f64) is the tensor pipe's fp64 path on sm_100a (no tcgen05 f64 kind)
        base.update({"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                     "peak_source": "measured DMMA (mma.sync f64) microbenchmark, profiles/peaks.json "
                                    "(MEASURED_PEAKS.json has no fp64 figure)"})
    elif bound == "alu32" and flops is not None:
        ach = flops / sec / 1e12
        peak = micro.get("ffma_tflops") or (148 * 128 * 2 * 1.965e9 / 1e12)
        base.update({"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                     "peak_source": "measured FFMA microbenchmark, profiles/peaks.json"})
    else:
        base.update({"bound": "latency", "achieved": None, "peak": None, "unit": None, "frac": None})
    return base


def algorithmic_work(stats_list, n: int, b: int, world: int = 1, m: int | None = None, tensor32: bool = True,
                     v32: bool = False):
    """Algorithmic flops / HBM bytes of the path's kernels summed over the
    given steps, per rank.  Gram of a pair (w = 2b columns,
    n rows): symmetric half incl. the diagonal, n w (w+1) flops, reading W
    once (per round the whole X: n^2 s bytes); update: 2 n w^2 flops and the
    read + write of n x w (s bytes) for X, and again for V when the stage
    accumulates V (fp64 refinement: the sweeps counted in v_sweeps64, all of
    them by default; fp32 stage: only on the V-route, v32); QRP: the lazy GEMV
    reads the (n-k)^2 trailing matrix at every step k (8 n^3 / 3 bytes)."""
    flops, byts, bound = {}, {}, {}
    nblk = -(-n // b)
    M = nblk + (nblk & 1) if world == 1 else -(-nblk // (2 * world)) * (2 * world)
    npairs = M // 2
    rounds = M - 1
    w = 2 * b
    for st in stats_list:
        for tag, s, key in (("f32", 4, "32"), ("f64", 8, "64")):
            sweeps = st["sweeps" + key]
            upd = sum(st["upd_trace" + key])
            # pairs skipped as unchanged (exact skip) compute no Gram
            evaluated = sweeps * rounds * npairs - sum(st.get("skip_trace" + key, []))
            g, u = f"pair_gram_{tag}", f"pair_update_{tag}"
            flops[g] = flops.get(g, 0.0) + evaluated * float(n) * w * (w + 1)
            byts[g] = byts.get(g, 0.0) + evaluated * float(n) * w * s
            # updated pairs whose V slabs are rotated too
            if tag == "f32":
                upd_v = upd if v32 else 0
            else:
                # the LAST v_sweeps64 sweeps accumulate V (sec. 3.4 V formation: the accumulating stage follows
                # the refinement without V)
                vsw = st.get("v_sweeps64", sweeps)
                upd_v = sum(st["upd_trace64"][sweeps - vsw:sweeps]) if vsw < sweeps else upd
            flops[u] = flops.get(u, 0.0) + (upd + upd_v) * 2.0 * n * w * w
            byts[u] = byts.get(u, 0.0) + (upd + upd_v) * 2 * float(n) * w * s
        flops["qrp_coop"] = flops.get("qrp_coop", 0.0) + 4.0 * n ** 3 / 3
        byts["qrp_coop"] = byts.get("qrp_coop", 0.0) + 8.0 * n ** 3 / 3
    # fp32 Gram/update are HBM-bound on the tensor cores (tcgen05) and ALU-bound on FFMA
    for k in ("pair_gram_f32", "pair_update_f32"):
        bound[k] = "hbm" if tensor32 else "alu32"
    bound["pair_gram_f64"] = "alu64"
    bound["pair_update_f64"] = "alu64"
    bound["qrp_coop"] = "hbm"
    return {"flops": {k: v / world for k, v in flops.items() if not k.startswith("qrp") or world == 1},
            "bytes": {k: v / world for k, v in byts.items() if not k.startswith("qrp") or world == 1},
            "bound": bound}


def time_config(mp, h, cfg, steps, warmup, root, device, stream, l2_flush, barrier, max_over_ranks):
    """Seconds per SVD of another config with the same handle and timing rules (device-resident input,
    L2 flushed between steps, CUDA events on the handle's stream, max over ranks)."""
    import numpy as np
    import torch
    import testmat
    m, n, _ = testmat.CONFIGS[cfg]
    A = U = S = V = None
    if root:
        a = testmat.cached_config(cfg)
        A = torch.from_numpy(np.ascontiguousarray(a.T)).t().to(device)
        U = mp.empty_col_major(m, n, torch.float64, device)
        V = mp.empty_col_major(n, n, torch.float64, device)
        S = torch.empty(n, dtype=torch.float64, device=device)
    st = None
    for _ in range(warmup):
        rc, st = mp.mpjsvd_factor(h, A, U, S, V, m, n, m, m, n)
    torch.cuda.synchronize()
    barrier()
    ms = []
    for _ in range(steps):
        l2_flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rc, st = mp.mpjsvd_factor(h, A, U, S, V, m, n, m, m, n)
        e1.record(stream)
        torch.cuda.synchronize()
        if rc < 0:
            raise mp.MpjsvdError(rc, f"mpjsvd_factor ({cfg})")
        ms.append(e0.elapsed_time(e1))
    v = max_over_ranks(statistics.mean(ms)) / 1e3
    d = st.as_dict()
    return {"value": v, "unit": "s", "steps": steps, "m": m, "n": n, "sweeps32": d["sweeps32"],
            "sweeps64": d["sweeps64"], "stage_ms": d["stage_ms"]}


def load_full_oracle_measurements():
    """Full-size O-MIX runs measured on a GPU box's host (bench.py --impl reference --full CFG), kept in
    profiles/cpu_oracle_full_*.json: the scale check of the bounded sample's n^3 extrapolation."""
    import glob
    out = []
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "cpu_oracle_full_*.json"))):
        try:
            d = json.load(open(p))
            out.append({k: d.get(k) for k in ("config", "seconds", "cores", "cpu", "sweeps32", "sweeps64",
                                              "extrapolated_seconds", "measured_over_extrapolated")})
        except Exception:
            pass
    return out


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    rank0, world0, _ = dist_env()
    if world0 != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world0}: launch one rank per GPU")
    if args.dist_check:
        dist_check(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2209_04626_b200 as mp
    import testmat

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    root = rank == 0

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    m, n, _ = testmat.CONFIGS[args.config]
    device = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    # experiment hook: MPJSVD_BENCH_OPTS="pdl_overlap=0,max_inner32=1" (Handle option overrides)
    extra = {}
    for kv in filter(None, os.environ.get("MPJSVD_BENCH_OPTS", "").split(",")):
        k, v = kv.split("=")
        extra[k.strip()] = float(v) if "." in v else int(v)
    h = mp.Handle(stream=stream.cuda_stream, block_cols=args.block_cols, **extra)
    if world > 1:
        h.comm_init_torch()          # NCCL communicator inside libmpjsvd.so (rank 0's id via torch.distributed)
    a = A = U = V = S = None
    if root:
        a = testmat.cached_config(args.config)
        A = torch.from_numpy(np.ascontiguousarray(a.T)).t().to(device)   # column-major, resident in HBM
        U = mp.empty_col_major(m, n, torch.float64, device)
        V = mp.empty_col_major(n, n, torch.float64, device)
        S = torch.empty(n, dtype=torch.float64, device=device)
    l2_flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=device)

    def step():
        rc, st = mp.mpjsvd_factor(h, A, U, S, V, m, n, m, m, n)
        if rc < 0:
            raise mp.MpjsvdError(rc, "mpjsvd_factor")
        return st.as_dict()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---------------- timed region: K steps, L2 flushed between steps, no per-kernel instrumentation
    stats = []
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        l2_flush.zero_()
        evs[i][0].record(stream)
        stats.append(step())
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / args.steps
    ms = max_over_ranks(ms)
    launches = int(sum(s["kernel_launches"] for s in stats))

    # ---------------- profiled pass (separate): per-kernel CUDA events on the launching stream; it feeds
    # the kernel shares and the roofline (an event pair per launch costs ~1.5 % of the step)
    prof, prof_ms, prof_steps = {}, None, 0
    if not args.no_profile:
        prof_steps = max(1, min(args.steps, 5))
        h.set_profiling(True)
        pe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(prof_steps)]
        pstats = []
        for i in range(prof_steps):
            l2_flush.zero_()
            pe[i][0].record(stream)
            pstats.append(step())
            pe[i][1].record(stream)
        torch.cuda.synchronize()
        prof = h.profile()
        h.set_profiling(False)
        prof_ms = max_over_ranks(sum(e0.elapsed_time(e1) for e0, e1 in pe) / prof_steps)

    # ---------------- result check (plumbing: torch on the device)
    orth_u = orth_v = res = None
    if root:
        eye = torch.eye(n, dtype=torch.float64, device=device)
        orth_u = float((U.T @ U - eye).abs().max())
        orth_v = float((V.T @ V - eye).abs().max())
        res = float(torch.linalg.norm(A - (U * S) @ V.T) / torch.linalg.norm(A))
        del eye

    # ---------------- e2e: host buffers through the same C-ABI call
    e2e = None
    if not args.no_e2e:
        Ah = Uh = Vh = Sh = None
        if root:
            Ah = torch.from_numpy(np.ascontiguousarray(a.T)).t().pin_memory()
            Uh = torch.empty((n, m), dtype=torch.float64).pin_memory().t()
            Vh = torch.empty((n, n), dtype=torch.float64).pin_memory().t()
            Sh = torch.empty(n, dtype=torch.float64).pin_memory()
        e2e_ms = []
        for i in range(max(1, args.steps)):
            l2_flush.zero_()
            torch.cuda.synchronize()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rc, _ = mp.mpjsvd_factor(h, Ah, Uh, Sh, Vh, m, n, m, m, n)
            e1.record(stream)
            torch.cuda.synchronize()
            if rc < 0:
                raise mp.MpjsvdError(rc, "mpjsvd_factor (host buffers)")
            e2e_ms.append(e0.elapsed_time(e1))
        e2e_v = max_over_ranks(statistics.mean(e2e_ms)) / 1e3
        e2e = {"value": e2e_v, "unit": "s", "h2d_bytes_per_step": int(m * n * 8),
               "d2h_bytes_per_step": int((m * n + n + n * n) * 8)}

    # ---------------- roofline of the dominant kernel
    peaks = load_peaks()
    v32 = int(h.options.switch_u) == 0
    work = algorithmic_work(pstats if prof else stats, n, args.block_cols, world, m, tensor32=True, v32=v32)
    try:
        # per (config, kernel): dram__bytes_read.sum + dram__bytes_write.sum per launch of the current code's
        # ncu --set full capture of this config (tools/ncu_summary.py traffic)
        work["traffic"] = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(args.config, {})
    except Exception:
        work["traffic"] = {}
    # the dominant single kernel (the overlapped solve+update brackets time two kernels together)
    single = {k: v for k, v in prof.items() if "solve_update" not in k}
    dominant = max(single.items(), key=lambda kv: kv[1][0]) if single else None
    roof = roofline_for(dominant[0], dominant[1][0], dominant[1][1], work, peaks, n, args.block_cols) \
        if dominant else None
    kernels = {k: {"ms_per_step": v[0] / prof_steps, "launches_per_step": v[1] / prof_steps,
                   "share": v[0] / max(1e-9, sum(x[0] for x in prof.values()))} for k, v in prof.items()}
    jacobi = {}
    # the overlapped brackets: the update's algorithmic bytes / flops over the bracket time (lower bound)
    for tag, kind in (("f32", "pair_update_f32"), ("f64", "pair_update_f64")):
        key = f"pair_solve_update_{tag}"
        if key in prof:
            work["flops"][key] = work["flops"].get(kind, 0.0)
            work["bytes"][key] = work["bytes"].get(kind, 0.0)
            work["bound"][key] = work["bound"].get(kind)
    for k in ("pair_gram_f64", "pair_update_f64", "pair_gram_f32", "pair_update_f32", "qrp_coop",
              "pair_solve_update_f32", "pair_solve_update_f64"):
        if k in prof:
            r = roofline_for(k, prof[k][0], prof[k][1], work, peaks, n, args.block_cols)
            jacobi[k] = {kk: r.get(kk) for kk in ("bound", "achieved", "peak", "unit", "frac", "hbm_gbs_achieved",
                                                  "hbm_frac", "avg_launch_us")}

    # ---------------- the metric's other size (n = 4096 next to 8192), same run, same timing rules
    also = {}
    for cfg in filter(None, (c.strip() for c in args.also.split(","))):
        if cfg == args.config:
            continue
        also[cfg] = time_config(mp, h, cfg, max(1, min(args.steps, 5)), max(3, min(args.warmup, 3)), root, device,
                                stream, l2_flush, barrier, max_over_ranks)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = oracle_sample(args.config, n, m)
        cpu.pop("sample_seconds", None)
        full = load_full_oracle_measurements()
        if full:
            cpu["full_size_measurements"] = full
    st0 = stats[-1]
    out = {
        "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f64+tf32x3",   # fp64 path; the fp32 seed stage's products on TF32 tensor cores, hi/lo split
        "data": "synthetic",
        "config": {"workload": args.config, "m": m, "n": n, "block_cols": args.block_cols,
                   "parallelism": f"column-block sharded x{world} (NCCL block exchange)" if world > 1
                   else "single-gpu",
                   "l2": "inputs (A 8n^2 B) and working set > L2; 512 MiB L2 flush between timed steps",
                   "recipe": testmat.CONFIGS[args.config][2]},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
        "sweeps32": st0["sweeps32"], "sweeps64": st0["sweeps64"],
        "upd_trace32": st0["upd_trace32"], "upd_trace64": st0["upd_trace64"],
        "inner_max_trace32": st0["inner_max_trace32"], "inner_max_trace64": st0["inner_max_trace64"],
        "inner_sum_trace32": st0["inner_sum_trace32"], "inner_sum_trace64": st0["inner_sum_trace64"],
        "skip_trace32": st0["skip_trace32"], "skip_trace64": st0["skip_trace64"],
        "stage_ms": st0["stage_ms"],
        "check": {"orth_u": orth_u, "orth_v": orth_v, "residual": res},
        "kernels": kernels, "jacobi_roofline": jacobi,
        "profiled": {"steps": prof_steps, "ms_per_step": prof_ms,
                     "note": "kernels / roofline / jacobi_roofline come from this separate pass with per-launch "
                             "CUDA events; value is timed without them"},
        "also": also,
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
