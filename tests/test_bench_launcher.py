"""bench.py's multi-GPU launch contract on CPU: `bench.py --gpus N` run as a plain process re-executes
itself under torch.distributed.run with N ranks (gloo here, NCCL on GPUs) and rank 0 prints one JSON line;
under a launcher, --gpus must equal WORLD_SIZE."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          timeout=300, env=e, cwd=ROOT)


def test_bench_relaunches_n_ranks():
    p = _run(["--gpus", "2", "--dist-check"])
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["world"] == 2 and d["rank_sum"] == 3 and d["gpus_arg"] == 2


def test_bench_rejects_world_mismatch():
    p = _run(["--gpus", "2", "--dist-check"], env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode != 0
    assert "WORLD_SIZE" in (p.stderr + p.stdout)
