"""Write oracle-only golden results for the full-size configs.

Usage:  python tests/golden/make_golden.py C3 [C4 C5 ...] [--threads N]

Calls ONLY oracle/ (O-MIX) on testmat.config_matrix(name) and stores, per
config, the input digest, the sweep counts / traces and sigma in
tests/golden/omix_<name>.json.  The GPU parity tests compare sweep counts
(+-1, BASELINE.json) and sigma against these files; sigma is compared
element by element only when the box regenerates a bit-identical input
(same digest), otherwise through the tiered tolerance.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import testmat  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=0)
    args = ap.parse_args()
    for name in args.configs:
        a = testmat.config_matrix(name)
        t0 = time.time()
        u, s, v, st, rc = oracle.mixed_svd(a, nthreads=args.threads)
        dt = time.time() - t0
        n = a.shape[1]
        out = {
            "config": name, "shape": list(a.shape), "digest": testmat.digest(a), "rc": rc,
            "oracle_seconds": dt, "threads": args.threads, "stats": st,
            "sigma": [float(x) for x in s],
            "orth_u": float(np.abs(u.T @ u - np.eye(n)).max()),
            "orth_v": float(np.abs(v.T @ v - np.eye(n)).max()),
            "residual": float(np.linalg.norm(a - (u * s) @ v.T) / np.linalg.norm(a)),
            "written_by": "tests/golden/make_golden.py (oracle O-MIX only)",
        }
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"omix_{name}.json")
        with open(path, "w") as f:
            json.dump(out, f)
        print(name, "rc", rc, "sweeps", st["sweeps32"], st["sweeps64"], "t", round(dt, 1),
              "orth", out["orth_u"], out["orth_v"], "res", out["residual"], flush=True)


if __name__ == "__main__":
    main()
