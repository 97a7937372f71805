"""Print the content digests of the full-size config inputs on this host
(checks that testmat regenerates bit-identical inputs on another machine)."""
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import threadpoolctl  # noqa: E402
import testmat  # noqa: E402

out = {"cpu": platform.processor(), "nproc": os.cpu_count(),
       "blas": [(d.get("architecture"), d.get("num_threads")) for d in threadpoolctl.threadpool_info()]}
try:
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            out["cpu"] = line.split(":", 1)[1].strip()
            break
except OSError:
    pass
for name in sys.argv[1:] or ["C3", "C4", "C5"]:
    t = time.time()
    a = testmat.config_matrix(name)
    out[name] = {"digest": testmat.digest(a), "gen_s": round(time.time() - t, 1)}
print(json.dumps(out))
