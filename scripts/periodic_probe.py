"""V(2,2)-cycles of the 512^3 periodic channel (x, z periodic, y Dirichlet
0/1): per-phase CUDA-event times (profiling mode) after two warm-up cycles.
python scripts/periodic_probe.py [n] [cycles]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 2
P, D = mg.MG_PERIODIC, mg.MG_DIRICHLET
s = mg.Multigrid((n, n, n), 1.0, [P, P, D, D, P, P], [0, 0, 0, 1, 0, 0], min_coarse=8)
s.set_rhs(np.random.default_rng(0).uniform(-1, 1, (n, n, n)))
for _ in range(2):
    s.vcycle()
s.set_profiling(True)
ts = []
for _ in range(cycles):
    s.vcycle()
    ts.append(s.last_cycle_times())
s.set_profiling(False)
keys = ["smooth0_ms", "restrict0_ms", "prolong0_ms", "norm_ms", "coarse_ms", "cycle_ms"]
print(" ".join("%s=%.4f" % (k, np.median([t[k] for t in ts])) for k in keys),
      "smooth0_launches=%d" % ts[0]["smooth0_launches"])
s.close()
