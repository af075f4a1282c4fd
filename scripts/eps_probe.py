"""Cycle-phase times of the variable-permittivity variant (N4: 78.5:1 random
jumps, channel BCs, V(2,2)) at n^3: python scripts/eps_probe.py [n] [cycles]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 4
shape = (n, n, n)
D, N = mg.MG_DIRICHLET, mg.MG_NEUMANN
s = mg.Multigrid(shape, 1.0, [N, N, D, D, N, N], [0, 0, 0, 1, 0, 0], min_coarse=8)
rng = np.random.default_rng(1)
s.set_permittivity(np.where(rng.uniform(size=shape) < 0.3, 78.5, 1.0))
s.set_rhs(np.random.default_rng(0).uniform(-1, 1, shape))
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
