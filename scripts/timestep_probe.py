"""Run a few time steps of the paper's regime (bench.py timestep_regime
workload) for profiling: python scripts/timestep_probe.py [steps]."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402
from paper_1410_6609_b200 import workloads as W  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = W.timestep_workload(n=512, seed=0)
s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8, nu1=3, nu2=3)
L = np.array(w.shape) * w.h
c = w.centers
for k in range(steps):
    if k:
        c = W.move_spheres(c, w.radii, L, k, seed=0, amplitude=0.005)
    F, n, r = s.timestep(c, w.radii, w.charges, cycles=1, subsample=2)
    print("step", k, "cycles", n, "res", r, "F0", F[0])
