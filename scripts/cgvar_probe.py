"""Time the masked (variable-coefficient) coarsest CG on config 5's coarsest
grid (32 x 8 x 8 with the beam): python scripts/cgvar_probe.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402
from paper_1410_6609_b200 import workloads as W  # noqa: E402

w = W.cfg5(scale=16, n_spheres=40)   # 128 x 32 x 32 -> coarsest 32 x 8 x 8
s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=w.min_coarse,
                 nu1=3, nu2=3)
s.set_mask(w.solid)
s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
for _ in range(2):
    s.vcycle()
L = s.nlevels - 1
it = s.coarse_solve()
t0 = time.perf_counter()
for _ in range(20):
    it = s.coarse_solve()
dt = (time.perf_counter() - t0) / 20
print("masked coarsest %s: iterations %d, %.1f us per solve (host-timed)"
      % (s.level_dims(L) if hasattr(s, "level_dims") else L, it, dt * 1e6))
s.close()
