"""Time the coarsest-grid CG alone on the coarsest grids of config 3 (8^3)
and of config 4 at P = 8 (64 x 8 x 8, channel BCs):
python scripts/cg_probe.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402

D, N = mg.MG_DIRICHLET, mg.MG_NEUMANN
for name, shape, bt, bv in [("cfg3 coarsest 8^3", (8, 8, 8), [D] * 6, [0.0] * 6),
                            ("cfg4 P=8 coarsest 64x8x8", (64, 8, 8),
                             [N, N, D, D, N, N], [0, 0, 0, 1, 0, 0]),
                            ("cfg5 coarsest 32x8x8", (32, 8, 8),
                             [N, N, D, D, N, N], [0, 0, 0, 1, 0, 0])]:
    s = mg.Multigrid(shape, 1.0 / 8, bt, bv, max_levels=1)
    f = np.random.default_rng(0).uniform(-1, 1, shape)
    s.set_field(0, mg.MG_FIELD_RHS, f)
    it = s.coarse_solve()
    t0 = time.perf_counter()
    for _ in range(20):
        it = s.coarse_solve()
    dt = (time.perf_counter() - t0) / 20
    print("%-28s iterations %4d  %.1f us per solve (host-timed, incl. sync)"
          % (name, it, dt * 1e6))
    s.close()
