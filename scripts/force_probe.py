"""Time mg_coulomb_forces on the time-stepping regime's workload (config-4
box 512^3, 7,417 spheres R=6, s_F=2): python scripts/force_probe.py [reps]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402
from paper_1410_6609_b200 import workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
w = W.cfg4(P=1, n=512, seed=0)
s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8, nu1=3, nu2=3)
s.set_rhs_from_spheres(w.centers, w.radii, w.charges, subsample=2)
for _ in range(3):
    s.vcycle()
F = s.coulomb_forces(w.centers, w.radii, w.charges, subsample=2)
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    F2 = s.coulomb_forces(w.centers, w.radii, w.charges, subsample=2)
    ts.append(time.perf_counter() - t0)
assert np.array_equal(F, F2)
print("forces: median %.3f ms over %d (|F| max %.3e)" % (1e3 * np.median(ts), reps,
                                                          np.abs(F).max()))
np.save(os.environ.get("FORCE_OUT", "/tmp/forces.npy"), F)
s.close()
