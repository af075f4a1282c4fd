"""A few config-5 V(3,3)-cycles (full size unless a scale is given), for
profiling: python scripts/cfg5_probe.py [scale] [cycles]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402
from paper_1410_6609_b200 import workloads as W  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = W.cfg5(scale=scale)
s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=w.min_coarse,
                 nu1=3, nu2=3)
s.set_mask(w.solid)
s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
for _ in range(cycles):
    print(s.vcycle())
