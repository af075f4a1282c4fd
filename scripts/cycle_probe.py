"""A few config-3 V-cycles at --size for profiling (no timing):
python scripts/cycle_probe.py [n] [cycles]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402
from paper_1410_6609_b200 import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = W.cfg3(n, seed=0, with_rhs=False)
s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8)
s.set_rhs(W.uniform_rhs(w.shape, 0))
for _ in range(cycles):
    print(s.vcycle())
