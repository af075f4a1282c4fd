"""Per-phase times of config-3 V-cycles (CUDA events between the level-0
phases, profiling mode): python scripts/cycle_times.py [n] [cycles] [fused]
(fused = 1: mg_opts.fused_norm, reading c11)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402
from paper_1410_6609_b200 import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 8
fused = len(sys.argv) > 3 and sys.argv[3] == "1"
w = W.cfg3(n, seed=0, with_rhs=False)
s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8, fused_norm=fused)
s.set_rhs(W.uniform_rhs(w.shape, 0))
for _ in range(3):
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
