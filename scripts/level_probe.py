"""Cycle time of the config-3 recipe at n^3 for n = 64 .. 512 under a few
coarse-end settings (default tail, tail from 64^3, no tail): the differences
between sizes give the cost of the levels below each size inside a cycle.
python scripts/level_probe.py [cycles]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402
from paper_1410_6609_b200 import workloads as W  # noqa: E402

cycles = int(sys.argv[1]) if len(sys.argv) > 1 else 40
variants = {"default": {}, "tail64": {"tail_cells": 64 ** 3},
            "notail": {"disable": mg.MG_OFF_TAIL}}
for n in (32, 64, 128, 256, 512):
    w = W.cfg3(n, seed=0, with_rhs=False)
    for name, kw in variants.items():
        st = torch.cuda.Stream()
        s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8,
                         stream=st, **kw)
        s.set_rhs(W.uniform_rhs(w.shape, 0))
        for _ in range(5):
            s.vcycle()
        ts = []
        for _ in range(cycles):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            s.vcycle()
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        s.set_profiling(True)
        s.vcycle()
        t = s.last_cycle_times()
        s.set_profiling(False)
        print("n=%4d %-8s cycle %.4f ms (min %.4f) launches %d coarse_ms %.4f paths %#x"
              % (n, name, np.median(ts), np.min(ts), s.cycle_launches,
                 t["coarse_ms"], s.cycle_paths), flush=True)
        s.close()
