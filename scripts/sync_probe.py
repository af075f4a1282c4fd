"""Back-to-back V-cycles with and without a host synchronisation between
them (mg_vcycle vs the cycles of mg_solve_async), same context and RHS:
python scripts/sync_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402
from paper_1410_6609_b200 import workloads as W  # noqa: E402

w = W.cfg3(512, seed=0, with_rhs=False)
stream = torch.cuda.Stream()
s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8, stream=stream)
fd = torch.from_numpy(W.uniform_rhs(w.shape, 0)).cuda()
od = torch.empty_like(fd)
s.set_rhs(fd)
for _ in range(3):
    s.vcycle()


def timed(fn):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for rep in range(3):
    t_sync = timed(lambda: [s.vcycle() for _ in range(20)]) / 20
    t0 = timed(lambda: (s.solve_async(fd, od, 0), s.wait()))
    t20 = timed(lambda: (s.solve_async(fd, od, 20), s.wait()))
    print("synced %.4f ms/cycle   enqueued %.4f ms/cycle" % (t_sync, (t20 - t0) / 20))
s.close()
