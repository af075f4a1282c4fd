"""Per-solve time of the config-3 end-to-end pipeline (mg_solve_async) with
host (pinned) or device buffers and 0 or 20 cycles per solve, to separate
copy cost, the layout conversions and the cycles:
python scripts/e2e_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402
from paper_1410_6609_b200 import workloads as W  # noqa: E402

w = W.cfg3(512, seed=0, with_rhs=False)
stream = torch.cuda.Stream()
s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8, stream=stream)
fh = torch.empty(w.shape, dtype=torch.float64, pin_memory=True)
fh.numpy()[...] = W.uniform_rhs(w.shape, 0)
fd = fh.cuda()
outs_h = [torch.empty(w.shape, dtype=torch.float64, pin_memory=True) for _ in range(2)]
outs_d = [torch.empty(w.shape, dtype=torch.float64, device="cuda") for _ in range(2)]
for name, f, outs in (("host", fh, outs_h), ("device", fd, outs_d)):
    for cycles in (0, 20):
        nsteps = 20
        s.solve_async(f, outs[0], 1)
        s.wait()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(nsteps):
            s.solve_async(f, outs[k % 2], cycles)
        s.wait()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / nsteps
        print("%-6s cycles %2d: %.2f ms per solve" % (name, cycles, ms))
# the same cycles through mg_vcycle (a host synchronisation per cycle)
s.set_rhs(fd)
for _ in range(3):
    s.vcycle()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(20):
    s.vcycle()
e1.record(stream)
torch.cuda.synchronize()
print("mg_vcycle x20: %.3f ms per cycle" % (e0.elapsed_time(e1) / 20))
s.close()
