"""Per-cycle device time over a config-3 solve from Phi = 0 (CUDA events
around each mg_vcycle), to see whether the cycle time depends on the
iterate (e.g. once the residual has reached the rounding floor):
python scripts/cycle_timeline.py [cycles] [n]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1410_6609_b200 import mg
    from paper_1410_6609_b200 import workloads as W
    cycles = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    w = W.cfg3(n, seed=0, with_rhs=False)
    st = torch.cuda.Stream()
    s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8, stream=st)
    s.set_rhs(W.uniform_rhs(w.shape, 0))
    s.vcycle()
    s.zero_solution()
    r0 = s.residual_norm()
    reset = int(os.environ.get("RESET_EVERY", "0"))
    for k in range(cycles):
        if reset and k and k % reset == 0:
            s.zero_solution()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        r = s.vcycle()
        b.record(st)
        torch.cuda.synchronize()
        print("cycle %2d  %.4f ms  r/r0 %.2e" % (k + 1, a.elapsed_time(b), r / r0), flush=True)
    s.close()


if __name__ == "__main__":
    main()
