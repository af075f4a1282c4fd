"""Timing of the sphere RHS (mg_set_rhs_from_spheres) on the bench's
workloads: the time-step regime (512^3, 7,417 spheres R = 6, s_f = 2) and
config 5 (2048 x 512 x 512, 50,000 spheres R = 4, s_f = 1).

    python scripts/sphere_probe.py [reps]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1410_6609_b200 import _build
    _build.build()
    from paper_1410_6609_b200 import mg
    from paper_1410_6609_b200 import workloads as W
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    st = torch.cuda.Stream()
    for name, w, sub in (("timestep 512^3 s_f=2", W.timestep_workload(512), 2),
                         ("cfg5 full s_f=1", W.cfg5(scale=1), 1)):
        s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8, stream=st)
        if w.solid is not None:
            s.set_mask(w.solid)
        ts = []
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            s.set_rhs_from_spheres(w.centers, w.radii, w.charges, subsample=sub)
            b.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print("%s: %d spheres, set_rhs_from_spheres %.3f ms (median of %d)"
              % (name, len(w.radii), float(np.median(ts)), reps), flush=True)
        s.close()


if __name__ == "__main__":
    main()
