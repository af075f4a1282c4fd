"""Coarse-end probes: the coarsest-grid CG alone on the coarsest grids of
config 3 (8^3), config 5 (32 x 8 x 8) and config 4 at P = 8 (64 x 8 x 8),
and V-cycles of config 3 at n^3 with and without the persistent tail kernel
(CUDA events around the whole cycle and the profiling categories).

    python scripts/cg_probe.py [n] [reps]

Run under ncu with -k regex:"cg|tail" for per-kernel captures.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1410_6609_b200 import _build
    _build.build()
    from paper_1410_6609_b200 import mg
    from paper_1410_6609_b200 import workloads as W
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    D, N = mg.MG_DIRICHLET, mg.MG_NEUMANN
    st = torch.cuda.Stream()
    for name, shape, bt, bv in [("cfg3 coarsest 8^3", (8, 8, 8), [D] * 6, [0.0] * 6),
                                ("cfg5 coarsest 32x8x8", (32, 8, 8),
                                 [N, N, D, D, N, N], [0, 0, 0, 1, 0, 0]),
                                ("cfg4 P=8 coarsest 64x8x8", (64, 8, 8),
                                 [N, N, D, D, N, N], [0, 0, 0, 1, 0, 0])]:
        for off in (0, mg.MG_OFF_CG_CLUSTER):
            s = mg.Multigrid(shape, 1.0, bt, bv, max_levels=1, stream=st, disable=off)
            f = np.random.default_rng(0).uniform(-1, 1, shape)
            s.set_field(0, mg.MG_FIELD_RHS, f)
            ts = []
            for _ in range(reps):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(st)
                it = s.coarse_solve()
                b.record(st)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            print("%-26s %-13s its %4d  %.1f us (events, median)"
                  % (name, "cluster" if s.cycle_paths & mg.MG_PATH_CG_CLUSTER else "single CTA",
                     it, 1e3 * float(np.median(ts))), flush=True)
            s.close()
    w = W.cfg3(n, seed=0, with_rhs=False)
    f = W.uniform_rhs(w.shape, 0)
    for off in (0, mg.MG_OFF_TAIL):
        s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8, stream=st,
                         disable=off)
        s.set_rhs(f)
        for _ in range(3):
            s.vcycle()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            s.vcycle()
        b.record(st)
        torch.cuda.synchronize()
        s.set_profiling(True)
        prof = []
        for _ in range(reps):
            s.vcycle()
            prof.append(s.last_cycle_times())
        s.set_profiling(False)
        med = {k: float(np.median([p[k] for p in prof])) for k in prof[0]}
        print("cfg3 %d^3 %-8s cycle %.4f ms  coarse %.4f  whole %.4f  launches %d"
              % (n, "tail" if not off else "per-step", a.elapsed_time(b) / reps,
                 med["coarse_ms"], med["whole_levels_ms"], s.cycle_launches), flush=True)
        s.close()


if __name__ == "__main__":
    main()
