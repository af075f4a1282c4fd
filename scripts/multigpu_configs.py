"""BASELINE configs 4 and 5 at their multi-GPU sizes through the x-slab
decomposition on ONE B200.

    python scripts/multigpu_configs.py [--P 1,2,4,8] [--configs cfg4,cfg5]
                                       [--out profiles/r02_multigpu_configs.md]

Per (config, P): the EMULATE backend (NCCL's data layout, every rank's
agglomerated copy) solves to 1e-8 and reports cycles and the residual
history; the LOOPBACK backend (one shared agglomerated copy -- what one
real rank computes) is profiled for the per-GPU cost of the agglomerated
levels + coarsest CG.  On one GPU the P slabs run one after another, so the
cycle time here is NOT a scaling measurement; the agglomerated-level figure
is the per-rank overhead a real P-GPU run would add.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def workload(W, cfg, P):
    if cfg == "cfg4":
        return W.cfg4(P=P, n=512, seed=0)
    return W.cfg5(scale=1)


def make(mg, w, P, backend, stream):
    kw = dict(min_coarse=w.min_coarse, nu1=w.nu1, nu2=w.nu2, stream=stream)
    if P > 1:
        kw.update(nranks=P, halo=backend)
    s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, **kw)
    if w.solid is not None:
        s.set_mask(w.solid)
    s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    return s


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", default="1,2,4,8")
    ap.add_argument("--configs", default="cfg4,cfg5")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_multigpu_configs.md"))
    args = ap.parse_args()
    from paper_1410_6609_b200 import _build
    _build.build()
    from paper_1410_6609_b200 import mg
    from paper_1410_6609_b200 import workloads as W
    stream = torch.cuda.Stream()
    rows = []
    for cfg in args.configs.split(","):
        for P in [int(x) for x in args.P.split(",")]:
            w = workload(W, cfg, P)
            dims, lnx, agg = mg.plan(w.shape, min_coarse=w.min_coarse, nranks=P,
                                     halo="emulate" if P > 1 else "none")
            t0 = time.time()
            s = make(mg, w, P, "emulate", stream)
            rc, cyc, hist = s.solve(w.tol, 40)
            setup_solve_s = time.time() - t0
            it = s.coarse_solve()
            s.close()
            torch.cuda.synchronize()
            # per-rank cost of the agglomerated part: LOOPBACK (one copy)
            s = make(mg, w, P, "loopback", stream)
            for _ in range(3):
                s.vcycle()
            s.set_profiling(True)
            prof = []
            for _ in range(5):
                s.vcycle()
                prof.append(s.last_cycle_times())
            s.set_profiling(False)
            s.close()
            torch.cuda.synchronize()
            med = {k: float(np.median([p[k] for p in prof])) for k in prof[0]}
            row = dict(cfg=cfg, P=P, shape=w.shape, spheres=len(w.radii),
                       levels=len(dims), agg_level=agg if P > 1 else None,
                       coarsest=dims[-1], cg_iters=it, rc=rc, cycles=cyc,
                       reduction=float(hist[-1] / hist[0]),
                       factor=float((hist[-1] / hist[0]) ** (1.0 / max(cyc, 1))),
                       cycle_ms_serial=med["cycle_ms"],
                       whole_levels_ms=med["whole_levels_ms"], cg_ms=med["cg_ms"],
                       coarse_ms=med["coarse_ms"], setup_solve_s=setup_solve_s)
            rows.append(row)
            print(json.dumps(row), flush=True)
    with open(args.out, "w") as fh:
        fh.write("# Configs 4 and 5 at P = 1, 2, 4, 8 through the x-slab decomposition "
                 "on one B200 (round 2)\n\n")
        fh.write("`python scripts/multigpu_configs.py` (EMULATE backend for the solves: "
                 "NCCL's data layout, per-rank agglomerated copies; LOOPBACK for the "
                 "per-rank cost of the agglomerated levels, one copy as one real rank "
                 "computes it). **The P slabs run serially on one GPU: `cycle ms "
                 "(serial)` is not a scaling measurement.** `whole levels ms` = levels "
                 ">= 1 held whole on every rank (the agglomerated levels) incl. the "
                 "coarsest CG, per cycle; `CG ms` the coarsest solve alone (CUDA events "
                 "in the captured graph, median of 5 cycles).\n\n")
        fh.write("| cfg | P | global cells | levels | agglomerated from | coarsest | CG its "
                 "| cycles to 1e-8 | mean factor | cycle ms (serial) | whole levels ms "
                 "| CG ms |\n|---|---|---|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            fh.write("| %s | %d | %s | %d | %s | %s | %d | %d | %.4f | %.2f | %.3f | %.3f |\n"
                     % (r["cfg"], r["P"], "x".join(map(str, r["shape"])), r["levels"],
                        "-" if r["agg_level"] is None else "level %d" % r["agg_level"],
                        "x".join(map(str, r["coarsest"])), r["cg_iters"], r["cycles"],
                        r["factor"], r["cycle_ms_serial"], r["whole_levels_ms"],
                        r["cg_ms"]))
        fh.write("\nRaw rows:\n\n```\n")
        for r in rows:
            fh.write(json.dumps(r) + "\n")
        fh.write("```\n")


if __name__ == "__main__":
    main()
