"""Run the five BASELINE.json configurations on one GPU and write a report.

For each config: hierarchy, schedule, cycles (fixed count or to the
relative tolerance), per-cycle time from CUDA events around mg_vcycle, V-cycle
throughput, asymptotic residual-reduction factor; for the configs the CPU
oracle finishes in reasonable time (1, 2, reduced 3/4/5) the GPU result is
compared with the oracle (Phi rel-L2, residual history).

usage: python scripts/run_configs.py [--out gpurun_out/r01_configs.md] [--full]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_gpu(mg, w, solid=None, max_cycles=60, **kw):
    import torch
    stream = torch.cuda.Stream()
    s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, stream=stream,
                     min_coarse=w.min_coarse, nu1=w.nu1, nu2=w.nu2,
                     coarse_tol=w.coarse_tol, **kw)
    if solid is not None:
        s.set_mask(solid)
    if w.rhs is not None:
        s.set_rhs(w.rhs)
    else:
        s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    r0 = s.residual_norm()
    hist = [r0]
    times = []
    ncyc = w.cycles if w.cycles else max_cycles
    for _ in range(ncyc):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        r = s.vcycle()
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
        hist.append(r)
        if w.tol and r <= w.tol * r0:
            break
    phi = s.get_solution()
    out = dict(levels=[s.level_dims(l) for l in range(s.nlevels)],
               cycles=len(hist) - 1, hist=hist,
               ms_per_cycle=float(np.median(times[1:] if len(times) > 2 else times)),
               launches=s.cycle_launches)
    s.close()
    return out, phi


def run_oracle(w, solid=None, max_cycles=60):
    import oracle
    o = oracle.Oracle(w.shape, w.h, w.bc_type, w.bc_value, solid=solid,
                      min_coarse=w.min_coarse, nu1=w.nu1, nu2=w.nu2,
                      coarse_tol=w.coarse_tol)
    if w.rhs is not None:
        o.set_rhs(w.rhs)
    else:
        o.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    t = time.perf_counter()
    if w.cycles:
        hist = [o.residual_norm()] + [o.vcycle() for _ in range(w.cycles)]
    else:
        st, cyc, hist = o.solve(w.tol, max_cycles)
        hist = list(hist)
    dt = time.perf_counter() - t
    return hist, o.phi(), dt


def floor_cycle(hist):
    """The cycle at which the residual reaches the fp64 rounding floor
    (reading c21): the first cycle below 1e-10 r_0 whose reduction factor
    r_k / r_{k-1} exceeds 0.5 (the V-cycle's own factor is 0.04-0.2); None
    if none."""
    for k in range(1, len(hist)):
        if hist[k - 1] < 1e-10 * hist[0] and hist[k] > 0.5 * hist[k - 1]:
            return k
    return None


def factor(hist):
    h = np.asarray(hist)
    h = h[h > 1e-13 * h[0]]
    if len(h) < 4:
        return float("nan")
    return float((h[-1] / h[-4]) ** (1.0 / 3.0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_configs.md"))
    ap.add_argument("--full", action="store_true",
                    help="also run configs 3/4/5 at full size on the GPU")
    a = ap.parse_args()
    from paper_1410_6609_b200 import _build
    _build.build()
    from paper_1410_6609_b200 import mg
    from paper_1410_6609_b200 import workloads as W

    cases = [("cfg1 32^3 sine, V(2,2), 10 cycles", W.cfg1(32), None, True),
             ("cfg2 256x64x64 channel + 200 spheres, V(2,2) to 1e-8", W.cfg2(seed=0), None, True),
             ("cfg3 reduced 128^3 random, V(2,2), 20 cycles", W.cfg3(128), None, True),
             ("cfg4 reduced 128^3 channel + spheres R=6 5%, V(2,2) to 1e-8", W.cfg4(P=1, n=128), None, True)]
    w5 = W.cfg5(scale=8, n_spheres=int(round(50000 / 512)))
    cases.append(("cfg5 reduced 256x64x64 beam mask + spheres, V(3,3) to 1e-8", w5, w5.solid, True))
    if a.full:
        cases.append(("cfg3 512^3 random, V(2,2), 20 cycles (full size)", W.cfg3(512), None, True))
        cases.append(("cfg4 512^3 channel + 7417 spheres R=6, V(2,2) to 1e-8 (P=1, full size)",
                      W.cfg4(P=1, n=512), None, True))
        w5f = W.cfg5(scale=1)
        cases.append(("cfg5 2048x512x512 beam mask + 50k spheres, V(3,3) to 1e-8 (P=1, full size)",
                      w5f, w5f.solid, False))
    rows = []
    for name, w, solid, with_oracle in cases:
        res, phi = run_gpu(mg, w, solid)
        cells = int(np.prod(w.shape))
        row = dict(name=name, shape=w.shape, cycles=res["cycles"],
                   ms_per_cycle=res["ms_per_cycle"],
                   mcells_s=cells / (res["ms_per_cycle"] * 1e-3) / 1e6,
                   factor=factor(res["hist"]), final_rel=res["hist"][-1] / res["hist"][0],
                   launches=res["launches"], levels=len(res["levels"]),
                   coarsest=res["levels"][-1], floor_cycle=floor_cycle(res["hist"]))
        fc = row["floor_cycle"]
        row["floor_rel"] = res["hist"][fc] / res["hist"][0] if fc else None
        if with_oracle:
            ho, po, dt = run_oracle(w, solid)
            n = min(len(ho), len(res["hist"]))
            row["oracle_cycles"] = len(ho) - 1
            row["phi_rel_l2"] = float(np.linalg.norm(phi - po) / np.linalg.norm(po))
            row["hist_max_rel"] = float(max(abs(a - b) / b for a, b in
                                            zip(res["hist"][:n], ho[:n])))
            # the history clause |dr_k| <= 1e-8 r_k + c r_0: the smallest c
            row["hist_floor_c"] = float(max(max(abs(a - b) - 1e-8 * b, 0.0) / ho[0]
                                            for a, b in zip(res["hist"][:n], ho[:n])))
            row["oracle_s"] = dt
        rows.append(row)
        print(json.dumps(row), flush=True)
    md = ["# Config runs on one B200 (round 2)", "",
          "Per-cycle time: median of CUDA events around `mg_vcycle` (graph "
          "launch + norm readback).  Oracle columns: the CPU oracle on the same "
          "inputs (host cores of the GPU box).  `floor at` = the cycle where the "
          "residual reaches the fp64 rounding floor (first cycle with r_k > 0.5 "
          "r_{k-1} once below 1e-10 r_0, reading c21) and r_k/r_0 there; `clause c` = the smallest c with "
          "|r_k(GPU) - r_k(oracle)| <= 1e-8 r_k + c r_0 over the history (the tests "
          "use c = 1e-15).", "",
          "| config | cells | levels (coarsest) | cycles | ms/cycle | Mcells/s | "
          "factor | r_k/r_0 | floor at (r/r_0) | Phi rel-L2 vs oracle | clause c | "
          "oracle cycles |",
          "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        md.append("| %s | %d | %d %s | %d | %.3f | %.0f | %.3f | %.1e | %s | %s | %s | %s |" % (
            r["name"], int(np.prod(r["shape"])), r["levels"], tuple(r["coarsest"]),
            r["cycles"], r["ms_per_cycle"], r["mcells_s"], r["factor"], r["final_rel"],
            ("%d (%.1e)" % (r["floor_cycle"], r["floor_rel"])) if r["floor_cycle"] else "not reached",
            "%.1e" % r["phi_rel_l2"] if "phi_rel_l2" in r else "-",
            "%.1e" % r["hist_floor_c"] if "hist_floor_c" in r else "-",
            r.get("oracle_cycles", "-")))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        fh.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
