"""Per-cycle times of the solver variants at 512^3 on one GPU (round report):
box (config 3), periodic channel (N3), solid beam mask (config-5 geometry
at 512^3 scale), variable permittivity with 78.5:1 jumps (N4).  Each: V(2,2)
cycles from a random RHS, median of CUDA-event times around mg_vcycle, and
the fraction of the variant's byte model at the measured HBM peak.

usage: python scripts/variant_bench.py [--n 512] [--out gpurun_out/r01_variants.md]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def model_bytes(levels, half, rr, pr, norm, nu=2):
    """Bytes per fine cell of a V(nu,nu)-cycle: per level 2 nu sweeps of two
    half-sweeps, residual+restriction and prolongation, times 8^-l; norm."""
    tot = 0.0
    for l in range(levels - 1):
        tot += (4 * nu * half + rr + pr) * 8.0 ** -l
    return tot + norm


def main():
    import torch
    from paper_1410_6609_b200 import mg
    from paper_1410_6609_b200 import workloads as W
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--cycles", type=int, default=8)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    n = a.n
    shape = (n, n, n)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    f = np.random.default_rng(0).uniform(-1, 1, shape)
    D, N, P = mg.MG_DIRICHLET, mg.MG_NEUMANN, mg.MG_PERIODIC
    rng = np.random.default_rng(1)
    eps = np.where(rng.uniform(size=shape) < 0.3, 78.5, 1.0)
    # (name, bt, bv, solid, eps, half-sweep, restriction, prolongation B/cell,
    #  norm B/cell by path: look-ahead / split / full pass)
    cases = [
        ("box (config 3 BCs)", [D] * 6, [0.0] * 6, None, None, 12, 17, 17, (4, 12, 16)),
        ("periodic channel: x, z periodic, y Dirichlet 0/1 (N3)",
         [P, P, D, D, P, P], [0, 0, 0, 1, 0, 0], None, None, 12, 17, 17, (4, 12, 16)),
        ("solid beam mask, channel BCs (config-5 geometry)",
         [N, N, D, D, N, N], [0, 0, 0, 1, 0, 0], W.beam_mask(shape), None,
         12.5, 18, 17.5, (4.5, 12.5, 17)),
        ("variable permittivity, 78.5:1 jumps, channel BCs (N4)",
         [N, N, D, D, N, N], [0, 0, 0, 1, 0, 0], None, eps, 12 + 32, 17 + 64, 17,
         (4, 12 + 32, 16 + 64)),
    ]
    rows = []
    for name, bt, bv, solid, ep, hs, rr, pr, norms in cases:
        stream = torch.cuda.Stream()
        s = mg.Multigrid(shape, 1.0, bt, bv, min_coarse=8, stream=stream)
        if solid is not None:
            s.set_mask(solid)
        if ep is not None:
            s.set_permittivity(ep)
        s.set_rhs(f)
        s.vcycle()
        times, res = [], []
        for _ in range(a.cycles):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res.append(s.vcycle())
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = float(np.median(times))
        paths = s.cycle_paths
        norm = norms[0] if paths & mg.MG_PATH_LOOKAHEAD else (
            norms[1] if paths & mg.MG_PATH_SPLIT_NORM else norms[2])
        mb = model_bytes(s.nlevels, hs, rr, pr, norm)
        frac = mb * n ** 3 / (ms * 1e-3) / 1e9 / peak
        fac = (res[-1] / res[0]) ** (1.0 / (len(res) - 1))
        rows.append((name, ms, n ** 3 / (ms * 1e-3) / 1e6, mb, frac, fac,
                     s.cycle_launches))
        s.close()
        del s
        torch.cuda.empty_cache()
    md = ["# Solver variants on one B200, %d^3, V(2,2) (round 2)" % n, "",
          "Median CUDA-event time of `mg_vcycle` (graph launch + residual norm "
          "readback) over %d cycles after one warm-up; byte model = the "
          "variant's algorithmic bytes per fine cell and cycle (SURVEY 8(d) "
          "plus the operator data the variant must read: 0.5 B/cell of face "
          "codes per half-sweep for the mask, 64 B per cell of fp64 records "
          "for the permittivity in the smoother, residual and norm -- the "
          "prolongation needs none without a mask; the norm: 4 B/cell with the "
          "look-ahead red sweep, else the split or full pass, as the recorded "
          "cycle took it); fraction at the measured peak %.1f GB/s." % (a.cycles, peak),
          "",
          "| variant | ms/cycle | Mcells/s | model B/cell | model-roofline fraction | factor/cycle | launches |",
          "|---|---|---|---|---|---|---|"]
    for r in rows:
        md.append("| %s | %.3f | %.0f | %.1f | %.3f | %.3f | %d |" % r)
    txt = "\n".join(md) + "\n"
    print(txt)
    if a.out:
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        open(a.out, "w").write(txt)


if __name__ == "__main__":
    main()
