"""A small tour of every kernel family for compute-sanitizer (SURVEY 4:
memcheck / racecheck / synccheck in CI): marching and direct half-sweeps,
residual kernels, prolongation, CG (single CTA and cluster), periodic,
masked and permittivity variants, sphere RHS and forces, fused norm,
loopback slabs, async copy-out.
python scripts/sanitize_probe.py   (run under compute-sanitizer)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1410_6609_b200 import mg  # noqa: E402
from paper_1410_6609_b200 import workloads as W  # noqa: E402

D, N, P = 0, 1, 2
rng = np.random.default_rng(0)


def run(shape, bt, bv, cycles=2, **kw):
    mask = kw.pop("mask", None)
    eps = kw.pop("eps", None)
    s = mg.Multigrid(shape, 1.0, bt, bv, **kw)
    if mask is not None:
        s.set_mask(mask)
    if eps is not None:
        s.set_permittivity(eps)
    s.set_rhs(rng.uniform(-1, 1, shape))
    for _ in range(cycles):
        s.vcycle()
    r = s.residual_norm()
    s.close()
    return r


chan = ([N, N, D, D, N, N], [0, 0, 0, 1, 0, 0])
print("box march", run((32, 16, 128), [D] * 6, [0.0] * 6, min_coarse=2))
print("box direct", run((16, 8, 12), *chan, min_coarse=2))
print("periodic", run((32, 16, 128), [P, P, D, D, P, P], [0, 0, 0, 1, 0, 0], min_coarse=2))
w = W.cfg5(scale=16, n_spheres=10)
print("mask", run(w.shape, *chan, mask=w.solid, min_coarse=w.min_coarse, nu1=3, nu2=3))
print("permittivity", run((16, 16, 24), *chan, eps=np.where(rng.uniform(size=(16, 16, 24)) < 0.3, 78.5, 1.0), min_coarse=2))
print("fused norm", run((32, 16, 128), *chan, min_coarse=2, fused_norm=True))
print("loopback", run((64, 16, 128), *chan, min_coarse=4, nranks=2, halo="loopback", agglomerate_below=4096))
# cluster CG on a 64 x 8 x 8 coarsest grid
s = mg.Multigrid((64, 8, 8), 1.0, *chan, max_levels=1)
s.set_field(0, mg.MG_FIELD_RHS, rng.uniform(-1, 1, (64, 8, 8)))
print("cluster cg its", s.coarse_solve())
s.close()
# spheres, forces, timestep, async copy-out
wk = W.cfg2(seed=0, shape=(64, 32, 128), n_spheres=10)
s = mg.Multigrid(wk.shape, wk.h, wk.bc_type, wk.bc_value, min_coarse=4)
F, n, r = s.timestep(wk.centers, wk.radii, wk.charges, cycles=2, subsample=2)
print("timestep", n, r, float(np.abs(F).max()))
out = torch.empty(wk.shape, dtype=torch.float64).pin_memory()
s.get_solution_async(out)
print("async", s.wait(), float(out.abs().max()))
s.close()
