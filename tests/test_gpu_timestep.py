"""Time-stepping regime (Alg.1)
through the C-ABI's mg_timestep, against the oracle doing the same steps:
RHS from the moved spheres (subsampling 2), warm-started V(3,3)
cycles (5 at the first step, then 1), Coulomb forces.

Per step: residual within the history clause of test_gpu_parity.py, Phi
rel-L2 <= 1e-10, forces rel 1e-9 (they are sums over the solved Phi, which
agrees to ~1e-13; the force sums differ only in order).
"""
import numpy as np
import pytest

import oracle
from paper_1410_6609_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1410_6609_b200 import _build
    _build.build()
    from paper_1410_6609_b200 import mg as M
    return M


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def run_steps(mg, w, steps, periodic=(False, False, False), sub=2,
              amplitude=0.3, **kw):
    s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value,
                     min_coarse=w.min_coarse, nu1=3, nu2=3, **kw)
    o = oracle.Oracle(w.shape, w.h, w.bc_type, w.bc_value,
                      min_coarse=w.min_coarse, nu1=3, nu2=3)
    c = w.centers
    out = []
    for k in range(steps):
        if k:
            c = W.move_spheres(c, w.radii, np.array(w.shape) * w.h, k,
                               seed=7, amplitude=amplitude, periodic=periodic)
        cyc = 5 if k == 0 else 1
        Fg, ncyc, rg = s.timestep(c, w.radii, w.charges, cycles=cyc,
                                  subsample=sub)
        o.set_rhs_from_spheres(c, w.radii, w.charges, subsample=sub)
        ro = None
        for _ in range(cyc):
            ro = o.vcycle()
        Fo = o.coulomb_forces(c, w.radii, w.charges, subsample=sub)
        out.append((ncyc, rg, ro, Fg, Fo, s.get_solution(), o.phi()))
    return out


def test_timestep_parity_channel(mg):
    w = W.timestep_workload(n=64, seed=1)
    assert len(w.radii) == 14
    res = run_steps(mg, w, 5)
    r0 = res[0][2]
    for k, (ncyc, rg, ro, Fg, Fo, pg, po) in enumerate(res):
        assert ncyc == (5 if k == 0 else 1)
        assert abs(rg - ro) <= 1e-8 * ro + 1e-15 * r0, (k, rg, ro)
        assert rel(pg, po) <= 1e-10
        assert np.abs(Fo).max() > 0
        assert np.allclose(Fg, Fo, rtol=1e-9, atol=1e-9 * np.abs(Fo).max())
    # warm start: one V(3,3) per step keeps the residual near the first
    # solve's level while the spheres move
    assert max(r[1] for r in res[1:]) < 50 * res[0][1]


def test_timestep_parity_periodic_channel(mg):
    """Periodic flow / span axes: moving spheres wrap around (images)."""
    w = W.timestep_workload(n=64, seed=2)
    w.bc_type, w.bc_value = W.periodic_channel_bc(1.0)
    c = w.centers.copy()
    c[0] = [0.4, 20.0, 63.7]            # straddles the x and z faces
    w.centers = c
    res = run_steps(mg, w, 4, periodic=(True, False, True), amplitude=0.8)
    r0 = res[0][2]
    for k, (ncyc, rg, ro, Fg, Fo, pg, po) in enumerate(res):
        assert abs(rg - ro) <= 1e-8 * ro + 1e-15 * r0, (k, rg, ro)
        assert rel(pg, po) <= 1e-10
        assert np.allclose(Fg, Fo, rtol=1e-9, atol=1e-9 * np.abs(Fo).max())


@pytest.mark.parametrize("halo,P,periodic", [("loopback", 2, False), ("loopback", 4, False),
                                             ("emulate", 2, False), ("loopback", 2, True),
                                             ("emulate", 4, True)])
def test_timestep_parity_slabs(mg, halo, P, periodic):
    """x-slab decomposition (one process, LOOPBACK device copies or the NCCL
    schedule EMULATEd), box and periodic channels: the batched step (RHS,
    cycle and forces enqueued back to back, one host wait) against the
    oracle."""
    w = W.timestep_workload(n=64, seed=5)
    per = (False, False, False)
    if periodic:
        w.bc_type, w.bc_value = W.periodic_channel_bc(1.0)
        per = (True, False, True)
    res = run_steps(mg, w, 3, periodic=per, amplitude=0.8 if periodic else 0.3,
                    nranks=P, halo=halo, agglomerate_below=512)
    r0 = res[0][2]
    for k, (ncyc, rg, ro, Fg, Fo, pg, po) in enumerate(res):
        assert ncyc == (5 if k == 0 else 1)
        assert abs(rg - ro) <= 1e-8 * ro + 1e-15 * r0, (k, rg, ro)
        assert rel(pg, po) <= 1e-10
        assert np.allclose(Fg, Fo, rtol=1e-9, atol=1e-9 * np.abs(Fo).max())


def test_timestep_tolerance_mode(mg):
    """cycles = 0: V-cycles while ||r|| > abs_tol (Alg.1), the
    same count as the oracle's loop."""
    w = W.timestep_workload(n=64, seed=3)
    s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8,
                     nu1=3, nu2=3)
    o = oracle.Oracle(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8,
                      nu1=3, nu2=3)
    tol = 1.5e-8     # the paper's monitored bound
    c = w.centers
    r0 = None
    for k in range(3):
        if k:
            c = W.move_spheres(c, w.radii, np.array(w.shape), k, seed=4,
                               amplitude=0.5)
        _, ncyc, rg = s.timestep(c, w.radii, w.charges, cycles=0, abs_tol=tol,
                                 subsample=2, forces=False)
        o.set_rhs_from_spheres(c, w.radii, w.charges, subsample=2)
        r = o.residual_norm()
        r0 = r if r0 is None else r0     # floor clause scale (reading c21)
        n = 0
        while r > tol:
            r = o.vcycle()
            n += 1
        assert ncyc == n and rg <= tol
        assert abs(rg - r) <= 1e-8 * r + 1e-15 * r0


def test_timestep_errors(mg):
    w = W.timestep_workload(n=32, seed=0)
    s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=4)
    with pytest.raises(mg.MGError) as e:
        s.timestep(w.centers, w.radii, w.charges, cycles=-1)
    assert e.value.code == mg.MG_ERR_ARG
    with pytest.raises(mg.MGError) as e:
        s.timestep(w.centers, w.radii, w.charges, cycles=0, abs_tol=0.0)
    assert e.value.code == mg.MG_ERR_ARG
    # an unreachable tolerance: NOTCONV, forces still returned on request
    s2 = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=4,
                      max_cycles=2)
    F, n, r = s2.timestep(w.centers, w.radii, w.charges, cycles=0,
                          abs_tol=1e-300, raise_notconv=False)
    assert n == 2 and F.shape == (len(w.radii), 3)


@pytest.mark.parametrize("cycles,forces", [(1, True), (1, False), (3, True)])
def test_timestep_empty_sphere_reported(mg, cycles, forces):
    """With cycles > 0 the step is enqueued back to back and the host waits
    once: a sphere that covers no cell centre is still reported (MG_ERR_ARG),
    after the step; the next valid step equals a fresh context's."""
    w = W.timestep_workload(n=32, seed=0)
    c = np.concatenate([w.centers, [[8.0, 8.0, 8.0]]])
    R = np.concatenate([w.radii, [0.2]])
    q = np.concatenate([w.charges, [1.0]])
    s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=4)
    with pytest.raises(mg.MGError) as e:
        s.timestep(c, R, q, cycles=cycles, forces=forces)
    assert e.value.code == mg.MG_ERR_ARG
    # the valid list afterwards: same forces and residual as a fresh context
    s.zero_solution()
    F1, n1, r1 = s.timestep(w.centers, w.radii, w.charges, cycles=cycles)
    s2 = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=4)
    F2, n2, r2 = s2.timestep(w.centers, w.radii, w.charges, cycles=cycles)
    assert n1 == n2 == cycles and r1 == r2
    assert np.array_equal(F1, F2)
    s.close()
    s2.close()


def test_timestep_parity_masked(mg):
    """Config 5's geometry (beam mask, channel walls) in the batched step:
    RHS with the solid cells zeroed, warm-started V(3,3), forces with solid
    gradient neighbours (reading d6), against the oracle."""
    w = W.cfg5(scale=16, n_spheres=40)
    s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=w.min_coarse,
                     nu1=3, nu2=3)
    s.set_mask(w.solid)
    o = oracle.Oracle(w.shape, w.h, w.bc_type, w.bc_value, solid=w.solid,
                      min_coarse=w.min_coarse, nu1=3, nu2=3)
    c = w.centers
    r0 = None
    for k in range(3):
        if k:
            c = W.move_spheres(c, w.radii, np.array(w.shape) * w.h, k, seed=11,
                               amplitude=0.3)
        cyc = 5 if k == 0 else 1
        Fg, n, rg = s.timestep(c, w.radii, w.charges, cycles=cyc)
        o.set_rhs_from_spheres(c, w.radii, w.charges)
        if r0 is None:
            r0 = o.residual_norm()
        ro = None
        for _ in range(cyc):
            ro = o.vcycle()
        Fo = o.coulomb_forces(c, w.radii, w.charges)
        assert n == cyc
        assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), o.rhs(0))
        assert abs(rg - ro) <= 1e-8 * ro + 1e-15 * r0, (k, rg, ro)
        assert rel(s.get_solution(), o.phi()) <= 1e-10
        assert np.allclose(Fg, Fo, rtol=1e-9, atol=1e-9 * np.abs(Fo).max())
    s.close()
