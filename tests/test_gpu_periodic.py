"""GPU parity of the periodic boundary conditions (PAPER.md
441-443 and 692-693) against the CPU oracle, through the C-ABI.

Same contract as test_gpu_parity.py: per-cell steps bitwise, whole cycles
Phi rel-L2 <= 1e-10 with the residual-history clause.  Sequences of several
half-sweeps exercise the ghost copies the smoothers store for the next
half-sweep (the periodic ghost rows / planes).
"""
import numpy as np
import pytest

import oracle
from paper_1410_6609_b200 import workloads as W

pytestmark = pytest.mark.gpu

D, N, P = 0, 1, 2
PBCS = {
    "xy": ([P, P, P, P, D, D], [0.0, 0.0, 0.0, 0.0, 0.0, 1.0]),
    "xz": ([P, P, D, N, P, P], [0.0, 0.0, 0.5, -0.25, 0.0, 0.0]),
    "y": ([D, N, P, P, N, D], [1.0, 0.3, 0.0, 0.0, -0.2, 2.0]),
    "z": ([N, D, D, N, P, P], [0.5, -1.0, 0.25, 0.0, 0.0, 0.0]),
    "xyz1": ([P, P, P, P, D, N], [0.0, 0.0, 0.0, 0.0, -1.0, 0.5]),
    "chan": ([P, P, D, D, P, P], [0.0, 0.0, 0.0, 1.0, 0.0, 0.0]),
}


@pytest.fixture(scope="module")
def mg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1410_6609_b200 import _build
    _build.build()
    from paper_1410_6609_b200 import mg as M
    return M


def pair(M, shape, h, bc, **kw):
    bt, bv = PBCS[bc]
    s = M.Multigrid(shape, h, bt, bv, **kw)
    okw = {k: v for k, v in kw.items()
           if k in ("min_coarse", "max_levels", "nu1", "nu2", "alpha",
                    "coarse_tol", "coarse_maxit")}
    o = oracle.Oracle(shape, h, bt, bv, **okw)
    return s, o


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def check_history(hg, ho):
    assert len(hg) == len(ho)
    r0 = ho[0]
    for a, b in zip(hg, ho):
        assert abs(a - b) <= 1e-8 * b + 1e-15 * r0, (a, b)


SHAPES = [((8, 8, 8), 1.0 / 8, "xy"),
          ((12, 10, 6), 1.0, "xz"),           # odd nz/2: ragged row tail
          ((2, 2, 4), 1.0, "xyz1"),           # width-2 periodic axes
          ((66, 34, 20), 1.0, "y"),
          ((16, 12, 10), 0.5, "z"),
          # marching TMA kernels (nz/2 >= 64): partial row tiles, x-chunks
          ((20, 16, 128), 1.0 / 16, "xy"),
          ((34, 12, 256), 1.0, "chan"),
          ((18, 24, 136), 0.5, "z"),
          ((4, 8, 512), 1.0, "xyz1")]


@pytest.mark.parametrize("shape,h,bc", SHAPES)
def test_periodic_half_sweeps_bitwise(mg, shape, h, bc):
    """Five alternating half-sweeps after a copy-in: each one reads the ghost
    copies written by the previous one (or by the copy-in fill)."""
    s, o = pair(mg, shape, h, bc, min_coarse=100)
    rng = np.random.default_rng(21)
    phi = rng.uniform(-1, 1, shape)
    f = rng.uniform(-1, 1, shape)
    s.set_solution(phi)
    s.set_field(0, mg.MG_FIELD_RHS, f)
    o.set_phi(phi)
    o.set_rhs_raw(f)
    for c in (0, 1, 0, 1, 1):
        s.smooth_half(0, c)
        o.smooth_half(0, c)
        assert np.array_equal(s.get_solution(), o.phi())


@pytest.mark.parametrize("shape,h,bc,mc", [
    ((8, 8, 8), 1.0 / 8, "xy", 1),
    ((16, 8, 12), 1.0, "xz", 2),
    ((64, 32, 32), 1.0, "chan", 4),
    ((32, 16, 128), 1.0, "z", 2),       # z-tiled TMA residual kernel
    ((16, 24, 512), 0.5, "xyz1", 2),
    ((48, 8, 136), 1.0, "y", 2)])
def test_periodic_residual_restrict_and_prolong_bitwise(mg, shape, h, bc, mc):
    s, o = pair(mg, shape, h, bc, min_coarse=mc)
    assert s.nlevels == o.nlevels >= 2
    rng = np.random.default_rng(22)
    for l in range(o.nlevels - 1):
        d = o.dims(l)
        phi = rng.uniform(-1, 1, d)
        f = rng.uniform(-1, 1, d)
        s.set_field(l, mg.MG_FIELD_PHI, phi)
        s.set_field(l, mg.MG_FIELD_RHS, f)
        o.set_phi(phi, l)
        o.set_rhs_raw(f, l)
        s.residual_restrict(l)
        o.restrict_residual(l)
        assert np.array_equal(s.get_field(l + 1, mg.MG_FIELD_RHS), o.rhs(l + 1))
        e = rng.uniform(-1, 1, o.dims(l + 1))
        s.set_field(l + 1, mg.MG_FIELD_PHI, e)
        o.set_phi(e, l + 1)
        s.prolong_correct(l)
        o.prolong_correct(l, 2.0)
        assert np.array_equal(s.get_field(l, mg.MG_FIELD_PHI), o.phi(l))
        # the next half-sweep reads the prolongation's periodic ghosts
        s.smooth_half(l, 0)
        o.smooth_half(l, 0)
        assert np.array_equal(s.get_field(l, mg.MG_FIELD_PHI), o.phi(l))


@pytest.mark.parametrize("bc", ["xy", "xz", "xyz1"])
def test_periodic_coarse_cg(mg, bc):
    shape = (16, 8, 8)
    s, o = pair(mg, shape, 1.0, bc, min_coarse=2)
    L = o.nlevels - 1
    f = np.random.default_rng(23).uniform(-1, 1, o.dims(L))
    s.set_field(L, mg.MG_FIELD_RHS, f)
    o.set_rhs_raw(f, L)
    it = s.coarse_solve()
    ito = o.cg(L, 1e-12, 1000)
    assert abs(it - ito) <= 2
    assert rel(s.get_field(L, mg.MG_FIELD_PHI), o.phi(L)) < 1e-11


@pytest.mark.parametrize("shape,h,bc,mc,nu", [
    ((32, 32, 32), 1.0 / 32, "xy", 4, (2, 2)),
    ((64, 32, 48), 0.5, "xz", 2, (2, 2)),
    ((64, 32, 32), 1.0, "chan", 4, (3, 3)),
    ((32, 16, 256), 1.0, "y", 2, (2, 2)),     # marching kernels
    ((64, 64, 128), 1.0, "xyz1", 4, (1, 1)),
    ((48, 24, 136), 0.5, "z", 2, (2, 0)),
    ((32, 32, 32), 1.0, "chan", 2, (0, 2))])
def test_periodic_vcycle_parity(mg, shape, h, bc, mc, nu):
    s, o = pair(mg, shape, h, bc, min_coarse=mc, nu1=nu[0], nu2=nu[1])
    f = np.random.default_rng(24).uniform(-1, 1, shape)
    s.set_rhs(f)
    o.set_rhs(f)
    hg = [s.residual_norm()]
    ho = [o.residual_norm()]
    for _ in range(6):
        hg.append(s.vcycle())
        ho.append(o.vcycle())
    check_history(hg, ho)
    assert rel(s.get_solution(), o.phi()) <= 1e-10


def test_periodic_closed_form_on_gpu(mg):
    """x, y periodic, z Dirichlet: u = sin(2 pi x) sin(2 pi y) sin(pi z) with
    f = 9 pi^2 u gives Phi_h = (9 pi^2 / lambda_h) u exactly (the oracle pin
    test_periodic_closed_form_and_order, here through the CUDA path)."""
    n = 64
    h = 1.0 / n
    x = (np.arange(n) + 0.5) * h
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    u = np.sin(2 * np.pi * X) * np.sin(2 * np.pi * Y) * np.sin(np.pi * Z)
    s = mg.Multigrid((n, n, n), h, [P, P, P, P, D, D], min_coarse=4,
                     coarse_tol=1e-14)
    s.set_rhs(9 * np.pi ** 2 * u)
    for _ in range(14):
        s.vcycle()
    lam = (8 * np.sin(np.pi * h) ** 2 + 4 * np.sin(np.pi * h / 2) ** 2) / h ** 2
    assert np.abs(s.get_solution() - 9 * np.pi ** 2 / lam * u).max() < 1e-10


@pytest.mark.parametrize("Pn", [2, 4])
def test_periodic_loopback_slabs_equal_single(mg, Pn):
    """x-periodic slab decomposition: the first and last slabs exchange
    ghost planes; result bitwise equal to one slab."""
    shape = (128, 32, 32)
    f = np.random.default_rng(25).uniform(-1, 1, shape)
    res = []
    for p in (1, Pn):
        kw = dict(min_coarse=4, agglomerate_below=512)
        if p > 1:
            kw.update(nranks=p, halo="loopback")
        s, _ = pair(mg, shape, 1.0, "chan", **kw)
        s.set_rhs(f)
        r = [s.vcycle() for _ in range(5)]
        res.append((r, s.get_solution()))
        s.close()
    assert np.array_equal(res[0][1], res[1][1])
    assert np.allclose(res[0][0], res[1][0], rtol=1e-13, atol=0)


@pytest.mark.parametrize("shape,bc", [((32, 24, 256), "xy"),
                                      ((64, 16, 128), "chan"),
                                      ((36, 20, 264), "z")])
def test_periodic_march_equals_direct(mg, shape, bc):
    f = np.random.default_rng(26).uniform(-1, 1, shape)
    out = []
    for no_march in (False, True):
        s, _ = pair(mg, shape, 1.0, bc, min_coarse=2,
                    disable=mg.MG_OFF_MARCH if no_march else 0)
        s.set_rhs(f)
        r = [s.vcycle() for _ in range(3)]
        out.append((r, s.get_solution()))
        s.close()
    assert np.array_equal(out[0][1], out[1][1])
    assert np.allclose(out[0][0], out[1][0], rtol=1e-13, atol=0)


def periodic_spheres(shape, h):
    L = np.array(shape) * h
    c = np.array([[0.3 * h, 0.5 * L[1], 0.5 * L[2]],          # wraps x
                  [0.5 * L[0], L[1] - 0.2 * h, 0.4 * L[2]],   # wraps y
                  [L[0] - 0.6 * h, 0.1 * h, L[2] - 0.3 * h],  # wraps x, y (+z)
                  [0.4 * L[0], 0.6 * L[1], 0.5 * L[2]]])
    r = np.array([3.0, 2.5, 3.5, 4.0]) * h
    q = np.array([1.0, -1.0, 2.0, -0.5])
    return c, r, q


@pytest.mark.parametrize("bc", ["xy", "chan", "xyz1"])
@pytest.mark.parametrize("norm,sub", [(0, 1), (1, 1), (0, 2)])
def test_periodic_sphere_rhs_bitwise(mg, bc, norm, sub):
    shape, h = (32, 24, 40), 0.5
    s, o = pair(mg, shape, h, bc, min_coarse=4)
    c, r, q = periodic_spheres(shape, h)
    s.set_rhs_from_spheres(c, r, q, normalization=norm, subsample=sub)
    o.set_rhs_from_spheres(c, r, q, normalization=norm, subsample=sub)
    fg = s.get_field(0, mg.MG_FIELD_RHS)
    assert np.array_equal(fg, o.rhs(0))
    assert fg[0].any() and fg[-1].any()   # the x-wrapping sphere on both sides


def test_periodic_forces_parity(mg):
    """Eq.14-15 on a periodic solution: spheres crossing periodic faces; the
    D3Q19 stencil reads the opposite side's cells."""
    shape, h = (32, 24, 40), 0.5
    s, o = pair(mg, shape, h, "chan", min_coarse=4)
    c, r, q = periodic_spheres(shape, h)
    s.set_rhs_from_spheres(c, r, q)
    o.set_rhs_from_spheres(c, r, q)
    s.solve(1e-10, 40)
    o.solve(1e-10, 40)
    Fg = s.coulomb_forces(c, r, q, subsample=2)
    o.set_phi(s.get_solution())
    Fo = o.coulomb_forces(c, r, q, subsample=2)
    assert np.abs(Fo).max() > 0
    assert np.allclose(Fg, Fo, rtol=1e-12, atol=1e-12 * np.abs(Fo).max())


def test_periodic_forces_loopback(mg):
    shape, h = (48, 24, 40), 0.5
    c, r, q = periodic_spheres(shape, h)
    phi = np.random.default_rng(27).uniform(-1, 1, shape)
    out = []
    for p in (1, 3):
        kw = dict(min_coarse=2, agglomerate_below=64)
        if p > 1:
            kw.update(nranks=p, halo="loopback")
        bt, bv = PBCS["xy"]
        s = mg.Multigrid(shape, h, bt, bv, **kw)
        s.set_solution(phi)
        out.append(s.coulomb_forces(c, r, q))
        s.close()
    assert np.allclose(out[0], out[1], rtol=1e-13, atol=1e-13 * np.abs(out[0]).max())


def test_periodic_errors(mg):
    bt, bv = PBCS["xy"]
    s = mg.Multigrid((16, 8, 8), 1.0, bt, bv, min_coarse=2)
    with pytest.raises(mg.MGError) as e:
        s.set_mask(np.zeros((16, 8, 8), np.uint8))
    assert e.value.code == mg.MG_ERR_BC
    with pytest.raises(mg.MGError) as e:
        s.set_bc_patch(4, 0, 2, 0, 2, D, 1.0)
    assert e.value.code == mg.MG_ERR_BC
    with pytest.raises(mg.MGError) as e:
        s.set_face_values(0, np.zeros(64))
    assert e.value.code == mg.MG_ERR_BC
    with pytest.raises(mg.MGError) as e:   # 2R + 2h > L_y = 8
        s.set_rhs_from_spheres([[8.0, 4.0, 4.0]], [3.5], [1.0])
    assert e.value.code == mg.MG_ERR_ARG
    with pytest.raises(mg.MGError) as e:   # centre outside [0, L_x)
        s.set_rhs_from_spheres([[-0.5, 4.0, 4.0]], [2.0], [1.0])
    assert e.value.code == mg.MG_ERR_ARG
    s.set_rhs_from_spheres([[15.9, 7.9, 4.0]], [2.0], [1.0])
    with pytest.raises(mg.MGError) as e:   # periodic on one face only
        mg.Multigrid((8, 8, 8), 1.0, [D, D, P, D, D, D])
    assert e.value.code == mg.MG_ERR_BC


@pytest.mark.parametrize("bc", ["xy", "chan", "z"])
def test_periodic_tail_kernel_equals_per_step(mg, bc):
    """Periodic coarse levels in the persistent tail kernel (ghost copies by
    the smoother, ghost refresh after the prolongation and the CG) == the
    per-step launches, bit for bit."""
    shape = (64, 32, 64)
    f = np.random.default_rng(27).uniform(-1, 1, shape)
    out = []
    for off in (0, mg.MG_OFF_TAIL):
        s, _ = pair(mg, shape, 1.0, bc, min_coarse=2, disable=off)
        s.set_rhs(f)
        r = [s.vcycle() for _ in range(3)]
        assert bool(s.cycle_paths & mg.MG_PATH_TAIL) == (off == 0)
        out.append((r, s.get_solution()))
        s.close()
    assert np.array_equal(out[0][1], out[1][1])
    assert out[0][0] == out[1][0]
