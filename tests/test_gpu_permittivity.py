"""GPU parity of the variable-permittivity path (reading
d10) against the oracle, through the C-ABI (mg_set_permittivity).

Per-cell steps and every level's operator are bitwise equal (power-of-two
h: the fp64 records are the oracle's stencils scaled by 2^k); whole solves
Phi rel-L2 <= 1e-10 with the residual-history clause of test_gpu_parity.py.
"""
import numpy as np
import pytest

import oracle
from paper_1410_6609_b200 import workloads as W

pytestmark = pytest.mark.gpu

D, N, P = 0, 1, 2
BCS = {
    "dirichlet": ([D] * 6, [1.0, -2.0, 0.5, 3.0, -1.0, 2.0]),
    "channel": ([N, N, D, D, N, N], [0.0, 0.0, 0.0, 1.0, 0.0, 0.0]),
    "mixed": ([N, D, N, D, N, D], [0.25, 1.0, -0.5, -1.0, 2.0, 0.0]),
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


def jumpy(shape, seed, ratio=78.5):
    """Two materials (1 and 78.5: a particle in water) in random blobs,
    times a smooth variation."""
    rng = np.random.default_rng(seed)
    base = np.where(rng.uniform(size=shape) < 0.3, ratio, 1.0)
    x = np.indices(shape).sum(0)
    return base * (1.0 + 0.25 * np.sin(0.7 * x))


def pair(M, shape, h, bc, eps, solid=None, **kw):
    bt, bv = BCS[bc]
    s = M.Multigrid(shape, h, bt, bv, **kw)
    okw = {k: v for k, v in kw.items()
           if k in ("min_coarse", "max_levels", "nu1", "nu2", "alpha",
                    "coarse_tol", "coarse_maxit")}
    o = oracle.Oracle(shape, h, bt, bv, solid=solid, **okw)
    if solid is not None:
        s.set_mask(solid)
    s.set_permittivity(eps)
    o.set_permittivity(eps)
    return s, o


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def check_history(hg, ho):
    assert len(hg) == len(ho)
    r0 = ho[0]
    for a, b in zip(hg, ho):
        assert abs(a - b) <= 1e-8 * b + 1e-15 * r0, (a, b)


@pytest.mark.parametrize("shape,h,bc,mask", [
    ((16, 8, 12), 0.5, "mixed", False),
    ((32, 16, 16), 1.0, "channel", True),
    ((12, 20, 12), 1.0, "dirichlet", False)])
def test_eps_operators_bitwise_every_level(mg, shape, h, bc, mask):
    solid = None
    if mask:
        solid = (np.random.default_rng(4).uniform(size=shape) < 0.1).astype(np.uint8)
    s, o = pair(mg, shape, h, bc, jumpy(shape, 1), solid=solid, min_coarse=2)
    assert s.nlevels == o.nlevels >= 2
    for l in range(o.nlevels):
        assert np.array_equal(s.get_stencil(l), o.stencil(l)), l


@pytest.mark.parametrize("bc", ["dirichlet", "channel", "mixed"])
def test_eps_rhs_adaptation_bitwise(mg, bc):
    shape = (16, 12, 10)
    s, o = pair(mg, shape, 0.5, bc, jumpy(shape, 2), min_coarse=2)
    f = np.random.default_rng(5).uniform(-1, 1, shape)
    s.set_rhs(f)
    o.set_rhs(f)
    assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), o.rhs(0))


@pytest.mark.parametrize("shape,h,bc", [((16, 8, 12), 0.5, "mixed"),
                                        ((32, 16, 128), 1.0, "channel"),
                                        ((12, 20, 12), 1.0, "dirichlet")])
def test_eps_steps_bitwise(mg, shape, h, bc):
    s, o = pair(mg, shape, h, bc, jumpy(shape, 3), min_coarse=2)
    rng = np.random.default_rng(6)
    for l in range(o.nlevels - 1):
        d = o.dims(l)
        phi = rng.uniform(-1, 1, d)
        f = rng.uniform(-1, 1, d)
        s.set_field(l, mg.MG_FIELD_PHI, phi)
        s.set_field(l, mg.MG_FIELD_RHS, f)
        o.set_phi(phi, l)
        o.set_rhs_raw(f, l)
        for c in (0, 1, 0):
            s.smooth_half(l, c)
            o.smooth_half(l, c)
            assert np.array_equal(s.get_field(l, mg.MG_FIELD_PHI), o.phi(l))
        s.residual_restrict(l)
        o.restrict_residual(l)
        assert np.array_equal(s.get_field(l + 1, mg.MG_FIELD_RHS), o.rhs(l + 1))
        e = rng.uniform(-1, 1, o.dims(l + 1))
        s.set_field(l + 1, mg.MG_FIELD_PHI, e)
        o.set_phi(e, l + 1)
        s.prolong_correct(l)
        o.prolong_correct(l, 2.0)
        assert np.array_equal(s.get_field(l, mg.MG_FIELD_PHI), o.phi(l))


@pytest.mark.parametrize("shape,bc,nu,mask", [
    ((32, 32, 32), "dirichlet", (2, 2), False),
    ((64, 32, 32), "channel", (3, 3), False),
    ((64, 32, 48), "mixed", (3, 3), True)])
def test_eps_solve_parity(mg, shape, bc, nu, mask):
    solid = None
    if mask:
        solid = W.beam_mask(shape)
    s, o = pair(mg, shape, 1.0, bc, jumpy(shape, 7), solid=solid, min_coarse=4,
                nu1=nu[0], nu2=nu[1])
    f = np.random.default_rng(8).uniform(-1, 1, shape)
    s.set_rhs(f)
    o.set_rhs(f)
    hg = [s.residual_norm()]
    ho = [o.residual_norm()]
    for _ in range(8):
        hg.append(s.vcycle())
        ho.append(o.vcycle())
    check_history(hg, ho)
    assert rel(s.get_solution(), o.phi()) <= 1e-10
    assert hg[-1] < 0.1 * hg[0]   # converges with 78.5:1 jumps (slowly with the beam)


def test_eps_spheres_in_water_parity(mg):
    """Charged spheres of permittivity 2 in water (78.5) in the config-2
    channel: RHS from the spheres, solve to 1e-8 (P:1534 'jumping
    dielectricity coefficients')."""
    w = W.cfg2(seed=0, shape=(64, 32, 32), n_spheres=8, radius=4.0)
    X = np.indices(w.shape).transpose(1, 2, 3, 0) + 0.5
    eps = np.full(w.shape, 78.5)
    for c, r in zip(w.centers, w.radii):
        eps[((X - c) ** 2).sum(-1) <= r * r] = 2.0
    s, o = pair(mg, w.shape, w.h, "channel", eps, min_coarse=4, nu1=3, nu2=3)
    s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    o.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    rc, cg, hg = s.solve(1e-8, 80)
    so, co, ho = o.solve(1e-8, 80)
    assert rc == 0 and so == 0 and cg == co
    check_history(hg, ho)
    assert rel(s.get_solution(), o.phi()) <= 1e-10


def test_eps_loopback_equals_single(mg):
    shape = (128, 32, 32)
    eps = jumpy(shape, 11)
    f = np.random.default_rng(12).uniform(-1, 1, shape)
    out = []
    for p in (1, 2):
        kw = dict(min_coarse=4, agglomerate_below=512)
        if p > 1:
            kw.update(nranks=p, halo="loopback")
        bt, bv = BCS["channel"]
        s = mg.Multigrid(shape, 1.0, bt, bv, **kw)
        s.set_permittivity(eps)
        s.set_rhs(f)
        r = [s.vcycle() for _ in range(4)]
        out.append((r, s.get_solution()))
        s.close()
    assert np.array_equal(out[0][1], out[1][1])
    assert np.allclose(out[0][0], out[1][0], rtol=1e-13, atol=0)


def test_eps_layered_medium_exact_on_gpu(mg):
    """Layers along x, Dirichlet 0 / 1 on the x faces: the discrete potential
    is the exact series-conductance solution (oracle pin, here on the GPU)."""
    nx, h = 64, 1.0 / 64
    shape = (nx, 16, 16)
    layer = np.where(np.arange(nx) < 24, 1.0, np.where(np.arange(nx) < 40, 80.0, 5.0))
    eps = np.broadcast_to(layer[:, None, None], shape).copy()
    s = mg.Multigrid(shape, h, [D, D, N, N, N, N], [0.0, 1.0, 0, 0, 0, 0],
                     min_coarse=2, nu1=3, nu2=3, coarse_tol=1e-14)
    s.set_permittivity(eps)
    s.set_rhs(np.zeros(shape))
    rc, _, _ = s.solve(1e-14, 300)
    assert rc == 0
    half = h / (2 * layer)
    R_centre = np.cumsum(np.concatenate([[0.0], 2 * half[:-1]])) + half
    exact = R_centre / (2 * half.sum())
    assert np.abs(s.get_solution() - exact[:, None, None]).max() < 1e-10


def test_eps_errors(mg):
    s = mg.Multigrid((8, 8, 8), 1.0, [D] * 6, min_coarse=2)
    e = np.ones((8, 8, 8))
    e[3, 3, 3] = -1.0
    with pytest.raises(mg.MGError) as ex:
        s.set_permittivity(e)
    assert ex.value.code == mg.MG_ERR_ARG
    sp = mg.Multigrid((8, 8, 8), 1.0, [P, P, D, D, D, D], min_coarse=2)
    with pytest.raises(mg.MGError) as ex:
        sp.set_permittivity(np.ones((8, 8, 8)))
    assert ex.value.code == mg.MG_ERR_BC
    s.set_permittivity(None)   # back to constant 1
