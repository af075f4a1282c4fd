"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Per-cell steps (smoother half-sweeps, residual + restriction, prolongation,
sphere RHS, BC adaptation, layout conversion) must be BITWISE equal for
power-of-two h ("Parity contract"); whole V-cycles must match in
Phi to relative L2 1e-10 and in residual history to 1e-8 relative (north_star)
with the rounding-floor clause |dr_k| <= 1e-8 r_k + 1e-15 r_0 (reading c21,
DESIGN.md: per-cell steps are bitwise, so the only differences are the CG and
norm reductions; an ulp-level difference in Phi moves the residual by about
eps*||A||*||Phi||, measured at 1.2e-16 r_0 on config 1).
"""
import numpy as np
import pytest

import oracle
from paper_1410_6609_b200 import workloads as W

pytestmark = pytest.mark.gpu

D, N = 0, 1
BCS = {
    "dirichlet0": ([D] * 6, [0.0] * 6),
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


def pair(M, shape, h, bc, **kw):
    bt, bv = BCS[bc]
    s = M.Multigrid(shape, h, bt, bv, **kw)
    okw = {k: v for k, v in kw.items()
           if k in ("min_coarse", "max_levels", "nu1", "nu2", "alpha",
                    "coarse_tol", "coarse_maxit")}
    o = oracle.Oracle(shape, h, bt, bv, **okw)
    return s, o


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


SHAPES = [((8, 8, 8), 1.0 / 8, "dirichlet"),
          ((12, 10, 6), 1.0, "mixed"),          # odd nz/2: ragged row tail
          ((32, 16, 64), 0.25, "channel"),      # many blocks
          ((2, 2, 2), 1.0, "dirichlet"),
          ((66, 34, 20), 1.0, "mixed"),
          # marching TMA kernel (nz/2 >= 64): full/partial row tiles and
          # x-chunks, pitch not a multiple of 8, 1..4 chunks per lane
          ((20, 16, 128), 1.0 / 16, "dirichlet"),
          ((34, 12, 256), 1.0, "mixed"),
          ((18, 24, 136), 0.5, "channel"),
          ((4, 8, 512), 1.0, "mixed")]


@pytest.mark.parametrize("shape,h,bc", SHAPES)
def test_layout_roundtrip(mg, shape, h, bc):
    s, _ = pair(mg, shape, h, bc, min_coarse=100)
    rng = np.random.default_rng(0)
    a = rng.standard_normal(shape)
    s.set_solution(a)
    assert np.array_equal(s.get_solution(), a)
    b = rng.standard_normal(shape)
    s.set_field(0, mg.MG_FIELD_RHS, b)
    assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), b)


@pytest.mark.parametrize("shape,h,bc", SHAPES)
@pytest.mark.parametrize("color", [0, 1])
def test_half_sweep_bitwise(mg, shape, h, bc, color):
    s, o = pair(mg, shape, h, bc, min_coarse=100)
    rng = np.random.default_rng(1 + color)
    phi = rng.uniform(-1, 1, shape)
    f = rng.uniform(-1, 1, shape)
    s.set_solution(phi)
    s.set_field(0, mg.MG_FIELD_RHS, f)
    o.set_phi(phi)
    o.set_rhs_raw(f)
    for c in (color, 1 - color, color):
        s.smooth_half(0, c)
        o.smooth_half(0, c)
        assert np.array_equal(s.get_solution(), o.phi())


def test_half_sweep_from_zero_bitwise(mg):
    shape = (16, 8, 12)
    s, o = pair(mg, shape, 1.0, "channel", min_coarse=100)
    f = np.random.default_rng(3).uniform(-1, 1, shape)
    s.set_solution(np.random.default_rng(4).uniform(-1, 1, shape))  # ignored
    s.set_field(0, mg.MG_FIELD_RHS, f)
    o.set_phi(np.zeros(shape))
    o.set_rhs_raw(f)
    s.smooth_half(0, 0, from_zero=True)
    o.smooth_half(0, 0)
    red = ((np.indices(shape).sum(0)) & 1) == 0
    assert np.array_equal(s.get_solution()[red], o.phi()[red])


@pytest.mark.parametrize("shape,h,bc,mc", [
    ((8, 8, 8), 1.0 / 8, "dirichlet", 2),
    ((16, 8, 12), 1.0, "mixed", 2),
    ((64, 32, 32), 1.0, "channel", 4),
    ((32, 32, 32), 1.0 / 32, "dirichlet0", 4),
    # z-tiled TMA residual+restriction kernel (nz/2 >= 64), 1 and 2 z-tiles
    ((32, 16, 128), 1.0, "mixed", 2),
    ((16, 24, 512), 0.5, "channel", 2),
    ((48, 8, 136), 1.0, "dirichlet", 2)])
def test_residual_restrict_and_prolong_bitwise(mg, shape, h, bc, mc):
    s, o = pair(mg, shape, h, bc, min_coarse=mc)
    assert s.nlevels == o.nlevels >= 2
    rng = np.random.default_rng(5)
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


@pytest.mark.parametrize("bc", ["dirichlet", "channel", "mixed"])
@pytest.mark.parametrize("h", [1.0, 0.5, 0.1])
def test_set_rhs_bc_adaptation_bitwise(mg, bc, h):
    """BC adaptation is bitwise for any h (same expressions)."""
    shape = (10, 12, 14)
    s, o = pair(mg, shape, h, bc, min_coarse=100)
    f = np.random.default_rng(6).uniform(-1, 1, shape)
    s.set_rhs(f)
    o.set_rhs(f)
    assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), o.rhs(0))


@pytest.mark.parametrize("norm", [0, 1])
@pytest.mark.parametrize("sub", [1, 2, 3])
def test_sphere_rhs_bitwise(mg, norm, sub):
    """Sphere RHS incl. subsampling s_f bitwise vs the oracle."""
    w = W.cfg2(seed=1)
    s, o = pair(mg, w.shape, w.h, "channel", min_coarse=4)
    s.set_rhs_from_spheres(w.centers, w.radii, w.charges, normalization=norm,
                           subsample=sub)
    o.set_rhs_from_spheres(w.centers, w.radii, w.charges, normalization=norm,
                           subsample=sub)
    assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), o.rhs(0))


def overlapping_spheres(L):
    """Clusters of 3-6 spheres around common centres (cells covered by up
    to 6 spheres), charges of mixed sign and magnitude so that the order of
    the additions changes the rounded sums."""
    rng = np.random.default_rng(31)
    c, R, q = [], [], []
    for base in ([0.3, 0.5, 0.5], [0.7, 0.4, 0.6], [0.5, 0.8, 0.3]):
        for m in range(3 + len(c) % 4):
            c.append(np.array(base) * L + rng.uniform(-1.5, 1.5, 3))
            R.append(rng.uniform(3.0, 5.0))
            q.append(rng.choice([-1, 1]) * 10.0 ** rng.uniform(-3, 1))
    # interleave the clusters so that covering spheres are not consecutive
    order = rng.permutation(len(c))
    return np.array(c)[order], np.array(R)[order], np.array(q)[order]


@pytest.mark.parametrize("norm", [0, 1])
@pytest.mark.parametrize("sub", [1, 2])
@pytest.mark.parametrize("P", [1, 2])
def test_sphere_rhs_overlapping_bitwise(mg, norm, sub, P):
    """Cells covered by 3 or more spheres: the GPU adds the densities in
    sphere order, like the oracle ("overlapping spheres add in sphere
    order"), so f is bitwise equal and run-to-run deterministic;
    also on loopback slabs."""
    shape = (48, 32, 40)
    c, R, q = overlapping_spheres(np.array(shape, float))
    kw = dict(nranks=P, halo="loopback", agglomerate_below=64) if P > 1 else {}
    s, o = pair(mg, shape, 1.0, "channel", min_coarse=4, **kw)
    o.set_rhs_from_spheres(c, R, q, normalization=norm, subsample=sub)
    ref = o.rhs(0)
    cover = sum((oracle.sphere_density(shape, 1.0, c[p:p + 1], R[p:p + 1], [1.0],
                                       normalization=1) != 0).astype(int)
                for p in range(len(R)))
    assert cover.max() >= 4
    for _ in range(2):
        s.set_rhs_from_spheres(c, R, q, normalization=norm, subsample=sub)
        assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), ref)


def test_sphere_rhs_overlapping_periodic(mg):
    """Overlapping spheres whose periodic images wrap (x and z periodic)."""
    shape = (32, 24, 40)
    bt = [2, 2, D, D, 2, 2]
    bv = [0.0, 0.0, 0.0, 1.0, 0.0, 0.0]
    c = np.array([[0.4, 12.0, 1.0], [1.5, 11.0, 39.5], [31.0, 12.5, 0.5],
                  [0.9, 12.2, 38.8], [2.0, 13.0, 2.5]])
    R = np.array([4.0, 3.5, 4.5, 3.0, 4.2])
    q = np.array([1.0, -0.37, 2.9e-2, 5.1, -1.3])
    s = mg.Multigrid(shape, 1.0, bt, bv, min_coarse=4)
    o = oracle.Oracle(shape, 1.0, bt, bv, min_coarse=4)
    for sub in (1, 3):
        s.set_rhs_from_spheres(c, R, q, subsample=sub)
        o.set_rhs_from_spheres(c, R, q, subsample=sub)
        assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), o.rhs(0))


def test_sphere_rhs_physical_units_and_errors(mg):
    shape, h = (32, 16, 24), 0.125
    c, q = W.random_spheres(np.array(shape) * h, 0.5, 6, seed=2)
    s, o = pair(mg, shape, h, "mixed", min_coarse=2)
    R = np.full(6, 0.5)
    s.set_rhs_from_spheres(c, R, q)
    o.set_rhs_from_spheres(c, R, q)
    assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), o.rhs(0))
    with pytest.raises(mg.MGError) as e:
        s.set_rhs_from_spheres(np.array([[0.3, 0.3, 0.3]]), [0.01], [1.0])
    assert e.value.code == mg.MG_ERR_ARG
    with pytest.raises(mg.MGError):
        s.set_rhs_from_spheres(c, -R, q)


def test_coarse_cg(mg):
    shape = (16, 8, 8)
    s, o = pair(mg, shape, 1.0, "mixed", min_coarse=2)
    L = o.nlevels - 1
    f = np.random.default_rng(8).uniform(-1, 1, o.dims(L))
    s.set_field(L, mg.MG_FIELD_RHS, f)
    o.set_rhs_raw(f, L)
    it = s.coarse_solve()
    ito = o.cg(L, 1e-12, 1000)
    assert abs(it - ito) <= 2
    assert rel(s.get_field(L, mg.MG_FIELD_PHI), o.phi(L)) < 1e-11


@pytest.mark.parametrize("shape,bt,bv", [
    ((64, 8, 8), [N, N, D, D, N, N], [0, 0, 0, 1, 0, 0]),     # config 4 P=8 coarsest
    ((64, 16, 8), [N, D, N, D, N, D], [0.25, 1.0, -0.5, -1.0, 2.0, 0.0]),
    ((16, 16, 24), [2, 2, D, N, 2, 2], [0, 0, 0.5, -0.25, 0, 0]),  # x, z periodic
    ((40, 10, 22), [D] * 6, [1.0, -2.0, 0.5, 3.0, -1.0, 2.0]),   # ragged chunks
])
def test_coarse_cg_cluster(mg, shape, bt, bv):
    """The cluster CG (8 CTAs, distributed shared memory) on large coarsest
    grids and the single-CTA CG (mg_opts.disable = MG_OFF_CG_CLUSTER): both
    the oracle's CG solution to 1e-11, iteration counts within 2 (the dot
    products sum in another order); the paths taken are checked."""
    f = np.random.default_rng(9).uniform(-1, 1, shape)
    o = oracle.Oracle(shape, 1.0, bt, bv, max_levels=1)
    o.set_rhs_raw(f, 0)
    ito = o.cg(0, 1e-12, 1000)
    out = []
    for cluster in (True, False):
        s = mg.Multigrid(shape, 1.0, bt, bv, max_levels=1,
                         disable=0 if cluster else mg.MG_OFF_CG_CLUSTER)
        s.set_field(0, mg.MG_FIELD_RHS, f)
        it = s.coarse_solve()
        assert bool(s.cycle_paths & mg.MG_PATH_CG_CLUSTER) == cluster
        out.append((it, s.get_field(0, mg.MG_FIELD_PHI)))
        s.close()
    assert abs(out[0][0] - ito) <= 2 and abs(out[1][0] - ito) <= 2
    assert rel(out[0][1], o.phi(0)) < 1e-11
    assert rel(out[1][1], o.phi(0)) < 1e-11


def check_history(hg, ho):
    assert len(hg) == len(ho)
    r0 = ho[0]
    for a, b in zip(hg, ho):
        assert abs(a - b) <= 1e-8 * b + 1e-15 * r0, (a, b)


def run_fixed(s, o, cycles):
    hg = [s.residual_norm()]
    ho = [o.residual_norm()]
    for _ in range(cycles):
        hg.append(s.vcycle())
        ho.append(o.vcycle())
    return hg, ho


def test_config1_parity(mg):
    w = W.cfg1(32)
    s, o = pair(mg, w.shape, w.h, "dirichlet0", min_coarse=4,
                coarse_tol=w.coarse_tol)
    s.set_rhs(w.rhs)
    o.set_rhs(w.rhs)
    hg, ho = run_fixed(s, o, w.cycles)
    check_history(hg, ho)
    assert rel(s.get_solution(), o.phi()) <= 1e-10
    # the discrete solution is c(h) u (closed form)
    u = w.rhs / (3 * np.pi ** 2)
    ch = (np.pi * w.h / 2) ** 2 / np.sin(np.pi * w.h / 2) ** 2
    assert np.abs(s.get_solution() - ch * u).max() < 1e-8


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_config2_parity(mg, seed):
    w = W.cfg2(seed=seed)
    s, o = pair(mg, w.shape, w.h, "channel", min_coarse=4)
    s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    o.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    rc, cg, hg = s.solve(w.tol, 60)
    so, co, ho = o.solve(w.tol, 60)
    assert rc == 0 and so == 0 and cg == co
    check_history(hg, ho)
    assert rel(s.get_solution(), o.phi()) <= 1e-10


@pytest.mark.parametrize("n", [64, 128])
def test_config3_reduced_parity(mg, n):
    w = W.cfg3(n, seed=0, cycles=20)
    s, o = pair(mg, w.shape, w.h, "dirichlet0", min_coarse=8)
    s.set_rhs(w.rhs)
    o.set_rhs(w.rhs)
    hg, ho = run_fixed(s, o, w.cycles)
    check_history(hg, ho)
    assert rel(s.get_solution(), o.phi()) <= 1e-10


def test_mixed_bc_schedules_parity(mg):
    shape = (64, 32, 48)
    for nu in ((1, 1), (3, 3), (2, 0), (0, 2)):
        s, o = pair(mg, shape, 0.5, "mixed", min_coarse=2, nu1=nu[0], nu2=nu[1])
        f = np.random.default_rng(9).uniform(-1, 1, shape)
        s.set_rhs(f)
        o.set_rhs(f)
        hg, ho = run_fixed(s, o, 6)
        check_history(hg, ho)
        assert rel(s.get_solution(), o.phi()) <= 1e-10


def test_graph_and_eager_identical(mg):
    w = W.cfg2(seed=0, shape=(64, 32, 32), n_spheres=10)
    out = []
    for g in (True, False):
        s, _ = pair(mg, w.shape, w.h, "channel", min_coarse=4, use_graph=g)
        s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
        r = [s.vcycle() for _ in range(4)]
        out.append((r, s.get_solution()))
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])


def test_zero_rhs_and_warm_start(mg):
    shape = (32, 16, 16)
    s, _ = pair(mg, shape, 1.0, "dirichlet0", min_coarse=2)
    s.set_rhs(np.zeros(shape))
    rc, cyc, hist = s.solve(1e-8, 5)
    assert rc == 0 and cyc == 0 and not s.get_solution().any()
    f = np.random.default_rng(0).uniform(-1, 1, shape)
    s.set_rhs(f)
    s.solve(1e-10, 50)
    r_warm = s.residual_norm()
    s.set_rhs(f)  # does not touch Phi (warm start)
    assert s.residual_norm() == r_warm


@pytest.mark.parametrize("P", [2, 4])
def test_loopback_slabs_equal_single(mg, P):
    """x-slab decomposition (P slabs on one GPU, halo by device copies) gives
    the 1-slab result bitwise in Phi (per-cell ops are bitwise and the
    agglomerated coarse levels are the same computation)."""
    w = W.cfg2(seed=0, shape=(128, 32, 32), n_spheres=20)
    res = []
    for p in (1, P):
        kw = dict(min_coarse=4, agglomerate_below=512)
        if p > 1:
            kw.update(nranks=p, halo="loopback")
        s, _ = pair(mg, w.shape, w.h, "channel", **kw)
        s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
        r = [s.vcycle() for _ in range(5)]
        res.append((r, s.get_solution()))
    assert np.array_equal(res[0][1], res[1][1])
    assert np.allclose(res[0][0], res[1][0], rtol=1e-13, atol=0)


def test_errors(mg):
    with pytest.raises(mg.MGError) as e:
        mg.Multigrid((8, 8, 8), 1.0, [N] * 6)
    assert e.value.code == mg.MG_ERR_BC
    with pytest.raises(mg.MGError) as e:
        mg.Multigrid((9, 8, 8), 1.0, [D] * 6)
    assert e.value.code == mg.MG_ERR_COARSEN
    with pytest.raises(mg.MGError) as e:
        mg.Multigrid((8, 8, 8), 1.0, [2] + [D] * 5)
    assert e.value.code == mg.MG_ERR_BC
    # divergence: a negative magnification blows the iteration up
    shape = (32, 32, 32)
    s = mg.Multigrid(shape, 1.0, [D] * 6, min_coarse=2, alpha=-8.0)
    s.set_rhs(np.random.default_rng(0).uniform(-1, 1, shape))
    with pytest.raises(mg.MGError) as e:
        for _ in range(20):
            s.vcycle()
    assert e.value.code == mg.MG_ERR_DIVERGED


@pytest.mark.parametrize("shape,bc", [((32, 24, 256), "mixed"),
                                      ((64, 16, 128), "channel"),
                                      ((16, 16, 512), "dirichlet"),
                                      ((36, 20, 264), "channel"),
                                      ((128, 64, 128), "mixed")])
def test_march_kernels_equal_direct_kernels(mg, shape, bc):
    """The TMA-marching kernels (half-sweep, prolongation fused with the
    first post-smoothing red sweep, residual+restriction, split norm) give
    the same V-cycle iterates as the direct-load kernels (mg_opts.disable =
    MG_OFF_MARCH), bit for bit."""
    f = np.random.default_rng(12).uniform(-1, 1, shape)
    out = []
    for no_march in (False, True):
        s, _ = pair(mg, shape, 1.0, bc, min_coarse=2,
                    disable=mg.MG_OFF_MARCH if no_march else 0)
        s.set_rhs(f)
        r = [s.vcycle() for _ in range(3)]
        march = mg.MG_PATH_MARCH | mg.MG_PATH_PROLONG_FUSED | mg.MG_PATH_SPLIT_NORM
        assert (s.cycle_paths & march) == (0 if no_march else march), s.cycle_paths
        out.append((r, s.get_solution()))
    assert np.array_equal(out[0][1], out[1][1])
    assert np.allclose(out[0][0], out[1][0], rtol=1e-13, atol=0)


def test_march_norm_matches_oracle(mg):
    shape = (48, 16, 256)
    s, o = pair(mg, shape, 1.0, "mixed", min_coarse=2)
    rng = np.random.default_rng(13)
    phi = rng.uniform(-1, 1, shape)
    f = rng.uniform(-1, 1, shape)
    s.set_solution(phi)
    s.set_rhs(f)
    o.set_phi(phi)
    o.set_rhs(f)
    assert abs(s.residual_norm() - o.residual_norm()) <= 1e-13 * o.residual_norm()



# --------------------------------------------------------------------------
# config 5: solid mask, variable (Galerkin) coefficients
# --------------------------------------------------------------------------
def mask_pair(M, shape, solid, bc="channel", **kw):
    bt, bv = BCS[bc]
    s = M.Multigrid(shape, 1.0, bt, bv, **kw)
    s.set_mask(solid)
    okw = {k: v for k, v in kw.items()
           if k in ("min_coarse", "nu1", "nu2", "coarse_tol", "coarse_maxit")}
    o = oracle.Oracle(shape, 1.0, bt, bv, solid=solid, **okw)
    return s, o


def random_mask(shape, frac, seed):
    return (np.random.default_rng(seed).uniform(size=shape) < frac).astype(np.uint8)


@pytest.mark.parametrize("kind", ["random", "beam"])
def test_mask_operators_equal_oracle_galerkin(mg, kind):
    """The GPU's face-transmissibility coarse operators equal the oracle's
    generic R A P stencils exactly on every level."""
    shape = (32, 16, 32)
    solid = random_mask(shape, 0.2, 1) if kind == "random" else W.beam_mask(shape)
    s, o = mask_pair(mg, shape, solid, min_coarse=1)
    assert s.nlevels == o.nlevels
    for l in range(o.nlevels):
        assert np.array_equal(s.get_stencil(l), o.stencil(l)), l


def test_mask_steps_bitwise(mg):
    shape = (32, 16, 32)
    solid = random_mask(shape, 0.15, 2)
    s, o = mask_pair(mg, shape, solid, bc="mixed", min_coarse=2)
    rng = np.random.default_rng(3)
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


def test_config5_reduced_parity(mg):
    """Config-5 recipe at 1/16 scale: beam mask, electrodes, spheres outside
    the beam, V(3,3) to 1e-8."""
    w = W.cfg5(scale=16, n_spheres=60)
    s, o = mask_pair(mg, w.shape, w.solid, min_coarse=w.min_coarse, nu1=3, nu2=3)
    s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    o.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), o.rhs(0))
    rc, cg, hg = s.solve(w.tol, 80)
    so, co, ho = o.solve(w.tol, 80)
    assert rc == 0 and so == 0 and cg == co
    check_history(hg, ho)
    assert rel(s.get_solution(), o.phi()) <= 1e-10
    assert not s.get_solution()[w.solid.astype(bool)].any()


def test_mask_loopback_equals_single(mg):
    w = W.cfg5(scale=16, n_spheres=40)
    res = []
    for p in (1, 4):
        kw = dict(min_coarse=8, nu1=3, nu2=3, agglomerate_below=256)
        if p > 1:
            kw.update(nranks=p, halo="loopback")
        bt, bv = BCS["channel"]
        s = mg.Multigrid(w.shape, 1.0, bt, bv, **kw)
        s.set_mask(w.solid)
        s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
        r = [s.vcycle() for _ in range(4)]
        res.append((r, s.get_solution()))
    assert np.array_equal(res[0][1], res[1][1])
    assert np.allclose(res[0][0], res[1][0], rtol=1e-13, atol=0)


@pytest.mark.parametrize("scale", [4])
def test_config5_march_codes_parity(mg, scale):
    """Config-5 recipe at 1/4 scale (512x128x128): levels aligned with the beam
    use byte face codes and the TMA-marching kernels (nz/2 = 64); V(3,3) to
    1e-8 against the oracle."""
    w = W.cfg5(scale=scale, n_spheres=400)
    s, o = mask_pair(mg, w.shape, w.solid, min_coarse=w.min_coarse, nu1=3, nu2=3)
    s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    o.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    rc, cg, hg = s.solve(w.tol, 40)
    so, co, ho = o.solve(w.tol, 40)
    assert rc == 0 and so == 0 and cg == co
    check_history(hg, ho)
    assert rel(s.get_solution(), o.phi()) <= 1e-10
    for l in range(o.nlevels):
        assert np.array_equal(s.get_stencil(l), o.stencil(l)), l


@pytest.mark.parametrize("codes", [True, False])
def test_mask_march_equals_var_kernels(mg, codes):
    """Masked V-cycles: byte-code marching kernels == variable-coefficient
    direct kernels (MG_OFF_MARCH), bit for bit (random mask: coarse levels
    not aligned)."""
    shape = (32, 16, 256)
    solid = random_mask(shape, 0.1, 7) if not codes else W.beam_mask(shape)
    f = np.random.default_rng(14).uniform(-1, 1, shape)
    out = []
    for no_march in (False, True):
        bt, bv = BCS["channel"]
        s = mg.Multigrid(shape, 1.0, bt, bv, min_coarse=2, nu1=3, nu2=3,
                         disable=mg.MG_OFF_MARCH if no_march else 0)
        s.set_mask(solid)
        s.set_rhs(f)
        r = [s.vcycle() for _ in range(3)]
        out.append((r, s.get_solution()))
    assert np.array_equal(out[0][1], out[1][1])
    assert np.allclose(out[0][0], out[1][0], rtol=1e-13, atol=0)



def test_bc_patch_parity(mg):
    """mg_set_bc_patch (partial-length electrodes, paper-faithful config-5
    variant, reading c17): operators on every level, RHS, and a V(3,3) solve
    match the oracle; combined with the beam mask."""
    w = W.cfg5(scale=16, n_spheres=40)
    nx = w.shape[0]
    bt, bv = BCS["channel"]
    s = mg.Multigrid(w.shape, 1.0, bt, bv, min_coarse=8, nu1=3, nu2=3)
    o = oracle.Oracle(w.shape, 1.0, bt, bv, solid=w.solid, min_coarse=8,
                      nu1=3, nu2=3)
    s.set_mask(w.solid)
    for face in (2, 3):  # electrodes only on the first 3/4 of the channel
        s.set_bc_patch(face, 3 * nx // 4, nx, 0, w.shape[2], N, 0.0)
        o.set_bc_patch(face, 3 * nx // 4, nx, 0, w.shape[2], N, 0.0)
    for l in range(o.nlevels):
        assert np.array_equal(s.get_stencil(l), o.stencil(l)), l
    s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    o.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), o.rhs(0))
    rc, cg, hg = s.solve(1e-8, 60)
    so, co, ho = o.solve(1e-8, 60)
    assert rc == 0 and so == 0 and cg == co
    check_history(hg, ho)
    assert rel(s.get_solution(), o.phi()) <= 1e-10
    with pytest.raises(mg.MGError):
        s.set_bc_patch(2, 0, nx + 1, 0, 1, D, 0.0)



def face_centres(shape, h, face):
    """Physical points of the boundary faces of the face cells, (a, b) order."""
    nx, ny, nz = shape
    ax = face // 2
    ext = [nx, ny, nz]
    others = [d for d in range(3) if d != ax]
    a = (np.arange(ext[others[0]]) + 0.5) * h
    b = (np.arange(ext[others[1]]) + 0.5) * h
    A, B = np.meshgrid(a, b, indexing="ij")
    X = [None, None, None]
    X[others[0]], X[others[1]] = A, B
    X[ax] = np.full(A.shape, 0.0 if face % 2 == 0 else ext[ax] * h)
    return X


def test_face_values_parity(mg):
    """Per-cell boundary values (mg_set_face_values) on mixed faces: RHS
    adaptation bitwise, solve parity with the oracle."""
    shape = (32, 16, 24)
    bt, bv = BCS["mixed"]
    s, o = pair(mg, shape, 0.5, "mixed", min_coarse=2)
    rng = np.random.default_rng(21)
    for q in range(6):
        X = face_centres(shape, 0.5, q)
        vals = np.sin(X[0]) * np.cos(X[1]) + X[2] + rng.uniform(-0.1, 0.1, X[0].shape)
        s.set_face_values(q, vals)
        o.set_face_values(q, vals)
    f = rng.uniform(-1, 1, shape)
    s.set_rhs(f)
    o.set_rhs(f)
    assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), o.rhs(0))
    rc, cg, hg = s.solve(1e-10, 60)
    so, co, ho = o.solve(1e-10, 60)
    assert rc == 0 and so == 0 and cg == co
    check_history(hg, ho)
    assert rel(s.get_solution(), o.phi()) <= 1e-10


def sphere_potential(X, c, R, Q):
    """Eq.18 with eps = 1."""
    r = np.sqrt((X[0] - c[0]) ** 2 + (X[1] - c[1]) ** 2 + (X[2] - c[2]) ** 2)
    out = np.where(r >= R, Q / (4 * np.pi * np.maximum(r, 1e-300)),
                   Q / (4 * np.pi) / (2 * R) * (3 - (r / R) ** 2))
    return out


def test_charged_sphere_potential_table4(mg):
    """Charged-sphere validation (Table 4): analytic
    Dirichlet data (Eq.18) on every boundary face cell, the paper's naive
    volume mapping with subsampling; the relative potential error is "well
    below 2 % in the L2 norm for all sphere sizes" and shrinks with s_f
    (PAPER.md:1124-1127).  128^3, R = 6 at an off-centre position."""
    n, h, R, Q = 128, 1.0, 6.0, 1.0
    shape = (n, n, n)
    c = np.array([64.23, 63.81, 64.37])
    x = (np.arange(n) + 0.5) * h
    Xc = np.meshgrid(x, x, x, indexing="ij")
    exact = sphere_potential(Xc, c, R, Q)
    errs = {}
    for sf in (1, 3):
        s = mg.Multigrid(shape, h, [D] * 6, [0.0] * 6, min_coarse=8)
        for q in range(6):
            s.set_face_values(q, sphere_potential(face_centres(shape, h, q), c, R, Q))
        s.set_rhs_from_spheres(c[None, :], [R], [Q],
                               normalization=mg.MG_CHARGE_PER_VOLUME, subsample=sf)
        rc, cyc, hist = s.solve(1e-10, 40)
        assert rc == 0
        e = (s.get_solution() - exact) / exact
        errs[sf] = (float(np.sqrt(np.mean(e ** 2))), float(np.abs(e).max()))
        s.close()
    assert errs[1][0] < 0.02 and errs[3][0] < 0.02
    assert errs[3][0] < errs[1][0]
    assert errs[1][1] < 0.11 and errs[3][1] < errs[1][1]


# --------------------------------------------------------------------------
# Coulomb force (Eq.14) with the D3Q19 gradient (Eq.15)
# --------------------------------------------------------------------------
def force_spheres(shape, h):
    """Spheres inside, touching each wall / corner, straddling slab planes,
    partly outside the domain, and one smaller than a cell."""
    L = np.array(shape) * h
    c = [L * [0.31, 0.52, 0.47], L * [0.5, 0.5, 0.5], [0.9 * h, 0.6 * h, 0.5 * L[2]],
         [L[0] - 0.7 * h, L[1] - 1.1 * h, L[2] - 0.4 * h], L * [0.25, 0.9, 0.1],
         [0.5 * L[0] + 0.1 * h, -0.8 * h, 0.6 * L[2]], L * [0.75, 0.3, 0.66]]
    r = [3.3 * h, 4.0 * h, 2.2 * h, 1.9 * h, 2.6 * h, 2.0 * h, 0.3 * h]
    q = [1.0, -2.5, 0.7, 1.3, -0.4, 2.0, 0.9]
    return np.array(c), np.array(r), np.array(q)


@pytest.mark.parametrize("norm", [0, 1])
@pytest.mark.parametrize("sub", [1, 2, 3])
def test_coulomb_forces_parity(mg, norm, sub):
    """GPU forces == oracle forces on the same Phi (sums differ only in
    order: relative 1e-12)."""
    shape, h = (48, 40, 36), 0.5
    s, o = pair(mg, shape, h, "mixed", min_coarse=2)
    rng = np.random.default_rng(31 + sub)
    x = [(np.arange(n) + 0.5) * h for n in shape]
    X = np.meshgrid(*x, indexing="ij")
    phi = np.sin(0.3 * X[0]) * np.cos(0.2 * X[1]) + 0.1 * X[2] \
        + 0.05 * rng.uniform(-1, 1, shape)
    s.set_solution(phi)
    o.set_phi(phi)
    c, r, q = force_spheres(shape, h)
    Fg = s.coulomb_forces(c, r, q, normalization=norm, subsample=sub)
    Fo = o.coulomb_forces(c, r, q, normalization=norm, subsample=sub)
    assert Fg.shape == (len(r), 3)
    assert np.abs(Fo).max() > 0
    assert np.allclose(Fg, Fo, rtol=1e-12, atol=1e-12 * np.abs(Fo).max())


def test_coulomb_forces_config4_recipe(mg):
    """The time-stepping regime's force step (config-4 recipe: R = 6 at 5 %
    volume, s_F = 2) on a 128 x 96 x 96 box: mostly interior spheres, which
    take the staged-gradient path, plus wall-touching ones."""
    shape = (128, 96, 96)
    w = W.cfg4(P=1, n=96, seed=2)
    c, q = W.random_spheres(shape, 6.0, 120, seed=4)
    r = np.full(len(q), 6.0)
    s, o = pair(mg, shape, 1.0, "channel", min_coarse=4)
    s.set_rhs_from_spheres(c, r, q, subsample=2)
    for _ in range(4):
        s.vcycle()
    o.set_phi(s.get_solution())
    Fg = s.coulomb_forces(c, r, q, subsample=2)
    Fo = o.coulomb_forces(c, r, q, subsample=2)
    assert np.abs(Fo).max() > 0
    assert np.allclose(Fg, Fo, rtol=1e-12, atol=1e-12 * np.abs(Fo).max())
    del w


def test_coulomb_forces_after_solve_and_masked(mg):
    """Forces on a solved config-5 (masked) potential: solid cells carry no
    force and are not gradient neighbours (reading d6)."""
    w = W.cfg5(scale=16, n_spheres=40)
    s, o = mask_pair(mg, w.shape, w.solid, min_coarse=w.min_coarse, nu1=3, nu2=3)
    s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    o.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    s.solve(w.tol, 60)
    o.solve(w.tol, 60)
    # sample positions touching the beam as well as the given spheres
    c = np.concatenate([w.centers, [[w.shape[0] * 0.5, w.shape[1] * 0.5,
                                     w.shape[2] * 0.5]]])
    r = np.concatenate([w.radii, [5.0]])
    q = np.concatenate([w.charges, [1.0]])
    Fg = s.coulomb_forces(c, r, q)
    o_phi = o.phi()
    o.set_phi(s.get_solution())       # same Phi: isolate the force step
    Fo = o.coulomb_forces(c, r, q)
    assert np.allclose(Fg, Fo, rtol=1e-12, atol=1e-12 * np.abs(Fo).max())
    o.set_phi(o_phi)
    Fo2 = o.coulomb_forces(c, r, q)   # and the oracle's own solve
    assert np.allclose(Fg, Fo2, rtol=1e-7, atol=1e-7 * np.abs(Fo2).max())


@pytest.mark.parametrize("P", [2, 3])
def test_coulomb_forces_loopback_slabs(mg, P):
    """x-slab split: spheres straddling slab planes read the ghost planes;
    partial sums combined in slab order equal the single-slab result."""
    shape, h = (48, 40, 36), 0.5
    rng = np.random.default_rng(5)
    phi = rng.uniform(-1, 1, shape)
    c, r, q = force_spheres(shape, h)
    c = np.concatenate([c, [[8.0, 10.0, 9.0], [16.0, 10.0, 9.0]]])  # x = 16, 32 cells
    r = np.concatenate([r, [3.0, 2.5]])
    q = np.concatenate([q, [1.0, -1.0]])
    out = []
    for p in (1, P):
        kw = dict(min_coarse=2, agglomerate_below=64)
        if p > 1:
            kw.update(nranks=p, halo="loopback")
        bt, bv = BCS["mixed"]
        s = mg.Multigrid(shape, h, bt, bv, **kw)
        s.set_solution(phi)
        out.append(s.coulomb_forces(c, r, q, subsample=2))
        s.close()
    assert np.allclose(out[0], out[1], rtol=1e-13, atol=1e-13 * np.abs(out[0]).max())


@pytest.mark.parametrize("sub,radii", [
    (1, [7.7, 9.3, 11.2, 2.4]),   # uniform adjoint, direct force, scatter fallback, shell
    (2, [7.6, 9.4, 4.1]),
    (16, [2.2, 1.3]),             # counts up to 4096: no value table
])
def test_sphere_kernel_paths_large_spheres(mg, sub, radii):
    """The size-dependent paths of the sphere kernels against the oracle:
    boxes whose padded counts exceed the shell form's list / mask space (the
    uniform adjoint sum), exceed the padded count array (the direct D3Q19
    sum), exceed the scatter's shared count array (per-cell sub-centre
    tests), and sub-cell counts above the value table (s = 16).  f bitwise,
    forces to 1e-12 of the largest."""
    shape, h = (64, 56, 48), 1.0
    s, o = pair(mg, shape, h, "mixed", min_coarse=4)
    L = np.array(shape) * h
    rng = np.random.default_rng(len(radii) + sub)
    c = np.array([L * [0.3 + 0.4 * k / len(radii), 0.5, 0.5] + rng.uniform(-0.5, 0.5, 3)
                  for k in range(len(radii))])
    r = np.array(radii) * h
    q = rng.uniform(-2, 2, len(radii))
    s.set_rhs_from_spheres(c, r, q, subsample=sub)
    o.set_rhs_from_spheres(c, r, q, subsample=sub)
    assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), o.rhs(0))
    x = [(np.arange(n) + 0.5) * h for n in shape]
    X = np.meshgrid(*x, indexing="ij")
    phi = np.sin(0.11 * X[0]) * np.cos(0.07 * X[1]) + 0.02 * X[2] \
        + 0.01 * rng.uniform(-1, 1, shape)
    s.set_solution(phi)
    o.set_phi(phi)
    Fg = s.coulomb_forces(c, r, q, subsample=sub)
    Fo = o.coulomb_forces(c, r, q, subsample=sub)
    assert np.abs(Fo).max() > 0
    assert np.abs(Fg - Fo).max() <= 1e-12 * np.abs(Fo).max()
    s.close()


def test_coulomb_force_errors(mg):
    s, _ = pair(mg, (8, 8, 8), 1.0, "dirichlet")
    c, r, q = np.zeros((1, 3)) + 4.0, np.array([2.0]), np.array([1.0])
    assert s.coulomb_forces(np.zeros((0, 3)), [], []).shape == (0, 3)
    with pytest.raises(mg.MGError):
        s.coulomb_forces(c, r, q, subsample=0)
    with pytest.raises(mg.MGError):
        s.coulomb_forces(c, [-1.0], q)
    with pytest.raises(mg.MGError):
        s.coulomb_forces(c, r, q, normalization=7)


def worst_volume_position(shape, h, R, sub, n_try, seed):
    """Near-centre position with the largest |e_rV| for subsampling `sub`
    (the paper's placement)."""
    rng = np.random.default_rng(seed)
    best, pos = -1.0, None
    V = 4.0 / 3.0 * np.pi * R ** 3
    for _ in range(n_try):
        cpos = (np.array(shape) // 2 + rng.uniform(0, 1, 3)) * h
        n = oracle.sphere_cell_count(shape, h, cpos, R, sub)
        e = n * (h / sub) ** 3 / V - 1.0
        if abs(e) > best:
            best, pos, ev = abs(e), cpos, e
    return pos, ev


def test_coulomb_force_homogeneous_field_table5(mg):
    """Table 5 setup: charged sphere in a homogeneous
    field (Phi_W = 0, Phi_E = -10, homogeneous Neumann elsewhere), naive
    volume mapping.  The field part of the discrete solution is exactly
    linear and the D3Q19 gradient is exact on it, so with s_Phi = s_F the
    relative force error equals the volume-mapping error e_rV of the
    position ("e_rFC is equal to e_rVmax for same subsampling factors",
    PAPER.md:1142) up to the small image self-force; for unequal factors it
    "changes only slightly" (|e| within the paper's 7.1 % table maximum)."""
    n, h, Q = 128, 1.0, 1.0
    shape = (n, n, n)
    bt = [D, D, N, N, N, N]
    bv = [0.0, -10.0, 0.0, 0.0, 0.0, 0.0]
    F0 = Q * 10.0 / (n * h)
    for R in (4.0, 6.0):
        for sF in (1, 2, 3):
            c, ev = worst_volume_position(shape, h, R, sF, 300, int(10 * R) + sF)
            for sP in (1, 2, 3):
                s = mg.Multigrid(shape, h, bt, bv, min_coarse=8)
                s.set_rhs_from_spheres(c[None, :], [R], [Q],
                                       normalization=mg.MG_CHARGE_PER_VOLUME,
                                       subsample=sP)
                rc, _, _ = s.solve(1e-12, 60)
                assert rc == 0
                F = s.coulomb_forces(c[None, :], [R], [Q],
                                     normalization=mg.MG_CHARGE_PER_VOLUME,
                                     subsample=sF)[0]
                s.close()
                e = (F[0] - F0) / F0
                assert abs(F[1]) < 0.05 * F0 and abs(F[2]) < 0.05 * F0
                if sP == sF:
                    assert abs(e - ev) < 2e-3, (R, sF, e, ev)
                else:
                    assert abs(e) < 0.08, (R, sF, sP, e)


def test_get_solution_async_overlapped_steps(mg):
    """mg_get_solution_async: the copy-outs of five consecutive sphere steps
    (more than the three staging slots), each overlapping the next step's
    RHS and cycles, equal the synchronous copy-outs bit for bit; also into
    device memory."""
    import torch
    w = W.cfg2(seed=2, shape=(128, 32, 32), n_spheres=20)
    steps = []
    for k in range(5):
        c = w.centers + 0.3 * k
        steps.append((c, w.radii, w.charges))
    ref = []
    s, _ = pair(mg, w.shape, w.h, "channel", min_coarse=4)
    for c, r, q in steps:
        s.zero_solution()
        s.set_rhs_from_spheres(c, r, q)
        for _ in range(3):
            s.vcycle()
        ref.append(s.get_solution())
    s.close()
    s, _ = pair(mg, w.shape, w.h, "channel", min_coarse=4)
    outs = [torch.empty(w.shape, dtype=torch.float64).pin_memory() for _ in steps]
    for (c, r, q), o in zip(steps, outs):
        s.zero_solution()
        s.set_rhs_from_spheres(c, r, q)
        for _ in range(3):
            s.vcycle()
        s.get_solution_async(o)
    s.wait()
    for o, e in zip(outs, ref):
        assert np.array_equal(o.numpy(), e)
    od = torch.empty(w.shape, dtype=torch.float64, device="cuda")
    s.get_solution_async(od)
    s.wait()
    assert np.array_equal(od.cpu().numpy(), ref[-1])
    s.close()


def test_solve_async_pipelined_equals_sync(mg):
    """mg_solve_async pipelining independent solves (pinned host buffers,
    uploads / downloads on copy streams overlapping the cycles) gives the
    same Phi and final residual as the synchronous calls, bit for bit; also
    with device buffers and two contexts on two streams."""
    import torch
    shape = (64, 32, 128)
    bt, bv = BCS["mixed"]
    fs = [np.random.default_rng(40 + k).uniform(-1, 1, shape) for k in range(5)]
    ref = []
    s = mg.Multigrid(shape, 1.0, bt, bv, min_coarse=2)
    for f in fs:
        s.zero_solution()
        s.set_rhs(f)
        r = [s.vcycle() for _ in range(5)][-1]
        ref.append((r, s.get_solution()))
    s.close()
    # one context, host buffers: the pipeline
    s = mg.Multigrid(shape, 1.0, bt, bv, min_coarse=2)
    fh = [torch.from_numpy(f).pin_memory() for f in fs]
    out = [torch.empty(shape, dtype=torch.float64).pin_memory() for _ in fs]
    for k in range(len(fs)):
        s.solve_async(fh[k], out[k], 5)
    r_last = s.wait()
    assert r_last == ref[-1][0]
    for k in range(len(fs)):
        assert np.array_equal(out[k].numpy(), ref[k][1])
    # device buffers, one problem at a time
    fd = torch.from_numpy(fs[2]).cuda()
    od = torch.empty(shape, dtype=torch.float64, device="cuda")
    s.solve_async(fd, od, 5)
    assert s.wait() == ref[2][0]
    assert np.array_equal(od.cpu().numpy(), ref[2][1])
    s.close()
    # two contexts on two streams
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    ctx = [mg.Multigrid(shape, 1.0, bt, bv, min_coarse=2, stream=st) for st in streams]
    out2 = [torch.empty(shape, dtype=torch.float64).pin_memory() for _ in fs]
    res = [None] * len(fs)
    for k in range(len(fs)):
        if k >= 2:
            res[k - 2] = ctx[k % 2].wait()
        ctx[k % 2].solve_async(fh[k], out2[k], 5)
    for k in (len(fs) - 2, len(fs) - 1):
        res[k] = ctx[k % 2].wait()
    for k in range(len(fs)):
        assert res[k] == ref[k][0]
        assert np.array_equal(out2[k].numpy(), ref[k][1])


def test_solve_async_slot_reuse_device_or_null_output(mg):
    """Seven pipelined solves from pinned host RHS with device or NULL
    outputs: the staging slot of problem k is rewritten by the upload of
    problem k + 3 only after problem k's RHS conversion has read it (ADVICE
    r1: with a NULL / device phi_out nothing else orders the two).  Each
    device output and the last residual equal the synchronous solves."""
    import torch
    shape = (128, 64, 128)
    bt, bv = BCS["channel"]
    fs = [np.random.default_rng(60 + k).uniform(-1, 1, shape) for k in range(7)]
    ref = []
    s = mg.Multigrid(shape, 1.0, bt, bv, min_coarse=2)
    for f in fs:
        s.zero_solution()
        s.set_rhs(f)
        r = [s.vcycle() for _ in range(8)][-1]
        ref.append((r, s.get_solution()))
    s.close()
    s = mg.Multigrid(shape, 1.0, bt, bv, min_coarse=2)
    fh = [torch.from_numpy(f).pin_memory() for f in fs]
    outs = [torch.empty(shape, dtype=torch.float64, device="cuda")
            if k % 2 == 0 or k == len(fs) - 1 else None for k in range(len(fs))]
    for k in range(len(fs)):
        s.solve_async(fh[k], outs[k], 8)
    assert s.wait() == ref[-1][0]
    for k, o in enumerate(outs):
        if o is not None:
            assert np.array_equal(o.cpu().numpy(), ref[k][1]), k
    s.close()


def test_async_buffer_size_checked(mg):
    import torch
    s = mg.Multigrid((16, 16, 16), 1.0, [D] * 6, min_coarse=2)
    with pytest.raises(mg.MGError):
        s.solve_async(torch.zeros(16 * 16 * 15, dtype=torch.float64).pin_memory(),
                      None, 1)
    with pytest.raises(mg.MGError):
        s.get_solution_async(torch.zeros(10, dtype=torch.float64, device="cuda"))
    with pytest.raises(mg.MGError):
        s.get_field(1, mg.MG_FIELD_PHI, np.zeros((16, 16, 16)))
    s.close()


@pytest.mark.parametrize("P", [2, 4])
def test_loopback_overlapped_exchange_equals_serial(mg, P):
    """Multi-slab half-sweeps with the ghost exchange overlapped (boundary
    planes first, exchange on the communication stream while the interior
    planes are swept) give the serial-exchange iterates (MG_OFF_OVERLAP) bit
    for bit."""
    shape = (256, 64, 128)
    f = np.random.default_rng(44).uniform(-1, 1, shape)
    out = []
    for no_overlap in (False, True):
        s, _ = pair(mg, shape, 1.0, "channel", min_coarse=4, nranks=P,
                    halo="loopback", agglomerate_below=4096,
                    disable=mg.MG_OFF_OVERLAP if no_overlap else 0)
        s.set_rhs(f)
        r = [s.vcycle() for _ in range(3)]
        assert bool(s.cycle_paths & mg.MG_PATH_OVERLAP) == (not no_overlap)
        out.append((r, s.get_solution()))
        s.close()
    assert np.array_equal(out[0][1], out[1][1])
    assert out[0][0] == out[1][0]


@pytest.mark.parametrize("shape,bc,P", [((32, 24, 256), "mixed", 1),
                                        ((36, 20, 264), "channel", 1),
                                        ((66, 34, 20), "mixed", 1),
                                        ((64, 24, 256), "mixed", 2),
                                        ((128, 16, 136), "channel", 4)])
def test_split_cycle_end_norm(mg, shape, bc, P):
    """The cycle-end norm split between the last black half-sweep (black
    residuals) and a red-only residual pass equals the full residual pass on
    the same state to rounding (1e-13), and the iterates are those of the
    unsplit cycle (MG_OFF_SPLIT_NORM) bit for bit -- also on loopback slabs,
    where the red residuals read the black ghosts exchanged after the last
    black sweep."""
    f = np.random.default_rng(14).uniform(-1, 1, shape)
    out = []
    kw = dict(nranks=P, halo="loopback", agglomerate_below=512) if P > 1 else {}
    for split in (True, False):
        s, _ = pair(mg, shape, 1.0, bc, min_coarse=2,
                    disable=0 if split else mg.MG_OFF_SPLIT_NORM, **kw)
        s.set_rhs(f)
        s.vcycle()
        # nzh < 64 grids have no marching kernels, hence no split
        expect = split and shape[2] // 2 >= 64
        assert bool(s.cycle_paths & mg.MG_PATH_SPLIT_NORM) == expect
        s.set_rhs(f)
        s.zero_solution()
        r = []
        for _ in range(3):
            r.append(s.vcycle())
            full = s.residual_norm()
            assert abs(r[-1] - full) <= 1e-13 * full, (r[-1], full)
        out.append((r, s.get_solution()))
        s.close()
    assert np.array_equal(out[0][1], out[1][1])
    assert np.allclose(out[0][0], out[1][0], rtol=1e-13, atol=0)


@pytest.mark.parametrize("shape,bc,nu,P", [((128, 128, 128), "dirichlet0", (2, 2), 1),
                                          ((64, 32, 128), "mixed", (3, 3), 1),
                                          ((64, 64, 64), "channel", (1, 1), 1),
                                          ((64, 48, 96), "mixed", (0, 2), 1),
                                          ((64, 48, 96), "mixed", (2, 0), 1),
                                          ((128, 64, 64), "channel", (2, 2), 2)])
def test_tail_kernel_equals_per_step_launches(mg, shape, bc, nu, P):
    """The persistent tail kernel (levels <= 32^3 down to the CG and back in
    one cluster kernel) gives the per-step launch path's iterates and norms
    bit for bit (the same device functions; the CG's thread count is the
    standalone kernel's), and the oracle's to 1e-10."""
    f = np.random.default_rng(17).uniform(-1, 1, shape)
    out = []
    kw = dict(nranks=P, halo="emulate", agglomerate_below=4096) if P > 1 else {}
    for off in (0, mg.MG_OFF_TAIL):
        s, o = pair(mg, shape, 1.0, bc, min_coarse=2, nu1=nu[0], nu2=nu[1],
                    disable=off, **kw)
        s.set_rhs(f)
        r = [s.vcycle() for _ in range(4)]
        assert bool(s.cycle_paths & mg.MG_PATH_TAIL) == (off == 0), s.cycle_paths
        out.append((r, s.get_solution()))
        s.close()
    assert np.array_equal(out[0][1], out[1][1])
    assert out[0][0] == out[1][0]
    o.set_rhs(f)
    ho = [o.vcycle() for _ in range(4)]
    check_history(out[0][0], ho)
    assert rel(out[0][1], o.phi()) <= 1e-10


@pytest.mark.parametrize("bc", ["channel", "periodic"])
def test_sphere_rhs_sequence_clears_previous(mg, bc):
    """Successive sphere RHS calls on one context: f after each call equals
    the oracle's fresh RHS bitwise -- moved spheres, a shorter and a longer
    list, an intervening full-field set_rhs, different subsampling."""
    shape = (64, 48, 64)
    if bc == "periodic":
        bt, bv = W.periodic_channel_bc(1.0)
    else:
        bt, bv = BCS["channel"]
    s = mg.Multigrid(shape, 1.0, bt, bv, min_coarse=4)
    o = oracle.Oracle(shape, 1.0, bt, bv, min_coarse=4)
    L = np.array(shape, float)
    c0, q0 = W.random_spheres(L, 4.0, 30, seed=5)
    per = (True, False, True) if bc == "periodic" else (False, False, False)
    steps = [(c0, q0, 1), (W.move_spheres(c0, np.full(30, 4.0), L, 1, amplitude=2.0,
                                          periodic=per), q0, 2),
             (c0[:11], q0[:11], 1), ("field", None, None), (c0, q0, 3)]
    for c, q, sub in steps:
        if isinstance(c, str):
            f = np.random.default_rng(2).uniform(-1, 1, shape)
            s.set_rhs(f)
            o.set_rhs(f)
        else:
            R = np.full(len(q), 4.0)
            s.set_rhs_from_spheres(c, R, q, subsample=sub)
            o.set_rhs_from_spheres(c, R, q, subsample=sub)
        assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), o.rhs(0))
    s.close()


@pytest.mark.parametrize("shape,bc,nu,P", [((256, 128, 128), "dirichlet0", (2, 2), 1),
                                          ((128, 64, 136), "mixed", (3, 3), 1),
                                          ((256, 64, 128), "channel", (2, 2), 2),
                                          ((256, 64, 128), "channel", (1, 2), 4)])
def test_restriction_with_first_red_sweep_equals_separate(mg, shape, bc, nu, P):
    """The restriction that also performs the next level's first red
    half-sweep from Phi = 0 (Phi_red = f w / d from the restricted f) gives
    the separate kernels' iterates and norms bit for bit (MG_OFF_RED0), also
    on EMULATE slabs (the red ghost exchange after the restriction)."""
    f = np.random.default_rng(19).uniform(-1, 1, shape)
    kw = dict(nranks=P, halo="emulate", agglomerate_below=4096) if P > 1 else {}
    out = []
    for off in (0, mg.MG_OFF_RED0):
        s, _ = pair(mg, shape, 1.0, bc, min_coarse=2, nu1=nu[0], nu2=nu[1],
                    disable=off, **kw)
        s.set_rhs(f)
        r = [s.vcycle() for _ in range(3)]
        assert bool(s.cycle_paths & mg.MG_PATH_RED0) == (off == 0)
        out.append((r, s.get_solution()))
        s.close()
    assert np.array_equal(out[0][1], out[1][1])
    assert out[0][0] == out[1][0]
