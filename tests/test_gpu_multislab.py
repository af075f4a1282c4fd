"""Row a4 (halo exchange) and a6 (agglomeration) against the ORACLE.

The x-slab decomposition (P:570-571 ghost exchange per level,
P:622-624, P:692-693 periodic arrangement) runs P slabs in one process on
one GPU, with two halo backends: LOOPBACK (ghost planes by device copies,
one shared agglomerated hierarchy) and EMULATE (NCCL's data layout: one
copy of the agglomerated levels per rank, the halo schedule mg_halo_schedule
matched message by message and the in-place all-gathers of the restricted
RHS, of the coarse operator records and of the norm executed as device
copies with NCCL's indexing).  Each run here is compared with the single-domain
CPU oracle -- not with the 1-slab CUDA run -- at sizes where level 0 takes
the TMA-marching kernels (nz/2 >= 64) and the coarse levels are agglomerated
(local cells < 64^3): Phi rel-L2 <= 1e-10, equal cycle counts and the
residual-history clause of tests/test_gpu_parity.py.
"""
import functools

import numpy as np
import pytest

import oracle
from paper_1410_6609_b200 import workloads as W

pytestmark = pytest.mark.gpu

BACKENDS = ["loopback", "emulate"]


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


def check_history(hg, ho):
    assert len(hg) == len(ho)
    r0 = ho[0]
    for a, b in zip(hg, ho):
        assert abs(a - b) <= 1e-8 * b + 1e-15 * r0, (a, b)


def _channel():
    return W.cfg2(seed=3, shape=(256, 64, 128), n_spheres=60)


def _periodic():
    w = W.cfg2(seed=4, shape=(256, 32, 128), n_spheres=40)
    w.bc_type, w.bc_value = W.periodic_channel_bc(1.0)
    return w


def _masked():
    return W.cfg5(scale=4, n_spheres=300)


CASES = {"channel": _channel, "periodic": _periodic, "masked": _masked}


@functools.lru_cache(maxsize=None)
def oracle_solve(case):
    w = CASES[case]()
    o = oracle.Oracle(w.shape, w.h, w.bc_type, w.bc_value, solid=w.solid,
                      min_coarse=w.min_coarse, nu1=w.nu1, nu2=w.nu2)
    o.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    st, cyc, hist = o.solve(w.tol, 40)
    assert st == 0
    return o.phi(), cyc, hist, o.rhs(0)


@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("case", sorted(CASES))
def test_slabs_solve_equals_oracle(mg, case, P, backend):
    w = CASES[case]()
    phi_o, cyc_o, hist_o, rhs_o = oracle_solve(case)
    s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=w.min_coarse,
                     nu1=w.nu1, nu2=w.nu2, nranks=P, halo=backend)
    dims, lnx, agg = mg.plan(w.shape, min_coarse=w.min_coarse, nranks=P, halo=backend)
    assert 1 <= agg < len(dims) - 1, "the case must agglomerate"
    if w.solid is not None:
        s.set_mask(w.solid)
    s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), rhs_o)
    rc, cyc, hist = s.solve(w.tol, 40)
    assert rc == 0 and cyc == cyc_o
    assert s.cycle_paths & mg.MG_PATH_MARCH
    check_history(hist, hist_o)
    assert rel(s.get_solution(), phi_o) <= 1e-10
    s.close()


@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("P", [2, 4])
def test_slabs_steps_bitwise_vs_oracle(mg, P, backend):
    """One level-0 half-sweep pair, the residual + restriction into the
    first agglomerated level, and the prolongation back, on slabs, against
    the oracle's steps bit for bit (the ghost planes the halo delivered are
    exactly the neighbours' cells)."""
    shape = (128, 32, 128)
    bt, bv = W.channel_bc(1.0)
    s = mg.Multigrid(shape, 1.0, bt, bv, min_coarse=4, nranks=P, halo=backend)
    o = oracle.Oracle(shape, 1.0, bt, bv, min_coarse=4)
    rng = np.random.default_rng(5)
    phi = rng.uniform(-1, 1, shape)
    f = rng.uniform(-1, 1, shape)
    s.set_solution(phi)
    s.set_rhs(f)
    o.set_phi(phi)
    o.set_rhs(f)
    for c in (0, 1, 0, 1):
        s.smooth_half(0, c)
        o.smooth_half(0, c)
    assert np.array_equal(s.get_solution(), o.phi())
    s.residual_restrict(0)
    o.restrict_residual(0)
    assert np.array_equal(s.get_field(1, mg.MG_FIELD_RHS), o.rhs(1))
    e = rng.uniform(-1, 1, o.dims(1))
    s.set_field(1, mg.MG_FIELD_PHI, e)
    o.set_phi(e, 1)
    s.prolong_correct(0)
    o.prolong_correct(0, 2.0)
    assert np.array_equal(s.get_solution(), o.phi())
    s.close()


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("kind", ["box", "periodic", "permittivity", "masked"])
def test_emulate_equals_loopback(mg, P, kind):
    """The NCCL layout (EMULATE) and the shared-copy layout (LOOPBACK) give
    the same iterates bit for bit and the same cycle norms (both sum the
    norm per rank, then in rank order)."""
    shape = (128, 32, 128)
    bt, bv = W.channel_bc(1.0)
    if kind == "periodic":
        bt, bv = W.periodic_channel_bc(1.0)
    f = np.random.default_rng(8).uniform(-1, 1, shape)
    out = []
    for backend in ("loopback", "emulate"):
        s = mg.Multigrid(shape, 1.0, bt, bv, min_coarse=4, nranks=P, halo=backend,
                         agglomerate_below=2048)
        if kind == "permittivity":
            eps = np.where(np.arange(shape[1])[None, :, None] < 16, 1.0, 78.5) \
                * np.ones(shape)
            s.set_permittivity(eps)
        if kind == "masked":
            s.set_mask(W.beam_mask(shape))
        s.set_rhs(f)
        r = [s.vcycle() for _ in range(3)]
        out.append((r, s.get_solution(), s.get_field(s.nlevels - 1, mg.MG_FIELD_PHI)))
        s.close()
    assert np.array_equal(out[0][1], out[1][1])
    assert np.array_equal(out[0][2], out[1][2])
    assert out[0][0] == out[1][0]


@pytest.mark.parametrize("halo", BACKENDS)
@pytest.mark.parametrize("nu", [(1, 0), (2, 0), (0, 1)])
def test_no_post_or_pre_smoothing_on_slabs(mg, halo, nu):
    """V(nu1, 0) on slabs: with no post-smoothing after the prolongation, the
    cycle-end norm reads the corrected red ghost planes -- the prolongation
    exchanges both colours (a case the deep randomised run found: (8, 4, 64),
    z periodic, V(1,0), 2 slabs); V(0, 1) for symmetry."""
    shape = (16, 8, 128)
    bt, bv = [0, 0, 0, 0, 2, 2], [0.0] * 6
    nu1, nu2 = nu
    kw = dict(min_coarse=2, nu1=nu1, nu2=nu2)
    f = np.random.default_rng(0).uniform(-1, 1, shape)
    o = oracle.Oracle(shape, 1.0, bt, bv, **kw)
    o.set_rhs(f)
    ho = [o.residual_norm()] + [o.vcycle() for _ in range(3)]
    s = mg.Multigrid(shape, 1.0, bt, bv, nranks=2, halo=halo, agglomerate_below=512, **kw)
    s.set_rhs(f)
    hg = [s.residual_norm()] + [s.vcycle() for _ in range(3)]
    check_history(hg, ho)
    assert rel(s.get_solution(), o.phi()) <= 1e-10
    s.close()
