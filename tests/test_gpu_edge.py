"""Edge and degenerate cases of the CUDA path against the oracle and the
mathematics (SURVEY 8(c) "whole solve" pins, `S:492`):

* an empty sphere list: f is exactly the BC adaptation (bitwise the oracle's),
  and with homogeneous BCs exactly 0 -- mg_solve returns at once (r_0 = 0)
  and a V-cycle keeps Phi = 0 bit for bit;
* linearity with a power-of-two factor: f -> 2f gives Phi -> 2 Phi bitwise
  (every per-cell operation commutes with exact scaling by 2);
* argument errors of the sphere mapping (R <= 0, subsample outside 1..16)
  leave f untouched; a sphere that covers no cell centre is reported;
* the smallest hierarchy (2 x 2 x 2, one level: CG only) and a single-level
  solve match the oracle.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

D, N = 0, 1


@pytest.fixture(scope="module")
def mg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1410_6609_b200 import _build
    _build.build()
    from paper_1410_6609_b200 import mg as M
    return M


def test_empty_sphere_list_homogeneous(mg):
    shape = (32, 16, 128)
    s = mg.Multigrid(shape, 1.0, [D] * 6, min_coarse=2)
    s.set_rhs_from_spheres(np.zeros((0, 3)), [], [])
    f = s.get_field(0, mg.MG_FIELD_RHS)
    assert not f.any()
    rc, cyc, hist = s.solve(1e-8, 10)
    assert rc == 0 and cyc == 0 and hist[0] == 0.0
    r = s.vcycle()
    assert r == 0.0
    assert not s.get_solution().any()
    s.close()


@pytest.mark.parametrize("shape", [(32, 16, 128), (12, 10, 6)])
def test_empty_sphere_list_bc_terms_only(mg, shape):
    bt = [N, D, N, D, N, D]
    bv = [0.25, 1.0, -0.5, -1.0, 2.0, 0.0]
    s = mg.Multigrid(shape, 0.5, bt, bv, min_coarse=2)
    o = oracle.Oracle(shape, 0.5, bt, bv, min_coarse=2)
    s.set_rhs_from_spheres(np.zeros((0, 3)), [], [])
    o.set_rhs_from_spheres(np.zeros((0, 3)), [], [])
    fg = s.get_field(0, mg.MG_FIELD_RHS)
    assert np.array_equal(fg, o.rhs(0))
    assert fg.any()
    r = [s.residual_norm()] + [s.vcycle() for _ in range(3)]
    ro = [o.residual_norm()] + [o.vcycle() for _ in range(3)]
    for a, b in zip(r, ro):  # reading c21's clause
        assert abs(a - b) <= 1e-8 * b + 1e-14 * ro[0]
    s.close()


def test_power_of_two_linearity(mg):
    shape = (34, 12, 256)
    f = np.random.default_rng(8).uniform(-1, 1, shape)
    out = []
    for scale in (1.0, 2.0):
        s = mg.Multigrid(shape, 0.25, [D] * 6, min_coarse=2)
        s.set_rhs(scale * f)
        r = [s.vcycle() for _ in range(3)]
        out.append((r, s.get_solution()))
        s.close()
    assert np.array_equal(2.0 * out[0][1], out[1][1])
    for a, b in zip(out[0][0], out[1][0]):
        assert abs(2.0 * a - b) <= 1e-13 * b


def test_sphere_argument_errors_leave_rhs(mg):
    shape = (16, 16, 16)
    s = mg.Multigrid(shape, 1.0, [D] * 6, min_coarse=2)
    rng = np.random.default_rng(2)
    f = rng.uniform(-1, 1, shape)
    s.set_rhs(f)
    f0 = s.get_field(0, mg.MG_FIELD_RHS)
    bad = [
        (np.array([[8.0, 8.0, 8.0]]), [0.0], [1.0], 1),     # R = 0
        (np.array([[8.0, 8.0, 8.0]]), [-2.0], [1.0], 1),    # R < 0
        (np.array([[8.0, 8.0, 8.0]]), [3.0], [1.0], 0),     # subsample 0
        (np.array([[8.0, 8.0, 8.0]]), [3.0], [1.0], 17),    # subsample 17
    ]
    for c, R, Q, sub in bad:
        with pytest.raises(mg.MGError) as e:
            s.set_rhs_from_spheres(c, R, Q, subsample=sub)
        assert e.value.code == mg.MG_ERR_ARG
        assert np.array_equal(s.get_field(0, mg.MG_FIELD_RHS), f0)
    # a sphere that covers no cell centre: found by the mapping itself
    with pytest.raises(mg.MGError) as e:
        s.set_rhs_from_spheres(np.array([[8.0, 8.0, 8.0]]), [0.2], [1.0])
    assert e.value.code == mg.MG_ERR_ARG
    s.close()


@pytest.mark.parametrize("shape,mc", [((2, 2, 2), 4), ((6, 6, 6), 8)])
def test_single_level_hierarchy(mg, shape, mc):
    """One level: the cycle is the CG solve of the whole grid."""
    bt = [D, N, D, N, D, N]
    bv = [1.0, 0.5, -1.0, 0.0, 0.25, 0.0]
    f = np.random.default_rng(3).uniform(-1, 1, shape)
    s = mg.Multigrid(shape, 1.0, bt, bv, min_coarse=mc)
    o = oracle.Oracle(shape, 1.0, bt, bv, min_coarse=mc)
    assert s.nlevels == o.nlevels == 1
    s.set_rhs(f)
    o.set_rhs(f)
    r, ro = s.vcycle(), o.vcycle()
    phi, po = s.get_solution(), o.phi()
    assert np.linalg.norm(phi - po) <= 1e-10 * np.linalg.norm(po)
    assert r <= 1e-10 * np.linalg.norm(f) and ro <= 1e-10 * np.linalg.norm(f)
    s.close()


def test_sphere_and_force_buffers_regrow(mg):
    """Growing sphere lists between force evaluations (the library caches
    its sphere and force buffers): forces equal those of a fresh context."""
    from paper_1410_6609_b200 import workloads as W
    shape = (64, 32, 32)
    res = []
    for fresh in (False, True):
        s = mg.Multigrid(shape, 1.0, [N, N, D, D, N, N],
                         [0.0, 0.0, 0.0, 1.0, 0.0, 0.0], min_coarse=4)
        F = None
        for k, n in enumerate((2, 5, 11)):
            c, q = W.random_spheres(shape, 3.0, n, seed=k)
            if fresh and k < 2:
                continue
            s.set_rhs_from_spheres(c, [3.0] * n, q)
            s.zero_solution()
            for _ in range(3):
                s.vcycle()
            F = s.coulomb_forces(c, [3.0] * n, q)
        res.append(F)
        s.close()
    assert res[0].shape == (11, 3)
    assert np.array_equal(res[0], res[1])
