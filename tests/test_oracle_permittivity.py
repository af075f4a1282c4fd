"""Pins of the oracle's variable-permittivity operator:
-div(eps grad Phi) = rho with eps constant per cell, harmonic face means
(reading d10), Galerkin coarse operators ("extensible for
discontinuous dielectricity coefficients ... by Galerkin coarsening";
P:1534 "jumping dielectricity coefficients").

Expected values: an independent flux-form dense operator (tests/dense.py),
the exact solution of a layered medium (series conductances), scaling
identities and the dense V-cycle matrix -- never the oracle itself or CUDA.
"""
import numpy as np
import pytest

import dense
import oracle

D, N, P = oracle.DIRICHLET, oracle.NEUMANN, oracle.PERIODIC

BCS = [([D] * 6, [1.0, -2.0, 0.5, 3.0, -1.0, 2.0]),
       ([N, N, D, D, N, N], [0.3, 0.0, 0.0, 1.0, -0.2, 0.0]),
       ([D, N, P, P, N, D], [1.0, 0.3, 0.0, 0.0, -0.2, 2.0])]


def jumpy(shape, seed, ratio=80.0):
    """Cell permittivity with jumps: two materials (1 and `ratio`, e.g. water
    78.5 vs a particle ~1) in random blobs plus a smooth variation."""
    rng = np.random.default_rng(seed)
    base = np.where(rng.uniform(size=shape) < 0.3, ratio, 1.0)
    x = np.indices(shape).sum(0)
    return base * (1.0 + 0.25 * np.sin(0.7 * x))


@pytest.mark.parametrize("bc", BCS)
def test_eps_operator_equals_flux_form(bc):
    """Finest operator == the flux-form dense matrix (harmonic means, ghost
    cells with eps_c) to rounding; RHS shift likewise."""
    bt, bv = bc
    shape, h = (6, 4, 8), 0.5
    eps = jumpy(shape, 1)
    o = oracle.Oracle(shape, h, bt, bv, min_coarse=1)
    o.set_permittivity(eps)
    per = tuple(bt[2 * a] == P for a in range(3))
    A = dense.stencil_to_dense(o.stencil(0), per)
    Af, b = dense.flux_operator_eps(shape, h, bt, eps, bv)
    assert np.allclose(A, Af, rtol=1e-15, atol=1e-13 * np.abs(Af).max())
    o.set_rhs(np.zeros(shape))
    assert np.allclose(o.rhs().reshape(-1), b, rtol=1e-15, atol=1e-13 * np.abs(b).max())
    assert np.array_equal(A, A.T)   # harmonic mean is symmetric bit for bit


@pytest.mark.parametrize("bc", BCS)
def test_eps_dense_direct_solve(bc):
    bt, bv = bc
    shape, h = (8, 8, 8), 0.5
    eps = jumpy(shape, 2)
    f = np.random.default_rng(3).uniform(-1, 1, shape)
    o = oracle.Oracle(shape, h, bt, bv, min_coarse=2, coarse_tol=1e-15,
                      coarse_maxit=5000, nu1=3, nu2=3)
    o.set_permittivity(eps)
    o.set_rhs(f)
    st, cyc, _ = o.solve(1e-13, 400)
    assert st == 0
    Af, b = dense.flux_operator_eps(shape, h, bt, eps, bv)
    u = np.linalg.solve(Af, f.reshape(-1) + b).reshape(shape)
    assert np.linalg.norm(o.phi() - u) / np.linalg.norm(u) < 1e-11


def test_eps_layered_medium_exact():
    """Layers of constant eps along x, Dirichlet 0 / 1 on the x faces,
    homogeneous Neumann elsewhere, no charge: with harmonic face means the
    discrete potential at the cell centres is the exact continuous one --
    piecewise linear, slope ~ 1/eps (series of half-cell resistances
    h / (2 eps))."""
    nx, h = 32, 1.0 / 32
    shape = (nx, 8, 8)
    layer = np.where(np.arange(nx) < 12, 1.0, np.where(np.arange(nx) < 20, 80.0, 5.0))
    eps = np.broadcast_to(layer[:, None, None], shape).copy()
    bt = [D, D, N, N, N, N]
    o = oracle.Oracle(shape, h, bt, [0.0, 1.0, 0, 0, 0, 0], min_coarse=2,
                      nu1=3, nu2=3, coarse_tol=1e-14)
    o.set_permittivity(eps)
    o.set_rhs(np.zeros(shape))
    st, _, _ = o.solve(1e-14, 300)
    assert st == 0
    # continuous solution: resistance from x = 0 to the centre of cell i
    half = h / (2 * layer)
    R_centre = np.cumsum(np.concatenate([[0.0], 2 * half[:-1]])) + half
    R_tot = 2 * half.sum()
    exact = R_centre / R_tot
    phi = o.phi()
    assert np.abs(phi - exact[:, None, None]).max() < 1e-11


def test_eps_constant_reduces_to_poisson():
    """eps = 1 gives the constant-coefficient operator bit for bit (power-of-
    two h); eps = 4 scales the operator by 4 exactly and Phi by 1/4 after
    the same cycles (homogeneous BCs)."""
    shape, h = (16, 8, 8), 0.25
    bt, bv = [D, N, D, D, N, N], [0.0] * 6
    f = np.random.default_rng(5).uniform(-1, 1, shape)
    o0 = oracle.Oracle(shape, h, bt, bv, min_coarse=2)
    o1 = oracle.Oracle(shape, h, bt, bv, min_coarse=2)
    o1.set_permittivity(np.ones(shape))
    for l in range(o0.nlevels):
        assert np.array_equal(o0.stencil(l), o1.stencil(l))
    o4 = oracle.Oracle(shape, h, bt, bv, min_coarse=2)
    o4.set_permittivity(np.full(shape, 4.0))
    for l in range(o0.nlevels):
        assert np.array_equal(o4.stencil(l), 4.0 * o0.stencil(l))
    o0.set_rhs(f)
    o4.set_rhs(f)
    for _ in range(4):
        o0.vcycle()
        o4.vcycle()
    assert np.array_equal(o4.phi(), o0.phi() / 4.0)


def test_eps_galerkin_equals_dense_RAP():
    """Coarse operators = dense R A P (averaging R, injection P) of the
    flux-form fine operator, to rounding (the oracle sums in a fixed order);
    still symmetric 7-point operators."""
    shape, h = (8, 8, 16), 0.5
    bt = [N, N, D, D, N, N]
    eps = jumpy(shape, 7)
    o = oracle.Oracle(shape, h, bt, [0.0] * 6, min_coarse=1)
    o.set_permittivity(eps)
    A, _ = dense.flux_operator_eps(shape, h, bt, eps)
    for l in range(o.nlevels - 1):
        Pm = dense.injection_P(o.dims(l))
        A = (Pm.T / 8.0) @ A @ Pm
        Ao = dense.stencil_to_dense(o.stencil(l + 1))
        assert np.allclose(Ao, A, rtol=1e-14, atol=1e-14 * np.abs(A).max())
        assert np.allclose(Ao, Ao.T, rtol=1e-15, atol=1e-15 * np.abs(A).max())


def test_eps_vcycle_equals_dense_iteration_matrix():
    shape = (16, 8, 8)
    bt = [D, D, N, N, D, N]
    eps = jumpy(shape, 9, ratio=20.0)
    o = oracle.Oracle(shape, 1.0, bt, [0.0] * 6, min_coarse=2,
                      coarse_tol=1e-15, coarse_maxit=5000)
    o.set_permittivity(eps)
    A0, _ = dense.flux_operator_eps(shape, 1.0, bt, eps)
    M, _ = dense.vcycle_matrices([o.dims(l) for l in range(o.nlevels)], 1.0, bt,
                                 2, 2, 2.0, A0=A0)
    x = np.random.default_rng(10).uniform(-1, 1, shape)
    o.set_rhs(np.zeros(shape))
    o.set_phi(x)
    o.vcycle()
    y = M @ x.reshape(-1)
    assert np.linalg.norm(o.phi().reshape(-1) - y) <= 1e-11 * np.linalg.norm(y)


def test_eps_rejects_nonpositive():
    o = oracle.Oracle((4, 4, 4), 1.0, [D] * 6)
    e = np.ones((4, 4, 4))
    e[1, 2, 3] = 0.0
    with pytest.raises(ValueError):
        o.set_permittivity(e)
