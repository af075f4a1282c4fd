"""Pins of the oracle's periodic boundary conditions.

PAPER.md:441-443: "Periodic BCs cyclically extend the domain.  They are
realised algorithmically by accessing unknowns in cells at opposite sides of
the domain."  Expected values come from closed forms (discrete eigenvectors of
the circulant operator), from dense / spectral constructions in tests/dense.py
(ghost layer = the opposite side's cells, independent of the oracle's folded
stencil), from the translation symmetry of the periodic problem, and from
brute-force minimum-image sphere coverage -- never from the oracle or the
CUDA path.
"""
import math

import numpy as np
import pytest

import dense
import oracle

D, N, P = oracle.DIRICHLET, oracle.NEUMANN, oracle.PERIODIC

PER_COMBOS = [
    ([P, P, P, P, D, D], [0.0, 0.0, 0.0, 0.0, 0.0, 1.0]),     # x, y periodic
    ([P, P, D, N, P, P], [0.0, 0.0, 0.5, -0.25, 0.0, 0.0]),   # x, z periodic
    ([D, N, P, P, N, D], [1.0, 0.3, 0.0, 0.0, -0.2, 2.0]),    # y periodic
    ([P, P, P, P, D, N], [0.0, 0.0, 0.0, 0.0, -1.0, 0.5]),    # one Dirichlet face
]


def _per(bt):
    return tuple(bt[2 * a] == P for a in range(3))


@pytest.mark.parametrize("bc", PER_COMBOS)
def test_periodic_dense_direct_solve(bc):
    """Converged MG = dense direct solve of the ghost-cell operator whose
    periodic ghosts are the opposite side's cells."""
    bt, bv = bc
    shape, h = (8, 8, 8), 0.5
    rng = np.random.default_rng(3)
    f = rng.uniform(-1, 1, shape)
    o = oracle.Oracle(shape, h, bt, bv, min_coarse=2, coarse_tol=1e-15,
                      coarse_maxit=4000)
    o.set_rhs(f)
    st, _, _ = o.solve(1e-14, 200)
    assert st == 0
    A = dense.dense_operator(shape, h, bt)
    b = (f + dense.bc_rhs_shift(shape, h, bt, bv)).reshape(-1)
    u = np.linalg.solve(A, b).reshape(shape)
    assert np.linalg.norm(o.phi() - u) / np.linalg.norm(u) < 1e-12


def test_periodic_kronecker_exact_solve():
    """64x32x16 with x, y periodic, z Dirichlet: fast diagonalisation of the
    circulant (x, y) and Dirichlet (z) 1D operators is the exact solution."""
    bt = [P, P, P, P, D, D]
    shape, h = (64, 32, 16), 1.0 / 16
    f = np.random.default_rng(8).uniform(-1, 1, shape)
    o = oracle.Oracle(shape, h, bt, [0.0] * 6, min_coarse=2)
    o.set_rhs(f)
    st, _, _ = o.solve(1e-13, 100)
    assert st == 0
    u = dense.kron_solve(f, h, bt)
    assert np.linalg.norm(o.phi() - u) / np.linalg.norm(u) < 1e-11


def _lam(h):
    """Eigenvalue of sin(2 pi x) sin(2 pi y) sin(pi z) at cell centres for the
    operator periodic in x, y (circulant: 4 sin^2(pi h)/h^2 per axis) and
    Dirichlet in z (ghost = -Phi_1: 4 sin^2(pi h/2)/h^2)."""
    return (8.0 * math.sin(math.pi * h) ** 2
            + 4.0 * math.sin(math.pi * h / 2) ** 2) / (h * h)


@pytest.mark.parametrize("n", [16, 32])
def test_periodic_closed_form_and_order(n):
    """Manufactured solution u = sin(2 pi x) sin(2 pi y) sin(pi z), f = 9 pi^2
    u: the discrete solution is exactly (9 pi^2 / lambda_h) u, an O(h^2)
    error (Eq.13)."""
    h = 1.0 / n
    x = (np.arange(n) + 0.5) * h
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    u = np.sin(2 * np.pi * X) * np.sin(2 * np.pi * Y) * np.sin(np.pi * Z)
    o = oracle.Oracle((n, n, n), h, [P, P, P, P, D, D], [0.0] * 6,
                      min_coarse=4, coarse_tol=1e-14)
    o.set_rhs(9 * np.pi ** 2 * u)
    for _ in range(14):
        o.vcycle()
    c = 9 * np.pi ** 2 / _lam(h)
    assert np.abs(o.phi() - c * u).max() < 1e-12
    e16 = 9 * np.pi ** 2 / _lam(1 / 16) - 1
    e32 = 9 * np.pi ** 2 / _lam(1 / 32) - 1
    assert abs(e16 / e32 - 4.0) < 0.03  # 4.02: asymptotic O(h^2)


@pytest.mark.parametrize("bc", PER_COMBOS[:3])
def test_periodic_galerkin_equals_dense_RAP_and_closed_form(bc):
    """A_c = R A P on a periodic grid: dense triple product ==
    the oracle's coarse stencils (wrapping neighbours) == 2^{-l} times the
    level's own ghost-cell operator, down to a coarse grid of width 2 along a
    periodic axis (x- and x+ then name the same neighbour)."""
    bt, _ = bc
    shape, h = (8, 8, 8), 0.5
    per = _per(bt)
    o = oracle.Oracle(shape, h, bt, [0.0] * 6, min_coarse=1)
    assert o.nlevels == 3 and o.dims(2) == (2, 2, 2)
    A = dense.stencil_to_dense(o.stencil(0), per)
    assert np.array_equal(A, dense.dense_operator(shape, h, bt))
    for l in range(o.nlevels - 1):
        Pm = dense.injection_P(o.dims(l))
        Ac = (Pm.T / 8.0) @ A @ Pm
        Ao = dense.stencil_to_dense(o.stencil(l + 1), per)
        assert np.array_equal(Ac, Ao)
        S = dense.dense_operator(o.dims(l + 1), h, bt)
        assert np.array_equal(Ao, S * 2.0 ** -(l + 1))
        A = Ao


@pytest.mark.parametrize("shape,mc,bc", [
    ((8, 8, 8), 4, PER_COMBOS[0]),
    ((16, 8, 8), 2, PER_COMBOS[1]),
    ((8, 8, 16), 2, PER_COMBOS[2]),
])
def test_periodic_vcycle_equals_dense_iteration_matrix(shape, mc, bc):
    """One V(2,2)-cycle with f = 0 maps phi to M phi, M the dense V-cycle
    error propagator built on the periodic ghost-cell operators."""
    bt = bc[0]
    o = oracle.Oracle(shape, 1.0, bt, [0.0] * 6, min_coarse=mc,
                      coarse_tol=1e-15, coarse_maxit=4000)
    shapes = [o.dims(l) for l in range(o.nlevels)]
    M, _ = dense.vcycle_matrices(shapes, 1.0, bt, 2, 2, 2.0)
    x = np.random.default_rng(12).uniform(-1, 1, shape)
    o.set_rhs(np.zeros(shape))
    o.set_phi(x)
    o.vcycle()
    y = M @ x.reshape(-1)
    assert np.linalg.norm(o.phi().reshape(-1) - y) <= 1e-12 * np.linalg.norm(y)


def test_periodic_shift_equivariance():
    """Translation symmetry of the periodic problem: shifting f by a multiple
    of 2^L cells along a periodic axis (colours and parents preserved on
    every level) shifts Phi after the same cycles; only the CG dot-product
    order differs, hence 1e-12 instead of bitwise."""
    shape = (32, 16, 16)
    bt = [P, P, P, P, D, D]
    f = np.random.default_rng(4).uniform(-1, 1, shape)
    res = []
    for sx, sy in ((0, 0), (8, 0), (16, 8)):
        o = oracle.Oracle(shape, 1.0, bt, [0.0] * 6, min_coarse=4)
        assert o.nlevels == 3
        o.set_rhs(np.roll(np.roll(f, sx, 0), sy, 1))
        for _ in range(3):
            o.vcycle()
        res.append(np.roll(np.roll(o.phi(), -sx, 0), -sy, 1))
    for r in res[1:]:
        assert np.linalg.norm(r - res[0]) <= 1e-12 * np.linalg.norm(res[0])


def test_periodic_sphere_images_bruteforce():
    """A sphere crossing periodic faces covers the cells within R of its
    nearest periodic image (minimum-image distance, brute force here); the
    charge stays exact (PER_CELLS) and a Dirichlet axis clips as before."""
    shape, h = (24, 20, 16), 1.0
    bt = [P, P, P, P, D, D]
    c = np.array([[0.7, 19.2, 8.0], [12.0, 10.0, 5.5], [23.5, 0.2, 14.0]])
    R = np.array([4.0, 3.0, 4.5])
    q = np.array([1.0, -1.0, 2.0])
    o = oracle.Oracle(shape, h, bt, [0.0] * 6, min_coarse=4)
    o.set_rhs_from_spheres(c, R, q)
    idx = [(np.arange(n) + 0.5) * h for n in shape]
    X, Y, Z = np.meshgrid(*idx, indexing="ij")
    rho = np.zeros(shape)
    L = np.array(shape) * h
    for p in range(len(q)):
        best = np.full(shape, np.inf)
        for mx in (-1, 0, 1):
            for my in (-1, 0, 1):
                d2 = ((X - (c[p, 0] + mx * L[0])) ** 2
                      + (Y - (c[p, 1] + my * L[1])) ** 2 + (Z - c[p, 2]) ** 2)
                best = np.minimum(best, d2)
        inside = best <= R[p] ** 2
        rho[inside] += q[p] / (inside.sum() * h ** 3)
    f = o.rhs()
    assert np.array_equal(f != 0, rho != 0)
    assert np.allclose(f, rho, rtol=1e-15, atol=1e-15)
    assert abs(f.sum() * h ** 3 - q.sum()) < 1e-12
    # the first sphere wraps in x and y: cells on both sides of each face
    assert f[0, 19, 8] != 0 and f[23, 0, 8] != 0 and f[23, 19, 8] != 0


def test_periodic_argument_rules():
    """Periodic faces come in pairs; spheres on a periodic axis need their
    centre inside [0, L) and 2R + 2h <= L (disjoint images); no BC patch or
    face values on a periodic face."""
    with pytest.raises(ValueError):
        oracle.Oracle((8, 8, 8), 1.0, [P, D, D, D, D, D], [0.0] * 6)
    o = oracle.Oracle((16, 8, 8), 1.0, [P, P, D, D, D, D], [0.0] * 6)
    with pytest.raises(ValueError):   # 2R + 2h > L_x = 16
        o.set_rhs_from_spheres([[8.0, 4.0, 4.0]], [7.5], [1.0])
    with pytest.raises(ValueError):   # centre outside [0, L_x)
        o.set_rhs_from_spheres([[16.5, 4.0, 4.0]], [2.0], [1.0])
    o.set_rhs_from_spheres([[15.5, 4.0, 4.0]], [2.0], [1.0])
    with pytest.raises(ValueError):
        o.set_bc_patch(0, 0, 2, 0, 2, D, 1.0)
    with pytest.raises(ValueError):
        o.set_face_values(1, np.zeros(64))


def test_periodic_gradient_wraps():
    """Eq.15 on a field varying along a periodic axis only: the D3Q19 sum
    collapses to the central difference (1/18 + 4/36 = 1/6; 3 S / h), and
    at the boundary cell the neighbour is the opposite side's cell."""
    shape, h = (16, 8, 8), 0.25
    bt = [P, P, P, P, P, P][:4] + [D, D]
    o = oracle.Oracle(shape, h, bt, [0.0] * 6, min_coarse=2)
    x = (np.arange(16) + 0.5) * h
    phi = np.broadcast_to(np.sin(2 * np.pi * x / 4.0)[:, None, None], shape).copy()
    for i in (0, 7, 15):
        g = o.gradient(phi, i, 3, 4)
        ref = (phi[(i + 1) % 16, 3, 4] - phi[(i - 1) % 16, 3, 4]) / (2 * h)
        assert abs(g[0] - ref) < 1e-13
        assert abs(g[1]) < 1e-14 and abs(g[2]) < 1e-14
