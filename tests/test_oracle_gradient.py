"""Pins of the oracle's gradient fallback at walls and solid cells.

PAPER.md:472-478 (Eq.15) gives the isotropic D3Q19 gradient and applies it
"where possible".  Reading d6 fixes what happens elsewhere: per
axis the central difference if both axis neighbours are fluid cells of the
domain, else the one-sided first-order difference toward the valid one,
else 0.  Each branch is pinned by a field on which it has a closed form that
the other branches do not share:

  linear     a.x + d       D3Q19, central and one-sided all give a exactly
  quadratic  x^2           central 2x, forward 2x + h, backward 2x - h
  x y^2      (x-component) D3Q19 y^2 + h^2/3 (third moment of the edge
                           links), central y^2

The cells are hand-placed (face, edge, corner, beside a solid, between two
solids) and every expected value is written out from these closed forms,
not from the oracle.
"""
import numpy as np
import pytest

import oracle

D, N = oracle.DIRICHLET, oracle.NEUMANN
SHAPE = (8, 9, 10)
H = 0.5


def _centres():
    return np.meshgrid(*[(np.arange(n) + 0.5) * H for n in SHAPE], indexing="ij")


def _oracle(solid=None, bc=(D, N, N, D, D, N)):
    return oracle.Oracle(SHAPE, H, list(bc), [0.0] * 6, solid=solid)


def _mask():
    """A few solid cells: (4,4,4) alone, and the pair (2,6,5), (4,6,5)
    enclosing the fluid cell (3,6,5) along x."""
    m = np.zeros(SHAPE, np.uint8)
    m[4, 4, 4] = 1
    m[2, 6, 5] = 1
    m[4, 6, 5] = 1
    return m


@pytest.mark.parametrize("solid", [None, "mask"])
def test_linear_field_exact_at_walls_corners_and_solids(solid):
    """Every branch is exact on a linear field: the gradient is a at every
    cell whose axis has at least one fluid neighbour (walls of either BC
    type, corners, cells beside a solid)."""
    m = _mask() if solid else None
    o = _oracle(m)
    X = _centres()
    a = np.array([0.75, -1.25, 2.0])
    phi = a[0] * X[0] + a[1] * X[1] + a[2] * X[2] + 0.3
    cells = [(0, 0, 0), (7, 8, 9), (0, 4, 5), (7, 4, 5), (3, 0, 5), (3, 8, 5),
             (3, 4, 0), (3, 4, 9), (0, 8, 0), (5, 5, 5)]
    if solid:
        cells += [(3, 4, 4), (5, 4, 4), (4, 3, 4), (4, 5, 4), (4, 4, 3), (4, 4, 5),
                  (3, 3, 4), (5, 5, 5)]
    for c in cells:
        assert np.allclose(o.gradient(phi, *c), a, rtol=0, atol=1e-12), c


def test_axis_between_two_solids_gives_zero():
    """Fluid cell (3,6,5) with solid x-neighbours (2,6,5), (4,6,5): no
    difference exists along x, so g_x = 0; y and z still see a (central)."""
    o = _oracle(_mask())
    X = _centres()
    a = np.array([0.75, -1.25, 2.0])
    phi = a[0] * X[0] + a[1] * X[1] + a[2] * X[2]
    g = o.gradient(phi, 3, 6, 5)
    assert g[0] == 0.0
    assert np.allclose(g[1:], a[1:], rtol=0, atol=1e-12)


def test_quadratic_one_sided_direction():
    """Phi = x^2 (x = (i+1/2) h): central 2x exactly; at the x- wall only the
    + neighbour exists -> forward (phi(x+h) - phi(x))/h = 2x + h; at the x+
    wall backward = 2x - h; beside the solid (4,4,4): cell (3,4,4) has only
    its - neighbour -> 2x - h, cell (5,4,4) only its + neighbour -> 2x + h."""
    for solid in (None, _mask()):
        o = _oracle(solid)
        X = _centres()
        phi = X[0] ** 2
        x = lambda i: (i + 0.5) * H  # noqa: E731
        assert np.isclose(o.gradient(phi, 0, 4, 5)[0], 2 * x(0) + H, rtol=0, atol=1e-12)
        assert np.isclose(o.gradient(phi, 7, 4, 5)[0], 2 * x(7) - H, rtol=0, atol=1e-12)
        assert np.isclose(o.gradient(phi, 3, 0, 5)[0], 2 * x(3), rtol=0, atol=1e-12)
        if solid is not None:
            assert np.isclose(o.gradient(phi, 3, 4, 4)[0], 2 * x(3) - H, rtol=0,
                              atol=1e-12)
            assert np.isclose(o.gradient(phi, 5, 4, 4)[0], 2 * x(5) + H, rtol=0,
                              atol=1e-12)
            # y / z components of x^2 vanish in every branch
            assert np.allclose(o.gradient(phi, 3, 4, 4)[1:], 0.0, atol=1e-13)


def test_isotropic_vs_central_selection():
    """Phi = x y^2: the D3Q19 x-component is y^2 + h^2/3 (the edge links
    carry the third moment), the central difference y^2.  Cells whose 18
    links are all fluid take Eq.15; a cell with one solid EDGE neighbour but
    fluid axis neighbours falls back to central; a wall cell likewise."""
    o = _oracle(_mask())
    X = _centres()
    phi = X[0] * X[1] ** 2
    y = lambda j: (j + 0.5) * H  # noqa: E731
    # interior, far from the solids: D3Q19
    assert np.isclose(o.gradient(phi, 5, 2, 2)[0], y(2) ** 2 + H * H / 3, rtol=0,
                      atol=1e-12)
    # (3,3,4): edge neighbour (4,4,4) (link (+1,+1,0)) is solid -> central
    assert np.isclose(o.gradient(phi, 3, 3, 4)[0], y(3) ** 2, rtol=0, atol=1e-12)
    # y-wall cell (5,0,3): its y- links leave the domain -> central in x
    assert np.isclose(o.gradient(phi, 5, 0, 3)[0], y(0) ** 2, rtol=0, atol=1e-12)
    # the same interior cell without a mask anywhere near: D3Q19 again
    o2 = _oracle(None)
    assert np.isclose(o2.gradient(phi, 3, 3, 4)[0], y(3) ** 2 + H * H / 3, rtol=0,
                      atol=1e-12)


def test_periodic_axis_neighbours_count_as_valid():
    """On a periodic x axis the wall cell i = 0 has both x-neighbours (the
    opposite side's cell is a neighbour), so a field periodic in
    x is differentiated centrally there: Phi = sin(2 pi x / Lx) gives
    (sin(t_1) - sin(t_-1))/(2h), t_-1 = t_{n-1} - 2 pi (the y-wall cell
    (0,0,5) is not eligible for the D3Q19 stencil)."""
    o = oracle.Oracle(SHAPE, H, [oracle.PERIODIC, oracle.PERIODIC, D, D, N, N],
                      [0.0] * 6)
    Lx = SHAPE[0] * H
    X = _centres()
    phi = np.sin(2 * np.pi * X[0] / Lx)
    t = lambda i: 2 * np.pi * (i + 0.5) * H / Lx  # noqa: E731
    g = o.gradient(phi, 0, 0, 5)  # y wall cell: not all 18 links valid
    assert np.isclose(g[0], (np.sin(t(1)) - np.sin(t(-1))) / (2 * H), rtol=0, atol=1e-12)
