"""Independent dense / spectral constructions used to pin the oracle.

Nothing here calls the oracle's operator code: matrices are built from the
*unfolded* 7-point stencil (Eq.13) applied to fields padded
with ghost cells whose values follow the paper's extrapolation rules
(PAPER.md:451-459):

    Dirichlet:  Phi_ghost = 2 g_d - Phi_1
    Neumann:    Phi_ghost = Phi_1 + h g_n     (reading c2, outward normal)

    Periodic:   Phi_ghost = Phi on the opposite side

so the folded stencil of the oracle and the ghost-cell form here are two
different constructions of the same operator.
"""
from __future__ import annotations

import numpy as np

DIRICHLET, NEUMANN, PERIODIC = 0, 1, 2


def _ghost_pad(u, h, bc_type, bc_value, homogeneous):
    """Pad u by one ghost layer per face with the paper's extrapolation.
    bc_type[face] / bc_value[face] may be scalars or arrays over the face
    (the two other axes in (x,y,z) order): per-face-cell patches."""
    p = np.pad(u, 1)
    for face in range(6):
        ax, side = divmod(face, 2)
        g = 0.0 if homogeneous else bc_value[face]
        sl_g = [slice(1, -1)] * 3
        sl_1 = [slice(1, -1)] * 3
        if side == 0:
            sl_g[ax], sl_1[ax] = 0, 1
        else:
            sl_g[ax], sl_1[ax] = -1, -2
        inner = p[tuple(sl_1)]
        if np.all(np.asarray(bc_type[face]) == PERIODIC):
            sl_o = [slice(1, -1)] * 3  # the opposite side's last cell layer
            sl_o[ax] = -2 if side == 0 else 1
            p[tuple(sl_g)] = p[tuple(sl_o)]
            continue
        t = np.broadcast_to(np.asarray(bc_type[face]), inner.shape)
        gg = np.broadcast_to(np.asarray(g, dtype=float), inner.shape)
        p[tuple(sl_g)] = np.where(t == DIRICHLET, 2.0 * gg - inner, inner + h * gg)
    return p


def neg_laplacian_ghost(u, h, bc_type, bc_value, homogeneous=True):
    """(-Lap_h u) with ghost cells from the BCs: (6 u - sum of 6 nbrs)/h^2."""
    p = _ghost_pad(u, h, bc_type, bc_value, homogeneous)
    c = p[1:-1, 1:-1, 1:-1]
    s = (p[:-2, 1:-1, 1:-1] + p[2:, 1:-1, 1:-1] + p[1:-1, :-2, 1:-1]
         + p[1:-1, 2:, 1:-1] + p[1:-1, 1:-1, :-2] + p[1:-1, 1:-1, 2:])
    return (6.0 * c - s) / (h * h)


def dense_operator(shape, h, bc_type):
    """Dense matrix of the homogeneous-BC operator, column by column."""
    n = int(np.prod(shape))
    A = np.zeros((n, n))
    e = np.zeros(n)
    for c in range(n):
        e[c] = 1.0
        A[:, c] = neg_laplacian_ghost(e.reshape(shape), h, bc_type,
                                      [0.0] * 6).reshape(-1)
        e[c] = 0.0
    return A


def bc_rhs_shift(shape, h, bc_type, bc_value):
    """b such that A u = f + b is the inhomogeneous ghost-cell system:
    b = -(-Lap_h applied to u=0 with inhomogeneous ghosts)."""
    z = np.zeros(shape)
    return -neg_laplacian_ghost(z, h, bc_type, bc_value, homogeneous=False)


def tridiag_1d(n, h, lo, hi):
    """1D ghost-cell operator along one axis (ends: D -> 3, N -> 1 over h^2;
    periodic: circulant)."""
    T = np.zeros((n, n))
    for i in range(n):
        T[i, i] = 2.0
        if i > 0:
            T[i, i - 1] = -1.0
        if i < n - 1:
            T[i, i + 1] = -1.0
    # end rows (2 u_1 - ghost - u_2): Dirichlet ghost = -u_1 -> 3,
    # Neumann ghost = +u_1 -> 1
    if lo == PERIODIC:  # circulant: the ends couple to each other
        T[0, -1] += -1.0
        T[-1, 0] += -1.0
        return T / (h * h)
    T[0, 0] = 3.0 if lo == DIRICHLET else 1.0
    T[-1, -1] = 3.0 if hi == DIRICHLET else 1.0
    return T / (h * h)


def kron_solve(f, h, bc_type):
    """Exact solve of A u = f by fast diagonalisation of
    A = Tx (x) I (x) I + I (x) Ty (x) I + I (x) I (x) Tz (box domains)."""
    nx, ny, nz = f.shape
    ev, V = [], []
    for ax, n in enumerate((nx, ny, nz)):
        T = tridiag_1d(n, h, bc_type[2 * ax], bc_type[2 * ax + 1])
        w, Q = np.linalg.eigh(T)
        ev.append(w)
        V.append(Q)
    g = np.einsum("ia,jb,kc,ijk->abc", V[0], V[1], V[2], f, optimize=True)
    lam = ev[0][:, None, None] + ev[1][None, :, None] + ev[2][None, None, :]
    g = g / lam
    return np.einsum("ia,jb,kc,abc->ijk", V[0], V[1], V[2], g, optimize=True)


def injection_P(fine_shape, unknown_fine=None, unknown_coarse=None):
    """Dense nearest-neighbour prolongation: child <- parent."""
    nx, ny, nz = fine_shape
    cx, cy, cz = nx // 2, ny // 2, nz // 2
    P = np.zeros((nx * ny * nz, cx * cy * cz))
    for i in range(nx):
        for j in range(ny):
            for k in range(nz):
                f = (i * ny + j) * nz + k
                c = ((i // 2) * cy + j // 2) * cz + k // 2
                if unknown_fine is not None and not unknown_fine[i, j, k]:
                    continue
                P[f, c] = 1.0
    return P


def stencil_to_dense(st, per=(False, False, False)):
    """Dense matrix from a 7-per-cell stencil field [c, x-, x+, y-, y+, z-, z+];
    neighbours across a periodic axis wrap to the opposite side."""
    nx, ny, nz, _ = st.shape
    n = nx * ny * nz
    A = np.zeros((n, n))
    off = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
    for i in range(nx):
        for j in range(ny):
            for k in range(nz):
                r = (i * ny + j) * nz + k
                A[r, r] += st[i, j, k, 0]
                for q, (a, b, c) in enumerate(off):
                    ii, jj, kk = i + a, j + b, k + c
                    if per[0]:
                        ii %= nx
                    if per[1]:
                        jj %= ny
                    if per[2]:
                        kk %= nz
                    if 0 <= ii < nx and 0 <= jj < ny and 0 <= kk < nz:
                        A[r, (ii * ny + jj) * nz + kk] += st[i, j, k, 1 + q]
                    else:
                        assert st[i, j, k, 1 + q] == 0.0
    return A


def rbgs_matrix(A, shape, color):
    """Error propagation of one red-black half-sweep of colour `color`:
    G = I - Pi_C D^{-1} A (rows of the updated colour replaced)."""
    nx, ny, nz = shape
    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz),
                          indexing="ij")
    sel = (((i + j + k) & 1) == color).reshape(-1).astype(float)
    D = np.diag(A)
    return np.eye(A.shape[0]) - (sel / D)[:, None] * A


def vcycle_matrices(shapes, h, bc_type, nu1, nu2, alpha, A0=None):
    """Dense V-cycle error-propagation matrix M_0 and approximate inverse B_0
    for a hierarchy of box levels `shapes` (finest first), Galerkin coarse
    operators A_{l+1} = R A_l P with R = P^T / 8, exact coarsest solve.
    A0: the finest operator (default: the constant-coefficient one)."""
    A = [dense_operator(shapes[0], h, bc_type) if A0 is None else A0]
    Ps = []
    for l in range(len(shapes) - 1):
        P = injection_P(shapes[l])
        Ps.append(P)
        A.append((P.T / 8.0) @ A[l] @ P)
    L = len(shapes)
    B = np.linalg.inv(A[L - 1])
    M = None
    for l in range(L - 2, -1, -1):
        n = A[l].shape[0]
        I = np.eye(n)
        S = rbgs_matrix(A[l], shapes[l], 1) @ rbgs_matrix(A[l], shapes[l], 0)
        pre = np.linalg.matrix_power(S, nu1)
        post = np.linalg.matrix_power(S, nu2)
        cgc = I - alpha * Ps[l] @ B @ (Ps[l].T / 8.0) @ A[l]
        M = post @ cgc @ pre
        B = (I - M) @ np.linalg.inv(A[l])
    return M, A


def flux_operator_eps(shape, h, bc_type, eps, bc_value=None):
    """Variable-permittivity finite-volume operator -div(eps grad) (N4) built
    from fluxes: the flux between cells c and n is eps_f (u_c - u_n) / h^2
    with eps_f the harmonic mean of the two cells' eps; across a boundary
    face the ghost cell carries eps_c and the paper's extrapolated value
    (Dirichlet 2 g - u_c, Neumann u_c + h g).  Returns the dense matrix of
    the homogeneous operator and the RHS shift b of the inhomogeneous BCs
    (A u = f + b).  Independent of the oracle's folded stencil."""
    nx, ny, nz = shape
    n = nx * ny * nz
    A = np.zeros((n, n))
    b = np.zeros(n)
    g = [0.0] * 6 if bc_value is None else bc_value
    idx = np.arange(n).reshape(shape)
    offs = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
    for i in range(nx):
        for j in range(ny):
            for k in range(nz):
                c = idx[i, j, k]
                ec = eps[i, j, k]
                for f, (a, bb, cc) in enumerate(offs):
                    ii, jj, kk = i + a, j + bb, k + cc
                    per = bc_type[f] == PERIODIC
                    if per:
                        ii, jj, kk = ii % nx, jj % ny, kk % nz
                    if 0 <= ii < nx and 0 <= jj < ny and 0 <= kk < nz:
                        en = eps[ii, jj, kk]
                        ef = 2.0 * ec * en / (ec + en)
                        A[c, c] += ef / h ** 2
                        A[c, idx[ii, jj, kk]] -= ef / h ** 2
                    elif bc_type[f] == DIRICHLET:
                        # ghost 2 g - u_c: eps_c (u_c - (2 g - u_c)) / h^2
                        A[c, c] += 2.0 * ec / h ** 2
                        b[c] += 2.0 * ec * g[f] / h ** 2
                    else:
                        # Neumann ghost u_c + h g: eps_c (u_c - u_c - h g) / h^2
                        b[c] += ec * g[f] / h
    return A, b
