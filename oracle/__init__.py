"""oracle -- TEST INFRASTRUCTURE ONLY.

Plain CPU fp64 oracle of the cell-centered multigrid Poisson solve of
Bartuschat & Ruede (arXiv 1410.6609), see ``mg_oracle.c`` for the passages
each step follows.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The CUDA product (``paper_1410_6609_b200``) never imports it and
shares no code with it.

This module is a thin ctypes wrapper: every number is computed in C.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmg_oracle.so")
SRC_PATH = os.path.join(_HERE, "mg_oracle.c")

DIRICHLET = 0
NEUMANN = 1
PERIODIC = 2
PER_CELLS = 0
PER_VOLUME = 1

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no FMA contraction, no fast-math)."""
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(
                os.path.getmtime(SRC_PATH),
                os.path.getmtime(os.path.join(_HERE, "mg_oracle.h")))):
        return LIB_PATH
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
           "-fPIC", "-shared", "-std=c11", "-o", LIB_PATH, SRC_PATH, "-lm"]
    subprocess.check_call(cmd, cwd=_HERE)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int)
        u8 = ctypes.POINTER(ctypes.c_uint8)
        i, d = ctypes.c_int, ctypes.c_double
        L.orc_create.restype = P
        L.orc_create.argtypes = [i, i, i, d, ip, dp, u8, i, i]
        L.orc_destroy.argtypes = [P]
        L.orc_num_levels.argtypes = [P]
        L.orc_level_dims.argtypes = [P, i, ip]
        for n in ("orc_get_stencil", "orc_get_phi", "orc_get_rhs"):
            getattr(L, n).argtypes = [P, i, dp]
        L.orc_get_unknown.argtypes = [P, i, u8]
        L.orc_set_phi.argtypes = [P, i, dp]
        L.orc_set_rhs_raw.argtypes = [P, i, dp]
        L.orc_set_rhs.argtypes = [P, dp]
        L.orc_set_rhs_from_spheres.argtypes = [P, i, dp, dp, dp, i]
        L.orc_sphere_cell_count.restype = ctypes.c_long
        L.orc_sphere_cell_count.argtypes = [i, i, i, d, d, d, d, d]
        L.orc_sphere_density.argtypes = [i, i, i, d, i, dp, dp, dp, i, dp]
        L.orc_bc_adapt.argtypes = [P]
        L.orc_smooth_half.argtypes = [P, i, i]
        L.orc_residual.argtypes = [P, i, dp]
        L.orc_restrict_residual.argtypes = [P, i]
        L.orc_prolong_correct.argtypes = [P, i, d]
        L.orc_cg.argtypes = [P, i, d, i]
        L.orc_apply.argtypes = [P, i, dp, dp]
        L.orc_set_schedule.argtypes = [P, i, i, d, d, i]
        L.orc_set_fused_norm.argtypes = [P, i]
        L.orc_residual_norm.restype = d
        L.orc_residual_norm.argtypes = [P]
        L.orc_vcycle.restype = d
        L.orc_vcycle.argtypes = [P]
        L.orc_solve.argtypes = [P, d, i, ip, dp]
        L.orc_last_cg_iters.argtypes = [P]
        L.orc_set_bc_patch.argtypes = [P, i, i, i, i, i, i, d]
        L.orc_set_face_values.argtypes = [P, i, dp]
        L.orc_set_permittivity.argtypes = [P, dp]
        L.orc_gradient.argtypes = [P, dp, i, i, i, dp]
        L.orc_coulomb_forces.argtypes = [P, i, dp, dp, dp, i, i, dp]
        L.orc_sphere_subcount.restype = ctypes.c_long
        L.orc_sphere_subcount.argtypes = [i, i, i, d, i, d, d, d, d]
        L.orc_sphere_density_sub.argtypes = [i, i, i, d, i, i, dp, dp, dp, i, dp]
        L.orc_set_rhs_from_spheres_sub.argtypes = [P, i, dp, dp, dp, i, i]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def sphere_cell_count(shape, h, center, radius, subsample=1) -> int:
    """Covered cells (s = 1) or covered sub-cells (s > 1) of one sphere."""
    nx, ny, nz = shape
    return int(lib().orc_sphere_subcount(nx, ny, nz, float(h), int(subsample),
                                         float(center[0]), float(center[1]),
                                         float(center[2]), float(radius)))


def sphere_density(shape, h, centers, radii, charges,
                   normalization=PER_CELLS, subsample=1) -> np.ndarray:
    nx, ny, nz = shape
    c = _f64(centers).reshape(-1)
    r = _f64(radii)
    q = _f64(charges)
    out = np.empty((nx, ny, nz), np.float64)
    lib().orc_sphere_density_sub(nx, ny, nz, float(h), int(subsample), len(r),
                                 _dp(c), _dp(r), _dp(q), int(normalization),
                                 _dp(out))
    return out


class Oracle:
    """One multigrid hierarchy on the CPU (natural layout, x slowest)."""

    def __init__(self, shape, h, bc_type, bc_value=None, solid=None,
                 min_coarse=4, max_levels=0, nu1=2, nu2=2, alpha=2.0,
                 coarse_tol=1e-12, coarse_maxit=1000, fused_norm=False):
        L = lib()
        nx, ny, nz = (int(s) for s in shape)
        if bc_value is None:
            bc_value = [0.0] * 6
        bt = (ctypes.c_int * 6)(*[int(t) for t in bc_type])
        bv = (ctypes.c_double * 6)(*[float(v) for v in bc_value])
        sp = None
        self._solid = None
        if solid is not None:
            self._solid = np.ascontiguousarray(solid, dtype=np.uint8)
            assert self._solid.shape == (nx, ny, nz)
            sp = self._solid.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
        self._h = L.orc_create(nx, ny, nz, float(h), bt, bv, sp,
                               int(min_coarse), int(max_levels))
        if not self._h:
            raise ValueError("oracle: bad arguments")
        self.h = float(h)
        L.orc_set_schedule(self._h, nu1, nu2, float(alpha), float(coarse_tol),
                           int(coarse_maxit))
        # reading c11: vcycle() reports the in-cycle residual norm
        L.orc_set_fused_norm(self._h, int(bool(fused_norm)))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_destroy(self._h)
            self._h = None

    # -- hierarchy ---------------------------------------------------------
    @property
    def nlevels(self) -> int:
        return lib().orc_num_levels(self._h)

    def dims(self, l):
        d = (ctypes.c_int * 3)()
        lib().orc_level_dims(self._h, l, d)
        return tuple(d)

    def stencil(self, l) -> np.ndarray:
        out = np.empty(self.dims(l) + (7,), np.float64)
        lib().orc_get_stencil(self._h, l, _dp(out))
        return out

    def unknown(self, l) -> np.ndarray:
        out = np.empty(self.dims(l), np.uint8)
        lib().orc_get_unknown(self._h, l,
                              out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
        return out

    def set_bc_patch(self, face, a0, a1, b0, b1, bc_type, value):
        if lib().orc_set_bc_patch(self._h, face, a0, a1, b0, b1, int(bc_type),
                                  float(value)) != 0:
            raise ValueError("oracle: bad patch")

    def set_permittivity(self, eps):
        """Cell permittivity (natural layout), None = constant 1 (N4)."""
        if eps is None:
            rc = lib().orc_set_permittivity(self._h, None)
        else:
            self._eps = _f64(eps)
            assert self._eps.shape == self.dims(0)
            rc = lib().orc_set_permittivity(self._h, _dp(self._eps))
        if rc != 0:
            raise ValueError("oracle: permittivity must be > 0")

    def set_face_values(self, face, values):
        v = _f64(values).reshape(-1)
        if lib().orc_set_face_values(self._h, int(face), _dp(v)) != 0:
            raise ValueError("oracle: bad face")

    def gradient(self, phi, i, j, k):
        """Isotropic D3Q19 gradient (Eq.15) of level-0 field phi at a cell."""
        phi = _f64(phi)
        g = np.empty(3)
        lib().orc_gradient(self._h, _dp(phi), int(i), int(j), int(k), _dp(g))
        return g

    def coulomb_forces(self, centers, radii, charges, normalization=PER_CELLS,
                       subsample=1):
        """Eq.14 forces (n, 3) of the spheres on the current Phi."""
        c = _f64(centers).reshape(-1)
        r = _f64(radii)
        q = _f64(charges)
        out = np.empty(3 * len(r))
        if lib().orc_coulomb_forces(self._h, len(r), _dp(c), _dp(r), _dp(q),
                                    int(normalization), int(subsample),
                                    _dp(out)) != 0:
            raise ValueError("oracle: bad sphere on a periodic axis")
        return out.reshape(-1, 3)

    # -- fields ------------------------------------------------------------
    def phi(self, l=0) -> np.ndarray:
        out = np.empty(self.dims(l), np.float64)
        lib().orc_get_phi(self._h, l, _dp(out))
        return out

    def set_phi(self, a, l=0):
        a = _f64(a)
        assert a.shape == self.dims(l)
        lib().orc_set_phi(self._h, l, _dp(a))

    def rhs(self, l=0) -> np.ndarray:
        out = np.empty(self.dims(l), np.float64)
        lib().orc_get_rhs(self._h, l, _dp(out))
        return out

    def set_rhs_raw(self, a, l=0):
        a = _f64(a)
        assert a.shape == self.dims(l)
        lib().orc_set_rhs_raw(self._h, l, _dp(a))

    def set_rhs(self, f):
        f = _f64(f)
        assert f.shape == self.dims(0)
        lib().orc_set_rhs(self._h, _dp(f))

    def set_rhs_from_spheres(self, centers, radii, charges,
                             normalization=PER_CELLS, subsample=1):
        c = _f64(centers).reshape(-1)
        r = _f64(radii)
        q = _f64(charges)
        rc = lib().orc_set_rhs_from_spheres_sub(self._h, len(r), _dp(c), _dp(r),
                                                _dp(q), int(normalization),
                                                int(subsample))
        if rc != 0:
            raise ValueError("oracle: a sphere covers no cell centre, or violates "
                             "the periodic-axis rule")

    # -- steps -------------------------------------------------------------
    def smooth_half(self, l, color):
        lib().orc_smooth_half(self._h, l, color)

    def residual(self, l=0) -> np.ndarray:
        out = np.empty(self.dims(l), np.float64)
        lib().orc_residual(self._h, l, _dp(out))
        return out

    def apply(self, x, l=0) -> np.ndarray:
        x = _f64(x)
        out = np.empty(self.dims(l), np.float64)
        lib().orc_apply(self._h, l, _dp(x), _dp(out))
        return out

    def restrict_residual(self, l):
        lib().orc_restrict_residual(self._h, l)

    def prolong_correct(self, l, alpha=2.0):
        lib().orc_prolong_correct(self._h, l, float(alpha))

    def cg(self, l, tol=1e-12, maxit=1000) -> int:
        return lib().orc_cg(self._h, l, float(tol), int(maxit))

    def residual_norm(self) -> float:
        return lib().orc_residual_norm(self._h)

    def vcycle(self) -> float:
        return lib().orc_vcycle(self._h)

    def solve(self, tol, max_cycles=100):
        cyc = ctypes.c_int(0)
        hist = np.zeros(max_cycles + 1, np.float64)
        st = lib().orc_solve(self._h, float(tol), int(max_cycles),
                             ctypes.byref(cyc), _dp(hist))
        return st, cyc.value, hist[:cyc.value + 1].copy()

    @property
    def last_cg_iters(self) -> int:
        return lib().orc_last_cg_iters(self._h)
