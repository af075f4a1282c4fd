"""Seeded synthetic inputs for the five BASELINE.json configurations.

This module holds input generators only -- none of the method's arithmetic.
It is the one module both the CUDA path's callers and the oracle's callers
use, so that both receive bit-identical inputs ("Input recipe").

Axis convention: arrays are (x, y, z) in C order, x slowest.  Physical
coordinates of cell (i, j, k) centre are ((i+1/2)h, (j+1/2)h, (k+1/2)h).
Face order for boundary conditions: x-, x+, y-, y+, z-, z+.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Tuple

import numpy as np

DIRICHLET = 0
NEUMANN = 1
PERIODIC = 2


@dataclasses.dataclass
class Workload:
    name: str
    shape: Tuple[int, int, int]
    h: float
    bc_type: List[int]
    bc_value: List[float]
    min_coarse: int
    nu1: int = 2
    nu2: int = 2
    coarse_tol: float = 1e-12       # CG relative tolerance (reading c8)
    cycles: Optional[int] = None    # fixed cycle count (cfg1, cfg3)
    tol: Optional[float] = None     # relative reduction target (cfg2, cfg4, cfg5)
    rhs: Optional[np.ndarray] = None        # natural-layout f (cfg1, cfg3)
    centers: Optional[np.ndarray] = None    # (n, 3) physical coordinates
    radii: Optional[np.ndarray] = None
    charges: Optional[np.ndarray] = None
    solid: Optional[np.ndarray] = None      # uint8 mask, natural layout (cfg5)

    @property
    def cells(self) -> int:
        return int(np.prod(self.shape))


def all_dirichlet():
    return [DIRICHLET] * 6, [0.0] * 6


def channel_bc(phi_top: float = 1.0):
    """Config 2/4: Phi=0 on the y=0 wall, Phi=phi_top on the far y wall,
    homogeneous Neumann on the x and z faces."""
    return ([NEUMANN, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, NEUMANN],
            [0.0, 0.0, 0.0, phi_top, 0.0, 0.0])


def sine_rhs(n: int) -> np.ndarray:
    """Config 1: f = 3 pi^2 sin(pi x) sin(pi y) sin(pi z) at cell centres of
    the unit cube with h = 1/n."""
    h = 1.0 / n
    x = (np.arange(n, dtype=np.float64) + 0.5) * h
    s = np.sin(np.pi * x)
    return (3.0 * np.pi ** 2) * (s[:, None, None] * s[None, :, None]
                                 * s[None, None, :])


def uniform_rhs(shape, seed: int) -> np.ndarray:
    """Config 3: i.i.d. U[-1, 1] in C order (x slowest)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, tuple(shape))


def random_spheres(extent, radius: float, n: int, seed: int,
                   exclude_box=None, max_tries: int = 200) -> Tuple[np.ndarray, np.ndarray]:
    """Random sequential addition of n non-overlapping spheres (reading c14):
    centres U[R, L-R] per axis, rejected if closer than 2R to an accepted
    centre (or, with exclude_box=((x0,x1),(y0,y1),(z0,z1)), closer than R to
    that box).  Then n charges, each +-1 with probability 1/2."""
    rng = np.random.default_rng(seed)
    L = np.asarray(extent, np.float64)
    R = float(radius)
    cell = 2.0 * R
    bins = {}
    out = np.empty((n, 3), np.float64)
    k = 0
    tries = 0
    limit = max_tries * max(n, 1)
    while k < n:
        tries += 1
        if tries > limit:
            raise RuntimeError("random_spheres: could not place all spheres")
        c = rng.uniform(R, L - R)
        if exclude_box is not None:
            d2 = 0.0
            for a in range(3):
                lo, hi = exclude_box[a]
                t = max(lo - c[a], 0.0, c[a] - hi)
                d2 += t * t
            if d2 < R * R:
                continue
        b = tuple((c // cell).astype(np.int64))
        ok = True
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    for j in bins.get((b[0] + dx, b[1] + dy, b[2] + dz), ()):
                        if float(np.sum((out[j] - c) ** 2)) < cell * cell:
                            ok = False
                            break
                    if not ok:
                        break
                if not ok:
                    break
            if not ok:
                break
        if not ok:
            continue
        out[k] = c
        bins.setdefault(b, []).append(k)
        k += 1
    charges = rng.choice(np.array([-1.0, 1.0]), size=n)
    return out, charges


def periodic_channel_bc(phi_top: float = 1.0):
    """The config-2/4 channel with periodic flow (x) and span (z) axes
    (P:441-443): Dirichlet 0 / phi_top on the y walls."""
    return ([PERIODIC, PERIODIC, DIRICHLET, DIRICHLET, PERIODIC, PERIODIC],
            [0.0, 0.0, 0.0, phi_top, 0.0, 0.0])


def move_spheres(centers, radii, extent, step: int, seed: int = 0,
                 amplitude: float = 0.05, periodic=(False, False, False)):
    """Synthetic particle motion of the time-stepping regime (SURVEY 8(f)
    N3).  In the paper the spheres move under the LBM / pe coupling of
    Alg.1 (out of scope here); this generator only supplies positions:
    step `step` displaces every centre by a vector with components drawn
    from U[-amplitude, amplitude] (default_rng((seed, step))), then reflects
    it into [R, L - R] on wall axes or wraps it into [0, L) on periodic
    axes.  Deterministic per (seed, step); overlaps are not prevented
    (charge densities of overlapping spheres add, mg.h)."""
    c = np.array(centers, np.float64, copy=True)
    R = np.asarray(radii, np.float64)
    L = np.asarray(extent, np.float64)
    rng = np.random.default_rng((int(seed), int(step)))
    c += rng.uniform(-amplitude, amplitude, c.shape)
    for a in range(3):
        if periodic[a]:
            c[:, a] = np.mod(c[:, a], L[a])
            c[c[:, a] >= L[a], a] = 0.0
        else:
            lo, hi = R, L[a] - R
            c[:, a] = np.where(c[:, a] < lo, 2 * lo - c[:, a], c[:, a])
            c[:, a] = np.where(c[:, a] > hi, 2 * hi - c[:, a], c[:, a])
    return c


def timestep_workload(n: int = 512, seed: int = 0) -> Workload:
    """The paper's scaling regime on config 4's single-GPU
    box: 512^3 channel, spheres R = 6 at 5 % volume (cfg4), RHS and force
    subsampling factor 2, V(3,3)-cycles, coarsest 8^3; 5 cycles at
    the first time step, then 1 per step."""
    w = cfg4(P=1, n=n, seed=seed)
    w.name = "timestep_%d" % n
    w.nu1 = w.nu2 = 3
    w.cycles = 1
    return w


def cfg1(n: int = 32, cycles: int = 10) -> Workload:
    bt, bv = all_dirichlet()
    # "exact coarse solve": CG to 1e-14 relative (reading c8)
    return Workload("cfg1_sine%d" % n, (n, n, n), 1.0 / n, bt, bv, min_coarse=4,
                    coarse_tol=1e-14, cycles=cycles, rhs=sine_rhs(n))


def cfg2(seed: int = 0, shape=(256, 64, 64), n_spheres: int = 200,
         radius: float = 4.0, tol: float = 1e-8) -> Workload:
    bt, bv = channel_bc(1.0)
    c, q = random_spheres(shape, radius, n_spheres, seed)
    return Workload("cfg2_channel_%dx%dx%d" % tuple(shape), tuple(shape), 1.0,
                    bt, bv, min_coarse=4, tol=tol, centers=c,
                    radii=np.full(n_spheres, radius), charges=q)


def cfg3(n: int = 512, seed: int = 0, cycles: int = 20,
         with_rhs: bool = True) -> Workload:
    bt, bv = all_dirichlet()
    rhs = uniform_rhs((n, n, n), seed) if with_rhs else None
    return Workload("cfg3_random%d" % n, (n, n, n), 1.0 / n, bt, bv,
                    min_coarse=8, cycles=cycles, rhs=rhs)


def cfg4_sphere_count(cells: int, radius: float = 6.0,
                      fraction: float = 0.05) -> int:
    return int(round(fraction * cells / (4.0 / 3.0 * math.pi * radius ** 3)))


def cfg4(P: int = 1, n: int = 512, seed: int = 0, radius: float = 6.0,
         tol: float = 1e-8) -> Workload:
    """Weak scaling: (n P) x n x n, slabs of n planes per GPU, channel BCs,
    spheres of radius 6 at 5% volume fraction."""
    shape = (n * P, n, n)
    bt, bv = channel_bc(1.0)
    ns = cfg4_sphere_count(int(np.prod(shape)), radius)
    c, q = random_spheres(shape, radius, ns, seed)
    return Workload("cfg4_weak_P%d_%d" % (P, n), shape, 1.0, bt, bv,
                    min_coarse=8, tol=tol, centers=c,
                    radii=np.full(ns, radius), charges=q)


def beam_box(shape):
    """Config 5 solid beam (reading c17): x in [3/4 nx, nx), y in
    [232/512 ny, 280/512 ny), all z -- the beam splitting the last quarter of
    the bifurcating channel."""
    nx, ny, nz = shape
    x0 = (3 * nx) // 4
    y0 = int(round(232 * ny / 512))
    y1 = max(int(round(280 * ny / 512)), y0 + 1)
    return (x0, nx), (y0, y1), (0, nz)


def beam_mask(shape) -> np.ndarray:
    (x0, x1), (y0, y1), (z0, z1) = beam_box(shape)
    m = np.zeros(tuple(shape), np.uint8)
    m[x0:x1, y0:y1, z0:z1] = 1
    return m


def cfg5(scale: int = 1, seed: int = 0, radius: float = 4.0,
         n_spheres: Optional[int] = None, tol: float = 1e-8) -> Workload:
    """Strong scaling: 2048 x 512 x 512 (divided by `scale`), h = 1, beam
    mask, Dirichlet 0 / 1 on the y = 0 / y = ny walls (full length), homogeneous
    Neumann elsewhere and on the beam walls; 50,000 spheres of radius 4 outside
    the beam (scaled by the volume), charges +-1; V(3,3) to 1e-8."""
    shape = (2048 // scale, 512 // scale, 512 // scale)
    bt, bv = channel_bc(1.0)
    if n_spheres is None:
        n_spheres = max(1, int(round(50000 / scale ** 3)))
    box = beam_box(shape)
    c, q = random_spheres(shape, radius, n_spheres, seed,
                          exclude_box=tuple((float(a), float(b)) for a, b in box))
    w = Workload("cfg5_beam_%dx%dx%d" % shape, shape, 1.0, bt, bv,
                 min_coarse=8, nu1=3, nu2=3, tol=tol, centers=c,
                 radii=np.full(n_spheres, radius), charges=q)
    w.solid = beam_mask(shape)
    return w
