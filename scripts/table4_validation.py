"""Charged-sphere potential validation (Table 4).

256^3 cells, h = 1, one sphere of radius R, analytic Dirichlet data (Eq.18,
eps = 1) on every boundary face cell, the paper's naive mapping Q/V x
(covered sub-cell fraction), subsampling s_f, V(2,2) to 1e-11.  Reports,
next to the paper's Table 4, e_rV at the sphere position used,
||e_rPhi||_L2 = sqrt(mean(e^2)) and ||e_rPhi||_inf (signed).

Position (reading d11).  The paper shifts the sphere "by a small
distance in all dimensions (up to +-0.51 dx/s_f)" from the domain centre and
evaluates the potential "for the position of e_rVmax".  The
count of covered sub-cell centres is piecewise constant in the position and
its extreme values live in small regions that uniform sampling misses (round
1's 3000-sample search stayed 1-2 sub-cells short of the paper's e_rVmax
for R = 4, 6).  Here a hill climb over the shift (in sub-cell units; the
count depends only on R s_f and the shift in units of dx/s_f) looks for a
position whose count gives the paper's printed e_rVmax exactly; the
potential is then computed there.  Where that count is not found the
closest one reached is used and the row says so.

usage: python scripts/table4_validation.py [--out profiles/r02_table4.md]
"""
import argparse
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

# R: s_f: (mean|erV|, erVmax, L2, inf) in %  -- Table 4
PAPER = {
    4: {1: (1.14, 7.06, 1.87, 10.9), 2: (0.284, 2.58, 0.622, 3.37),
        3: (0.145, -1.43, 0.568, -2.06), 4: (0.081, 0.72, 0.192, 1.13)},
    6: {1: (0.638, -2.74, 0.927, -4.48), 2: (0.140, -1.43, 0.568, -2.19),
        3: (0.065, -0.33, 0.290, -0.80), 4: (0.039, -0.25, 0.273, -0.61)},
    8: {1: (0.285, 2.58, 0.622, 3.37), 2: (0.081, 0.72, 0.192, 0.97),
        3: (0.040, -0.25, 0.273, -0.67), 4: (0.021, -0.14, 0.251, -0.48)},
    9: {1: (0.258, 1.91, 0.444, 2.48), 2: (0.066, -0.33, 0.290, -0.82),
        3: (0.028, 0.32, 0.185, 0.44), 4: (0.018, -0.11, 0.244, -0.39)},
    12: {1: (0.146, -1.43, 0.567, -2.02), 2: (0.040, -0.25, 0.273, -0.58),
         3: (0.018, -0.11, 0.244, -0.39), 4: (0.009, -0.10, 0.243, -0.39)},
}


def lattice_counts(rs, offs):
    """Unit-lattice points (i + 1/2, j + 1/2, k + 1/2) within radius rs of
    each offset (the covered sub-cell centres of a sphere of radius R s_f in
    units of dx/s_f): per (i, j) column the k-interval, vectorised."""
    n = int(rs) + 2
    g = np.arange(-n, n + 1) + 0.5
    out = np.empty(len(offs), np.int64)
    for t, o in enumerate(offs):
        dx2 = (g - o[0]) ** 2
        dy2 = (g - o[1]) ** 2
        rem = rs * rs - (dx2[:, None] + dy2[None, :])
        ok = rem >= 0
        r = np.sqrt(np.where(ok, rem, 0.0))
        lo = np.ceil(o[2] - r - 0.5)
        hi = np.floor(o[2] + r - 0.5)
        out[t] = int(np.where(ok, np.maximum(hi - lo + 1, 0), 0).sum())
    return out


def search(rs, target, sign, V, rng, restarts=8, rounds=80, pop=3000, cand=300):
    """Hill climbs on the shift (unit-lattice units) toward the count whose
    e_rV prints as the paper's value `target` (%, 2 decimals), approached
    from the sign side; several restarts.  Returns (count, offset)."""
    tc = V * (1 + target / 100.0)
    def score(x):
        return -np.abs(x - tc) + 1e-3 * sign * x
    def hit(x):
        return abs(100.0 * (x - V) / V - target) <= 0.005
    best, bc = None, None
    for _ in range(restarts):
        P = rng.uniform(0, 1, (pop, 3))
        c = lattice_counts(rs, P)
        i = int(np.argmax(score(c)))
        cur, cc0 = P[i], int(c[i])
        step = 0.05
        for _ in range(rounds):
            if hit(cc0):
                break
            C = cur + rng.normal(0, step, (cand, 3))
            cc = lattice_counts(rs, C)
            j = int(np.argmax(score(cc)))
            if score(cc[j]) >= score(cc0):
                cur, cc0 = C[j], int(cc[j])
            step = max(step * 0.93, 1e-4)
        if bc is None or score(cc0) > score(bc):
            best, bc = cur, cc0
        if hit(bc):
            break
    return bc, best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_table4.md"))
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--radii", default="4,6,8,9,12")
    a = ap.parse_args()
    import oracle
    from paper_1410_6609_b200 import _build
    _build.build()
    from paper_1410_6609_b200 import mg
    from test_gpu_parity import face_centres, sphere_potential
    n, h, Q = a.n, 1.0, 1.0
    shape = (n, n, n)
    x = (np.arange(n) + 0.5) * h
    Xc = np.meshgrid(x, x, x, indexing="ij")
    rows = []
    for R in [int(r) for r in a.radii.split(",")]:
        V = 4.0 / 3.0 * math.pi * R ** 3
        for sf in (1, 2, 3, 4):
            p = PAPER[R][sf]
            rs = R * sf
            Vs = V * sf ** 3
            rng = np.random.default_rng(R * 10 + sf)
            cnt, off = search(rs, p[1], 1 if p[1] > 0 else -1, Vs, rng)
            # the sphere centre: domain centre + shift, the shift in dx/s_f
            # units congruent to the lattice offset (n s_f / 2 is an integer)
            # and inside +-0.5 dx/s_f
            c = n / 2.0 + (np.mod(off + 0.5, 1.0) - 0.5) / sf
            exact_cnt = oracle.sphere_cell_count(shape, h, c, R, sf)  # the library rule
            ev = 100.0 * (exact_cnt / sf ** 3 - V) / V
            s = mg.Multigrid(shape, h, [0] * 6, [0.0] * 6, min_coarse=8)
            for q in range(6):
                s.set_face_values(q, sphere_potential(face_centres(shape, h, q), c, R, Q))
            s.set_rhs_from_spheres(c[None, :], [float(R)], [Q],
                                   normalization=mg.MG_CHARGE_PER_VOLUME, subsample=sf)
            rc, cyc, hist = s.solve(1e-11, 60)
            exact = sphere_potential(Xc, c, R, Q)
            e = (s.get_solution() - exact) / exact
            l2 = 100 * float(np.sqrt(np.mean(e ** 2)))
            im = int(np.argmax(np.abs(e)))
            inf = 100 * float(e.reshape(-1)[im])
            s.close()
            rows.append((R, sf, ev, p[1], abs(ev - p[1]) <= 0.005, l2, p[2], inf, p[3],
                         cyc))
            print(rows[-1], flush=True)
    md = ["# Charged-sphere potential validation (Table 4), round 2", "",
          "%d^3 cells, h = 1, analytic Dirichlet data (Eq.18) on every boundary "
          "face cell, the paper's naive volume mapping (Q/V x covered sub-cell "
          "fraction) with subsampling s_f, V(2,2) to 1e-11 (`python "
          "scripts/table4_validation.py`).  The sphere sits at a shift (within one "
          "dx/s_f of the domain centre) whose covered-count gives the paper's "
          "printed e_rVmax, found by hill climbs on the shift (reading d11, "
          "DESIGN.md); `match` = e_rV prints as the paper's value (2 decimals).  Paper values: "
          "PAPER.md:1089-1118." % n, "",
          "| R | s_f | e_rV % (ours / paper e_rVmax) | match | L2 e_rPhi % (ours / paper) "
          "| inf e_rPhi % (ours / paper) | cycles |",
          "|---|---|---|---|---|---|---|"]
    for R, sf, ev, pev, ok, l2, pl2, inf, pinf, cyc in rows:
        md.append("| %d | %d | %.3f / %.2f | %s | %.3f / %.3f | %.2f / %.2f | %d |"
                  % (R, sf, ev, pev, "yes" if ok else "no", l2, pl2, inf, pinf, cyc))
    with open(a.out, "w") as fh:
        fh.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
