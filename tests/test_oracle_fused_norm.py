"""Oracle pins for reading c11: the optional fused
termination norm -- the cycle reports the norm of the level-0 residual it
computes after pre-smoothing (the one restricted to level 1) instead of a
separate post-cycle pass (the termination check is "negligible";
Alg.1).

Pinned against things other than the oracle's own norm routine:
* the iterates are those of the default mode, bit for bit (the norm only
  observes);
* the reported value is ||f + b - A phi|| of the pre-smoothed iterate with A
  the dense ghost-cell operator of tests/dense.py and b its BC shift (an
  independent assembly), phi reproduced from the previous iterate by the four
  pre-smoothing half-sweeps;
* solve() with the fused norm stops with the true residual below tol * r0.
"""
import numpy as np

import dense
import oracle

D, N = dense.DIRICHLET, dense.NEUMANN
SHAPE = (16, 8, 12)
H = 0.5
BT = [D, N, D, N, N, D]
BV = [0.25, -0.5, 1.0, 0.0, 0.75, -1.0]


def make(fused, f):
    o = oracle.Oracle(SHAPE, H, BT, BV, min_coarse=2, fused_norm=fused)
    o.set_rhs(f)
    return o


def dense_residual_norm(phi, f):
    A = dense.dense_operator(SHAPE, H, BT)
    b = dense.bc_rhs_shift(SHAPE, H, BT, BV)
    r = (f + b).reshape(-1) - A @ phi.reshape(-1)
    return float(np.linalg.norm(r))


def test_fused_norm_is_the_pre_smoothed_residual():
    f = np.random.default_rng(4).uniform(-1, 1, SHAPE)
    a, b = make(False, f), make(True, f)
    assert b.nlevels >= 2
    for _ in range(4):
        phi_before = b.phi()
        ra, rb = a.vcycle(), b.vcycle()
        # the norm only observes: identical iterates
        assert np.array_equal(a.phi(), b.phi())
        assert ra == a.residual_norm()
        # the pre-smoothed iterate, rebuilt step by step
        c = make(False, f)
        c.set_phi(phi_before)
        for _ in range(2):
            c.smooth_half(0, 0)
            c.smooth_half(0, 1)
        ref = dense_residual_norm(c.phi(), f)
        assert abs(rb - ref) <= 1e-12 * ref, (rb, ref)
        assert rb != ra


def test_fused_norm_solve_reaches_tolerance():
    f = np.random.default_rng(5).uniform(-1, 1, SHAPE)
    o = make(True, f)
    st, cyc, hist = o.solve(1e-9, 60)
    assert st == 0 and cyc >= 2
    assert hist[-1] <= 1e-9 * hist[0] < hist[-2]
    # the true residual of the final iterate is below the stopping value
    true = dense_residual_norm(o.phi(), f)
    assert true <= hist[-1]
    # the default mode needs no fewer cycles than one less
    st2, cyc2, _ = make(False, f).solve(1e-9, 60)
    assert st2 == 0 and abs(cyc2 - cyc) <= 1


def test_fused_norm_single_level_is_post_cycle():
    """No restriction on a single level: the post-cycle norm is reported."""
    f = np.random.default_rng(6).uniform(-1, 1, (6, 6, 6))
    o = oracle.Oracle((6, 6, 6), 1.0, [D] * 6, min_coarse=8, fused_norm=True)
    assert o.nlevels == 1
    o.set_rhs(f)
    r = o.vcycle()
    assert r == o.residual_norm()
