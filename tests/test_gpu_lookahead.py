"""The look-ahead red sweep (mg_api.cu lookahead_tail): a cycle's
norm takes its red residuals from the NEXT cycle's first red half-sweep,
written to a second red buffer, so the committed iterate is never touched by
work of a cycle that may not run.

Checked here: with and without it (mg_opts.disable MG_OFF_LOOKAHEAD) the
iterates are bitwise equal after every cycle and the norms agree to 1e-13
(red partials summed over another CTA grouping); both against the oracle;
and every API call that changes Phi, f or the operator between cycles (which
must drop the look-ahead) -- set_solution, set_rhs, zero_solution, a manual
half-sweep, a stopped solve, the asynchronous pipeline, eager (no graph)
cycles and profiling toggles -- leaves the two contexts bitwise equal.
"""
import numpy as np
import pytest

import oracle
from paper_1410_6609_b200 import workloads as W

pytestmark = pytest.mark.gpu

D, N, P = 0, 1, 2
# level 0 on the marching kernels (nz / 2 >= 64)
CASES = {
    "box": ((48, 40, 128), [D] * 6, [0.0, 0.5, -1.0, 0.0, 0.25, 0.0], 1.0 / 64),
    "neumann": ((32, 64, 136), [N, D, D, N, N, D], [0.1, 0.0, 0.5, -0.2, 0.0, 1.0], 0.5),
    "periodic": ((32, 32, 128), [P, P, P, P, D, D], [0.0, 0.0, 0.0, 0.0, 1.0, -1.0], 1.0),
}


@pytest.fixture(scope="module")
def mg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1410_6609_b200 import _build
    _build.build()
    from paper_1410_6609_b200 import mg as M
    return M


def pair(mg, case, **kw):
    shape, bt, bv, h = CASES[case]
    a = mg.Multigrid(shape, h, bt, bv, min_coarse=4, **kw)
    b = mg.Multigrid(shape, h, bt, bv, min_coarse=4, disable=mg.MG_OFF_LOOKAHEAD, **kw)
    return a, b


def same(a, b):
    assert np.array_equal(a.get_solution(), b.get_solution())


@pytest.mark.parametrize("case", sorted(CASES))
def test_lookahead_equals_plain_and_oracle(mg, case):
    shape, bt, bv, h = CASES[case]
    a, b = pair(mg, case)
    f = np.random.default_rng(5).uniform(-1, 1, shape)
    o = oracle.Oracle(shape, h, bt, bv, min_coarse=4)
    for s in (a, b):
        s.set_rhs(f)
    o.set_rhs(f)
    ho = [o.residual_norm()]
    ha, hb = [a.residual_norm()], [b.residual_norm()]
    for k in range(4):
        ha.append(a.vcycle())
        hb.append(b.vcycle())
        ho.append(o.vcycle())
        same(a, b)
        assert abs(ha[-1] - hb[-1]) <= 1e-13 * hb[-1], (k, ha[-1], hb[-1])
    assert a.cycle_paths & mg.MG_PATH_LOOKAHEAD
    assert not b.cycle_paths & mg.MG_PATH_LOOKAHEAD
    assert b.cycle_paths & mg.MG_PATH_SPLIT_NORM
    for x, y in zip(ha, ho):  # the history clause (reading c21)
        assert abs(x - y) <= 1e-8 * y + 1e-15 * ho[0], (x, y)
    po = o.phi()
    assert np.linalg.norm(a.get_solution() - po) <= 1e-10 * np.linalg.norm(po)
    # one launch fewer per cycle (the red residual pass)
    assert a.cycle_launches == b.cycle_launches - 1
    a.close()
    b.close()


@pytest.mark.parametrize("halo", ["loopback", "emulate"])
@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("case", ["box", "periodic"])
@pytest.mark.parametrize("overlap", [True, False])
def test_lookahead_slabs(mg, halo, nranks, case, overlap):
    """x-slabs (the NCCL data layout on one GPU for EMULATE): the look-ahead
    sweeps of every slab, the black ghost exchange before them and the red
    ghost exchange of the other buffers after them -- bitwise equal to the
    plain cycle, the norm to 1e-13, and to the oracle (history clause)."""
    shape, bt, bv, h = CASES[case]
    if shape[0] % (2 * nranks):
        pytest.skip("slabs of an odd plane count")
    kw = dict(nranks=nranks, halo=halo, agglomerate_below=4096,
              disable=0 if overlap else mg.MG_OFF_OVERLAP)
    a = mg.Multigrid(shape, h, bt, bv, min_coarse=4, **kw)
    kw["disable"] |= mg.MG_OFF_LOOKAHEAD
    b = mg.Multigrid(shape, h, bt, bv, min_coarse=4, **kw)
    f = np.random.default_rng(11).uniform(-1, 1, shape)
    o = oracle.Oracle(shape, h, bt, bv, min_coarse=4)
    for s in (a, b):
        s.set_rhs(f)
    o.set_rhs(f)
    ho = [o.residual_norm()]
    for k in range(3):
        ra, rb = a.vcycle(), b.vcycle()
        ho.append(o.vcycle())
        same(a, b)
        assert abs(ra - rb) <= 1e-13 * rb
        assert abs(ra - ho[-1]) <= 1e-8 * ho[-1] + 1e-15 * ho[0]
    assert a.cycle_paths & mg.MG_PATH_LOOKAHEAD
    assert bool(a.cycle_paths & mg.MG_PATH_OVERLAP) == overlap
    # a new iterate between cycles drops the look-ahead (the prologue runs
    # the exchanges itself)
    x = np.random.default_rng(12).uniform(-1, 1, shape)
    for s in (a, b):
        s.set_solution(x)
    for _ in range(2):
        ra, rb = a.vcycle(), b.vcycle()
        same(a, b)
    a.close()
    b.close()


@pytest.mark.parametrize("kind", ["beam", "random"])
def test_lookahead_masked(mg, kind):
    """Solid masks (byte-code levels, config 5's setting): the look-ahead
    sweep skips the solid cells' residuals and copies their values into the
    other buffer, so Phi -- solid cells included, whatever set_solution put
    there -- stays bitwise the plain cycle's; both against the oracle."""
    shape = (64, 32, 128)
    bt = [N, N, D, D, N, N]
    bv = [0.0, 0.0, 0.0, 1.0, 0.0, 0.0]
    if kind == "beam":
        solid = W.beam_mask(shape)
    else:
        solid = (np.random.default_rng(3).uniform(size=shape) < 0.1).astype(np.uint8)
    a = mg.Multigrid(shape, 1.0, bt, bv, min_coarse=4, nu1=3, nu2=3)
    b = mg.Multigrid(shape, 1.0, bt, bv, min_coarse=4, nu1=3, nu2=3,
                     disable=mg.MG_OFF_LOOKAHEAD)
    o = oracle.Oracle(shape, 1.0, bt, bv, solid=solid, min_coarse=4, nu1=3, nu2=3)
    rng = np.random.default_rng(4)
    f = rng.uniform(-1, 1, shape)
    for s in (a, b):
        s.set_mask(solid)
        s.set_rhs(f)
    o.set_rhs(f)
    ho = [o.residual_norm()]
    for _ in range(3):
        ra, rb = a.vcycle(), b.vcycle()
        ho.append(o.vcycle())
        same(a, b)
        assert abs(ra - rb) <= 1e-13 * rb
        assert abs(ra - ho[-1]) <= 1e-8 * ho[-1] + 1e-15 * ho[0]
    assert a.cycle_paths & mg.MG_PATH_LOOKAHEAD
    po = o.phi()
    assert np.linalg.norm(a.get_solution() - po) <= 1e-10 * np.linalg.norm(po)
    # nonzero values in solid cells survive the cycles on both paths alike
    x = rng.uniform(-1, 1, shape)
    for s in (a, b):
        s.set_solution(x)
    for _ in range(2):
        a.vcycle()
        b.vcycle()
        same(a, b)
    a.close()
    b.close()


def test_lookahead_interleaved_api_calls(mg):
    shape = CASES["box"][0]
    rng = np.random.default_rng(9)
    a, b = pair(mg, "box")
    f1, f2 = rng.uniform(-1, 1, shape), rng.uniform(-1, 1, shape)

    def both(fn):
        ra, rb = fn(a), fn(b)
        same(a, b)
        return ra, rb

    def cyc(s):
        return s.vcycle()

    both(lambda s: s.set_rhs(f1))
    for _ in range(2):
        both(cyc)
    # a new iterate between cycles
    phi = rng.uniform(-1, 1, shape)
    both(lambda s: s.set_solution(phi))
    ra, rb = both(cyc)
    assert abs(ra - rb) <= 1e-13 * rb
    # a new RHS between cycles
    both(lambda s: s.set_rhs(f2))
    both(cyc)
    # a manual half-sweep of level 0 between cycles
    both(lambda s: s.smooth_half(0, 0))
    both(cyc)
    both(lambda s: s.smooth_half(0, 1))
    both(cyc)
    # zeroed iterate
    both(lambda s: s.zero_solution())
    both(cyc)
    # a stopped solve returns the iterate of its last cycle (not the look-ahead)
    both(lambda s: s.set_rhs(f1))
    ra, rb = both(lambda s: s.solve(1e-6, 30))
    assert ra[1] == rb[1] and ra[0] == rb[0] == 0
    # and continuing afterwards
    both(cyc)
    # profiling on / off between cycles (the graphs are re-recorded)
    both(lambda s: s.set_profiling(True))
    both(cyc)
    both(lambda s: s.set_profiling(False))
    both(cyc)
    a.close()
    b.close()


def test_lookahead_eager_cycles(mg):
    shape = CASES["periodic"][0]
    a, b = pair(mg, "periodic", use_graph=False)
    f = np.random.default_rng(2).uniform(-1, 1, shape)
    for s in (a, b):
        s.set_rhs(f)
    for _ in range(3):
        ra, rb = a.vcycle(), b.vcycle()
        same(a, b)
        assert abs(ra - rb) <= 1e-13 * rb
    assert a.cycle_paths & mg.MG_PATH_LOOKAHEAD
    a.close()
    b.close()


def test_lookahead_async_pipeline(mg):
    import torch
    shape = CASES["box"][0]
    st = torch.cuda.Stream()
    a, b = pair(mg, "box", stream=st)
    rng = np.random.default_rng(13)
    fs = [rng.uniform(-1, 1, shape) for _ in range(3)]
    outs = {}
    for name, s in (("a", a), ("b", b)):
        res = [np.empty(shape) for _ in fs]
        for f, r in zip(fs, res):
            s.solve_async(f, r, 5)
        s.wait()
        outs[name] = res
    for x, y in zip(outs["a"], outs["b"]):
        assert np.array_equal(x, y)
    a.close()
    b.close()


def test_timestep_single_cycle_plain(mg):
    # one cycle per new RHS takes the plain form (the look-ahead would be
    # discarded by the next RHS)
    w = W.cfg4(P=1, n=128, seed=0)
    a = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=w.min_coarse, nu1=3,
                     nu2=3)
    b = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=w.min_coarse, nu1=3,
                     nu2=3, disable=mg.MG_OFF_LOOKAHEAD)
    for s in (a, b):
        s.timestep(w.centers, w.radii, w.charges, cycles=1)
    assert not a.cycle_paths & mg.MG_PATH_LOOKAHEAD
    same(a, b)
    for s in (a, b):
        s.timestep(w.centers, w.radii, w.charges, cycles=2)
    assert a.cycle_paths & mg.MG_PATH_LOOKAHEAD
    same(a, b)
    a.close()
    b.close()


hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings, strategies as st  # noqa: E402

OPS = ["vcycle", "vcycle", "vcycle", "set_rhs", "set_solution", "zero", "smooth0",
       "smooth1", "residual_norm", "get_solution", "solve", "profiling", "mask_bc",
       "solve_async"]


@settings(max_examples=30, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])
@given(st.sampled_from(sorted(CASES)), st.lists(st.sampled_from(OPS), min_size=4, max_size=14),
       st.integers(0, 2 ** 16))
def test_lookahead_random_call_sequences(mg, case, ops, seed):
    """Random sequences of API calls on a look-ahead context and a plain one
    (MG_OFF_LOOKAHEAD): after every call Phi is bitwise equal and the
    returned norms agree to 1e-13."""
    shape, bt, bv, h = CASES[case]
    rng = np.random.default_rng(seed)
    a, b = pair(mg, case)
    f = rng.uniform(-1, 1, shape)
    for s in (a, b):
        s.set_rhs(f)
    prof = False
    for op in ops:
        if op == "vcycle":
            ra, rb = a.vcycle(), b.vcycle()
            assert abs(ra - rb) <= 1e-13 * rb
        elif op == "set_rhs":
            f = rng.uniform(-1, 1, shape)
            a.set_rhs(f)
            b.set_rhs(f)
        elif op == "set_solution":
            x = rng.uniform(-1, 1, shape)
            a.set_solution(x)
            b.set_solution(x)
        elif op == "zero":
            a.zero_solution()
            b.zero_solution()
        elif op in ("smooth0", "smooth1"):
            a.smooth_half(0, int(op[-1]))
            b.smooth_half(0, int(op[-1]))
        elif op == "residual_norm":
            assert a.residual_norm() == b.residual_norm()
        elif op == "get_solution":
            pass
        elif op == "solve":
            ra, rb = a.solve(1e-5, 6), b.solve(1e-5, 6)
            assert ra[1] == rb[1]
        elif op == "profiling":
            prof = not prof
            a.set_profiling(prof)
            b.set_profiling(prof)
        elif op == "mask_bc":
            # new boundary values on one face (f changes by the BC adaptation)
            if bt[1] != P:
                v = rng.uniform(-1, 1, (shape[1], shape[2]))
                a.set_face_values(1, v)
                b.set_face_values(1, v)
        elif op == "solve_async":
            outs = [np.empty(shape), np.empty(shape)]
            a.solve_async(f, outs[0], 2)
            b.solve_async(f, outs[1], 2)
            a.wait()
            b.wait()
            assert np.array_equal(outs[0], outs[1])
        same(a, b)
    a.close()
    b.close()
