"""Random API call sequences on a look-ahead and a plain context, printing each
call (debugging aid for tests/test_gpu_lookahead.py):
python scripts/la_repro.py [n_sequences] [first]"""
import faulthandler
import os
import sys

import numpy as np

faulthandler.enable()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_1410_6609_b200 import _build  # noqa: E402
_build.build()
from paper_1410_6609_b200 import mg  # noqa: E402
from test_gpu_lookahead import CASES, OPS, P  # noqa: E402

nseq = int(sys.argv[1]) if len(sys.argv) > 1 else 30
q0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for q in range(q0, nseq):
    rng = np.random.default_rng(q)
    case = sorted(CASES)[q % 3]
    shape, bt, bv, h = CASES[case]
    ops = [OPS[i] for i in rng.integers(0, len(OPS), rng.integers(4, 15))]
    print("seq", q, case, ops, flush=True)
    a = mg.Multigrid(shape, h, bt, bv, min_coarse=4)
    b = mg.Multigrid(shape, h, bt, bv, min_coarse=4, disable=mg.MG_OFF_LOOKAHEAD)
    f = rng.uniform(-1, 1, shape)
    for s in (a, b):
        s.set_rhs(f)
    prof = False
    for op in ops:
        print("  ", op, flush=True)
        if op == "vcycle":
            ra, rb = a.vcycle(), b.vcycle()
            assert abs(ra - rb) <= 1e-13 * rb, (ra, rb)
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
            x, y = a.residual_norm(), b.residual_norm()
            assert x == y, (x, y)
        elif op == "solve":
            ra, rb = a.solve(1e-5, 6), b.solve(1e-5, 6)
            assert ra[1] == rb[1], (ra, rb)
        elif op == "profiling":
            prof = not prof
            a.set_profiling(prof)
            b.set_profiling(prof)
        elif op == "mask_bc":
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
        assert np.array_equal(a.get_solution(), b.get_solution()), op
    print("  close", flush=True)
    a.close()
    b.close()
print("ok")
