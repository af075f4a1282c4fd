"""One random-parity case against the oracle under path switches (debugging
aid): python scripts/repro_case.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from paper_1410_6609_b200 import _build  # noqa: E402
_build.build()
from paper_1410_6609_b200 import mg  # noqa: E402

shape, bt, bv, h, nu1, nu2, mc, slabs, seed = ((8, 4, 64), [0, 0, 0, 0, 2, 2], [0.0] * 6,
                                               1.0, 1, 0, 1, 2, 0)
kw = dict(min_coarse=mc, nu1=nu1, nu2=nu2)
f = np.random.default_rng(seed).uniform(-1, 1, shape)
o = oracle.Oracle(shape, h, bt, bv, **kw)
o.set_rhs(f)
ho = [o.residual_norm()] + [o.vcycle() for _ in range(3)]
print("oracle", ho, "levels", o.nlevels)
for sl in (1, 2):
    for dis in (0, mg.MG_OFF_MARCH, mg.MG_OFF_OVERLAP, mg.MG_OFF_TAIL, mg.MG_OFF_RED0,
                mg.MG_OFF_LOOKAHEAD, mg.MG_OFF_SPLIT_NORM, 255):
        extra = dict(nranks=sl, halo="loopback", agglomerate_below=512) if sl > 1 else {}
        s = mg.Multigrid(shape, h, bt, bv, disable=dis, **kw, **extra)
        s.set_rhs(f)
        hg = [s.residual_norm()] + [s.vcycle() for _ in range(3)]
        ok = all(abs(a - b) <= 1e-8 * b + 1e-15 * ho[0] for a, b in zip(hg, ho))
        print("slabs", sl, "disable", dis, "levels", s.nlevels, "paths", hex(s.cycle_paths),
              "ok" if ok else "MISMATCH", ["%.6g" % x for x in hg])
        s.close()
