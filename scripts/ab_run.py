"""A/B runner for kernel experiments: run a script with the binding pointed
at another build of the library (ab/*.so, untracked).
    python scripts/ab_run.py ab/libmg_X.so scripts/cg_probe.py [args...]"""
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1410_6609_b200 import _build, mg  # noqa: E402

_build.build = lambda *a, **k: mg.LIB_PATH  # do not rebuild the default library
mg.LIB_PATH = os.path.abspath(sys.argv[1])
sys.argv = sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
