"""Build libmg_cuda.so in-tree with nvcc for sm_100a (no JIT, no torch ext)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmg_cuda.so")
ROOT = os.path.dirname(HERE)


def _nccl_include() -> str:
    try:
        import nvidia.nccl  # type: ignore
        for p in nvidia.nccl.__path__:
            inc = os.path.join(p, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except Exception:
        pass
    return "/usr/include"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return (sources() + glob.glob(os.path.join(CSRC, "*.h"))
            + glob.glob(os.path.join(CSRC, "*.cuh"))
            + [os.path.join(ROOT, "include", "mg.h"), __file__])


def nvcc_cmd(out=LIB, extra=()):
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    return [nvcc, "-O3", "-std=c++17",
            "-gencode", "arch=compute_100a,code=sm_100a",
            "-lineinfo", "-fmad=false", "-Xptxas", "-v",
            "-Xcompiler", "-fPIC,-ffp-contract=off",
            "-shared", "-I" + _nccl_include(), "-I" + os.path.join(ROOT, "include"),
            *extra, "-o", out, *sources(), "-ldl"]


def build(force: bool = False, verbose: bool = False) -> str:
    if (not force and os.path.exists(LIB)
            and os.path.getmtime(LIB) >= max(os.path.getmtime(p) for p in _deps())):
        return LIB
    cmd = nvcc_cmd()
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stderr[-4000:])
    if verbose:
        print(res.stderr)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
