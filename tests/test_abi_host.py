"""CPU-only checks of the C-ABI library: it loads without a GPU, exports every
function include/mg.h declares, and its host-side planning (hierarchy rule,
slab ownership, agglomeration level, workspace size) is right."""
import os
import re

import numpy as np
import pytest

import oracle
from paper_1410_6609_b200 import _build, mg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    _build.build()
    oracle.build()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "mg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(mg_[a-z_0-9]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 20
    L = mg.lib()
    for n in names:
        assert hasattr(L, n), n


def test_every_declaration_is_documented():
    """Each entry point of include/mg.h is preceded by a comment block (its
    semantics, arguments, errors; the paper passage where there is one), and
    the header cites the paper (P:line) for the operations it defines."""
    src = open(os.path.join(ROOT, "include", "mg.h")).read()
    decls = list(re.finditer(r"^(?:int|void|size_t|const char \*|void \*)\s*\**\s*"
                             r"(mg_[a-z_0-9]+)\s*\(", src, flags=re.M))
    assert len(decls) >= 20
    for m in decls:
        # a comment block ends right above the declaration or above the
        # contiguous group of declarations it belongs to (no blank line)
        end = src.rfind("*/", 0, m.start())
        gap = src[end + 2:m.start()]
        assert end >= 0 and "\n\n" not in gap, "undocumented: " + m.group(1)
    cites = re.findall(r"P:\d+", src)
    assert len(cites) >= 20
    for op in ("mg_set_rhs_from_spheres", "mg_vcycle", "mg_solve", "mg_coulomb_forces",
               "mg_timestep", "mg_set_permittivity", "mg_residual_norm"):
        i = src.index(op + "(")
        block = src[src.rindex("/*", 0, i):i]
        assert "P:" in block or "Alg." in block or "reading" in block, op


def test_no_oracle_in_product():
    """The product never references the oracle (no shared code)."""
    pkg = os.path.join(ROOT, "paper_1410_6609_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "mg_oracle" not in txt, f
                assert "orc_" not in txt, f


def test_create_without_gpu_fails_loudly():
    """No CPU fallback: without a device the library returns an error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(mg.MGError):
        mg.Multigrid((8, 8, 8), 1.0, [0] * 6)
    bc = (mg.mg_bc * 6)(*[mg.mg_bc(0, 0.0)] * 6)
    assert not mg.lib().mg_create(8, 8, 8, 1.0, bc)
    assert b"MG_ERR_CUDA" in mg.lib().mg_last_error(None)


def test_missing_extension_fails_loudly(monkeypatch, tmp_path):
    """No CPU fallback: with the shared library absent, loading it (and so
    every product call) raises ImportError instead of computing anything
    elsewhere; a solver's construction raises too (MGError first when no
    device is present, ImportError from the loader on a GPU box)."""
    monkeypatch.setattr(mg, "_lib", None)
    monkeypatch.setattr(mg, "LIB_PATH", str(tmp_path / "libmg_cuda.so"))
    with pytest.raises(ImportError, match="no CPU fallback"):
        mg.lib()
    with pytest.raises((ImportError, mg.MGError)):
        mg.Multigrid((8, 8, 8), 1.0, [0] * 6)


@pytest.mark.parametrize("shape,mc", [((32, 32, 32), 4), ((256, 64, 64), 4),
                                      ((512, 512, 512), 8), ((64, 16, 48), 2),
                                      ((24, 24, 24), 2), ((2, 2, 2), 1)])
def test_plan_hierarchy_equals_oracle(shape, mc):
    dims, lnx, agg = mg.plan(shape, min_coarse=mc)
    o = oracle.Oracle(shape, 1.0, [0] * 6, min_coarse=mc) \
        if np.prod(shape) <= 64 ** 3 * 8 else None
    if o is not None:
        assert dims == [o.dims(l) for l in range(o.nlevels)]
    assert agg == len(dims)
    assert all(x == 0 for x in lnx)


def test_plan_multi_rank_agglomeration():
    # config 4 at P = 8: 4096 x 512 x 512, slabs of 512 planes
    dims, lnx, agg = mg.plan((4096, 512, 512), min_coarse=8, nranks=8,
                             halo="nccl")
    assert dims[-1] == (64, 8, 8)
    assert lnx[0] == 512 and lnx[1] == 256 and lnx[2] == 128 and lnx[3] == 64
    # local 64^3 at level 3 is kept distributed; level 4 (32^3 local) is whole
    assert agg == 4
    # config 5 at P = 8: 2048 x 512 x 512
    dims, lnx, agg = mg.plan((2048, 512, 512), min_coarse=8, nranks=8,
                             halo="nccl")
    assert dims[-1] == (32, 8, 8)
    assert agg == 3  # level 3 local 32 x 64 x 64 < 64^3


def test_plan_errors():
    with pytest.raises(mg.MGError) as e:
        mg.plan((7, 8, 8))
    assert e.value.code == mg.MG_ERR_COARSEN
    with pytest.raises(mg.MGError):
        mg.plan((0, 8, 8))
    with pytest.raises(mg.MGError):
        mg.plan((48, 8, 8), nranks=5, halo="nccl")
    with pytest.raises(mg.MGError):
        mg.plan((6, 8, 8), nranks=2, halo="nccl")  # 3 planes per rank


def test_workspace_bytes_model():
    """Split layout: 4 fields per level, ghost planes/rows, pitch
    nz/2 -> x4; no device query (the same bytes on any SM count).  One
    level-0 slab: a fifth level-0 array, the look-ahead red buffer."""
    nb = mg.workspace_bytes((512, 512, 512), min_coarse=8)
    fine = 5 * 514 * 514 * 256 * 8  # (any slab count: one look-ahead array per slab)
    assert fine < nb < fine * 1.2
    nb1 = mg.workspace_bytes((512, 512, 512), min_coarse=8, disable=mg.MG_OFF_LOOKAHEAD)
    assert nb - nb1 == 514 * 514 * 256 * 8
    assert mg.workspace_bytes((512, 512, 512), min_coarse=8, fused_norm=True) == nb1
    nb2 = mg.workspace_bytes((1024, 512, 512), min_coarse=8, nranks=2,
                             halo="nccl")
    slab = 5 * 514 * 514 * 256 * 8
    assert slab < nb2 < slab * 1.2
    assert mg.workspace_bytes((7, 8, 8)) == 0


def test_opts_struct_matches_header():
    """The ctypes mirror of mg_opts ends with the fields mg.h declares last,
    and the MG_OFF_* / MG_PATH_* bits equal the header's."""
    src = open(os.path.join(ROOT, "include", "mg.h")).read()
    body = src[src.index("typedef struct {\n  int nu1"):src.index("} mg_opts;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"(\w+)(?:\[\d+\])?;", body)
    names = [n for n, _ in mg.mg_opts._fields_]
    assert fields[-5:] == names[-5:] == ["use_graph", "fused_norm", "disable",
                                         "nccl_timeout_ms", "tail_cells"]
    for m in re.finditer(r"#define (MG_(?:OFF|PATH)_\w+) (\d+)", src):
        assert getattr(mg, m.group(1)) == int(m.group(2)), m.group(1)


def test_nccl_unique_id_on_cpu():
    try:
        uid = mg.nccl_unique_id()
    except mg.MGError as e:
        pytest.skip("libnccl not loadable here: %s" % e)
    assert len(uid) == 128 and any(uid)


def test_move_spheres_generator():
    """Synthetic motion for the time-stepping regime: deterministic per
    (seed, step), bounded displacement, reflected into [R, L-R] on wall axes,
    wrapped into [0, L) on periodic axes."""
    from paper_1410_6609_b200 import workloads as W
    w = W.timestep_workload(n=64, seed=1)
    L = np.array(w.shape, float)
    a = W.move_spheres(w.centers, w.radii, L, 3, seed=9, amplitude=0.5)
    b = W.move_spheres(w.centers, w.radii, L, 3, seed=9, amplitude=0.5)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, W.move_spheres(w.centers, w.radii, L, 4, seed=9))
    assert np.abs(a - w.centers).max() <= 0.5 + 1e-12
    R = w.radii[:, None]
    assert np.all(a >= R) and np.all(a <= L - R)
    c = np.array([[0.1, 32.0, 63.95]])
    p = W.move_spheres(c, [6.0], L, 1, seed=0, amplitude=0.2,
                       periodic=(True, False, True))
    assert np.all((p[:, [0, 2]] >= 0) & (p[:, [0, 2]] < L[[0, 2]]))
