"""Python binding of libmg_cuda.so (include/mg.h) -- argument marshalling only.

Every step of the solve runs in the CUDA library; PyTorch is used for device
memory (the workspace is a torch uint8 tensor), the current CUDA stream and,
for multi-GPU runs, the broadcast of the NCCL unique id through
torch.distributed.  There is no CPU fallback: importing this module without
the built extension, or creating a solver without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmg_cuda.so")

MG_OK = 0
MG_ERR_ARG = -1
MG_ERR_BC = -2
MG_ERR_COARSEN = -3
MG_ERR_CUDA = -4
MG_ERR_NCCL = -5
MG_ERR_NOMEM = -6
MG_ERR_DIVERGED = -7
MG_ERR_NOTCONV = -8

MG_DIRICHLET = 0
MG_NEUMANN = 1
MG_PERIODIC = 2
MG_HOST = 0
MG_DEVICE = 1
MG_CHARGE_PER_CELLS = 0
MG_CHARGE_PER_VOLUME = 1
MG_FIELD_PHI = 0
MG_FIELD_RHS = 1
MG_HALO_NONE = 0
MG_HALO_NCCL = 1
MG_HALO_LOOPBACK = 2
MG_HALO_EMULATE = 3
# mg_opts.disable bits / mg_cycle_paths bits (include/mg.h)
MG_OFF_MARCH, MG_OFF_OVERLAP, MG_OFF_SPLIT_NORM = 1, 2, 4
MG_OFF_CG_CLUSTER, MG_OFF_MASK_CODES, MG_OFF_TAIL, MG_OFF_RED0 = 8, 16, 32, 64
MG_PATH_MARCH, MG_PATH_OVERLAP, MG_PATH_SPLIT_NORM, MG_PATH_CG_CLUSTER = 1, 2, 4, 8
MG_PATH_CG_VAR, MG_PATH_PROLONG_FUSED, MG_PATH_FUSED_NORM, MG_PATH_TAIL = 16, 32, 64, 128
MG_PATH_RED0 = 256
MG_OFF_LOOKAHEAD, MG_PATH_LOOKAHEAD = 128, 512

_HALO = {"none": MG_HALO_NONE, "nccl": MG_HALO_NCCL, "loopback": MG_HALO_LOOPBACK,
         "emulate": MG_HALO_EMULATE}


class MGError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class mg_bc(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("value", ctypes.c_double)]


class mg_opts(ctypes.Structure):
    _fields_ = [("nu1", ctypes.c_int), ("nu2", ctypes.c_int),
                ("alpha", ctypes.c_double), ("min_coarse", ctypes.c_int),
                ("max_levels", ctypes.c_int),
                ("agglomerate_below", ctypes.c_longlong),
                ("coarse_tol", ctypes.c_double), ("coarse_maxit", ctypes.c_int),
                ("max_cycles", ctypes.c_int), ("device", ctypes.c_int),
                ("stream", ctypes.c_void_p), ("rank", ctypes.c_int),
                ("nranks", ctypes.c_int), ("halo_backend", ctypes.c_int),
                ("nccl_id", ctypes.c_ubyte * 128),
                ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t),
                ("use_graph", ctypes.c_int), ("fused_norm", ctypes.c_int),
                ("disable", ctypes.c_int), ("nccl_timeout_ms", ctypes.c_int),
                ("tail_cells", ctypes.c_longlong)]


_lib = None


def lib():
    """Load libmg_cuda.so; raises if the extension has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                "libmg_cuda.so is missing: run __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, i, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        dp = ctypes.c_void_p  # pointers passed as integers (host or device)
        ip = ctypes.POINTER(ctypes.c_int)
        L.mg_default_opts.argtypes = [ctypes.POINTER(mg_opts)]
        L.mg_default_opts.restype = None
        L.mg_plan.argtypes = [i, i, i, ctypes.POINTER(mg_opts), ip, ip,
                              ctypes.POINTER(ctypes.c_int * 3), ip]
        L.mg_workspace_bytes.argtypes = [i, i, i, ctypes.POINTER(mg_opts)]
        L.mg_workspace_bytes.restype = ctypes.c_size_t
        L.mg_create.argtypes = [i, i, i, d, ctypes.POINTER(mg_bc)]
        L.mg_create.restype = P
        L.mg_create_ex.argtypes = [i, i, i, d, ctypes.POINTER(mg_bc),
                                   ctypes.POINTER(mg_opts)]
        L.mg_create_ex.restype = P
        L.mg_destroy.argtypes = [P]
        L.mg_destroy.restype = None
        L.mg_last_error.argtypes = [P]
        L.mg_last_error.restype = ctypes.c_char_p
        L.mg_last_error_code.argtypes = []
        L.mg_strerror.argtypes = [i]
        L.mg_strerror.restype = ctypes.c_char_p
        L.mg_nccl_unique_id.argtypes = [ctypes.c_ubyte * 128]
        L.mg_halo_schedule.argtypes = [i, i, i, ctypes.c_int * 12]
        L.mg_set_rhs_from_spheres.argtypes = [P, i, dp, dp, dp, i, i]
        L.mg_set_rhs.argtypes = [P, dp, i]
        L.mg_vcycle.argtypes = [P, ctypes.POINTER(ctypes.c_double)]
        L.mg_solve_async.argtypes = [P, dp, i, dp, i, i]
        L.mg_wait.argtypes = [P, ctypes.POINTER(ctypes.c_double)]
        L.mg_get_solution_async.argtypes = [P, dp, i]
        L.mg_solve.argtypes = [P, d, ip, dp]
        L.mg_solve_n.argtypes = [P, d, i, ip, dp]
        L.mg_residual_norm.argtypes = [P, ctypes.POINTER(ctypes.c_double)]
        L.mg_get_solution.argtypes = [P, dp, i]
        L.mg_set_solution.argtypes = [P, dp, i]
        L.mg_zero_solution.argtypes = [P]
        L.mg_num_levels.argtypes = [P]
        L.mg_level_dims.argtypes = [P, i, ctypes.c_int * 3]
        L.mg_get_field.argtypes = [P, i, i, dp, i]
        L.mg_set_field.argtypes = [P, i, i, dp, i]
        L.mg_smooth_half.argtypes = [P, i, i, i]
        L.mg_residual_restrict.argtypes = [P, i]
        L.mg_prolong_correct.argtypes = [P, i]
        L.mg_coarse_solve.argtypes = [P, ip]
        L.mg_set_mask.argtypes = [P, dp, i]
        L.mg_set_bc_patch.argtypes = [P, i, i, i, i, i, i, d]
        L.mg_set_face_values.argtypes = [P, i, dp]
        L.mg_set_permittivity.argtypes = [P, dp, i]
        L.mg_coulomb_forces.argtypes = [P, i, dp, dp, dp, i, i, dp]
        L.mg_timestep.argtypes = [P, i, dp, dp, dp, i, i, i, d, dp, i, ip,
                                  ctypes.POINTER(ctypes.c_double)]
        L.mg_get_stencil.argtypes = [P, i, dp, i]
        L.mg_set_profiling.argtypes = [P, i]
        L.mg_last_cycle_times.argtypes = [P, ctypes.c_double * 8]
        L.mg_last_cycle_times_ex.argtypes = [P, ctypes.c_double * 12, i]
        L.mg_cycle_launches.argtypes = [P]
        L.mg_cycle_paths.argtypes = [P]
        L.mg_stream.argtypes = [P]
        L.mg_stream.restype = ctypes.c_void_p
        _lib = L
    return _lib


def _check(rc, ctx=None):
    if rc != MG_OK:
        msg = lib().mg_last_error(ctx).decode()
        raise MGError(rc, msg)
    return rc


MG_OP_SEND, MG_OP_RECV = 0, 1
MG_PLANE_FIRST, MG_PLANE_LAST, MG_GHOST_LO, MG_GHOST_HI = 1, 2, 3, 4


def halo_schedule(nranks: int, rank: int, periodic_x: bool):
    """Ordered ghost-plane operations [(op, peer, plane), ...] the library
    posts in one NCCL group on this rank (mg_halo_schedule; host logic)."""
    ops = (ctypes.c_int * 12)()
    n = lib().mg_halo_schedule(int(nranks), int(rank), 1 if periodic_x else 0, ops)
    if n < 0:
        raise MGError(n, "bad rank / nranks")
    return [tuple(ops[3 * k:3 * k + 3]) for k in range(n)]


def default_opts() -> mg_opts:
    o = mg_opts()
    lib().mg_default_opts(ctypes.byref(o))
    return o


def make_opts(nu1=2, nu2=2, alpha=2.0, min_coarse=4, max_levels=0,
              agglomerate_below=64 ** 3, coarse_tol=1e-12, coarse_maxit=1000,
              max_cycles=100, device=0, rank=0, nranks=1, halo="none",
              nccl_id: Optional[bytes] = None, use_graph=True,
              fused_norm=False, disable=0, nccl_timeout_ms=600000,
              tail_cells=0) -> mg_opts:
    o = default_opts()
    o.nu1, o.nu2, o.alpha = nu1, nu2, alpha
    o.min_coarse, o.max_levels = min_coarse, max_levels
    o.agglomerate_below = int(agglomerate_below)
    o.coarse_tol, o.coarse_maxit, o.max_cycles = coarse_tol, coarse_maxit, max_cycles
    o.device, o.rank, o.nranks = device, rank, nranks
    o.halo_backend = _HALO[halo] if isinstance(halo, str) else int(halo)
    if nccl_id is not None:
        ctypes.memmove(o.nccl_id, bytes(nccl_id), 128)
    o.use_graph = 1 if use_graph else 0
    o.fused_norm = 1 if fused_norm else 0  # reading c11 (include/mg.h)
    o.disable = int(disable)  # MG_OFF_* bits
    o.nccl_timeout_ms = int(nccl_timeout_ms)
    o.tail_cells = int(tail_cells)
    return o


def plan(shape, **kw):
    """Level plan (no GPU needed): (dims per level, local_nx, agg_level)."""
    o = make_opts(**kw)
    nl, agg = ctypes.c_int(), ctypes.c_int()
    dims = (ctypes.c_int * 3 * 32)()
    lnx = (ctypes.c_int * 32)()
    _check(lib().mg_plan(int(shape[0]), int(shape[1]), int(shape[2]),
                         ctypes.byref(o), ctypes.byref(nl), ctypes.byref(agg),
                         dims, lnx))
    L = nl.value
    return [tuple(dims[l]) for l in range(L)], list(lnx[:L]), agg.value


def workspace_bytes(shape, **kw) -> int:
    o = make_opts(**kw)
    return int(lib().mg_workspace_bytes(int(shape[0]), int(shape[1]),
                                        int(shape[2]), ctypes.byref(o)))


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _check(lib().mg_nccl_unique_id(buf))
    return bytes(buf)


def _host_ptr(a: np.ndarray):
    return a.ctypes.data


class Multigrid:
    """One solver context (see include/mg.h).

    shape: global (nx, ny, nz); bc_type / bc_value: 6 faces x-,x+,y-,y+,z-,z+.
    The workspace is a torch uint8 CUDA tensor owned by this object.
    """

    def __init__(self, shape: Sequence[int], h: float, bc_type, bc_value=None,
                 *, device: int = 0, torch_workspace: bool = True, stream=None,
                 **kw):
        import torch
        if not torch.cuda.is_available():
            raise MGError(MG_ERR_CUDA, "no CUDA device: the multigrid solver "
                                       "has no CPU path")
        self._torch = torch
        if bc_value is None:
            bc_value = [0.0] * 6
        bcs = (mg_bc * 6)(*[mg_bc(int(t), float(v))
                            for t, v in zip(bc_type, bc_value)])
        self.shape = tuple(int(s) for s in shape)
        o = make_opts(device=device, **kw)
        self._plan_kw = {k: v for k, v in kw.items()
                         if k in ("min_coarse", "max_levels", "agglomerate_below",
                                  "nranks", "rank", "halo")}
        self._plan = None
        self._stream = stream  # a torch.cuda.Stream kept alive while in use
        if stream is not None:
            o.stream = stream.cuda_stream
        self.nranks = o.nranks
        self.rank = o.rank
        self.halo = o.halo_backend
        self.device = torch.device("cuda", device)
        self._ws = None
        if torch_workspace:
            nb = lib().mg_workspace_bytes(*self.shape, ctypes.byref(o))
            if nb == 0:
                raise MGError(lib().mg_last_error_code(),
                              lib().mg_last_error(None).decode())
            self._ws = torch.empty(nb + 256, dtype=torch.uint8, device=self.device)
            o.workspace = self._ws.data_ptr()
            o.workspace_bytes = nb + 256
        self._ctx = lib().mg_create_ex(*self.shape, float(h), bcs, ctypes.byref(o))
        if not self._ctx:
            raise MGError(lib().mg_last_error_code(),
                          lib().mg_last_error(None).decode())
        self.h = float(h)

    def close(self):
        if getattr(self, "_ctx", None):
            lib().mg_destroy(self._ctx)
            self._ctx = None
        self._ws = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- geometry -----------------------------------------------------------
    @property
    def nlevels(self) -> int:
        return lib().mg_num_levels(self._ctx)

    def level_dims(self, level: int):
        d = (ctypes.c_int * 3)()
        _check(lib().mg_level_dims(self._ctx, level, d), self._ctx)
        return tuple(d)

    def local_shape(self, level: int = 0):
        """Shape of the arrays exchanged for `level` (the slab for NCCL)."""
        if self._plan is None:
            self._plan = plan(self.shape, **self._plan_kw)
        dims, lnx, agg = self._plan
        d = dims[level]
        if self.nranks > 1 and self.halo == MG_HALO_NCCL and level < agg:
            return (lnx[level], d[1], d[2])
        return d

    # -- data movement (host numpy arrays or torch CUDA tensors) -------------
    def _io_args(self, a, level=0):
        """Pointer and MG_HOST / MG_DEVICE of a natural-layout buffer of
        `level` (the library copies prod(local_shape(level)) doubles)."""
        torch = self._torch
        n = int(np.prod(self.local_shape(level)))
        if isinstance(a, torch.Tensor):
            assert a.dtype == torch.float64 and a.is_contiguous()
            if a.numel() != n:
                raise MGError(MG_ERR_ARG, "buffer of %d values, need %d" % (a.numel(), n))
            if a.is_cuda:
                torch.cuda.current_stream(a.device).synchronize()
                return a.data_ptr(), MG_DEVICE
            return a.data_ptr(), MG_HOST
        assert isinstance(a, np.ndarray) and a.dtype == np.float64 \
            and a.flags["C_CONTIGUOUS"]
        if a.size != n:
            raise MGError(MG_ERR_ARG, "buffer of %d values, need %d" % (a.size, n))
        return _host_ptr(a), MG_HOST

    def set_rhs(self, f):
        ptr, where = self._io_args(f)
        _check(lib().mg_set_rhs(self._ctx, ptr, where), self._ctx)

    def set_rhs_from_spheres(self, centers, radii, charges,
                             normalization=MG_CHARGE_PER_CELLS, subsample=1):
        c = np.ascontiguousarray(centers, np.float64).reshape(-1)
        r = np.ascontiguousarray(radii, np.float64)
        q = np.ascontiguousarray(charges, np.float64)
        _check(lib().mg_set_rhs_from_spheres(self._ctx, len(r), _host_ptr(c),
                                             _host_ptr(r), _host_ptr(q),
                                             normalization, subsample),
               self._ctx)

    def coulomb_forces(self, centers, radii, charges,
                       normalization=MG_CHARGE_PER_CELLS, subsample=1):
        """Eq.14 forces (n, 3) on the spheres from the current solution."""
        c = np.ascontiguousarray(centers, np.float64).reshape(-1)
        r = np.ascontiguousarray(radii, np.float64)
        q = np.ascontiguousarray(charges, np.float64)
        out = np.empty(3 * len(r), np.float64)
        _check(lib().mg_coulomb_forces(self._ctx, len(r), _host_ptr(c),
                                       _host_ptr(r), _host_ptr(q), normalization,
                                       subsample, _host_ptr(out)), self._ctx)
        return out.reshape(-1, 3)

    def solve_async(self, f, phi_out, cycles: int):
        """Enqueue f -> Phi = 0 -> `cycles` V-cycles -> phi_out on the
        context's stream without host synchronisation (mg_solve_async); use
        pinned host tensors (or CUDA tensors) to overlap transfers with the
        cycles of another context.  Call wait() before reading phi_out."""
        fp, fw = self._io_args_nosync(f)
        pp, pw = self._io_args_nosync(phi_out)
        _check(lib().mg_solve_async(self._ctx, fp, fw, pp, pw, int(cycles)),
               self._ctx)

    def get_solution_async(self, out):
        """Enqueue the copy-out of Phi into `out` (a pinned host or CUDA
        float64 tensor of the slab's shape) without host synchronisation
        (mg_get_solution_async); the download overlaps the work enqueued
        next.  Call wait() before reading `out`."""
        p, w = self._io_args_nosync(out)
        _check(lib().mg_get_solution_async(self._ctx, p, w), self._ctx)

    def wait(self) -> float:
        r = ctypes.c_double(0.0)
        _check(lib().mg_wait(self._ctx, ctypes.byref(r)), self._ctx)
        return r.value

    def _io_args_nosync(self, a):
        """Pointer of a level-0 slab buffer for the asynchronous calls: the
        library copies prod(local_shape(0)) doubles through it, so the size
        is checked here (an undersized buffer would be read or written out
        of bounds long after the call returned)."""
        if a is None:
            return None, MG_HOST
        torch = self._torch
        n = int(np.prod(self.local_shape(0)))
        if isinstance(a, torch.Tensor):
            assert a.dtype == torch.float64 and a.is_contiguous()
            if a.numel() != n:
                raise MGError(MG_ERR_ARG, "buffer of %d values, need %d" % (a.numel(), n))
            return a.data_ptr(), (MG_DEVICE if a.is_cuda else MG_HOST)
        assert isinstance(a, np.ndarray) and a.dtype == np.float64 \
            and a.flags["C_CONTIGUOUS"]
        if a.size != n:
            raise MGError(MG_ERR_ARG, "buffer of %d values, need %d" % (a.size, n))
        return _host_ptr(a), MG_HOST

    def timestep(self, centers, radii, charges, cycles=1, abs_tol=0.0,
                 normalization=MG_CHARGE_PER_CELLS, subsample=1, forces=True,
                 force_subsample=None, raise_notconv=True):
        """One time step of Alg.1's potential part (mg_timestep): RHS from
        the spheres, `cycles` warm-started V-cycles (or, cycles=0, cycles
        until ||r|| <= abs_tol), then the Coulomb forces.  Returns
        (forces (n, 3) or None, cycles run, final residual norm)."""
        c = np.ascontiguousarray(centers, np.float64).reshape(-1)
        r = np.ascontiguousarray(radii, np.float64)
        q = np.ascontiguousarray(charges, np.float64)
        out = np.empty(3 * len(r), np.float64) if forces else None
        cyc = ctypes.c_int(0)
        res = ctypes.c_double(0.0)
        fs = subsample if force_subsample is None else force_subsample
        rc = lib().mg_timestep(self._ctx, len(r), _host_ptr(c), _host_ptr(r),
                               _host_ptr(q), normalization, subsample,
                               int(cycles), float(abs_tol),
                               _host_ptr(out) if forces else None, int(fs),
                               ctypes.byref(cyc), ctypes.byref(res))
        if rc != MG_OK and (rc != MG_ERR_NOTCONV or raise_notconv):
            _check(rc, self._ctx)
        return (out.reshape(-1, 3) if forces else None), cyc.value, res.value

    def get_solution(self, out=None):
        if out is None:
            out = np.empty(self.local_shape(0), np.float64)
        ptr, where = self._io_args(out)
        _check(lib().mg_get_solution(self._ctx, ptr, where), self._ctx)
        return out

    def set_solution(self, a):
        ptr, where = self._io_args(a)
        _check(lib().mg_set_solution(self._ctx, ptr, where), self._ctx)

    def zero_solution(self):
        _check(lib().mg_zero_solution(self._ctx), self._ctx)

    def get_field(self, level, field, out=None):
        if out is None:
            out = np.empty(self.local_shape(level), np.float64)
        ptr, where = self._io_args(out, level)
        _check(lib().mg_get_field(self._ctx, level, field, ptr, where), self._ctx)
        return out

    def set_field(self, level, field, a):
        ptr, where = self._io_args(a, level)
        _check(lib().mg_set_field(self._ctx, level, field, ptr, where), self._ctx)

    def set_mask(self, solid):
        """Solid cells (nonzero) of the WHOLE domain, natural layout."""
        if solid is None:
            _check(lib().mg_set_mask(self._ctx, None, MG_HOST), self._ctx)
            return
        a = np.ascontiguousarray(solid, dtype=np.uint8)
        self._mask_keep = a
        _check(lib().mg_set_mask(self._ctx, a.ctypes.data, MG_HOST), self._ctx)

    def set_bc_patch(self, face, a0, a1, b0, b1, bc_type, value):
        """Per-face-cell BC on a rectangle of face `face` (include/mg.h)."""
        _check(lib().mg_set_bc_patch(self._ctx, int(face), int(a0), int(a1),
                                     int(b0), int(b1), int(bc_type),
                                     float(value)), self._ctx)

    def set_permittivity(self, eps):
        """Cell permittivity (whole domain, natural layout); None = 1."""
        if eps is None:
            _check(lib().mg_set_permittivity(self._ctx, None, MG_HOST), self._ctx)
            return
        e = np.ascontiguousarray(eps, np.float64)
        _check(lib().mg_set_permittivity(self._ctx, _host_ptr(e), MG_HOST),
               self._ctx)

    def set_face_values(self, face, values):
        """Per-cell boundary values of face `face` (in-face (a, b) order)."""
        v = np.ascontiguousarray(values, np.float64)
        _check(lib().mg_set_face_values(self._ctx, int(face), v.ctypes.data),
               self._ctx)

    def get_stencil(self, level=0):
        out = np.empty(self.local_shape(level) + (7,), np.float64)
        _check(lib().mg_get_stencil(self._ctx, level, out.ctypes.data, MG_HOST),
               self._ctx)
        return out

    # -- solve ----------------------------------------------------------------
    def vcycle(self) -> float:
        r = ctypes.c_double()
        _check(lib().mg_vcycle(self._ctx, ctypes.byref(r)), self._ctx)
        return r.value

    def residual_norm(self) -> float:
        r = ctypes.c_double()
        _check(lib().mg_residual_norm(self._ctx, ctypes.byref(r)), self._ctx)
        return r.value

    def solve(self, tol: float, max_cycles: int = 100, raise_notconv=False):
        max_cycles = int(max_cycles)
        if max_cycles < 1:
            raise MGError(MG_ERR_ARG, "max_cycles must be >= 1")
        hist = np.zeros(max_cycles + 1, np.float64)
        cyc = ctypes.c_int()
        rc = lib().mg_solve_n(self._ctx, float(tol), max_cycles, ctypes.byref(cyc),
                              _host_ptr(hist))
        if rc != MG_OK and (rc != MG_ERR_NOTCONV or raise_notconv):
            _check(rc, self._ctx)
        return rc, cyc.value, hist[:cyc.value + 1].copy()

    # -- single steps -----------------------------------------------------------
    def smooth_half(self, level, color, from_zero=False):
        _check(lib().mg_smooth_half(self._ctx, level, color, int(from_zero)),
               self._ctx)

    def residual_restrict(self, level):
        _check(lib().mg_residual_restrict(self._ctx, level), self._ctx)

    def prolong_correct(self, level):
        _check(lib().mg_prolong_correct(self._ctx, level), self._ctx)

    def coarse_solve(self) -> int:
        it = ctypes.c_int()
        _check(lib().mg_coarse_solve(self._ctx, ctypes.byref(it)), self._ctx)
        return it.value

    # -- measurement --------------------------------------------------------------
    def set_profiling(self, on: bool):
        _check(lib().mg_set_profiling(self._ctx, int(bool(on))), self._ctx)

    def last_cycle_times(self) -> dict:
        out = (ctypes.c_double * 12)()
        _check(lib().mg_last_cycle_times_ex(self._ctx, out, 12), self._ctx)
        keys = ["smooth0_ms", "smooth0_launches", "restrict0_ms", "prolong0_ms",
                "norm_ms", "coarse_ms", "cycle_ms", "launches",
                "smooth0_launches_ex", "smooth0_halfsweeps", "whole_levels_ms",
                "cg_ms"]
        return dict(zip(keys, list(out)))

    @property
    def cycle_launches(self) -> int:
        return lib().mg_cycle_launches(self._ctx)

    @property
    def cycle_paths(self) -> int:
        """MG_PATH_* bits of the kernel paths the last recorded cycle took."""
        return lib().mg_cycle_paths(self._ctx)

    @property
    def stream_ptr(self) -> int:
        return lib().mg_stream(self._ctx)
