// Host orchestration and C-ABI (include/mg.h) of libmg_cuda.so.
//
// One context = this process's part of the multigrid hierarchy:
//   levels l <  nd : "distributed" -- x-slabs of nx_l/P planes, one per rank
//                    (NCCL backend: this rank's slab; LOOPBACK: all P slabs)
//   levels l >= nd : held whole (single grid); with P > 1 every rank holds a
//                    copy and computes it redundantly (agglomeration by
//                    in-place all-gather of the restricted RHS, P:746 /
//                    north_star "agglomerated onto one GPU" -- DESIGN.md).
//                    LOOPBACK shares one copy among its slabs; EMULATE keeps
//                    one copy per emulated rank, gathered by device copies
//                    with NCCL's indexing (the NCCL data layout, one GPU).
// With P == 1, nd = 0: every level is a single grid.
//
// The V-cycle is recorded once into a CUDA graph and replayed.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <nvtx3/nvToolsExt.h>
#include <time.h>

#include <chrono>
#include <string>
#include <vector>

#include "../../include/mg.h"
#include "mg_internal.h"

using mg::Grid;

namespace {

// NVTX range around a public call (SURVEY 5 tracing; header-only NVTX v3:
// a no-op unless a profiler injects itself)
struct Nvtx {
  explicit Nvtx(const char *name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

thread_local std::string g_err;
thread_local int g_err_code = 0;

int fail(int code, const char *fmt, ...) {
  g_err_code = code;
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = std::string(mg_strerror(code)) + ": " + buf;
  return code;
}

// ---- NCCL, loaded on demand (no link-time dependency) -----------------------
struct Nccl {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t);
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t);
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t,
                            ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char *(*GetErrorString)(ncclResult_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *);
  ncclResult_t (*CommAbort)(ncclComm_t);
};
Nccl g_nccl;

bool load_nccl() {
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
#define SYM(name, field)                                             \
  *(void **)(&g_nccl.field) = dlsym(h, name);                        \
  if (!g_nccl.field) return false;
  SYM("ncclGetUniqueId", GetUniqueId);
  SYM("ncclCommInitRank", CommInitRank);
  SYM("ncclCommDestroy", CommDestroy);
  SYM("ncclSend", Send);
  SYM("ncclRecv", Recv);
  SYM("ncclAllGather", AllGather);
  SYM("ncclGroupStart", GroupStart);
  SYM("ncclGroupEnd", GroupEnd);
  SYM("ncclGetErrorString", GetErrorString);
  SYM("ncclCommGetAsyncError", CommGetAsyncError);
  SYM("ncclCommAbort", CommAbort);
#undef SYM
  g_nccl.ok = true;
  return true;
}

// ---- plan ---------------------------------------------------------------------
struct Plan {
  int L = 0, nd = 0, P = 1;
  int dims[32][3];
  int nxl[32];
};

int make_plan(int nx, int ny, int nz, const mg_opts *o, Plan *pl) {
  if (nx <= 0 || ny <= 0 || nz <= 0)
    return fail(MG_ERR_ARG, "dimensions must be positive (%d,%d,%d)", nx, ny, nz);
  if (nx % 2 || ny % 2 || nz % 2)
    return fail(MG_ERR_COARSEN,
                "dimensions must be even: the coarsest level is a multiple of "
                "two (P:506-507); got (%d,%d,%d)", nx, ny, nz);
  const int P = o->nranks < 1 ? 1 : o->nranks;
  const int maxl = (o->max_levels <= 0 || o->max_levels > 32) ? 32 : o->max_levels;
  int d[3] = {nx, ny, nz};
  pl->L = 0;
  pl->P = P;
  while (true) {
    for (int a = 0; a < 3; a++) pl->dims[pl->L][a] = d[a];
    pl->L++;
    if (pl->L >= maxl) break;
    bool ok = true;
    for (int a = 0; a < 3; a++)
      if (d[a] % 2 || (d[a] / 2) % 2) ok = false;
    int mn = d[0] < d[1] ? d[0] : d[1];
    if (d[2] < mn) mn = d[2];
    if (mn <= o->min_coarse) ok = false;
    if (!ok) break;
    for (int a = 0; a < 3; a++) d[a] /= 2;
  }
  for (int l = 0; l < 32; l++) pl->nxl[l] = 0;
  if (P == 1) {
    pl->nd = 0;
    return MG_OK;
  }
  if (nx % P)
    return fail(MG_ERR_ARG, "nx=%d not divisible by nranks=%d", nx, P);
  if (pl->L < 2)
    return fail(MG_ERR_COARSEN, "multi-slab solve needs at least two levels");
  if ((nx / P) % 2)
    return fail(MG_ERR_COARSEN, "planes per rank (%d) must be even", nx / P);
  int nd = 1;
  for (int l = 1; l < pl->L - 1; l++) {
    if (pl->dims[l][0] % P) break;
    const int nxl = pl->dims[l][0] / P;
    if (nxl % 2) break;
    const long long cells = (long long)nxl * pl->dims[l][1] * pl->dims[l][2];
    if (cells < o->agglomerate_below) break;
    nd = l + 1;
  }
  pl->nd = nd;
  for (int l = 0; l < nd; l++) pl->nxl[l] = pl->dims[l][0] / P;
  return MG_OK;
}

int round4(int v) { return (v + 3) & ~3; }

Grid make_grid(const Plan &pl, int l, int slab, double h, const int *dface) {
  Grid g;
  memset(&g, 0, sizeof g);
  g.nx = pl.dims[l][0];
  g.ny = pl.dims[l][1];
  g.nz = pl.dims[l][2];
  if (l < pl.nd) {
    g.nxl = pl.nxl[l];
    g.x0 = slab * pl.nxl[l];
  } else {
    g.nxl = g.nx;
    g.x0 = 0;
  }
  g.nzh = g.nz / 2;
  g.pz = round4(g.nzh);
  g.plane = (long long)(g.ny + 2) * g.pz;
  g.c = ldexp(1.0 / (h * h), -l);
  g.w = ldexp(h * h, l);
  for (int q = 0; q < 6; q++) g.dface[q] = dface[q];
  return g;
}

}  // namespace

// ---- context --------------------------------------------------------------------
// TMA descriptors of a grid's two Phi arrays (for the marching half-sweep)
struct TmPair {
  alignas(64) unsigned char r[128];   // whole-row boxes (half-sweeps)
  alignas(64) unsigned char b[128];
  alignas(64) unsigned char rr[128];  // z-tiled boxes (residual kernels)
  alignas(64) unsigned char rb[128];
  bool ok = false, ok_resid = false;
};

struct mg_ctx {
  Plan pl;
  std::vector<std::vector<TmPair>> tm;
  // kernel paths (mg_opts.disable clears them; include/mg.h MG_OFF_*)
  int use_march = 1;  // TMA plane-marching kernels where the grid allows
  // multi-slab overlap: boundary planes first, the ghost exchange on s_comm
  // while the interior planes are swept
  int overlap = 1;
  int paths = 0;      // MG_PATH_* taken by the last recorded V-cycle
  int nsm = 148;      // SMs of the device (cudaDevAttrMultiProcessorCount)
  cudaStream_t s_comm = nullptr;
  // sphere RHS: the clear of f runs on s_aux while the sphere kernels that do
  // not touch f (bins, neighbour lists, counts) run on the context's stream
  cudaStream_t s_aux = nullptr;
  cudaEvent_t ev_aux0 = nullptr, ev_aux1 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_sync = nullptr;  // NCCL contexts: polled by sync()
  std::vector<std::vector<Grid>> vlo, vhi, vin;   // per level, slab: views
  std::vector<std::vector<TmPair>> tmin;          // TMA maps of the interior views
  bool masked = false;            // variable coefficients (mask and/or patches)
  std::vector<void *> mask_bufs;  // codes / coefficients (library-owned)
  std::vector<uint8_t> solid_h;   // global solid mask (empty: none)
  std::vector<double> eps_h;      // global cell permittivity (empty: 1)
  bool patched = false;           // per-face-cell BC arrays in use
  bool types_uniform = true;      // every face cell has its face's BC type
  std::vector<uint8_t> fty_h[6];  // face-cell BC types
  std::vector<double> fva_h[6];   // face-cell BC values
  mg::FaceBC fbc{};               // device copies (patched only)
  unsigned char *dsolid = nullptr;  // device copy of the global solid mask
  double h;
  mg_bc bc[6];
  mg_opts o;
  int P = 1, rank = 0, backend = MG_HALO_NONE;
  int nslab = 1, slab0 = 0;  // slabs held on distributed levels
  int ncopy = 1;             // copies of each agglomerated level (EMULATE: P)
  std::vector<size_t> pbase; // norm partials of level-0 slab s at partials + pbase[s]
  std::vector<std::vector<Grid>> g;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  char *ws = nullptr;
  size_t ws_bytes = 0;
  bool own_ws = false;
  double *partials = nullptr;  // norm partial sums (carve: upper bound)
  double *normv = nullptr;     // [0] local sum, [1] global sum, [2..2+P) gathered
  double *cg_scr = nullptr;
  int *cg_iters = nullptr;
  double *h_norm = nullptr;    // pinned, mapped
  double *h_norm_dev = nullptr;  // its device view (written by k_publish)
  int *h_iters = nullptr;      // pinned
  double *stage = nullptr;     // lazily allocated natural-layout staging
  size_t stage_bytes = 0;
  // mg_solve_async pipeline: three staging slots (upload of problem k+1,
  // download of problem k-1 and the current problem's unpack never share
  // one), copy streams, slot events
  double *astg[3] = {nullptr, nullptr, nullptr};
  size_t astg_bytes = 0;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_in[3] = {}, ev_out[3] = {}, ev_d2h[3] = {};
  // ev_free[q]: recorded on the context's stream after its last read of slot
  // q (the RHS conversion); the next upload into the slot waits for it
  cudaEvent_t ev_free[3] = {};
  bool d2h_used[3] = {false, false, false}, free_used[3] = {false, false, false};
  unsigned long long async_k = 0;
  double *sph = nullptr;       // lazily allocated sphere list
  size_t sph_cap = 0;
  int *bins = nullptr;         // sphere bins (counts + items), grown on demand
  size_t bins_cap = 0;         // ints
  double *fbuf = nullptr;      // force step: sphere list + partial sums
  double *hpin = nullptr;      // pinned host staging for sphere lists and
  size_t hpin_cap = 0;         // force partials (doubles), grown, kept
  size_t fbuf_cap = 0;         // (doubles), grown on demand, kept
  unsigned long long *counts = nullptr;
  cudaGraphExec_t graph = nullptr;
  bool in_cycle = false;  // enqueue_vcycle is recording (vs a single step)
  // look-ahead red sweep: a second level-0 red buffer per slab;
  // g[0] / tm[0] (and the level-0 overlap views) view the committed iterate,
  // g0alt / tm0alt (vlo0alt, ...) the other buffers, which hold the next
  // cycle's first red half-sweep when la_valid.  One graph per orientation
  // (red0: which buffers g[0] views).
  std::vector<double *> red0_alt;
  std::vector<Grid> g0alt, vlo0alt, vhi0alt, vin0alt;
  std::vector<TmPair> tm0alt, tmin0alt;
  int red0 = 0;
  bool la_valid = false;
  cudaGraphExec_t graph_la[2] = {nullptr, nullptr};
  double prev_norm = -1.0;
  ncclComm_t comm = nullptr;
  int dev = 0;
  // measurement: kernel launches per recorded V-cycle, optional event marks
  int launches = 0;
  int cycle_launches = 0;
  bool prof = false, prof_last = false;
  std::vector<cudaEvent_t> ev;
  int nev = 0;
  std::vector<int> mark_cat;  // category of the interval ending at mark i
};

namespace {

// partial sums of the grid-stride norm kernels: 8 per SM, for up to 256 SMs
// (the workspace size must not depend on a device query)
constexpr int kMaxNormBlocks = 8 * 256;

// bump allocation over the workspace; with base == nullptr only sizes
struct Carver {
  char *base;
  size_t off = 0;
  void *take(size_t bytes) {
    off = (off + 255) & ~(size_t)255;
    void *p = base ? base + off : nullptr;
    off += bytes;
    return p;
  }
};

// contexts that get the look-ahead red sweep's second buffers: a
// pre-smoothing red sweep to look ahead to, the true cycle-end norm
bool lookahead_capable(const mg_ctx *c) {
  return c->pl.L >= 2 && c->o.nu1 >= 1 && c->o.nu2 >= 1 && !c->o.fused_norm &&
         !(c->o.disable & MG_OFF_LOOKAHEAD);
}

size_t carve(mg_ctx *c, char *base) {
  Carver cv{base};
  const int L = c->pl.L;
  c->g.assign(L, {});
  // centre contribution of a face: Dirichlet +1, Neumann -1, periodic 0
  int dface[6];
  for (int q = 0; q < 6; q++)
    dface[q] = c->bc[q].type == MG_DIRICHLET ? 1 : (c->bc[q].type == MG_NEUMANN ? -1 : 0);
  for (int l = 0; l < L; l++) {
    const int ns = l < c->pl.nd ? c->nslab : c->ncopy;
    for (int s = 0; s < ns; s++) {
      Grid gr = make_grid(c->pl, l, l < c->pl.nd ? c->slab0 + s : 0, c->h, dface);
      gr.nsm = c->nsm;
      for (int a = 0; a < 3; a++) gr.per[a] = c->bc[2 * a].type == MG_PERIODIC;
      gr.gx = gr.per[0] && gr.nxl == gr.nx;  // whole grid: own x ghosts
      const size_t bytes = (size_t)mg::grid_elems(gr) * sizeof(double);
      gr.phiR = (double *)cv.take(bytes);
      gr.phiB = (double *)cv.take(bytes);
      gr.fR = (double *)cv.take(bytes);
      gr.fB = (double *)cv.take(bytes);
      c->g[l].push_back(gr);
    }
  }
  // look-ahead red sweep: a second red array per level-0 slab
  c->red0_alt.clear();
  if (lookahead_capable(c))
    for (const Grid &g : c->g[0])
      c->red0_alt.push_back((double *)cv.take((size_t)mg::grid_elems(g) * sizeof(double)));
  // one region of norm partials per level-0 slab: residual-kernel partials
  // plus (split norm) the smoother's, or the grid-stride kernels' (fewer)
  size_t npart = 0;
  c->pbase.clear();
  for (const Grid &g : c->g[0]) {
    c->pbase.push_back(npart);
    const size_t nb = (size_t)mg::march_blocks_max(g);
    npart += 2 * (nb > (size_t)kMaxNormBlocks ? nb : (size_t)kMaxNormBlocks);
  }
  c->partials = (double *)cv.take(sizeof(double) * npart);
  c->normv = (double *)cv.take(sizeof(double) * (2 + c->P));
  c->cg_scr = (double *)cv.take(sizeof(double) *
                                mg::coarse_cg_scratch_doubles(c->g[L - 1][0]));
  c->cg_iters = (int *)cv.take(sizeof(int) * 4);
  c->counts = (unsigned long long *)cv.take(sizeof(unsigned long long) * 4);
  return cv.off + 256;
}

bool ck(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return true;
  fail(MG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return false;
}

#define CK(expr)                               \
  do {                                         \
    if (!ck((expr), #expr)) return MG_ERR_CUDA; \
  } while (0)

int nccl_ck(ncclResult_t r, const char *what) {
  if (r == ncclSuccess) return MG_OK;
  return fail(MG_ERR_NCCL, "%s: %s", what, g_nccl.GetErrorString(r));
}

bool distributed(const mg_ctx *c, int l) { return l < c->pl.nd && c->P > 1; }

// profiling categories (mg_last_cycle_times)
// CAT_COARSE: distributed levels >= 1; CAT_AGG: levels >= 1 held whole
// (agglomerated, or every level >= 1 of a single slab) without the CG;
// CAT_CG: the coarsest-grid solve
enum { CAT_NONE = -1, CAT_SMOOTH0 = 0, CAT_RESTRICT0 = 2, CAT_PROLONG0 = 3,
       CAT_NORM = 4, CAT_COARSE = 5, CAT_AGG = 6, CAT_CG = 7, kNumCat = 8 };
constexpr int kMaxMarks = 512;

// record an event closing an interval of category `cat` (CAT_NONE opens one)
void mark(mg_ctx *c, int cat) {
  if (!c->prof || c->nev >= kMaxMarks) return;
  // external record: a real event node when the stream is being captured
  // (outside a capture -- eager cycles, single steps -- a plain record)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->stream, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(c->ev[c->nev], c->stream, cudaEventRecordExternal);
  else
    cudaEventRecord(c->ev[c->nev], c->stream);
  c->mark_cat[c->nev] = cat;
  c->nev++;
}

// the grid slab / copy s of level l restricts to and prolongs from: its
// own slab on distributed levels, else the agglomerated level (EMULATE: the
// copy of rank s)
const Grid &coarse_of(const mg_ctx *c, int l, int s) {
  return (l + 1 < c->pl.nd) ? c->g[l + 1][s] : c->g[l + 1][c->ncopy > 1 ? s : 0];
}

// grids of level l whose cells the caller's arrays hold: the slabs of a
// distributed level, one copy of an agglomerated level
size_t io_grids(const mg_ctx *c, int l) {
  return l < c->pl.nd ? c->g[l].size() : 1;
}

bool periodic_x(const mg_ctx *c) { return c->bc[0].type == MG_PERIODIC; }
bool any_periodic(const mg_ctx *c) {
  for (int q = 0; q < 6; q++)
    if (c->bc[q].type == MG_PERIODIC) return true;
  return false;
}

// reading c11: the cycle reports the norm of the level-0 residual computed
// for the restriction (after pre-smoothing); one level has no restriction
bool fused_norm_on(const mg_ctx *c) { return c->o.fused_norm && c->pl.L > 1; }
int norm_partials(mg_ctx *c, size_t s, double *partials);
int finish_norm(mg_ctx *c, const int *cnt);
constexpr int kMaxSlabs = 64;  // level-0 slabs held by one context

// ghost-plane exchange of one colour array (0 phiR, 1 phiB) on level l.  On a
// periodic x axis the first and last slabs are neighbours too (P:692-693:
// "processes are configured in a periodic arrangement").  Every rank posts
// its sends / receives in the same order -- (last plane -> right, left ghost
// <- left), then (first plane -> left, right ghost <- right) -- so that
// repeated peers (P = 2 with wrap) match message by message.
int halo(mg_ctx *c, int l, int which, cudaStream_t st = nullptr) {
  if (!distributed(c, l)) return MG_OK;
  if (!st) st = c->stream;
  auto arr = [&](const Grid &g) { return which ? g.phiB : g.phiR; };
  const bool wrap = periodic_x(c);
  if (c->backend == MG_HALO_LOOPBACK) {
    const int ns = c->nslab;
    for (int s = 0; s < ns; s++) {
      if (s + 1 == ns && !wrap) break;
      const Grid &a = c->g[l][s], &b = c->g[l][(s + 1) % ns];
      const size_t bytes = sizeof(double) * a.plane;
      CK(cudaMemcpyAsync(arr(b), arr(a) + (long long)a.nxl * a.plane, bytes,
                         cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(arr(a) + (long long)(a.nxl + 1) * a.plane,
                         arr(b) + b.plane, bytes, cudaMemcpyDeviceToDevice,
                         st));
    }
    return MG_OK;
  }
  auto plane_of = [](const Grid &g, int code) {
    return code == MG_PLANE_FIRST ? 1
           : code == MG_PLANE_LAST ? g.nxl
           : code == MG_GHOST_LO   ? 0
                                   : g.nxl + 1;
  };
  if (c->backend == MG_HALO_EMULATE) {
    // every emulated rank's schedule executed as NCCL would match it: the
    // k-th receive of rank r from peer q takes the k-th send of q to r
    int ops[kMaxSlabs][4][3], nops[kMaxSlabs];
    for (int r = 0; r < c->P; r++) nops[r] = mg_halo_schedule(c->P, r, wrap ? 1 : 0, ops[r]);
    for (int r = 0; r < c->P; r++) {
      for (int k = 0; k < nops[r]; k++) {
        if (ops[r][k][0] != MG_OP_RECV) continue;
        const int q = ops[r][k][1];
        int nth = 0;
        for (int m = 0; m < k; m++) nth += ops[r][m][0] == MG_OP_RECV && ops[r][m][1] == q;
        int src = -1;
        for (int m = 0, seen = 0; m < nops[q]; m++)
          if (ops[q][m][0] == MG_OP_SEND && ops[q][m][1] == r && seen++ == nth) src = m;
        if (src < 0) return fail(MG_ERR_NCCL, "halo schedule: unmatched receive");
        const Grid &gr = c->g[l][r], &gq = c->g[l][q];
        CK(cudaMemcpyAsync(arr(gr) + (long long)plane_of(gr, ops[r][k][2]) * gr.plane,
                           arr(gq) + (long long)plane_of(gq, ops[q][src][2]) * gq.plane,
                           sizeof(double) * gr.plane, cudaMemcpyDeviceToDevice, st));
      }
    }
    return MG_OK;
  }
  const Grid &g = c->g[l][0];
  double *A = arr(g);
  const size_t n = (size_t)g.plane;
  int ops[4][3];
  const int nops = mg_halo_schedule(c->P, c->rank, wrap ? 1 : 0, ops);
  int rc;
  if ((rc = nccl_ck(g_nccl.GroupStart(), "ncclGroupStart"))) return rc;
  for (int k = 0; k < nops; k++) {
    double *buf = A + (long long)plane_of(g, ops[k][2]) * g.plane;
    if (ops[k][0] == MG_OP_SEND)
      g_nccl.Send(buf, n, ncclDouble, ops[k][1], c->comm, st);
    else
      g_nccl.Recv(buf, n, ncclDouble, ops[k][1], c->comm, st);
  }
  return nccl_ck(g_nccl.GroupEnd(), "ncclGroupEnd(halo)");
}

// Agglomeration of level l (held whole): rank r computed the planes
// [1 + r nx/P, 1 + (r+1) nx/P) of `narr` arrays (elements of `esize` bytes,
// base(g, a) the array a of grid g); every rank receives the others'
// portions.  NCCL: in-place all-gathers in one group; EMULATE: the same
// byte ranges copied between the ranks' copies; LOOPBACK: nothing (one
// shared copy).
template <typename Base>
int gather_portions(mg_ctx *c, int l, int narr, size_t esize, Base base) {
  if (c->P == 1 || c->backend == MG_HALO_LOOPBACK) return MG_OK;
  const Grid &G = c->g[l][0];
  const size_t cnt = (size_t)(G.nx / c->P) * G.plane * esize;  // bytes per rank
  const size_t first = (size_t)G.plane * esize;                  // ghost plane 0
  if (c->backend == MG_HALO_EMULATE) {
    for (int r = 0; r < c->P; r++)
      for (int t = 0; t < c->P; t++) {
        if (t == r) continue;
        for (int a = 0; a < narr; a++) {
          char *src = (char *)base(c->g[l][r], a) + first + r * cnt;
          char *dst = (char *)base(c->g[l][t], a) + first + r * cnt;
          CK(cudaMemcpyAsync(dst, src, cnt, cudaMemcpyDeviceToDevice, c->stream));
        }
      }
    return MG_OK;
  }
  int rc;
  if ((rc = nccl_ck(g_nccl.GroupStart(), "ncclGroupStart"))) return rc;
  for (int a = 0; a < narr; a++) {
    char *b = (char *)base(G, a) + first;
    g_nccl.AllGather(b + c->rank * cnt, b, cnt, ncclChar, c->comm, c->stream);
  }
  return nccl_ck(g_nccl.GroupEnd(), "ncclGroupEnd(agglomerate)");
}

// periodic ghost rows / planes of the grids of level l held here, for the
// writers of Phi that do not store ghost copies (prolongation, CG, copy-in)
void periodic_fill(mg_ctx *c, int l) {
  for (const Grid &g : c->g[l]) {
    if (!(g.gx || g.per[1])) continue;
    mg::launch_periodic_fill(g, c->stream);
    c->launches++;
  }
}

// plane-range view of a slab grid: planes [pb, pb + n) as a slab of n planes
Grid plane_view(const Grid &g, int pb, int n) {
  Grid v = g;
  const long long off = (long long)pb * g.plane;
  v.phiR += off;
  v.phiB += off;
  v.fR += off;
  v.fB += off;
  v.nxl = n;
  v.x0 = g.x0 + pb;
  return v;
}

// overlap the ghost exchange of level l with the interior planes?
bool overlap_level(const mg_ctx *c, int l) {
  return c->overlap && distributed(c, l) && !c->masked && !c->vin.empty() &&
         !c->vin[l].empty();
}

// half-sweep of a distributed level with the exchange overlapped: the two
// boundary planes of every slab first (the planes the neighbours need), then
// the exchange on s_comm while the interior planes are swept; the next step
// waits for the exchange (its boundary planes read the received ghosts).
int smooth_half_overlap(mg_ctx *c, int l, int color, int from_zero) {
  for (size_t s = 0; s < c->g[l].size(); s++) {
    mg::launch_smooth(c->vlo[l][s], color, from_zero, c->stream);
    mg::launch_smooth(c->vhi[l][s], color, from_zero, c->stream);
    c->launches += 2;
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->ev_fork, c->stream));
  CK(cudaStreamWaitEvent(c->s_comm, c->ev_fork, 0));
  int rc = halo(c, l, color, c->s_comm);
  if (rc) return rc;
  CK(cudaEventRecord(c->ev_join, c->s_comm));
  for (size_t s = 0; s < c->g[l].size(); s++) {
    const Grid &v = c->vin[l][s];
    const TmPair &t = c->tmin[l][s];
    if (!from_zero && t.ok && c->use_march)
      mg::launch_smooth_march(v, color ? t.r : t.b, color, c->stream);
    else
      mg::launch_smooth(v, color, from_zero, c->stream);
    c->launches++;
  }
  CK(cudaGetLastError());
  CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  return MG_OK;
}

int smooth_half(mg_ctx *c, int l, int color, int from_zero) {
  if (overlap_level(c, l)) {
    c->paths |= MG_PATH_OVERLAP;
    if (l == 0) mark(c, CAT_NONE);
    int rc = smooth_half_overlap(c, l, color, from_zero);
    if (l == 0) mark(c, CAT_SMOOTH0);
    return rc;
  }
  if (l == 0) mark(c, CAT_NONE);
  for (size_t s = 0; s < c->g[l].size(); s++) {
    const Grid &g = c->g[l][s];
    const TmPair &t = c->tm[l][s];
    if (c->masked && !(g.codeR && !from_zero && t.ok && c->use_march))
      mg::launch_smooth_var(g, color, from_zero, c->stream);
    else if (!from_zero && t.ok && c->use_march)
      mg::launch_smooth_march(g, color ? t.r : t.b, color, c->stream);
    else
      mg::launch_smooth(g, color, from_zero, c->stream);
    c->launches++;
  }
  if (l == 0) mark(c, CAT_SMOOTH0);
  CK(cudaGetLastError());
  return halo(c, l, color);
}

// f_{l+1} = R (f_l - A Phi_l); at the agglomeration level every rank then
// all-gathers the restricted RHS (in place) so that each holds the whole level
// red0: the restriction also performs level l+1's first red half-sweep from
// Phi = 0 (box domains; mg_opts.disable MG_OFF_RED0 turns it off)
int restrict_level(mg_ctx *c, int l, bool red0 = false) {
  if (l == 0) mark(c, CAT_NONE);
  const bool with_norm = l == 0 && fused_norm_on(c);
  int cnt[kMaxSlabs] = {0};  // norm partials per slab (fused norm, reading c11)
  for (int s = 0; s < (int)c->g[l].size(); s++) {
    const TmPair &t = c->tm[l][s];
    const bool march = t.ok_resid && c->use_march;
    double *part = with_norm ? c->partials + c->pbase[s] : nullptr;
    if (with_norm && !(march && (!c->masked || c->g[l][s].codeR))) {
      // no fused kernel for this grid: the same residual's norm, one pass
      cnt[s] = norm_partials(c, s, part);
      c->launches++;
    }
    if (c->masked && !(c->g[l][s].codeR && march)) {
      mg::launch_resid_restrict_var(c->g[l][s], coarse_of(c, l, s), c->stream);
    } else if (march) {
      if (with_norm)
        cnt[s] = mg::launch_resid_restrict_norm_march(c->g[l][s], coarse_of(c, l, s), t.rr,
                                                      t.rb, part, c->stream, red0);
      else
        mg::launch_resid_restrict_march(c->g[l][s], coarse_of(c, l, s), t.rr, t.rb,
                                        c->stream, red0);
    } else {
      mg::launch_resid_restrict(c->g[l][s], coarse_of(c, l, s), red0, c->stream);
    }
    c->launches++;
  }
  if (l == 0) mark(c, CAT_RESTRICT0);
  CK(cudaGetLastError());
  if (with_norm) {
    int rc = finish_norm(c, cnt);
    if (rc) return rc;
  }
  if (l + 1 == c->pl.nd && c->P > 1)
    return gather_portions(c, l + 1, 2, sizeof(double), [](const Grid &g, int a) {
      return (void *)(a ? g.fB : g.fR);
    });
  if (red0) {  // the red half-sweep's ghost exchange
    c->paths |= MG_PATH_RED0;
    return halo(c, l + 1, 0);
  }
  return MG_OK;
}

// may the restriction of level l perform level l+1's first red half-sweep
// (from Phi = 0)?  Levels above `top` (the tail's first level), box grids
// without mask, not into the first agglomerated level (its red Phi would
// need the gather too), pre-smoothing on
bool red0_fused(const mg_ctx *c, int l, int top) {
  return !(c->o.disable & MG_OFF_RED0) && c->o.nu1 >= 1 && !c->masked && !any_periodic(c) &&
         l + 1 < top && !(c->P > 1 && l + 1 == c->pl.nd);
}

int prolong_level(mg_ctx *c, int l) {
  if (l == 0) mark(c, CAT_NONE);
  for (int s = 0; s < (int)c->g[l].size(); s++) {
    if (c->masked)
      mg::launch_prolong_var(c->g[l][s], coarse_of(c, l, s), c->o.alpha, c->stream);
    else
      mg::launch_prolong(c->g[l][s], coarse_of(c, l, s), 0, c->o.alpha, c->stream);
    c->launches++;
  }
  periodic_fill(c, l);
  if (l == 0) mark(c, CAT_PROLONG0);
  CK(cudaGetLastError());
  // both colours' ghosts: the next red half-sweep reads the black ones, and
  // without post-smoothing (nu2 = 0, or a single step) the norm or the next
  // step reads the red ones too
  int rc = halo(c, l, 1);
  if (!rc && (c->o.nu2 == 0 || !c->in_cycle)) rc = halo(c, l, 0);
  return rc;
}

// can level l use the fused prolongation + first post-smoothing red sweep?
bool can_fuse_prolong(const mg_ctx *c, int l) {
  if (!c->use_march || c->o.nu2 < 1) return false;
  for (size_t s = 0; s < c->tm[l].size(); s++) {
    if (!c->tm[l][s].ok) return false;
    if (c->masked && !c->g[l][s].codeR) return false;  // float records: no
  }
  return true;
}

// Phi_l += alpha P Phi_{l+1} fused with the red half-sweep that follows it
int prolong_red_level(mg_ctx *c, int l) {
  if (l == 0) mark(c, CAT_NONE);
  for (int s = 0; s < (int)c->g[l].size(); s++) {
    mg::launch_prolong_smooth_march(c->g[l][s], coarse_of(c, l, s),
                                    c->tm[l][s].b, 0, c->o.alpha, c->stream);
    c->launches++;
  }
  if (l == 0) {
    mark(c, CAT_PROLONG0);
    c->paths |= MG_PATH_PROLONG_FUSED;
  }
  CK(cudaGetLastError());
  return halo(c, l, 0);  // black is recomputed by the next half-sweep
}

// the coarsest grids of agglomerated runs (>= 4,096 unknowns) run CG on an
// 8-CTA cluster unless mg_opts.disable has MG_OFF_CG_CLUSTER
bool cg_cluster_on(const mg_ctx *c) { return !(c->o.disable & MG_OFF_CG_CLUSTER); }

int coarse_solve(mg_ctx *c) {
  // every copy of the coarsest level (EMULATE: one per rank, redundantly)
  for (const Grid &g : c->g[c->pl.L - 1]) {
    if (c->masked) {
      mg::launch_coarse_cg_var(g, c->cg_scr, c->o.coarse_tol, c->o.coarse_maxit,
                               c->cg_iters, c->stream);
      c->paths |= MG_PATH_CG_VAR;
    } else if (cg_cluster_on(c) && mg::coarse_cg_cluster_supported(g)) {
      mg::launch_coarse_cg_cluster(g, c->o.coarse_tol, c->o.coarse_maxit, c->cg_iters,
                                   c->stream);
      c->paths |= MG_PATH_CG_CLUSTER;
    } else {
      mg::launch_coarse_cg(g, c->cg_scr, c->o.coarse_tol, c->o.coarse_maxit,
                           c->cg_iters, c->stream);
    }
    c->launches++;
  }
  periodic_fill(c, c->pl.L - 1);  // the prolongation reads coarse ghosts
  CK(cudaGetLastError());
  return MG_OK;
}

// enqueue ||f - A Phi||^2 of level 0 into c->normv[1] and a copy to h_norm
// partial sums of r^2 over level-0 grid s (fixed order); returns their count
int norm_partials(mg_ctx *c, size_t s, double *partials) {
  const Grid &g = c->g[0][s];
  const TmPair &t = c->tm[0][s];
  if (c->masked && !(g.codeR && t.ok_resid && c->use_march))
    return mg::launch_norm_partials_var(g, partials, c->stream);
  if (t.ok_resid && c->use_march) {
    mg::launch_norm_march(g, t.rr, t.rb, partials, c->stream);
    return mg::norm_march_blocks(g);
  }
  return mg::launch_norm_partials(g, partials, c->stream);
}

int enqueue_norm(mg_ctx *c) {
  int cnt[kMaxSlabs] = {0};
  mark(c, CAT_NONE);
  for (size_t s = 0; s < c->g[0].size(); s++) {
    cnt[s] = norm_partials(c, s, c->partials + c->pbase[s]);
    c->launches++;
  }
  return finish_norm(c, cnt);
}

// ||r||^2 from the partials (cnt[s] of them for level-0 slab s, at
// partials + pbase[s]), published to the mapped host word.  One slab: their
// ordered sum.  P slabs / ranks: per slab (rank) the ordered sum into
// normv[2 + rank], an in-place all-gather of the P values (NCCL), then their
// sum in rank order -- the same roundings in every backend.
int finish_norm(mg_ctx *c, const int *cnt) {
  if (c->P == 1) {
    mg::launch_sum_publish(c->partials + c->pbase[0], cnt[0], c->normv, c->normv + 1,
                           c->h_norm_dev, c->stream);
    c->launches++;
  } else {
    for (size_t s = 0; s < c->g[0].size(); s++) {
      mg::launch_sum_ordered(c->partials + c->pbase[s], cnt[s],
                             c->normv + 2 + c->slab0 + s, c->stream);
      c->launches++;
    }
    CK(cudaGetLastError());
    if (c->backend == MG_HALO_NCCL) {
      int rc = nccl_ck(g_nccl.AllGather(c->normv + 2 + c->rank, c->normv + 2, 1,
                                        ncclDouble, c->comm, c->stream),
                       "ncclAllGather(norm)");
      if (rc) return rc;
    }
    mg::launch_sum_ordered(c->normv + 2, c->P, c->normv + 1, c->stream);
    mg::launch_publish(c->normv + 1, c->normv + 1, c->h_norm_dev, c->stream);
    c->launches += 2;
  }
  mark(c, CAT_NORM);
  CK(cudaGetLastError());
  return MG_OK;
}

// split cycle-end norm: the last black half-sweep of level 0 sums the black
// residuals (k_smooth_march<..., NORM>), a red-only residual pass the rest:
// 12 + 12 instead of 12 + 16 B/cell for that pair.  Every level-0 slab needs
// both marching kernels; MG_OFF_SPLIT_NORM turns it off.
bool split_norm_ok(const mg_ctx *c) {
  if ((c->o.disable & MG_OFF_SPLIT_NORM) || fused_norm_on(c) || c->pl.L < 2 ||
      c->o.nu2 < 1 || !c->use_march)
    return false;
  for (size_t s = 0; s < c->g[0].size(); s++) {
    const TmPair &t = c->tm[0][s];
    if (!(t.ok && t.ok_resid && (!c->masked || c->g[0][s].codeR))) return false;
  }
  return true;
}

// the split norm's two passes, after the last red post-smoothing half-sweep
// of level 0: black sweep + black residual partials on every slab, the black
// ghost exchange (the red residuals read the new black ghosts), red residual
// partials, the ordered sum
int split_norm_tail(mg_ctx *c) {
  mark(c, CAT_NONE);
  int cnt[kMaxSlabs] = {0};
  for (size_t s = 0; s < c->g[0].size(); s++) {
    cnt[s] = mg::launch_smooth_norm_march(c->g[0][s], c->tm[0][s].r, 1,
                                          c->partials + c->pbase[s], c->stream);
    c->launches++;
  }
  mark(c, CAT_SMOOTH0);
  CK(cudaGetLastError());
  int rc;
  if ((rc = halo(c, 0, 1))) return rc;
  mark(c, CAT_NONE);
  for (size_t s = 0; s < c->g[0].size(); s++) {
    cnt[s] += mg::launch_norm_red_march(c->g[0][s], c->tm[0][s].rr, c->tm[0][s].rb,
                                        c->partials + c->pbase[s] + cnt[s], c->stream);
    c->launches++;
  }
  CK(cudaGetLastError());
  c->paths |= MG_PATH_SPLIT_NORM;
  return finish_norm(c, cnt);
}

// Look-ahead red sweep: the cycle-end norm needs the red
// residuals of the new iterate, f - c (d Phi_R - s), s the sum of its black
// neighbours -- the same s the NEXT cycle's first red half-sweep computes.
// So the last kernel of a cycle is that half-sweep, written to the second
// red buffer (the committed iterate stays intact: a solve that stops here
// returns exactly the oracle's iterate), with the red residuals of the
// current Phi_R read beside it: 4 B/cell more than the sweep instead of a
// 12 B/cell residual pass.  The next cycle starts from the other buffer and
// skips that sweep.  Anything that changes Phi, f or the operator on level
// 0 drops the look-ahead (la_drop); the next cycle then runs it first.
bool lookahead_ok(const mg_ctx *c) {
  // (masked levels: split_norm_ok requires the byte codes on every slab)
  if (c->red0_alt.empty() || !split_norm_ok(c)) return false;
  for (const TmPair &t : c->tm0alt)
    if (!(t.ok && t.ok_resid)) return false;
  // the overlapped half-sweeps need the other buffers' interior views too
  return !overlap_level(c, 0) || c->vin0alt.size() == c->g[0].size();
}

void la_drop(mg_ctx *c) { c->la_valid = false; }

// recorded V-cycle graphs (re-recorded on next use)
void drop_graphs(mg_ctx *c) {
  if (c->graph) cudaGraphExecDestroy(c->graph);
  c->graph = nullptr;
  for (int k = 0; k < 2; k++) {
    if (c->graph_la[k]) cudaGraphExecDestroy(c->graph_la[k]);
    c->graph_la[k] = nullptr;
  }
}

// committed view <-> look-ahead view
void la_swap(mg_ctx *c) {
  std::swap(c->g[0], c->g0alt);
  std::swap(c->tm[0], c->tm0alt);
  if (!c->vin0alt.empty()) {
    std::swap(c->vlo[0], c->vlo0alt);
    std::swap(c->vhi[0], c->vhi0alt);
    std::swap(c->vin[0], c->vin0alt);
    std::swap(c->tmin[0], c->tmin0alt);
  }
  c->red0 ^= 1;
}

// the look-ahead sweeps of every level-0 slab, from the committed red
// values into the other buffers, with their red residual partials (cnt[s]
// of slab s at partials + pbase[s] + off[s]); then the red ghost exchange
// of the other buffers (the next cycle's black sweep reads them)
int lookahead_sweeps(mg_ctx *c, int *cnt) {
  for (size_t s = 0; s < c->g[0].size(); s++) {
    cnt[s] += mg::launch_smooth_lookahead_march(c->g0alt[s], c->tm[0][s].b,
                                                c->g[0][s].phiR,
                                                c->partials + c->pbase[s] + cnt[s],
                                                c->stream);
    c->launches++;
  }
  CK(cudaGetLastError());
  la_swap(c);
  const int rc = halo(c, 0, 0);
  la_swap(c);
  return rc;
}

// the look-ahead of the committed iterate (eager: before the first
// look-ahead cycle after a change); its residual partials are not used.
// The black ghosts are exchanged first (the committed iterate may come
// from mg_set_solution or a single step).
int la_prologue(mg_ctx *c) {
  int rc;
  if ((rc = halo(c, 0, 1))) return rc;
  int cnt[kMaxSlabs] = {0};
  if ((rc = lookahead_sweeps(c, cnt))) return rc;
  c->la_valid = true;
  return MG_OK;
}

// the end of a look-ahead cycle, after the last red post-smoothing
// half-sweep: black sweep + black residual partials on every slab, the black
// ghost exchange, the look-ahead red sweeps into the other buffers + red
// residual partials, their ghost exchange, the ordered sums
int lookahead_tail(mg_ctx *c) {
  mark(c, CAT_NONE);
  int cnt[kMaxSlabs] = {0};
  for (size_t s = 0; s < c->g[0].size(); s++) {
    cnt[s] = mg::launch_smooth_norm_march(c->g[0][s], c->tm[0][s].r, 1,
                                          c->partials + c->pbase[s], c->stream);
    c->launches++;
  }
  CK(cudaGetLastError());
  int rc;
  if ((rc = halo(c, 0, 1))) return rc;
  mark(c, CAT_SMOOTH0);
  if ((rc = lookahead_sweeps(c, cnt))) return rc;
  c->paths |= MG_PATH_SPLIT_NORM | MG_PATH_LOOKAHEAD;
  return finish_norm(c, cnt);
}

// first level of the persistent tail kernel (k_vcycle_tail), or L for none:
// the first level >= 1 held whole on every rank with at most
// mg_opts.tail_cells cells, if the levels from there down are box or
// periodic grids whose coarsest solve is the single-CTA CG
int tail_level(const mg_ctx *c) {
  const int L = c->pl.L;
  if ((c->o.disable & MG_OFF_TAIL) || c->masked || L < 3) return L;
  const long long cap = c->o.tail_cells > 0 ? c->o.tail_cells : 32768;
  int ls = L;
  for (int l = c->pl.nd > 1 ? c->pl.nd : 1; l < L - 1; l++)
    if ((long long)c->pl.dims[l][0] * c->pl.dims[l][1] * c->pl.dims[l][2] <= cap) {
      ls = l;
      break;
    }
  if (ls >= L - 1 || L - ls > mg::kTailMax) return L;
  const Grid &gc = c->g[L - 1][0];
  if (!mg::vcycle_tail_supported(gc)) return L;
  if (cg_cluster_on(c) && mg::coarse_cg_cluster_supported(gc)) return L;
  return ls;
}

// levels ls..L-1 (copy s of each) in one persistent cluster kernel
int tail_launch(mg_ctx *c, int ls) {
  for (int s = 0; s < c->ncopy; s++) {
    mg::TailLevels T;
    T.n = c->pl.L - ls;
    for (int k = 0; k < T.n; k++) T.g[k] = c->g[ls + k][c->ncopy > 1 ? s : 0];
    if (mg::launch_vcycle_tail(T, c->o.nu1, c->o.nu2, c->o.alpha, c->o.coarse_tol,
                               c->o.coarse_maxit, c->cg_scr, c->cg_iters, c->stream))
      return fail(MG_ERR_CUDA, "tail kernel launch: %s",
                  cudaGetErrorString(cudaGetLastError()));
    c->launches++;
  }
  c->paths |= MG_PATH_TAIL;
  return MG_OK;
}

// profiling category of the work on level l >= 1 (not level 0)
int level_cat(const mg_ctx *c, int l) {
  if (l < 1 || l > c->pl.L - 2) return CAT_NONE;
  return distributed(c, l) ? CAT_COARSE : CAT_AGG;
}

// la: a look-ahead cycle (lookahead_ok): level 0's first red half-sweep was
// done by the previous cycle (or la_prologue), the cycle ends with
// lookahead_tail
int enqueue_vcycle_(mg_ctx *c, bool la);
int enqueue_vcycle(mg_ctx *c, bool la = false) {
  c->in_cycle = true;
  const int rc = enqueue_vcycle_(c, la);
  c->in_cycle = false;
  return rc;
}
int enqueue_vcycle_(mg_ctx *c, bool la) {
  const int L = c->pl.L;
  int rc;
  c->launches = 0;
  c->nev = 0;
  c->paths = 0;
  if (c->use_march && !c->tm[0].empty() && c->tm[0][0].ok) c->paths |= MG_PATH_MARCH;
  if (fused_norm_on(c)) c->paths |= MG_PATH_FUSED_NORM;
  // levels top..L-1 are the tail kernel's (or just the coarsest's CG)
  const int ls = tail_level(c);
  const int top = ls < L ? ls : L - 1;
  // profiling marks on levels >= 1 only where the category changes (every
  // mark is an event node in the graph)
  for (int l = 0; l < top; l++) {
    if (l >= 2 && level_cat(c, l - 1) != level_cat(c, l)) mark(c, level_cat(c, l - 1));
    if (c->o.nu1 == 0 && l > 0)
      for (const Grid &g : c->g[l]) {
        CK(cudaMemsetAsync(g.phiR, 0, sizeof(double) * mg::grid_elems(g), c->stream));
        CK(cudaMemsetAsync(g.phiB, 0, sizeof(double) * mg::grid_elems(g), c->stream));
      }
    for (int s = 0; s < c->o.nu1; s++) {
      // (l > 0, s == 0: from Phi = 0 -- done by the restriction of level l-1;
      // l == 0, s == 0 in a look-ahead cycle: done by the previous cycle)
      if (!(s == 0 && l == 0 && la) && !(s == 0 && l > 0 && red0_fused(c, l - 1, top)))
        if ((rc = smooth_half(c, l, 0, (l > 0 && s == 0) ? 1 : 0))) return rc;
      if ((rc = smooth_half(c, l, 1, 0))) return rc;
    }
    if ((rc = restrict_level(c, l, red0_fused(c, l, top)))) return rc;
  }
  const int before = level_cat(c, top - 1);  // CAT_NONE: level 0 came last
  int open_cat;  // category of the interval open after the coarse end
  if (ls < L) {
    if (before != CAT_NONE && before != CAT_AGG) mark(c, before);
    if ((rc = tail_launch(c, ls))) return rc;
    open_cat = CAT_AGG;
  } else {
    if (before != CAT_NONE) mark(c, before);
    if ((rc = coarse_solve(c))) return rc;
    mark(c, CAT_CG);
    open_cat = CAT_NONE;
  }
  for (int l = top - 1; l >= 0; l--) {
    if (l < top - 1) open_cat = level_cat(c, l + 1);
    if (open_cat != CAT_NONE && (l == 0 || open_cat != level_cat(c, l))) mark(c, open_cat);
    const bool fuse = can_fuse_prolong(c, l);
    if (fuse) {
      if ((rc = prolong_red_level(c, l))) return rc;
    } else {
      if ((rc = prolong_level(c, l))) return rc;
    }
    const bool split_n = l == 0 && split_norm_ok(c);
    for (int s = 0; s < c->o.nu2; s++) {
      if (!(fuse && s == 0))
        if ((rc = smooth_half(c, l, 0, 0))) return rc;
      if (split_n && s == c->o.nu2 - 1) break;  // the last black: split_norm_tail
      if ((rc = smooth_half(c, l, 1, 0))) return rc;
    }
    if (split_n) {
      if ((rc = la ? lookahead_tail(c) : split_norm_tail(c))) return rc;
      c->cycle_launches = c->launches;
      c->prof_last = c->prof;
      return MG_OK;
    }
  }
  // fused norm (c11): already published by the level-0 restriction
  rc = fused_norm_on(c) ? MG_OK : enqueue_norm(c);
  c->cycle_launches = c->launches;
  c->prof_last = c->prof;
  return rc;
}

// Wait for the context's stream.  NCCL contexts poll instead of blocking
// (failure detection): the stream's completion, the
// communicator's asynchronous error and a timeout (mg_opts.nccl_timeout_ms);
// a failed or timed-out communicator is aborted -- so that a dead peer does
// not hang the caller -- and the call returns MG_ERR_NCCL (the context can
// then only be destroyed).
int sync(mg_ctx *c) {
  if (c->backend != MG_HALO_NCCL || c->P == 1) {
    CK(cudaStreamSynchronize(c->stream));
    return MG_OK;
  }
  if (!c->comm) return fail(MG_ERR_NCCL, "the communicator was aborted");
  CK(cudaEventRecord(c->ev_sync, c->stream));
  const auto t0 = std::chrono::steady_clock::now();
  for (long spin = 0;; spin++) {
    const cudaError_t e = cudaEventQuery(c->ev_sync);
    if (e == cudaSuccess) return MG_OK;
    if (e != cudaErrorNotReady) return ck(e, "cudaEventQuery") ? MG_OK : MG_ERR_CUDA;
    ncclResult_t ae = ncclSuccess;
    const bool nccl_err = g_nccl.CommGetAsyncError(c->comm, &ae) != ncclSuccess ||
                          (ae != ncclSuccess && ae != ncclInProgress);
    const double ms = std::chrono::duration<double, std::milli>(
                          std::chrono::steady_clock::now() - t0).count();
    const bool late = c->o.nccl_timeout_ms > 0 && ms > c->o.nccl_timeout_ms;
    if (nccl_err || late) {
      g_nccl.CommAbort(c->comm);
      c->comm = nullptr;
      return nccl_err ? fail(MG_ERR_NCCL, "communicator error: %s",
                             g_nccl.GetErrorString(ae))
                      : fail(MG_ERR_NCCL, "no progress for %d ms (a peer died?); "
                             "communicator aborted", c->o.nccl_timeout_ms);
    }
    if (spin > 64) {  // past the first microseconds: yield the core
      const timespec ts{0, 20000};
      nanosleep(&ts, nullptr);
    }
  }
}

// staging buffer for natural-layout host/device transfers of level l
int stage_for(mg_ctx *c, size_t bytes) {
  if (c->stage_bytes >= bytes) return MG_OK;
  if (c->stage) cudaFree(c->stage);
  c->stage = nullptr;
  c->stage_bytes = 0;
  CK(cudaMalloc(&c->stage, bytes));
  c->stage_bytes = bytes;
  return MG_OK;
}

// pinned host staging of >= n doubles; returned idle: no copy enqueued on
// the context's stream reads or writes it any more
double *host_pinned(mg_ctx *c, size_t n) {
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return nullptr;
  if (n > c->hpin_cap) {
    if (c->hpin) cudaFreeHost(c->hpin);
    c->hpin = nullptr;
    c->hpin_cap = 0;
    if (cudaMallocHost(&c->hpin, n * sizeof(double)) != cudaSuccess) return nullptr;
    c->hpin_cap = n;
  }
  return c->hpin;
}

size_t level_cells_held(const mg_ctx *c, int l) {
  size_t n = 0;
  for (size_t s = 0; s < io_grids(c, l); s++) {
    const Grid &g = c->g[l][s];
    n += (size_t)g.nxl * g.ny * g.nz;
  }
  return n;
}

int field_io(mg_ctx *c, int l, int field, double *buf, int where, bool in,
             bool do_sync = true) {
  if (l < 0 || l >= c->pl.L) return fail(MG_ERR_ARG, "level %d out of range", l);
  if (field != MG_FIELD_PHI && field != MG_FIELD_RHS)
    return fail(MG_ERR_ARG, "bad field %d", field);
  if (!buf) return fail(MG_ERR_ARG, "null pointer");
  const size_t n = level_cells_held(c, l);
  double *dev = buf;
  int rc;
  if (where == MG_HOST) {
    if ((rc = stage_for(c, n * sizeof(double)))) return rc;
    dev = c->stage;
    if (in)
      CK(cudaMemcpyAsync(dev, buf, n * sizeof(double), cudaMemcpyHostToDevice,
                         c->stream));
  } else if (where != MG_DEVICE) {
    return fail(MG_ERR_ARG, "bad 'where' %d", where);
  }
  size_t off = 0;
  for (size_t s = 0; s < c->g[l].size(); s++) {
    const Grid &g = c->g[l][s];
    if (in)
      mg::launch_pack(g, field, dev + off, c->stream);  // every copy
    else if (s < io_grids(c, l))
      mg::launch_unpack(g, field, dev + off, c->stream);
    if (s + 1 < io_grids(c, l)) off += (size_t)g.nxl * g.ny * g.nz;
  }
  CK(cudaGetLastError());
  if (in) {
    // refresh ghost planes of both colours for a distributed level, and the
    // periodic ghosts of grids held whole
    if (field == MG_FIELD_PHI) {
      periodic_fill(c, l);
      CK(cudaGetLastError());
      if ((rc = halo(c, l, 0))) return rc;
      if ((rc = halo(c, l, 1))) return rc;
    }
  } else if (where == MG_HOST) {
    CK(cudaMemcpyAsync(buf, dev, n * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream));
  }
  return do_sync ? sync(c) : MG_OK;
}

int bc_adapt(mg_ctx *c) {
  const double alpha = -1.0 * (1.0 / (c->h * c->h));
  double terms[6];
  int types[6];
  for (int q = 0; q < 6; q++) {
    const double g = c->bc[q].value;
    types[q] = c->bc[q].type;
    terms[q] = c->bc[q].type == MG_DIRICHLET ? 2.0 * alpha * g : alpha * (c->h * g);
  }
  for (const Grid &g : c->g[0]) {
    mg::launch_zero_solid(g, c->stream);  // masked cells are not unknowns
    if (c->patched)
      mg::launch_bc_adapt_faces(g, c->fbc, alpha, c->h, c->stream);
    else
      mg::launch_bc_adapt(g, terms, types, c->stream);
  }
  CK(cudaGetLastError());
  return MG_OK;
}

void free_mask(mg_ctx *c) {
  for (void *p : c->mask_bufs) cudaFree(p);
  c->mask_bufs.clear();
  for (auto &lv : c->g)
    for (Grid &g : lv) {
      g.codeR = g.codeB = nullptr;
      g.coefR = g.coefB = nullptr;
      g.c64R = g.c64B = nullptr;
      g.ukR = g.ukB = nullptr;
      g.all_unknown = 0;
    }
  c->masked = false;
}

// the look-ahead view of level 0 = the committed view with the other red
// buffer (after any change of the level-0 grid's coefficient fields)
void sync_alt_view(mg_ctx *c) {
  for (size_t s = 0; s < c->g0alt.size(); s++) {
    double *alt = c->g0alt[s].phiR;
    c->g0alt[s] = c->g[0][s];
    c->g0alt[s].phiR = alt;
  }
}

int residual_norm_now(mg_ctx *c, double *out) {
  int rc = enqueue_norm(c);
  if (rc) return rc;
  if ((rc = sync(c))) return rc;
  *out = sqrt(*c->h_norm);
  return MG_OK;
}

// spheres on a periodic axis: centre in [0, n h) and 2R + 2h <= n h, so the
// periodic images of a sphere cover disjoint cells (mg.h)
int check_sphere(const mg_ctx *c, int p, const double *ctr, double R) {
  if (!(R > 0.0)) return fail(MG_ERR_ARG, "sphere %d: radius <= 0", p);
  for (int a = 0; a < 3; a++) {
    if (c->bc[2 * a].type != MG_PERIODIC) continue;
    const double len = (double)c->pl.dims[0][a] * c->h;
    if (!(ctr[a] >= 0.0 && ctr[a] < len) || !(2.0 * R + 2.0 * c->h <= len))
      return fail(MG_ERR_ARG,
                  "sphere %d on periodic axis %d: need centre in [0, %g) and "
                  "2R + 2h <= %g", p, a, len, len);
  }
  return MG_OK;
}

}  // namespace

// ==== C-ABI ======================================================================
extern "C" {

void mg_default_opts(mg_opts *o) {
  memset(o, 0, sizeof *o);
  o->nu1 = 2;
  o->nu2 = 2;
  o->alpha = 2.0;
  o->min_coarse = 4;
  o->max_levels = 0;
  o->agglomerate_below = 64LL * 64 * 64;
  o->coarse_tol = 1e-12;
  o->coarse_maxit = 1000;
  o->max_cycles = 100;
  o->device = 0;
  o->stream = nullptr;
  o->rank = 0;
  o->nranks = 1;
  o->halo_backend = MG_HALO_NONE;
  o->workspace = nullptr;
  o->workspace_bytes = 0;
  o->use_graph = 1;
  o->nccl_timeout_ms = 600000;
}

const char *mg_strerror(int code) {
  switch (code) {
    case MG_OK: return "MG_OK";
    case MG_ERR_ARG: return "MG_ERR_ARG";
    case MG_ERR_BC: return "MG_ERR_BC";
    case MG_ERR_COARSEN: return "MG_ERR_COARSEN";
    case MG_ERR_CUDA: return "MG_ERR_CUDA";
    case MG_ERR_NCCL: return "MG_ERR_NCCL";
    case MG_ERR_NOMEM: return "MG_ERR_NOMEM";
    case MG_ERR_DIVERGED: return "MG_ERR_DIVERGED";
    case MG_ERR_NOTCONV: return "MG_ERR_NOTCONV";
    default: return "MG_ERR_UNKNOWN";
  }
}

const char *mg_last_error(const mg_ctx *) { return g_err.c_str(); }

int mg_halo_schedule(int nranks, int rank, int periodic_x, int ops[4][3]) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !ops) return MG_ERR_ARG;
  const int left = rank > 0 ? rank - 1 : (periodic_x ? nranks - 1 : -1);
  const int right = rank < nranks - 1 ? rank + 1 : (periodic_x ? 0 : -1);
  int n = 0;
  auto put = [&](int op, int peer, int plane) {
    ops[n][0] = op;
    ops[n][1] = peer;
    ops[n][2] = plane;
    n++;
  };
  if (nranks == 1) return 0;
  if (right >= 0) put(MG_OP_SEND, right, MG_PLANE_LAST);
  if (left >= 0) put(MG_OP_RECV, left, MG_GHOST_LO);
  if (left >= 0) put(MG_OP_SEND, left, MG_PLANE_FIRST);
  if (right >= 0) put(MG_OP_RECV, right, MG_GHOST_HI);
  return n;
}

int mg_last_error_code(void) { return g_err_code; }

int mg_plan(int nx, int ny, int nz, const mg_opts *o, int *nlevels,
            int *agg_level, int dims[][3], int *local_nx) {
  mg_opts d;
  if (!o) {
    mg_default_opts(&d);
    o = &d;
  }
  Plan pl;
  int rc = make_plan(nx, ny, nz, o, &pl);
  if (rc) return rc;
  if (nlevels) *nlevels = pl.L;
  if (agg_level) *agg_level = pl.P > 1 ? pl.nd : pl.L;
  for (int l = 0; l < pl.L; l++) {
    if (dims)
      for (int a = 0; a < 3; a++) dims[l][a] = pl.dims[l][a];
    if (local_nx) local_nx[l] = pl.nxl[l];
  }
  return MG_OK;
}

static int validate(int nx, int ny, int nz, double h, const mg_bc *bc,
                    const mg_opts *o) {
  if (!bc) return fail(MG_ERR_ARG, "bc is NULL");
  if (!(h > 0.0)) return fail(MG_ERR_ARG, "h must be positive");
  bool anyD = false;
  for (int q = 0; q < 6; q++) {
    if (bc[q].type != MG_DIRICHLET && bc[q].type != MG_NEUMANN &&
        bc[q].type != MG_PERIODIC)
      return fail(MG_ERR_BC, "face %d: unknown type %d", q, bc[q].type);
    anyD = anyD || bc[q].type == MG_DIRICHLET;
  }
  for (int a = 0; a < 3; a++)
    if ((bc[2 * a].type == MG_PERIODIC) != (bc[2 * a + 1].type == MG_PERIODIC))
      return fail(MG_ERR_BC, "axis %d: periodic faces come in pairs (P:441-443)", a);
  if (!anyD)
    return fail(MG_ERR_BC, "no Dirichlet face: the operator is singular");
  if (o->nu1 < 0 || o->nu2 < 0 || o->nu1 + o->nu2 < 1)
    return fail(MG_ERR_ARG, "need nu1, nu2 >= 0 and nu1 + nu2 >= 1");
  if (o->nranks < 1 || o->rank < 0 || o->rank >= o->nranks)
    return fail(MG_ERR_ARG, "bad rank %d / nranks %d", o->rank, o->nranks);
  if (o->nranks > 1 && o->halo_backend != MG_HALO_NCCL &&
      o->halo_backend != MG_HALO_LOOPBACK && o->halo_backend != MG_HALO_EMULATE)
    return fail(MG_ERR_ARG, "nranks > 1 needs the NCCL, LOOPBACK or EMULATE backend");
  if (o->nranks > kMaxSlabs && o->halo_backend != MG_HALO_NCCL)
    return fail(MG_ERR_ARG, "at most %d slabs in one process", kMaxSlabs);
  (void)nx;
  (void)ny;
  (void)nz;
  return MG_OK;
}

size_t mg_workspace_bytes(int nx, int ny, int nz, const mg_opts *o) {
  mg_opts d;
  if (!o) {
    mg_default_opts(&d);
    o = &d;
  }
  mg_ctx c;
  c.o = *o;
  if (make_plan(nx, ny, nz, o, &c.pl)) return 0;
  c.P = c.pl.P;
  const bool local = c.P > 1 && o->halo_backend != MG_HALO_NCCL;
  c.nslab = local ? c.P : 1;
  c.slab0 = local ? 0 : o->rank;
  c.ncopy = (c.P > 1 && o->halo_backend == MG_HALO_EMULATE) ? c.P : 1;
  c.h = 1.0;
  for (int q = 0; q < 6; q++) c.bc[q].type = MG_DIRICHLET;
  return carve(&c, nullptr);
}

int mg_nccl_unique_id(unsigned char out[128]) {
  if (!out) return fail(MG_ERR_ARG, "null pointer");
  if (!load_nccl()) return fail(MG_ERR_NCCL, "cannot load libnccl.so.2");
  ncclUniqueId id;
  int rc = nccl_ck(g_nccl.GetUniqueId(&id), "ncclGetUniqueId");
  if (rc) return rc;
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
  return MG_OK;
}

mg_ctx *mg_create_ex(int nx, int ny, int nz, double h, const mg_bc *bc,
                     const mg_opts *opts) {
  mg_opts d;
  if (!opts) {
    mg_default_opts(&d);
    opts = &d;
  }
  if (validate(nx, ny, nz, h, bc, opts)) return nullptr;
  mg_ctx *c = new mg_ctx();
  c->o = *opts;
  c->h = h;
  for (int q = 0; q < 6; q++) c->bc[q] = bc[q];
  if (make_plan(nx, ny, nz, opts, &c->pl)) {
    delete c;
    return nullptr;
  }
  c->P = c->pl.P;
  c->rank = opts->rank;
  c->backend = c->P > 1 ? opts->halo_backend : MG_HALO_NONE;
  c->nslab = (c->backend == MG_HALO_LOOPBACK || c->backend == MG_HALO_EMULATE) ? c->P : 1;
  c->slab0 = c->backend == MG_HALO_NCCL ? c->rank : 0;
  c->ncopy = c->backend == MG_HALO_EMULATE ? c->P : 1;
  c->dev = opts->device;
  auto bail = [&](cudaError_t e, const char *what) -> mg_ctx * {
    fail(MG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    mg_destroy(c);
    return nullptr;
  };
  cudaError_t e = cudaSetDevice(c->dev);
  if (e != cudaSuccess) return bail(e, "cudaSetDevice");
  e = cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, c->dev);
  if (e != cudaSuccess) return bail(e, "cudaDeviceGetAttribute(SM count)");
  if (c->nsm > 256) c->nsm = 256;  // kMaxNormBlocks bounds 8 CTAs per SM
  if (opts->stream) {
    c->stream = (cudaStream_t)opts->stream;
  } else {
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return bail(e, "cudaStreamCreate");
    c->own_stream = true;
  }
  const size_t need = carve(c, nullptr);
  if (opts->workspace) {
    if (opts->workspace_bytes < need) {
      fail(MG_ERR_NOMEM, "workspace of %zu bytes < %zu needed",
           opts->workspace_bytes, need);
      mg_destroy(c);
      return nullptr;
    }
    c->ws = (char *)opts->workspace;
    c->ws_bytes = opts->workspace_bytes;
  } else {
    e = cudaMalloc(&c->ws, need);
    if (e != cudaSuccess) {
      fail(MG_ERR_NOMEM, "cudaMalloc(%zu): %s", need, cudaGetErrorString(e));
      mg_destroy(c);
      return nullptr;
    }
    c->own_ws = true;
    c->ws_bytes = need;
  }
  // align the base to 256 bytes
  char *base = (char *)(((uintptr_t)c->ws + 255) & ~(uintptr_t)255);
  if ((size_t)(base - c->ws) + need > c->ws_bytes) {
    fail(MG_ERR_NOMEM, "workspace too small after alignment");
    mg_destroy(c);
    return nullptr;
  }
  carve(c, base);
  c->tm.assign(c->pl.L, {});
  for (int l = 0; l < c->pl.L; l++) {
    c->tm[l].resize(c->g[l].size());
    for (size_t s = 0; s < c->g[l].size(); s++) {
      const Grid &g = c->g[l][s];
      TmPair &t = c->tm[l][s];
      t.ok = mg::march_supported(g) && mg::make_tmap_field(g, g.phiR, t.r) &&
             mg::make_tmap_field(g, g.phiB, t.b);
      t.ok_resid = mg::resid_march_supported(g) &&
                   mg::make_tmap_resid(g, g.phiR, t.rr) &&
                   mg::make_tmap_resid(g, g.phiB, t.rb);
    }
  }
  for (size_t s = 0; s < c->red0_alt.size(); s++) {
    Grid ga = c->g[0][s];
    ga.phiR = c->red0_alt[s];
    c->g0alt.push_back(ga);
    const TmPair &t0 = c->tm[0][s];
    TmPair t = t0;  // the Phi^B maps are shared
    t.ok = t0.ok && mg::make_tmap_field(ga, ga.phiR, t.r);
    t.ok_resid = t0.ok_resid && mg::make_tmap_resid(ga, ga.phiR, t.rr);
    c->tm0alt.push_back(t);
  }
  // multi-slab overlap: views of the boundary / interior planes of every
  // distributed level (slabs of >= 4 planes), a communication stream
  if (c->P > 1 && !(opts->disable & MG_OFF_OVERLAP)) {
    c->vlo.assign(c->pl.L, {});
    c->vhi.assign(c->pl.L, {});
    c->vin.assign(c->pl.L, {});
    c->tmin.assign(c->pl.L, {});
    for (int l = 0; l < c->pl.nd; l++) {
      if (c->g[l][0].nxl < 4) continue;
      c->tmin[l].resize(c->g[l].size());
      for (size_t s = 0; s < c->g[l].size(); s++) {
        const Grid &g = c->g[l][s];
        c->vlo[l].push_back(plane_view(g, 0, 1));
        c->vhi[l].push_back(plane_view(g, g.nxl - 1, 1));
        const Grid vi = plane_view(g, 1, g.nxl - 2);
        c->vin[l].push_back(vi);
        TmPair &t = c->tmin[l][s];
        t.ok = mg::march_supported(vi) && mg::make_tmap_field(vi, vi.phiR, t.r) &&
               mg::make_tmap_field(vi, vi.phiB, t.b);
      }
    }
    // the same views of the look-ahead buffers (level 0)
    if (!c->g0alt.empty() && !c->vin[0].empty()) {
      for (size_t s = 0; s < c->g0alt.size(); s++) {
        const Grid &g = c->g0alt[s];
        c->vlo0alt.push_back(plane_view(g, 0, 1));
        c->vhi0alt.push_back(plane_view(g, g.nxl - 1, 1));
        const Grid vi = plane_view(g, 1, g.nxl - 2);
        c->vin0alt.push_back(vi);
        TmPair t;
        t.ok = mg::march_supported(vi) && mg::make_tmap_field(vi, vi.phiR, t.r) &&
               mg::make_tmap_field(vi, vi.phiB, t.b);
        c->tmin0alt.push_back(t);
      }
    }
    e = cudaStreamCreateWithFlags(&c->s_comm, cudaStreamNonBlocking);
    if (e != cudaSuccess) return bail(e, "cudaStreamCreate(comm)");
    e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
    if (e != cudaSuccess) return bail(e, "cudaEventCreate");
    e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
    if (e != cudaSuccess) return bail(e, "cudaEventCreate");
  } else {
    c->overlap = 0;
  }
  if (opts->disable & MG_OFF_MARCH) c->use_march = 0;
  e = cudaMemsetAsync(base, 0, need - 256, c->stream);
  if (e != cudaSuccess) return bail(e, "cudaMemsetAsync");
  e = cudaHostAlloc(&c->h_norm, sizeof(double) * 2, cudaHostAllocMapped);
  if (e != cudaSuccess) return bail(e, "cudaHostAlloc");
  e = cudaHostGetDevicePointer(&c->h_norm_dev, c->h_norm, 0);
  if (e != cudaSuccess) return bail(e, "cudaHostGetDevicePointer");
  e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return bail(e, "cudaStreamSynchronize");
  if (c->backend == MG_HALO_NCCL) {
    if (!load_nccl()) {
      fail(MG_ERR_NCCL, "cannot load libnccl.so.2");
      mg_destroy(c);
      return nullptr;
    }
    e = cudaEventCreateWithFlags(&c->ev_sync, cudaEventDisableTiming);
    if (e != cudaSuccess) return bail(e, "cudaEventCreate(sync)");
    ncclUniqueId id;
    memcpy(&id, opts->nccl_id, sizeof id);
    if (nccl_ck(g_nccl.CommInitRank(&c->comm, c->P, id, c->rank),
                "ncclCommInitRank")) {
      c->comm = nullptr;
      mg_destroy(c);
      return nullptr;
    }
  }
  return c;
}

mg_ctx *mg_create(int nx, int ny, int nz, double h, const mg_bc *bc) {
  return mg_create_ex(nx, ny, nz, h, bc, nullptr);
}

void mg_destroy(mg_ctx *c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  for (int k = 0; k < 2; k++)
    if (c->graph_la[k]) cudaGraphExecDestroy(c->graph_la[k]);
  for (auto &e : c->ev) cudaEventDestroy(e);
  if (c->comm && g_nccl.ok) g_nccl.CommDestroy(c->comm);
  if (c->stage) cudaFree(c->stage);
  if (c->s_comm) {
    cudaStreamSynchronize(c->s_comm);
    cudaStreamDestroy(c->s_comm);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->ev_sync) cudaEventDestroy(c->ev_sync);
  if (c->s_aux) {
    cudaStreamSynchronize(c->s_aux);
    cudaStreamDestroy(c->s_aux);
  }
  if (c->ev_aux0) cudaEventDestroy(c->ev_aux0);
  if (c->ev_aux1) cudaEventDestroy(c->ev_aux1);
  if (c->s_h2d) cudaStreamSynchronize(c->s_h2d);
  if (c->s_d2h) cudaStreamSynchronize(c->s_d2h);
  for (int q = 0; q < 3; q++) {
    if (c->astg[q]) cudaFree(c->astg[q]);
    if (c->ev_in[q]) cudaEventDestroy(c->ev_in[q]);
    if (c->ev_out[q]) cudaEventDestroy(c->ev_out[q]);
    if (c->ev_d2h[q]) cudaEventDestroy(c->ev_d2h[q]);
    if (c->ev_free[q]) cudaEventDestroy(c->ev_free[q]);
  }
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  if (c->sph) cudaFree(c->sph);
  if (c->bins) cudaFree(c->bins);
  if (c->fbuf) cudaFree(c->fbuf);
  if (c->hpin) cudaFreeHost(c->hpin);
  for (void *p : c->mask_bufs) cudaFree(p);
  if (c->h_norm) cudaFreeHost(c->h_norm);
  if (c->own_ws && c->ws) cudaFree(c->ws);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int mg_num_levels(const mg_ctx *c) { return c ? c->pl.L : MG_ERR_ARG; }

int mg_level_dims(const mg_ctx *c, int l, int dims[3]) {
  if (!c || !dims || l < 0 || l >= c->pl.L) return fail(MG_ERR_ARG, "bad level");
  for (int a = 0; a < 3; a++) dims[a] = c->pl.dims[l][a];
  return MG_OK;
}

int mg_set_rhs(mg_ctx *c, const double *f, int where) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  la_drop(c);
  int rc = field_io(c, 0, MG_FIELD_RHS, const_cast<double *>(f), where, true);
  if (rc) return rc;
  if ((rc = bc_adapt(c))) return rc;
  c->prev_norm = -1.0;
  return sync(c);
}

// enqueue the sphere RHS (no host synchronisation); *check: the empty-sphere
// flag (mapped h_norm[1]) is being computed and must be read after a sync
static int rhs_from_spheres(mg_ctx *c, int n, const double *centers, const double *radii,
                            const double *charges, int normalization, int subsample,
                            bool *check_out) {
  *check_out = false;
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  la_drop(c);
  if (n < 0) return fail(MG_ERR_ARG, "n < 0");
  if (subsample < 1 || subsample > 16)
    return fail(MG_ERR_ARG, "subsample must be in 1..16");
  if (normalization != MG_CHARGE_PER_CELLS && normalization != MG_CHARGE_PER_VOLUME)
    return fail(MG_ERR_ARG, "bad normalization");
  if (n > 0 && (!centers || !radii || !charges)) return fail(MG_ERR_ARG, "null array");
  for (int p = 0; p < n; p++)
    if (int rc = check_sphere(c, p, centers + 3 * (size_t)p, radii[p])) return rc;
  // the sphere list through pinned staging (an asynchronous upload)
  double *h5 = n > 0 ? host_pinned(c, 5 * (size_t)n) : nullptr;
  if (n > 0 && !h5) return fail(MG_ERR_CUDA, "pinned staging allocation failed");
  for (int p = 0; p < n; p++) {
    for (int a = 0; a < 3; a++) h5[5 * (size_t)p + a] = centers[3 * (size_t)p + a];
    h5[5 * (size_t)p + 3] = radii[p];
    h5[5 * (size_t)p + 4] = charges[p];
  }
  if ((size_t)n > c->sph_cap) {
    if (c->sph) cudaFree(c->sph);
    c->sph = nullptr;
    c->sph_cap = 0;
    CK(cudaMalloc(&c->sph, sizeof(double) * 5 * (size_t)n + sizeof(unsigned long long) * (size_t)n));
    c->sph_cap = (size_t)n;
  }
  unsigned long long *cnt = (unsigned long long *)(c->sph + 5 * c->sph_cap);
  // f := 0 on the side stream (bandwidth-bound) overlapping the bins,
  // neighbour lists and counts (ALU-bound, not touching f); joined before
  // the scatter
  if (!c->s_aux) {
    CK(cudaStreamCreateWithFlags(&c->s_aux, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->ev_aux0, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_aux1, cudaEventDisableTiming));
  }
  CK(cudaEventRecord(c->ev_aux0, c->stream));
  CK(cudaStreamWaitEvent(c->s_aux, c->ev_aux0, 0));
  for (const Grid &g : c->g[0]) {
    CK(cudaMemsetAsync(g.fR, 0, sizeof(double) * mg::grid_elems(g), c->s_aux));
    CK(cudaMemsetAsync(g.fB, 0, sizeof(double) * mg::grid_elems(g), c->s_aux));
  }
  CK(cudaEventRecord(c->ev_aux1, c->s_aux));
  if (n > 0) {
    CK(cudaMemcpyAsync(c->sph, h5, sizeof(double) * 5 * (size_t)n,
                       cudaMemcpyHostToDevice, c->stream));
    // bins of the centres for the scatter's neighbour search: wider than
    // 2 R_max + 2 cells, at most 64 per axis; on periodic axes the bin width
    // divides the extent (exact wrap of bin indices)
    mg::SphereBins B;
    B.rmax = 0.0;
    for (int p = 0; p < n; p++) B.rmax = radii[p] > B.rmax ? radii[p] : B.rmax;
    const int bcmin = (int)ceil(2.0 * B.rmax / c->h) + 2;
    size_t nbins = 1;
    for (int a = 0; a < 3; a++) {
      const int ext = c->pl.dims[0][a];
      int bc = bcmin > (ext + 63) / 64 ? bcmin : (ext + 63) / 64;
      if (bc > ext) bc = ext;
      if (c->bc[2 * a].type == MG_PERIODIC)
        while (ext % bc) bc++;
      B.bc[a] = bc;
      B.nb[a] = (ext + bc - 1) / bc;
      nbins *= (size_t)B.nb[a];
    }
    // + neighbour lists: nn[n], nbr[n kNbMax], list[2n], nlist[2]
    const size_t need = nbins * (1 + mg::kBinCap) + (size_t)n * (3 + mg::kNbMax) + 2;
    if (need > c->bins_cap) {
      if (c->bins) cudaFree(c->bins);
      c->bins = nullptr;
      c->bins_cap = 0;
      CK(cudaMalloc(&c->bins, need * sizeof(int)));
      c->bins_cap = need;
    }
    B.count = c->bins;
    B.items = c->bins + nbins;
    mg::SphereLists S;
    S.nn = B.items + nbins * mg::kBinCap;
    S.nbr = S.nn + n;
    S.list = S.nbr + (size_t)n * mg::kNbMax;
    S.nlist = S.list + 2 * (size_t)n;
    CK(cudaMemsetAsync(B.count, 0, nbins * sizeof(int), c->stream));
    CK(cudaMemsetAsync(S.nlist, 0, 2 * sizeof(int), c->stream));
    mg::launch_sphere_bin(c->g[0][0], c->h, n, c->sph, B, c->stream);
    mg::launch_sphere_neighbours(c->g[0][0], c->h, n, c->sph, B, S, c->stream);
    mg::launch_sphere_counts(c->g[0][0], c->h, subsample, n, c->sph, cnt, c->stream);
    CK(cudaStreamWaitEvent(c->stream, c->ev_aux1, 0));  // f cleared
    for (const Grid &g : c->g[0])
      mg::launch_sphere_scatter(g, c->h, subsample, n, c->sph, normalization, cnt, S,
                                c->stream);
    CK(cudaGetLastError());
  }
  CK(cudaStreamWaitEvent(c->stream, c->ev_aux1, 0));  // (n == 0: the clear alone)
  int rc = bc_adapt(c);
  if (rc) return rc;
  c->prev_norm = -1.0;
  // the empty-sphere check reads back through mapped memory: a copy-engine
  // transfer would queue behind a pending bulk download (get_solution_async)
  const bool check = normalization == MG_CHARGE_PER_CELLS && n > 0;
  if (check) mg::launch_first_empty(cnt, n, c->h_norm_dev + 1, c->stream);
  CK(cudaGetLastError());
  *check_out = check;
  return MG_OK;
}

// the empty-sphere verdict of rhs_from_spheres (after a sync)
static int empty_sphere_check(mg_ctx *c, bool check) {
  if (check && c->h_norm[1] >= 0.0)
    return fail(MG_ERR_ARG, "sphere %d covers no cell centre", (int)c->h_norm[1]);
  return MG_OK;
}

int mg_set_rhs_from_spheres(mg_ctx *c, int n, const double *centers,
                            const double *radii, const double *charges,
                            int normalization, int subsample) {
  Nvtx nv("mg_set_rhs_from_spheres");
  bool check;
  int rc = rhs_from_spheres(c, n, centers, radii, charges, normalization, subsample, &check);
  if (rc) return rc;
  if ((rc = sync(c))) return rc;
  return empty_sphere_check(c, check);
}

// enqueue one V-cycle (graph launch, recorded on first use); no host sync.
// allow_la: the look-ahead form where the context supports it (else, and
// for a single cycle after a change of f -- mg_timestep --, the plain form)
static int enqueue_cycle(mg_ctx *c, bool allow_la = true) {
  int rc;
  if (allow_la && lookahead_ok(c)) {
    if (!c->la_valid && (rc = la_prologue(c))) return rc;
    la_swap(c);  // the cycle continues from the look-ahead buffer
    c->la_valid = false;  // (until the cycle is enqueued)
    if (c->o.use_graph) {
      cudaGraphExec_t &gx = c->graph_la[c->red0];
      if (!gx) {
        cudaGraph_t gr;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        rc = enqueue_vcycle(c, true);
        cudaError_t e = cudaStreamEndCapture(c->stream, &gr);
        if (!rc && e != cudaSuccess)
          rc = fail(MG_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
        if (!rc && cudaGraphInstantiate(&gx, gr, 0) != cudaSuccess)
          rc = fail(MG_ERR_CUDA, "cudaGraphInstantiate failed");
        if (e == cudaSuccess) cudaGraphDestroy(gr);
        if (rc) {
          la_swap(c);  // back to the committed iterate (look-ahead dropped)
          return rc;
        }
      }
      CK(cudaGraphLaunch(gx, c->stream));
    } else if ((rc = enqueue_vcycle(c, true))) {
      return rc;
    }
    c->la_valid = true;
    return MG_OK;
  }
  la_drop(c);
  if (c->o.use_graph) {
    if (!c->graph) {
      cudaGraph_t gr;
      CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      rc = enqueue_vcycle(c);
      cudaError_t e = cudaStreamEndCapture(c->stream, &gr);
      if (rc) return rc;
      CK(e);
      CK(cudaGraphInstantiate(&c->graph, gr, 0));
      cudaGraphDestroy(gr);
    }
    CK(cudaGraphLaunch(c->graph, c->stream));
    return MG_OK;
  }
  return enqueue_vcycle(c);
}

// natural <-> split conversion of level 0 from / to a device buffer
static int pack0(mg_ctx *c, int field, const double *dev) {
  size_t off = 0;
  for (const Grid &g : c->g[0]) {
    mg::launch_pack(g, field, dev + off, c->stream);
    off += (size_t)g.nxl * g.ny * g.nz;
  }
  CK(cudaGetLastError());
  return MG_OK;
}
static int unpack0(mg_ctx *c, int field, double *dev) {
  size_t off = 0;
  for (const Grid &g : c->g[0]) {
    mg::launch_unpack(g, field, dev + off, c->stream);
    off += (size_t)g.nxl * g.ny * g.nz;
  }
  CK(cudaGetLastError());
  return MG_OK;
}

static int async_setup(mg_ctx *c, size_t bytes) {
  if (!c->s_h2d) {
    CK(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    for (int q = 0; q < 3; q++) {
      CK(cudaEventCreateWithFlags(&c->ev_in[q], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_out[q], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_d2h[q], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_free[q], cudaEventDisableTiming));
    }
  }
  if (c->astg_bytes < bytes) {
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaStreamSynchronize(c->s_h2d));
    CK(cudaStreamSynchronize(c->s_d2h));
    for (int q = 0; q < 3; q++) {
      if (c->astg[q]) cudaFree(c->astg[q]);
      c->astg[q] = nullptr;
      c->d2h_used[q] = false;
      c->free_used[q] = false;
    }
    c->astg_bytes = 0;
    for (int q = 0; q < 3; q++) CK(cudaMalloc(&c->astg[q], bytes));
    c->astg_bytes = bytes;
  }
  return MG_OK;
}

// Pipeline of independent solves: problem k uses staging slot k % 3.  The
// H2D of its f runs on the context's h2d stream (after the D2H that last
// used the slot), the cycles on the context's stream, the D2H of Phi on the
// d2h stream -- so problem k+1's upload and problem k-1's download overlap
// problem k's cycles, while the cycles of consecutive problems stay
// serialised on one stream.
int mg_solve_async(mg_ctx *c, const double *f, int where_f, double *phi_out,
                   int where_phi, int cycles) {
  Nvtx nv("mg_solve_async");
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  la_drop(c);
  if (cycles < 0) return fail(MG_ERR_ARG, "cycles < 0");
  if (!f) return fail(MG_ERR_ARG, "null f");
  if ((where_f != MG_HOST && where_f != MG_DEVICE) ||
      (phi_out && where_phi != MG_HOST && where_phi != MG_DEVICE))
    return fail(MG_ERR_ARG, "bad 'where'");
  const size_t n = level_cells_held(c, 0);
  int rc;
  if ((rc = async_setup(c, n * sizeof(double)))) return rc;
  const int q = (int)(c->async_k++ % 3);
  double *stg = c->astg[q];
  if (where_f == MG_HOST) {
    // the slot's previous users must be done with it: a download of Phi
    // (ev_d2h) and the context stream's last read of it (ev_free: an RHS
    // conversion, whatever the previous problem's phi_out was)
    if (c->d2h_used[q]) CK(cudaStreamWaitEvent(c->s_h2d, c->ev_d2h[q], 0));
    if (c->free_used[q]) CK(cudaStreamWaitEvent(c->s_h2d, c->ev_free[q], 0));
    CK(cudaMemcpyAsync(stg, f, n * sizeof(double), cudaMemcpyHostToDevice, c->s_h2d));
    CK(cudaEventRecord(c->ev_in[q], c->s_h2d));
    CK(cudaStreamWaitEvent(c->stream, c->ev_in[q], 0));
    if ((rc = pack0(c, MG_FIELD_RHS, stg))) return rc;
    CK(cudaEventRecord(c->ev_free[q], c->stream));
    c->free_used[q] = true;
  } else if ((rc = pack0(c, MG_FIELD_RHS, f))) {
    return rc;
  }
  if ((rc = bc_adapt(c))) return rc;
  for (const Grid &g : c->g[0]) {
    CK(cudaMemsetAsync(g.phiR, 0, sizeof(double) * mg::grid_elems(g), c->stream));
    CK(cudaMemsetAsync(g.phiB, 0, sizeof(double) * mg::grid_elems(g), c->stream));
  }
  c->prev_norm = -1.0;
  for (int k = 0; k < cycles; k++)
    if ((rc = enqueue_cycle(c))) return rc;
  if (phi_out) {
    if (where_phi == MG_HOST) {
      if ((rc = unpack0(c, MG_FIELD_PHI, stg))) return rc;
      CK(cudaEventRecord(c->ev_out[q], c->stream));
      CK(cudaStreamWaitEvent(c->s_d2h, c->ev_out[q], 0));
      CK(cudaMemcpyAsync(phi_out, stg, n * sizeof(double), cudaMemcpyDeviceToHost,
                         c->s_d2h));
      CK(cudaEventRecord(c->ev_d2h[q], c->s_d2h));
      c->d2h_used[q] = true;
    } else if ((rc = unpack0(c, MG_FIELD_PHI, phi_out))) {
      return rc;
    }
  }
  return MG_OK;
}

int mg_get_solution_async(mg_ctx *c, double *out, int where) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  if (!out) return fail(MG_ERR_ARG, "null out");
  if (where != MG_HOST && where != MG_DEVICE) return fail(MG_ERR_ARG, "bad 'where'");
  if (where == MG_DEVICE) return unpack0(c, MG_FIELD_PHI, out);
  const size_t n = level_cells_held(c, 0);
  int rc;
  if ((rc = async_setup(c, n * sizeof(double)))) return rc;
  const int q = (int)(c->async_k++ % 3);
  double *stg = c->astg[q];
  // the slot's previous download must have left it before it is rewritten
  if (c->d2h_used[q]) CK(cudaStreamWaitEvent(c->stream, c->ev_d2h[q], 0));
  if ((rc = unpack0(c, MG_FIELD_PHI, stg))) return rc;
  CK(cudaEventRecord(c->ev_out[q], c->stream));
  CK(cudaStreamWaitEvent(c->s_d2h, c->ev_out[q], 0));
  CK(cudaMemcpyAsync(out, stg, n * sizeof(double), cudaMemcpyDeviceToHost, c->s_d2h));
  CK(cudaEventRecord(c->ev_d2h[q], c->s_d2h));
  c->d2h_used[q] = true;
  return MG_OK;
}

int mg_wait(mg_ctx *c, double *res_norm_out) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  int rc = sync(c);
  if (rc) return rc;
  if (c->s_d2h) CK(cudaStreamSynchronize(c->s_d2h));
  if (c->s_h2d) CK(cudaStreamSynchronize(c->s_h2d));
  const double r = sqrt(*c->h_norm);
  if (res_norm_out) *res_norm_out = r;
  if (!(r == r)) return fail(MG_ERR_DIVERGED, "residual is NaN");
  return MG_OK;
}

static int vcycle(mg_ctx *c, double *res_norm_out, bool allow_la) {
  int rc;
  if ((rc = enqueue_cycle(c, allow_la))) return rc;
  if ((rc = sync(c))) return rc;
  const double r = sqrt(*c->h_norm);
  if (res_norm_out) *res_norm_out = r;
  const double prev = c->prev_norm;
  c->prev_norm = r;
  if (!(r == r) || (prev >= 0.0 && r > 10.0 * prev))
    return fail(MG_ERR_DIVERGED, "residual %g after %g", r, prev);
  return MG_OK;
}

int mg_vcycle(mg_ctx *c, double *res_norm_out) {
  Nvtx nv("mg_vcycle");
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  return vcycle(c, res_norm_out, true);
}

int mg_residual_norm(mg_ctx *c, double *out) {
  Nvtx nv("mg_residual_norm");
  if (!c || !out) return fail(MG_ERR_ARG, "null pointer");
  return residual_norm_now(c, out);
}

int mg_solve_n(mg_ctx *c, double tol, int max_cycles, int *cycles_out, double *hist) {
  Nvtx nv("mg_solve");
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  const int kmax = max_cycles > 0 ? max_cycles : c->o.max_cycles;
  double r0;
  int rc = residual_norm_now(c, &r0);
  if (rc) return rc;
  if (hist) hist[0] = r0;
  c->prev_norm = r0;
  int k = 0;
  int status = r0 == 0.0 ? MG_OK : MG_ERR_NOTCONV;
  while (status == MG_ERR_NOTCONV && k < kmax) {
    double rk;
    rc = mg_vcycle(c, &rk);
    k++;
    if (hist) hist[k] = rk;
    if (rc) {
      status = rc;
      break;
    }
    if (rk <= tol * r0) status = MG_OK;
  }
  if (cycles_out) *cycles_out = k;
  if (status == MG_ERR_NOTCONV)
    fail(MG_ERR_NOTCONV, "not converged after %d cycles", k);
  return status;
}

int mg_solve(mg_ctx *c, double tol, int *cycles_out, double *hist) {
  return mg_solve_n(c, tol, 0, cycles_out, hist);
}

int mg_get_solution(mg_ctx *c, double *out, int where) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  return field_io(c, 0, MG_FIELD_PHI, out, where, false);
}

int mg_set_solution(mg_ctx *c, const double *in, int where) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  la_drop(c);
  c->prev_norm = -1.0;
  return field_io(c, 0, MG_FIELD_PHI, const_cast<double *>(in), where, true);
}

int mg_zero_solution(mg_ctx *c) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  la_drop(c);
  for (const Grid &g : c->g[0]) {
    CK(cudaMemsetAsync(g.phiR, 0, sizeof(double) * mg::grid_elems(g), c->stream));
    CK(cudaMemsetAsync(g.phiB, 0, sizeof(double) * mg::grid_elems(g), c->stream));
  }
  c->prev_norm = -1.0;
  return sync(c);
}

int mg_get_field(mg_ctx *c, int level, int field, double *out, int where) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  return field_io(c, level, field, out, where, false);
}

int mg_set_field(mg_ctx *c, int level, int field, const double *in, int where) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  la_drop(c);
  return field_io(c, level, field, const_cast<double *>(in), where, true);
}

int mg_smooth_half(mg_ctx *c, int level, int color, int from_zero) {
  if (!c || level < 0 || level >= c->pl.L || (color != 0 && color != 1))
    return fail(MG_ERR_ARG, "bad arguments");
  la_drop(c);
  int rc = smooth_half(c, level, color, from_zero);
  if (rc) return rc;
  return sync(c);
}

int mg_residual_restrict(mg_ctx *c, int level) {
  if (!c || level < 0 || level >= c->pl.L - 1) return fail(MG_ERR_ARG, "bad level");
  la_drop(c);
  int rc = restrict_level(c, level);
  if (rc) return rc;
  return sync(c);
}

int mg_prolong_correct(mg_ctx *c, int level) {
  if (!c || level < 0 || level >= c->pl.L - 1) return fail(MG_ERR_ARG, "bad level");
  la_drop(c);
  int rc = prolong_level(c, level);
  if (rc) return rc;
  return sync(c);
}

int mg_coarse_solve(mg_ctx *c, int *iters) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  la_drop(c);
  int rc = coarse_solve(c);
  if (rc) return rc;
  if (iters) CK(cudaMemcpyAsync(c->h_norm + 1, c->cg_iters, sizeof(int),
                                cudaMemcpyDeviceToHost, c->stream));
  if ((rc = sync(c))) return rc;
  if (iters) memcpy(iters, c->h_norm + 1, sizeof(int));
  return MG_OK;
}

}  // extern "C"

namespace {

// (Re)build the variable-coefficient representation from the solid mask and
// the face-cell BCs: level-0 float records (mask + patch types), Galerkin
// coarse records level by level, and byte codes on every level whose records
// all have kappa in {0,1} and position-derived delta.
int rebuild_coefficients_(mg_ctx *c);
int rebuild_coefficients(mg_ctx *c) {
  const int rc = rebuild_coefficients_(c);
  sync_alt_view(c);
  return rc;
}
int rebuild_coefficients_(mg_ctx *c) {
  CK(cudaStreamSynchronize(c->stream));
  drop_graphs(c);
  free_mask(c);
  c->fbc = mg::FaceBC{};
  c->dsolid = nullptr;
  if (c->solid_h.empty() && !c->patched && c->eps_h.empty()) return MG_OK;
  const bool need_var = !c->solid_h.empty() || !c->types_uniform || !c->eps_h.empty();
  unsigned char *dmask = nullptr;
  if (!c->solid_h.empty()) {
    CK(cudaMalloc(&dmask, c->solid_h.size()));
    c->mask_bufs.push_back(dmask);
    CK(cudaMemcpyAsync(dmask, c->solid_h.data(), c->solid_h.size(),
                       cudaMemcpyHostToDevice, c->stream));
    c->dsolid = dmask;
  }
  if (c->patched)
    for (int q = 0; q < 6; q++) {
      unsigned char *t = nullptr;
      double *v = nullptr;
      CK(cudaMalloc(&t, c->fty_h[q].size()));
      c->mask_bufs.push_back(t);
      CK(cudaMalloc(&v, c->fva_h[q].size() * sizeof(double)));
      c->mask_bufs.push_back(v);
      CK(cudaMemcpyAsync(t, c->fty_h[q].data(), c->fty_h[q].size(),
                         cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(v, c->fva_h[q].data(), c->fva_h[q].size() * sizeof(double),
                         cudaMemcpyHostToDevice, c->stream));
      c->fbc.ty[q] = t;
      c->fbc.va[q] = v;
    }
  if (!need_var) {  // only boundary values vary: box-domain operator, RHS only
    c->prev_norm = -1.0;
    return sync(c);
  }
  if (!c->eps_h.empty()) {
    // variable permittivity (N4): fp64 records on every level, level 0 from
    // eps, coarse levels by Galerkin R A P in the oracle's order
    double *deps = nullptr;
    CK(cudaMalloc(&deps, c->eps_h.size() * sizeof(double)));
    c->mask_bufs.push_back(deps);
    CK(cudaMemcpyAsync(deps, c->eps_h.data(), c->eps_h.size() * sizeof(double),
                       cudaMemcpyHostToDevice, c->stream));
    for (int l = 0; l < c->pl.L; l++)
      for (Grid &g : c->g[l]) {
        const size_t nb = (size_t)mg::grid_elems(g) * 8 * sizeof(double);
        double *r = nullptr, *b = nullptr;
        CK(cudaMalloc(&r, nb));
        c->mask_bufs.push_back(r);
        CK(cudaMalloc(&b, nb));
        c->mask_bufs.push_back(b);
        CK(cudaMemsetAsync(r, 0, nb, c->stream));
        CK(cudaMemsetAsync(b, 0, nb, c->stream));
        g.c64R = r;
        g.c64B = b;
        g.all_unknown = dmask == nullptr;
      }
    for (Grid &g : c->g[0])
      mg::launch_level0_coef64(g, dmask, deps, c->fbc, const_cast<double *>(g.c64R),
                               const_cast<double *>(g.c64B), c->stream);
    for (int l = 1; l < c->pl.L; l++) {
      for (int s = 0; s < (int)c->g[l - 1].size(); s++) {
        const Grid &cg = coarse_of(c, l - 1, s);
        mg::launch_coarse_coef64(c->g[l - 1][s], cg, const_cast<double *>(cg.c64R),
                                 const_cast<double *>(cg.c64B), c->stream);
      }
      if (l == c->pl.nd && c->P > 1) {  // records: 8 doubles per element
        int rc = gather_portions(c, l, 2, 8 * sizeof(double), [](const Grid &g, int a) {
          return (void *)(a ? g.c64B : g.c64R);
        });
        if (rc) return rc;
      }
    }
    CK(cudaGetLastError());
    c->masked = true;
    for (const Grid &g : c->g[0]) mg::launch_zero_solid(g, c->stream);
    c->prev_norm = -1.0;
    return sync(c);
  }
  // float records on every level
  for (int l = 0; l < c->pl.L; l++)
    for (Grid &g : c->g[l]) {
      const size_t ne = (size_t)mg::grid_elems(g);
      float *r = nullptr, *b = nullptr;
      CK(cudaMalloc(&r, ne * 8 * sizeof(float)));
      c->mask_bufs.push_back(r);
      CK(cudaMalloc(&b, ne * 8 * sizeof(float)));
      c->mask_bufs.push_back(b);
      CK(cudaMemsetAsync(r, 0, ne * 8 * sizeof(float), c->stream));
      CK(cudaMemsetAsync(b, 0, ne * 8 * sizeof(float), c->stream));
      g.coefR = r;
      g.coefB = b;
    }
  for (Grid &g : c->g[0])
    mg::launch_level0_coef(g, dmask, c->fbc, const_cast<float *>(g.coefR),
                           const_cast<float *>(g.coefB), c->stream);
  int *dfail = nullptr;
  CK(cudaMalloc(&dfail, sizeof(int)));
  c->mask_bufs.push_back(dfail);
  for (int l = 0; l < c->pl.L; l++) {
    if (l > 0) {
      for (int s = 0; s < (int)c->g[l - 1].size(); s++) {
        const Grid &cg = coarse_of(c, l - 1, s);
        mg::launch_coarse_coef(c->g[l - 1][s], cg, const_cast<float *>(cg.coefR),
                               const_cast<float *>(cg.coefB), c->stream);
      }
      if (l == c->pl.nd && c->P > 1) {  // records: 8 floats per element
        int rc = gather_portions(c, l, 2, 8 * sizeof(float), [](const Grid &g, int a) {
          return (void *)(a ? g.coefB : g.coefR);
        });
        if (rc) return rc;
      }
    }
    // level l aligned (every kappa 0 or 1, delta from the position)?  codes
    CK(cudaMemsetAsync(dfail, 0, sizeof(int), c->stream));
    std::vector<std::pair<unsigned char *, unsigned char *>> codes;
    for (Grid &g : c->g[l]) {
      const size_t ne = (size_t)mg::grid_elems(g);
      unsigned char *r = nullptr, *b = nullptr;
      CK(cudaMalloc(&r, ne));
      c->mask_bufs.push_back(r);
      CK(cudaMalloc(&b, ne));
      c->mask_bufs.push_back(b);
      CK(cudaMemsetAsync(r, 0, ne, c->stream));
      CK(cudaMemsetAsync(b, 0, ne, c->stream));
      mg::launch_coef_to_code(g, r, b, dfail, c->stream);
      codes.push_back({r, b});
      g.ukR = r;  // (bit 6 = D != 0 whether or not the codes are exact)
      g.ukB = b;
    }
    int hfail = 1;
    CK(cudaMemcpyAsync(&hfail, dfail, sizeof(int), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (!hfail && !(c->o.disable & MG_OFF_MASK_CODES))
      for (size_t s = 0; s < c->g[l].size(); s++) {
        Grid &g = c->g[l][s];
        g.codeR = codes[s].first;
        g.codeB = codes[s].second;
        g.coefR = g.coefB = nullptr;
      }
  }
  CK(cudaGetLastError());
  c->masked = true;
  for (const Grid &g : c->g[0]) mg::launch_zero_solid(g, c->stream);
  c->prev_norm = -1.0;
  return sync(c);
}

}  // namespace

extern "C" {

int mg_set_mask(mg_ctx *c, const uint8_t *solid, int where) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  la_drop(c);
  if (solid && any_periodic(c))
    return fail(MG_ERR_BC, "a solid mask on a domain with periodic faces is "
                           "not supported");
  const size_t N = (size_t)c->pl.dims[0][0] * c->pl.dims[0][1] * c->pl.dims[0][2];
  if (!solid) {
    c->solid_h.clear();
  } else {
    c->solid_h.resize(N);
    if (where == MG_DEVICE)
      CK(cudaMemcpy(c->solid_h.data(), solid, N, cudaMemcpyDeviceToHost));
    else
      memcpy(c->solid_h.data(), solid, N);
  }
  return rebuild_coefficients(c);
}

static void init_face_arrays(mg_ctx *c);

int mg_set_permittivity(mg_ctx *c, const double *eps, int where) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  la_drop(c);
  const size_t N = (size_t)c->pl.dims[0][0] * c->pl.dims[0][1] * c->pl.dims[0][2];
  if (!eps) {
    c->eps_h.clear();
    return rebuild_coefficients(c);
  }
  if (any_periodic(c))
    return fail(MG_ERR_BC, "a variable permittivity on a domain with periodic "
                           "faces is not supported");
  std::vector<double> e(N);
  if (where == MG_DEVICE)
    CK(cudaMemcpy(e.data(), eps, N * sizeof(double), cudaMemcpyDeviceToHost));
  else if (where == MG_HOST)
    memcpy(e.data(), eps, N * sizeof(double));
  else
    return fail(MG_ERR_ARG, "bad 'where' %d", where);
  for (size_t k = 0; k < N; k++)
    if (!(e[k] > 0.0)) return fail(MG_ERR_ARG, "eps[%zu] = %g is not > 0", k, e[k]);
  c->eps_h.swap(e);
  init_face_arrays(c);  // the eps-weighted RHS adaptation runs per face cell
  return rebuild_coefficients(c);
}

static void init_face_arrays(mg_ctx *c) {
  if (c->patched) return;
  const int ext[3] = {c->pl.dims[0][0], c->pl.dims[0][1], c->pl.dims[0][2]};
  for (int q = 0; q < 6; q++) {
    const int aq = q / 2;
    const size_t n = (size_t)ext[aq == 0 ? 1 : 0] * ext[aq == 2 ? 1 : 2];
    c->fty_h[q].assign(n, (uint8_t)c->bc[q].type);
    c->fva_h[q].assign(n, c->bc[q].value);
  }
  c->patched = true;
}

int mg_set_bc_patch(mg_ctx *c, int face, int a0, int a1, int b0, int b1,
                    int type, double value) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  la_drop(c);
  if (face < 0 || face > 5) return fail(MG_ERR_ARG, "bad face %d", face);
  if (type != MG_DIRICHLET && type != MG_NEUMANN)
    return fail(MG_ERR_BC, "patch type must be Dirichlet or Neumann");
  if (any_periodic(c))
    return fail(MG_ERR_BC, "boundary patches on a domain with periodic faces "
                           "are not supported");
  const int ext[3] = {c->pl.dims[0][0], c->pl.dims[0][1], c->pl.dims[0][2]};
  const int ax = face / 2;
  const int na = ext[ax == 0 ? 1 : 0], nb = ext[ax == 2 ? 1 : 2];
  if (a0 < 0 || b0 < 0 || a1 > na || b1 > nb || a0 > a1 || b0 > b1)
    return fail(MG_ERR_ARG, "patch [%d,%d)x[%d,%d) outside face %d (%dx%d)", a0,
                a1, b0, b1, face, na, nb);
  init_face_arrays(c);
  for (int x = a0; x < a1; x++)
    for (int y = b0; y < b1; y++) {
      c->fty_h[face][(size_t)x * nb + y] = (uint8_t)type;
      c->fva_h[face][(size_t)x * nb + y] = value;
    }
  c->types_uniform = true;
  for (int q = 0; q < 6; q++)
    for (uint8_t t : c->fty_h[q])
      if (t != (uint8_t)c->bc[q].type) c->types_uniform = false;
  return rebuild_coefficients(c);
}

int mg_set_face_values(mg_ctx *c, int face, const double *values) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  la_drop(c);
  if (face < 0 || face > 5 || !values) return fail(MG_ERR_ARG, "bad arguments");
  if (c->bc[face].type == MG_PERIODIC)
    return fail(MG_ERR_BC, "face %d is periodic: it has no boundary values", face);
  init_face_arrays(c);
  memcpy(c->fva_h[face].data(), values, c->fva_h[face].size() * sizeof(double));
  return rebuild_coefficients(c);
}

static int coulomb_forces(mg_ctx *c, int n, const double *centers,
                          const double *radii, const double *charges,
                          int normalization, int subsample, double *forces_out,
                          const unsigned long long *counts,
                          const double *dsph_given = nullptr);

int mg_coulomb_forces(mg_ctx *c, int n, const double *centers,
                      const double *radii, const double *charges,
                      int normalization, int subsample, double *forces_out) {
  Nvtx nv("mg_coulomb_forces");
  return coulomb_forces(c, n, centers, radii, charges, normalization, subsample,
                        forces_out, nullptr);
}

// counts: the per-sphere covered sub-cell counts on the device if the RHS of
// the same spheres was just set with the same subsampling (mg_timestep)
static int coulomb_forces(mg_ctx *c, int n, const double *centers,
                          const double *radii, const double *charges,
                          int normalization, int subsample, double *forces_out,
                          const unsigned long long *counts,
                          const double *dsph_given) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  if (n < 0 || (n > 0 && (!centers || !radii || !charges || !forces_out)))
    return fail(MG_ERR_ARG, "bad arrays");
  if (subsample < 1 || subsample > 16)
    return fail(MG_ERR_ARG, "subsample must be in 1..16");
  if (normalization != MG_CHARGE_PER_CELLS && normalization != MG_CHARGE_PER_VOLUME)
    return fail(MG_ERR_ARG, "bad normalization");
  if (n == 0) return MG_OK;
  std::vector<double> h5;
  if (!dsph_given) {  // (a given device list was checked when it was uploaded)
    h5.resize(5 * (size_t)n);
    for (int p = 0; p < n; p++) {
      if (int rc = check_sphere(c, p, centers + 3 * (size_t)p, radii[p])) return rc;
      for (int q = 0; q < 3; q++) h5[5 * (size_t)p + q] = centers[3 * (size_t)p + q];
      h5[5 * (size_t)p + 3] = radii[p];
      h5[5 * (size_t)p + 4] = charges[p];
    }
  }
  int rc;
  // both colours' ghost planes current (the gradient reads across slabs)
  if ((rc = halo(c, 0, 0)) || (rc = halo(c, 0, 1))) return rc;
  const size_t ns = c->g[0].size();
  const size_t nrow = 3 * (size_t)n;
  // device: sphere list + per-slab partials (+ all-gathered partials)
  const size_t nb = 5 * (size_t)n + nrow * (ns + (size_t)c->P);
  if (nb > c->fbuf_cap) {
    CK(cudaStreamSynchronize(c->stream));
    if (c->fbuf) cudaFree(c->fbuf);
    c->fbuf = nullptr;
    c->fbuf_cap = 0;
    CK(cudaMalloc(&c->fbuf, nb * sizeof(double)));
    c->fbuf_cap = nb;
  }
  double *buf = c->fbuf;
  double *dsph = buf, *dpart = buf + 5 * (size_t)n, *dall = dpart + nrow * ns;
  if (dsph_given) {
    dsph = const_cast<double *>(dsph_given);
  } else if (cudaMemcpyAsync(dsph, h5.data(), 5 * (size_t)n * sizeof(double),
                             cudaMemcpyHostToDevice, c->stream) != cudaSuccess) {
    return fail(MG_ERR_CUDA, "copy of the sphere list failed");
  }
  for (size_t s = 0; s < ns; s++)
    mg::launch_coulomb(c->g[0][s], c->dsolid, c->h, subsample, n, dsph,
                       normalization, dpart + nrow * s, counts, c->stream);
  size_t nparts = ns;
  double *src = dpart;
  if (c->P > 1 && c->backend == MG_HALO_NCCL) {
    rc = nccl_ck(g_nccl.AllGather(dpart, dall, nrow, ncclDouble, c->comm, c->stream),
                 "ncclAllGather(forces)");
    nparts = (size_t)c->P;
    src = dall;
  }
  double *hq = nullptr;
  if (!rc) {
    hq = host_pinned(c, nrow * nparts);
    if (!hq || cudaMemcpyAsync(hq, src, nrow * nparts * sizeof(double),
                               cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess)
      rc = fail(MG_ERR_CUDA, "force readback failed");
  }
  if (rc) return rc;
  const double h3 = c->h * c->h * c->h;
  for (size_t r = 0; r < nrow; r++) {
    double s = 0.0;
    for (size_t k = 0; k < nparts; k++) s = s + hq[k * nrow + r];  // slab order
    forces_out[r] = -h3 * s;
  }
  return MG_OK;
}

int mg_timestep(mg_ctx *c, int n, const double *centers, const double *radii,
                const double *charges, int normalization, int subsample,
                int cycles, double abs_tol, double *forces_out,
                int force_subsample, int *cycles_out, double *res_out) {
  Nvtx nv("mg_timestep");
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  if (cycles < 0) return fail(MG_ERR_ARG, "cycles < 0");
  if (cycles == 0 && !(abs_tol > 0.0))
    return fail(MG_ERR_ARG, "cycles == 0 needs abs_tol > 0");
  int k = 0;
  double r = -1.0;
  int rc;
  if (cycles > 0) {
    // The RHS, the cycles and the forces are enqueued back to back; the host
    // waits once, at the end (the forces' readback or a final sync), and
    // then checks the empty-sphere flag and the last cycle's norm.  Earlier
    // cycles of a multi-cycle step keep their per-cycle check.  One cycle
    // per new RHS takes the plain form: the look-ahead sweep would be
    // discarded by the next step's RHS (4 B/cell more than the norm pass).
    bool check;
    if ((rc = rhs_from_spheres(c, n, centers, radii, charges, normalization, subsample,
                               &check)))
      return rc;
    for (; k < cycles - 1; k++)
      if ((rc = vcycle(c, &r, true))) break;
    if (rc) {
      if (cycles_out) *cycles_out = k;
      if (res_out) *res_out = r;
      sync(c);
      if (int e = empty_sphere_check(c, check)) return e;
      return rc;
    }
    const double prev = c->prev_norm;
    if ((rc = enqueue_cycle(c, cycles > 1))) return rc;
    k++;
    if (forces_out) {
      const unsigned long long *cnt =
          (force_subsample == subsample && n > 0)
              ? reinterpret_cast<const unsigned long long *>(c->sph + 5 * c->sph_cap)
              : nullptr;
      rc = coulomb_forces(c, n, centers, radii, charges, normalization, force_subsample,
                          forces_out, cnt, n > 0 ? c->sph : nullptr);  // (syncs)
    } else {
      rc = sync(c);
    }
    if (int e = empty_sphere_check(c, check)) return e;
    if (rc) return rc;
    r = sqrt(*c->h_norm);
    c->prev_norm = r;
    if (cycles_out) *cycles_out = k;
    if (res_out) *res_out = r;
    if (!(r == r) || (prev >= 0.0 && r > 10.0 * prev))
      return fail(MG_ERR_DIVERGED, "residual %g after %g", r, prev);
    return MG_OK;
  }
  if ((rc = mg_set_rhs_from_spheres(c, n, centers, radii, charges, normalization,
                                    subsample)))
    return rc;
  {  // Alg.1: while residual >= tol, perform a V-cycle
    if ((rc = residual_norm_now(c, &r))) return rc;
    c->prev_norm = r;
    while (r > abs_tol && k < c->o.max_cycles) {
      k++;
      if ((rc = mg_vcycle(c, &r))) break;
    }
    if (!rc && r > abs_tol)
      rc = fail(MG_ERR_NOTCONV, "residual %g > %g after %d cycles", r, abs_tol, k);
  }
  if (cycles_out) *cycles_out = k;
  if (res_out) *res_out = r;
  if (rc && rc != MG_ERR_NOTCONV) return rc;
  if (forces_out) {
    // the RHS kernel counted the spheres' covered sub-cells already
    const unsigned long long *cnt =
        (force_subsample == subsample && n > 0)
            ? reinterpret_cast<const unsigned long long *>(c->sph + 5 * c->sph_cap)
            : nullptr;
    // ... and the same sphere list is already on the device (c->sph)
    const int frc = coulomb_forces(c, n, centers, radii, charges, normalization,
                                   force_subsample, forces_out, cnt,
                                   n > 0 ? c->sph : nullptr);
    if (frc) return frc;
  }
  return rc;
}

int mg_get_stencil(mg_ctx *c, int l, double *out, int where) {
  if (!c || !out || l < 0 || l >= c->pl.L) return fail(MG_ERR_ARG, "bad arguments");
  const size_t n = level_cells_held(c, l);
  double *dev = out;
  int rc;
  if (where == MG_HOST) {
    if ((rc = stage_for(c, 7 * n * sizeof(double)))) return rc;
    dev = c->stage;
  }
  size_t off = 0;
  for (size_t s = 0; s < io_grids(c, l); s++) {
    const Grid &g = c->g[l][s];
    mg::launch_get_stencil(g, dev + 7 * off, c->stream);
    off += (size_t)g.nxl * g.ny * g.nz;
  }
  CK(cudaGetLastError());
  if (where == MG_HOST)
    CK(cudaMemcpyAsync(out, dev, 7 * n * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream));
  return sync(c);
}

int mg_set_profiling(mg_ctx *c, int on) {
  if (!c) return fail(MG_ERR_ARG, "null ctx");
  if (on && c->ev.empty()) {
    c->ev.resize(kMaxMarks);
    c->mark_cat.assign(kMaxMarks, CAT_NONE);
    for (auto &e : c->ev) CK(cudaEventCreate(&e));
  }
  if ((on != 0) != c->prof) drop_graphs(c);
  c->prof = on != 0;
  return MG_OK;
}

// per-category sums of the last profiled cycle's intervals (ms), and the
// number of level-0 half-sweep intervals
static int cycle_cats(mg_ctx *c, double cat_ms[kNumCat], int *nsmooth, double *total) {
  if (!c->prof_last || c->nev < 2) return fail(MG_ERR_ARG, "profiling was off");
  for (int q = 0; q < kNumCat; q++) cat_ms[q] = 0.0;
  *nsmooth = 0;
  for (int i = 1; i < c->nev; i++) {
    const int cat = c->mark_cat[i];
    if (cat == CAT_NONE) continue;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev[i - 1], c->ev[i]));
    cat_ms[cat] += ms;
    if (cat == CAT_SMOOTH0) (*nsmooth)++;
  }
  float tot = 0.f;
  CK(cudaEventElapsedTime(&tot, c->ev[0], c->ev[c->nev - 1]));
  *total = tot;
  return MG_OK;
}

int mg_last_cycle_times(mg_ctx *c, double out[8]) {
  if (!c || !out) return fail(MG_ERR_ARG, "null pointer");
  double cat[kNumCat], tot;
  int ns;
  int rc = cycle_cats(c, cat, &ns, &tot);
  if (rc) return rc;
  out[0] = cat[CAT_SMOOTH0];
  out[1] = ns;
  out[2] = cat[CAT_RESTRICT0];
  out[3] = cat[CAT_PROLONG0];
  out[4] = cat[CAT_NORM];
  out[5] = cat[CAT_COARSE] + cat[CAT_AGG] + cat[CAT_CG];  // levels >= 1 incl. CG
  out[6] = tot;
  out[7] = c->cycle_launches;
  return MG_OK;
}

int mg_last_cycle_times_ex(mg_ctx *c, double *out, int n) {
  if (!c || !out || n < 10) return fail(MG_ERR_ARG, "need 10 outputs");
  int rc = mg_last_cycle_times(c, out);
  if (rc) return rc;
  out[8] = out[1];  // level-0 smoothing launches
  out[9] = out[1];  // half-sweeps they perform (one per launch)
  if (n >= 12) {
    double cat[kNumCat], tot;
    int ns;
    if ((rc = cycle_cats(c, cat, &ns, &tot))) return rc;
    out[10] = cat[CAT_AGG] + cat[CAT_CG];  // levels >= 1 held whole, incl. CG
    out[11] = cat[CAT_CG];                 // the coarsest-grid solve
  }
  return MG_OK;
}

int mg_cycle_launches(const mg_ctx *c) { return c ? c->cycle_launches : MG_ERR_ARG; }

int mg_cycle_paths(const mg_ctx *c) { return c ? c->paths : MG_ERR_ARG; }

void *mg_stream(const mg_ctx *c) { return c ? (void *)c->stream : nullptr; }

}  // extern "C"
