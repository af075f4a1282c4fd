// One full RBGS sweep (red half-sweep, then black) in one
// plane-marching kernel for sm_100a -- the two-stage form of temporal
// blocking.
//
// A CTA owns TY rows x ZT half-entries of a chunk of x-planes.  Black plane t
// (input B0) streams into a TMA ring; red is computed on plane t-1 over the
// tile grown by one row and two half-entries on each side (what the black
// update needs), kept in a three-plane shared-memory ring, and black is
// computed on plane t-2 from it.  Per fine cell the sweep reads Phi^B, f^R,
// f^B and writes Phi^R, Phi^B once: 20 bytes instead of 2 x 12 for two
// half-sweep kernels.  The red halo rows / half-entries are the only
// recomputation (10/8 rows, 132/128 half-entries).
//
// Per-cell arithmetic is exactly that of k_smooth_march (bitwise):
//     Phi_c = (f_c * w + s) / d,  s = ((((x- + x+) + y-) + y+) + z-) + z+.
// The final black goes to a second black array (the input black is still
// read by neighbouring CTAs through their halos); the host alternates the
// two arrays between passes.  PROLONG: the prolongation + magnified
// correction of black is applied to each input plane as it
// arrives, as in k_smooth_march<true> (red is overwritten unread).
// FROMZERO: the input black is 0 (first pre-smoothing sweep of a coarse
// level).  Box domains, levels held whole, no periodic axis, no mask.
#include <cuda.h>
#include <cstdlib>
#include <cuda_runtime.h>

#include "mg_internal.h"
#include "mg_tma.cuh"

namespace mg {

namespace {

constexpr int kTY2 = 16;           // core rows per tile
constexpr int kZT2 = 64;           // core half-entries per tile
constexpr int kW0 = kZT2 + 8;      // input tile width: half-entries kz0-4 ..
constexpr int kWR = kZT2 + 4;      // red tile width:   half-entries kz0-2 ..
constexpr int kR0 = kTY2 + 4;      // input rows j0-2 .. j0+TY+1
constexpr int kRR = kTY2 + 2;      // red rows   j0-1 .. j0+TY
constexpr int kS2 = 6;             // input ring: 3 in use + 3 in flight
constexpr int kAhead = kS2 - 3;    // TMA issue distance (planes)
constexpr int kSlot0 = kR0 * kW0;  // doubles per input slot
constexpr int kSlotR = kRR * kWR;  // doubles per red slot
constexpr int kPairsR = kWR / 2;   // red pairs per row (34)
constexpr int kRT = (kRR * kPairsR + kThreadsM - 1) / kThreadsM;  // 3
constexpr int kBT = kTY2 * (kZT2 / 2) / kThreadsM;                // 2
static_assert(kZT2 / 2 == 32, "one black pair per lane per row");

__host__ __device__ constexpr size_t sweep2_smem() {
  return (size_t)(kS2 * kSlot0 + 3 * kSlotR) * 8 + kS2 * 8;
}

// diagonal 6 + sum of the face terms of the y and z faces a cell touches, for
// the two cells (z0 = 2k + p, z0 + 2) of a pair and both parities p, as four
// 4-bit fields [p][e] (values 3..9); the x term is added per plane
__device__ __forceinline__ unsigned pack_dyz(const Grid &g, int j, int k) {
  const int dy = (j == 0 ? g.dface[2] : 0) + (j == g.ny - 1 ? g.dface[3] : 0);
  unsigned r = 0;
#pragma unroll
  for (int p = 0; p < 2; p++)
#pragma unroll
    for (int e = 0; e < 2; e++) {
      const int z = 2 * k + p + 2 * e;
      const int d = 6 + dy + (z == 0 ? g.dface[4] : 0) + (z == g.nz - 1 ? g.dface[5] : 0);
      r |= (unsigned)d << (4 * (2 * p + e));
    }
  return r;
}

// RN(a / d) (bitwise IEEE) with the shared reciprocal table; branch-free so
// that the independent tasks of a thread interleave
__device__ __forceinline__ double div_cell(double a, int d, const double *rcp) {
  return div_small(a, (double)d, rcp[d]);
}

}  // namespace

template <bool PROLONG, bool FROMZERO>
__global__ void __launch_bounds__(kThreadsM, 2)
    k_sweep2(Grid g, const __grid_constant__ CUtensorMap tmB, double *bout,
             Grid C, double alpha, int ich) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *ring0 = reinterpret_cast<double *>(smem);
  double *ringR = ring0 + (size_t)kS2 * kSlot0;
  unsigned long long *bars =
      reinterpret_cast<unsigned long long *>(ringR + (size_t)3 * kSlotR);
  __shared__ double rcp[16];

  const int nzt = (g.nzh + kZT2 - 1) / kZT2;
  const int nrt = (g.ny + kTY2 - 1) / kTY2;
  int b = blockIdx.x;
  const int zt = b % nzt;
  b /= nzt;
  const int rt = b % nrt;
  const int xc = b / nrt;
  const int kz0 = zt * kZT2, j0 = rt * kTY2;
  const int i0 = xc * ich;
  const int i1 = min(i0 + ich, g.nxl);
  const int tfirst = i0 - 2, tlast = i1 + 1;  // input planes
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned box_bytes = (unsigned)(kSlot0 * 8);

  fill_rcp16(rcp);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kS2; s++) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (FROMZERO)
    for (int e = threadIdx.x; e < kS2 * kSlot0; e += kThreadsM) ring0[e] = 0.0;
  __syncthreads();
  auto issue = [&](int t) {
    const int s = (t - tfirst) % kS2;
    mbar_expect_tx(&bars[s], box_bytes);
    tma_load_3d(ring0 + (size_t)s * kSlot0, &tmB, kz0 - 4, j0 - 2 + 1, t + 1, &bars[s]);
  };
  if (!FROMZERO && threadIdx.x == 0)
    for (int t = tfirst; t <= min(tfirst + kAhead, tlast); t++) issue(t);

  const int ny = g.ny, nzh = g.nzh;
  const long long plane = g.plane;
  const double w = g.w;

  // ---- red tasks: the kRR x kPairsR pairs of the red tile; task e = thread +
  // 256 m (row e / 34, pair e % 34).  Per task, fixed over the march: tile
  // offsets, the in-plane memory offset, validity, core-ness, the y/z diagonal
  int r_in[kRT], r_out[kRT], r_off[kRT], r_j[kRT];
  unsigned r_d[kRT];
  bool r_ok[kRT], r_core[kRT], r_pair[kRT];
#pragma unroll
  for (int m = 0; m < kRT; m++) {
    const int e = threadIdx.x + kThreadsM * m;
    const int rr = e / kPairsR, cr = 2 * (e % kPairsR);
    const int j = j0 - 1 + rr, k = kz0 - 2 + cr;
    r_ok[m] = e < kRR * kPairsR && j >= 0 && j < ny && k >= 0 && k < nzh;
    r_core[m] = r_ok[m] && rr >= 1 && rr <= kTY2 && cr >= 2 && cr < 2 + kZT2;
    r_pair[m] = k + 1 < nzh;
    r_in[m] = e < kRR * kPairsR ? (rr + 1) * kW0 + cr + 2 : kW0 + 2;  // in-tile
    r_out[m] = e < kRR * kPairsR ? rr * kWR + cr : -1;
    r_off[m] = (j + 1) * g.pz + k;
    r_j[m] = j;
    r_d[m] = r_ok[m] ? pack_dyz(g, j, k) : 0u;
  }
  // ---- black tasks: row warp + 8 m, pair lane (the core of the tile)
  int b_out[kBT], b_off[kBT], b_j[kBT];
  unsigned b_d[kBT];
  bool b_ok[kBT], b_pair[kBT];
  const int kb = kz0 + 2 * lane;
#pragma unroll
  for (int m = 0; m < kBT; m++) {
    const int rr = warp + 8 * m + 1;  // red-tile row of the black row
    const int j = j0 + warp + 8 * m;
    b_ok[m] = j < ny && kb < nzh;
    b_pair[m] = kb + 1 < nzh;
    b_out[m] = rr * kWR + 2 * lane + 2;
    b_off[m] = (j + 1) * g.pz + kb;
    b_j[m] = j;
    b_d[m] = b_ok[m] ? pack_dyz(g, j, kb) : 0u;
  }

  auto load_fr = [&](int i, double2 *fr) {
    const bool pin = i >= 0 && i < g.nxl;
    const double *base = g.fR + (long long)(i + 1) * plane;
#pragma unroll
    for (int m = 0; m < kRT; m++)
      fr[m] = (pin && r_ok[m]) ? *reinterpret_cast<const double2 *>(base + r_off[m])
                               : make_double2(0.0, 0.0);
  };
  auto load_fb = [&](int i, double2 *fb) {
    const bool pin = i >= i0 && i < i1;
    const double *base = g.fB + (long long)(i + 1) * plane;
#pragma unroll
    for (int m = 0; m < kBT; m++)
      fb[m] = (pin && b_ok[m]) ? *reinterpret_cast<const double2 *>(base + b_off[m])
                               : make_double2(0.0, 0.0);
  };

  // PROLONG: black input plane i += alpha * e(parent), in-level cells only;
  // tasks = (row rb, pair pc) of the kR0 x kW0/2 input tile, e loaded a step ahead
  constexpr int kPT = (kR0 * (kW0 / 2) + kThreadsM - 1) / kThreadsM;
  auto load_e = [&](int i, double2 *E) {
    const int I = (g.x0 + i) >> 1;
    const bool pin = i >= 0 && i < g.nxl;
    const double *cR = C.phiR + (long long)(I - C.x0 + 1) * C.plane;
    const double *cB = C.phiB + (long long)(I - C.x0 + 1) * C.plane;
#pragma unroll
    for (int m = 0; m < kPT; m++) {
      const int e = threadIdx.x + kThreadsM * m;
      const int rb = e / (kW0 / 2), pc = e % (kW0 / 2);
      const int j = j0 - 2 + rb, k = kz0 - 4 + 2 * pc;
      double2 v = make_double2(0.0, 0.0);
      if (pin && rb < kR0 && j >= 0 && j < ny && k >= 0 && k < nzh) {
        const int J = j >> 1;
        const long long o = (long long)(J + 1) * C.pz + (k >> 1);
        const int c0 = (I + J + k) & 1;  // colour of coarse z = k
        v.x = c0 ? cB[o] : cR[o];
        if (k + 1 < nzh) v.y = c0 ? cR[o] : cB[o];
      }
      E[m] = v;
    }
  };

  double2 fr[kRT], fb[kBT], E[PROLONG ? kPT : 1];
  load_fr(tfirst + 1, fr);  // red of step tfirst+2 is plane tfirst+1
  load_fb(i0, fb);          // black of step i0+2 is plane i0
  if (PROLONG) load_e(tfirst, E);
  int sR = 0;  // red ring slot of plane t-1 (slot(plane) = base + plane mod 3)

  for (int t = tfirst; t <= tlast; t++) {
    const int s0 = (t - tfirst) % kS2;
    // plane t+kAhead goes to the slot of plane t-3, free since step t-1 ended
    if (!FROMZERO && threadIdx.x == 0 && t > tfirst && t + kAhead <= tlast) {
      fence_proxy_async();
      issue(t + kAhead);
    }
    if (!FROMZERO) mbar_wait(&bars[s0], ((t - tfirst) / kS2) & 1);
    double *in_t = ring0 + (size_t)s0 * kSlot0;
    if (PROLONG) {
      double2 En[kPT];
      if (t + 1 <= tlast) load_e(t + 1, En);
#pragma unroll
      for (int m = 0; m < kPT; m++) {
        const int e = threadIdx.x + kThreadsM * m;
        if (e < kR0 * (kW0 / 2)) {
          double2 v = reinterpret_cast<double2 *>(in_t)[e];
          v.x = v.x + alpha * E[m].x;
          v.y = v.y + alpha * E[m].y;
          reinterpret_cast<double2 *>(in_t)[e] = v;
        }
        E[m] = En[m];
      }
      __syncthreads();
    }
    // ---- stage 1: red on plane t-1 (needs input planes t-2, t-1, t)
    const int ir = t - 1;
    if (t >= tfirst + 2) {
      double2 frn[kRT];
      load_fr(ir + 1, frn);
      const double *Im = ring0 + (size_t)((t - 2 - tfirst) % kS2) * kSlot0;
      const double *Ic = ring0 + (size_t)((t - 1 - tfirst) % kS2) * kSlot0;
      const double *Ip = in_t;
      double *Rout = ringR + (size_t)sR * kSlotR;
      const bool pin = ir >= 0 && ir < g.nxl;
      const bool core_plane = ir >= i0 && ir < i1;
      const int ii = g.x0 + ir;
      const int dx = (ii == 0 ? g.dface[0] : 0) + (ii == g.nx - 1 ? g.dface[1] : 0);
      double *outR = g.phiR + (long long)(ir + 1) * plane;
#pragma unroll
      for (int m = 0; m < kRT; m++) {
        const int p = (ii + r_j[m]) & 1;  // red: z = 2k + p
        const double *c = Ic + r_in[m];
        const double2 xm = lds2(Im + r_in[m]);
        const double2 xp = lds2(Ip + r_in[m]);
        const double2 ym = lds2(c - kW0);
        const double2 yp = lds2(c + kW0);
        const double2 zc = lds2(c);
        const double zx = c[p ? 2 : -1];
        const double zm0 = p ? zc.x : zx, zp0 = p ? zc.y : zc.x;
        const double zm1 = p ? zc.y : zc.x, zp1 = p ? zx : zc.y;
        const double s0 = ((((xm.x + xp.x) + ym.x) + yp.x) + zm0) + zp0;
        const double s1 = ((((xm.y + xp.y) + ym.y) + yp.y) + zm1) + zp1;
        const unsigned dd = r_d[m] >> (8 * p);
        const bool ok = pin && r_ok[m];
        double2 v;
        v.x = div_cell(fr[m].x * w + s0, ok ? (int)(dd & 15u) + dx : 6, rcp);
        v.y = div_cell(fr[m].y * w + s1, ok ? (int)((dd >> 4) & 15u) + dx : 6, rcp);
        if (!ok) v.x = 0.0;
        if (!ok || !r_pair[m]) v.y = 0.0;
        if (core_plane && r_core[m]) {
          if (r_pair[m])
            *reinterpret_cast<double2 *>(outR + r_off[m]) = v;
          else
            outR[r_off[m]] = v.x;
        }
        if (r_out[m] >= 0) *reinterpret_cast<double2 *>(Rout + r_out[m]) = v;
      }
#pragma unroll
      for (int m = 0; m < kRT; m++) fr[m] = frn[m];
    }
    __syncthreads();
    // ---- stage 2: black on plane t-2 (needs red planes t-3, t-2, t-1)
    const int ib = t - 2;
    if (ib >= i0 && ib < i1) {
      double2 fbn[kBT];
      load_fb(ib + 1, fbn);
      const double *Rm = ringR + (size_t)((sR + 1) % 3) * kSlotR;  // plane t-3
      const double *Rc = ringR + (size_t)((sR + 2) % 3) * kSlotR;  // plane t-2
      const double *Rp = ringR + (size_t)sR * kSlotR;              // plane t-1
      const int ii = g.x0 + ib;
      const int dx = (ii == 0 ? g.dface[0] : 0) + (ii == g.nx - 1 ? g.dface[1] : 0);
      double *outB = bout + (long long)(ib + 1) * plane;
#pragma unroll
      for (int m = 0; m < kBT; m++) {
        const int p = (ii + b_j[m] + 1) & 1;  // black: z = 2k + p
        const double *c = Rc + b_out[m];
        const double2 xm = lds2(Rm + b_out[m]);
        const double2 xp = lds2(Rp + b_out[m]);
        const double2 ym = lds2(c - kWR);
        const double2 yp = lds2(c + kWR);
        const double2 zc = lds2(c);
        const double zx = c[p ? 2 : -1];
        const double zm0 = p ? zc.x : zx, zp0 = p ? zc.y : zc.x;
        const double zm1 = p ? zc.y : zc.x, zp1 = p ? zx : zc.y;
        const double s0 = ((((xm.x + xp.x) + ym.x) + yp.x) + zm0) + zp0;
        const double s1 = ((((xm.y + xp.y) + ym.y) + yp.y) + zm1) + zp1;
        const unsigned dd = b_d[m] >> (8 * p);
        double2 v;
        v.x = div_cell(fb[m].x * w + s0, b_ok[m] ? (int)(dd & 15u) + dx : 6, rcp);
        v.y = div_cell(fb[m].y * w + s1, b_ok[m] ? (int)((dd >> 4) & 15u) + dx : 6, rcp);
        if (b_ok[m]) {
          if (b_pair[m])
            *reinterpret_cast<double2 *>(outB + b_off[m]) = v;
          else
            outB[b_off[m]] = v.x;
        }
      }
#pragma unroll
      for (int m = 0; m < kBT; m++) fb[m] = fbn[m];
    }
    __syncthreads();  // ring slots of this step are free for the next one
    sR = (sR + 1) % 3;
  }
}

// ---- host side ------------------------------------------------------------------
bool sweep2_supported(const Grid &g) {
  return g.nxl == g.nx && !is_periodic(g) && !g.codeR && !g.coefR && !g.c64R &&
         g.nx >= 2 && g.ny >= kTY2 && g.nzh >= kZT2;
}

bool make_tmap_sweep2(const Grid &g, const double *base, void *out128) {
  return encode_box(g, base, out128, kW0, kR0);
}

template <bool P, bool Z>
static void launch_s2(const Grid &g, const Grid &c, const CUtensorMap *tm,
                      double *bout, double alpha, cudaStream_t s) {
  const int nzt = (g.nzh + kZT2 - 1) / kZT2;
  const int nrt = (g.ny + kTY2 - 1) / kTY2;
  // x chunks: long (the chunk re-reads 4 input planes and recomputes 2 red
  // planes) but at least ~6 waves of 2 CTAs per SM
  int ich = 64;
  if (const char *e = getenv("MG_S2_ICH")) ich = atoi(e);
  while (ich > 4 && (long long)((g.nxl + ich - 1) / ich) * nrt * nzt < 148 * 2 * 6) ich >>= 1;
  const int nxc = (g.nxl + ich - 1) / ich;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_sweep2<P, Z>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sweep2_smem());
    configured = true;
  }
  k_sweep2<P, Z><<<nxc * nrt * nzt, kThreadsM, sweep2_smem(), s>>>(g, *tm, bout, c,
                                                                   alpha, ich);
}

void launch_sweep2(const Grid &g, const Grid &c, const void *tm_in128, double *bout,
                   bool prolong, bool from_zero, double alpha, cudaStream_t s) {
  const CUtensorMap *tm = reinterpret_cast<const CUtensorMap *>(tm_in128);
  if (prolong)
    launch_s2<true, false>(g, c, tm, bout, alpha, s);
  else if (from_zero)
    launch_s2<false, true>(g, c, tm, bout, alpha, s);
  else
    launch_s2<false, false>(g, c, tm, bout, alpha, s);
}

}  // namespace mg
