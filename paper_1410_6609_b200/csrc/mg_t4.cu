// Temporally blocked smoother for sm_100a: the four half-sweeps of a V(2,2)
// pre- or post-smoothing pass (red, black, red, black)
// in ONE plane-marching kernel.
//
// The split layout keeps each colour in its own array, so a half-sweep of
// colour c reads only the other colour and its own f.  Four half-sweeps in a
// row therefore form a wavefront along x: when black plane t (input B0) has
// arrived, red R1 can be computed on plane t-1, then black B1 on t-2, red R2
// on t-3 and black B2 on t-4.  A CTA owns a (TY rows x ZT half-entries) tile
// of a chunk of planes and keeps the intermediate planes of R1, B1, R2 in
// shared-memory rings; every stage is computed on a tile grown by one cell
// per remaining stage on each side (rows and half-indices), so the CTA needs
// no data of its neighbours' intermediate stages.  Per fine cell the pass
// reads Phi^B, f^R, f^B once and writes Phi^R, Phi^B once (plus the halo
// overhead) instead of 4 x 12 bytes.
//
// The per-cell arithmetic is exactly that of every other smoother kernel
// (bitwise):  Phi_c = (f_c * w + s) / d,  s = ((((x- + x+) + y-) + y+) + z-) + z+,
// cells outside the level read as 0 (the folded boundary).
//
// The final black values are written to a second Phi^B buffer (the input
// black array is still read by neighbouring CTAs' halos); the host swaps the
// two black buffers between the pre- and post-smoothing passes.
//
// POST variant: the prolongation + magnified correction of the other colour
// is applied to the black input tile before the first red
// stage, exactly as in k_smooth_march<true> (red is overwritten unread).
// Box domains, one slab (or a level held whole), no mask, no periodic axis.
#include <cuda.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "mg_internal.h"
#include "mg_tma.cuh"

namespace mg {

namespace {

constexpr int kZT4 = 64;    // half-entries per tile (core)
constexpr int kSlots4 = 5;  // input ring: 3 in use + 2 in flight
// halos per stage s = 0 (input B0), 1 (R1), 2 (B1), 3 (R2), 4 (B2, core):
// rows 4 - s (what the remaining stages need); half-index columns rounded up
// to even numbers so that every tile row starts at an even global half-index
// and the cells are processed in 16-byte pairs (k, k+1)
__host__ __device__ constexpr int hr4(int s) { return 4 - s; }
__host__ __device__ constexpr int hc4(int s) {
  return s == 0 ? 6 : (s == 1 ? 4 : (s == 2 ? 4 : (s == 3 ? 2 : 0)));
}

template <int TY>
struct T4 {
  static constexpr int NT = TY * 32;  // threads
  __host__ __device__ static constexpr int rows(int s) { return TY + 2 * hr4(s); }
  __host__ __device__ static constexpr int cols(int s) { return kZT4 + 2 * hc4(s); }
  __host__ __device__ static constexpr int tile(int s) { return rows(s) * cols(s); }
  __host__ __device__ static constexpr int pairs(int s) { return rows(s) * cols(s) / 2; }
  __host__ __device__ static constexpr int per_thread(int s) {
    return (pairs(s) + NT - 1) / NT;
  }
  static constexpr int off1 = kSlots4 * tile(0);
  static constexpr int off2 = off1 + 3 * tile(1);
  static constexpr int off3 = off2 + 3 * tile(2);
  static constexpr int total = off3 + 3 * tile(3);  // doubles
  static constexpr size_t smem = (size_t)total * 8 + kSlots4 * 8;
};

}  // namespace

// g: the level (phiR written, phiB = output black buffer); tmB: the input
// black array (B0).  Stage colours: 1 red, 2 black, 3 red, 4 black.
template <int TY, bool PROLONG, bool FROMZERO>
__global__ void __launch_bounds__(TY * 32, (TY <= 8) ? 2 : 1)
    k_sweep4(Grid g, const __grid_constant__ CUtensorMap tmB, Grid C,
             double alpha, int ich) {
  using T = T4<TY>;
  extern __shared__ __align__(128) unsigned char smem[];
  double *sb = reinterpret_cast<double *>(smem);
  unsigned long long *bars =
      reinterpret_cast<unsigned long long *>(smem + (size_t)T::total * 8);
  const int nzt = (g.nzh + kZT4 - 1) / kZT4;
  const int nrt = (g.ny + TY - 1) / TY;
  int b = blockIdx.x;
  const int zt = b % nzt;
  b /= nzt;
  const int rt = b % nrt;
  const int xc = b / nrt;
  const int k0 = zt * kZT4, j0 = rt * TY;
  const int i0 = xc * ich;
  const int i1 = min(i0 + ich, g.nxl);
  const unsigned box_bytes = (unsigned)(T::tile(0) * 8);
  const int tfirst = i0 - 4, tlast = i1 - 1 + 4;  // input planes

  auto issue = [&](int t) {
    const int s = (t - tfirst) % kSlots4;
    mbar_expect_tx(&bars[s], box_bytes);
    tma_load_3d(sb + (size_t)s * T::tile(0), &tmB, k0 - hc4(0), j0 - hr4(0) + 1,
                t + 1, &bars[s]);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots4; s++) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (FROMZERO)
    for (int e = threadIdx.x; e < kSlots4 * T::tile(0); e += T::NT) sb[e] = 0.0;
  // RN(1/d) for the possible centres d = 0..12 (IEEE division, once)
  __shared__ double rcp[16];
  fill_rcp16(rcp);
  __syncthreads();
  if (!FROMZERO && threadIdx.x == 0)
    for (int t = tfirst; t <= min(tfirst + 2, tlast); t++) issue(t);

  // Per-thread pair descriptors, fixed for the whole kernel (only the plane
  // changes from step to step).  Pair m of stage s is tile element
  // e = tid + m NT -> row r = e / PW, column c = 2 (e % PW); packed:
  //   bits 0-3 / 4-7   centre d of the first cell for red-row parity 0 / 1
  //   bits 8-11/12-15  centre of the second cell (parity 0 / 1), x part excl.
  //   bit 16 row and first half-index inside the level, bit 17 second one
  //   bit 18 core (written to the output array), bit 19 row parity j & 1,
  //   bit 20 pair exists (e < pairs)
  struct Pd {
    int pk, q, fo;  // packed flags, input-tile offset, global row offset
  };
  auto make_pd = [&](auto S, int m) {
    constexpr int s = decltype(S)::value;
    constexpr int PW = T::cols(s) / 2;
    constexpr int Wi = (s > 0) ? T::cols(s - 1) : T::cols(0);
    constexpr int dc = (s > 0) ? hc4(s - 1) - hc4(s) : 0;
    const int e = threadIdx.x + m * T::NT;
    const int r = e / PW, c = 2 * (e % PW);
    const int j = j0 - hr4(s) + r, k = k0 - hc4(s) + c;
    Pd d;
    d.q = (r + 1) * Wi + c + dc;
    d.fo = (j + 1) * g.pz + k;
    int pk = 0;
    if (e < T::pairs(s)) {
      pk |= 1 << 20;
      const bool rin = j >= 0 && j < g.ny;
      if (rin && k >= 0 && k < g.nzh) pk |= 1 << 16;
      if (rin && k + 1 >= 0 && k + 1 < g.nzh) pk |= 1 << 17;
      if (j >= j0 && j < j0 + TY && k >= k0 && k < k0 + kZT4 && rin) pk |= 1 << 18;
      pk |= (j & 1) << 19;
      const int dy = 6 + (j == 0 ? g.dface[2] : 0) + (j == g.ny - 1 ? g.dface[3] : 0);
      for (int pp = 0; pp < 2; pp++) {
        const int z0 = 2 * k + pp;
        const int d0 = dy + (z0 == 0 ? g.dface[4] : 0) + (z0 == g.nz - 1 ? g.dface[5] : 0);
        const int d1 = dy + (z0 + 2 == g.nz - 1 ? g.dface[5] : 0);
        pk |= (d0 & 15) << (4 * pp);
        pk |= (d1 & 15) << (8 + 4 * pp);
      }
    }
    d.pk = pk;
    return d;
  };
  using S0 = std::integral_constant<int, 0>;
  using S1 = std::integral_constant<int, 1>;
  using S2 = std::integral_constant<int, 2>;
  using S3 = std::integral_constant<int, 3>;
  using S4 = std::integral_constant<int, 4>;
  constexpr int M1 = T::per_thread(1), M2 = T::per_thread(2), M3 = T::per_thread(3),
                M4 = T::per_thread(4), M0 = T::per_thread(0);
  Pd p1[M1], p2[M2], p3[M3], p4[M4];
#pragma unroll
  for (int m = 0; m < M1; m++) p1[m] = make_pd(S1{}, m);
#pragma unroll
  for (int m = 0; m < M2; m++) p2[m] = make_pd(S2{}, m);
#pragma unroll
  for (int m = 0; m < M3; m++) p3[m] = make_pd(S3{}, m);
#pragma unroll
  for (int m = 0; m < M4; m++) p4[m] = make_pd(S4{}, m);

  // f of the stage's colour on plane i (0 outside the level), a step ahead
  auto load_f = [&](auto S, int i, const Pd *pd, double2 *buf) {
    constexpr int s = decltype(S)::value;
    constexpr int M = T::per_thread(s);
    const double *f = ((s & 1) ? g.fR : g.fB) + (long long)(i + 1) * g.plane;
    const bool pin = i >= 0 && i < g.nxl;
#pragma unroll
    for (int m = 0; m < M; m++)
      buf[m] = (pin && (pd[m].pk & (1 << 16)))
                   ? *reinterpret_cast<const double2 *>(f + pd[m].fo)
                   : make_double2(0.0, 0.0);
  };
  // stage s on plane i from stage s-1 planes i-1, i, i+1
  auto stage = [&](auto S, int i, const double *__restrict__ Pm,
                   const double *__restrict__ Pc, const double *__restrict__ Pp,
                   double *__restrict__ out, const Pd *pd, const double2 *fb) {
    constexpr int s = decltype(S)::value;
    constexpr int M = T::per_thread(s);
    constexpr int Wi = T::cols(s - 1);
    constexpr int PW = T::cols(s) / 2;
    constexpr int col = (s & 1) ? 0 : 1;
    double *gout = (s == 3) ? g.phiR : (s == 4 ? g.phiB : nullptr);
    const bool pin = i >= 0 && i < g.nxl;
    const int ii = g.x0 + i;
    const int dxp = (ii == 0 ? g.dface[0] : 0) + (ii == g.nx - 1 ? g.dface[1] : 0);
    const bool core_plane = i >= i0 && i < i1;
    double *grow = gout ? gout + (long long)(i + 1) * g.plane : nullptr;
    const int par = (ii + col) & 1;
    double2 vv[M];
#pragma unroll
    for (int m = 0; m < M; m++) {
      const int pk = pd[m].pk;
      double2 v = make_double2(0.0, 0.0);
      if (pin && (pk & (1 << 16))) {
        const int p = par ^ ((pk >> 19) & 1);
        const int q = pd[m].q;
        double zm0, zp0, zm1, zp1;
        double2 a, bb, ym, yp;
        if (FROMZERO && s == 1) {
          a = bb = ym = yp = make_double2(0.0, 0.0);
          zm0 = zp0 = zm1 = zp1 = 0.0;
        } else {
          a = lds2(Pm + q);
          bb = lds2(Pp + q);
          ym = lds2(Pc + q - Wi);
          yp = lds2(Pc + q + Wi);
          const double2 zc = lds2(Pc + q);
          if (p == 0) {
            zm0 = Pc[q - 1];
            zp0 = zc.x;
            zm1 = zc.x;
            zp1 = zc.y;
          } else {
            zm0 = zc.x;
            zp0 = zc.y;
            zm1 = zc.y;
            zp1 = Pc[q + 2];
          }
        }
        const double s0 = ((((a.x + bb.x) + ym.x) + yp.x) + zm0) + zp0;
        const double s1 = ((((a.y + bb.y) + ym.y) + yp.y) + zm1) + zp1;
        const int d0 = ((pk >> (4 * p)) & 15) + dxp;
        const int d1 = ((pk >> (8 + 4 * p)) & 15) + dxp;
        v.x = div_small(fb[m].x * g.w + s0, (double)d0, rcp[d0]);
        if (pk & (1 << 17)) v.y = div_small(fb[m].y * g.w + s1, (double)d1, rcp[d1]);
        if (gout && core_plane && (pk & (1 << 18))) {
          double *o = grow + pd[m].fo;
          if (pk & (1 << 17))
            *reinterpret_cast<double2 *>(o) = v;
          else
            o[0] = v.x;
        }
      }
      vv[m] = v;
      (void)PW;
    }
    if (s < 4) {
#pragma unroll
      for (int m = 0; m < M; m++) {
        const int e = threadIdx.x + m * T::NT;
        if (pd[m].pk & (1 << 20))
          reinterpret_cast<double2 *>(out)[e] = vv[m];  // pair e: row e/PW, col 2(e%PW)
      }
    }
  };

  // PROLONG: coarse corrections of the input tile's black pairs of plane i:
  // black half-indices k, k+1 (k even) have parents at coarse z = k, k+1,
  // one red and one black coarse cell at coarse half-index k/2
  auto load_e = [&](int i, double2 *buf) {
    const int ii = g.x0 + i;
    const int I = ii >> 1;
    const double *cb = C.phiR + (long long)(I - C.x0 + 1) * C.plane;
    const long long dB = C.phiB - C.phiR;
    const bool pin = i >= 0 && i < g.nxl;
#pragma unroll
    for (int m = 0; m < M0; m++) {
      const int e = threadIdx.x + m * T::NT;
      constexpr int PW = T::cols(0) / 2;
      const int r = e / PW, c = 2 * (e % PW);
      const int j = j0 - hr4(0) + r, k = k0 - hc4(0) + c;
      double2 v = make_double2(0.0, 0.0);
      if (pin && r < T::rows(0) && j >= 0 && j < g.ny && k >= 0 && k < g.nzh) {
        const int J = j >> 1;
        const double *row = cb + (J + 1) * C.pz + (k >> 1);
        const int c0 = (I + J + k) & 1;  // colour of coarse z = k
        v.x = c0 ? row[dB] : row[0];
        if (k + 1 < g.nzh) v.y = c0 ? row[0] : row[dB];
      }
      buf[m] = v;
    }
  };

  double2 f1[M1], f2[M2], f3[M3], f4[M4], ec[PROLONG ? M0 : 1];
  load_f(S1{}, tfirst - 1, p1, f1);
  load_f(S2{}, tfirst - 2, p2, f2);
  load_f(S3{}, tfirst - 3, p3, f3);
  load_f(S4{}, tfirst - 4, p4, f4);
  if (PROLONG) load_e(tfirst, ec);
  // ring slots: input (5), stage tiles (3 each); the slot of plane t is
  // advanced incrementally
  int sin0 = 0;                       // slot of input plane t
  int sr1 = ((tfirst - 1) % 3 + 3) % 3;  // slot of R1 plane t - 1 (etc.)
  int sb1 = ((tfirst - 2) % 3 + 3) % 3;
  int sr2 = ((tfirst - 3) % 3 + 3) % 3;
  auto nx3 = [](int v) { return v == 2 ? 0 : v + 1; };
  auto pv3 = [](int v) { return v == 0 ? 2 : v - 1; };
  auto pv5 = [](int v) { return v == 0 ? kSlots4 - 1 : v - 1; };
  double *const R1 = sb + T::off1, *const B1 = sb + T::off2, *const R2 = sb + T::off3;

  for (int t = tfirst; t <= tlast; t++) {
    if (!FROMZERO && threadIdx.x == 0 && t + 2 <= tlast && t > tfirst) {
      fence_proxy_async();
      issue(t + 2);
    }
    // next step's f / e, in flight while this step computes
    double2 n1[M1], n2[M2], n3[M3], n4[M4], ne[PROLONG ? M0 : 1];
    load_f(S1{}, t, p1, n1);
    load_f(S2{}, t - 1, p2, n2);
    load_f(S3{}, t - 2, p3, n3);
    load_f(S4{}, t - 3, p4, n4);
    if (PROLONG) load_e(t + 1, ne);
    if (!FROMZERO) mbar_wait(&bars[sin0], ((t - tfirst) / kSlots4) & 1);
    double *in_t = sb + (size_t)sin0 * T::tile(0);
    if (PROLONG) {
      // B0(t) += alpha * e(parent) on the cells of the level (e = 0 elsewhere)
      double2 *B = reinterpret_cast<double2 *>(in_t);
#pragma unroll
      for (int m = 0; m < M0; m++) {
        const int e = threadIdx.x + m * T::NT;
        if (e < T::pairs(0) && t >= 0 && t < g.nxl) {
          double2 v = B[e];
          v.x = v.x + alpha * ec[m].x;
          v.y = v.y + alpha * ec[m].y;
          B[e] = v;
        }
      }
      __syncthreads();
    }
    const int s1m = pv5(sin0), s2m = pv5(s1m);
    if (t - 1 >= i0 - 3 && t - 1 <= i1 + 2)
      stage(S1{}, t - 1, sb + (size_t)s2m * T::tile(0), sb + (size_t)s1m * T::tile(0),
            in_t, R1 + (size_t)sr1 * T::tile(1), p1, f1);
    __syncthreads();
    if (t - 2 >= i0 - 2 && t - 2 <= i1 + 1)
      stage(S2{}, t - 2, R1 + (size_t)pv3(pv3(sr1)) * T::tile(1),
            R1 + (size_t)pv3(sr1) * T::tile(1), R1 + (size_t)sr1 * T::tile(1),
            B1 + (size_t)sb1 * T::tile(2), p2, f2);
    __syncthreads();
    if (t - 3 >= i0 - 1 && t - 3 <= i1)
      stage(S3{}, t - 3, B1 + (size_t)pv3(pv3(sb1)) * T::tile(2),
            B1 + (size_t)pv3(sb1) * T::tile(2), B1 + (size_t)sb1 * T::tile(2),
            R2 + (size_t)sr2 * T::tile(3), p3, f3);
    __syncthreads();
    if (t - 4 >= i0 && t - 4 <= i1 - 1)
      stage(S4{}, t - 4, R2 + (size_t)pv3(pv3(sr2)) * T::tile(3),
            R2 + (size_t)pv3(sr2) * T::tile(3), R2 + (size_t)sr2 * T::tile(3), nullptr,
            p4, f4);
    __syncthreads();  // ring slots of this step are free for the next one
#pragma unroll
    for (int m = 0; m < M1; m++) f1[m] = n1[m];
#pragma unroll
    for (int m = 0; m < M2; m++) f2[m] = n2[m];
#pragma unroll
    for (int m = 0; m < M3; m++) f3[m] = n3[m];
#pragma unroll
    for (int m = 0; m < M4; m++) f4[m] = n4[m];
    if (PROLONG) {
#pragma unroll
      for (int m = 0; m < M0; m++) ec[m] = ne[m];
    }
    sin0 = sin0 + 1 == kSlots4 ? 0 : sin0 + 1;
    sr1 = nx3(sr1);
    sb1 = nx3(sb1);
    sr2 = nx3(sr2);
  }
}

// ---- host side ------------------------------------------------------------------
bool sweep4_supported(const Grid &g) {
  return g.nxl == g.nx && !is_periodic(g) && !g.codeR && !g.coefR && !g.c64R &&
         g.nx >= 2 && g.ny >= 2 && g.nzh >= 1;
}

bool make_tmap_sweep4(const Grid &g, const double *base, void *out128) {
  return encode_box(g, base, out128, kZT4 + 2 * hc4(0), 8 + 2 * hr4(0)) &&
         encode_box(g, base, reinterpret_cast<unsigned char *>(out128) + 128,
                    kZT4 + 2 * hc4(0), 16 + 2 * hr4(0));
}

template <int TY, bool P, bool Z>
static void launch_t4(const Grid &g, const Grid &c, const CUtensorMap *tm,
                      double alpha, cudaStream_t s) {
  using T = T4<TY>;
  const int nzt = (g.nzh + kZT4 - 1) / kZT4;
  const int nrt = (g.ny + TY - 1) / TY;
  // x-chunks: long enough to amortise the 2 x 4 wavefront planes, short
  // enough for ~2 waves of CTAs
  const int per_sm = (TY <= 8) ? 2 : 1;
  int ich = 64;
  while (ich > 8 && (long long)((g.nxl + ich - 1) / ich) * nzt * nrt < 148 * per_sm * 2)
    ich >>= 1;
  const int nxc = (g.nxl + ich - 1) / ich;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_sweep4<TY, P, Z>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::smem);
    configured = true;
  }
  k_sweep4<TY, P, Z><<<nxc * nrt * nzt, T::NT, T::smem, s>>>(g, *tm, c, alpha, ich);
}

// tm256: two tensor maps (box rows TY=8 + 8, TY=16 + 8) of the input black
// array; g.phiB = the output black buffer
void launch_sweep4(const Grid &g, const Grid &c, const void *tm256, bool prolong,
                   bool from_zero, double alpha, int ty, cudaStream_t s) {
  const CUtensorMap *tm8 = reinterpret_cast<const CUtensorMap *>(tm256);
  const CUtensorMap *tm16 = tm8 + 1;
  if (ty == 16) {
    if (prolong)
      launch_t4<16, true, false>(g, c, tm16, alpha, s);
    else if (from_zero)
      launch_t4<16, false, true>(g, c, tm16, alpha, s);
    else
      launch_t4<16, false, false>(g, c, tm16, alpha, s);
  } else {
    if (prolong)
      launch_t4<8, true, false>(g, c, tm8, alpha, s);
    else if (from_zero)
      launch_t4<8, false, true>(g, c, tm8, alpha, s);
    else
      launch_t4<8, false, false>(g, c, tm8, alpha, s);
  }
}

}  // namespace mg
