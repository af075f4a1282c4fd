// Plane-marching kernels for sm_100a with TMA-staged neighbours.
//
// A CTA owns TY rows (j) of one x-chunk of ICH planes and marches along x.
// Neighbour planes -- rows j0-1 .. j0+TY (one halo row each side) -- stream
// into shared-memory rings with cp.async.bulk.tensor (TMA) completing on
// per-slot mbarriers, issued three planes ahead by one thread.  Every
// neighbour value therefore crosses L2->SM once per CTA (plus 2/TY halo
// rows) instead of ~5 times for direct loads; own f is prefetched one plane
// ahead in registers and results are written with 16-byte stores.
//
//   k_smooth_march<false>  RBGS half-sweep, the dominant kernel
//   k_smooth_march<true>   prolongation + magnified correction of the other
//                          colour fused with the half-sweep
//                          that follows it (the first post-smoothing red
//                          sweep): red cells are overwritten by that sweep,
//                          so only black needs the correction -- the result
//                          equals prolong-then-sweep bit for bit.
//   k_resid_march<RESTRICT> residual + 8-child averaging restriction
//   k_resid_march<NORM>     residual norm partial sums (Alg.1)
//
// Per-cell arithmetic is exactly that of mg_kernels.cu (bitwise identical):
//     Phi_c = (f_c * w + s) / d,  r_c = f_c - c (d Phi_c - s),
//     s = ((((x- + x+) + y-) + y+) + z-) + z+.
#include <cuda.h>
#include <cuda_runtime.h>

#include "mg_internal.h"
#include "mg_tma.cuh"

namespace mg {



// ============================================================================
// half-sweep (optionally fused with the prolongation of the other colour)
// one TMA box = (pz doubles) x (TY+2 rows) x (1 plane)
// ============================================================================
// VAR: 0 box domain, 1 solid mask (byte codes), 2 periodic axes -- compile-
// time variants, so the box-domain kernel carries neither code path
enum { VAR_BOX = 0, VAR_MASK = 1, VAR_PER = 2 };

// rows of <= 128 half-entries (NCH <= 2: level 1 and below at 512^3) fit 3
// CTAs per SM (<= 85 registers, no spills; 4 spilled and were no faster)
// NORM 1: also the residual of every updated cell after the sweep (its
// neighbours are the other colour, final), f - c (d u - s) with the residual
// kernels' expression, r^2 summed into one partial per CTA (fixed order) --
// the last black half-sweep of a cycle then leaves only the red residuals to
// the norm pass (12 instead of 16 B/cell).
// NORM 2 (the look-ahead red sweep): the residual of each updated
// cell BEFORE the sweep, u = oldv (the own colour's current values; the sweep
// writes its results to g's own array, a different buffer): the same s and
// d serve the residual and the update, so the red residuals of the iterate
// cost 4 B/cell more than the sweep instead of a 12 B/cell pass.
template <bool PROLONG, int NCH, int VAR, int NORM = 0>
__global__ void __launch_bounds__(kThreadsM, NCH <= 2 ? 3 : 2)
    k_smooth_march(Grid g, const __grid_constant__ CUtensorMap tm_oth,
                   int color, Grid C, double alpha, double *partials,
                   const double *__restrict__ oldv) {
  constexpr bool MASK = VAR == VAR_MASK;
  constexpr bool PER = VAR == VAR_PER;
  extern __shared__ __align__(128) unsigned char smem[];
  const int pz = g.pz;
  const int sd = slot_doubles(pz);
  double *ring = reinterpret_cast<double *>(smem);
  unsigned long long *bars =
      reinterpret_cast<unsigned long long *>(smem + (size_t)kSlots * sd * 8);
  const unsigned box_bytes = (unsigned)((kTY + 2) * pz * 8);

  const int nrt = (g.ny + kTY - 1) / kTY;
  const int ich = chunk_planes(g.nxl, nrt, g.nsm);
  const int rt = blockIdx.x % nrt;
  const int xc = blockIdx.x / nrt;
  const int j0 = rt * kTY;
  const int i0 = xc * ich;
  const int i1 = min(i0 + ich, g.nxl);
  const int nplanes = (i1 - i0) + 2;  // local planes i0-1 .. i1
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; s++) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // prologue: planes q = 0..3 (local plane i0-1+q, array plane i0+q)
  if (threadIdx.x == 0) {
    const int np = nplanes < 4 ? nplanes : 4;
    for (int q = 0; q < np; q++) {
      mbar_expect_tx(&bars[q], box_bytes);
      tma_load_3d(ring + (size_t)q * sd, &tm_oth, 0, j0, i0 + q, &bars[q]);
    }
  }

  const int j = j0 + warp;
  const bool row_ok = j < g.ny;
  double *__restrict__ own = color ? g.phiB : g.phiR;
  const double *__restrict__ fown = color ? g.fB : g.fR;
  // NCH: lane chunks of 64 half-entries per warp pass, ceil(nzh / 64)

  // PROLONG: add alpha * e(parent) to the ring copy of local plane il (rows
  // j0-1 .. j0+TY).  The corrected other colour is NOT written back: the
  // half-sweep of the other colour that follows overwrites every one of its
  // cells without reading them (and a write-back would race with the TMA
  // halo reads of neighbouring CTAs).  The coarse values are loaded one plane
  // ahead (load_e) so their latency hides behind the previous plane's work.
  // Work split: task t = (coarse row jr, 64-wide chunk c), t = warp + TY*m:
  // the tile rows j0-1 .. j0+TY have the parent rows J = j0/2 - 1 + jr,
  // jr = 0 .. TY/2 + 1; the two sibling rows 2J, 2J+1 (tile rows 2jr-1,
  // 2jr, where inside the tile) share the coarse values, loaded once.
  constexpr int kJR = kTY / 2 + 2;
  constexpr int ntask = kJR * NCH;
  constexpr int kTPW = (ntask + kTY - 1) / kTY;  // tasks per warp
  int tK[kTPW], tCoff[kTPW], tJp[kTPW], tRowA[kTPW];
  bool tOkA[kTPW], tOkB[kTPW];
  auto row_valid = [&](int jj) {
    // rows of the level, plus (y periodic) the ghost rows -1 / ny that hold
    // the opposite side's cells and need their parents' correction too
    return (PER && g.per[1]) ? (jj >= -1 && jj <= g.ny) : (jj >= 0 && jj < g.ny);
  };
#pragma unroll
  for (int m = 0; m < kTPW; m++) {
    const int t = warp + kTY * m;
    const int jr = t / NCH, c = t % NCH;
    const int J = (j0 >> 1) - 1 + jr;
    const int k = 2 * lane + 64 * c;
    const bool ok = PROLONG && t < ntask && k < g.nzh;
    const int rrA = 2 * jr - 1, rrB = 2 * jr;  // tile rows of 2J, 2J+1
    tOkA[m] = ok && rrA >= 0 && row_valid(2 * J);
    tOkB[m] = ok && rrB <= kTY + 1 && row_valid(2 * J + 1);
    tRowA[m] = rrA * pz;
    tK[m] = k;
    tCoff[m] = (J + 1) * C.pz + (k >> 1);
    tJp[m] = J & 1;
  }
  auto load_e = [&](int q, double2 *E) {
    const int i = g.x0 + i0 - 1 + q;
    // x periodic: ghost planes -1 / nx hold the opposite side's cells, their
    // parents sit in the coarse ghost planes (I = -1 / nx/2), kept current
    const bool pok = (PER && g.per[0]) || (i >= 0 && i < g.nx);
    const int I = i >> 1;
    const long long poff = (long long)(I - C.x0 + 1) * C.plane;
    const int Ip = I & 1;
#pragma unroll
    for (int m = 0; m < kTPW; m++) {
      E[m] = make_double2(0.0, 0.0);
      if (!(pok && (tOkA[m] || tOkB[m]))) continue;
      // parents of half-indices k, k+1 are coarse z = k, k+1: one red and
      // one black coarse cell at coarse half-index k/2 (k even)
      const int c0 = (Ip + tJp[m]) & 1;
      const long long cb = poff + tCoff[m];
      E[m].x = (c0 ? C.phiB : C.phiR)[cb];
      E[m].y = (c0 ? C.phiR : C.phiB)[cb];
      // (MASK: a solid cell of the other colour may receive a correction in
      // this smem copy -- it is never written back, and the red update
      // weights a solid neighbour by kappa = 0, so its value is unused)
    }
  };
  auto apply_e = [&](int q, const double2 *E) {
    const int i = g.x0 + i0 - 1 + q;
    if (!(PER && g.per[0]) && (i < 0 || i >= g.nx)) return;  // physical ghost: 0
    double *slot = ring + (size_t)(q % kSlots) * sd;
    auto add = [&](double *row, int k, const double2 e) {
      double2 v = lds2(row + k);
      v.x = v.x + alpha * e.x;
      v.y = v.y + alpha * e.y;
      if (k + 1 < g.nzh)
        *reinterpret_cast<double2 *>(row + k) = v;
      else
        row[k] = v.x;
    };
#pragma unroll
    for (int m = 0; m < kTPW; m++) {
      if (tOkA[m]) add(slot + tRowA[m], tK[m], E[m]);
      if (tOkB[m]) add(slot + tRowA[m] + pz, tK[m], E[m]);
    }
  };
  // parent rows J = j0/2 - 1 .. j0/2 + TY/2 of coarse plane i >> 1 (array
  // rows J + 1, contiguous), both colours
  auto prefetch_parent_rows = [&](int i) {
    if (!((PER && g.per[0]) || (i >= 0 && i < g.nx))) return;
    const long long off =
        (long long)((i >> 1) - C.x0 + 1) * C.plane + (long long)(j0 >> 1) * C.pz;
    const int rows = min(kJR, C.ny + 2 - (j0 >> 1));
    const unsigned bytes = (unsigned)(rows * C.pz * 8);
    prefetch_l2_bulk(C.phiR + off, bytes);
    prefetch_l2_bulk(C.phiB + off, bytes);
  };
  if (PROLONG && threadIdx.x == 0)
    for (int q = 0; q < 4 && q < nplanes; q += 2) prefetch_parent_rows(g.x0 + i0 - 1 + q);
  double2 E[kTPW];
  if (PROLONG && nplanes > 2) load_e(2, E);

  // f (and, masked, the own face codes) of the first plane into registers
  double2 fr[NCH];
  unsigned cr[NCH];
  const unsigned char *__restrict__ cown = color ? g.codeB : g.codeR;
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    const int k = 2 * lane + 64 * c;
    cr[c] = 0x4040u;
    if (row_ok && k < g.nzh) {
      const long long o = (long long)(i0 + 1) * g.plane + (long long)(j + 1) * pz + k;
      fr[c] = *reinterpret_cast<const double2 *>(fown + o);
      if (MASK) cr[c] = *reinterpret_cast<const unsigned short *>(cown + o);
    }
  }

  double nacc = 0.0;  // NORM: sum of r^2 of this thread's updated cells
  if (NORM == 2 && threadIdx.x == 0)  // the first two planes' own rows
    for (int il = i0; il < i1 && il < i0 + 2; il++)
      prefetch_l2_bulk(oldv + (long long)(il + 1) * g.plane + (long long)(j0 + 1) * pz,
                       (unsigned)(min(kTY, g.ny - j0) * pz * 8));
  for (int il = i0; il < i1; il++) {
    const int q = il - i0 + 1;  // ring index of the current plane
    __syncthreads();            // everybody is done with plane q-2's slot
    if (threadIdx.x == 0 && q + 3 < nplanes) {
      const int s = (q + 3) % kSlots;
      fence_proxy_async();
      mbar_expect_tx(&bars[s], box_bytes);
      tma_load_3d(ring + (size_t)s * sd, &tm_oth, 0, j0, i0 + q + 3, &bars[s]);
    }
    // NORM 2: the tile's rows of the own colour two planes ahead into L2 (one
    // bulk prefetch: the rows are contiguous), then this plane's values into
    // registers (issued before the ring waits)
    if (NORM == 2 && threadIdx.x == 0 && il + 2 < i1)
      prefetch_l2_bulk(oldv + (long long)(il + 3) * g.plane + (long long)(j0 + 1) * pz,
                       (unsigned)(min(kTY, g.ny - j0) * pz * 8));
    // PROLONG: the parent rows of local plane q + 4 (both colours) into L2,
    // once per coarse plane, ahead of load_e's register loads
    if (PROLONG && threadIdx.x == 0 && q + 4 < nplanes) {
      const int i4 = g.x0 + i0 - 1 + q + 4;
      if (!(i4 & 1) || q == 1) prefetch_parent_rows(i4);
    }
    double2 ov[NCH];
    if (NORM == 2) {
#pragma unroll
      for (int c = 0; c < NCH; c++) {
        const int k = 2 * lane + 64 * c;
        ov[c] = make_double2(0.0, 0.0);
        if (row_ok && k < g.nzh)
          ov[c] = *reinterpret_cast<const double2 *>(
              oldv + (long long)(il + 1) * g.plane + (long long)(j + 1) * pz + k);
      }
    }
    // wait for planes q-1 (first step only), q (first step only), q+1
    if (q == 1) {
      mbar_wait(&bars[0], 0);
      mbar_wait(&bars[1], 0);
    }
    mbar_wait(&bars[(q + 1) % kSlots], ((q + 1) / kSlots) & 1);
    if (PROLONG) {
      if (q == 1) {
        double2 E0[kTPW];
        load_e(0, E0);
        apply_e(0, E0);
        load_e(1, E0);
        apply_e(1, E0);
      }
      apply_e(q + 1, E);
      // fine planes 2I and 2I+1 share the parent plane I: keep E (the same
      // tasks, the same coarse values) instead of loading it again
      const int ia = g.x0 + i0 + q, ib = ia + 1;  // global planes q+1, q+2
      if (q + 2 < nplanes && (ia >> 1) != (ib >> 1)) load_e(q + 2, E);
      __syncthreads();
    }

    // prefetch f of the next plane
    double2 fn[NCH];
    unsigned cn[NCH];
    const bool more = il + 1 < i1;
#pragma unroll
    for (int c = 0; c < NCH; c++) {
      const int k = 2 * lane + 64 * c;
      cn[c] = 0x4040u;
      if (more && row_ok && k < g.nzh) {
        const long long o = (long long)(il + 2) * g.plane + (long long)(j + 1) * pz + k;
        fn[c] = *reinterpret_cast<const double2 *>(fown + o);
        if (MASK) cn[c] = *reinterpret_cast<const unsigned short *>(cown + o);
      }
    }
    if (row_ok) {
      const double *cur = ring + (size_t)(q % kSlots) * sd + (warp + 1) * pz;
      const double *xm = ring + (size_t)((q - 1) % kSlots) * sd + (warp + 1) * pz;
      const double *xp = ring + (size_t)((q + 1) % kSlots) * sd + (warp + 1) * pz;
      const int i = g.x0 + il;
      const int p = (i + j + color) & 1;
      double *orow = own + (long long)(il + 1) * g.plane + (long long)(j + 1) * pz;
#pragma unroll
      for (int c = 0; c < NCH; c++) {
        const int k = 2 * lane + 64 * c;
        if (k >= g.nzh) continue;
        const double2 a = lds2(xm + k);
        const double2 b = lds2(xp + k);
        const double2 ym = lds2(cur - pz + k);
        const double2 yp = lds2(cur + pz + k);
        const double2 zc = lds2(cur + k);
        double zm0, zp0, zm1, zp1;
        if (p == 0) {
          zm0 = z_lo<PER>(g, cur, k);
          zp0 = zc.x;
          zm1 = zc.x;
          zp1 = zc.y;
        } else {
          zm0 = zc.x;
          zp0 = z_hi0<PER>(g, cur, k, zc.y);
          zm1 = zc.y;
          zp1 = z_hi<PER>(g, cur, k);
        }
        const int z0 = 2 * k + p;
        double s0, s1, d0, d1;
        unsigned cd0 = 64, cd1 = 64;
        if (MASK && !__all_sync(__activemask(), cr[c] == kOpenPair)) {
          const unsigned cc2 = cr[c];
          cd0 = cc2 & 0xffu;
          cd1 = (k + 1 < g.nzh) ? (cc2 >> 8) : 0u;
          s0 = ksum(cd0, a.x, b.x, ym.x, yp.x, zm0, zp0);
          s1 = ksum(cd1, a.y, b.y, ym.y, yp.y, zm1, zp1);
          d0 = kdiag(g, cd0, i, j, z0);
          d1 = kdiag(g, cd1, i, j, z0 + 2);
        } else if (MASK) {
          // the whole warp on fluid cells with all six faces open (the bulk
          // of a masked level): kappa = 1 everywhere and no domain face, so
          // ksum is the plain sum and kdiag = popc(63) = 6 -- the same bits
          if (k + 1 >= g.nzh) cd1 = 0u;
          s0 = ((((a.x + b.x) + ym.x) + yp.x) + zm0) + zp0;
          s1 = ((((a.y + b.y) + ym.y) + yp.y) + zm1) + zp1;
          d0 = d1 = 6.0;
        } else {
          s0 = ((((a.x + b.x) + ym.x) + yp.x) + zm0) + zp0;
          s1 = ((((a.y + b.y) + ym.y) + yp.y) + zm1) + zp1;
          d0 = (double)centre_dm(g, i, j, z0);
          d1 = (double)centre_dm(g, i, j, z0 + 2);
        }
        double2 out;
        // exact division (bitwise IEEE) with RN(1/d) from the constant-memory
        // table (a broadcast for the warp-uniform interior d = 6; measured
        // faster than a shared-memory table or an IEEE division on boundary
        // cells)
        out.x = div_small(fr[c].x * g.w + s0, d0, c_rcp16[(int)d0]);
        out.y = div_small(fr[c].y * g.w + s1, d1, c_rcp16[(int)d1]);
        if (NORM) {
          const double u0 = NORM == 2 ? ov[c].x : out.x;
          const double u1 = NORM == 2 ? ov[c].y : out.y;
          const double r0 = (cd0 & 64) ? fr[c].x - g.c * (d0 * u0 - s0) : 0.0;
          const double r1 =
              (k + 1 < g.nzh && (cd1 & 64)) ? fr[c].y - g.c * (d1 * u1 - s1) : 0.0;
          nacc = nacc + r0 * r0;
          nacc = nacc + r1 * r1;
        }
        if (NORM == 2 && MASK) {
          // the look-ahead writes another buffer: a cell that is not an
          // unknown (solid) keeps its value there too
          if (!(cd0 & 64)) out.x = ov[c].x;
          if (!(cd1 & 64)) out.y = ov[c].y;
          cd0 = 64;
          cd1 = k + 1 < g.nzh ? 64u : 0u;
        }
        const bool both = k + 1 < g.nzh && (cd0 & 64) && (cd1 & 64);
        if (both) {
          *reinterpret_cast<double2 *>(orow + k) = out;
          if (PER) ghost_copies(g, own, il, j, k, out);
        } else {  // ragged row end or a solid cell (not an unknown: untouched)
          if (cd0 & 64) orow[k] = out.x;
          if (k + 1 < g.nzh && (cd1 & 64)) orow[k + 1] = out.y;
          if (PER) ghost_copies(g, own, il, j, k, out.x);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < NCH; c++) {
      fr[c] = fn[c];
      cr[c] = cn[c];
    }
  }
  if (NORM) {  // deterministic block reduction (warp tree, warps in order)
    __shared__ double nred[kTY];
    double v = nacc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) nred[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double sum = 0.0;
      for (int w = 0; w < kTY; w++) sum = sum + nred[w];
      partials[blockIdx.x] = sum;
    }
  }
}

// ============================================================================
// residual kernels: two rings (Phi^R, Phi^B), z-tiles of ZT half-entries with
// one halo element each side; box = (ZT+2) x (TY+2 rows) x (1 plane)
// ============================================================================
// MODE_BOTH: restriction plus the norm partials of the same residual (the
// fused termination norm, reading c11)
// MODE_NORM_RED: the norm partials of the red residuals only (the black ones
// were summed by the last black half-sweep, k_smooth_march<..., NORM>)
enum { MODE_RESTRICT = 0, MODE_NORM = 1, MODE_BOTH = 2, MODE_NORM_RED = 3 };

template <int MODE, int VAR>
__global__ void __launch_bounds__(kThreadsM, 2)
    k_resid_march(Grid g, const __grid_constant__ CUtensorMap tmR,
                  const __grid_constant__ CUtensorMap tmB, Grid C,
                  double *partials, int red0) {
  constexpr bool MASK = VAR == VAR_MASK;
  constexpr bool PER = VAR == VAR_PER;
  extern __shared__ __align__(128) unsigned char smem[];
  const int W = rbox0(g);  // smem row width = TMA box width
  const int sd = rslot_doubles();
  double *ringR = reinterpret_cast<double *>(smem);
  double *ringB = ringR + (size_t)kSlots * sd;
  double *xch = ringB + (size_t)kSlots * sd;  // [TY/2][ZT] row-pair exchange
  unsigned long long *bars =
      reinterpret_cast<unsigned long long *>(xch + (kTY / 2) * kZT);
  __shared__ double red_sh[32];
  const unsigned box_bytes = (unsigned)((kTY + 2) * W * 8);

  const int nzt = rntiles(g);
  const int nrt = (g.ny + kTY - 1) / kTY;
  int b = blockIdx.x;
  const int zt = b % nzt;
  b /= nzt;
  const int rt = b % nrt;
  const int xc = b / nrt;
  const int ich = chunk_planes(g.nxl, nrt * nzt, g.nsm);
  const int kz0 = zt * kZT;
  const int c0z = rtile_c0(g, kz0);
  const int zoff = kz0 - c0z;  // smem column of half-index kz0
  const int j0 = rt * kTY;
  const int i0 = xc * ich;
  const int i1 = min(i0 + ich, g.nxl);
  const int nplanes = (i1 - i0) + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; s++) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int q) {
    const int s = q % kSlots;
    mbar_expect_tx(&bars[s], 2 * box_bytes);
    tma_load_3d(ringR + (size_t)s * sd, &tmR, c0z, j0, i0 + q, &bars[s]);
    tma_load_3d(ringB + (size_t)s * sd, &tmB, c0z, j0, i0 + q, &bars[s]);
  };
  if (threadIdx.x == 0) {
    const int np = nplanes < 4 ? nplanes : 4;
    for (int q = 0; q < np; q++) issue(q);
  }

  const int j = j0 + warp;
  const bool row_ok = j < g.ny;
  double acc = 0.0;
  double sdx0[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // restriction, even plane

  // f (and, masked, face codes) of both colours, first plane
  double2 fR[2], fB[2];
  unsigned cR[2] = {0x4040u, 0x4040u}, cB[2] = {0x4040u, 0x4040u};
#pragma unroll
  for (int c = 0; c < 2; c++) {
    const int k = kz0 + 2 * lane + 64 * c;
    if (row_ok && k < g.nzh) {
      const long long o = (long long)(i0 + 1) * g.plane + (long long)(j + 1) * g.pz + k;
      fR[c] = *reinterpret_cast<const double2 *>(g.fR + o);
      if (MODE != MODE_NORM_RED) fB[c] = *reinterpret_cast<const double2 *>(g.fB + o);
      if (MASK) {
        cR[c] = *reinterpret_cast<const unsigned short *>(g.codeR + o);
        cB[c] = *reinterpret_cast<const unsigned short *>(g.codeB + o);
      }
    }
  }

  // periodic z: the other colour's row ends (half-indices nzh-1 and 0) of
  // plane il, [wlo(own R), wlo(own B), whi(own R), whi(own B)], read by the
  // tiles at the row ends with direct loads (the arrays are not written
  // here), one plane ahead so that their latency hides behind a plane
  double wr[4] = {0.0, 0.0, 0.0, 0.0};
  auto load_wrap = [&](int il, double *w) {
    if (!(PER && g.per[2]) || !row_ok) return;
    const long long ro = (long long)(il + 1) * g.plane + (long long)(j + 1) * g.pz;
    if (zt == 0) {
      w[0] = g.phiB[ro + g.nzh - 1];
      w[1] = g.phiR[ro + g.nzh - 1];
    }
    if (zt == nzt - 1) {
      w[2] = g.phiB[ro];
      w[3] = g.phiR[ro];
    }
  };
  if (PER) load_wrap(i0, wr);

  // f of the row tile's rows (all z-tiles: contiguous rows) two planes
  // ahead into L2, by the z-tile 0 CTA, ahead of the register prefetch
  auto prefetch_f = [&](int il) {
    const long long o = (long long)(il + 1) * g.plane + (long long)(j0 + 1) * g.pz;
    const unsigned bytes = (unsigned)(min(kTY, g.ny - j0) * g.pz * 8);
    prefetch_l2_bulk(g.fR + o, bytes);
    if (MODE != MODE_NORM_RED) prefetch_l2_bulk(g.fB + o, bytes);
  };
  if (zt == 0 && threadIdx.x == 0)
    for (int il = i0 + 1; il < i1 && il < i0 + 3; il++) prefetch_f(il);
  for (int il = i0; il < i1; il++) {
    const int q = il - i0 + 1;
    __syncthreads();
    if (threadIdx.x == 0 && q + 3 < nplanes) {
      fence_proxy_async();
      issue(q + 3);
    }
    if (zt == 0 && threadIdx.x == 0 && il + 3 < i1) prefetch_f(il + 3);
    if (q == 1) {
      mbar_wait(&bars[0], 0);
      mbar_wait(&bars[1], 0);
    }
    mbar_wait(&bars[(q + 1) % kSlots], ((q + 1) / kSlots) & 1);

    double2 nR[2], nB[2];
    unsigned ncR[2] = {0x4040u, 0x4040u}, ncB[2] = {0x4040u, 0x4040u};
    const bool more = il + 1 < i1;
    double nwr[4] = {0.0, 0.0, 0.0, 0.0};
    if (PER && more) load_wrap(il + 1, nwr);
#pragma unroll
    for (int c = 0; c < 2; c++) {
      const int k = kz0 + 2 * lane + 64 * c;
      if (more && row_ok && k < g.nzh) {
        const long long o = (long long)(il + 2) * g.plane + (long long)(j + 1) * g.pz + k;
        nR[c] = *reinterpret_cast<const double2 *>(g.fR + o);
        if (MODE != MODE_NORM_RED) nB[c] = *reinterpret_cast<const double2 *>(g.fB + o);
        if (MASK) {
          ncR[c] = *reinterpret_cast<const unsigned short *>(g.codeR + o);
          ncB[c] = *reinterpret_cast<const unsigned short *>(g.codeB + o);
        }
      }
    }
    const int i = g.x0 + il;
    double pr[2][2];  // [chunk][element] red + black pair sums (restriction)
#pragma unroll
    for (int c = 0; c < 2; c++) pr[c][0] = pr[c][1] = 0.0;
    if (row_ok) {
      const size_t oc = (size_t)(q % kSlots) * sd + (warp + 1) * W + zoff;
      const size_t om = (size_t)((q - 1) % kSlots) * sd + (warp + 1) * W + zoff;
      const size_t op = (size_t)((q + 1) % kSlots) * sd + (warp + 1) * W + zoff;
      const double wlo[2] = {wr[0], wr[1]}, whi[2] = {wr[2], wr[3]};  // [own colour]
      // the centre's x / y face terms are the row's (hoisted); z adds only at
      // the row ends -- the same integer as centre_dm
      const int dxy = 6 + (i == 0 ? g.dface[0] : 0) + (i == g.nx - 1 ? g.dface[1] : 0) +
                      (j == 0 ? g.dface[2] : 0) + (j == g.ny - 1 ? g.dface[3] : 0);
      auto dcen = [&](int z) {
        return (double)(dxy + (z == 0 ? g.dface[4] : 0) + (z == g.nz - 1 ? g.dface[5] : 0));
      };
#pragma unroll
      for (int c = 0; c < 2; c++) {
        const int kl = 2 * lane + 64 * c;  // tile-relative half-index
        const int k = kz0 + kl;
        if (k >= g.nzh) continue;
        // the warp's cells of both colours all fluid with six open faces:
        // the plain-box arithmetic gives the same bits (see the smoother)
        const bool open =
            MASK && __all_sync(__activemask(), cR[c] == kOpenPair && cB[c] == kOpenPair);
        double r[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // [colour][element]
#pragma unroll
        for (int col = 0; col < (MODE == MODE_NORM_RED ? 1 : 2); col++) {
          const double *O = col ? ringR : ringB;  // other colour's ring
          const double *M = col ? ringB : ringR;  // own colour's ring
          const int p = (i + j + col) & 1;
          const double2 a = lds2(O + om + kl);
          const double2 bb = lds2(O + op + kl);
          const double2 ym = lds2(O + oc - W + kl);
          const double2 yp = lds2(O + oc + W + kl);
          const double2 zc = lds2(O + oc + kl);
          const double2 u = lds2(M + oc + kl);
          // z neighbours; the halo element is 0 outside the level, or on a
          // periodic z axis the row's opposite end (not in this z-tile: a
          // direct load of the other colour, unchanged during this kernel)
          double zm0, zp0, zm1, zp1;
          if (p == 0) {
            zm0 = (k > 0) ? O[oc + kl - 1] : wlo[col];
            zp0 = zc.x;
            zm1 = zc.x;
            zp1 = zc.y;
          } else {
            zm0 = zc.x;
            zp0 = (PER && g.per[2] && k + 1 >= g.nzh) ? whi[col] : zc.y;
            zm1 = zc.y;
            zp1 = (k + 2 < g.nzh) ? O[oc + kl + 2] : whi[col];
          }
          const int z0 = 2 * k + p;
          double s0, s1, d0, d1;
          unsigned cd0 = 64, cd1 = 64;
          if (MASK && !open) {
            const unsigned cc2 = col ? cB[c] : cR[c];
            cd0 = cc2 & 0xffu;
            cd1 = (k + 1 < g.nzh) ? (cc2 >> 8) : 0u;
            s0 = ksum(cd0, a.x, bb.x, ym.x, yp.x, zm0, zp0);
            s1 = ksum(cd1, a.y, bb.y, ym.y, yp.y, zm1, zp1);
            d0 = kdiag(g, cd0, i, j, z0);
            d1 = kdiag(g, cd1, i, j, z0 + 2);
          } else if (MASK) {
            if (k + 1 >= g.nzh) cd1 = 0u;
            s0 = ((((a.x + bb.x) + ym.x) + yp.x) + zm0) + zp0;
            s1 = ((((a.y + bb.y) + ym.y) + yp.y) + zm1) + zp1;
            d0 = d1 = 6.0;
          } else {
            s0 = ((((a.x + bb.x) + ym.x) + yp.x) + zm0) + zp0;
            s1 = ((((a.y + bb.y) + ym.y) + yp.y) + zm1) + zp1;
            d0 = dcen(z0);
            d1 = dcen(z0 + 2);
          }
          const double t0 = d0 * u.x - s0;
          const double t1 = d1 * u.y - s1;
          const double2 fo = col ? fB[c] : fR[c];
          r[col][0] = (cd0 & 64) ? fo.x - g.c * t0 : 0.0;
          r[col][1] = (k + 1 < g.nzh && (cd1 & 64)) ? fo.y - g.c * t1 : 0.0;
        }
        if (MODE != MODE_RESTRICT) {
          acc = acc + r[0][0] * r[0][0];
          acc = acc + r[0][1] * r[0][1];
          acc = acc + r[1][0] * r[1][0];
          acc = acc + r[1][1] * r[1][1];
        }
        if ((MODE == MODE_RESTRICT || MODE == MODE_BOTH)) {
          // z-children of coarse K = k are the red and black cells at
          // half-index k (commutative pair: r_dz0 + r_dz1)
          pr[c][0] = r[0][0] + r[1][0];
          pr[c][1] = r[0][1] + r[1][1];
        }
      }
    }
    if ((MODE == MODE_RESTRICT || MODE == MODE_BOTH)) {
      // y-children: rows 2J (even warp) + 2J+1 (odd warp), in that order
      if (warp & 1) {
#pragma unroll
        for (int c = 0; c < 2; c++) {
          const int kl = 2 * lane + 64 * c;
          xch[(warp >> 1) * kZT + kl] = pr[c][0];
          xch[(warp >> 1) * kZT + kl + 1] = pr[c][1];
        }
      }
      __syncthreads();
      if (!(warp & 1) && row_ok) {
        const bool odd_plane = (il & 1);
        const int J = j >> 1;
        const int I = i >> 1;
#pragma unroll
        for (int c = 0; c < 2; c++) {
          const int kl = 2 * lane + 64 * c;
          const int k = kz0 + kl;
          if (k >= g.nzh) continue;
          const double s0 = pr[c][0] + xch[(warp >> 1) * kZT + kl];
          const double s1 = pr[c][1] + xch[(warp >> 1) * kZT + kl + 1];
          if (!odd_plane) {
            sdx0[c][0] = s0;
            sdx0[c][1] = s1;
          } else {
            // coarse cells K = k and k+1: one of each colour at K/2 = k/2
            const long long cb = (long long)(I - C.x0 + 1) * C.plane +
                                 (long long)(J + 1) * C.pz + (k >> 1);
            const int c0 = (I + J + k) & 1;
            const double fk0 = 0.125 * (sdx0[c][0] + s0);
            const double fk1 = 0.125 * (sdx0[c][1] + s1);
            (c0 ? C.fB : C.fR)[cb] = fk0;
            if (k + 1 < g.nzh) (c0 ? C.fR : C.fB)[cb] = fk1;
            if (red0) {
              // the coarse level's first red half-sweep from Phi = 0:
              // Phi_red = (f w + 0) / d, the expression of k_smooth's
              // from-zero sweep on the red cell among K = k, k+1
              const int kr = c0 ? k + 1 : k;
              if (kr < C.nz) {
                const double fr = c0 ? fk1 : fk0;
                const double d = (double)centre_dm(C, I, J, kr);
                C.phiR[cb] = div_small(fr * C.w + 0.0, d, c_rcp16[(int)d]);
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 2; c++) {
      fR[c] = nR[c];
      fB[c] = nB[c];
      cR[c] = ncR[c];
      cB[c] = ncB[c];
    }
    if (PER)
#pragma unroll
      for (int e = 0; e < 4; e++) wr[e] = nwr[e];
  }
  if (MODE != MODE_RESTRICT) {
    // deterministic block reduction
    double v = acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red_sh[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < kTY; w++) s = s + red_sh[w];
      partials[blockIdx.x] = s;
    }
  }
}

// ---- host side ------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType,
                                    cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *,
                                    const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault,
                                &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  }
  return fn;
}

bool march_supported(const Grid &g) {
  // whole row in one TMA box (<= 256 elements), at least one full row tile
  return g.pz <= 256 && g.nzh >= 64 && g.ny >= kTY && g.nxl >= 2 &&
         get_encode() != nullptr;
}

static size_t smooth_smem_bytes(const Grid &g) {
  return (size_t)kSlots * slot_doubles(g.pz) * 8 + kSlots * 8;
}

static size_t resid_smem_bytes() {
  return (size_t)2 * kSlots * rslot_doubles() * 8 + (kTY / 2) * kZT * 8 +
         kSlots * 8;
}

static bool encode(const Grid &g, const double *base, void *out128,
                   cuuint32_t box0) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  CUtensorMap *tm = reinterpret_cast<CUtensorMap *>(out128);
  cuuint64_t dims[3] = {(cuuint64_t)g.pz, (cuuint64_t)(g.ny + 2),
                        (cuuint64_t)(g.nxl + 2)};
  cuuint64_t strides[2] = {(cuuint64_t)g.pz * 8, (cuuint64_t)g.plane * 8};
  cuuint32_t box[3] = {box0, (cuuint32_t)(kTY + 2), 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                   const_cast<double *>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_box(const Grid &g, const double *base, void *out128, unsigned box0,
                unsigned box1) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  CUtensorMap *tm = reinterpret_cast<CUtensorMap *>(out128);
  cuuint64_t dims[3] = {(cuuint64_t)g.pz, (cuuint64_t)(g.ny + 2),
                        (cuuint64_t)(g.nxl + 2)};
  cuuint64_t strides[2] = {(cuuint64_t)g.pz * 8, (cuuint64_t)g.plane * 8};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                   const_cast<double *>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_field(const Grid &g, const double *base, void *out128) {
  return encode(g, base, out128, (cuuint32_t)g.pz);
}

bool make_tmap_resid(const Grid &g, const double *base, void *out128) {
  return encode(g, base, out128, (cuuint32_t)rbox0(g));
}

// raise a kernel's dynamic shared-memory limit to `bytes` (once per size)
template <typename K>
static void set_smem(K kernel, size_t bytes, size_t *configured) {
  if (bytes > *configured) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)bytes);
    *configured = bytes;
  }
}

static int smooth_blocks(const Grid &g) {
  const int nrt = (g.ny + kTY - 1) / kTY;
  const int ich = chunk_planes(g.nxl, nrt, g.nsm);
  return nrt * ((g.nxl + ich - 1) / ich);
}

template <bool P, int NCH, int M, int NORM = 0>
static void launch_sm(const Grid &g, const Grid &c, const CUtensorMap *tm,
                      int color, double alpha, cudaStream_t s,
                      double *partials = nullptr, const double *oldv = nullptr) {
  const size_t smem = smooth_smem_bytes(g);
  static size_t configured = 0;
  set_smem(k_smooth_march<P, NCH, M, NORM>, smem, &configured);
  k_smooth_march<P, NCH, M, NORM><<<smooth_blocks(g), kThreadsM, smem, s>>>(
      g, *tm, color, c, alpha, partials, oldv);
}

template <bool P, int M, int NORM = 0>
static void launch_sm_n(const Grid &g, const Grid &c, const void *tm128,
                        int color, double alpha, cudaStream_t s,
                        double *partials = nullptr, const double *oldv = nullptr) {
  const CUtensorMap *tm = reinterpret_cast<const CUtensorMap *>(tm128);
  switch ((g.nzh + 63) >> 6) {
    case 1: launch_sm<P, 1, M, NORM>(g, c, tm, color, alpha, s, partials, oldv); break;
    case 2: launch_sm<P, 2, M, NORM>(g, c, tm, color, alpha, s, partials, oldv); break;
    case 3: launch_sm<P, 3, M, NORM>(g, c, tm, color, alpha, s, partials, oldv); break;
    default: launch_sm<P, 4, M, NORM>(g, c, tm, color, alpha, s, partials, oldv); break;
  }
}

static int variant(const Grid &g) {
  return g.codeR ? VAR_MASK : (is_periodic(g) ? VAR_PER : VAR_BOX);
}

void launch_smooth_march(const Grid &g, const void *tm_oth128, int color,
                         cudaStream_t s) {
  switch (variant(g)) {
    case VAR_MASK: launch_sm_n<false, VAR_MASK>(g, g, tm_oth128, color, 0.0, s); break;
    case VAR_PER: launch_sm_n<false, VAR_PER>(g, g, tm_oth128, color, 0.0, s); break;
    default: launch_sm_n<false, VAR_BOX>(g, g, tm_oth128, color, 0.0, s); break;
  }
}

int launch_smooth_norm_march(const Grid &g, const void *tm_oth128, int color,
                             double *partials, cudaStream_t s) {
  switch (variant(g)) {
    case VAR_MASK:
      launch_sm_n<false, VAR_MASK, 1>(g, g, tm_oth128, color, 0.0, s, partials);
      break;
    case VAR_PER:
      launch_sm_n<false, VAR_PER, 1>(g, g, tm_oth128, color, 0.0, s, partials);
      break;
    default:
      launch_sm_n<false, VAR_BOX, 1>(g, g, tm_oth128, color, 0.0, s, partials);
      break;
  }
  return smooth_blocks(g);
}

// the look-ahead red half-sweep (NORM 2): reads Phi^B (ring), f^R and the
// current Phi^R (oldv), writes the swept Phi^R to g.phiR (another buffer)
// and the red residual partials of the current iterate; box, periodic and
// masked (byte-code) grids
int launch_smooth_lookahead_march(const Grid &g, const void *tm_oth128,
                                  const double *oldv, double *partials,
                                  cudaStream_t s) {
  switch (variant(g)) {
    case VAR_MASK: launch_sm_n<false, VAR_MASK, 2>(g, g, tm_oth128, 0, 0.0, s, partials, oldv); break;
    case VAR_PER: launch_sm_n<false, VAR_PER, 2>(g, g, tm_oth128, 0, 0.0, s, partials, oldv); break;
    default: launch_sm_n<false, VAR_BOX, 2>(g, g, tm_oth128, 0, 0.0, s, partials, oldv); break;
  }
  return smooth_blocks(g);
}

void launch_prolong_smooth_march(const Grid &g, const Grid &c,
                                 const void *tm_oth128, int color, double alpha,
                                 cudaStream_t s) {
  switch (variant(g)) {
    case VAR_MASK: launch_sm_n<true, VAR_MASK>(g, c, tm_oth128, color, alpha, s); break;
    case VAR_PER: launch_sm_n<true, VAR_PER>(g, c, tm_oth128, color, alpha, s); break;
    default: launch_sm_n<true, VAR_BOX>(g, c, tm_oth128, color, alpha, s); break;
  }
}

static int resid_blocks(const Grid &g) {
  const int nzt = rntiles(g);
  const int nrt = (g.ny + kTY - 1) / kTY;
  const int ich = chunk_planes(g.nxl, nrt * nzt, g.nsm);
  const int nxc = (g.nxl + ich - 1) / ich;
  return nzt * nrt * nxc;
}

bool resid_march_supported(const Grid &g) {
  return g.nzh >= 64 && g.pz <= 256 && g.ny >= kTY && g.nxl >= 2 &&
         (g.nxl % 2) == 0 && (g.ny % 2) == 0 && get_encode() != nullptr;
}

template <int MODE, int M>
static void launch_rm(const Grid &g, const Grid &c, const void *tmR,
                      const void *tmB, double *partials, cudaStream_t s, int red0 = 0) {
  static size_t configured = 0;
  set_smem(k_resid_march<MODE, M>, resid_smem_bytes(), &configured);
  k_resid_march<MODE, M><<<resid_blocks(g), kThreadsM, resid_smem_bytes(), s>>>(
      g, *reinterpret_cast<const CUtensorMap *>(tmR),
      *reinterpret_cast<const CUtensorMap *>(tmB), c, partials, red0);
}

void launch_resid_restrict_march(const Grid &g, const Grid &c, const void *tmR,
                                 const void *tmB, cudaStream_t s, int red0) {
  switch (variant(g)) {
    case VAR_MASK: launch_rm<MODE_RESTRICT, VAR_MASK>(g, c, tmR, tmB, nullptr, s); break;
    case VAR_PER: launch_rm<MODE_RESTRICT, VAR_PER>(g, c, tmR, tmB, nullptr, s); break;
    default: launch_rm<MODE_RESTRICT, VAR_BOX>(g, c, tmR, tmB, nullptr, s, red0); break;
  }
}

int norm_march_blocks(const Grid &g) { return resid_blocks(g); }

// CTA count of the marching kernels for any SM count (x-chunks of 2 planes,
// the shortest chunk_planes picks): sizes the partial-sum buffers without a
// device query
int march_blocks_max(const Grid &g) {
  return rntiles(g) * ((g.ny + kTY - 1) / kTY) * ((g.nxl + 1) / 2);
}

int launch_norm_red_march(const Grid &g, const void *tmR, const void *tmB,
                          double *partials, cudaStream_t s) {
  switch (variant(g)) {
    case VAR_MASK: launch_rm<MODE_NORM_RED, VAR_MASK>(g, g, tmR, tmB, partials, s); break;
    case VAR_PER: launch_rm<MODE_NORM_RED, VAR_PER>(g, g, tmR, tmB, partials, s); break;
    default: launch_rm<MODE_NORM_RED, VAR_BOX>(g, g, tmR, tmB, partials, s); break;
  }
  return resid_blocks(g);
}

int launch_resid_restrict_norm_march(const Grid &g, const Grid &c, const void *tmR,
                                     const void *tmB, double *partials,
                                     cudaStream_t s, int red0) {
  switch (variant(g)) {
    case VAR_MASK: launch_rm<MODE_BOTH, VAR_MASK>(g, c, tmR, tmB, partials, s); break;
    case VAR_PER: launch_rm<MODE_BOTH, VAR_PER>(g, c, tmR, tmB, partials, s); break;
    default: launch_rm<MODE_BOTH, VAR_BOX>(g, c, tmR, tmB, partials, s, red0); break;
  }
  return resid_blocks(g);
}

void launch_norm_march(const Grid &g, const void *tmR, const void *tmB,
                       double *partials, cudaStream_t s) {
  switch (variant(g)) {
    case VAR_MASK: launch_rm<MODE_NORM, VAR_MASK>(g, g, tmR, tmB, partials, s); break;
    case VAR_PER: launch_rm<MODE_NORM, VAR_PER>(g, g, tmR, tmB, partials, s); break;
    default: launch_rm<MODE_NORM, VAR_BOX>(g, g, tmR, tmB, partials, s); break;
  }
}

}  // namespace mg
