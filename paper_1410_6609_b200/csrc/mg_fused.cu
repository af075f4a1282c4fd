// Fused "last black half-sweep + residual epilogue" marching kernels (sm_100a).
//
//   k_black_resid<RESTRICT>  black half-sweep fused with the
//                            residual + 8-child averaging restriction
//                            that ends pre-smoothing
//   k_black_resid<NORM>      black half-sweep fused with the residual norm
//                            (Alg.1) that ends the cycle
//
// Saves a full pass (12 B/cell) each.  The red residual at plane q needs the
// NEW black values at planes q-1..q+1 and at rows j0-1 / j0+TY owned by the
// neighbouring CTAs, so each CTA recomputes black on a one-row and
// one-element halo (from final red, read through a 12-row TMA ring) and runs
// the residual one plane behind the black update.  Values are computed with
// exactly the expressions of the unfused kernels, so the result is bitwise
// identical.  Used on levels held whole (no slab interfaces).
#include <cuda.h>
#include <cuda_runtime.h>

#include "mg_internal.h"
#include "mg_tma.cuh"

namespace mg {

namespace {

constexpr int kRS = 6;              // red ring slots (4 planes in use + 2 ahead)
constexpr int kRRows = kTY + 4;     // red rows j0-2 .. j0+TY+1
constexpr int kBRows = kTY + 2;     // new-black rows j0-1 .. j0+TY
constexpr int kBW = kZT + 4;        // new-black row width; column of k = k-kz0+2

__host__ __device__ inline int ring_doubles(const Grid &g) {
  return round128(kRRows * rbox0(g) * 8) / 8;
}

}  // namespace

enum { FMODE_RESTRICT = 0, FMODE_NORM = 1 };

template <int MODE>
__global__ void __launch_bounds__(kThreadsM, 2)
    k_black_resid(Grid g, const __grid_constant__ CUtensorMap tmR, Grid C,
                  double *partials) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int W = rbox0(g);
  const int sd = ring_doubles(g);
  double *ring = reinterpret_cast<double *>(smem);
  double *bbuf = ring + (size_t)kRS * sd;                 // [3][kBRows][kBW]
  double *xch = bbuf + 3 * kBRows * kBW;                  // [TY/2][ZT]
  unsigned long long *bars =
      reinterpret_cast<unsigned long long *>(xch + (kTY / 2) * kZT);
  __shared__ double red_sh[kTY];
  const unsigned box_bytes = (unsigned)(kRRows * W * 8);

  const int nzt = rntiles(g);
  const int nrt = (g.ny + kTY - 1) / kTY;
  int b = blockIdx.x;
  const int zt = b % nzt;
  b /= nzt;
  const int rt = b % nrt;
  const int xc = b / nrt;
  const int ich = chunk_planes(g.nxl, nrt * nzt);
  const int kz0 = zt * kZT;
  const int c0z = rtile_c0(g, kz0);
  const int zoff = kz0 - c0z;
  const int j0 = rt * kTY;
  const int c1 = j0 > 0 ? j0 - 1 : 0;       // TMA row coordinate (array row)
  const int i0 = xc * ich;
  const int i1 = min(i0 + ich, g.nxl);
  const int rp0 = i0 >= 2 ? i0 - 2 : -1;    // first red plane in the ring
  const int rp1 = min(i1 + 1, g.nxl);       // last one (array plane <= nxl+1)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kend = min(kz0 + kZT, g.nzh);   // own elements [kz0, kend)

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRS; s++) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int lp = rp0; lp <= min(i0 + 2, rp1); lp++) {
      const int s = (lp - rp0) % kRS;
      mbar_expect_tx(&bars[s], box_bytes);
      tma_load_3d(ring + (size_t)s * sd, &tmR, c0z, c1, lp + 1, &bars[s]);
    }

  // ---- static per-thread geometry ----
  // ring / bbuf element of (local row jj, half-index k): base + row offset + k
  const int rbase = zoff - kz0;                    // ring column of k = rbase+k
  auto rrow = [&](int jj) { return (jj + 1 - c1) * W + rbase; };
  auto brow = [&](int jj) { return (jj - j0 + 1) * kBW + 2 - kz0; };
  const double w = g.w, cc = g.c;
  const int df4 = g.dface[4], df5 = g.dface[5];
  auto dz = [&](int z) { return (z == 0 ? df4 : 0) + (z == g.nz - 1 ? df5 : 0); };
  auto drow = [&](int jj) {
    return 6 + (jj == 0 ? g.dface[2] : 0) + (jj == g.ny - 1 ? g.dface[3] : 0);
  };
  // phase-1 tasks: t = warp + 8 m (t < 20): row rr = t >> 1, chunk c = t & 1
  constexpr int kTasks = kBRows * 2;
  int tj[3], tk[3], tro[3], tbo[3], tdr[3];
  bool tok[3];
#pragma unroll
  for (int m = 0; m < 3; m++) {
    const int t = warp + kTY * m;
    const int rr = t >> 1, c = t & 1;
    tj[m] = j0 - 1 + rr;
    tk[m] = kz0 + 2 * lane + 64 * c;
    tok[m] = t < kTasks && tj[m] >= 0 && tj[m] < g.ny && tk[m] < kend;
    tro[m] = t < kTasks ? rrow(tj[m]) : 0;
    tbo[m] = t < kTasks ? brow(tj[m]) : 0;
    tdr[m] = t < kTasks && tj[m] >= 0 && tj[m] < g.ny ? drow(tj[m]) : 6;
  }
  // z-halo scalar tasks (warps 4..7, lanes 0..4): h = 0..19
  const int h = (warp >= 4 && lane < 5) ? (warp - 4) * 5 + lane : -1;
  const int hj = h >= 0 ? j0 - 1 + (h >> 1) : 0;
  const int hk = h >= 0 ? ((h & 1) ? kz0 + kZT : kz0 - 1) : 0;
  const bool hok = h >= 0 && hj >= 0 && hj < g.ny && hk >= 0 && hk < g.nzh;
  const int hro = hok ? rrow(hj) : 0, hbo = h >= 0 ? brow(hj) : 0;
  const int hdr = hok ? drow(hj) : 6;
  // phase-2 row: j = j0 + warp
  const int j = j0 + warp;
  const bool jok = j < g.ny;
  const int jro = rrow(j), jbo = brow(j), jdr = jok ? drow(j) : 6;

  const double *__restrict__ fB = g.fB;
  const double *__restrict__ fR = g.fR;
  const long long pl = g.plane;
  auto goff = [&](int il, int jj) -> long long {
    return (long long)(il + 1) * pl + (long long)(jj + 1) * g.pz;
  };
  auto in_x = [&](int il) { const int i = g.x0 + il; return i >= 0 && i < g.nx; };

  // prefetch registers (one plane ahead)
  double2 fBt[3];      // phase-1 tasks, plane bq
  double fBh = 0.0;    // halo task, plane bq
  double2 fRo[2], fBo[2];  // own row, plane rq (= bq - 1)
  double2 fRn[2], fBn[2];  // own row, plane bq (next rq)
  auto load_tasks = [&](int il) {
    const bool ok = in_x(il);
#pragma unroll
    for (int m = 0; m < 3; m++) {
      fBt[m] = make_double2(0.0, 0.0);
      if (ok && tok[m])
        fBt[m] = *reinterpret_cast<const double2 *>(fB + goff(il, tj[m]) + tk[m]);
    }
    fBh = (ok && hok) ? fB[goff(il, hj) + hk] : 0.0;
  };
  auto load_own = [&](int il, double2 *r, double2 *bb) {
    const bool ok = in_x(il) && jok;
#pragma unroll
    for (int c = 0; c < 2; c++) {
      const int k = kz0 + 2 * lane + 64 * c;
      r[c] = bb[c] = make_double2(0.0, 0.0);
      if (ok && k < kend) {
        r[c] = *reinterpret_cast<const double2 *>(fR + goff(il, j) + k);
        bb[c] = *reinterpret_cast<const double2 *>(fB + goff(il, j) + k);
      }
    }
  };
  load_tasks(i0 - 1);
  fRo[0] = fRo[1] = fBo[0] = fBo[1] = make_double2(0.0, 0.0);

  double acc = 0.0;
  double sdx0[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  int sq = (i0 - 1 - rp0) % kRS;  // ring slot of plane bq
  int bm = ((i0 - 1) % 3 + 3) % 3;  // bbuf slot of plane bq

  for (int bq = i0 - 1; bq <= i1; bq++) {
    __syncthreads();  // previous step done: bbuf slot of bq and ring slot of bq-3 free
    if (threadIdx.x == 0 && bq + 3 <= rp1 && bq + 3 > min(i0 + 2, rp1)) {
      fence_proxy_async();
      const int s = (sq + 3) % kRS;
      mbar_expect_tx(&bars[s], box_bytes);
      tma_load_3d(ring + (size_t)s * sd, &tmR, c0z, c1, bq + 4, &bars[s]);
    }
    if (bq == i0 - 1) {
      for (int lp = rp0; lp <= bq + 1; lp++) {
        const int r = lp - rp0;
        mbar_wait(&bars[r % kRS], (r / kRS) & 1);
      }
    } else if (bq + 1 <= rp1) {
      const int r = bq + 1 - rp0;
      mbar_wait(&bars[r % kRS], (r / kRS) & 1);
    }
    const double *Rc = ring + (size_t)sq * sd;                          // bq
    const double *Rp = ring + (size_t)((sq + 1) % kRS) * sd;            // bq+1
    const double *Rm = ring + (size_t)((sq + kRS - 1) % kRS) * sd;      // bq-1
    const double *Rmm = ring + (size_t)((sq + kRS - 2) % kRS) * sd;     // bq-2
    double *Bc = bbuf + (size_t)bm * kBRows * kBW;                       // bq
    const double *Bm = bbuf + (size_t)((bm + 2) % 3) * kBRows * kBW;     // bq-1
    const double *Bmm = bbuf + (size_t)((bm + 1) % 3) * kBRows * kBW;    // bq-2
    load_own(bq, fRn, fBn);  // own-row f of plane bq (residual of next step)

    // ---- phase 1: new black at plane bq, rows j0-1 .. j0+TY, z halo ----
    const int ib = g.x0 + bq;
    const bool plane_ok = ib >= 0 && ib < g.nx;
    const int dpl = (ib == 0 ? g.dface[0] : 0) + (ib == g.nx - 1 ? g.dface[1] : 0);
    const bool own_plane = bq >= i0 && bq < i1;
#pragma unroll
    for (int m = 0; m < 3; m++) {
      if (warp + kTY * m >= kTasks) continue;
      const int k = tk[m];
      double2 out = make_double2(0.0, 0.0);
      if (plane_ok && tok[m]) {
        const int jj = tj[m];
        const int p = (ib + jj + 1) & 1;  // black cells at z = 2k + p
        const double *cur = Rc + tro[m];
        const double2 a = lds2(Rm + tro[m] + k);
        const double2 bb = lds2(Rp + tro[m] + k);
        const double2 ym = lds2(cur - W + k);
        const double2 yp = lds2(cur + W + k);
        const double2 zc = lds2(cur + k);
        double zm0, zp0, zm1, zp1;
        if (p == 0) {
          zm0 = (k > 0) ? cur[k - 1] : 0.0;
          zp0 = zc.x;
          zm1 = zc.x;
          zp1 = zc.y;
        } else {
          zm0 = zc.x;
          zp0 = zc.y;
          zm1 = zc.y;
          zp1 = (k + 2 < g.nzh) ? cur[k + 2] : 0.0;
        }
        const double s0 = ((((a.x + bb.x) + ym.x) + yp.x) + zm0) + zp0;
        const double s1 = ((((a.y + bb.y) + ym.y) + yp.y) + zm1) + zp1;
        const int z0 = 2 * k + p;
        // exact division (bitwise IEEE) with the constant-memory RN(1/d)
        const int i0d = tdr[m] + dpl + dz(z0), i1d = tdr[m] + dpl + dz(z0 + 2);
        out.x = div_small(fBt[m].x * w + s0, (double)i0d, c_rcp16[i0d]);
        out.y = (k + 1 < g.nzh) ? div_small(fBt[m].y * w + s1, (double)i1d, c_rcp16[i1d])
                                : 0.0;
        if (own_plane && jj >= j0 && jj < j0 + kTY) {
          double *dst = g.phiB + goff(bq, jj);
          if (k + 1 < g.nzh)
            *reinterpret_cast<double2 *>(dst + k) = out;
          else
            dst[k] = out.x;
        }
      }
      *reinterpret_cast<double2 *>(Bc + tbo[m] + k) = out;
    }
    if (h >= 0) {  // z-halo element (the other z-tile's edge), 0 outside
      double v = 0.0;
      if (plane_ok && hok) {
        const int p = (ib + hj + 1) & 1;
        const int z = 2 * hk + p;
        const double *cur = Rc + hro;
        const double zm = (z > 0) ? cur[hk - 1 + p] : 0.0;
        const double zp = (z < g.nz - 1) ? cur[hk + p] : 0.0;
        const double s = ((((Rm[hro + hk] + Rp[hro + hk]) + cur[hk - W]) +
                           cur[hk + W]) +
                          zm) +
                         zp;
        const int di = hdr + dpl + dz(z);
        v = div_small(fBh * w + s, (double)di, c_rcp16[di]);
      }
      Bc[hbo + hk] = v;
    }
    load_tasks(bq + 1);  // phase-1 f_B of the next plane
    __syncthreads();     // new black of plane bq complete

    // ---- phase 2: residuals at plane rq = bq - 1, own row j0 + warp ----
    const int rq = bq - 1;
    double pr[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const bool do_res = rq >= i0 && rq < i1;
    if (do_res && jok) {
      const int i = g.x0 + rq;
      const int pR = (i + j) & 1, pB = pR ^ 1;
      const int dpr = (i == 0 ? g.dface[0] : 0) + (i == g.nx - 1 ? g.dface[1] : 0) + jdr;
#pragma unroll
      for (int c = 0; c < 2; c++) {
        const int k = kz0 + 2 * lane + 64 * c;
        if (k >= kend) continue;
        double r0, r1, q0, q1;
        {  // red: own red (ring, plane rq), neighbours new black
          const double *bc = Bm + jbo;
          const double2 a = lds2(Bmm + jbo + k);
          const double2 bb = lds2(Bc + jbo + k);
          const double2 ym = lds2(bc - kBW + k);
          const double2 yp = lds2(bc + kBW + k);
          const double2 zc = lds2(bc + k);
          double zm0, zp0, zm1, zp1;
          if (pR == 0) {
            zm0 = (k > 0) ? bc[k - 1] : 0.0;
            zp0 = zc.x;
            zm1 = zc.x;
            zp1 = zc.y;
          } else {
            zm0 = zc.x;
            zp0 = zc.y;
            zm1 = zc.y;
            zp1 = (k + 2 < g.nzh) ? bc[k + 2] : 0.0;
          }
          const double s0 = ((((a.x + bb.x) + ym.x) + yp.x) + zm0) + zp0;
          const double s1 = ((((a.y + bb.y) + ym.y) + yp.y) + zm1) + zp1;
          const double2 u = lds2(Rm + jro + k);
          const int z0 = 2 * k + pR;
          const double d0 = (double)(dpr + dz(z0));
          const double d1 = (double)(dpr + dz(z0 + 2));
          const double t0 = d0 * u.x - s0;
          const double t1 = d1 * u.y - s1;
          r0 = fRo[c].x - cc * t0;
          r1 = (k + 1 < g.nzh) ? fRo[c].y - cc * t1 : 0.0;
        }
        {  // black: own new black (bbuf, plane rq), neighbours red (ring)
          const double *cur = Rm + jro;
          const double2 a = lds2(Rmm + jro + k);
          const double2 bb = lds2(Rc + jro + k);
          const double2 ym = lds2(cur - W + k);
          const double2 yp = lds2(cur + W + k);
          const double2 zc = lds2(cur + k);
          double zm0, zp0, zm1, zp1;
          if (pB == 0) {
            zm0 = (k > 0) ? cur[k - 1] : 0.0;
            zp0 = zc.x;
            zm1 = zc.x;
            zp1 = zc.y;
          } else {
            zm0 = zc.x;
            zp0 = zc.y;
            zm1 = zc.y;
            zp1 = (k + 2 < g.nzh) ? cur[k + 2] : 0.0;
          }
          const double s0 = ((((a.x + bb.x) + ym.x) + yp.x) + zm0) + zp0;
          const double s1 = ((((a.y + bb.y) + ym.y) + yp.y) + zm1) + zp1;
          const double2 u = lds2(Bm + jbo + k);
          const int z0 = 2 * k + pB;
          const double d0 = (double)(dpr + dz(z0));
          const double d1 = (double)(dpr + dz(z0 + 2));
          const double t0 = d0 * u.x - s0;
          const double t1 = d1 * u.y - s1;
          q0 = fBo[c].x - cc * t0;
          q1 = (k + 1 < g.nzh) ? fBo[c].y - cc * t1 : 0.0;
        }
        if (MODE == FMODE_NORM) {
          acc = acc + r0 * r0;
          acc = acc + r1 * r1;
          acc = acc + q0 * q0;
          acc = acc + q1 * q1;
        } else {
          pr[c][0] = r0 + q0;
          pr[c][1] = r1 + q1;
        }
      }
    }
    if (MODE == FMODE_RESTRICT && do_res) {
      if (warp & 1) {
#pragma unroll
        for (int c = 0; c < 2; c++) {
          const int kl = 2 * lane + 64 * c;
          *reinterpret_cast<double2 *>(xch + (warp >> 1) * kZT + kl) =
              make_double2(pr[c][0], pr[c][1]);
        }
      }
      __syncthreads();
      if (!(warp & 1) && jok) {
        const bool odd_plane = (rq & 1);
        const int J = j >> 1;
        const int I = (g.x0 + rq) >> 1;
#pragma unroll
        for (int c = 0; c < 2; c++) {
          const int kl = 2 * lane + 64 * c;
          const int k = kz0 + kl;
          if (k >= kend) continue;
          const double2 o = lds2(xch + (warp >> 1) * kZT + kl);
          const double s0 = pr[c][0] + o.x;
          const double s1 = pr[c][1] + o.y;
          if (!odd_plane) {
            sdx0[c][0] = s0;
            sdx0[c][1] = s1;
          } else {
            const long long cb = (long long)(I - C.x0 + 1) * C.plane +
                                 (long long)(J + 1) * C.pz + (k >> 1);
            const int ccol = (I + J + k) & 1;
            (ccol ? C.fB : C.fR)[cb] = 0.125 * (sdx0[c][0] + s0);
            if (k + 1 < g.nzh) (ccol ? C.fR : C.fB)[cb] = 0.125 * (sdx0[c][1] + s1);
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 2; c++) {
      fRo[c] = fRn[c];
      fBo[c] = fBn[c];
    }
    sq = (sq + 1 == kRS) ? 0 : sq + 1;
    bm = (bm + 1 == 3) ? 0 : bm + 1;
  }
  if (MODE == FMODE_NORM) {
    double v = acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red_sh[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int ww = 0; ww < kTY; ww++) s = s + red_sh[ww];
      partials[blockIdx.x] = s;
    }
  }
}

// ---- host side ----------------------------------------------------------------
static size_t fused_smem_bytes(const Grid &g) {
  return (size_t)kRS * ring_doubles(g) * 8 + (size_t)3 * kBRows * kBW * 8 +
         (size_t)(kTY / 2) * kZT * 8 + kRS * 8;
}

bool fused_supported(const Grid &g) {
  // whole levels only (no slab interface), same tile rules as the residual
  // kernels, and the smem budget of 2 CTAs per SM
  return g.x0 == 0 && g.nxl == g.nx && resid_march_supported(g) &&
         fused_smem_bytes(g) <= 112 * 1024;
}

bool make_tmap_red12(const Grid &g, const double *base, void *out128) {
  return encode_box(g, base, out128, (unsigned)rbox0(g), (unsigned)kRRows);
}

static int fused_blocks(const Grid &g) {
  const int nzt = rntiles(g);
  const int nrt = (g.ny + kTY - 1) / kTY;
  const int ich = chunk_planes(g.nxl, nrt * nzt);
  return nzt * nrt * ((g.nxl + ich - 1) / ich);
}

template <int MODE>
static void launch_fused(const Grid &g, const Grid &c, const void *tm,
                         double *partials, cudaStream_t s) {
  const size_t smem = fused_smem_bytes(g);
  static size_t configured = 0;
  if (smem > configured) {
    cudaFuncSetAttribute(k_black_resid<MODE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  k_black_resid<MODE><<<fused_blocks(g), kThreadsM, smem, s>>>(
      g, *reinterpret_cast<const CUtensorMap *>(tm), c, partials);
}

void launch_black_restrict(const Grid &g, const Grid &c, const void *tm_red12,
                           cudaStream_t s) {
  launch_fused<FMODE_RESTRICT>(g, c, tm_red12, nullptr, s);
}

int launch_black_norm(const Grid &g, const void *tm_red12, double *partials,
                      cudaStream_t s) {
  launch_fused<FMODE_NORM>(g, g, tm_red12, partials, s);
  return fused_blocks(g);
}

}  // namespace mg
