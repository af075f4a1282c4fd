// The end of a look-ahead V-cycle on one box-domain level-0 slab in ONE
// plane-marching kernel (sm_100a): the last black post-smoothing half-sweep
// (with its residual partials, k_smooth_march<..., NORM 1>) and the
// look-ahead red half-sweep (k_smooth_march<..., NORM 2>) that follows it.
//
// Separately the two read Phi_R (ring) + f_B and write Phi_B (12 B/cell),
// then read Phi_B (ring) + f_R + Phi_R and write Phi_R' (16 B/cell).  Here
// a CTA owns TY rows of an x-chunk; the old red planes stream in through a
// TMA ring of TY + 4 rows, the new black is computed on TY + 2 rows (one
// halo row each side, redundant with the neighbouring tiles) and on one
// halo plane at each chunk end, kept in a three-plane shared-memory ring, and
// the look-ahead red of plane i - 1 is computed from it while plane i's black
// is done.  No CTA reads global black or writes global red during the
// kernel (the new black of the tile's own rows is written in place, the new
// red to the other red buffer), so the redundant halos need no
// synchronisation.  20 B/cell instead of 28.
//
// Per-cell arithmetic is exactly that of k_smooth_march (bitwise):
//     Phi_c = (f_c * w + s) / d,  r_c = f_c - c (d u - s),
//     s = ((((x- + x+) + y-) + y+) + z-) + z+.
#include <cuda.h>
#include <cuda_runtime.h>

#include "mg_internal.h"
#include "mg_tma.cuh"

namespace mg {

namespace {

constexpr int kRR = kTY + 4;  // red ring rows: j0-2 .. j0+TY+1
constexpr int kBR = kTY + 2;  // black ring rows: j0-1 .. j0+TY
constexpr int kSR = 5;        // red ring slots: planes u .. u+2 in use, 2 in flight
constexpr int kWPR = 2;                // warps per row: interleaved 64-wide chunks
constexpr int kWarps = kBR * kWPR;     // black rows; rows 1..TY also do red
constexpr int kThreadsF = kWarps * 32;

__host__ __device__ inline int rslot12(int pz) { return round128(kRR * pz * 8) / 8; }
__host__ __device__ inline int bslot10(int pz) { return kBR * pz; }

}  // namespace

template <int NCH>
__global__ void __launch_bounds__(kThreadsF, 1)
    k_black_lookahead(Grid g, const __grid_constant__ CUtensorMap tm_red12,
                      double *__restrict__ red_out, double *partials) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int pz = g.pz;
  const int rsd = rslot12(pz), bsd = bslot10(pz);
  double *rring = reinterpret_cast<double *>(smem);
  double *bring = rring + (size_t)kSR * rsd;
  unsigned long long *bars = reinterpret_cast<unsigned long long *>(bring + 3 * (size_t)bsd);
  const unsigned box_bytes = (unsigned)(kRR * pz * 8);

  const int nrt = (g.ny + kTY - 1) / kTY;
  const int ich = chunk_planes(g.nxl, nrt, g.nsm);
  const int rt = blockIdx.x % nrt;
  const int xc = blockIdx.x / nrt;
  const int j0 = rt * kTY;
  const int i0 = xc * ich;
  const int i1 = min(i0 + ich, g.nxl);
  const int nq = (i1 - i0) + 2;  // black planes i0-1 .. i1 (local q = 0 .. nq-1)
  const int nu = nq + 2;         // red planes i0-2 .. i1+1 (ring index u)
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warp = wid / kWPR, part = wid % kWPR;  // row, chunk set
  constexpr int CPW = (NCH + kWPR - 1) / kWPR;    // chunks per warp

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSR; s++) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // red plane u (global i0 - 2 + u) = array plane i0 - 1 + u, array rows
  // j0 - 1 .. j0 + TY + 2 (global rows j0 - 2 ..); out of the array: zeros
  auto issue = [&](int u) {
    const int s = u % kSR;
    mbar_expect_tx(&bars[s], box_bytes);
    tma_load_3d(rring + (size_t)s * rsd, &tm_red12, 0, j0 - 1, i0 - 1 + u, &bars[s]);
  };
  if (threadIdx.x == 0)
    for (int u = 0; u < 4 && u < nu; u++) issue(u);

  // this warp's black row jb and (warps 1..TY) red row jr = jb
  const int jb = j0 - 1 + warp;
  const bool brow = jb >= 0 && jb < g.ny;
  const bool own = warp >= 1 && warp <= kTY && jb < g.ny;
  const double *__restrict__ fB = g.fB;
  const double *__restrict__ fR = g.fR;
  double *__restrict__ phiB = g.phiB;
  // chunk cc of this warp: c = part + kWPR cc (< NCH), half-indices
  // k = 2 lane + 64 c
  auto fload = [&](const double *f, int i, int j, double2 *dst) {
#pragma unroll
    for (int cc = 0; cc < CPW; cc++) {
      const int c = part + kWPR * cc;
      const int k = 2 * lane + 64 * c;
      dst[cc] = make_double2(0.0, 0.0);
      if (c < NCH && i >= 0 && i < g.nxl && j >= 0 && j < g.ny && k < g.nzh)
        dst[cc] = *reinterpret_cast<const double2 *>(
            f + (long long)(i + 1) * g.plane + (long long)(j + 1) * pz + k);
    }
  };
  double2 fb[CPW], fr[CPW];
  fload(fB, i0 - 1, jb, fb);   // black plane q = 0
  fload(fR, i0, own ? jb : -1, fr);  // red plane i0 (q = 2)

  double nacc = 0.0;
  int waited = 0;  // red ring planes waited for
  for (int q = 0; q < nq; q++) {
    const int i = i0 - 1 + q;  // global black plane
    __syncthreads();           // ring slots of planes u = q - 1 (red), q - 3 (black) free
    if (threadIdx.x == 0 && q + 4 < nu) {
      fence_proxy_async();
      issue(q + 4);
    }
    // red planes u = q, q + 1, q + 2 (global i - 1, i, i + 1)
    for (; waited <= q + 2 && waited < nu; waited++)
      mbar_wait(&bars[waited % kSR], (waited / kSR) & 1);
    double2 fbn[CPW];
    fload(fB, i + 1, jb, fbn);
    // ---- black of plane i, row jb ----
    double *brow_out = bring + (size_t)(q % 3) * bsd + (size_t)warp * pz;
    if (brow && i >= 0 && i < g.nx) {
      const double *rc = rring + (size_t)((q + 1) % kSR) * rsd + (size_t)(warp + 1) * pz;
      const double *rxm = rring + (size_t)(q % kSR) * rsd + (size_t)(warp + 1) * pz;
      const double *rxp = rring + (size_t)((q + 2) % kSR) * rsd + (size_t)(warp + 1) * pz;
      const int p = (i + jb + 1) & 1;
      const bool store = own && q >= 1 && q <= nq - 2;
      double *orow = phiB + (long long)(i + 1) * g.plane + (long long)(jb + 1) * pz;
#pragma unroll
      for (int cc = 0; cc < CPW; cc++) {
        const int c = part + kWPR * cc;
        const int k = 2 * lane + 64 * c;
        if (c >= NCH || k >= g.nzh) continue;
        const double2 a = lds2(rxm + k);
        const double2 b = lds2(rxp + k);
        const double2 ym = lds2(rc - pz + k);
        const double2 yp = lds2(rc + pz + k);
        const double2 zc = lds2(rc + k);
        double zm0, zp0, zm1, zp1;
        if (p == 0) {
          zm0 = z_lo<false>(g, rc, k);
          zp0 = zc.x;
          zm1 = zc.x;
          zp1 = zc.y;
        } else {
          zm0 = zc.x;
          zp0 = z_hi0<false>(g, rc, k, zc.y);
          zm1 = zc.y;
          zp1 = z_hi<false>(g, rc, k);
        }
        const int z0 = 2 * k + p;
        const double s0 = ((((a.x + b.x) + ym.x) + yp.x) + zm0) + zp0;
        const double s1 = ((((a.y + b.y) + ym.y) + yp.y) + zm1) + zp1;
        const double d0 = (double)centre_dm(g, i, jb, z0);
        const double d1 = (double)centre_dm(g, i, jb, z0 + 2);
        double2 out;
        out.x = div_small(fb[cc].x * g.w + s0, d0, c_rcp16[(int)d0]);
        out.y = div_small(fb[cc].y * g.w + s1, d1, c_rcp16[(int)d1]);
        const bool two = k + 1 < g.nzh;
        if (!two) out.y = 0.0;
        *reinterpret_cast<double2 *>(brow_out + k) = out;
        if (store) {
          const double r0 = fb[cc].x - g.c * (d0 * out.x - s0);
          const double r1 = two ? fb[cc].y - g.c * (d1 * out.y - s1) : 0.0;
          nacc = nacc + r0 * r0;
          nacc = nacc + r1 * r1;
          if (two)
            *reinterpret_cast<double2 *>(orow + k) = out;
          else
            orow[k] = out.x;
        }
      }
    } else {
      // a ghost row / plane: black 0 (folded boundary)
#pragma unroll
      for (int cc = 0; cc < CPW; cc++) {
        const int c = part + kWPR * cc;
        const int k = 2 * lane + 64 * c;
        if (c < NCH && k < g.nzh)
          *reinterpret_cast<double2 *>(brow_out + k) = make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int cc = 0; cc < CPW; cc++) fb[cc] = fbn[cc];
    __syncthreads();  // black plane i complete
    // ---- look-ahead red of plane ir = i - 1 (own planes), own rows ----
    const int ir = i - 1;
    if (q >= 2) {
      double2 frn[CPW];
      fload(fR, ir + 1, own ? jb : -1, frn);
      if (own) {
        const double *bc = bring + (size_t)((q - 1) % 3) * bsd + (size_t)warp * pz;
        const double *bxm = bring + (size_t)((q - 2) % 3) * bsd + (size_t)warp * pz;
        const double *bxp = bring + (size_t)(q % 3) * bsd + (size_t)warp * pz;
        // old red of plane ir, row jb: ring plane u = q (global i0 - 2 + q = ir)
        const double *rold = rring + (size_t)(q % kSR) * rsd + (size_t)(warp + 1) * pz;
        const int p = (ir + jb) & 1;
        double *orow = red_out + (long long)(ir + 1) * g.plane + (long long)(jb + 1) * pz;
#pragma unroll
        for (int cc = 0; cc < CPW; cc++) {
          const int c = part + kWPR * cc;
          const int k = 2 * lane + 64 * c;
          if (c >= NCH || k >= g.nzh) continue;
          const double2 a = lds2(bxm + k);
          const double2 b = lds2(bxp + k);
          const double2 ym = lds2(bc - pz + k);
          const double2 yp = lds2(bc + pz + k);
          const double2 zc = lds2(bc + k);
          const double2 ov = lds2(rold + k);
          double zm0, zp0, zm1, zp1;
          if (p == 0) {
            zm0 = z_lo<false>(g, bc, k);
            zp0 = zc.x;
            zm1 = zc.x;
            zp1 = zc.y;
          } else {
            zm0 = zc.x;
            zp0 = z_hi0<false>(g, bc, k, zc.y);
            zm1 = zc.y;
            zp1 = z_hi<false>(g, bc, k);
          }
          const int z0 = 2 * k + p;
          const double s0 = ((((a.x + b.x) + ym.x) + yp.x) + zm0) + zp0;
          const double s1 = ((((a.y + b.y) + ym.y) + yp.y) + zm1) + zp1;
          const double d0 = (double)centre_dm(g, ir, jb, z0);
          const double d1 = (double)centre_dm(g, ir, jb, z0 + 2);
          double2 out;
          out.x = div_small(fr[cc].x * g.w + s0, d0, c_rcp16[(int)d0]);
          out.y = div_small(fr[cc].y * g.w + s1, d1, c_rcp16[(int)d1]);
          const bool two = k + 1 < g.nzh;
          const double r0 = fr[cc].x - g.c * (d0 * ov.x - s0);
          const double r1 = two ? fr[cc].y - g.c * (d1 * ov.y - s1) : 0.0;
          nacc = nacc + r0 * r0;
          nacc = nacc + r1 * r1;
          if (two)
            *reinterpret_cast<double2 *>(orow + k) = out;
          else
            orow[k] = out.x;
        }
      }
#pragma unroll
      for (int cc = 0; cc < CPW; cc++) fr[cc] = frn[cc];
    }
  }
  // deterministic block reduction (warp tree, warps in order)
  __shared__ double nred[kWarps];
  double v = nacc;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) nred[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int w = 0; w < kWarps; w++) sum = sum + nred[w];
    partials[blockIdx.x] = sum;
  }
}

size_t black_lookahead_smem(const Grid &g) {
  return ((size_t)kSR * rslot12(g.pz) + 3 * (size_t)bslot10(g.pz)) * 8 + kSR * 8;
}

bool black_lookahead_supported(const Grid &g) {
  return !is_periodic(g) && !g.codeR && !g.coefR && !g.c64R && g.nxl == g.nx &&
         g.nzh <= 256 && black_lookahead_smem(g) <= 220 * 1024;
}

bool make_tmap_red12(const Grid &g, const double *base, void *out128) {
  return encode_box(g, base, out128, (unsigned)g.pz, (unsigned)kRR);
}

template <int NCH>
static void launch_bl(const Grid &g, const CUtensorMap *tm, double *red_out,
                      double *partials, int blocks, cudaStream_t s) {
  const size_t smem = black_lookahead_smem(g);
  static size_t configured = 0;
  if (smem > configured) {
    cudaFuncSetAttribute(k_black_lookahead<NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    configured = smem;
  }
  k_black_lookahead<NCH><<<blocks, kThreadsF, smem, s>>>(g, *tm, red_out, partials);
}

int launch_black_lookahead(const Grid &g, const void *tm_red12, double *red_out,
                           double *partials, cudaStream_t s) {
  const int nrt = (g.ny + kTY - 1) / kTY;
  const int ich = chunk_planes(g.nxl, nrt, g.nsm);
  const int blocks = nrt * ((g.nxl + ich - 1) / ich);
  const CUtensorMap *tm = reinterpret_cast<const CUtensorMap *>(tm_red12);
  switch ((g.nzh + 63) >> 6) {
    case 1: launch_bl<1>(g, tm, red_out, partials, blocks, s); break;
    case 2: launch_bl<2>(g, tm, red_out, partials, blocks, s); break;
    case 3: launch_bl<3>(g, tm, red_out, partials, blocks, s); break;
    default: launch_bl<4>(g, tm, red_out, partials, blocks, s); break;
  }
  return blocks;
}

}  // namespace mg
