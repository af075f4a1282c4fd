// Coulomb force on charged spheres (Eq.14) with the isotropic
// D3Q19 gradient (Eq.15) -- SURVEY §8(f) N2, the step after the
// potential solve in Alg.1.
//
//   grad Phi(x_b) = (1/w_1) sum_{q=2..19} w_q Phi(x_b + e_q) e_q / dx^2,
//   w_1 = 1/3, faces 1/18, edges 1/36; per component
//   S = sum_q w_q c_q Phi_q in a fixed order, g = (3 S) / h.
//   Reading d6: D3Q19 where all 18 neighbours are fluid cells of
//   the domain, else per axis central / one-sided differences.
//   F_p = -h^3 sum_b grad Phi(x_b) rho_p(x_b), rho_p the sphere's own
//   (subsampled) charge density with the RHS mapping's expressions.
// One CTA per sphere: the covered sub-cell count of the whole domain (given
// by the RHS of the same step, or counted here), the per-cell counts of the
// sphere's box in shared memory (x intervals, mg_sphere.cuh), then the slab's
// sum -- on interior boxes in adjoint form over a shell of cells (reading
// d13, adjoint_force_shell), else cell by cell with the gradient of reading
// d6; per-slab partial sums, summed on the host in slab / rank order.
#include <cuda_runtime.h>

#include "mg_internal.h"
#include "mg_sphere.cuh"

namespace mg {

namespace {

constexpr int kTF = 256;

// D3Q19 directions e_q (q = 2..19 of Eq.15, rest direction omitted), as a
// constexpr function so that the unrolled loops fold every component
__host__ __device__ constexpr int kq(int q, int a) {
  const int t[18][3] = {
      {1, 0, 0},  {-1, 0, 0}, {0, 1, 0},   {0, -1, 0}, {0, 0, 1},  {0, 0, -1},
      {1, 1, 0},  {-1, -1, 0}, {1, -1, 0}, {-1, 1, 0}, {1, 0, 1},  {-1, 0, -1},
      {1, 0, -1}, {-1, 0, 1}, {0, 1, 1},   {0, -1, -1}, {0, 1, -1}, {0, -1, 1}};
  return t[q][a];
}

__device__ __forceinline__ int wrapi(int i, int n, int per) {
  return !per ? i : (i < 0 ? i + n : (i >= n ? i - n : i));
}

// fluid cell of the (global) domain?  solid: global natural-layout mask or
// null.  Periodic axes: the opposite side's cell.
__device__ __forceinline__ bool valid_cell(const Grid &g, const unsigned char *solid,
                                           int i, int j, int k) {
  i = wrapi(i, g.nx, g.per[0]);
  j = wrapi(j, g.ny, g.per[1]);
  k = wrapi(k, g.nz, g.per[2]);
  if (i < 0 || j < 0 || k < 0 || i >= g.nx || j >= g.ny || k >= g.nz) return false;
  return !solid || solid[((long long)i * g.ny + j) * g.nz + k] == 0;
}

// level-0 Phi at global cell (i, j, k) held by this slab (incl. ghost planes:
// an x index one past the slab is its ghost plane, which on a periodic x
// axis holds the opposite side's plane; y and z wrap explicitly)
__device__ __forceinline__ double phi_at(const Grid &g, int i, int j, int k) {
  j = wrapi(j, g.ny, g.per[1]);
  k = wrapi(k, g.nz, g.per[2]);
  const int iw = wrapi(i, g.nx, g.per[0]);  // colour of the cell it mirrors
  const long long e = (long long)(i - g.x0 + 1) * g.plane +
                      (long long)(j + 1) * g.pz + (k >> 1);
  return (((iw + j + k) & 1) ? g.phiB : g.phiR)[e];
}

// LD(i, j, k): Phi at a global cell
template <class LD>
__device__ __forceinline__ void gradient(const Grid &g, const unsigned char *solid,
                                         double h, int i, int j, int k, double *gr,
                                         const LD &ld) {
  bool all = true;
#pragma unroll
  for (int q = 0; q < 18; q++)
    all = all && valid_cell(g, solid, i + kq(q, 0), j + kq(q, 1), k + kq(q, 2));
  if (all) {
    // per component the oracle's sum S_a = sum_q (+-) w_q Phi_q in the fixed
    // q order (terms with c_q = 0 skipped): each neighbour is loaded once and
    // added to the components it contributes to, in q order per component
    double S[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 18; q++) {
      const double v = ld(i + kq(q, 0), j + kq(q, 1), k + kq(q, 2));
      const double w = q < 6 ? 1.0 / 18.0 : 1.0 / 36.0;
#pragma unroll
      for (int a = 0; a < 3; a++) {
        const int c = kq(q, a);
        if (c == 0) continue;
        S[a] = c > 0 ? S[a] + w * v : S[a] - w * v;
      }
    }
#pragma unroll
    for (int a = 0; a < 3; a++) gr[a] = (3.0 * S[a]) / h;
    return;
  }
  const double c0 = ld(i, j, k);
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const int pi = i + (a == 0), pj = j + (a == 1), pk = k + (a == 2);
    const int mi = i - (a == 0), mj = j - (a == 1), mk = k - (a == 2);
    const bool vp = valid_cell(g, solid, pi, pj, pk);
    const bool vm = valid_cell(g, solid, mi, mj, mk);
    if (vp && vm)
      gr[a] = (ld(pi, pj, pk) - ld(mi, mj, mk)) / (2.0 * h);
    else if (vp)
      gr[a] = (ld(pi, pj, pk) - c0) / h;
    else if (vm)
      gr[a] = (c0 - ld(mi, mj, mk)) / h;
    else
      gr[a] = 0.0;
  }
}

// The all-valid D3Q19 gradient of gradient() for a cell whose 18 neighbours
// are known to be fluid cells of the domain (no mask, no periodic wrap, box
// inside the level): the same loads in the same q order, addressed directly
// in the split layout (neighbour colour = own colour ^ parity of the offset).
__device__ __forceinline__ void gradient_interior(const Grid &g, double h, int i,
                                                  int j, int k, double *gr) {
  const long long base = (long long)(i - g.x0 + 1) * g.plane + (long long)(j + 1) * g.pz;
  const int c0 = (i + j + k) & 1;
  // same-colour neighbours (offset parity even) in the own array, the others
  // in the other one: two row pointers, no per-load colour select
  const double *own = (c0 ? g.phiB : g.phiR) + base;
  const double *oth = (c0 ? g.phiR : g.phiB) + base;
  const long long P = g.plane, Z = g.pz;
  const int kh0 = k >> 1;
  // half-index of z + dk relative to the row: (k + dk) >> 1
  const int khm = (k - 1) >> 1, khp = (k + 1) >> 1;
  double S[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int q = 0; q < 18; q++) {
    const int di = kq(q, 0), dj = kq(q, 1), dk = kq(q, 2);
    const double *arr = ((di + dj + dk) & 1) ? oth : own;
    const int kh = dk < 0 ? khm : (dk > 0 ? khp : kh0);
    const double v = arr[di * P + dj * Z + kh];
    const double w = q < 6 ? 1.0 / 18.0 : 1.0 / 36.0;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const int c = kq(q, a);
      if (c == 0) continue;
      S[a] = c > 0 ? S[a] + w * v : S[a] - w * v;
    }
  }
#pragma unroll
  for (int a = 0; a < 3; a++) gr[a] = (3.0 * S[a]) / h;
}

__device__ __forceinline__ double bsum(double v, double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); w++) s = s + sh[w];
  __syncthreads();
  return s;
}

// the three force components reduced together (one barrier pair), each in
// the fixed warp-shuffle tree + warp order of bsum
__device__ __forceinline__ void bsum3(double *v, double (*sh)[32]) {
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[a] += __shfl_down_sync(0xffffffffu, v[a], o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0)
    for (int a = 0; a < 3; a++) sh[a][wid] = v[a];
  __syncthreads();
  for (int a = 0; a < 3; a++) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) s = s + sh[a][w];
    v[a] = s;
  }
}

}  // namespace

// padded per-cell counts of one box image (2 rim cells per side)
constexpr int kPad = 12288;

// The K stencil at padded index idx (see adjoint_force below).
__device__ __forceinline__ void k_stencil(const unsigned short *q, int X, int Y, int &kx,
                                          int &ky, int &kz) {
  kx = 2 * ((int)q[-X] - (int)q[X]);
  ky = 2 * ((int)q[-Y] - (int)q[Y]);
  kz = 2 * ((int)q[-1] - (int)q[1]);
  int e;
  e = q[-X - Y]; kx += e; ky += e;
  e = q[-X + Y]; kx += e; ky -= e;
  e = q[X - Y];  kx -= e; ky += e;
  e = q[X + Y];  kx -= e; ky -= e;
  e = q[-X - 1]; kx += e; kz += e;
  e = q[-X + 1]; kx += e; kz -= e;
  e = q[X - 1];  kx -= e; kz += e;
  e = q[X + 1];  kx -= e; kz -= e;
  e = q[-Y - 1]; ky += e; kz += e;
  e = q[-Y + 1]; ky += e; kz -= e;
  e = q[Y - 1];  ky -= e; kz += e;
  e = q[Y + 1];  ky -= e; kz -= e;
}

// The force of one sphere image over an interior box (every cell of the box
// and its D3Q19 neighbours inside the level, no mask, no wrap) in adjoint
// form.  The gradient is linear in Phi, so
//   sum_b c_b S_a(b) = sum_b c_b sum_q w_q e_qa Phi(b + e_q)
//                    = (1/36) sum_y Phi(y) K_a(y),
//   K_a(y) = sum_q m_q e_qa c(y - e_q),  m = 2 (faces), 1 (edges),
// an integer stencil of the covered counts c (exact).  K vanishes wherever
// the 3^3 neighbourhood is uniformly covered or empty, so only the cells of
// a shell around the sphere surface load Phi -- once each, instead of once
// per covered neighbour.  cc: the counts on the padded box, x planes outside
// [xa, xb] zero.  Returns sum_y Phi(y) K_a(y) per component (the caller
// scales by (3 / h) (1 / 36) rho_per_count); the sum is reordered against
// the oracle's cell-by-cell one (rounding only).
__device__ __forceinline__ void adjoint_force(const Grid &g, const sph::Box &bx, int xa,
                                              int xb, const unsigned short *cc, double *G) {
  const int Q2 = bx.n[2] + 4, Q1 = bx.n[1] + 4;
  const int X = Q1 * Q2, Y = Q2;
  const int nv = bx.n[1] + 2, nw = bx.n[2] + 2, nu = xb - xa + 3;
  const int tot = nu * nv * nw;
  // thread t's cell (uo, v, w) of the rim box, advanced by blockDim.x per
  // step with carries (no division in the loop)
  const int B = blockDim.x;
  const int dw = B % nw, dv = (B / nw) % nv, du = B / (nw * nv);
  int w = threadIdx.x % nw, v = (threadIdx.x / nw) % nv, uo = threadIdx.x / (nw * nv);
  const int u0 = xa - bx.lo[0] - 1;
  double g0 = 0.0, g1 = 0.0, g2 = 0.0;  // (registers, added to G at the end)
  for (int t = threadIdx.x; t < tot; t += B) {
    const int u = u0 + uo;
    const int idx = ((u + 2) * Q1 + v + 1) * Q2 + w + 1;
    int kx, ky, kz;
    k_stencil(cc + idx, X, Y, kx, ky, kz);
    if ((kx | ky | kz) != 0) {
      const int i = bx.lo[0] + u, j = bx.lo[1] + v - 1, k = bx.lo[2] + w - 1;
      const long long o = (long long)(i - g.x0 + 1) * g.plane + (long long)(j + 1) * g.pz +
                          (k >> 1);
      const double phi = (((i + j + k) & 1) ? g.phiB : g.phiR)[o];
      g0 = g0 + phi * (double)kx;
      g1 = g1 + phi * (double)ky;
      g2 = g2 + phi * (double)kz;
    }
    w += dw;
    if (w >= nw) { w -= nw; v++; }
    v += dv;
    if (v >= nv) { v -= nv; uo++; }
    uo += du;
  }
  G[0] = G[0] + g0;
  G[1] = G[1] + g1;
  G[2] = G[2] + g2;
}

constexpr int kShellRounds = 4;  // column rounds of the shell list (ncol <= 4 blockDim)

// Shell form of adjoint_force: K(y) vanishes unless y lies within one cell
// of a covered cell and not amid full ones, so the rim-box columns first
// mark their candidate cells -- from per-column bit masks of the covered
// (cm) and fully covered (fm) cells of the 3 x 3 neighbouring columns --
// and append them to a shared list (warp scans + per-warp totals: a fixed
// order), which the block then works through evenly.  cm / fm: per padded column ((n1 + 2) x (n2 + 2),
// rim columns zero), bit ci + 1 for box cell ci.  Returns false (nothing
// accumulated) when the list would not fit; the caller then runs
// adjoint_force.
__device__ __forceinline__ bool adjoint_force_shell(const Grid &g, const sph::Box &bx,
                                                    const unsigned short *cc,
                                                    const unsigned *cm, const unsigned *fm,
                                                    unsigned *list, int cap, int *wsum,
                                                    double *G) {
  const int Q2 = bx.n[2] + 4, Q1 = bx.n[1] + 4;
  const int X = Q1 * Q2, Y = Q2;
  const int nv = bx.n[1] + 2, nw = bx.n[2] + 2, ncol = nv * nw;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  // up to kShellRounds column rounds; list order = (round, warp, lane,
  // bit): a deterministic order, so the sums are reproducible
  unsigned need[kShellRounds];
  int excl[kShellRounds];
#pragma unroll
  for (int r = 0; r < kShellRounds; r++) {
    const int t = r * blockDim.x + threadIdx.x;
    need[r] = 0;
    if (t < ncol) {
      const int v = t / nw, w = t - v * nw;
      unsigned any = 0, all = ~0u;
#pragma unroll
      for (int dv = -1; dv <= 1; dv++)
#pragma unroll
        for (int dw = -1; dw <= 1; dw++) {
          const int vv = v + dv, ww = w + dw;
          if (vv < 0 || vv >= nv || ww < 0 || ww >= nw) {
            all = 0;
            continue;
          }
          const unsigned c = cm[vv * nw + ww], f = fm[vv * nw + ww];
          any |= c | (c << 1) | (c >> 1);
          all &= f & (f << 1) & (f >> 1);
        }
      need[r] = any & ~all;
    }
    const int cnt = __popc(need[r]);
    int incl = cnt;  // warp inclusive scan of the counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    excl[r] = incl - cnt;
    if (lane == 31) wsum[r * nwarp + wid] = incl;
  }
  __syncthreads();
  int L = 0;
  for (int k = 0; k < kShellRounds * nwarp; k++) L += wsum[k];
  if (L > cap) return false;  // (block-uniform)
#pragma unroll
  for (int r = 0; r < kShellRounds; r++) {
    const int t = r * blockDim.x + threadIdx.x;
    int base = excl[r];
    for (int k = 0; k < r * nwarp + wid; k++) base += wsum[k];
    const int v = t / nw, w = t - v * nw;
    unsigned nd = need[r];
    while (nd) {
      const int b = __ffs(nd) - 1;  // bit b: box-relative x index b - 1
      nd &= nd - 1;
      list[base++] = (unsigned)(((b + 1) * Q1 + v + 1) * Q2 + w + 1) | ((unsigned)b << 14) |
                     ((unsigned)v << 19) | ((unsigned)w << 24);
    }
  }
  __syncthreads();
  double g0 = 0.0, g1 = 0.0, g2 = 0.0;
  for (int t = threadIdx.x; t < L; t += blockDim.x) {
    const unsigned e = list[t];
    int kx, ky, kz;
    k_stencil(cc + (e & 0x3fffu), X, Y, kx, ky, kz);
    if ((kx | ky | kz) == 0) continue;
    const int i = bx.lo[0] + (int)((e >> 14) & 31u) - 1;
    const int j = bx.lo[1] + (int)((e >> 19) & 31u) - 1;
    const int k = bx.lo[2] + (int)((e >> 24) & 31u) - 1;
    const long long o = (long long)(i - g.x0 + 1) * g.plane + (long long)(j + 1) * g.pz +
                        (k >> 1);
    const double phi = (((i + j + k) & 1) ? g.phiB : g.phiR)[o];
    g0 = g0 + phi * (double)kx;
    g1 = g1 + phi * (double)ky;
    g2 = g2 + phi * (double)kz;
  }
  G[0] = G[0] + g0;
  G[1] = G[1] + g1;
  G[2] = G[2] + g2;
  return true;
}

// counts: the global covered sub-cell count of each sphere if already known
// (the RHS kernel of the same step, same subsampling), else null
// 4 CTAs per SM: the per-sphere CTAs are latency-bound, so residency beats
// registers
// PER: periodic images (up to 27); otherwise the sphere itself only, without
// the 27-entry image array (registers / stack of the common case)
template <bool PER>
__global__ void __launch_bounds__(kTF, 4)
    k_coulomb(Grid g, const unsigned char *solid, double h, int s,
              const double *sph, int normalization, double *part,
              const unsigned long long *counts) {
  __shared__ double sh[32];
  __shared__ sph::Tab tab;
  __shared__ unsigned short cc[kPad];
  __shared__ int wsum[kShellRounds * (kTF / 32)];
  const int p = blockIdx.x;
  const double R = sph[5 * p + 3], Q = sph[5 * p + 4];
  const double R2 = R * R;
  const double hs = h / (double)s;
  double img[PER ? 27 : 1][3];
  int nimg = 1;
  if (PER) {
    nimg = sph::images(g, h, sph[5 * p], sph[5 * p + 1], sph[5 * p + 2],
                       reinterpret_cast<double(*)[3]>(img));
  } else {
    img[0][0] = sph[5 * p];
    img[0][1] = sph[5 * p + 1];
    img[0][2] = sph[5 * p + 2];
  }
  long long cnt = 0;  // the sphere's covered sub-cells of the whole domain
  for (int m = 0; !counts && m < nimg; m++) {
    const sph::Box bx = sph::box_of(g, h, img[m], R);
    if (bx.cells() == 0) continue;
    if (sph::tables(tab, bx, s, hs, img[m])) {
      cnt += sph::image_count(tab, bx, s, R2);
      continue;
    }
    const int ncol = bx.n[1] * bx.n[2];
    for (int col = threadIdx.x; col < ncol; col += blockDim.x) {
      const int cj = col / bx.n[2], ck = col % bx.n[2];
      for (int ci = 0; ci < bx.n[0]; ci++)
        cnt += sph::sub_count(bx.lo[0] + ci, bx.lo[1] + cj, bx.lo[2] + ck, s, hs,
                              img[m][0], img[m][1], img[m][2], R);
    }
  }
  const double np = counts ? (double)counts[p] : bsum((double)cnt, sh);
  double F[3] = {0.0, 0.0, 0.0}, G[3] = {0.0, 0.0, 0.0};
  const bool any = np > 0.0 || normalization == 1;
  const double rho0 = Q / ((4.0 / 3.0) * 3.14159265358979323846 * (R * R * R));
  for (int m = 0; any && m < nimg; m++) {
    const sph::Box bx = sph::box_of(g, h, img[m], R);
    const int xa = bx.lo[0] > g.x0 ? bx.lo[0] : g.x0;
    const int xb = min(bx.lo[0] + bx.n[0] - 1, g.x0 + g.nxl - 1);
    if (bx.cells() == 0 || xa > xb) continue;
    const int Q1 = bx.n[1] + 4, Q2 = bx.n[2] + 4;
    const bool tb = sph::tables(tab, bx, s, hs, img[m]) &&
                    (long long)(bx.n[0] + 4) * Q1 * Q2 <= kPad;
    // every cell of this box (and its D3Q19 neighbours) inside the level,
    // no mask, no wrap: the adjoint form applies
    const bool interior = !solid && !is_periodic(g) && xa - 1 >= 0 && xb + 1 < g.nx &&
                          bx.lo[1] - 1 >= 0 && bx.lo[1] + bx.n[1] < g.ny &&
                          bx.lo[2] - 1 >= 0 && bx.lo[2] + bx.n[2] < g.nz;
    const int ncol = bx.n[1] * bx.n[2];
    if (tb) {  // the slab's covered counts on the padded box
      // the shell form's column masks after the padded counts (u32-aligned)
      const int pv = ((bx.n[0] + 4) * Q1 * Q2 + 1) & ~1;
      const int nv = bx.n[1] + 2, nw = bx.n[2] + 2;
      const bool shell = interior && bx.n[0] <= 30 && nv <= 32 && nw <= 32 &&
                         nv * nw <= kShellRounds * (int)blockDim.x &&
                         pv + 4 * nv * nw <= kPad;
      unsigned *cm = reinterpret_cast<unsigned *>(cc + pv), *fm = cm + nv * nw;
      if (interior) {
        const int nz = shell ? pv + 4 * nv * nw : (bx.n[0] + 4) * Q1 * Q2;
        for (int e = threadIdx.x; e < nz; e += blockDim.x) cc[e] = 0;
        __syncthreads();
      }
      const int s3 = s * s * s;
      for (int col = threadIdx.x; col < ncol; col += blockDim.x) {
        const int cj = col / bx.n[2], ck = col % bx.n[2];
        const int base = (2 * Q1 + cj + 2) * Q2 + ck + 2;
        sph::column_counts(tab, bx, s, R2, cj, ck, cc, base, Q1 * Q2, xa - bx.lo[0],
                           xb - bx.lo[0]);
        if (shell) {  // (the thread's own column)
          unsigned c = 0, f = 0;
          for (int ci = 0; ci < bx.n[0]; ci++) {
            const int v = cc[base + ci * Q1 * Q2];
            c |= (v > 0 ? 2u : 0u) << ci;
            f |= (v == s3 ? 2u : 0u) << ci;
          }
          cm[(cj + 1) * nw + ck + 1] = c;
          fm[(cj + 1) * nw + ck + 1] = f;
        }
      }
      if (interior) {
        __syncthreads();
        if (!shell || !adjoint_force_shell(g, bx, cc, cm, fm, reinterpret_cast<unsigned *>(&tab),
                                           (int)(sizeof(sph::Tab) / sizeof(unsigned)), wsum, G))
          adjoint_force(g, bx, xa, xb, cc, G);
        continue;
      }
    }
    auto ld_glb = [&](int x, int y, int z) { return phi_at(g, x, y, z); };
    for (int col = threadIdx.x; col < ncol; col += blockDim.x) {
      const int cj = col / bx.n[2], ck = col % bx.n[2];
      const int j = bx.lo[1] + cj, k = bx.lo[2] + ck;
      for (int i = xa; i <= xb; i++) {
        // (the thread's own column of cc)
        const int c = tb ? (int)cc[((i - bx.lo[0] + 2) * Q1 + cj + 2) * Q2 + ck + 2]
                         : sph::sub_count(i, j, k, s, hs, img[m][0], img[m][1],
                                          img[m][2], R);
        if (!c || !valid_cell(g, solid, i, j, k)) continue;
        const double rho = (normalization == 1)
                               ? rho0 * ((double)c / (double)(s * s * s))
                               : (Q * (double)c) / (np * (h * h * h));
        double gr[3];
        if (interior)
          gradient_interior(g, h, i, j, k, gr);
        else
          gradient(g, solid, h, i, j, k, gr, ld_glb);
#pragma unroll
        for (int a = 0; a < 3; a++) F[a] = F[a] + gr[a] * rho;
      }
    }
  }
  // the adjoint sums: F += (3 / h) (1 / 36) rho_per_count sum_y Phi K
  const double unit = !any ? 0.0
                     : (normalization == 1) ? rho0 / (double)(s * s * s)
                                            : Q / (np * (h * h * h));
  const double scale = ((3.0 / h) / 36.0) * unit;
#pragma unroll
  for (int a = 0; a < 3; a++) F[a] = F[a] + G[a] * scale;
  __shared__ double sh3[3][32];
  bsum3(F, sh3);
  if (threadIdx.x == 0)
    for (int a = 0; a < 3; a++) part[3 * p + a] = F[a];
}

void launch_coulomb(const Grid &g, const unsigned char *solid_global, double h,
                    int subsample, int n, const double *sph, int normalization,
                    double *partials, const unsigned long long *counts,
                    cudaStream_t s) {
  if (n <= 0) return;
  if (is_periodic(g))
    k_coulomb<true><<<n, kTF, 0, s>>>(g, solid_global, h, subsample, sph,
                                      normalization, partials, counts);
  else
    k_coulomb<false><<<n, kTF, 0, s>>>(g, solid_global, h, subsample, sph,
                                       normalization, partials, counts);
}

}  // namespace mg
