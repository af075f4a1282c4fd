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
// One CTA per sphere: count the covered sub-cells of the whole domain, then
// accumulate the slab's cells; per-slab partial sums, summed on the host in
// slab / rank order.
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

}  // namespace

__global__ void __launch_bounds__(kTF)
    k_coulomb(Grid g, const unsigned char *solid, double h, int s,
              const double *sph, int normalization, double *part) {
  __shared__ double sh[32];
  __shared__ sph::Tab tab;
  const int p = blockIdx.x;
  const double R = sph[5 * p + 3], Q = sph[5 * p + 4];
  const double R2 = R * R;
  const double hs = h / (double)s;
  double img[27][3];
  const int nimg = sph::images(g, h, sph[5 * p], sph[5 * p + 1], sph[5 * p + 2], img);
  long long cnt = 0;  // threads own (j, k) columns of the box, walk along x
  for (int m = 0; m < nimg; m++) {
    const sph::Box bx = sph::box_of(g, h, img[m], R);
    if (bx.cells() == 0) continue;
    const bool tb = sph::tables(tab, bx, s, hs, img[m]);
    const int ncol = bx.n[1] * bx.n[2];
    for (int col = threadIdx.x; col < ncol; col += blockDim.x) {
      const int cj = col / bx.n[2], ck = col % bx.n[2];
      for (int ci = 0; ci < bx.n[0]; ci++)
        cnt += tb ? sph::count_tab(tab, ci, cj, ck, s, R2)
                  : sph::sub_count(bx.lo[0] + ci, bx.lo[1] + cj, bx.lo[2] + ck, s,
                                   hs, img[m][0], img[m][1], img[m][2], R);
    }
  }
  const double np = bsum((double)cnt, sh);
  double F[3] = {0.0, 0.0, 0.0};
  const bool any = np > 0.0 || normalization == 1;
  const double rho0 = Q / ((4.0 / 3.0) * 3.14159265358979323846 * (R * R * R));
  for (int m = 0; any && m < nimg; m++) {
    const sph::Box bx = sph::box_of(g, h, img[m], R);
    const int xa = bx.lo[0] > g.x0 ? bx.lo[0] : g.x0;
    const int xb = min(bx.lo[0] + bx.n[0] - 1, g.x0 + g.nxl - 1);
    if (bx.cells() == 0 || xa > xb) continue;
    const bool tb = sph::tables(tab, bx, s, hs, img[m]);
    auto ld_glb = [&](int x, int y, int z) { return phi_at(g, x, y, z); };
    const int ncol = bx.n[1] * bx.n[2];
    for (int col = threadIdx.x; col < ncol; col += blockDim.x) {
      const int cj = col / bx.n[2], ck = col % bx.n[2];
      const int j = bx.lo[1] + cj, k = bx.lo[2] + ck;
      for (int i = xa; i <= xb; i++) {
        const int c = tb ? sph::count_tab(tab, i - bx.lo[0], cj, ck, s, R2)
                         : sph::sub_count(i, j, k, s, hs, img[m][0], img[m][1],
                                          img[m][2], R);
        if (!c || !valid_cell(g, solid, i, j, k)) continue;
        const double rho = (normalization == 1)
                               ? rho0 * ((double)c / (double)(s * s * s))
                               : (Q * (double)c) / (np * (h * h * h));
        double gr[3];
        gradient(g, solid, h, i, j, k, gr, ld_glb);
#pragma unroll
        for (int a = 0; a < 3; a++) F[a] = F[a] + gr[a] * rho;
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const double v = bsum(F[a], sh);
    if (threadIdx.x == 0) part[3 * p + a] = v;
  }
}

void launch_coulomb(const Grid &g, const unsigned char *solid_global, double h,
                    int subsample, int n, const double *sph, int normalization,
                    double *partials, cudaStream_t s) {
  if (n <= 0) return;
  k_coulomb<<<n, kTF, 0, s>>>(g, solid_global, h, subsample, sph, normalization,
                              partials);
}

}  // namespace mg
