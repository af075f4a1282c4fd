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

namespace mg {

namespace {

constexpr int kTF = 256;

__constant__ int kQ19[18][3] = {
    {1, 0, 0},  {-1, 0, 0}, {0, 1, 0},   {0, -1, 0}, {0, 0, 1},  {0, 0, -1},
    {1, 1, 0},  {-1, -1, 0}, {1, -1, 0}, {-1, 1, 0}, {1, 0, 1},  {-1, 0, -1},
    {1, 0, -1}, {-1, 0, 1}, {0, 1, 1},   {0, -1, -1}, {0, 1, -1}, {0, -1, 1}};

__device__ __forceinline__ bool insph(int i, int j, int k, double h, double cx,
                                      double cy, double cz, double R) {
  const double dx = ((double)i + 0.5) * h - cx;
  const double dy = ((double)j + 0.5) * h - cy;
  const double dz = ((double)k + 0.5) * h - cz;
  const double d2 = (dx * dx + dy * dy) + dz * dz;
  return d2 <= R * R;
}

__device__ __forceinline__ int subcnt(int i, int j, int k, int s, double hs,
                                      double cx, double cy, double cz, double R) {
  int c = 0;
  for (int a = 0; a < s; a++)
    for (int b = 0; b < s; b++)
      for (int d = 0; d < s; d++)
        c += insph(i * s + a, j * s + b, k * s + d, hs, cx, cy, cz, R) ? 1 : 0;
  return c;
}

__device__ __forceinline__ void bbox_f(int n, double h, double c, double R,
                                       int *lo, int *hi) {
  int a = (int)floor((c - R) / h - 0.5) - 1;
  int b = (int)ceil((c + R) / h - 0.5) + 1;
  *lo = a < 0 ? 0 : a;
  *hi = b > n - 1 ? n - 1 : b;
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

// periodic images of a sphere centre: the enumeration of k_spheres / the
// oracle (m in {-1,0,1} on periodic axes, (mx,my,mz) lexicographic)
__device__ __forceinline__ int images_f(const Grid &g, double h, double cx,
                                        double cy, double cz, double img[27][3]) {
  int n = 0;
  for (int mx = -g.per[0]; mx <= g.per[0]; mx++)
    for (int my = -g.per[1]; my <= g.per[1]; my++)
      for (int mz = -g.per[2]; mz <= g.per[2]; mz++) {
        img[n][0] = mx ? cx + (double)mx * ((double)g.nx * h) : cx;
        img[n][1] = my ? cy + (double)my * ((double)g.ny * h) : cy;
        img[n][2] = mz ? cz + (double)mz * ((double)g.nz * h) : cz;
        n++;
      }
  return n;
}

__device__ void gradient(const Grid &g, const unsigned char *solid, double h,
                         int i, int j, int k, double *gr) {
  bool all = true;
#pragma unroll
  for (int q = 0; q < 18; q++)
    all = all && valid_cell(g, solid, i + kQ19[q][0], j + kQ19[q][1], k + kQ19[q][2]);
  if (all) {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      double S = 0.0;
#pragma unroll
      for (int q = 0; q < 18; q++) {
        const int c = kQ19[q][a];
        if (c == 0) continue;
        const double w = q < 6 ? 1.0 / 18.0 : 1.0 / 36.0;
        const double v = phi_at(g, i + kQ19[q][0], j + kQ19[q][1], k + kQ19[q][2]);
        S = c > 0 ? S + w * v : S - w * v;
      }
      gr[a] = (3.0 * S) / h;
    }
    return;
  }
  const double c0 = phi_at(g, i, j, k);
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const int pi = i + (a == 0), pj = j + (a == 1), pk = k + (a == 2);
    const int mi = i - (a == 0), mj = j - (a == 1), mk = k - (a == 2);
    const bool vp = valid_cell(g, solid, pi, pj, pk);
    const bool vm = valid_cell(g, solid, mi, mj, mk);
    if (vp && vm)
      gr[a] = (phi_at(g, pi, pj, pk) - phi_at(g, mi, mj, mk)) / (2.0 * h);
    else if (vp)
      gr[a] = (phi_at(g, pi, pj, pk) - c0) / h;
    else if (vm)
      gr[a] = (c0 - phi_at(g, mi, mj, mk)) / h;
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
  const int p = blockIdx.x;
  const double R = sph[5 * p + 3], Q = sph[5 * p + 4];
  const double hs = h / (double)s;
  double img[27][3];
  const int nimg = images_f(g, h, sph[5 * p], sph[5 * p + 1], sph[5 * p + 2], img);
  double cnt = 0.0;
  for (int m = 0; m < nimg; m++) {
    const double cx = img[m][0], cy = img[m][1], cz = img[m][2];
    int i0, i1, j0, j1, k0, k1;
    bbox_f(g.nx, h, cx, R, &i0, &i1);
    bbox_f(g.ny, h, cy, R, &j0, &j1);
    bbox_f(g.nz, h, cz, R, &k0, &k1);
    const int ni = i1 - i0 + 1, nj = j1 - j0 + 1, nk = k1 - k0 + 1;
    const long long nbox = (ni > 0 && nj > 0 && nk > 0) ? (long long)ni * nj * nk : 0;
    for (long long t = threadIdx.x; t < nbox; t += blockDim.x) {
      const int k = k0 + (int)(t % nk);
      const long long q = t / nk;
      const int j = j0 + (int)(q % nj);
      const int i = i0 + (int)(q / nj);
      cnt += (double)subcnt(i, j, k, s, hs, cx, cy, cz, R);
    }
  }
  const double np = bsum(cnt, sh);
  double F[3] = {0.0, 0.0, 0.0};
  const bool any = np > 0.0 || normalization == 1;
  const double rho0 = Q / ((4.0 / 3.0) * 3.14159265358979323846 * (R * R * R));
  for (int m = 0; any && m < nimg; m++) {
    const double cx = img[m][0], cy = img[m][1], cz = img[m][2];
    int i0, i1, j0, j1, k0, k1;
    bbox_f(g.nx, h, cx, R, &i0, &i1);
    bbox_f(g.ny, h, cy, R, &j0, &j1);
    bbox_f(g.nz, h, cz, R, &k0, &k1);
    const int nj = j1 - j0 + 1, nk = k1 - k0 + 1;
    const int xa = i0 > g.x0 ? i0 : g.x0;
    const int xb = i1 < g.x0 + g.nxl - 1 ? i1 : g.x0 + g.nxl - 1;
    if (xa > xb || nj <= 0 || nk <= 0) continue;
    const long long nloc = (long long)(xb - xa + 1) * nj * nk;
    for (long long t = threadIdx.x; t < nloc; t += blockDim.x) {
      const int k = k0 + (int)(t % nk);
      const long long q = t / nk;
      const int j = j0 + (int)(q % nj);
      const int i = xa + (int)(q / nj);
      const int c = subcnt(i, j, k, s, hs, cx, cy, cz, R);
      if (!c || !valid_cell(g, solid, i, j, k)) continue;
      const double rho = (normalization == 1)
                             ? rho0 * ((double)c / (double)(s * s * s))
                             : (Q * (double)c) / (np * (h * h * h));
      double gr[3];
      gradient(g, solid, h, i, j, k, gr);
#pragma unroll
      for (int a = 0; a < 3; a++) F[a] = F[a] + gr[a] * rho;
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
