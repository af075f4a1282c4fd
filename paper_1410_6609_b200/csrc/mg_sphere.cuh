// Sphere geometry shared by the RHS kernel (k_spheres, mg_kernels.cu) and the
// Coulomb-force kernel (k_coulomb, mg_force.cu): the charge mapping of
// "each cell whose center is overlapped", inclusive
// test |x - c|^2 <= R^2 (reading c13), subsampling factor s (the
// s^3 sub-cell centres ((i s + a + 1/2) h/s, ...)), periodic images
// (P:441-443).
//
// The inside test is d2 = (dx*dx + dy*dy) + dz*dz <= R*R with
// dx = ((double)(i s + a) + 0.5) * hs - cx, each product rounded on its own
// (-fmad=false).  tables() stores the per-axis products dx*dx of one
// sphere image in shared memory, so a test is two additions and a compare
// that reproduce d2 bit for bit.
#pragma once
#include <cuda_runtime.h>

#include "mg_internal.h"

namespace mg {
namespace sph {

constexpr int kTab = 512;  // table entries per axis: (bbox cells) * s
constexpr int kVal = 513;  // tabulated cell values per covered count (s <= 8)

// shared-memory tables of one sphere image: per axis the squared distances
// of the sub-cell centre coordinates (d[a][(i - lo) s + sub]) and, per cell,
// their minimum / maximum over the cell's s sub-positions
struct Tab {
  double d[3][kTab];
  double mn[3][kTab], mx[3][kTab];
};

__device__ __forceinline__ bool inside(int i, int j, int k, double h, double cx,
                                       double cy, double cz, double R) {
  const double dx = ((double)i + 0.5) * h - cx;
  const double dy = ((double)j + 0.5) * h - cy;
  const double dz = ((double)k + 0.5) * h - cz;
  const double d2 = (dx * dx + dy * dy) + dz * dz;
  return d2 <= R * R;
}

// covered sub-cell centres of cell (i,j,k), direct evaluation (fallback)
__device__ __forceinline__ int sub_count(int i, int j, int k, int s, double hs,
                                         double cx, double cy, double cz,
                                         double R) {
  int cnt = 0;
  for (int a = 0; a < s; a++)
    for (int b = 0; b < s; b++)
      for (int c = 0; c < s; c++)
        cnt += inside(i * s + a, j * s + b, k * s + c, hs, cx, cy, cz, R) ? 1 : 0;
  return cnt;
}

// cells whose centre (or a sub-cell centre) can lie within R of c, with a
// safety margin, clipped to [0, n)
__device__ __forceinline__ void bbox(int n, double h, double c, double R,
                                     int *lo, int *hi) {
  int a = (int)floor((c - R) / h - 0.5) - 1;
  int b = (int)ceil((c + R) / h - 0.5) + 1;
  *lo = a < 0 ? 0 : a;
  *hi = b > n - 1 ? n - 1 : b;
}

// periodic images: m in {-1,0,1} on periodic axes, centre c + m (n h) (the
// coordinate untouched for m = 0), (mx, my, mz) lexicographic -- the
// oracle's enumeration.  The host checks 2R + 2h <= n h on periodic axes.
__device__ __forceinline__ int images(const Grid &g, double h, double cx,
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

// the images of a sphere centre: 27 on grids with periodic axes, the
// centre itself otherwise (then no local-memory array)
template <bool PER>
struct Images {
  double c[PER ? 27 : 1][3];
  int n;
};
template <bool PER>
__device__ __forceinline__ void make_images(const Grid &g, double h, double cx, double cy,
                                            double cz, Images<PER> &im) {
  if constexpr (PER) {
    im.n = images(g, h, cx, cy, cz, im.c);
  } else {
    im.c[0][0] = cx;
    im.c[0][1] = cy;
    im.c[0][2] = cz;
    im.n = 1;
  }
}

// bounding box of one image: lo[a], n[a] cells per axis (0 if empty)
struct Box {
  int lo[3], n[3];
  __device__ long long cells() const { return (long long)n[0] * n[1] * n[2]; }
};

__device__ __forceinline__ Box box_of(const Grid &g, double h, const double c[3],
                                      double R) {
  Box b;
  const int ext[3] = {g.nx, g.ny, g.nz};
  for (int a = 0; a < 3; a++) {
    int lo, hi;
    bbox(ext[a], h, c[a], R, &lo, &hi);
    b.lo[a] = lo;
    b.n[a] = hi >= lo ? hi - lo + 1 : 0;
  }
  return b;
}

// Build the tables of one image (block-uniform result: false when a table
// would not fit, then callers use sub_count).  Starts and ends with a
// barrier, so it may be called once per image in a loop.
__device__ __forceinline__ bool tables(Tab &T, const Box &b, int s, double hs,
                                       const double c[3]) {
  __syncthreads();
  for (int a = 0; a < 3; a++)
    if (b.n[a] * s > kTab) return false;
  for (int a = 0; a < 3; a++) {
    for (int e = threadIdx.x; e < b.n[a] * s; e += blockDim.x) {
      const int i = b.lo[a] + e / s, sub = e % s;
      const double d = ((double)(i * s + sub) + 0.5) * hs - c[a];
      T.d[a][e] = d * d;
    }
    for (int ci = threadIdx.x; ci < b.n[a]; ci += blockDim.x) {
      double lo = 0.0, hi = 0.0;
      for (int sub = 0; sub < s; sub++) {  // the same products as T.d
        const double d = ((double)((b.lo[a] + ci) * s + sub) + 0.5) * hs - c[a];
        const double q = d * d;
        lo = sub ? fmin(lo, q) : q;
        hi = sub ? fmax(hi, q) : q;
      }
      T.mn[a][ci] = lo;
      T.mx[a][ci] = hi;
    }
  }
  __syncthreads();
  return true;
}

// covered sub-cells of box cell (ci, cj, ck) (box-relative) from the tables.
// IEEE addition is monotonic, so fl(fl(x+y)+z) of the per-axis minima
// (maxima) bounds every sub-centre's d2 from below (above): a cell whose
// lower bound exceeds R^2 has no covered sub-centre, one whose upper bound
// is <= R^2 has all s^3 -- exactly what the per-sub-centre test gives.
__device__ __forceinline__ int count_tab(const Tab &T, int ci, int cj, int ck,
                                         int s, double R2) {
  if ((T.mn[0][ci] + T.mn[1][cj]) + T.mn[2][ck] > R2) return 0;
  if ((T.mx[0][ci] + T.mx[1][cj]) + T.mx[2][ck] <= R2) return s * s * s;
  int cnt = 0;
  const double *tx = T.d[0] + ci * s, *ty = T.d[1] + cj * s, *tz = T.d[2] + ck * s;
  for (int a = 0; a < s; a++)
    for (int b = 0; b < s; b++) {
      const double t = tx[a] + ty[b];
      for (int c = 0; c < s; c++) cnt += (t + tz[c] <= R2) ? 1 : 0;
    }
  return cnt;
}

}  // namespace sph
}  // namespace mg
