// Sphere geometry shared by the RHS kernels (k_sphere_count,
// k_sphere_scatter, mg_kernels.cu) and the Coulomb-force kernel (k_coulomb,
// mg_force.cu): the charge mapping of
// "each cell whose center is overlapped", inclusive
// test |x - c|^2 <= R^2 (reading c13), subsampling factor s (the
// s^3 sub-cell centres ((i s + a + 1/2) h/s, ...)), periodic images
// (P:441-443).
//
// The inside test is d2 = (dx*dx + dy*dy) + dz*dz <= R*R with
// dx = ((double)(i s + a) + 0.5) * hs - cx, each product rounded on its own
// (-fmad=false).  tables() stores the per-axis products dx*dx of one
// sphere image in shared memory, so a test is two additions and a compare
// that reproduce d2 bit for bit; x_interval() finds the covered x
// sub-positions of a (y, z) sub-row as one interval (reading d9).
#pragma once
#include <cuda_runtime.h>

#include "mg_internal.h"

namespace mg {
namespace sph {

constexpr int kTab = 512;  // table entries per axis: (bbox cells) * s
constexpr int kVal = 513;  // tabulated cell values per covered count (s <= 8)

// shared-memory tables of one sphere image: per axis the squared distances
// of the sub-cell centre coordinates (d[a][(i - lo) s + sub]); emin = the x
// entry of least distance (the d[0] entries do not increase before it and do
// not decrease from it on)
struct Tab {
  double d[3][kTab];
  int emin;
};

// per-cell covered counts of one box, in shared memory (box cells <= kCells)
constexpr int kCells = 12288;

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
  // one thread per (axis, cell), the cell's s entries in a loop
  const int nc = b.n[0] + b.n[1] + b.n[2];
  for (int t = threadIdx.x; t < nc; t += blockDim.x) {
    const int a = t < b.n[0] ? 0 : (t < b.n[0] + b.n[1] ? 1 : 2);
    const int ci = t - (a > 0 ? b.n[0] : 0) - (a > 1 ? b.n[1] : 0);
    const int i = b.lo[a] + ci;
    for (int sub = 0; sub < s; sub++) {
      const int e = ci * s + sub;
      const double d = ((double)(i * s + sub) + 0.5) * hs - c[a];
      T.d[a][e] = d * d;
      // x: the first entry whose coordinate is >= the centre (x strictly
      // increases with e): the least square is there or just before it
      if (a == 0) {
        const bool first = d >= 0.0 && (e == 0 || ((double)(i * s + sub) - 0.5) * hs - c[a] < 0.0);
        const bool none = e == b.n[0] * s - 1 && d < 0.0;  // all left of c
        if (first || none) T.emin = none ? e + 1 : e;
      }
    }
  }
  __syncthreads();
  const int ne = b.n[0] * s;
  if (ne > 0) {
    const int e0 = T.emin;  // (every thread reads it; one more barrier)
    __syncthreads();
    if (threadIdx.x == 0)
      T.emin = (e0 > 0 && (e0 == ne || T.d[0][e0 - 1] <= T.d[0][e0])) ? e0 - 1 : e0;
  }
  __syncthreads();
  return true;
}

// floor(x / s) for 0 <= x < 2^10, s <= 16, with M = ceil(2^16 / s): the
// multiplier's excess adds less than x 2^-16 < 1/s to x / s
__device__ __forceinline__ int div_s(int x, unsigned M) { return (int)(((unsigned)x * M) >> 16); }
__host__ __device__ constexpr unsigned div_magic(int s) { return (65536u + (unsigned)s - 1u) / (unsigned)s; }

// The x sub-positions e (box-relative) of one sub-row -- fixed y and z
// squares ty, tz -- inside the sphere: (d[0][e] + ty) + tz <= R^2, the
// inside test's own operations.  IEEE addition is monotonic, so the test
// holds on an interval around emin, found by two binary searches.  Returns
// the interval [lo, hi] (hi < lo: empty).
__device__ __forceinline__ int2 x_interval(const Tab &T, int ne, double ty, double tz,
                                           double R2) {
  const double *dx = T.d[0];
  const int em = T.emin;
  if (!((dx[em] + ty) + tz <= R2)) return make_int2(1, 0);
  int a = 0, z = em;  // first inside position in [0, em]
  while (a < z) {
    const int m = (a + z) >> 1;
    if ((dx[m] + ty) + tz <= R2) z = m; else a = m + 1;
  }
  const int lo = a;
  a = em;
  z = ne - 1;  // last inside position in [em, ne)
  while (a < z) {
    const int m = (a + z + 1) >> 1;
    if ((dx[m] + ty) + tz <= R2) a = m; else z = m - 1;
  }
  return make_int2(lo, a);
}

// covered sub-cell count of every cell ci = 0..n0-1 of box column (cj, ck):
// cnt[base + ci * st] (cells with ci outside [sa, sb] -- another slab's --
// are stored as 0); returns the column's total over all ci.  Exactly the
// per-sub-centre test: the s^2 sub-rows' x intervals added cell by cell.
__device__ __forceinline__ int column_counts(const Tab &T, const Box &b, int s, double R2,
                                             int cj, int ck, unsigned short *cnt,
                                             int base, int st, int sa, int sb) {
  const int n0 = b.n[0], ne = n0 * s;
  const unsigned M = div_magic(s);
  for (int ci = 0; ci < n0; ci++) cnt[base + ci * st] = 0;
  int tot = 0;
  for (int y = 0; y < s; y++) {
    const double ty = T.d[1][cj * s + y];
    for (int z = 0; z < s; z++) {
      const int2 iv = x_interval(T, ne, ty, T.d[2][ck * s + z], R2);
      if (iv.y < iv.x) continue;
      tot += iv.y - iv.x + 1;
      const int c0 = max(div_s(iv.x, M), sa), c1 = min(div_s(iv.y, M), sb);
      for (int ci = c0; ci <= c1; ci++) {
        const int n = min(iv.y, ci * s + s - 1) - max(iv.x, ci * s) + 1;
        cnt[base + ci * st] = (unsigned short)(cnt[base + ci * st] + n);
      }
    }
  }
  return tot;
}

// the covered sub-cell total of one image: warps take the y sub-rows, lanes
// the z sub-rows
__device__ __forceinline__ long long image_count(const Tab &T, const Box &b, int s,
                                                 double R2) {
  const int ny = b.n[1] * s, nz = b.n[2] * s, ne = b.n[0] * s;
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  long long tot = 0;
  for (int y = threadIdx.x >> 5; y < ny; y += nw)
    for (int z = lane; z < nz; z += 32) {
      const int2 iv = x_interval(T, ne, T.d[1][y], T.d[2][z], R2);
      if (iv.y >= iv.x) tot += iv.y - iv.x + 1;
    }
  return tot;
}

}  // namespace sph
}  // namespace mg
