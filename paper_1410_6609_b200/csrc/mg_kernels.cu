// sm_100a kernels of the cell-centered multigrid solve (arXiv 1410.6609).
//
// Compiled with -fmad=false: every per-cell formula is evaluated with the
// operand order and single roundings written here, no FMA contraction, so
// smoother / residual / restriction / prolongation / sphere rasterisation are
// bitwise reproducible ("Parity contract").
//
// Operator (Galerkin closed form): on level l of a box domain
//     A_l = c_l * S_l,  c_l = 2^-l / h^2,
// S_l the folded integer 7-point stencil of the level's own grid: centre
// d = 6 + sum over touched faces (+1 Dirichlet, -1 Neumann), neighbours -1.
// Hence no stencil is stored: the centre comes from the cell position.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "mg_internal.h"
#include "mg_sphere.cuh"

namespace mg {

static constexpr int kThreads = 256;
static constexpr double kPi = 3.14159265358979323846;

__device__ __forceinline__ int centre_d(const Grid &g, int i, int j, int z) {
  int d = 6;
  if (i == 0) d += g.dface[0];
  if (i == g.nx - 1) d += g.dface[1];
  if (j == 0) d += g.dface[2];
  if (j == g.ny - 1) d += g.dface[3];
  if (z == 0) d += g.dface[4];
  if (z == g.nz - 1) d += g.dface[5];
  return d;
}

__device__ __forceinline__ long long rowbase(const Grid &g, int il, int j) {
  return (long long)(il + 1) * g.plane + (long long)(j + 1) * g.pz;
}

__device__ __forceinline__ double2 ld2(const double *p) {
  return *reinterpret_cast<const double2 *>(p);
}

// ---------------------------------------------------------------------------
// RBGS half-sweep.  One thread updates two cells of colour
// `color` (half-indices k, k+1 of one row):
//     Phi_c = (f_c * w + s) / d,  s = ((((x- + x+) + y-) + y+) + z-) + z+
// which equals (f_c - sum_q a_q Phi_q) / a_cc of the oracle bit for bit when
// c_l is a power of two.  The other colour's x/y neighbours share
// the half-index k; the z neighbours are O(k-1+p), O(k+p), p = z & 1.
// ---------------------------------------------------------------------------
// pairs (row, half-index pair) a half-sweep of g updates, one per thread
__host__ __device__ inline long long smooth_items(const Grid &g) {
  return (long long)g.nxl * g.ny * ((g.nzh + 1) >> 1);
}

// the two cells of pair t (no __restrict__: the persistent tail kernel
// calls it on arrays other CTAs of its cluster wrote before a barrier)
template <bool PER>
__device__ __forceinline__ void smooth_pair(const Grid &g, int color, int from_zero,
                                            long long t) {
  const int nk2 = (g.nzh + 1) >> 1;  // odd nzh: the last pair is half used
  const int k2 = (int)(t % nk2);
  const long long r = t / nk2;
  const int j = (int)(r % g.ny);
  const int il = (int)(r / g.ny);
  const int i = g.x0 + il;
  const int p = (i + j + color) & 1;
  double *own = color ? g.phiB : g.phiR;
  const double *oth = color ? g.phiR : g.phiB;
  const double *f = color ? g.fB : g.fR;
  const long long b = rowbase(g, il, j);
  const int k = 2 * k2;
  const double2 fo = ld2(f + b + k);
  double s0, s1;
  if (from_zero) {
    s0 = 0.0;
    s1 = 0.0;
  } else {
    const double2 xm = ld2(oth + b - g.plane + k);
    const double2 xp = ld2(oth + b + g.plane + k);
    const double2 ym = ld2(oth + b - g.pz + k);
    const double2 yp = ld2(oth + b + g.pz + k);
    const double2 zc = ld2(oth + b + k);
    double zm0, zp0, zm1, zp1;
    if (p == 0) {
      zm0 = z_lo<PER>(g, oth + b, k);
      zp0 = zc.x;
      zm1 = zc.x;
      zp1 = zc.y;
    } else {
      zm0 = zc.x;
      zp0 = z_hi0<PER>(g, oth + b, k, zc.y);
      zm1 = zc.y;
      zp1 = z_hi<PER>(g, oth + b, k);
    }
    s0 = ((((xm.x + xp.x) + ym.x) + yp.x) + zm0) + zp0;
    s1 = ((((xm.y + xp.y) + ym.y) + yp.y) + zm1) + zp1;
  }
  const int z0 = 2 * k + p;
  const double d0 = (double)centre_d(g, i, j, z0);
  const double d1 = (double)centre_d(g, i, j, z0 + 2);
  double2 out;
  out.x = div_small(fo.x * g.w + s0, d0, c_rcp16[(int)d0]);
  out.y = div_small(fo.y * g.w + s1, d1, c_rcp16[(int)d1]);
  if (k + 1 < g.nzh) {
    *reinterpret_cast<double2 *>(own + b + k) = out;
    if (PER) ghost_copies(g, own, il, j, k, out);
  } else {
    own[b + k] = out.x;
    if (PER) ghost_copies(g, own, il, j, k, out.x);
  }
}

template <bool PER>
__global__ void __launch_bounds__(kThreads)
    k_smooth(Grid g, int color, int from_zero) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < smooth_items(g)) smooth_pair<PER>(g, color, from_zero, t);
}

void launch_smooth(const Grid &g, int color, int from_zero, cudaStream_t s) {
  const long long total = (long long)g.nxl * g.ny * ((g.nzh + 1) >> 1);
  if (total <= 0) return;
  const unsigned blocks = (unsigned)((total + kThreads - 1) / kThreads);
  if (is_periodic(g))
    k_smooth<true><<<blocks, kThreads, 0, s>>>(g, color, from_zero);
  else
    k_smooth<false><<<blocks, kThreads, 0, s>>>(g, color, from_zero);
}

// residual r = f - c (d Phi - s) at (il, j, z) of a grid: the oracle's
// f - (a_cc Phi + sum_q a_q Phi_q) with the same roundings
template <bool PER>
__device__ __forceinline__ double resid_at(const Grid &g, int il, int j,
                                           int z) {
  const int i = g.x0 + il;
  const int col = (i + j + z) & 1;
  const int k = z >> 1;
  const int p = z & 1;
  const double *own = col ? g.phiB : g.phiR;
  const double *oth = col ? g.phiR : g.phiB;
  const double *f = col ? g.fB : g.fR;
  const long long b = rowbase(g, il, j);
  // z-1 / z+1 are the other colour's half-indices k-1+p / k+p; on a
  // periodic z axis z = -1 / nz wrap to nz-1 / 0 (half-indices nzh-1 / 0)
  const double zm = (z > 0) ? oth[b + k - 1 + p] : ((PER && g.per[2]) ? oth[b + g.nzh - 1] : 0.0);
  const double zp = (z < g.nz - 1) ? oth[b + k + p] : ((PER && g.per[2]) ? oth[b] : 0.0);
  const double s = ((((oth[b - g.plane + k] + oth[b + g.plane + k]) +
                      oth[b - g.pz + k]) +
                     oth[b + g.pz + k]) +
                    zm) +
                   zp;
  const double d = (double)centre_d(g, i, j, z);
  const double t = d * own[b + k] - s;
  return f[b + k] - g.c * t;
}

// ---------------------------------------------------------------------------
// Fused residual + restriction: f_{l+1}(C) = 1/8 * pairwise sum of the
// residuals of C's 8 children, child bits (dx,dy,dz), dz fastest.  The fine
// residual is never stored.  One thread per coarse cell.
// ---------------------------------------------------------------------------
__host__ __device__ inline long long restrict_items(const Grid &F) {
  return (long long)(F.nxl >> 1) * (F.ny >> 1) * (F.nz >> 1);
}

// red0: also the coarse level's first red half-sweep from Phi = 0 on the
// coarse cell if it is red (box domains; the from-zero sweep's expression)
template <bool PER>
__device__ __forceinline__ void restrict_cell(const Grid &F, const Grid &C, long long t,
                                              int red0 = 0) {
  const int ncz = F.nz >> 1, ncy = F.ny >> 1;
  const int K = (int)(t % ncz);
  const long long q = t / ncz;
  const int J = (int)(q % ncy);
  const int Il = (int)(q / ncy);
  double r[8];
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 2; b++)
#pragma unroll
      for (int c = 0; c < 2; c++)
        r[a * 4 + b * 2 + c] = resid_at<PER>(F, 2 * Il + a, 2 * J + b, 2 * K + c);
  const double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  const int Ig = (F.x0 >> 1) + Il;
  const int col = (Ig + J + K) & 1;
  double *cf = col ? C.fB : C.fR;
  const double fc = 0.125 * s;
  cf[rowbase(C, Ig - C.x0, J) + (K >> 1)] = fc;
  if (red0 && col == 0) {
    const double d = (double)centre_d(C, Ig, J, K);
    C.phiR[rowbase(C, Ig - C.x0, J) + (K >> 1)] = div_small(fc * C.w + 0.0, d,
                                                             c_rcp16[(int)d]);
  }
}

template <bool PER>
__global__ void __launch_bounds__(kThreads)
    k_resid_restrict(Grid F, Grid C, int red0) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < restrict_items(F)) restrict_cell<PER>(F, C, t, red0);
}

void launch_resid_restrict(const Grid &f, const Grid &c, int red0,
                           cudaStream_t s) {
  const long long total =
      (long long)(f.nxl >> 1) * (f.ny >> 1) * (f.nz >> 1);
  if (total <= 0) return;
  const unsigned blocks = (unsigned)((total + kThreads - 1) / kThreads);
  if (is_periodic(f))
    k_resid_restrict<true><<<blocks, kThreads, 0, s>>>(f, c, 0);
  else
    k_resid_restrict<false><<<blocks, kThreads, 0, s>>>(f, c, red0);
}

// ---------------------------------------------------------------------------
// Prolongation + magnified correction:
//     Phi(c) = Phi(c) + alpha * e(parent(c)),  parent = (i/2, j/2, z/2).
// Red and black cells with half-index k both have parent z-index Z = k.
// ---------------------------------------------------------------------------
__host__ __device__ inline long long prolong_items(const Grid &F) {
  return (long long)F.nxl * F.ny * F.nzh;
}

__device__ __forceinline__ void prolong_cell(const Grid &F, const Grid &C, double alpha,
                                             long long t) {
  const int k = (int)(t % F.nzh);
  const long long q = t / F.nzh;
  const int j = (int)(q % F.ny);
  const int il = (int)(q / F.ny);
  const int I = (F.x0 + il) >> 1, J = j >> 1, Z = k;
  const double *ce = ((I + J + Z) & 1) ? C.phiB : C.phiR;
  const double e = ce[rowbase(C, I - C.x0, J) + (Z >> 1)];
  const long long b = rowbase(F, il, j) + k;
  F.phiR[b] = F.phiR[b] + alpha * e;
  F.phiB[b] = F.phiB[b] + alpha * e;
}

__global__ void __launch_bounds__(kThreads)
    k_prolong(Grid F, Grid C, double alpha) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < prolong_items(F)) prolong_cell(F, C, alpha, t);
}

void launch_prolong(const Grid &f, const Grid &c, int /*cofs*/, double alpha,
                    cudaStream_t s) {
  const long long total = (long long)f.nxl * f.ny * f.nzh;
  if (total <= 0) return;
  const unsigned blocks = (unsigned)((total + kThreads - 1) / kThreads);
  k_prolong<<<blocks, kThreads, 0, s>>>(f, c, alpha);
}

// ---------------------------------------------------------------------------
// Residual norm (Alg.1): per-block partial sums of r^2 with a
// fixed grid and a fixed reduction tree (deterministic), then an ordered sum.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  v = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.0;
  if (wid == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sh[0] = v;
  }
  __syncthreads();
  v = sh[0];
  __syncthreads();
  return v;
}

// residual of the two cells of colour `col` at half-indices k, k+1 of row
// (il, j): same expression as resid_at, vectorised along the row
template <bool PER>
__device__ __forceinline__ void resid_pair(const Grid &g, int il, int j, int k,
                                           int col, double &r0, double &r1) {
  const int i = g.x0 + il;
  const int p = (i + j + col) & 1;  // own cells at z = 2k + p, 2k + 2 + p
  const double *own = col ? g.phiB : g.phiR;
  const double *oth = col ? g.phiR : g.phiB;
  const double *f = col ? g.fB : g.fR;
  const long long b = rowbase(g, il, j);
  const double2 xm = ld2(oth + b - g.plane + k);
  const double2 xp = ld2(oth + b + g.plane + k);
  const double2 ym = ld2(oth + b - g.pz + k);
  const double2 yp = ld2(oth + b + g.pz + k);
  const double2 zc = ld2(oth + b + k);
  const double2 u = ld2(own + b + k);
  const double2 fo = ld2(f + b + k);
  double zm0, zp0, zm1, zp1;
  if (p == 0) {
    zm0 = z_lo<PER>(g, oth + b, k);
    zp0 = zc.x;
    zm1 = zc.x;
    zp1 = zc.y;
  } else {
    zm0 = zc.x;
    zp0 = z_hi0<PER>(g, oth + b, k, zc.y);
    zm1 = zc.y;
    zp1 = z_hi<PER>(g, oth + b, k);
  }
  const double s0 = ((((xm.x + xp.x) + ym.x) + yp.x) + zm0) + zp0;
  const double s1 = ((((xm.y + xp.y) + ym.y) + yp.y) + zm1) + zp1;
  const int z0 = 2 * k + p;
  const double d0 = (double)centre_d(g, i, j, z0);
  const double d1 = (double)centre_d(g, i, j, z0 + 2);
  const double t0 = d0 * u.x - s0;
  const double t1 = d1 * u.y - s1;
  r0 = fo.x - g.c * t0;
  r1 = (k + 1 < g.nzh) ? fo.y - g.c * t1 : 0.0;
}

// one thread per (row, double2 position), both colours: 4 cells
template <bool PER>
__global__ void __launch_bounds__(kThreads)
    k_norm_partials(Grid g, double *partials) {
  __shared__ double sh[32];
  const int nk2 = (g.nzh + 1) >> 1;
  const long long total = (long long)g.nxl * g.ny * nk2;
  double acc = 0.0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
       t < total; t += (long long)gridDim.x * blockDim.x) {
    const int k2 = (int)(t % nk2);
    const long long r = t / nk2;
    const int j = (int)(r % g.ny);
    const int il = (int)(r / g.ny);
    double a0, a1, b0, b1;
    resid_pair<PER>(g, il, j, 2 * k2, 0, a0, a1);
    resid_pair<PER>(g, il, j, 2 * k2, 1, b0, b1);
    acc = acc + a0 * a0;
    acc = acc + a1 * a1;
    acc = acc + b0 * b0;
    acc = acc + b1 * b1;
  }
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

int launch_norm_partials(const Grid &g, double *partials, cudaStream_t s) {
  const long long total = (long long)g.nxl * g.ny * ((g.nzh + 1) >> 1);
  long long nb = (total + kThreads - 1) / kThreads;
  if (nb > norm_blocks_max(g)) nb = norm_blocks_max(g);
  if (nb < 1) nb = 1;
  if (is_periodic(g))
    k_norm_partials<true><<<(unsigned)nb, kThreads, 0, s>>>(g, partials);
  else
    k_norm_partials<false><<<(unsigned)nb, kThreads, 0, s>>>(g, partials);
  return (int)nb;
}

__global__ void __launch_bounds__(kThreads)
    k_sum_ordered(const double *parts, int n, double *out) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) acc = acc + parts[t];
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) out[0] = s;
}

void launch_sum_ordered(const double *parts, int n, double *out,
                        cudaStream_t s) {
  k_sum_ordered<<<1, kThreads, 0, s>>>(parts, n, out);
}

// k_sum_ordered and k_publish in one launch (one slab): out[0] = dev_dst[0]
// = host_dst[0] = the ordered sum
__global__ void __launch_bounds__(kThreads)
    k_sum_publish(const double *parts, int n, double *out, double *dev_dst,
                  double *host_dst) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) acc = acc + parts[t];
  const double v = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    out[0] = v;
    dev_dst[0] = v;
    host_dst[0] = v;
    __threadfence_system();
  }
}

void launch_sum_publish(const double *parts, int n, double *out, double *dev_dst,
                        double *host_dst, cudaStream_t s) {
  k_sum_publish<<<1, kThreads, 0, s>>>(parts, n, out, dev_dst, host_dst);
}

// dev_dst[0] = host_dst[0] = src[0]; host_dst is mapped pinned memory, so
// the value reaches the host without a copy-engine transfer (which would
// queue behind bulk copies on the same engine)
__global__ void k_publish(const double *src, double *dev_dst, double *host_dst) {
  const double v = src[0];
  dev_dst[0] = v;
  host_dst[0] = v;
  __threadfence_system();
}

void launch_publish(const double *src, double *dev_dst, double *host_dst,
                    cudaStream_t s) {
  k_publish<<<1, 1, 0, s>>>(src, dev_dst, host_dst);
}

// index of the first sphere whose covered count is 0 (or -1), written to
// mapped host memory like k_publish (no copy-engine transfer)
__global__ void __launch_bounds__(1024)
    k_first_empty(const unsigned long long *counts, int n, double *host_dst) {
  __shared__ int first;
  if (threadIdx.x == 0) first = n;
  __syncthreads();
  for (int p = threadIdx.x; p < n; p += blockDim.x)
    if (counts[p] == 0ull) atomicMin(&first, p);
  __syncthreads();
  if (threadIdx.x == 0) {
    host_dst[0] = first < n ? (double)first : -1.0;
    __threadfence_system();
  }
}

void launch_first_empty(const unsigned long long *counts, int n, double *host_dst,
                        cudaStream_t s) {
  if (n > 0) k_first_empty<<<1, 1024, 0, s>>>(counts, n, host_dst);
}

// ---------------------------------------------------------------------------
// Coarsest-grid CG: one CTA, from x = 0, stop at ||r|| <= tol
// ||b|| or maxit.  Up to kCgSmemMax unknowns and eight per thread: the
// register-resident Chronopoulos-Gear form below (cg_cta_cg); otherwise this
// Hestenes-Stiefel loop.  Vectors in natural order, in shared memory
// when they fit (else in `scratch`, L1/L2-resident); the operator is the same
// closed form as the smoother.  Dot products: per-thread partials in a fixed
// order, warp shuffle tree, then every thread sums the warp partials in
// warp order (one barrier per dot; two alternating partial arrays).
// Two barriers per iteration: the direction p = r + beta p is not formed in
// a pass of its own but where the next matrix-vector product needs it --
// each thread evaluates r[k] + beta * p_old[k] (the same expression, hence
// the same bits) for its cell and the six neighbours and stores its own
// p_new in the other of two p buffers (p_old stays readable: no barrier).
// ---------------------------------------------------------------------------
static constexpr int kCgThreads = 512;  // cg_threads' largest count
static constexpr long long kCgSmemMax = 4096;  // unknowns with smem vectors

__device__ __forceinline__ long long split_index(const Grid &g, int il, int j,
                                                 int z, int *col) {
  *col = (g.x0 + il + j + z) & 1;
  return rowbase(g, il, j) + (z >> 1);
}

// sum over the block of per-thread values; one barrier; all threads get it.
// Fixed trees: the warp's butterfly, then the warp partials (zero-padded to
// 32) by a butterfly in every warp -- log-depth dependency chains, where a
// serial sum over the warps would put nw dependent fp64 additions on the
// CG's critical path every iteration.
__device__ __forceinline__ double cg_allsum(double v, double *part) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  const int lane = threadIdx.x & 31;
  double s = lane < nw ? part[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// doubles of a CG work area for N unknowns: x, r, two p buffers, q, then the
// per-element neighbour bits (2 bytes) and centre (1 byte)
__host__ __device__ inline size_t cg_area_doubles(long long N) {
  return 5 * (size_t)N + ((size_t)N * 3 + 7) / 8;
}

// CG on grid g by the calling CTA (every thread must call it; the first
// nthr of them hold elements -- the others add zeros to the dot products,
// which leaves the sums' bits unchanged); `base`: a work area of
// cg_area_doubles(N) (shared or global memory: callers pass a __shared__
// array and a global pointer in separate calls, so that the inlined copy
// for shared memory uses shared-memory loads); part: 2 x 32 doubles of
// shared memory.  The neighbour values are loaded unconditionally from a
// valid index and selected (no branches in the matrix-vector product).
template <bool PER>
__device__ __forceinline__ void cg_cta(const Grid &g, double *base, double (*part)[64],
                                       double tol, int maxit, int *iters_out,
                                       int nthr) {
  using NB = typename std::conditional<PER, unsigned short, unsigned char>::type;
  const int N = g.nx * g.ny * g.nz;
  double *x = base, *r = base + N, *pa = base + 2 * N, *pbuf = base + 3 * N,
         *q = base + 4 * N;
  // per-element geometry, computed once: neighbour bits (x-,x+,y-,y+,z-,z+):
  // bits 0-5 neighbour inside the level, bits 6-11 neighbour across a
  // periodic face (the opposite side's cell); and the centre d
  // (closed-form operator A = c (d - neighbours))
  NB *nb = reinterpret_cast<NB *>(base + 5 * N);
  signed char *dc = reinterpret_cast<signed char *>(nb + N);
  const int sx = g.ny * g.nz, sy = g.nz;
  const int wx = (g.nx - 1) * sx, wy = (g.ny - 1) * sy, wz = g.nz - 1;
  const int nend = (int)threadIdx.x < nthr ? N : 0;  // idle threads: no elements
  int pb = 0;
  double acc = 0.0;
  for (int n = threadIdx.x; n < nend; n += nthr) {
    const int z = n % g.nz;
    const int t = n / g.nz;
    const int j = t % g.ny, i = t / g.ny;
    const int in[6] = {i > 0, i < g.nx - 1, j > 0, j < g.ny - 1, z > 0, z < g.nz - 1};
    unsigned m = 0;
#pragma unroll
    for (int a = 0; a < 6; a++)
      m |= in[a] ? (1u << a) : ((PER && g.per[a >> 1]) ? (64u << a) : 0u);
    nb[n] = (NB)m;
    dc[n] = (signed char)centre_d(g, i, j, z);
    int col;
    const long long idx = split_index(g, i, j, z, &col);
    const double b = col ? g.fB[idx] : g.fR[idx];
    x[n] = 0.0;
    r[n] = b;
    pa[n] = 0.0;  // p_old of the first iteration: p = r + 0 * 0 = r
    acc = acc + b * b;
  }
  double rho = cg_allsum(acc, part[pb]);  // barrier also publishes r, nb, dc
  pb ^= 1;
  const double bnorm = sqrt(rho);
  const double c = g.c;
  double beta = 0.0;
  double *po = pa, *pn = pbuf;  // p of the last iteration / of this one
  int it = 0;
  if (bnorm > 0.0) {
    while (it < maxit) {
      acc = 0.0;
      for (int n = threadIdx.x; n < nend; n += nthr) {
        const unsigned m = nb[n];
        // p = r + beta p_old at neighbour (bit `in`: inside; bit `pe`: across
        // a periodic face) -- a valid index is loaded either way, the value
        // selected
        auto nbr = [&](unsigned in, unsigned pe, int kin, int kpe) {
          const bool vi = (m & in) != 0, vp = PER && (m & pe) != 0;
          const int k = vi ? kin : (vp ? kpe : n);
          const double v = r[k] + beta * po[k];
          return (vi || vp) ? v : 0.0;
        };
        const double xm = nbr(1, 64, n - sx, n + wx);
        const double xp = nbr(2, 128, n + sx, n - wx);
        const double ym = nbr(4, 256, n - sy, n + wy);
        const double yp = nbr(8, 512, n + sy, n - wy);
        const double zm = nbr(16, 1024, n - 1, n + wz);
        const double zp = nbr(32, 2048, n + 1, n - wz);
        const double s = ((((xm + xp) + ym) + yp) + zm) + zp;
        const double p = r[n] + beta * po[n];
        pn[n] = p;
        const double qn = c * ((double)dc[n] * p - s);
        q[n] = qn;
        acc = acc + p * qn;
      }
      const double pq = cg_allsum(acc, part[pb]);
      pb ^= 1;
      const double a = rho / pq;
      acc = 0.0;
      for (int n = threadIdx.x; n < nend; n += nthr) {
        x[n] = x[n] + a * pn[n];
        const double rn = r[n] - a * q[n];
        r[n] = rn;
        acc = acc + rn * rn;
      }
      const double rho1 = cg_allsum(acc, part[pb]);
      pb ^= 1;
      it++;
      if (sqrt(rho1) <= tol * bnorm) break;
      beta = rho1 / rho;
      rho = rho1;
      double *t = po;
      po = pn;
      pn = t;
    }
  }
  __syncthreads();
  for (int n = threadIdx.x; n < nend; n += nthr) {
    const int z = n % g.nz;
    const int t = n / g.nz;
    int col;
    const long long idx = split_index(g, t / g.ny, t % g.ny, z, &col);
    (col ? g.phiB : g.phiR)[idx] = x[n];
  }
  if (threadIdx.x == 0 && iters_out) *iters_out = it;
}

// doubles of the register-resident CG's shared area: r with a zero slot at
// N, then x
__host__ __device__ inline size_t cg_reg_doubles(long long N) { return 2 * (size_t)N + 1; }

// CG on grid g by the calling CTA, N <= E * nthr unknowns held in registers
// (element n = threadIdx.x + e * nthr): the Chronopoulos-Gear arrangement of
// the conjugate-gradient recurrences (reading c8): w = A r, gamma = (r, r)
// and delta = (w, r) summed in ONE reduction, then
//     beta = gamma / gamma_old,  alpha = gamma / (delta - beta gamma / alpha_old),
//     p = r + beta p,  s = w + beta s (= A p),  x += alpha p,  r -= alpha s,
// the same iterates as Hestenes-Stiefel in exact arithmetic (the stopping
// test on the recursively updated r, ||r|| <= tol ||b||, and the iteration
// count as cg_cta).  Shared memory holds r for the neighbours (the six
// neighbour offsets are computed once; outside the level they point at a
// zero slot) and x (updated off the dependency chain: registers for eight
// elements per thread would spill).  One reduction and one plain barrier per iteration instead of
// two reductions, six neighbour loads instead of twelve.
template <bool PER, int E>
__device__ __forceinline__ void cg_cta_cg(const Grid &g, double *sm, double (*part)[64],
                                          double tol, int maxit, int *iters_out,
                                          int nthr, int bar, int bcnt) {
  const int N = g.nx * g.ny * g.nz;
  double *rs = sm, *xs = sm + N + 1;
  const int sx = g.ny * g.nz, sy = g.nz;
  const int wx = (g.nx - 1) * sx, wy = (g.ny - 1) * sy, wz = g.nz - 1;
  unsigned nb[E][3];  // six 16-bit offsets (N <= kCgSmemMax < 65536)
  double r[E], p[E], sv[E], w[E];
  unsigned long long dpk = 0;  // the centre integers d (<= 12), 4 bits each
  bool act[E];
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int n = (int)threadIdx.x + e * nthr;
    act[e] = (int)threadIdx.x < nthr && n < N;
    r[e] = p[e] = sv[e] = w[e] = 0.0;
#pragma unroll
    for (int a = 0; a < 3; a++) nb[e][a] = (unsigned)N * 0x10001u;
    if (act[e]) {
      const int z = n % g.nz;
      const int t = n / g.nz;
      const int j = t % g.ny, i = t / g.ny;
      const bool in[6] = {i > 0, i < g.nx - 1, j > 0, j < g.ny - 1, z > 0, z < g.nz - 1};
      const int kin[6] = {n - sx, n + sx, n - sy, n + sy, n - 1, n + 1};
      const int kpe[6] = {n + wx, n - wx, n + wy, n - wy, n + wz, n - wz};
      int k6[6];
#pragma unroll
      for (int a = 0; a < 6; a++)
        k6[a] = in[a] ? kin[a] : ((PER && g.per[a >> 1]) ? kpe[a] : N);
#pragma unroll
      for (int a = 0; a < 3; a++)
        nb[e][a] = (unsigned)k6[2 * a] | ((unsigned)k6[2 * a + 1] << 16);
      dpk |= (unsigned long long)centre_d(g, i, j, z) << (4 * e);
      int col;
      const long long idx = split_index(g, i, j, z, &col);
      const double b = col ? g.fB[idx] : g.fR[idx];
      r[e] = b;
      rs[n] = b;
      xs[n] = 0.0;
    }
  }
  if (threadIdx.x == 0) rs[N] = 0.0;
  const double c = g.c;
  int pb = 0;
  // w = A r from the published r; partial sums of (r, r) and (w, r)
  auto matvec = [&](double &gg, double &dl) {
    gg = 0.0;
    dl = 0.0;
#pragma unroll
    for (int e = 0; e < E; e++) {
      auto v = [&](int a) {
        return rs[(int)((nb[e][a >> 1] >> (16 * (a & 1))) & 0xffffu)];
      };
      const double s = ((((v(0) + v(1)) + v(2)) + v(3)) + v(4)) + v(5);
      const double d = (double)(int)((dpk >> (4 * e)) & 15u);
      w[e] = c * (d * r[e] - s);
      if (act[e]) {
        gg = gg + r[e] * r[e];
        dl = dl + w[e] * r[e];
      }
    }
  };
  bar_part(bar, bcnt);  // r published
  double gg, dl;
  matvec(gg, dl);
  double2 gd = cg_allsum2(gg, dl, part[pb], bar, bcnt);
  pb ^= 1;
  double gamma = gd.x;
  const double bnorm = sqrt(gamma);
  int it = 0;
  if (bnorm > 0.0) {
    double alpha = gamma / gd.y;
    // beta gamma / alpha_old = gamma^2 k with k = 1 / (gamma_old alpha_old),
    // formed a step ahead: one division on the chain after the reduction
    double kinv = 1.0 / (gamma * alpha);
#pragma unroll
    for (int e = 0; e < E; e++) {
      p[e] = r[e];
      sv[e] = w[e];
    }
    while (it < maxit) {
#pragma unroll
      for (int e = 0; e < E; e++) {
        r[e] = r[e] - alpha * sv[e];
        if (act[e]) {
          const int n = (int)threadIdx.x + e * nthr;
          rs[n] = r[e];
          xs[n] = xs[n] + alpha * p[e];
        }
      }
      bar_part(bar, bcnt);  // r published (the reads of the last product are
                            // done: they precede the reduction's barrier)
      it++;
      matvec(gg, dl);
      gd = cg_allsum2(gg, dl, part[pb], bar, bcnt);
      pb ^= 1;
      if (sqrt(gd.x) <= tol * bnorm) break;
      const double beta = gd.x / gamma;
      alpha = gd.x / (gd.y - (gd.x * gd.x) * kinv);
      kinv = 1.0 / (gd.x * alpha);
      gamma = gd.x;
#pragma unroll
      for (int e = 0; e < E; e++) {
        p[e] = r[e] + beta * p[e];
        sv[e] = w[e] + beta * sv[e];
      }
    }
  }
#pragma unroll
  for (int e = 0; e < E; e++) {
    if (!act[e]) continue;
    const int n = (int)threadIdx.x + e * nthr;
    const int z = n % g.nz;
    const int t = n / g.nz;
    int col;
    const long long idx = split_index(g, t / g.ny, t % g.ny, z, &col);
    (col ? g.phiB : g.phiR)[idx] = xs[n];
  }
  if (threadIdx.x == 0 && iters_out) *iters_out = it;
}

// the register-resident CG for the elements per thread N needs (<= MAXE,
// at most 8), else false (the caller runs cg_cta)
template <bool PER, int MAXE = 8>
__device__ __forceinline__ bool cg_cta_fast(const Grid &g, double *sm, double (*part)[64],
                                            double tol, int maxit, int *iters_out,
                                            int nthr, int bar = 0, int bcnt = 0) {
  const int N = g.nx * g.ny * g.nz;
  const int E = (N + nthr - 1) / nthr;
  if (E <= 1)
    cg_cta_cg<PER, 1>(g, sm, part, tol, maxit, iters_out, nthr, bar, bcnt);
  else if (E <= 2)
    cg_cta_cg<PER, 2>(g, sm, part, tol, maxit, iters_out, nthr, bar, bcnt);
  else if (MAXE >= 4 && E <= 4)
    cg_cta_cg<PER, 4>(g, sm, part, tol, maxit, iters_out, nthr, bar, bcnt);
  else if (MAXE >= 8 && E <= 8)
    cg_cta_cg<PER, 8>(g, sm, part, tol, maxit, iters_out, nthr, bar, bcnt);
  else
    return false;
  return true;
}

template <bool PER>
__global__ void __launch_bounds__(kCgThreads)
    k_coarse_cg(Grid g, double *scr, double tol, int maxit, int *iters_out) {
  extern __shared__ double cg_sm[];
  __shared__ double part[2][64];
  const long long N = (long long)g.nx * g.ny * g.nz;
  if (N <= kCgSmemMax) {
    if (!cg_cta_fast<PER>(g, cg_sm, part, tol, maxit, iters_out, (int)blockDim.x))
      cg_cta<PER>(g, cg_sm, part, tol, maxit, iters_out, (int)blockDim.x);
  } else {
    cg_cta<PER>(g, scr, part, tol, maxit, iters_out, (int)blockDim.x);
  }
}

size_t coarse_cg_scratch_doubles(const Grid &g) {
  return cg_area_doubles((long long)g.nx * g.ny * g.nz);
}

// (round 2, Chronopoulos-Gear, scripts/cg_probe.py: unknowns per thread
// capped at 2 / 4 / 8 / 16 instead -- i.e. fewer threads -- are slower or no
// faster on 8^3, 32 x 8 x 8, 64 x 8 x 8; one z-row per thread with its z
// neighbours in registers is slower too: 68 vs 57 us on 8^3)
// 256 threads below 2048 unknowns, 512 from there (more warps hide the smem
// latency of the per-thread loops: 64 x 8 x 8, config 4's coarsest at P = 8,
// 476 vs 557 us in round 1; 1024 threads are slower again)
// (round 2 A/B, scripts/cg_probe.py: caps of 64/128 per block are slower,
// 512/1024 no faster -- the iteration is bound by its dependency chain; a
// separate p = r + beta p pass with a third barrier is slower on 8^3 and
// faster on 32 x 8 x 8, 3.275 vs 3.268 ms per config-3 cycle)
static int cg_threads(const Grid &g) {
  const long long N = (long long)g.nx * g.ny * g.nz;
  int threads = (int)((N + 31) / 32 * 32);
  const int cap = N >= 2048 ? 512 : 256;
  return threads > cap ? cap : threads;
}

template <bool PER>
static void launch_cg(const Grid &g, double *scratch, double tol, int maxit,
                      int *iters_out, cudaStream_t s) {
  const long long N = (long long)g.nx * g.ny * g.nz;
  const int threads = cg_threads(g);
  size_t smem = 0;
  if (N <= kCgSmemMax) {
    smem = cg_area_doubles(N) * sizeof(double);
    static size_t configured = 48 * 1024;
    if (smem > configured) {
      cudaFuncSetAttribute(k_coarse_cg<PER>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      configured = smem;
    }
  }
  k_coarse_cg<PER><<<1, threads, smem, s>>>(g, scratch, tol, maxit, iters_out);
}

void launch_coarse_cg(const Grid &g, double *scratch, double tol, int maxit,
                      int *iters_out, cudaStream_t s) {
  if (is_periodic(g))
    launch_cg<true>(g, scratch, tol, maxit, iters_out, s);
  else
    launch_cg<false>(g, scratch, tol, maxit, iters_out, s);
}

// ---------------------------------------------------------------------------
// RHS from charged spheres (centre rule P:273, inclusive c13;
// subsampling P:485-489; periodic images P:441-443).  Two kernels, one CTA
// per sphere each:
//   k_sphere_count    n_p = covered sub-cells of the whole (global) domain
//                     over all images (per-axis tables, mg_sphere.cuh)
//   k_sphere_scatter  the density of the covered cells of this slab.  A cell
//                     covered by several spheres is written once, by the
//                     lowest-index one, as ((0 + rho_p1) + rho_p2) + ... in
//                     ascending sphere order -- the oracle's "overlapping
//                     spheres add in sphere order" exactly, and deterministic
//                     (no atomics).  The other spheres that can reach a cell
//                     of sphere p are found first (k_sphere_neighbours): a
//                     uniform grid of bins (k_sphere_bin, bins wider than any
//                     two radii) gives the candidates of the bins around p,
//                     which pass a conservative distance test and are sorted
//                     into an ascending list.  A full bin or more than kNbMax
//                     neighbours make every cell scan all spheres instead --
//                     slow, still exact.  Isolated spheres (the common case)
//                     store their cells without the neighbour checks.  Per
//                     box column the covered counts come from the sub-rows'
//                     x intervals (sph::column_counts, reading d9).
// sph holds (cx, cy, cz, R, Q) per sphere.  Every cell not covered keeps the
// value it has (the caller zeroes f first).
// ---------------------------------------------------------------------------
template <bool PER>
__global__ void __launch_bounds__(kThreads)
    k_sphere_count(Grid g, double h, int s, const double *sph,
                   unsigned long long *counts) {
  __shared__ double sh[32];
  __shared__ sph::Tab tab;
  const int p = blockIdx.x;
  const double R = sph[5 * p + 3];
  const double R2 = R * R;
  const double hs = h / (double)s;
  sph::Images<PER> im;
  sph::make_images<PER>(g, h, sph[5 * p], sph[5 * p + 1], sph[5 * p + 2], im);
  const int nimg = im.n;
  auto &img = im.c;
  // threads share the (y, z) sub-rows of the box: each adds the length of
  // its x interval (sph::x_interval); integer counts are exact in any order
  long long cnt = 0;
  for (int m = 0; m < nimg; m++) {
    const sph::Box bx = sph::box_of(g, h, img[m], R);
    if (bx.cells() == 0) continue;
    if (sph::tables(tab, bx, s, hs, img[m])) {
      cnt += sph::image_count(tab, bx, s, R2);
      continue;
    }
    const int ncol = bx.n[1] * bx.n[2];  // (a box too long for the tables)
    for (int col = threadIdx.x; col < ncol; col += blockDim.x) {
      const int cj = col / bx.n[2], ck = col % bx.n[2];
      for (int ci = 0; ci < bx.n[0]; ci++)
        cnt += sph::sub_count(bx.lo[0] + ci, bx.lo[1] + cj, bx.lo[2] + ck, s, hs,
                              img[m][0], img[m][1], img[m][2], R);
    }
  }
  const double np = block_sum((double)cnt, sh);
  if (threadIdx.x == 0) counts[p] = (unsigned long long)np;
}


// floor division for possibly negative cell indices
__device__ __forceinline__ int fdiv(int a, int b) {
  return a >= 0 ? a / b : -((-a + b - 1) / b);
}

// the bin of a sphere centre: cell index floor(c / h) per axis (clamped to
// the domain), bc cells per bin
__device__ __forceinline__ int bin_axis(const SphereBins &B, const Grid &g, int ax,
                                        double c, double h) {
  const int ext[3] = {g.nx, g.ny, g.nz};
  int ic = (int)floor(c / h);
  ic = min(max(ic, 0), ext[ax] - 1);
  return min(ic / B.bc[ax], B.nb[ax] - 1);
}

__global__ void __launch_bounds__(kThreads)
    k_sphere_bin(Grid g, double h, int n, const double *sph, SphereBins B) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int b = (bin_axis(B, g, 0, sph[5 * p], h) * B.nb[1] +
                 bin_axis(B, g, 1, sph[5 * p + 1], h)) * B.nb[2] +
                bin_axis(B, g, 2, sph[5 * p + 2], h);
  const int slot = atomicAdd(B.count + b, 1);
  if (slot < kBinCap) B.items[(size_t)b * kBinCap + slot] = p;
}

// can spheres a and b cover sub-cell centres of a common cell?  Then the
// centres are at most Ra + Rb + sqrt(3) h apart (two points of one cell);
// conservative: the (minimum-image on periodic axes) centre distance
// <= Ra + Rb + 2h
__device__ __forceinline__ bool spheres_near(const Grid &g, double h, const double *a,
                                             const double *b) {
  const int ext[3] = {g.nx, g.ny, g.nz};
  const double lim = a[3] + b[3] + 2.0 * h;
  double d2 = 0.0;
#pragma unroll
  for (int ax = 0; ax < 3; ax++) {
    double d = fabs(b[ax] - a[ax]);
    if (g.per[ax]) {
      const double L = (double)ext[ax] * h;
      if (d > 0.5 * L) d = L - d;
    }
    if (d > lim) return false;
    d2 += d * d;
  }
  return d2 <= lim * lim;
}

// covered sub-cell centres of cell (i,j,k) by sphere q: the image nearest to
// the cell on periodic axes (the oracle's image coordinate c + m (n h); the
// images of one sphere reach disjoint cells, so at most this one covers it)
__device__ __forceinline__ int cover_count(const Grid &g, double h, int s, double hs,
                                           const double *q, int i, int j, int k) {
  const int ext[3] = {g.nx, g.ny, g.nz};
  const int ic[3] = {i, j, k};
  double c[3];
#pragma unroll
  for (int ax = 0; ax < 3; ax++) {
    const double x = ((double)ic[ax] + 0.5) * h;
    double best = q[ax];
    if (g.per[ax]) {
      const double L = (double)ext[ax] * h;
      const double lo = q[ax] + -1.0 * L, hi = q[ax] + 1.0 * L;
      if (fabs(x - lo) < fabs(x - best)) best = lo;
      if (fabs(x - hi) < fabs(x - best)) best = hi;
    }
    if (fabs(x - best) > q[3] + h) return 0;  // no sub-centre within R
    c[ax] = best;
  }
  return sph::sub_count(i, j, k, s, hs, c[0], c[1], c[2], q[3]);
}

// the oracle's cell value of sphere q for `cnt` covered sub-cells
__device__ __forceinline__ double sphere_value(const double *q, double np, int cnt,
                                               int s3, double h, int normalization) {
  if (normalization == 1) {
    const double R = q[3];
    const double rho0 = q[4] / ((4.0 / 3.0) * kPi * (R * R * R));
    return rho0 * ((double)cnt / (double)s3);
  }
  return (q[4] * (double)cnt) / (np * (h * h * h));
}

// neighbour lists: for sphere p the spheres that may share a cell with it --
// the candidates of the bins within R_p + R_max + 2h (+ 2 cells of margin)
// of p's centre cell on every axis (periodic axes wrap; their bins divide
// the axis), then the distance test, then an ascending sort (ranks; the
// entries are distinct).  nn[p] = their number (kNbMax + 1: a full bin or
// more than kNbMax neighbours -- the scatter then scans every sphere);
// p is appended to the list of isolated spheres (nn = 0) or of the others.
constexpr int kNbThreads = 64;

__global__ void __launch_bounds__(kNbThreads)
    k_sphere_neighbours(Grid g, double h, int n, const double *sph, SphereBins B,
                        SphereLists S) {
  __shared__ int cand[kNbMax];
  __shared__ int ncand, overflow;
  const int p = blockIdx.x;
  const double *me = sph + 5 * p;
  if (threadIdx.x == 0) {
    ncand = 0;
    overflow = 0;
  }
  __syncthreads();
  const int ext[3] = {g.nx, g.ny, g.nz};
  int b0[3], nbr[3];
#pragma unroll
  for (int ax = 0; ax < 3; ax++) {
    int ic = (int)floor(me[ax] / h);
    ic = min(max(ic, 0), ext[ax] - 1);
    const int E = (int)((me[3] + B.rmax + 2.0 * h) / h) + 2;
    int lo = fdiv(ic - E, B.bc[ax]), hi = fdiv(ic + E, B.bc[ax]);
    if (!g.per[ax]) {
      lo = max(lo, 0);
      hi = min(hi, B.nb[ax] - 1);
    }
    nbr[ax] = min(hi - lo + 1, B.nb[ax]);
    b0[ax] = lo;
  }
  const int nbins = nbr[0] * nbr[1] * nbr[2];
  for (int t = threadIdx.x; t < nbins; t += blockDim.x) {
    int bb[3] = {t / (nbr[1] * nbr[2]), (t / nbr[2]) % nbr[1], t % nbr[2]};
#pragma unroll
    for (int ax = 0; ax < 3; ax++) {
      bb[ax] += b0[ax];
      if (g.per[ax]) bb[ax] = ((bb[ax] % B.nb[ax]) + B.nb[ax]) % B.nb[ax];
    }
    const int b = (bb[0] * B.nb[1] + bb[1]) * B.nb[2] + bb[2];
    const int m = B.count[b];
    if (m > kBinCap) {
      overflow = 1;
      continue;
    }
    for (int e = 0; e < m; e++) {
      const int q = B.items[(size_t)b * kBinCap + e];
      if (q == p || !spheres_near(g, h, me, sph + 5 * q)) continue;
      const int slot = atomicAdd(&ncand, 1);
      if (slot < kNbMax) cand[slot] = q;
    }
  }
  __syncthreads();
  const int nc = ncand;
  int *out = S.nbr + (size_t)p * kNbMax;
  if (nc <= kNbMax)
    for (int t = threadIdx.x; t < nc; t += blockDim.x) {
      const int q = cand[t];
      int r = 0;
      for (int u = 0; u < nc; u++) r += cand[u] < q;
      out[r] = q;
    }
  if (threadIdx.x == 0) {
    const int nn = (overflow || nc > kNbMax) ? kNbMax + 1 : nc;
    S.nn[p] = nn;
    const int k = nn ? 1 : 0;
    S.list[(size_t)k * n + atomicAdd(S.nlist + k, 1)] = p;
  }
}

// The density of the covered cells of this slab, one CTA per sphere: the
// spheres with neighbours first (list 1: the cell is written by its
// lowest-index covering sphere with the ordered sum), then the isolated
// ones (list 0: every covered cell is the sphere's alone, one plain store
// per cell) -- the heavier CTAs start first.  Grid = n.
template <bool PER>
__global__ void __launch_bounds__(kThreads, 4)
    k_sphere_scatter(Grid g, double h, int s, int n, const double *sph,
                     int normalization, const unsigned long long *counts,
                     SphereLists S) {
  __shared__ sph::Tab tab;
  __shared__ double vt[sph::kVal];  // cell value by covered count (s^3 <= kVal-1)
  __shared__ unsigned short cc[sph::kCells];  // covered counts of the box cells
  const int n1 = S.nlist[1];
  const bool OVERLAP = (int)blockIdx.x < n1;
  const int k = OVERLAP ? 1 : 0;
  const int slot = OVERLAP ? (int)blockIdx.x : (int)blockIdx.x - n1;
  if (slot >= S.nlist[k]) return;
  const int p = S.list[(size_t)k * n + slot];
  const double *me = sph + 5 * p;
  const double R = me[3];
  const double R2 = R * R;
  const double hs = h / (double)s;
  const int s3 = s * s * s;
  const double np = (double)counts[p];
  if (normalization != 1 && np == 0.0) return;  // covers nothing
  const int nn = OVERLAP ? S.nn[p] : 0;
  const int *nbl = S.nbr + (size_t)p * kNbMax;
  const bool scan_all = nn > kNbMax;  // list overflow: every sphere per cell
  const int ntry = scan_all ? n : nn;
  const bool vtab = s3 < sph::kVal;
  if (vtab)
    for (int c = threadIdx.x; c <= s3; c += blockDim.x)
      vt[c] = sphere_value(me, np, c, s3, h, normalization);
  sph::Images<PER> im;
  sph::make_images<PER>(g, h, me[0], me[1], me[2], im);
  const int nimg = im.n;
  auto &img = im.c;
  for (int m = 0; m < nimg; m++) {
    sph::Box bx = sph::box_of(g, h, img[m], R);
    // this slab's planes of the box
    const int xa = bx.lo[0] > g.x0 ? bx.lo[0] : g.x0;
    const int xb = min(bx.lo[0] + bx.n[0] - 1, g.x0 + g.nxl - 1);
    if (bx.cells() == 0 || xa > xb) continue;
    // (tables() also publishes vt)
    const bool tb = sph::tables(tab, bx, s, hs, img[m]) && bx.cells() <= sph::kCells;
    const int ncol = bx.n[1] * bx.n[2];
    for (int col = threadIdx.x; col < ncol; col += blockDim.x) {
      const int cj = col / bx.n[2], ck = col % bx.n[2];
      const int j = bx.lo[1] + cj, kz = bx.lo[2] + ck;
      // the column's counts from its sub-rows' x intervals (the thread's own
      // entries of cc: no barrier)
      if (tb)
        sph::column_counts(tab, bx, s, R2, cj, ck, cc, col, ncol, xa - bx.lo[0],
                           xb - bx.lo[0]);
      for (int i = xa; i <= xb; i++) {
        const int c = tb ? (int)cc[col + (i - bx.lo[0]) * ncol]
                         : sph::sub_count(i, j, kz, s, hs, img[m][0], img[m][1],
                                          img[m][2], R);
        if (!c) continue;
        double v = 0.0;
        if (OVERLAP) {
          // the lowest-index covering sphere writes the cell
          bool mine = true;
          int t = 0;
          for (; t < ntry; t++) {
            const int q = scan_all ? t : nbl[t];
            if (q >= p) break;
            if (scan_all && !spheres_near(g, h, me, sph + 5 * q)) continue;
            const double *sq = sph + 5 * q;
            if (normalization != 1 && counts[q] == 0ull) continue;
            if (cover_count(g, h, s, hs, sq, i, j, kz)) {
              mine = false;
              break;
            }
          }
          if (!mine) continue;
          v = v + (vtab ? vt[c] : sphere_value(me, np, c, s3, h, normalization));
          for (; t < ntry; t++) {
            const int q = scan_all ? t : nbl[t];
            if (q == p) continue;
            if (scan_all && !spheres_near(g, h, me, sph + 5 * q)) continue;
            const double *sq = sph + 5 * q;
            const double nq = (double)counts[q];
            if (normalization != 1 && nq == 0.0) continue;
            const int cq = cover_count(g, h, s, hs, sq, i, j, kz);
            if (cq) v = v + sphere_value(sq, nq, cq, s3, h, normalization);
          }
        } else {
          v = v + (vtab ? vt[c] : sphere_value(me, np, c, s3, h, normalization));
        }
        const long long idx = rowbase(g, i - g.x0, j) + (kz >> 1);
        (((i + j + kz) & 1) ? g.fB : g.fR)[idx] = v;
      }
    }
  }
}

void launch_sphere_counts(const Grid &g, double h, int s, int n, const double *sph,
                          unsigned long long *counts, cudaStream_t st) {
  if (n <= 0) return;
  if (is_periodic(g))
    k_sphere_count<true><<<n, kThreads, 0, st>>>(g, h, s, sph, counts);
  else
    k_sphere_count<false><<<n, kThreads, 0, st>>>(g, h, s, sph, counts);
}

void launch_sphere_bin(const Grid &g, double h, int n, const double *sph,
                       const SphereBins &B, cudaStream_t st) {
  if (n <= 0) return;
  k_sphere_bin<<<(n + kThreads - 1) / kThreads, kThreads, 0, st>>>(g, h, n, sph, B);
}

void launch_sphere_neighbours(const Grid &g, double h, int n, const double *sph,
                              const SphereBins &B, const SphereLists &S, cudaStream_t st) {
  if (n <= 0) return;
  k_sphere_neighbours<<<n, kNbThreads, 0, st>>>(g, h, n, sph, B, S);
}

void launch_sphere_scatter(const Grid &g, double h, int s, int n, const double *sph,
                           int normalization, const unsigned long long *counts,
                           const SphereLists &S, cudaStream_t st) {
  if (n <= 0) return;
  static bool carve = false;  // 4 CTAs of ~40 KB static shared memory per SM
  if (!carve) {
    cudaFuncSetAttribute(k_sphere_scatter<false>,
                         cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_sphere_scatter<true>,
                         cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    carve = true;
  }
  if (is_periodic(g))
    k_sphere_scatter<true><<<n, kThreads, 0, st>>>(g, h, s, n, sph, normalization, counts, S);
  else
    k_sphere_scatter<false><<<n, kThreads, 0, st>>>(g, h, s, n, sph, normalization, counts, S);
}
// ---------------------------------------------------------------------------
// Finest-grid RHS adaptation: f -= term_q for every
// face q the cell touches, in face order.  term_q = (2 alpha) g_d for
// Dirichlet, alpha (h g_n) for Neumann, alpha = -1/h^2 (host-computed, the
// oracle's expressions).  One thread per row; boundary rows do every cell,
// interior rows only z = 0 and z = nz-1.
// ---------------------------------------------------------------------------
struct Terms {
  double t[6];
};

__device__ __forceinline__ void bc_cell(const Grid &g, const Terms &T, int il,
                                        int j, int z) {
  const int i = g.x0 + il;
  const long long e = rowbase(g, il, j) + (z >> 1);
  // masked cells are not unknowns (their f stays 0)
  if (g.codeR && !((((i + j + z) & 1) ? g.codeB : g.codeR)[e] & 64)) return;
  double *f = ((i + j + z) & 1) ? g.fB : g.fR;
  double v = f[e];
  const bool on[6] = {i == 0, i == g.nx - 1, j == 0,
                      j == g.ny - 1, z == 0, z == g.nz - 1};
#pragma unroll
  for (int q = 0; q < 6; q++)
    if (on[q] && !g.per[q >> 1]) v = v - T.t[q];  // periodic: no boundary
  f[e] = v;
}

// every boundary cell exactly once, one thread per cell (each cell's face
// terms in face order in that thread):
//   part A: z = 0 and z = nz-1 of every row            (rows x 2)
//   part B: rows j = 0, ny-1 of every plane, 0 < z < nz-1   (nxl x 2 x (nz-2))
//   part C: planes i = 0, nx-1 held here, 0 < j < ny-1, 0 < z < nz-1
__global__ void __launch_bounds__(kThreads)
    k_bc_adapt(Grid g, Terms T, long long nA, long long nB, int pc0, int pc1) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int nzi = g.nz - 2;
  if (t < nA) {
    const int side = (int)(t & 1);
    const long long r = t >> 1;
    const int j = (int)(r % g.ny), il = (int)(r / g.ny);
    if (side && g.nz == 1) return;
    bc_cell(g, T, il, j, side ? g.nz - 1 : 0);
    return;
  }
  t -= nA;
  if (t < nB) {
    const int z = 1 + (int)(t % nzi);
    const long long r = t / nzi;
    const int side = (int)(r & 1), il = (int)(r >> 1);
    if (side && g.ny == 1) return;
    bc_cell(g, T, il, side ? g.ny - 1 : 0, z);
    return;
  }
  t -= nB;
  const long long per_plane = (long long)(g.ny - 2) * nzi;
  const int z = 1 + (int)(t % nzi);
  const long long r = t / nzi;
  const int j = 1 + (int)(r % (g.ny - 2));
  const int pl = (int)(r / (g.ny - 2));  // 0: plane pc0, 1: plane pc1
  if (per_plane <= 0 || pl > 1) return;
  const int il = pl ? pc1 : pc0;
  if (il < 0 || (pl && pc1 == pc0)) return;
  bc_cell(g, T, il, j, z);
}

void launch_bc_adapt(const Grid &g, const double *terms, const int * /*types*/,
                     cudaStream_t s) {
  Terms T;
  for (int q = 0; q < 6; q++) T.t[q] = terms[q];
  const long long nzi = g.nz > 2 ? g.nz - 2 : 0;
  const long long nA = 2LL * g.nxl * g.ny;
  const long long nB = g.ny > 0 ? 2LL * g.nxl * nzi : 0;
  // local planes of the x faces held by this slab (-1: none)
  const int pc0 = (g.x0 == 0) ? 0 : -1;
  const int pc1 = (g.x0 + g.nxl == g.nx) ? g.nxl - 1 : -1;
  const long long nC = (g.ny > 2 ? 2LL * (g.ny - 2) * nzi : 0);
  const long long total = nA + nB + nC;
  if (g.nxl <= 0 || total <= 0) return;
  int a0 = pc0, a1 = pc1;
  if (a0 < 0) {  // only the last plane: put it first
    a0 = a1;
    a1 = -1;
  }
  k_bc_adapt<<<(unsigned)((total + kThreads - 1) / kThreads), kThreads, 0, s>>>(
      g, T, nA, nB, a0, a1 < 0 ? a0 : a1);
}

// ---------------------------------------------------------------------------
// natural (x slowest) <-> checkerboard-split conversion at the API boundary
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
    k_pack(Grid g, int field, const double *nat) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.nxl * g.ny * g.nz) return;
  const int z = (int)(t % g.nz);
  const long long q = t / g.nz;
  const int j = (int)(q % g.ny);
  const int il = (int)(q / g.ny);
  int col;
  const long long idx = split_index(g, il, j, z, &col);
  double *dst = field ? (col ? g.fB : g.fR) : (col ? g.phiB : g.phiR);
  dst[idx] = nat[t];
}

__global__ void __launch_bounds__(kThreads)
    k_unpack(Grid g, int field, double *nat) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.nxl * g.ny * g.nz) return;
  const int z = (int)(t % g.nz);
  const long long q = t / g.nz;
  const int j = (int)(q % g.ny);
  const int il = (int)(q / g.ny);
  int col;
  const long long idx = split_index(g, il, j, z, &col);
  const double *src = field ? (col ? g.fB : g.fR) : (col ? g.phiB : g.phiR);
  nat[t] = src[idx];
}

// even nz: one CTA per row (il, j), thread k moves the natural pair
// (2k, 2k+1) -- one 16-byte access -- to half-index k of both colour arrays
// (no 64-bit index division per cell)
__global__ void __launch_bounds__(kThreads)
    k_pack_rows(Grid g, int field, const double *nat) {
  const int j = (int)(blockIdx.x % (unsigned)g.ny);
  const int il = (int)(blockIdx.x / (unsigned)g.ny);
  const bool p0 = (g.x0 + il + j) & 1;  // colour of z = 2k
  const double2 *src = reinterpret_cast<const double2 *>(nat + (long long)blockIdx.x * g.nz);
  const long long rb = rowbase(g, il, j);
  double *R = (field ? g.fR : g.phiR) + rb;
  double *B = (field ? g.fB : g.phiB) + rb;
  for (int k = threadIdx.x; k < g.nzh; k += blockDim.x) {
    const double2 v = src[k];
    R[k] = p0 ? v.y : v.x;
    B[k] = p0 ? v.x : v.y;
  }
}

__global__ void __launch_bounds__(kThreads)
    k_unpack_rows(Grid g, int field, double *nat) {
  const int j = (int)(blockIdx.x % (unsigned)g.ny);
  const int il = (int)(blockIdx.x / (unsigned)g.ny);
  const bool p0 = (g.x0 + il + j) & 1;
  double2 *dst = reinterpret_cast<double2 *>(nat + (long long)blockIdx.x * g.nz);
  const long long rb = rowbase(g, il, j);
  const double *R = (field ? g.fR : g.phiR) + rb;
  const double *B = (field ? g.fB : g.phiB) + rb;
  for (int k = threadIdx.x; k < g.nzh; k += blockDim.x) {
    const double r = R[k], b = B[k];
    dst[k] = p0 ? make_double2(b, r) : make_double2(r, b);
  }
}

static unsigned row_threads(int n) {
  return n < kThreads ? (unsigned)((n + 31) / 32 * 32) : (unsigned)kThreads;
}

// natural buffers from the caller (torch / cudaMalloc) are 16-byte aligned;
// the row kernels need even nz and an aligned base, else the per-cell ones
static bool rows_ok(const Grid &g, const void *nat) {
  return (g.nz % 2) == 0 && ((reinterpret_cast<uintptr_t>(nat) & 15) == 0) &&
         (long long)g.nxl * g.ny < (1LL << 31);
}

void launch_pack(const Grid &g, int field, const double *nat, cudaStream_t s) {
  const long long total = (long long)g.nxl * g.ny * g.nz;
  if (total <= 0) return;
  if (rows_ok(g, nat))
    k_pack_rows<<<(unsigned)(g.nxl * g.ny), row_threads(g.nzh), 0, s>>>(g, field, nat);
  else
    k_pack<<<(unsigned)((total + kThreads - 1) / kThreads), kThreads, 0, s>>>(g, field,
                                                                               nat);
}

void launch_unpack(const Grid &g, int field, double *nat, cudaStream_t s) {
  const long long total = (long long)g.nxl * g.ny * g.nz;
  if (total <= 0) return;
  if (rows_ok(g, nat))
    k_unpack_rows<<<(unsigned)(g.nxl * g.ny), row_threads(g.nzh), 0, s>>>(g, field, nat);
  else
    k_unpack<<<(unsigned)((total + kThreads - 1) / kThreads), kThreads, 0, s>>>(g, field,
                                                                                 nat);
}

// ---------------------------------------------------------------------------
// Periodic ghost refresh ("near boundary values are then
// copied to the periodic neighbour's ghost layer"): every ghost element of
// both Phi colours that mirrors an interior cell is copied from it -- ghost
// rows 0 / ny+1 of the interior planes (y periodic) and the whole ghost
// planes 0 / nxl+1 incl. their ghost rows (x periodic, grid held whole).
// Sources are interior elements only, so one pass needs no ordering.
// ---------------------------------------------------------------------------
__host__ __device__ inline long long periodic_fill_items(const Grid &g) {
  if (!(g.gx || g.per[1])) return 0;
  return ((g.gx ? 2LL * (g.ny + 2) : 0) + (g.per[1] ? 2LL * g.nxl : 0)) * g.nzh;
}

__device__ __forceinline__ void periodic_fill_elem(const Grid &g, long long t) {
  const long long rowsx = g.gx ? 2LL * (g.ny + 2) : 0;        // planes 0, nxl+1
  const int k = (int)(t % g.nzh);
  const long long r = t / g.nzh;
  int ap, ar;  // ghost element's array plane / row
  if (r < rowsx) {
    ap = (r / (g.ny + 2)) ? g.nxl + 1 : 0;
    ar = (int)(r % (g.ny + 2));
  } else {
    const long long q = r - rowsx;
    ap = 1 + (int)(q >> 1);
    ar = (q & 1) ? g.ny + 1 : 0;
  }
  int sp = ap, sr = ar;  // its interior source
  if (g.gx) sp = ap == 0 ? g.nxl : (ap == g.nxl + 1 ? 1 : ap);
  if (g.per[1]) sr = ar == 0 ? g.ny : (ar == g.ny + 1 ? 1 : ar);
  if (sr == 0 || sr == g.ny + 1) return;  // non-periodic ghost row: stays 0
  const long long dst = (long long)ap * g.plane + (long long)ar * g.pz + k;
  const long long src = (long long)sp * g.plane + (long long)sr * g.pz + k;
  g.phiR[dst] = g.phiR[src];
  g.phiB[dst] = g.phiB[src];
}

__global__ void __launch_bounds__(kThreads) k_periodic_fill(Grid g) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < periodic_fill_items(g)) periodic_fill_elem(g, t);
}

void launch_periodic_fill(const Grid &g, cudaStream_t s) {
  if (!(g.gx || g.per[1])) return;
  const long long rows = (g.gx ? 2LL * (g.ny + 2) : 0) + (g.per[1] ? 2LL * g.nxl : 0);
  const long long total = rows * g.nzh;
  if (total <= 0) return;
  k_periodic_fill<<<(unsigned)((total + kThreads - 1) / kThreads), kThreads, 0, s>>>(g);
}



// ---------------------------------------------------------------------------
// The coarse end of the V-cycle in one persistent kernel (the "tail"): the
// levels ls..L-1 of a cycle -- pre-smoothing, residual + restriction down to
// the coarsest grid, CG there, prolongation + correction and post-smoothing
// back up to level ls -- run by one thread-block
// cluster, the steps separated by cluster barriers (barrier.cluster
// arrive.release / wait.acquire: the global-memory writes of one step are
// visible to every CTA of the cluster in the next).  On these small,
// L2-resident levels (<= 32^3 cells) every step of the launch-per-step path
// costs a kernel launch of a few microseconds for well under a microsecond
// of work.  The per-cell arithmetic is the device functions the per-step
// kernels use (smooth_pair, restrict_cell, prolong_cell, periodic_fill_elem,
// cg_cta with the standalone CG's thread count), so the iterates are bitwise
// those of the per-step path.
// ---------------------------------------------------------------------------
namespace {
namespace cgr = cooperative_groups;
}

template <bool PER>
__global__ void __launch_bounds__(kTailThreads)
    k_vcycle_tail(TailLevels T, int nu1, int nu2, double alpha, double tol, int maxit,
                  int cg_nthr, double *cg_scr, int *iters_out) {
  extern __shared__ double tail_sm[];
  __shared__ double part[2][64];
  cgr::cluster_group cl = cgr::this_cluster();
  const long long t0 = (long long)cl.block_rank() * blockDim.x + threadIdx.x;
  const long long nt = (long long)cl.num_blocks() * blockDim.x;
  auto half = [&](const Grid &g, int color, int from_zero) {
    const long long n = smooth_items(g);
    for (long long t = t0; t < n; t += nt) smooth_pair<PER>(g, color, from_zero, t);
    cl.sync();
  };
  auto fill = [&](const Grid &g) {
    if (!PER) return;
    const long long n = periodic_fill_items(g);
    if (n == 0) return;
    for (long long t = t0; t < n; t += nt) periodic_fill_elem(g, t);
    cl.sync();
  };
  for (int l = 0; l + 1 < T.n; l++) {
    const Grid &g = T.g[l];
    if (nu1 == 0) {  // Phi of a coarse level starts from 0
      const long long ne = grid_elems(g);
      for (long long e = t0; e < ne; e += nt) {
        g.phiR[e] = 0.0;
        g.phiB[e] = 0.0;
      }
      cl.sync();
    }
    for (int s = 0; s < nu1; s++) {
      half(g, 0, s == 0);  // the first red sweep from Phi = 0
      half(g, 1, 0);
    }
    const long long n = restrict_items(g);
    for (long long t = t0; t < n; t += nt) restrict_cell<PER>(g, T.g[l + 1], t);
    cl.sync();
  }
  const Grid &gc = T.g[T.n - 1];
  if (cl.block_rank() == 0) {
    const long long N = (long long)gc.nx * gc.ny * gc.nz;
    // (at most four elements per thread here -- eight would spill --:
    // vcycle_tail_supported keeps larger coarsest grids out of the tail, so
    // that the tail and the standalone CG run the same arithmetic.)  Only
    // the standalone CG's threads take part, behind barrier 1: the same
    // warps, so the same reduction trees, with fewer warps to wait for.
    const int pad = (cg_nthr + 31) / 32 * 32;
    if (N <= kCgSmemMax && (N + cg_nthr - 1) / cg_nthr <= 4) {
      if ((int)threadIdx.x < pad)
        cg_cta_fast<PER, 4>(gc, tail_sm, part, tol, maxit, iters_out, cg_nthr,
                            pad < (int)blockDim.x ? 1 : 0, pad);
    } else if (N <= kCgSmemMax) {
      cg_cta<PER>(gc, tail_sm, part, tol, maxit, iters_out, cg_nthr);
    } else {
      cg_cta<PER>(gc, cg_scr, part, tol, maxit, iters_out, cg_nthr);
    }
  }
  cl.sync();
  fill(gc);
  for (int l = T.n - 2; l >= 0; l--) {
    const Grid &g = T.g[l];
    const long long n = prolong_items(g);
    for (long long t = t0; t < n; t += nt) prolong_cell(g, T.g[l + 1], alpha, t);
    cl.sync();
    fill(g);
    for (int s = 0; s < nu2; s++) {
      half(g, 0, 0);
      half(g, 1, 0);
    }
  }
}

int tail_cluster_ctas() {
  static int n = -1;
  if (n < 0) {
    // the largest cluster (<= 16, non-portable above 8) the device runs
    cudaFuncSetAttribute(k_vcycle_tail<false>,
                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_vcycle_tail<true>,
                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    n = 0;
    for (int c = 16; c >= 1 && n == 0; c /= 2) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c);
      cfg.blockDim = dim3(kTailThreads);
      cfg.dynamicSmemBytes = 0;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, k_vcycle_tail<false>, &cfg) ==
              cudaSuccess &&
          ncl > 0)
        n = c;
    }
    cudaGetLastError();
  }
  return n;
}

bool vcycle_tail_supported(const Grid &coarsest) {
  const long long N = (long long)coarsest.nx * coarsest.ny * coarsest.nz;
  const int thr = cg_threads(coarsest);
  return tail_cluster_ctas() > 0 && N <= kCgSmemMax && thr <= kTailThreads &&
         (N + thr - 1) / thr <= 4 &&
         coarsest.nxl == coarsest.nx;
}

template <bool PER>
static int launch_tail(const TailLevels &T, int nu1, int nu2, double alpha, double tol,
                       int maxit, double *cg_scr, int *iters_out, cudaStream_t s) {
  const Grid &gc = T.g[T.n - 1];
  const long long N = (long long)gc.nx * gc.ny * gc.nz;
  const size_t smem = cg_area_doubles(N) * sizeof(double);
  static size_t configured = 48 * 1024;
  if (smem > configured) {
    cudaFuncSetAttribute(k_vcycle_tail<PER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    configured = smem;
  }
  const int nc = tail_cluster_ctas();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nc);
  cfg.blockDim = dim3(kTailThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = nc;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_vcycle_tail<PER>, T, nu1, nu2, alpha, tol, maxit,
                            cg_threads(gc), cg_scr, iters_out) == cudaSuccess
             ? 0
             : -1;
}

int launch_vcycle_tail(const TailLevels &T, int nu1, int nu2, double alpha, double tol,
                       int maxit, double *cg_scr, int *iters_out, cudaStream_t s) {
  if (is_periodic(T.g[0]))
    return launch_tail<true>(T, nu1, nu2, alpha, tol, maxit, cg_scr, iters_out, s);
  return launch_tail<false>(T, nu1, nu2, alpha, tol, maxit, cg_scr, iters_out, s);
}

}  // namespace mg
