// Coarsest-grid CG on a thread-block cluster (sm_100a): the same
// Hestenes-Stiefel iteration as k_coarse_cg -- x = 0, r = p = b, q = A p,
// alpha = rho / (p.q), x += alpha p, r -= alpha q, stop at
// sqrt(rho') <= tol ||b|| or maxit, p = r + beta p -- with the unknowns
// (natural order) split into kCK contiguous chunks, one per CTA of the
// cluster, each chunk's vectors in that CTA's shared memory.  The matrix-
// vector product reads neighbour values of other chunks through distributed
// shared memory; dot products are per-CTA partials (fixed shuffle trees over
// the warp and over the warps) that every thread sums by a fixed pairwise
// tree in cluster-rank order after a cluster barrier, so all CTAs take the
// same decisions.  The large coarsest grids of
// agglomerated multi-GPU runs (64 x 8 x 8 at P = 8) spread over kCK SMs.
// Round 1 (three cluster barriers per iteration, partials read remotely):
// 0.42 ms for 64 x 8 x 8 vs 0.48 ms single-CTA; clusters of 4 (0.51) and 16
// (0.45, non-portable) were slower.  Round 2: the Chronopoulos-Gear kernel
// below (k_coarse_cg_cluster_cg) for chunks of up to 2048 unknowns: 0.24 ms
// per 64 x 8 x 8 solve (events; this Hestenes-Stiefel kernel 0.39).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "mg_internal.h"

namespace cgr = cooperative_groups;

namespace mg {

namespace {

constexpr int kCK = 8;          // CTAs per cluster (portable size)
constexpr int kCT = 512;        // threads per CTA
constexpr int kChunkMax = 4096; // unknowns per CTA

__device__ __forceinline__ int centre_dc(const Grid &g, int i, int j, int z) {
  int d = 6;
  if (i == 0) d += g.dface[0];
  if (i == g.nx - 1) d += g.dface[1];
  if (j == 0) d += g.dface[2];
  if (j == g.ny - 1) d += g.dface[3];
  if (z == 0) d += g.dface[4];
  if (z == g.nz - 1) d += g.dface[5];
  return d;
}

__device__ __forceinline__ long long split_at(const Grid &g, int n, int *col) {
  const int z = n % g.nz, t = n / g.nz;
  const int j = t % g.ny, i = t / g.ny;
  *col = (g.x0 + i + j + z) & 1;
  return (long long)(i + 1) * g.plane + (long long)(j + 1) * g.pz + (z >> 1);
}

// this CTA's partial of a dot product (valid in warp 0): fixed butterfly
// trees over the warp, then over the warp partials (zero-padded to 32)
__device__ __forceinline__ double cta_partial(double v, double *wpart) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) wpart[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? wpart[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  return s;
}

}  // namespace

// Two cluster barriers per iteration: (1) the direction p = r + beta p_old
// is formed where the matrix-vector product needs it (own cell and the six
// neighbours, read from the owners' r and p_old -- the same expression, so
// the same bits as a separate update pass) and stored into the other of two
// p buffers; (2) each CTA pushes its dot-product partial into slot [rank] of
// every CTA's shared memory before the barrier, so that after it the sum in
// rank order reads local shared memory only.
template <bool PER>
__global__ void __cluster_dims__(kCK, 1, 1) __launch_bounds__(kCT)
    k_coarse_cg_cluster(Grid g, double tol, int maxit, int *iters_out, int chunk) {
  using NB = typename std::conditional<PER, unsigned short, unsigned char>::type;
  cgr::cluster_group cl = cgr::this_cluster();
  const int rank = (int)cl.block_rank();
  extern __shared__ __align__(16) double cgs[];
  __shared__ double slots[2][kCK];        // every CTA's partials (pushed here)
  __shared__ double wpart[kCT / 32];
  __shared__ const double *rr[kCK];       // every CTA's r (distributed smem)
  __shared__ const double *rpa[kCK];      // every CTA's p buffers
  __shared__ const double *rpb[kCK];
  __shared__ double *rslot[kCK];          // every CTA's slots

  const int N = g.nx * g.ny * g.nz;
  const int n0 = rank * chunk;
  const int nl = max(0, min(chunk, N - n0));  // unknowns of this CTA
  double *pa = cgs, *pb = cgs + chunk, *x = cgs + 2 * chunk, *r = cgs + 3 * chunk,
         *q = cgs + 4 * chunk;
  NB *nb = reinterpret_cast<NB *>(cgs + 5 * chunk);
  signed char *dc = reinterpret_cast<signed char *>(nb + chunk);
  if (threadIdx.x < kCK) {
    rr[threadIdx.x] = cl.map_shared_rank(r, (int)threadIdx.x);
    rpa[threadIdx.x] = cl.map_shared_rank(pa, (int)threadIdx.x);
    rpb[threadIdx.x] = cl.map_shared_rank(pb, (int)threadIdx.x);
    rslot[threadIdx.x] = cl.map_shared_rank(&slots[0][0], (int)threadIdx.x);
  }
  const int sx = g.ny * g.nz, sy = g.nz;
  const int wx = (g.nx - 1) * sx, wy = (g.ny - 1) * sy, wz = g.nz - 1;

  // geometry (neighbour bits as k_coarse_cg: 0-5 inside, 6-11 periodic) and b
  double acc = 0.0;
  for (int e = threadIdx.x; e < nl; e += blockDim.x) {
    const int n = n0 + e;
    const int z = n % g.nz, t = n / g.nz;
    const int j = t % g.ny, i = t / g.ny;
    const int in[6] = {i > 0, i < g.nx - 1, j > 0, j < g.ny - 1, z > 0, z < g.nz - 1};
    unsigned m = 0;
#pragma unroll
    for (int a = 0; a < 6; a++)
      m |= in[a] ? (1u << a) : ((PER && g.per[a >> 1]) ? (64u << a) : 0u);
    nb[e] = (NB)m;
    dc[e] = (signed char)centre_dc(g, i, j, z);
    int col;
    const long long idx = split_at(g, n, &col);
    const double b = col ? g.fB[idx] : g.fR[idx];
    x[e] = 0.0;
    r[e] = b;
    pb[e] = 0.0;  // p_old of the first iteration: p = r + 0 * 0 = r
    acc = acc + b * b;
  }
  __syncthreads();  // the pointer tables
  int sl = 0;
  // sum over the cluster in rank order; one CTA barrier + one cluster barrier
  auto cluster_sum = [&](double v) {
    const double s = cta_partial(v, wpart);
    if (threadIdx.x == 0)
#pragma unroll
      for (int k = 0; k < kCK; k++) rslot[k][sl * kCK + rank] = s;
    cl.sync();
    // the CTA partials in rank order, as a fixed pairwise tree
    double t[kCK];
#pragma unroll
    for (int k = 0; k < kCK; k++) t[k] = slots[sl][k];
#pragma unroll
    for (int w = 1; w < kCK; w <<= 1)
#pragma unroll
      for (int k = 0; k + w < kCK; k += 2 * w) t[k] = t[k] + t[k + w];
    sl ^= 1;
    return t[0];
  };
  double rho = cluster_sum(acc);  // the barrier also publishes r
  const double bnorm = sqrt(rho);
  const double c = g.c;
  double beta = 0.0;
  int it = 0;
  if (bnorm > 0.0) {
    while (it < maxit) {
      // p_old in buffer a on odd iterations, b on even ones (p_new the other)
      const bool old_a = (it & 1) != 0;
      double *pn = old_a ? pb : pa;
      const double *po = old_a ? pa : pb;
      // p = r + beta p_old of global unknown m: own chunk from local shared
      // memory (shared-memory loads), other chunks through DSMEM
      auto P = [&](int m) {
        const int e = m - n0;
        if ((unsigned)e < (unsigned)chunk) return r[e] + beta * po[e];
        const int k = m / chunk, ek = m - k * chunk;
        const double *pk = old_a ? rpa[k] : rpb[k];
        return rr[k][ek] + beta * pk[ek];
      };
      acc = 0.0;
      for (int e = threadIdx.x; e < nl; e += blockDim.x) {
        const int n = n0 + e;
        const unsigned m = nb[e];
        const double xm = (m & 1) ? P(n - sx) : ((PER && (m & 64)) ? P(n + wx) : 0.0);
        const double xp = (m & 2) ? P(n + sx) : ((PER && (m & 128)) ? P(n - wx) : 0.0);
        const double ym = (m & 4) ? P(n - sy) : ((PER && (m & 256)) ? P(n + wy) : 0.0);
        const double yp = (m & 8) ? P(n + sy) : ((PER && (m & 512)) ? P(n - wy) : 0.0);
        const double zm = (m & 16) ? P(n - 1) : ((PER && (m & 1024)) ? P(n + wz) : 0.0);
        const double zp = (m & 32) ? P(n + 1) : ((PER && (m & 2048)) ? P(n - wz) : 0.0);
        const double s = ((((xm + xp) + ym) + yp) + zm) + zp;
        const double p = P(n);
        pn[e] = p;
        const double qn = c * ((double)dc[e] * p - s);
        q[e] = qn;
        acc = acc + p * qn;
      }
      const double pq = cluster_sum(acc);
      const double a = rho / pq;
      acc = 0.0;
      for (int e = threadIdx.x; e < nl; e += blockDim.x) {
        x[e] = x[e] + a * pn[e];
        const double rn = r[e] - a * q[e];
        r[e] = rn;
        acc = acc + rn * rn;
      }
      const double rho1 = cluster_sum(acc);
      it++;
      if (sqrt(rho1) <= tol * bnorm) break;
      beta = rho1 / rho;
      rho = rho1;
    }
  }
  for (int e = threadIdx.x; e < nl; e += blockDim.x) {
    int col;
    const long long idx = split_at(g, n0 + e, &col);
    (col ? g.phiB : g.phiR)[idx] = x[e];
  }
  if (rank == 0 && threadIdx.x == 0 && iters_out) *iters_out = it;
  cl.sync();  // no CTA exits while another may still read its smem
}

// The Chronopoulos-Gear form (reading c8; k_coarse_cg's cg_cta_cg) on the
// cluster, per-unknown r, p, s = Ap, w = Ar, x in registers (E per thread):
// per iteration the updates, r published in shared memory, then
//   barrier.cluster.arrive.release
//   w = A r and the partial dots of the unknowns whose six neighbours are in
//     this CTA's chunk (no remote value needed)
//   barrier.cluster.wait.acquire
//   the unknowns with a neighbour in another chunk (distributed shared memory)
//   the two partials (gamma = (r, r), delta = (w, r)) pushed into every CTA's
//   slots, cluster barrier, their sum in rank order
// so the first barrier's latency hides behind the interior products and
// only one reduction is needed.  Neighbour handles: >= 0 a local index (the
// zero slot `chunk` outside the level), < 0 the global unknown -h-1 of
// another chunk.
template <bool PER, int E>
__global__ void __cluster_dims__(kCK, 1, 1) __launch_bounds__(kCT)
    k_coarse_cg_cluster_cg(Grid g, double tol, int maxit, int *iters_out, int chunk) {
  cgr::cluster_group cl = cgr::this_cluster();
  const int rank = (int)cl.block_rank();
  extern __shared__ __align__(16) double cgs[];
  __shared__ double slots[2][2 * kCK];  // every CTA's (gamma, delta) partials
  __shared__ double wpart[2][kCT / 32];
  __shared__ const double *rr[kCK];     // every CTA's r (distributed smem)
  __shared__ double *rslot[kCK];        // every CTA's slots
  const int N = g.nx * g.ny * g.nz;
  const int n0 = rank * chunk;
  const int nl = max(0, min(chunk, N - n0));
  double *rs = cgs;  // chunk + 1 (zero slot)
  if (threadIdx.x < kCK) {
    rr[threadIdx.x] = cl.map_shared_rank(rs, (int)threadIdx.x);
    rslot[threadIdx.x] = cl.map_shared_rank(&slots[0][0], (int)threadIdx.x);
  }
  const int sx = g.ny * g.nz, sy = g.nz;
  const int wx = (g.nx - 1) * sx, wy = (g.ny - 1) * sy, wz = g.nz - 1;
  int hd[E][6];
  bool act[E], inner[E];
  unsigned long long dpk = 0;
  double r[E], p[E], sv[E], w[E], x[E];
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int el = (int)threadIdx.x + e * (int)blockDim.x;
    act[e] = el < nl;
    inner[e] = true;
    r[e] = p[e] = sv[e] = w[e] = x[e] = 0.0;
#pragma unroll
    for (int a = 0; a < 6; a++) hd[e][a] = chunk;
    if (act[e]) {
      const int n = n0 + el;
      const int z = n % g.nz, t = n / g.nz;
      const int j = t % g.ny, i = t / g.ny;
      const bool in[6] = {i > 0, i < g.nx - 1, j > 0, j < g.ny - 1, z > 0, z < g.nz - 1};
      const int kin[6] = {n - sx, n + sx, n - sy, n + sy, n - 1, n + 1};
      const int kpe[6] = {n + wx, n - wx, n + wy, n - wy, n + wz, n - wz};
#pragma unroll
      for (int a = 0; a < 6; a++) {
        const int m = in[a] ? kin[a] : ((PER && g.per[a >> 1]) ? kpe[a] : -1);
        if (m < 0) {
          hd[e][a] = chunk;  // outside the level: the zero slot
        } else if (m >= n0 && m < n0 + chunk) {
          hd[e][a] = m - n0;
        } else {
          hd[e][a] = -m - 1;
          inner[e] = false;
        }
      }
      dpk |= (unsigned long long)centre_dc(g, i, j, z) << (4 * e);
      int col;
      const long long idx = split_at(g, n, &col);
      r[e] = col ? g.fB[idx] : g.fR[idx];
      rs[el] = r[e];
    }
  }
  if (threadIdx.x == 0) rs[chunk] = 0.0;
  const double c = g.c;
  int sl = 0;
  auto nbv = [&](int h) {
    if (h >= 0) return rs[h];
    const int m = -h - 1;
    const int k = m / chunk;
    return rr[k][m - k * chunk];
  };
  auto product = [&](int e, double &gg, double &dl) {
    const double s = ((((nbv(hd[e][0]) + nbv(hd[e][1])) + nbv(hd[e][2])) + nbv(hd[e][3])) +
                      nbv(hd[e][4])) + nbv(hd[e][5]);
    const double d = (double)(int)((dpk >> (4 * e)) & 15u);
    w[e] = c * (d * r[e] - s);
    gg = gg + r[e] * r[e];
    dl = dl + w[e] * r[e];
  };
  // w = A r (r published in shared memory before the call) and the global
  // (gamma, delta), as described above
  auto product_sum = [&]() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    double gi = 0.0, di = 0.0, gb = 0.0, db = 0.0;
#pragma unroll
    for (int e = 0; e < E; e++)
      if (act[e] && inner[e]) product(e, gi, di);
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
#pragma unroll
    for (int e = 0; e < E; e++)
      if (act[e] && !inner[e]) product(e, gb, db);
    double v0 = gi + gb, v1 = di + db;  // per thread: interior then boundary
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v0 += __shfl_xor_sync(0xffffffffu, v0, o);
      v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    }
    if ((threadIdx.x & 31) == 0) {
      wpart[0][threadIdx.x >> 5] = v0;
      wpart[1][threadIdx.x >> 5] = v1;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int nw = (int)(blockDim.x >> 5);
      double a0 = threadIdx.x < nw ? wpart[0][threadIdx.x] : 0.0;
      double a1 = threadIdx.x < nw ? wpart[1][threadIdx.x] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      }
      if (threadIdx.x < kCK) {
        rslot[threadIdx.x][sl * 2 * kCK + rank] = a0;
        rslot[threadIdx.x][sl * 2 * kCK + kCK + rank] = a1;
      }
    }
    cl.sync();
    double t0[kCK], t1[kCK];
#pragma unroll
    for (int k = 0; k < kCK; k++) {
      t0[k] = slots[sl][k];
      t1[k] = slots[sl][kCK + k];
    }
#pragma unroll
    for (int wd = 1; wd < kCK; wd <<= 1)
#pragma unroll
      for (int k = 0; k + wd < kCK; k += 2 * wd) {
        t0[k] = t0[k] + t0[k + wd];
        t1[k] = t1[k] + t1[k + wd];
      }
    sl ^= 1;
    return make_double2(t0[0], t1[0]);
  };
  __syncthreads();  // the pointer tables and r of this CTA
  double2 gd = product_sum();
  double gamma = gd.x;
  const double bnorm = sqrt(gamma);
  int it = 0;
  if (bnorm > 0.0) {
    double alpha = gamma / gd.y;
#pragma unroll
    for (int e = 0; e < E; e++) {
      p[e] = r[e];
      sv[e] = w[e];
    }
    while (it < maxit) {
#pragma unroll
      for (int e = 0; e < E; e++) {
        x[e] = x[e] + alpha * p[e];
        r[e] = r[e] - alpha * sv[e];
        if (act[e]) rs[(int)threadIdx.x + e * (int)blockDim.x] = r[e];
      }
      it++;
      gd = product_sum();
      if (sqrt(gd.x) <= tol * bnorm) break;
      const double beta = gd.x / gamma;
      alpha = gd.x / (gd.y - beta * (gd.x / alpha));
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
    int col;
    const long long idx = split_at(g, n0 + (int)threadIdx.x + e * (int)blockDim.x, &col);
    (col ? g.phiB : g.phiR)[idx] = x[e];
  }
  if (rank == 0 && threadIdx.x == 0 && iters_out) *iters_out = it;
  cl.sync();  // no CTA exits while another may still read its smem
}

bool coarse_cg_cluster_supported(const Grid &g) {
  const long long N = (long long)g.nx * g.ny * g.nz;
  // from 4096 unknowns (64 x 8 x 8: 0.42 vs 0.48 ms single-CTA); on 32 x 8 x 8
  // the three cluster barriers per iteration cost more than they save
  return g.nxl == g.nx && g.x0 == 0 && N >= 4096 && (N + kCK - 1) / kCK <= kChunkMax;
}

// the Chronopoulos-Gear cluster kernel for chunks of up to 4 unknowns per
// thread (N <= 8 x 2048); larger chunks take the Hestenes-Stiefel one
template <bool PER, int E>
static void launch_cc_cg(const Grid &g, double tol, int maxit, int *iters_out,
                         int chunk, cudaStream_t s) {
  const size_t smem = (size_t)(chunk + 1) * sizeof(double);
  static size_t configured = 48 * 1024;
  if (smem > configured) {
    cudaFuncSetAttribute(k_coarse_cg_cluster_cg<PER, E>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  k_coarse_cg_cluster_cg<PER, E><<<kCK, kCT, smem, s>>>(g, tol, maxit, iters_out, chunk);
}

template <bool PER>
static void launch_cc(const Grid &g, double tol, int maxit, int *iters_out,
                      cudaStream_t s) {
  const int N = g.nx * g.ny * g.nz;
  const int chunk = (N + kCK - 1) / kCK;
  if (chunk <= kCT) return launch_cc_cg<PER, 1>(g, tol, maxit, iters_out, chunk, s);
  if (chunk <= 2 * kCT) return launch_cc_cg<PER, 2>(g, tol, maxit, iters_out, chunk, s);
  if (chunk <= 4 * kCT) return launch_cc_cg<PER, 4>(g, tol, maxit, iters_out, chunk, s);
  using NB = typename std::conditional<PER, unsigned short, unsigned char>::type;
  const size_t smem = (size_t)chunk * (5 * sizeof(double) + sizeof(NB) + 1);
  static size_t configured = 0;
  static bool nonportable = false;
  if (kCK > 8 && !nonportable) {
    cudaFuncSetAttribute(k_coarse_cg_cluster<PER>,
                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    nonportable = true;
  }
  if (smem > configured) {
    cudaFuncSetAttribute(k_coarse_cg_cluster<PER>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  const int threads = chunk < kCT ? (chunk + 31) / 32 * 32 : kCT;
  k_coarse_cg_cluster<PER><<<kCK, threads, smem, s>>>(g, tol, maxit, iters_out, chunk);
}

void launch_coarse_cg_cluster(const Grid &g, double tol, int maxit, int *iters_out,
                              cudaStream_t s) {
  if (is_periodic(g))
    launch_cc<true>(g, tol, maxit, iters_out, s);
  else
    launch_cc<false>(g, tol, maxit, iters_out, s);
}

}  // namespace mg
