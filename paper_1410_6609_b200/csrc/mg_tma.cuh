// Shared device helpers of the plane-marching TMA kernels (mg_march.cu):
// mbarrier / TMA PTX wrappers, tile geometry.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "mg_internal.h"

namespace mg {
namespace {

constexpr int kTY = 8;        // rows per CTA (one warp per row)
constexpr int kICH = 16;      // max planes per CTA (x-chunk)
constexpr int kSlots = 5;     // ring depth: planes q-1, q, q+1 in use, 2 in flight
constexpr int kThreadsM = kTY * 32;
constexpr int kZT = 128;      // z-tile (half-entries) of the residual kernels

__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(cnt));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar,
                                               unsigned bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar,
                                          unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(20000u)  // suspend-time hint (ns): yield, do not spin
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *tm,
                                            int c0, int c1, int c2,
                                            unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::"
      "bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(c1), "r"(c2),
      "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// bulk prefetch of `bytes` (a multiple of 16) of global memory into L2
__device__ __forceinline__ void prefetch_l2_bulk(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ int centre_dm(const Grid &g, int i, int j, int z) {
  int d = 6;
  if (i == 0) d += g.dface[0];
  if (i == g.nx - 1) d += g.dface[1];
  if (j == 0) d += g.dface[2];
  if (j == g.ny - 1) d += g.dface[3];
  if (z == 0) d += g.dface[4];
  if (z == g.nz - 1) d += g.dface[5];
  return d;
}

// masked levels with byte codes (bits 0-5 kappa in {0,1} for faces x-,x+,
// y-,y+,z-,z+, bit 6 fluid): number of Dirichlet faces the cell touches,
// and t = sum_q kappa_q phi_q in the fixed face order (kappa as 0.0 / 1.0,
// the same products and order as the variable-coefficient kernels)
__device__ __forceinline__ int ndir_m(const Grid &g, int i, int j, int z) {
  return (i == 0 && g.dface[0] > 0) + (i == g.nx - 1 && g.dface[1] > 0) +
         (j == 0 && g.dface[2] > 0) + (j == g.ny - 1 && g.dface[3] > 0) +
         (z == 0 && g.dface[4] > 0) + (z == g.nz - 1 && g.dface[5] > 0);
}

// kappa in {0,1}: kappa*phi is phi or a signed zero; selecting +0 instead
// changes at most the sign of an exactly-zero sum, never a nonzero value
// face codes of a pair of fluid cells with all six faces open (kappa = 1):
// 0x7F per cell (bit 6 fluid, bits 0-5 the faces)
constexpr unsigned kOpenPair = 0x7F7Fu;

__device__ __forceinline__ double ksum(unsigned cd, double xm, double xp,
                                       double ym, double yp, double zm,
                                       double zp) {
  const double t0 = (cd & 1) ? xm : 0.0, t1 = (cd & 2) ? xp : 0.0;
  const double t2 = (cd & 4) ? ym : 0.0, t3 = (cd & 8) ? yp : 0.0;
  const double t4 = (cd & 16) ? zm : 0.0, t5 = (cd & 32) ? zp : 0.0;
  return ((((t0 + t1) + t2) + t3) + t4) + t5;
}

__device__ __forceinline__ double kdiag(const Grid &g, unsigned cd, int i, int j,
                                        int z) {
  return (double)(__popc(cd & 63u) + 2 * ndir_m(g, i, j, z));
}

__host__ __device__ inline int round128(int bytes) { return (bytes + 127) / 128 * 128; }

// smoother ring slot: (TY + 2) rows of pz doubles
__host__ __device__ inline int slot_doubles(int pz) {
  return round128((kTY + 2) * pz * 8) / 8;
}

// residual kernels: z-tiles of ZT half-entries.  A row of pz <= ZT + 3 is
// one tile loaded whole (box = pz); longer rows are cut into tiles whose TMA
// box (ZT + 4 wide, start a multiple of 4) lies inside [0, pz): the z-halo
// element of a seam comes from the overlap, never from out-of-bounds reads.
constexpr int kZB = kZT + 4;
__host__ __device__ inline bool rsingle(const Grid &g) { return g.nzh <= kZT; }
__host__ __device__ inline int rbox0(const Grid &g) { return rsingle(g) ? g.pz : kZB; }
__host__ __device__ inline int rntiles(const Grid &g) {
  return rsingle(g) ? 1 : (g.nzh + kZT - 1) / kZT;
}
__host__ __device__ inline int rtile_c0(const Grid &g, int kz0) {
  if (rsingle(g)) return 0;
  int c0 = kz0 - 4;
  if (c0 < 0) c0 = 0;
  if (c0 > g.pz - kZB) c0 = g.pz - kZB;
  return c0;
}
// residual ring slot: (TY + 2) rows of rbox0 doubles
__host__ __device__ inline int rslot_doubles() {
  return round128((kTY + 2) * kZB * 8) / 8;
}

// x-chunk length: 16 planes, halved (down to 2, even for the restriction
// pairs) while the grid would have fewer than ~8 CTAs per SM (nsm: the
// device's SM count)
__host__ __device__ inline int chunk_planes(int nxl, int tiles_per_plane_set, int nsm) {
  int ich = kICH;
  while (ich > 2 && (long long)((nxl + ich - 1) / ich) * tiles_per_plane_set < nsm * 8)
    ich >>= 1;
  return ich;
}

__device__ __forceinline__ double2 lds2(const double *p) {
  return *reinterpret_cast<const double2 *>(p);
}

}  // namespace

}  // namespace mg
