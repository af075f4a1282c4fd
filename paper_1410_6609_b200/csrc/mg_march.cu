// Plane-marching RBGS half-sweep for sm_100a with TMA-staged neighbours.
//
// The dominant kernel of the V-cycle.  A CTA owns
// TY rows (j) of one x-chunk of ICH planes and marches along x.  The other
// colour's planes -- rows j0-1 .. j0+TY (one ghost/halo row each side), the
// whole row in z -- stream into a 5-slot shared-memory ring with
// cp.async.bulk.tensor (TMA) completing on per-slot mbarriers, issued three
// planes ahead by one thread.  Each value of the other colour therefore
// crosses L2->SM once per CTA (plus 2/TY halo rows), instead of ~5 times for
// the direct-load kernel; own f is prefetched one plane ahead in registers
// and own Phi is written with 16-byte stores.
//
// The per-cell arithmetic is exactly that of k_smooth (bitwise identical):
//     Phi_c = (f_c * w + s) / d,  s = ((((x- + x+) + y-) + y+) + z-) + z+
#include <cuda.h>
#include <cuda_runtime.h>

#include "mg_internal.h"

namespace mg {

namespace {

constexpr int kTY = 8;        // rows per CTA (one warp per row)
constexpr int kICH = 16;      // planes per CTA
constexpr int kSlots = 5;     // ring depth: planes q-1, q, q+1 in use, 2 in flight
constexpr int kThreadsM = kTY * 32;

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
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
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

__host__ __device__ inline int slot_doubles(int pz) {
  // (TY + 2) rows of pz doubles, rounded up to 128 bytes
  return (((kTY + 2) * pz * 8 + 127) / 128) * 128 / 8;
}

}  // namespace

// one TMA box = (pz doubles) x (TY+2 rows) x (1 plane)
__global__ void __launch_bounds__(kThreadsM, 2)
    k_smooth_march(Grid g, const __grid_constant__ CUtensorMap tm_oth,
                   int color) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int pz = g.pz;
  const int sd = slot_doubles(pz);
  double *ring = reinterpret_cast<double *>(smem);
  unsigned long long *bars =
      reinterpret_cast<unsigned long long *>(smem + (size_t)kSlots * sd * 8);
  const unsigned box_bytes = (unsigned)((kTY + 2) * pz * 8);

  const int nrt = (g.ny + kTY - 1) / kTY;
  const int rt = blockIdx.x % nrt;
  const int xc = blockIdx.x / nrt;
  const int j0 = rt * kTY;
  const int i0 = xc * kICH;
  const int i1 = min(i0 + kICH, g.nxl);
  const int nplanes = (i1 - i0) + 2;  // local planes i0-1 .. i1
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; s++) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // prologue: planes q = 0..3 (local plane i0-1+q, array plane i0+q)
  if (threadIdx.x == 0) {
    const int np = nplanes < 4 ? nplanes : 4;
    for (int q = 0; q < np; q++) {
      mbar_expect_tx(&bars[q], box_bytes);
      tma_load_3d(ring + (size_t)q * sd, &tm_oth, 0, j0, i0 + q, &bars[q]);
    }
  }

  const int j = j0 + warp;
  const bool row_ok = j < g.ny;
  double *__restrict__ own = color ? g.phiB : g.phiR;
  const double *__restrict__ fown = color ? g.fB : g.fR;
  const int nch = (g.nzh + 63) >> 6;  // 64 half-entries per warp pass

  // f of the first plane into registers
  double2 fr[4];
#pragma unroll
  for (int c = 0; c < 4; c++) {
    const int k = 2 * lane + 64 * c;
    if (c < nch && row_ok && k < g.nzh)
      fr[c] = *reinterpret_cast<const double2 *>(
          fown + (long long)(i0 + 1) * g.plane + (long long)(j + 1) * pz + k);
  }

  for (int il = i0; il < i1; il++) {
    const int q = il - i0 + 1;  // ring index of the current plane
    __syncthreads();            // everybody is done with plane q-2's slot
    if (threadIdx.x == 0 && q + 3 < nplanes && q + 3 >= 4) {
      const int s = (q + 3) % kSlots;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bars[s], box_bytes);
      tma_load_3d(ring + (size_t)s * sd, &tm_oth, 0, j0, i0 + q + 3, &bars[s]);
    }
    // wait for planes q-1 (first step only), q (first step only), q+1
    if (q == 1) {
      mbar_wait(&bars[0], 0);
      mbar_wait(&bars[1], 0);
    }
    mbar_wait(&bars[(q + 1) % kSlots], ((q + 1) / kSlots) & 1);

    // prefetch f of the next plane
    double2 fn[4];
    const bool more = il + 1 < i1;
#pragma unroll
    for (int c = 0; c < 4; c++) {
      const int k = 2 * lane + 64 * c;
      if (more && c < nch && row_ok && k < g.nzh)
        fn[c] = *reinterpret_cast<const double2 *>(
            fown + (long long)(il + 2) * g.plane + (long long)(j + 1) * pz + k);
    }
    if (row_ok) {
      const double *cur = ring + (size_t)(q % kSlots) * sd + (warp + 1) * pz;
      const double *xm = ring + (size_t)((q - 1) % kSlots) * sd + (warp + 1) * pz;
      const double *xp = ring + (size_t)((q + 1) % kSlots) * sd + (warp + 1) * pz;
      const int i = g.x0 + il;
      const int p = (i + j + color) & 1;
      double *orow = own + (long long)(il + 1) * g.plane + (long long)(j + 1) * pz;
#pragma unroll
      for (int c = 0; c < 4; c++) {
        const int k = 2 * lane + 64 * c;
        if (c >= nch || k >= g.nzh) continue;
        const double2 a = *reinterpret_cast<const double2 *>(xm + k);
        const double2 b = *reinterpret_cast<const double2 *>(xp + k);
        const double2 ym = *reinterpret_cast<const double2 *>(cur - pz + k);
        const double2 yp = *reinterpret_cast<const double2 *>(cur + pz + k);
        const double2 zc = *reinterpret_cast<const double2 *>(cur + k);
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
        const double s0 = ((((a.x + b.x) + ym.x) + yp.x) + zm0) + zp0;
        const double s1 = ((((a.y + b.y) + ym.y) + yp.y) + zm1) + zp1;
        const int z0 = 2 * k + p;
        const double d0 = (double)centre_dm(g, i, j, z0);
        const double d1 = (double)centre_dm(g, i, j, z0 + 2);
        double2 out;
        out.x = (fr[c].x * g.w + s0) / d0;
        out.y = (fr[c].y * g.w + s1) / d1;
        if (k + 1 < g.nzh)
          *reinterpret_cast<double2 *>(orow + k) = out;
        else
          orow[k] = out.x;
      }
    }
#pragma unroll
    for (int c = 0; c < 4; c++) fr[c] = fn[c];
  }
}

// ---- host side ------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType,
                                    cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *,
                                    const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault,
                                &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  }
  return fn;
}

bool march_supported(const Grid &g) {
  // whole row in one TMA box (<= 256 elements), at least one full row tile
  return g.pz <= 256 && g.nzh >= 64 && g.ny >= kTY && g.nxl >= 2 &&
         get_encode() != nullptr;
}

size_t march_smem_bytes(const Grid &g) {
  return (size_t)kSlots * slot_doubles(g.pz) * 8 + kSlots * 8;
}

bool make_tmap_field(const Grid &g, const double *base, void *out128) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  CUtensorMap *tm = reinterpret_cast<CUtensorMap *>(out128);
  cuuint64_t dims[3] = {(cuuint64_t)g.pz, (cuuint64_t)(g.ny + 2),
                        (cuuint64_t)(g.nxl + 2)};
  cuuint64_t strides[2] = {(cuuint64_t)g.pz * 8, (cuuint64_t)g.plane * 8};
  cuuint32_t box[3] = {(cuuint32_t)g.pz, (cuuint32_t)(kTY + 2), 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                   const_cast<double *>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

void launch_smooth_march(const Grid &g, const void *tm_oth128, int color,
                         cudaStream_t s) {
  const int nrt = (g.ny + kTY - 1) / kTY;
  const int nxc = (g.nxl + kICH - 1) / kICH;
  const size_t smem = march_smem_bytes(g);
  static size_t configured = 0;
  if (smem > configured) {
    cudaFuncSetAttribute(k_smooth_march,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    configured = smem;
  }
  const CUtensorMap *tm = reinterpret_cast<const CUtensorMap *>(tm_oth128);
  k_smooth_march<<<nrt * nxc, kThreadsM, smem, s>>>(g, *tm, color);
}

}  // namespace mg
