// Internal declarations shared by the kernels (mg_kernels.cu) and the host
// orchestration (mg_api.cu) of libmg_cuda.so.  Not part of the C-ABI.
//
// Storage of one level of one slab ("Grid"): checkerboard-split layout
// ("rearranging the unknowns in a checker-board manner").  Each of
// the four fields Phi^R, Phi^B, f^R, f^B is an array
//     [nxl + 2 planes][ny + 2 rows][pz]   (x slowest, z fastest)
// holding, for row (i, j), the cells of that colour in z order: the red cell
// with half-index k sits at z = 2k + p, p = (i + j) & 1 (global i), the black
// one at z = 2k + 1 - p.  Plane 0 / nxl+1 and row 0 / ny+1 are ghost layers
// (0 on physical boundaries, neighbour data on slab interfaces).  pz >= nz/2,
// a multiple of 4 doubles, so every row starts 32-byte aligned.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mg {

struct Grid {
  double *phiR, *phiB, *fR, *fB;
  int nx, ny, nz;    // global dims of the level
  int nxl, x0;       // planes held here, global x index of the first one
  int nzh, pz;       // nz/2, row pitch in doubles
  long long plane;   // (ny + 2) * pz
  double c;          // operator scale 2^-l / h^2   (A_l = c * S_l)
  double w;          // 2^l h^2 = 1/c
  int dface[6];      // centre contribution of a face: +1 Dirichlet, -1 Neumann
  // solid mask (config 5), null on box domains.  Galerkin operator in face-
  // transmissibility form: a_q = -c kappa_q, a_cc = c (sum kappa + 2 delta).
  //   level 0:  code[e] bits 0-5 = kappa_q in {0,1} (face order x-,x+,y-,y+,
  //             z-,z+), bit 6 = fluid; delta from the Dirichlet faces touched
  //   level>0:  coef[8 e + q] = kappa_q (q < 6), coef[8 e + 6] = sum kappa +
  //             2 delta (0 = solid), coef[8 e + 7] = delta  (all dyadic, exact)
  const unsigned char *codeR, *codeB;
  const float *coefR, *coefB;
  // variable permittivity (N4, reading d10): fp64 records per cell
  // [kappa_q (6), D, eps_c (level 0) / 0]: a_q = -c kappa_q, a_cc = c D, with
  // real-valued kappa (harmonic face means on level 0, Galerkin R A P below)
  const double *c64R, *c64B;
  // every cell of the level is an unknown (records without a solid mask):
  // kernels that only need the unknown flag skip the records
  int all_unknown;
  // byte flags of the float records (bit 6 = an unknown, coef D != 0), kept
  // for kernels that only need that flag when the records are not codes
  const unsigned char *ukR, *ukB;
  // periodic axes ("accessing unknowns in cells at opposite sides
  // of the domain"): per[a] = 1 for a periodic axis (dface = 0 on its faces).
  // Ghost layers then hold the opposite side's cells: rows 0 / ny+1 mirror
  // rows ny / 1 (y periodic); planes 0 / nxl+1 mirror planes nxl / 1 when
  // the grid is held whole (gx = 1), otherwise the halo exchange wraps.  z
  // has no ghosts: kernels wrap the half-index of z neighbours (per[2]).
  int per[3];
  int gx;  // x periodic and the grid held whole: its writers fill x ghosts
  // streaming multiprocessors of the context's device (grid sizing of the
  // plane-marching and reduction kernels; cudaDevAttrMultiProcessorCount)
  int nsm;
};

__host__ __device__ inline long long grid_elems(const Grid &g) {
  return (long long)(g.nxl + 2) * g.plane;
}

// Periodic ghost copies of a value just written at (il, j, half-index k) of a
// colour array: the same colour array at the mirrored plane / row (nx, ny
// even keep the colour; corners when both apply).  Writers of Phi call this
// so that every reader finds current ghosts; the colour written is never
// read by the kernel writing it.
template <typename T>
__device__ __forceinline__ void ghost_copies(const Grid &g, double *arr, int il,
                                             int j, int k, T v) {
  const bool ex = g.gx && (il == 0 || il == g.nxl - 1);
  const bool ey = g.per[1] && (j == 0 || j == g.ny - 1);
  if (!(ex || ey)) return;
  // target planes / rows: the cell's own, then the mirrors (-1: none)
  const int pl[3] = {il + 1, (g.gx && il == 0) ? g.nxl + 1 : -1,
                     (g.gx && il == g.nxl - 1) ? 0 : -1};
  const int rw[3] = {j + 1, (g.per[1] && j == 0) ? g.ny + 1 : -1,
                     (g.per[1] && j == g.ny - 1) ? 0 : -1};
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = 0; b < 3; b++)
      if ((a || b) && pl[a] >= 0 && rw[b] >= 0)
        *reinterpret_cast<T *>(arr + (long long)pl[a] * g.plane +
                               (long long)rw[b] * g.pz + k) = v;
}

// sums over the block of two per-thread values at once; one barrier; every
// thread gets both.  part: 64 doubles.  Up to 16 warps the warp partials are
// read by lanes l and l + 16 alike, so four butterfly levels give every lane
// the same bits; up to 32 warps, five levels.
// a barrier of the first cnt threads of the block (id 0: the whole block)
__device__ __forceinline__ void bar_part(int id, int cnt) {
  if (id == 0)
    __syncthreads();
  else
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory");
}

// (bar, cnt: the barrier of the participating threads -- the first cnt of
// the block, a multiple of 32 -- when not the whole block)
__device__ __forceinline__ double2 cg_allsum2(double v0, double v1, double *part,
                                              int bar = 0, int cnt = 0) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, o);
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    part[w] = v0;
    part[32 + w] = v1;
  }
  bar_part(bar, cnt);
  const int nw = ((bar ? cnt : (int)blockDim.x) + 31) >> 5;
  if (nw <= 16) {
    const int l = lane & 15;
    double s0 = l < nw ? part[l] : 0.0, s1 = l < nw ? part[32 + l] : 0.0;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    return make_double2(s0, s1);
  }
  double s0 = lane < nw ? part[lane] : 0.0, s1 = lane < nw ? part[32 + lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  return make_double2(s0, s1);
}

// other-colour z neighbours of the own cells at half-indices k, k+1 of a row
// (red cells at z = 2k + p): zm0 = z-1 of the first, zp1 = z+1 of the second;
// the others are the row's entries k and k+1.  Outside the level: 0 (folded
// boundary) or, on a periodic z axis, the opposite end of the row.  PER is a
// compile-time switch: box-domain kernels carry no periodic logic at all.
template <bool PER>
__device__ __forceinline__ double z_lo(const Grid &g, const double *row, int k) {
  return (k > 0) ? row[k - 1] : ((PER && g.per[2]) ? row[g.nzh - 1] : 0.0);
}
template <bool PER>
__device__ __forceinline__ double z_hi(const Grid &g, const double *row, int k) {
  return (k + 2 < g.nzh) ? row[k + 2] : ((PER && g.per[2]) ? row[0] : 0.0);
}
// z+1 of the FIRST own cell (p = 1) is the entry k+1; when k is the row's
// last half-index (odd nzh) that entry is padding (0, the folded boundary),
// and on a periodic z axis it is the row's first entry instead
template <bool PER>
__device__ __forceinline__ double z_hi0(const Grid &g, const double *row, int k,
                                        double next) {
  return (PER && g.per[2] && k + 1 >= g.nzh) ? row[0] : next;
}

// Correctly rounded a / d for a small positive integer d (a smoother's
// centre, 1..15) from rd = RN(1/d): q0 = RN(a rd) is within 2 ulp of a/d;
// one FMA residual step brings it within 1 ulp, and the final Markstein step
// q = RN(q1 + RN(a - d q1) rd) -- exact residual by the FMA, rd within half
// an ulp of 1/d -- is RN(a/d) (no overflow / underflow at the smoothers'
// magnitudes).  Bitwise equal to IEEE a / d (except possibly the sign of an
// exact zero) at a quarter of the instructions; the half-sweep parity tests
// check it against the oracle's IEEE `/`.
__device__ __forceinline__ double div_small(double a, double d, double rd) {
  const double q0 = __dmul_rn(a, rd);
  const double r0 = __fma_rn(-q0, d, a);
  const double q1 = __fma_rn(r0, rd, q0);
  const double r1 = __fma_rn(-q1, d, a);
  return __fma_rn(r1, rd, q1);
}

// a / d for a centre d: the exact reciprocal path for the interior centre 6
// (RN(1/6) is a compile-time constant), IEEE division on boundary cells
__device__ __forceinline__ double div_centre(double a, double d) {
  constexpr double kRcp6 = 1.0 / 6.0;
  return d == 6.0 ? div_small(a, 6.0, kRcp6) : a / d;
}

// RN(1/d), d = 0..15 (entry 0 unused), in constant memory (one copy per
// translation unit); the initialisers are IEEE divisions, so div_small with
// these reciprocals is exactly RN(a/d).  A warp-uniform index (the interior
// centre 6) is a broadcast.
static __constant__ double c_rcp16[16] = {0.0,      1.0 / 1,  1.0 / 2,  1.0 / 3,
                                          1.0 / 4,  1.0 / 5,  1.0 / 6,  1.0 / 7,
                                          1.0 / 8,  1.0 / 9,  1.0 / 10, 1.0 / 11,
                                          1.0 / 12, 1.0 / 13, 1.0 / 14, 1.0 / 15};

// RN(1/d) for d = 0..15 into a shared table (IEEE division; entry 0 unused)
__device__ __forceinline__ void fill_rcp16(double *rcp) {
  if (threadIdx.x < 16) rcp[threadIdx.x] = threadIdx.x ? 1.0 / (double)threadIdx.x : 0.0;
}

// upper bound of the grid-stride norm kernels' CTA count (8 per SM): the
// number of partial sums they write
__host__ __device__ inline int norm_blocks_max(const Grid &g) { return 8 * g.nsm; }

__host__ __device__ inline bool is_periodic(const Grid &g) {
  return g.per[0] || g.per[1] || g.per[2];
}

// ---- kernel launchers (mg_kernels.cu) ---------------------------------------
// the coarse end of a V-cycle in one persistent cluster kernel: levels
// g[0..n-1] (whole grids, g[n-1] the coarsest), see k_vcycle_tail
constexpr int kTailMax = 12;
constexpr int kTailThreads = 512;
struct TailLevels {
  Grid g[kTailMax];
  int n;
};
// CTAs of the tail's cluster on this device (0: clusters unavailable)
int tail_cluster_ctas();
bool vcycle_tail_supported(const Grid &coarsest);
// 0, or -1 if the launch failed
int launch_vcycle_tail(const TailLevels &T, int nu1, int nu2, double alpha, double tol,
                       int maxit, double *cg_scr, int *iters_out, cudaStream_t s);
void launch_smooth(const Grid &g, int color, int from_zero, cudaStream_t s);
// red0 != 0 (box domains): also the coarse level's first red half-sweep
// from Phi = 0 (the coarse red Phi from the restricted f alone)
void launch_resid_restrict(const Grid &f, const Grid &c, int red0,
                           cudaStream_t s);
void launch_prolong(const Grid &f, const Grid &c, int cofs, double alpha,
                    cudaStream_t s);
// partial sums of r^2 over the grid into partials[0..nblk), returns nblk
int launch_norm_partials(const Grid &g, double *partials, cudaStream_t s);
// out[0] = sum of parts[0..n) in a fixed order
void launch_sum_ordered(const double *parts, int n, double *out,
                        cudaStream_t s);
void launch_sum_publish(const double *parts, int n, double *out, double *dev_dst,
                        double *host_dst, cudaStream_t s);
// dev_dst[0] = host_dst[0] = src[0] (host_dst: device view of mapped pinned
// host memory)
// coarsest CG on a thread-block cluster (mg_cg_cluster.cu): grids held
// whole with 4096 .. 8 x 4096 unknowns
bool coarse_cg_cluster_supported(const Grid &g);
void launch_coarse_cg_cluster(const Grid &g, double tol, int maxit, int *iters_out,
                              cudaStream_t s);
void launch_publish(const double *src, double *dev_dst, double *host_dst,
                    cudaStream_t s);
// first sphere index with a zero covered count (-1: none) -> mapped host word
void launch_first_empty(const unsigned long long *counts, int n, double *host_dst,
                        cudaStream_t s);
void launch_coarse_cg(const Grid &g, double *scratch, double tol, int maxit,
                      int *iters_out, cudaStream_t s);
size_t coarse_cg_scratch_doubles(const Grid &g);
// sphere RHS (mg_kernels.cu): covered sub-cell counts of the whole domain
// (any grid of level 0), then the density of grid g's covered cells, each
// cell written once in ascending sphere order (deterministic)
void launch_sphere_counts(const Grid &g, double h, int subsample, int n,
                          const double *sph, unsigned long long *counts,
                          cudaStream_t s);
// uniform bins of sphere centres for the neighbour search of the scatter:
// nb[a] bins of bc[a] cells per axis (on periodic axes bc divides the
// extent), count[bin] (zeroed by the caller) and up to kBinCap sphere
// indices per bin; rmax = the largest radius
constexpr int kBinCap = 16;
struct SphereBins {
  int nb[3], bc[3];
  int *count, *items;
  double rmax;
};
// per-sphere neighbour lists (kNbMax entries each), their lengths, and the
// spheres split into isolated ones (list[0..nlist[0])) and the others
// (list[n..n+nlist[1])); nlist zeroed by the caller
constexpr int kNbMax = 128;
struct SphereLists {
  int *nn, *nbr, *list, *nlist;
};
void launch_sphere_bin(const Grid &g, double h, int n, const double *sph,
                       const SphereBins &B, cudaStream_t s);
void launch_sphere_neighbours(const Grid &g, double h, int n, const double *sph,
                              const SphereBins &B, const SphereLists &S, cudaStream_t st);
void launch_sphere_scatter(const Grid &g, double h, int subsample, int n,
                           const double *sph, int normalization,
                           const unsigned long long *counts, const SphereLists &S,
                           cudaStream_t s);
void launch_bc_adapt(const Grid &g, const double *terms, const int *types,
                     cudaStream_t s);
// plane-marching TMA half-sweep (mg_march.cu)
bool march_supported(const Grid &g);
bool make_tmap_field(const Grid &g, const double *base, void *out128);
void launch_smooth_march(const Grid &g, const void *tm_oth128, int color,
                         cudaStream_t s);
// prolongation of the other colour fused with the half-sweep of `color`
void launch_prolong_smooth_march(const Grid &g, const Grid &c,
                                 const void *tm_oth128, int color, double alpha,
                                 cudaStream_t s);
// residual kernels (two rings, z-tiled boxes)
bool resid_march_supported(const Grid &g);
bool make_tmap_resid(const Grid &g, const double *base, void *out128);
void launch_resid_restrict_march(const Grid &g, const Grid &c, const void *tmR,
                                 const void *tmB, cudaStream_t s, int red0 = 0);
int norm_march_blocks(const Grid &g);
int march_blocks_max(const Grid &g);
// split norm of a cycle's end: the last black half-sweep with the black
// residuals' partials, then the red residuals' partials (12 B/cell); both
// return their partial counts
int launch_smooth_norm_march(const Grid &g, const void *tm_oth128, int color,
                             double *partials, cudaStream_t s);
int launch_norm_red_march(const Grid &g, const void *tmR, const void *tmB,
                          double *partials, cudaStream_t s);
// the look-ahead red half-sweep: the next cycle's first red half-sweep
// written to g.phiR (a second buffer) from the current Phi^R in oldv, with the
// current iterate's red residual partials; returns their count
int launch_smooth_lookahead_march(const Grid &g, const void *tm_oth128,
                                  const double *oldv, double *partials,
                                  cudaStream_t s);
// residual + restriction that also writes the norm partials of that residual
// (one per CTA, fixed order); returns the partial count
int launch_resid_restrict_norm_march(const Grid &g, const Grid &c, const void *tmR,
                                     const void *tmB, double *partials,
                                     cudaStream_t s, int red0 = 0);
void launch_norm_march(const Grid &g, const void *tmR, const void *tmB,
                       double *partials, cudaStream_t s);
bool encode_box(const Grid &g, const double *base, void *out128, unsigned box0,
                unsigned box1);
// per-face-cell boundary conditions (mg_set_bc_patch); null = face-uniform.
// Face q cell (a, b): q<2 -> (j, z), q<4 -> (i, z), else (i, j); index a*nb+b
struct FaceBC {
  const unsigned char *ty[6];  // MG_DIRICHLET / MG_NEUMANN per face cell
  const double *va[6];         // g_d / g_n per face cell
};
// level-0 float coefficient records from the mask (nullable) and face BCs
void launch_level0_coef(const Grid &g, const unsigned char *solid_global,
                        const FaceBC &fb, float *coefR, float *coefB,
                        cudaStream_t s);
void launch_bc_adapt_faces(const Grid &g, const FaceBC &fb, double alpha,
                           double h, cudaStream_t s);
// Coulomb force partial sums (mg_force.cu): part[3p+a] = sum_b g_a rho_p
// counts: per-sphere global covered sub-cell counts if known (the same
// step's RHS with the same subsampling), else null (counted here)
void launch_coulomb(const Grid &g, const unsigned char *solid_global, double h,
                    int subsample, int n, const double *sph, int normalization,
                    double *partials, const unsigned long long *counts,
                    cudaStream_t s);
// masked (variable-coefficient) path, mg_mask.cu
void launch_mask_codes(const Grid &g, const unsigned char *solid_global,
                       unsigned char *codeR, unsigned char *codeB,
                       cudaStream_t s);
void launch_coarse_coef(const Grid &f, const Grid &c, float *coefR,
                        float *coefB, cudaStream_t s);
void launch_coef_to_code(const Grid &g, unsigned char *codeR,
                         unsigned char *codeB, int *fail, cudaStream_t s);
void launch_smooth_var(const Grid &g, int color, int from_zero, cudaStream_t s);
void launch_resid_restrict_var(const Grid &f, const Grid &c, cudaStream_t s);
void launch_prolong_var(const Grid &f, const Grid &c, double alpha,
                        cudaStream_t s);
int launch_norm_partials_var(const Grid &g, double *partials, cudaStream_t s);
void launch_coarse_cg_var(const Grid &g, double *scratch, double tol, int maxit,
                          int *iters_out, cudaStream_t s);
void launch_zero_solid(const Grid &g, cudaStream_t s);
// fp64 records (permittivity): level 0 from eps (+ mask, face BC types), and
// Galerkin R A P in the oracle's summation order for the coarse levels
void launch_level0_coef64(const Grid &g, const unsigned char *solid_global,
                          const double *eps_global, const FaceBC &fb,
                          double *recR, double *recB, cudaStream_t s);
void launch_coarse_coef64(const Grid &f, const Grid &c, double *recR,
                          double *recB, cudaStream_t s);
void launch_get_stencil(const Grid &g, double *out7, cudaStream_t s);
// natural <-> split conversion of one field of a grid (phi: 0, f: 1)
void launch_pack(const Grid &g, int field, const double *nat, cudaStream_t s);
// refresh the periodic ghost rows / planes of both Phi colours from the
// interior (after writers that do not store ghost copies themselves)
void launch_periodic_fill(const Grid &g, cudaStream_t s);
void launch_unpack(const Grid &g, int field, double *nat, cudaStream_t s);

}  // namespace mg
