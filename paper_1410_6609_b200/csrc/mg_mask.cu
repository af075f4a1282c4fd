// Variable-coefficient (solid-mask) kernels for sm_100a: config 5.
//
// With solid cells (P:653-697 flags; reading c19: a masked cell is not an
// unknown and its faces are homogeneous Neumann) the Galerkin operator
// R A P of every level has an exact face-transmissibility form:
//     a_q  = -c_l * kappa_q,   kappa_q = (# fluid-fluid fine face pairs
//                                        across the coarse face) / 4^l,
//     a_cc =  c_l * (sum_q kappa_q + 2 delta),   delta = (# fluid fine cells
//                                        on Dirichlet faces of the block) / 4^l
// (row sums are preserved by R A P because P 1 = 1 on fluid cells).  Every
// coefficient is a dyadic rational with <= 13 significant bits, exact in
// fp32 and fp64, so the GPU values equal the oracle's generic RAP stencils
// bit for bit.  Level 0 stores one byte per cell (6 face bits + fluid bit),
// coarse levels 8 floats per cell: kappa[6], D = sum kappa + 2 delta, delta.
//
// Per-cell arithmetic (bitwise equal to the oracle's (f - sum a_q phi_q)/a_cc
// when c_l is a power of two):
//     t   = ((((k0 x- + k1 x+) + k2 y-) + k3 y+) + k4 z-) + k5 z+
//     Phi = (f w + t) / D,       r = f - c (D Phi - t)
#include <cuda_runtime.h>

#include "mg_internal.h"

namespace mg {

namespace {

constexpr int kT = 256;

__device__ __forceinline__ long long rb(const Grid &g, int il, int j) {
  return (long long)(il + 1) * g.plane + (long long)(j + 1) * g.pz;
}

__device__ __forceinline__ int ndir(const Grid &g, int i, int j, int z) {
  int n = 0;
  if (i == 0 && g.dface[0] > 0) n++;
  if (i == g.nx - 1 && g.dface[1] > 0) n++;
  if (j == 0 && g.dface[2] > 0) n++;
  if (j == g.ny - 1 && g.dface[3] > 0) n++;
  if (z == 0 && g.dface[4] > 0) n++;
  if (z == g.nz - 1 && g.dface[5] > 0) n++;
  return n;
}

struct Coef {
  double k[6];
  double D;      // 0 for solid cells
  double delta;
};

// coefficients of the cell of colour col at split element e, global (i,j,z)
__device__ __forceinline__ void coef_at(const Grid &g, int col, long long e,
                                        int i, int j, int z, Coef &C) {
  if (g.c64R) {  // permittivity: fp64 records, 64-byte aligned, 16-byte loads
    const double2 *r = reinterpret_cast<const double2 *>((col ? g.c64B : g.c64R) + 8 * e);
    const double2 r0 = r[0], r1 = r[1], r2 = r[2], r3 = r[3];
    C.k[0] = r0.x;
    C.k[1] = r0.y;
    C.k[2] = r1.x;
    C.k[3] = r1.y;
    C.k[4] = r2.x;
    C.k[5] = r2.y;
    C.D = r3.x;
    C.delta = r3.y;
  } else if (g.coefR == nullptr) {
    const unsigned cd = (col ? g.codeB : g.codeR)[e];
    int n = 0;
#pragma unroll
    for (int q = 0; q < 6; q++) {
      const int b = (cd >> q) & 1;
      C.k[q] = b ? 1.0 : 0.0;
      n += b;
    }
    if (cd & 64) {
      C.delta = (double)ndir(g, i, j, z);
      C.D = (double)n + 2.0 * C.delta;
    } else {
      C.delta = 0.0;
      C.D = 0.0;
    }
  } else {  // float records, 32-byte aligned, 16-byte loads
    const float4 *r = reinterpret_cast<const float4 *>((col ? g.coefB : g.coefR) + 8 * e);
    const float4 r0 = r[0], r1 = r[1];
    C.k[0] = (double)r0.x;
    C.k[1] = (double)r0.y;
    C.k[2] = (double)r0.z;
    C.k[3] = (double)r0.w;
    C.k[4] = (double)r1.x;
    C.k[5] = (double)r1.y;
    C.D = (double)r1.z;
    C.delta = (double)r1.w;
  }
}

// t = sum_q kappa_q phi_q of the cell (il, j, z) (other colour array O)
__device__ __forceinline__ double nbsum(const Grid &g, const double *O,
                                        long long e, int z, const Coef &C) {
  const int p = z & 1;
  const double xm = O[e - g.plane], xp = O[e + g.plane];
  const double ym = O[e - g.pz], yp = O[e + g.pz];
  const double zm = (z > 0) ? O[e - 1 + p] : 0.0;
  const double zp = (z < g.nz - 1) ? O[e + p] : 0.0;
  return ((((C.k[0] * xm + C.k[1] * xp) + C.k[2] * ym) + C.k[3] * yp) +
          C.k[4] * zm) +
         C.k[5] * zp;
}

__device__ __forceinline__ double resid_var(const Grid &g, int il, int j, int z) {
  const int i = g.x0 + il;
  const int col = (i + j + z) & 1;
  const long long e = rb(g, il, j) + (z >> 1);
  Coef C;
  coef_at(g, col, e, i, j, z, C);
  if (C.D == 0.0) return 0.0;
  const double *own = col ? g.phiB : g.phiR;
  const double *oth = col ? g.phiR : g.phiB;
  const double *f = col ? g.fB : g.fR;
  const double t = nbsum(g, oth, e, z, C);
  const double u = C.D * own[e] - t;
  return f[e] - g.c * u;
}

__device__ __forceinline__ double block_sum_m(double v, double *sh) {
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

inline unsigned nblk(long long n) { return (unsigned)((n + kT - 1) / kT); }

}  // namespace

// ---- level-0 face codes from the global solid mask ---------------------------
__global__ void __launch_bounds__(kT)
    k_mask_codes(Grid g, const unsigned char *solid, unsigned char *codeR,
                 unsigned char *codeB) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.nxl * g.ny * g.nz) return;
  const int z = (int)(t % g.nz);
  const long long q = t / g.nz;
  const int j = (int)(q % g.ny);
  const int il = (int)(q / g.ny);
  const int i = g.x0 + il;
  auto fluid = [&](int a, int b, int c) -> bool {
    if (a < 0 || b < 0 || c < 0 || a >= g.nx || b >= g.ny || c >= g.nz) return false;
    return solid[((long long)a * g.ny + b) * g.nz + c] == 0;
  };
  unsigned char cd = 0;
  if (fluid(i, j, z)) {
    cd = 64;
    if (fluid(i - 1, j, z)) cd |= 1;
    if (fluid(i + 1, j, z)) cd |= 2;
    if (fluid(i, j - 1, z)) cd |= 4;
    if (fluid(i, j + 1, z)) cd |= 8;
    if (fluid(i, j, z - 1)) cd |= 16;
    if (fluid(i, j, z + 1)) cd |= 32;
  }
  (((i + j + z) & 1) ? codeB : codeR)[rb(g, il, j) + (z >> 1)] = cd;
}

void launch_mask_codes(const Grid &g, const unsigned char *solid_global,
                       unsigned char *codeR, unsigned char *codeB,
                       cudaStream_t s) {
  const long long n = (long long)g.nxl * g.ny * g.nz;
  if (n > 0) k_mask_codes<<<nblk(n), kT, 0, s>>>(g, solid_global, codeR, codeB);
}

// ---- level-0 records from mask + per-face-cell BCs ------------------------------
__device__ __forceinline__ long long face_idx(const Grid &g, int q, int i, int j,
                                              int z) {
  if (q < 2) return (long long)j * g.nz + z;
  if (q < 4) return (long long)i * g.nz + z;
  return (long long)i * g.ny + j;
}

__device__ __forceinline__ bool face_dirichlet(const Grid &g, const FaceBC &fb,
                                               int q, int i, int j, int z) {
  if (fb.ty[q]) return fb.ty[q][face_idx(g, q, i, j, z)] == 0;
  return g.dface[q] > 0;
}

__global__ void __launch_bounds__(kT)
    k_level0_coef(Grid g, const unsigned char *solid, FaceBC fb, float *coefR,
                  float *coefB) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.nxl * g.ny * g.nz) return;
  const int z = (int)(t % g.nz);
  const long long q = t / g.nz;
  const int j = (int)(q % g.ny);
  const int il = (int)(q / g.ny);
  const int i = g.x0 + il;
  auto fluid = [&](int a, int b, int c) -> bool {
    return !solid || solid[((long long)a * g.ny + b) * g.nz + c] == 0;
  };
  float rec[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (fluid(i, j, z)) {
    const int di[6] = {-1, 1, 0, 0, 0, 0}, dj[6] = {0, 0, -1, 1, 0, 0},
              dk[6] = {0, 0, 0, 0, -1, 1};
    float D = 0.f, del = 0.f;
    for (int f = 0; f < 6; f++) {
      const int a = i + di[f], b = j + dj[f], c = z + dk[f];
      if (a < 0 || b < 0 || c < 0 || a >= g.nx || b >= g.ny || c >= g.nz) {
        if (face_dirichlet(g, fb, f, i, j, z)) del += 1.f;
      } else if (fluid(a, b, c)) {
        rec[f] = 1.f;
        D += 1.f;
      }
    }
    rec[6] = D + 2.f * del;
    rec[7] = del;
  }
  const int col = (i + j + z) & 1;
  float *out = (col ? coefB : coefR) + 8 * (rb(g, il, j) + (z >> 1));
  for (int r = 0; r < 8; r++) out[r] = rec[r];
}

void launch_level0_coef(const Grid &g, const unsigned char *solid_global,
                        const FaceBC &fb, float *coefR, float *coefB,
                        cudaStream_t s) {
  const long long n = (long long)g.nxl * g.ny * g.nz;
  if (n > 0) k_level0_coef<<<nblk(n), kT, 0, s>>>(g, solid_global, fb, coefR, coefB);
}

// ---- finest-grid RHS adaptation with per-face-cell BCs ---------------
// same expressions as the uniform kernel: f -= (2 alpha) g (Dirichlet) or
// alpha (h g) (Neumann), in face order; solid cells skipped
__global__ void __launch_bounds__(kT)
    k_bc_adapt_faces(Grid g, FaceBC fb, double alpha, double h) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.nxl * g.ny) return;
  const int j = (int)(t % g.ny);
  const int il = (int)(t / g.ny);
  const int i = g.x0 + il;
  const bool full = (i == 0 || i == g.nx - 1 || j == 0 || j == g.ny - 1);
  const long long b = rb(g, il, j);
  const int step = full ? 1 : (g.nz - 1 > 0 ? g.nz - 1 : 1);
  for (int z = 0; z < g.nz; z += step) {
    const int col = (i + j + z) & 1;
    const long long e = b + (z >> 1);
    if (g.codeR || g.coefR || g.c64R) {  // masked cells are not unknowns
      Coef C;
      coef_at(g, col, e, i, j, z, C);
      if (C.D == 0.0) continue;
    }
    double *f = col ? g.fB : g.fR;
    double v = f[e];
    // variable permittivity (d10): alpha = -eps_c / h^2, the oracle's form
    const double al =
        g.c64R ? -((col ? g.c64B : g.c64R)[8 * e + 7] * (1.0 / (h * h))) : alpha;
    const bool on[6] = {i == 0, i == g.nx - 1, j == 0, j == g.ny - 1, z == 0,
                        z == g.nz - 1};
    for (int q = 0; q < 6; q++) {
      if (!on[q] || g.per[q >> 1]) continue;  // periodic: no boundary term
      const long long fi = face_idx(g, q, i, j, z);
      const bool dir = fb.ty[q] ? fb.ty[q][fi] == 0 : g.dface[q] > 0;
      const double gv = fb.va[q][fi];
      v = dir ? v - 2.0 * al * gv : v - al * (h * gv);
    }
    f[e] = v;
  }
}

void launch_bc_adapt_faces(const Grid &g, const FaceBC &fb, double alpha,
                           double h, cudaStream_t s) {
  const long long n = (long long)g.nxl * g.ny;
  if (n > 0) k_bc_adapt_faces<<<nblk(n), kT, 0, s>>>(g, fb, alpha, h);
}

// ---- Galerkin coarse coefficients (face-transmissibility form) ---------------
__global__ void __launch_bounds__(kT)
    k_coarse_coef(Grid F, Grid C, float *coefR, float *coefB) {
  const int ncz = F.nz >> 1, ncy = F.ny >> 1, ncx = F.nxl >> 1;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)ncx * ncy * ncz) return;
  const int K = (int)(t % ncz);
  const long long q = t / ncz;
  const int J = (int)(q % ncy);
  const int Il = (int)(q / ncy);
  float kap[6] = {0, 0, 0, 0, 0, 0};
  float del = 0.f;
  for (int a = 0; a < 2; a++)
    for (int b = 0; b < 2; b++)
      for (int c = 0; c < 2; c++) {
        const int il = 2 * Il + a, j = 2 * J + b, z = 2 * K + c;
        const int i = F.x0 + il;
        const int col = (i + j + z) & 1;
        Coef cf;
        coef_at(F, col, rb(F, il, j) + (z >> 1), i, j, z, cf);
        // child faces on the coarse cell's boundary: x- (a=0), x+ (a=1), ...
        kap[a == 0 ? 0 : 1] += (float)cf.k[a == 0 ? 0 : 1];
        kap[b == 0 ? 2 : 3] += (float)cf.k[b == 0 ? 2 : 3];
        kap[c == 0 ? 4 : 5] += (float)cf.k[c == 0 ? 4 : 5];
        del += (float)cf.delta;
      }
  float D = 0.f;
#pragma unroll
  for (int r = 0; r < 6; r++) {
    kap[r] *= 0.25f;
    D += kap[r];
  }
  del *= 0.25f;
  D += 2.f * del;
  const int Ig = (F.x0 >> 1) + Il;
  const int col = (Ig + J + K) & 1;
  float *out = (col ? coefB : coefR) + 8 * (rb(C, Ig - C.x0, J) + (K >> 1));
#pragma unroll
  for (int r = 0; r < 6; r++) out[r] = kap[r];
  out[6] = D;
  out[7] = del;
}

void launch_coarse_coef(const Grid &f, const Grid &c, float *coefR,
                        float *coefB, cudaStream_t s) {
  const long long n = (long long)(f.nxl >> 1) * (f.ny >> 1) * (f.nz >> 1);
  if (n > 0) k_coarse_coef<<<nblk(n), kT, 0, s>>>(f, c, coefR, coefB);
}

// ---- fp64 records for a variable permittivity (N4, reading d10) ----------------
// level 0, the oracle's assemble_finest_eps in kappa units (a = -kappa / h^2,
// a_cc = D / h^2, exact scalings for power-of-two h): per face in order x-,
// x+, y-, y+, z-, z+: fluid neighbour kappa = (2 eps_c eps_n)/(eps_c + eps_n)
// and D += kappa; Dirichlet boundary D += 2 eps_c; Neumann / solid nothing.
__global__ void __launch_bounds__(kT)
    k_level0_coef64(Grid g, const unsigned char *solid, const double *eps,
                    FaceBC fb, double *recR, double *recB) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.nxl * g.ny * g.nz) return;
  const int z = (int)(t % g.nz);
  const long long q = t / g.nz;
  const int j = (int)(q % g.ny);
  const int il = (int)(q / g.ny);
  const int i = g.x0 + il;
  auto gidx = [&](int a, int b, int c) { return ((long long)a * g.ny + b) * g.nz + c; };
  auto fluid = [&](int a, int b, int c) -> bool {
    return !solid || solid[gidx(a, b, c)] == 0;
  };
  double rec[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (fluid(i, j, z)) {
    const int di[6] = {-1, 1, 0, 0, 0, 0}, dj[6] = {0, 0, -1, 1, 0, 0},
              dk[6] = {0, 0, 0, 0, -1, 1};
    const double ec = eps[gidx(i, j, z)];
    double D = 0.0;
    for (int f = 0; f < 6; f++) {
      const int a = i + di[f], b = j + dj[f], c = z + dk[f];
      if (a < 0 || b < 0 || c < 0 || a >= g.nx || b >= g.ny || c >= g.nz) {
        if (face_dirichlet(g, fb, f, i, j, z)) D = D + 2.0 * ec;
      } else if (fluid(a, b, c)) {
        const double en = eps[gidx(a, b, c)];
        const double ef = (2.0 * ec * en) / (ec + en);
        rec[f] = ef;
        D = D + ef;
      }
    }
    rec[6] = D;
    rec[7] = ec;
  }
  const int col = (i + j + z) & 1;
  double *out = (col ? recB : recR) + 8 * (rb(g, il, j) + (z >> 1));
  for (int r = 0; r < 8; r++) out[r] = rec[r];
}

void launch_level0_coef64(const Grid &g, const unsigned char *solid_global,
                          const double *eps_global, const FaceBC &fb,
                          double *recR, double *recB, cudaStream_t s) {
  const long long n = (long long)g.nxl * g.ny * g.nz;
  if (n > 0)
    k_level0_coef64<<<nblk(n), kT, 0, s>>>(g, solid_global, eps_global, fb, recR, recB);
}

// Galerkin R A P in the oracle's order (galerkin(): children
// (a,b,c) lexicographic, per child its centre then faces x-..z+; a face to a
// sibling adds to the centre, any other to that face), in kappa units: the
// fine centre D and -kappa of sibling faces into sD, kappa into sK[q]; the
// coarse record is 0.25 * (sD, sK) (= 1/8 and the level scale 2, exact).
// kappa = 0 (boundary / solid neighbour) adds an exact zero.
__global__ void __launch_bounds__(kT)
    k_coarse_coef64(Grid F, Grid C, double *recR, double *recB) {
  const int ncz = F.nz >> 1, ncy = F.ny >> 1, ncx = F.nxl >> 1;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)ncx * ncy * ncz) return;
  const int K = (int)(t % ncz);
  const long long q = t / ncz;
  const int J = (int)(q % ncy);
  const int Il = (int)(q / ncy);
  double sD = 0.0, sK[6] = {0, 0, 0, 0, 0, 0};
  bool any = false;
  for (int a = 0; a < 2; a++)
    for (int b = 0; b < 2; b++)
      for (int c = 0; c < 2; c++) {
        const int il = 2 * Il + a, j = 2 * J + b, z = 2 * K + c;
        const int i = F.x0 + il;
        const int col = (i + j + z) & 1;
        const double *r = (col ? F.c64B : F.c64R) + 8 * (rb(F, il, j) + (z >> 1));
        if (r[6] == 0.0) continue;  // solid: not an unknown
        any = true;
        sD = sD + r[6];
        const bool sib[6] = {a == 1, a == 0, b == 1, b == 0, c == 1, c == 0};
#pragma unroll
        for (int f = 0; f < 6; f++) {
          if (r[f] == 0.0) continue;  // boundary or solid neighbour
          if (sib[f])
            sD = sD - r[f];
          else
            sK[f] = sK[f] + r[f];
        }
      }
  const int Ig = (F.x0 >> 1) + Il;
  const int col = (Ig + J + K) & 1;
  double *out = (col ? recB : recR) + 8 * (rb(C, Ig - C.x0, J) + (K >> 1));
  for (int f = 0; f < 6; f++) out[f] = any ? 0.25 * sK[f] : 0.0;
  out[6] = any ? 0.25 * sD : 0.0;
  out[7] = 0.0;
}

void launch_coarse_coef64(const Grid &f, const Grid &c, double *recR,
                          double *recB, cudaStream_t s) {
  const long long n = (long long)(f.nxl >> 1) * (f.ny >> 1) * (f.nz >> 1);
  if (n > 0) k_coarse_coef64<<<nblk(n), kT, 0, s>>>(f, c, recR, recB);
}

// ---- float records -> byte codes, when every kappa is 0 or 1 ------------------
// (the mask is aligned with this level's cells: then the level can use the
// byte-code marching kernels).  *fail is set if any cell is not representable.
__global__ void __launch_bounds__(kT)
    k_coef_to_code(Grid g, unsigned char *codeR, unsigned char *codeB, int *fail) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.nxl * g.ny * g.nz) return;
  const int z = (int)(t % g.nz);
  const long long q = t / g.nz;
  const int j = (int)(q % g.ny);
  const int il = (int)(q / g.ny);
  const int i = g.x0 + il;
  const int col = (i + j + z) & 1;
  const long long e = rb(g, il, j) + (z >> 1);
  const float *r = (col ? g.coefB : g.coefR) + 8 * e;
  unsigned char cd = 0;
  if (r[6] != 0.f) {
    cd = 64;
    int n = 0;
    for (int f = 0; f < 6; f++) {
      if (r[f] == 1.f) {
        cd |= (unsigned char)(1 << f);
        n++;
      } else if (r[f] != 0.f) {
        atomicOr(fail, 1);
      }
    }
    const int nd = ndir(g, i, j, z);
    if (r[7] != (float)nd || r[6] != (float)(n + 2 * nd)) atomicOr(fail, 1);
  }
  (col ? codeB : codeR)[e] = cd;
}

void launch_coef_to_code(const Grid &g, unsigned char *codeR, unsigned char *codeB,
                         int *fail, cudaStream_t s) {
  const long long n = (long long)g.nxl * g.ny * g.nz;
  if (n > 0) k_coef_to_code<<<nblk(n), kT, 0, s>>>(g, codeR, codeB, fail);
}

// ---- RBGS half-sweep, variable coefficients -----------------------------------
__global__ void __launch_bounds__(kT)
    k_smooth_var(Grid g, int color, int from_zero) {
  // one CTA per row (il, j), threads along the half-index k
  const int j = (int)(blockIdx.x % (unsigned)g.ny);
  const int il = (int)(blockIdx.x / (unsigned)g.ny);
  const int i = g.x0 + il;
  const int p = (i + j + color) & 1;
  const long long r0 = rb(g, il, j);
  const double *oth = color ? g.phiR : g.phiB;
  const double *f = color ? g.fB : g.fR;
  double *own = color ? g.phiB : g.phiR;
  for (int k = threadIdx.x; k < g.nzh; k += blockDim.x) {
    const int z = 2 * k + p;
    if (z >= g.nz) break;
    const long long e = r0 + k;
    Coef C;
    coef_at(g, color, e, i, j, z, C);
    if (C.D == 0.0) continue;  // solid: not an unknown
    const double tsum = from_zero ? 0.0 : nbsum(g, oth, e, z, C);
    own[e] = (f[e] * g.w + tsum) / C.D;
  }
}

// threads per row-CTA: the row's half-indices rounded up to a warp, <= kT
inline unsigned row_threads(int n) { return n < kT ? (unsigned)((n + 31) / 32 * 32) : kT; }

void launch_smooth_var(const Grid &g, int color, int from_zero, cudaStream_t s) {
  const long long rows = (long long)g.nxl * g.ny;
  if (rows > 0 && g.nzh > 0)
    k_smooth_var<<<(unsigned)rows, row_threads(g.nzh), 0, s>>>(g, color, from_zero);
}

// ---- residual + restriction ----------------------------------------------------
__global__ void __launch_bounds__(kT) k_resid_restrict_var(Grid F, Grid C) {
  const int ncz = F.nz >> 1, ncy = F.ny >> 1, ncx = F.nxl >> 1;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)ncx * ncy * ncz) return;
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
        r[a * 4 + b * 2 + c] = resid_var(F, 2 * Il + a, 2 * J + b, 2 * K + c);
  const double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  const int Ig = (F.x0 >> 1) + Il;
  const int col = (Ig + J + K) & 1;
  (col ? C.fB : C.fR)[rb(C, Ig - C.x0, J) + (K >> 1)] = 0.125 * s;
}

void launch_resid_restrict_var(const Grid &f, const Grid &c, cudaStream_t s) {
  const long long n = (long long)(f.nxl >> 1) * (f.ny >> 1) * (f.nz >> 1);
  if (n > 0) k_resid_restrict_var<<<nblk(n), kT, 0, s>>>(f, c);
}

// ---- prolongation + magnified correction, fluid cells only --------------------
// one CTA per fine row (il, j), threads along z (no 64-bit index division)
__global__ void __launch_bounds__(kT) k_prolong_var(Grid F, Grid C, double alpha) {
  const int j = (int)(blockIdx.x % (unsigned)F.ny);
  const int il = (int)(blockIdx.x / (unsigned)F.ny);
  const int i = F.x0 + il;
  const int I = i >> 1, J = j >> 1;
  const long long rf = rb(F, il, j), rc = rb(C, I - C.x0, J);
  for (int z = threadIdx.x; z < F.nz; z += blockDim.x) {
    const int col = (i + j + z) & 1;
    const long long e = rf + (z >> 1);
    if (!F.all_unknown) {  // unknowns only; without a mask all cells are
      Coef cf;
      coef_at(F, col, e, i, j, z, cf);
      if (cf.D == 0.0) continue;
    }
    const int Z = z >> 1;
    const double ec = (((I + J + Z) & 1) ? C.phiB : C.phiR)[rc + (Z >> 1)];
    double *u = col ? F.phiB : F.phiR;
    u[e] = u[e] + alpha * ec;
  }
}

void launch_prolong_var(const Grid &f, const Grid &c, double alpha, cudaStream_t s) {
  const long long rows = (long long)f.nxl * f.ny;
  if (rows > 0 && f.nz > 0)
    k_prolong_var<<<(unsigned)rows, row_threads(f.nz), 0, s>>>(f, c, alpha);
}

// ---- residual norm partials -------------------------------------------------------
__global__ void __launch_bounds__(kT) k_norm_var(Grid g, double *partials) {
  __shared__ double sh[32];
  const long long total = (long long)g.nxl * g.ny * g.nz;
  double acc = 0.0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int z = (int)(t % g.nz);
    const long long q = t / g.nz;
    const int j = (int)(q % g.ny);
    const int il = (int)(q / g.ny);
    const double r = resid_var(g, il, j, z);
    acc = acc + r * r;
  }
  const double s = block_sum_m(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

int launch_norm_partials_var(const Grid &g, double *partials, cudaStream_t s) {
  const long long total = (long long)g.nxl * g.ny * g.nz;
  long long nb = (total + kT - 1) / kT;
  if (nb > norm_blocks_max(g)) nb = norm_blocks_max(g);
  if (nb < 1) nb = 1;
  k_norm_var<<<(unsigned)nb, kT, 0, s>>>(g, partials);
  return (int)nb;
}

// ---- coarsest-grid CG, variable coefficients (one CTA, vectors in scratch) -----
__device__ __forceinline__ double cg_sum_v(double v, double *part) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double s = 0.0;
  for (int w = 0; w < nw; w++) s = s + part[w];
  return s;
}

__device__ __forceinline__ double cg_apply_var(const Grid &g, const double *v,
                                               long long n) {
  const int z = (int)(n % g.nz);
  const long long q = n / g.nz;
  const int j = (int)(q % g.ny);
  const int i = (int)(q / g.ny);
  const int col = (i + j + z) & 1;
  Coef C;
  coef_at(g, col, rb(g, i, j) + (z >> 1), i, j, z, C);
  if (C.D == 0.0) return 0.0;
  const long long sx = (long long)g.ny * g.nz, sy = g.nz;
  const double xm = (i > 0) ? v[n - sx] : 0.0;
  const double xp = (i < g.nx - 1) ? v[n + sx] : 0.0;
  const double ym = (j > 0) ? v[n - sy] : 0.0;
  const double yp = (j < g.ny - 1) ? v[n + sy] : 0.0;
  const double zm = (z > 0) ? v[n - 1] : 0.0;
  const double zp = (z < g.nz - 1) ? v[n + 1] : 0.0;
  const double t = ((((C.k[0] * xm + C.k[1] * xp) + C.k[2] * ym) + C.k[3] * yp) +
                    C.k[4] * zm) +
                   C.k[5] * zp;
  return g.c * (C.D * v[n] - t);
}

__global__ void __launch_bounds__(1024)
    k_coarse_cg_var(Grid g, double *scr, double tol, int maxit, int *iters_out) {
  __shared__ double part[2][32];
  const long long N = (long long)g.nx * g.ny * g.nz;
  double *x = scr, *r = scr + N, *p = scr + 2 * N, *q = scr + 3 * N;
  int pb = 0;
  double acc = 0.0;
  for (long long n = threadIdx.x; n < N; n += blockDim.x) {
    const int z = (int)(n % g.nz);
    const long long t = n / g.nz;
    const int j = (int)(t % g.ny), i = (int)(t / g.ny);
    const int col = (i + j + z) & 1;
    const long long e = rb(g, i, j) + (z >> 1);
    Coef C;
    coef_at(g, col, e, i, j, z, C);
    const double b = (C.D == 0.0) ? 0.0 : (col ? g.fB[e] : g.fR[e]);
    x[n] = 0.0;
    r[n] = b;
    p[n] = b;
    acc = acc + b * b;
  }
  double rho = cg_sum_v(acc, part[pb]);
  pb ^= 1;
  const double bnorm = sqrt(rho);
  int it = 0;
  if (bnorm > 0.0) {
    while (it < maxit) {
      acc = 0.0;
      for (long long n = threadIdx.x; n < N; n += blockDim.x) {
        const double qn = cg_apply_var(g, p, n);
        q[n] = qn;
        acc = acc + p[n] * qn;
      }
      const double pq = cg_sum_v(acc, part[pb]);
      pb ^= 1;
      const double a = rho / pq;
      acc = 0.0;
      for (long long n = threadIdx.x; n < N; n += blockDim.x) {
        x[n] = x[n] + a * p[n];
        const double rn = r[n] - a * q[n];
        r[n] = rn;
        acc = acc + rn * rn;
      }
      const double rho1 = cg_sum_v(acc, part[pb]);
      pb ^= 1;
      it++;
      if (sqrt(rho1) <= tol * bnorm) break;
      const double beta = rho1 / rho;
      for (long long n = threadIdx.x; n < N; n += blockDim.x) p[n] = r[n] + beta * p[n];
      __syncthreads();
      rho = rho1;
    }
  }
  __syncthreads();
  for (long long n = threadIdx.x; n < N; n += blockDim.x) {
    const int z = (int)(n % g.nz);
    const long long t = n / g.nz;
    const int j = (int)(t % g.ny), i = (int)(t / g.ny);
    const int col = (i + j + z) & 1;
    (col ? g.phiB : g.phiR)[rb(g, i, j) + (z >> 1)] = x[n];
  }
  if (threadIdx.x == 0 && iters_out) *iters_out = it;
}

// coarsest levels up to kCgVarSmem unknowns: the register-resident kernel
// below (9 doubles of shared memory per unknown: r, x, 6 kappa, D)
static constexpr int kCgVarSmem = 2304;

// The Chronopoulos-Gear form of the same CG (reading c8; k_coarse_cg's
// cg_cta_cg): per unknown n = threadIdx.x + e * blockDim (e < E) r, p,
// s = A p, w = A r in registers, the coefficients (6 kappa, D), r for the
// neighbours (zero slot at N) and x in shared memory; one two-value
// reduction and one barrier per iteration.  A solid cell (D = 0) has b = 0
// and a zero row, so its r, p, x stay 0.
template <int E>
__global__ void __launch_bounds__(512)
    k_coarse_cg_var_cg(Grid g, double tol, int maxit, int *iters_out) {
  extern __shared__ double sm[];
  __shared__ double part[2][64];
  const int N = g.nx * g.ny * g.nz;
  double *rs = sm, *xs = sm + N + 1;
  double *kap = sm + 2 * N + 1;  // [6][N]
  double *Dd = kap + 6 * N;      // [N]
  const int sx = g.ny * g.nz, sy = g.nz;
  const int nthr = (int)blockDim.x;
  unsigned nb[E][3];  // six 16-bit neighbour indices (N <= kCgVarSmem)
  double r[E], p[E], sv[E], w[E];
  bool act[E];
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int n = (int)threadIdx.x + e * nthr;
    act[e] = n < N;
    r[e] = p[e] = sv[e] = w[e] = 0.0;
#pragma unroll
    for (int a = 0; a < 3; a++) nb[e][a] = (unsigned)N * 0x10001u;
    if (act[e]) {
      const int z = n % g.nz;
      const int t = n / g.nz;
      const int j = t % g.ny, i = t / g.ny;
      const int col = (i + j + z) & 1;
      const long long el = rb(g, i, j) + (z >> 1);
      Coef C;
      coef_at(g, col, el, i, j, z, C);
      for (int f = 0; f < 6; f++) kap[f * N + n] = C.k[f];
      Dd[n] = C.D;
      const int k6[6] = {i > 0 ? n - sx : N, i < g.nx - 1 ? n + sx : N,
                         j > 0 ? n - sy : N, j < g.ny - 1 ? n + sy : N,
                         z > 0 ? n - 1 : N,  z < g.nz - 1 ? n + 1 : N};
#pragma unroll
      for (int a = 0; a < 3; a++)
        nb[e][a] = (unsigned)k6[2 * a] | ((unsigned)k6[2 * a + 1] << 16);
      const double b = (C.D == 0.0) ? 0.0 : (col ? g.fB[el] : g.fR[el]);
      r[e] = b;
      rs[n] = b;
      xs[n] = 0.0;
    }
  }
  if (threadIdx.x == 0) rs[N] = 0.0;
  const double c = g.c;
  int pb = 0;
  auto matvec = [&](double &gg, double &dl) {
    gg = 0.0;
    dl = 0.0;
#pragma unroll
    for (int e = 0; e < E; e++) {
      if (!act[e]) continue;
      const int n = (int)threadIdx.x + e * nthr;
      auto v = [&](int a) {
        return rs[(int)((nb[e][a >> 1] >> (16 * (a & 1))) & 0xffffu)];
      };
      const double D = Dd[n];
      double wn = 0.0;
      if (D != 0.0) {
        const double t = ((((kap[n] * v(0) + kap[N + n] * v(1)) + kap[2 * N + n] * v(2)) +
                           kap[3 * N + n] * v(3)) +
                          kap[4 * N + n] * v(4)) +
                         kap[5 * N + n] * v(5);
        wn = c * (D * r[e] - t);
      }
      w[e] = wn;
      gg = gg + r[e] * r[e];
      dl = dl + wn * r[e];
    }
  };
  __syncthreads();  // r and the coefficients published
  double gg, dl;
  matvec(gg, dl);
  double2 gd = cg_allsum2(gg, dl, part[pb]);
  pb ^= 1;
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
        r[e] = r[e] - alpha * sv[e];
        if (act[e]) {
          const int n = (int)threadIdx.x + e * nthr;
          rs[n] = r[e];
          xs[n] = xs[n] + alpha * p[e];
        }
      }
      __syncthreads();  // r published
      it++;
      matvec(gg, dl);
      gd = cg_allsum2(gg, dl, part[pb]);
      pb ^= 1;
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
  __syncthreads();
  for (int n = threadIdx.x; n < N; n += nthr) {
    const int z = n % g.nz;
    const int t = n / g.nz;
    const int j = t % g.ny, i = t / g.ny;
    const int col = (i + j + z) & 1;
    (col ? g.phiB : g.phiR)[rb(g, i, j) + (z >> 1)] = xs[n];
  }
  if (threadIdx.x == 0 && iters_out) *iters_out = it;
}

void launch_coarse_cg_var(const Grid &g, double *scratch, double tol, int maxit,
                          int *iters_out, cudaStream_t s) {
  const long long N = (long long)g.nx * g.ny * g.nz;
  if (N <= kCgVarSmem) {
    // the Chronopoulos-Gear kernel: up to 8 unknowns per thread
    int threads = (int)((N + 31) / 32 * 32);
    const int cap = N >= 2048 ? 512 : 256;  // as k_coarse_cg
    if (threads > cap) threads = cap;
    const int E = (int)((N + threads - 1) / threads);
    const size_t smem = (9 * (size_t)N + 1) * sizeof(double);
    static size_t configured = 48 * 1024;
    if (smem > configured) {
      cudaFuncSetAttribute(k_coarse_cg_var_cg<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(k_coarse_cg_var_cg<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(k_coarse_cg_var_cg<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(k_coarse_cg_var_cg<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      configured = smem;
    }
    if (E <= 1)
      k_coarse_cg_var_cg<1><<<1, threads, smem, s>>>(g, tol, maxit, iters_out);
    else if (E <= 2)
      k_coarse_cg_var_cg<2><<<1, threads, smem, s>>>(g, tol, maxit, iters_out);
    else if (E <= 4)
      k_coarse_cg_var_cg<4><<<1, threads, smem, s>>>(g, tol, maxit, iters_out);
    else
      k_coarse_cg_var_cg<8><<<1, threads, smem, s>>>(g, tol, maxit, iters_out);
    return;
  }
  int threads = (int)((N + 31) / 32 * 32);
  if (threads > 1024) threads = 1024;
  k_coarse_cg_var<<<1, threads, 0, s>>>(g, scratch, tol, maxit, iters_out);
}

// ---- f := 0 on solid cells (the oracle's "masked cells are not unknowns") -----
// f := 0 on the cells that are not unknowns.  Byte flags (bit 64 <=> an
// unknown, D != 0 -- the codes, or the flags of the float records): one warp
// per row (il, j), four flags per 32-bit load (rows start at multiples of 4
// elements), rows grid-strided over the warps.  Otherwise the records, one
// CTA per row.
__global__ void __launch_bounds__(kT) k_zero_solid(Grid g) {
  const unsigned char *uR = g.coefR ? g.ukR : g.codeR, *uB = g.coefR ? g.ukB : g.codeB;
  const unsigned rows = (unsigned)g.nxl * (unsigned)g.ny;
  if (uR && !g.c64R) {
    const int lane = threadIdx.x & 31;
    const unsigned nw = gridDim.x * (blockDim.x >> 5);
    const int nq = (g.nzh + 3) >> 2;  // 4-element groups per row half
    for (unsigned row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
         row += nw) {
      const int j = (int)(row % (unsigned)g.ny);
      const int il = (int)(row / (unsigned)g.ny);
      const int i = g.x0 + il;
      const long long r = rb(g, il, j);
      for (int q = lane; q < nq; q += 32)
#pragma unroll
        for (int col = 0; col < 2; col++) {
          const unsigned w = *reinterpret_cast<const unsigned *>((col ? uB : uR) + r + 4 * q);
          const int p = (i + j + col) & 1;
          double *f = (col ? g.fB : g.fR) + r + 4 * q;
#pragma unroll
          for (int b = 0; b < 4; b++) {
            const int z = 2 * (4 * q + b) + p;
            if (z < g.nz && !((w >> (8 * b)) & 64u)) f[b] = 0.0;
          }
        }
    }
    return;
  }
  for (unsigned row = blockIdx.x; row < rows; row += gridDim.x) {
    const int j = (int)(row % (unsigned)g.ny);
    const int il = (int)(row / (unsigned)g.ny);
    const int i = g.x0 + il;
    const long long r = rb(g, il, j);
    for (int z = threadIdx.x; z < g.nz; z += blockDim.x) {
      const int col = (i + j + z) & 1;
      const long long e = r + (z >> 1);
      Coef C;
      coef_at(g, col, e, i, j, z, C);
      if (C.D == 0.0) (col ? g.fB : g.fR)[e] = 0.0;
    }
  }
}

void launch_zero_solid(const Grid &g, cudaStream_t s) {
  const long long rows = (long long)g.nxl * g.ny;
  if (rows > 0 && g.nz > 0 && (g.codeR || g.coefR || g.c64R)) {
    const long long nb = rows < (long long)g.nsm * 8 ? rows : (long long)g.nsm * 8;
    k_zero_solid<<<(unsigned)nb, kT, 0, s>>>(g);
  }
}

// ---- operator of a level as 7 coefficients per cell, natural layout ------------
__global__ void __launch_bounds__(kT) k_get_stencil(Grid g, double *out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.nxl * g.ny * g.nz) return;
  const int z = (int)(t % g.nz);
  const long long q = t / g.nz;
  const int j = (int)(q % g.ny);
  const int il = (int)(q / g.ny);
  const int i = g.x0 + il;
  double *o = out + 7 * t;
  if (g.codeR || g.coefR || g.c64R) {
    const int col = (i + j + z) & 1;
    Coef C;
    coef_at(g, col, rb(g, il, j) + (z >> 1), i, j, z, C);
    o[0] = g.c * C.D;
    for (int r = 0; r < 6; r++) o[1 + r] = (C.D == 0.0) ? 0.0 : -g.c * C.k[r];
  } else {
    int d = 6;
    const bool on[6] = {i == 0, i == g.nx - 1, j == 0, j == g.ny - 1, z == 0,
                        z == g.nz - 1};
    for (int r = 0; r < 6; r++) {
      if (on[r]) d += g.dface[r];
      o[1 + r] = on[r] ? 0.0 : -g.c;
    }
    o[0] = g.c * (double)d;
  }
}

void launch_get_stencil(const Grid &g, double *out7, cudaStream_t s) {
  const long long n = (long long)g.nxl * g.ny * g.nz;
  if (n > 0) k_get_stencil<<<nblk(n), kT, 0, s>>>(g, out7);
}

}  // namespace mg
