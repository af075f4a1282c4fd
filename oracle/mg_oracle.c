/*
 * oracle/mg_oracle.c -- TEST INFRASTRUCTURE ONLY (parity oracle).
 *
 * A plain, slow, obviously correct CPU fp64 implementation of the cell-centered
 * multigrid solve of the finite-volume Poisson equation in
 *   Bartuschat & Ruede, "Parallel Multiphysics Simulations of Charged Particles
 *   in Microfluidic Flows", arXiv 1410.6609  (PAPER.md, cited as P:<line>).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.  It shares no code with the CUDA product and the product
 * never loads it.  Compiled with -O2 -ffp-contract=off (no FMA contraction,
 * no fast-math); OpenMP only over independent per-cell loops, so the result
 * is bitwise the same for any thread count.
 *
 * Every step follows the paper in its order and notation:
 *   Poisson equation          -Lap Phi = rho/eps            Eq.12
 *   7-point FV stencil        -1/dx^2 [.. 6 .. -1 ..]      Eq.13
 *   Dirichlet/Neumann folding [0 (beta-+alpha) gamma]
 *   charge density            Q/V on cells whose centre is in the sphere P:481
 *   hierarchy                 coarsen while dims even
 *   Galerkin coarsening       A_c = R A P, R average, P nearest neighbour P:514-516
 *   magnified correction      phi += alpha P e, alpha = 2
 *   red-black Gauss-Seidel    checkerboard half-sweeps
 *   V(nu1,nu2)-cycles
 *   coarsest solve by CG
 *   residual L2 termination   Alg.1
 * Readings where the paper is silent are listed in DESIGN.md (c1..c21 of
 * SURVEY.md section 8(c)); each is cited at its use below.
 */
#include "mg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define MAXLEV 32
#define ORC_PI 3.14159265358979323846

typedef struct {
  int nx, ny, nz;
  long n;
  double *A;          /* 7 per cell: centre, x-, x+, y-, y+, z-, z+ */
  uint8_t *unk;       /* 1 = unknown cell, 0 = solid (masked) */
  double *phi, *f, *r;
  int per[3];         /* periodic axes, same on every level */
} level_t;

struct orc_hier {
  int nlev;
  level_t L[MAXLEV];
  double h;
  int bct[6];
  double bcv[6];
  int per[3]; /* periodic axes */
  /* per face-cell BC (patches, "specified in input files"):
   * face q has area A_q, cell (a,b) in the two remaining axes in (x,y,z)
   * order; NULL = the face-uniform bct/bcv */
  int *fty[6];
  double *fva[6];
  /* cell permittivity (N4, natural layout of level 0); NULL = constant 1,
   * the paper's "spatially constant permittivity" */
  double *eps;
  int nu1, nu2;
  double alpha;
  double coarse_tol;
  int coarse_maxit;
  int last_cg_iters;
  /* reading c11: report the norm of the fine residual the cycle computes
   * after pre-smoothing (for the restriction) instead of a post-cycle pass */
  int fused_norm;
  double in_cycle_norm;
};

static inline long IDX(const level_t *L, int i, int j, int k) {
  return ((long)i * L->ny + j) * L->nz + k;
}

/* in-face coordinates of cell (i,j,k) on face q: the two other axes, in
 * (x,y,z) order; index a*nb + b with nb the extent of the second one */
static inline long face_index(const level_t *L, int q, int i, int j, int k) {
  if (q < 2) return (long)j * L->nz + k;
  if (q < 4) return (long)i * L->nz + k;
  return (long)i * L->ny + j;
}

static inline int face_type(const orc_hier *H, int q, int i, int j, int k) {
  return H->fty[q] ? H->fty[q][face_index(&H->L[0], q, i, j, k)] : H->bct[q];
}

static inline double face_value(const orc_hier *H, int q, int i, int j, int k) {
  return H->fva[q] ? H->fva[q][face_index(&H->L[0], q, i, j, k)] : H->bcv[q];
}

/* Periodic BCs "cyclically extend the domain ... by accessing unknowns in
 * cells at opposite sides of the domain": an index one past a
 * periodic face wraps to the opposite side. */
static inline int wrap(int i, int n, int per) {
  if (!per) return i;
  if (i < 0) return i + n;
  if (i >= n) return i - n;
  return i;
}

/* value of a field at (i,j,k), 0 outside the level (the folded boundary
 * coefficient is 0 there, so the value never matters); wrapped
 * on periodic axes */
static inline double get(const level_t *L, const double *v, int i, int j,
                         int k) {
  i = wrap(i, L->nx, L->per[0]);
  j = wrap(j, L->ny, L->per[1]);
  k = wrap(k, L->nz, L->per[2]);
  if (i < 0 || j < 0 || k < 0 || i >= L->nx || j >= L->ny || k >= L->nz)
    return 0.0;
  return v[IDX(L, i, j, k)];
}

static void level_alloc(level_t *L, int nx, int ny, int nz) {
  L->nx = nx;
  L->ny = ny;
  L->nz = nz;
  L->n = (long)nx * ny * nz;
  L->A = (double *)calloc((size_t)L->n * 7, sizeof(double));
  L->unk = (uint8_t *)calloc((size_t)L->n, 1);
  L->phi = (double *)calloc((size_t)L->n, sizeof(double));
  L->f = (double *)calloc((size_t)L->n, sizeof(double));
  L->r = (double *)calloc((size_t)L->n, sizeof(double));
}

static void level_free(level_t *L) {
  free(L->A);
  free(L->unk);
  free(L->phi);
  free(L->f);
  free(L->r);
}

/* Finest-level stencil: Eq.13 gives -Lap_dx = (1/dx^2)[6; -1 x 6]
 * as the operator A of -Lap Phi = f (reading c1).  Boundary folding per
 * direction, P:451-459 with alpha the coefficient toward the boundary:
 *   Dirichlet: centre beta -> beta - alpha, alpha -> 0
 *   Neumann:   centre beta -> beta + alpha, alpha -> 0
 * A solid (masked) neighbour is a homogeneous Neumann face (reading c19). */
static void assemble_finest_eps(orc_hier *H);
static void galerkin(orc_hier *H, int l);

static void assemble_finest(orc_hier *H) {
  if (H->eps) {
    assemble_finest_eps(H);
    return;
  }
  level_t *L = &H->L[0];
  const double inv = 1.0 / (H->h * H->h);
  const int di[6] = {-1, 1, 0, 0, 0, 0};
  const int dj[6] = {0, 0, -1, 1, 0, 0};
  const int dk[6] = {0, 0, 0, 0, -1, 1};
  for (int i = 0; i < L->nx; i++)
    for (int j = 0; j < L->ny; j++)
      for (int k = 0; k < L->nz; k++) {
        long c = IDX(L, i, j, k);
        double *a = &L->A[7 * c];
        if (!L->unk[c]) {
          for (int q = 0; q < 7; q++) a[q] = 0.0;
          continue;
        }
        double beta = 6.0 * inv;
        for (int q = 0; q < 6; q++) {
          double alpha = -1.0 * inv;
          int ii = wrap(i + di[q], L->nx, L->per[0]);
          int jj = wrap(j + dj[q], L->ny, L->per[1]);
          int kk = wrap(k + dk[q], L->nz, L->per[2]);
          int outside = ii < 0 || jj < 0 || kk < 0 || ii >= L->nx ||
                        jj >= L->ny || kk >= L->nz;
          if (outside) {
            if (face_type(H, q, i, j, k) == ORC_DIRICHLET)
              beta = beta - alpha;
            else
              beta = beta + alpha;
            alpha = 0.0;
          } else if (!L->unk[IDX(L, ii, jj, kk)]) {
            beta = beta + alpha; /* homogeneous Neumann toward a solid cell */
            alpha = 0.0;
          }
          a[1 + q] = alpha;
        }
        a[0] = beta;
      }
}

/* Variable permittivity (the solver "is extensible for
 * discontinuous dielectricity coefficients ... by Galerkin coarsening",
 * P:513-516; "jumping dielectricity coefficients"):
 * -div(eps grad Phi) = rho, finite volumes on the same cells.
 * Reading d10: the flux across the face between cells c and n uses the
 * harmonic mean eps_f = (2 eps_c eps_n) / (eps_c + eps_n) (flux continuity
 * for a coefficient constant per cell); a boundary face uses eps_c, folded as
 * P:451-459 with alpha = -eps_c/h^2: Dirichlet adds 2 eps_c/h^2 to the
 * centre, Neumann nothing; a solid neighbour is a homogeneous Neumann face.
 * The centre sums the face terms in face order. */
static void assemble_finest_eps(orc_hier *H) {
  level_t *L = &H->L[0];
  const double inv = 1.0 / (H->h * H->h);
  const int di[6] = {-1, 1, 0, 0, 0, 0};
  const int dj[6] = {0, 0, -1, 1, 0, 0};
  const int dk[6] = {0, 0, 0, 0, -1, 1};
  for (int i = 0; i < L->nx; i++)
    for (int j = 0; j < L->ny; j++)
      for (int k = 0; k < L->nz; k++) {
        long c = IDX(L, i, j, k);
        double *a = &L->A[7 * c];
        for (int q = 0; q < 7; q++) a[q] = 0.0;
        if (!L->unk[c]) continue;
        const double ec = H->eps[c];
        double beta = 0.0;
        for (int q = 0; q < 6; q++) {
          int ii = wrap(i + di[q], L->nx, L->per[0]);
          int jj = wrap(j + dj[q], L->ny, L->per[1]);
          int kk = wrap(k + dk[q], L->nz, L->per[2]);
          int outside = ii < 0 || jj < 0 || kk < 0 || ii >= L->nx ||
                        jj >= L->ny || kk >= L->nz;
          if (outside) {
            if (face_type(H, q, i, j, k) == ORC_DIRICHLET)
              beta = beta + 2.0 * (ec * inv);
          } else if (L->unk[IDX(L, ii, jj, kk)]) {
            const double en = H->eps[IDX(L, ii, jj, kk)];
            const double ef = (2.0 * ec * en) / (ec + en);
            beta = beta + ef * inv;
            a[1 + q] = -(ef * inv);
          }
        }
        a[0] = beta;
      }
}

int orc_set_permittivity(orc_hier *H, const double *eps) {
  level_t *L = &H->L[0];
  free(H->eps);
  H->eps = NULL;
  if (eps) {
    for (long c = 0; c < L->n; c++)
      if (!(eps[c] > 0.0)) return -1;
    H->eps = (double *)malloc(sizeof(double) * (size_t)L->n);
    memcpy(H->eps, eps, sizeof(double) * (size_t)L->n);
  }
  assemble_finest(H);
  for (int l = 0; l + 1 < H->nlev; l++) galerkin(H, l);
  return 0;
}

/* Galerkin coarsening A_c = R A P: P = nearest-neighbour
 * (piecewise constant) injection of a coarse value to its unknown children,
 * R = (1/8) P^T (averaging).  Written as a stencil product: entry (I,J) of
 * R A P is (1/8) * sum over children i of I and j of J of A(i,j). */
static void galerkin(orc_hier *H, int l) {
  const level_t *F = &H->L[l];
  level_t *C = &H->L[l + 1];
  const int di[6] = {-1, 1, 0, 0, 0, 0};
  const int dj[6] = {0, 0, -1, 1, 0, 0};
  const int dk[6] = {0, 0, 0, 0, -1, 1};
  for (int I = 0; I < C->nx; I++)
    for (int J = 0; J < C->ny; J++)
      for (int K = 0; K < C->nz; K++) {
        long cI = IDX(C, I, J, K);
        double s[7] = {0, 0, 0, 0, 0, 0, 0};
        int any = 0;
        for (int a = 0; a < 2; a++)
          for (int b = 0; b < 2; b++)
            for (int c = 0; c < 2; c++) {
              int i = 2 * I + a, j = 2 * J + b, k = 2 * K + c;
              long fi = IDX(F, i, j, k);
              if (!F->unk[fi]) continue;
              any = 1;
              const double *A = &F->A[7 * fi];
              s[0] += A[0];
              for (int q = 0; q < 6; q++) {
                int ii = wrap(i + di[q], F->nx, F->per[0]);
                int jj = wrap(j + dj[q], F->ny, F->per[1]);
                int kk = wrap(k + dk[q], F->nz, F->per[2]);
                if (ii < 0 || jj < 0 || kk < 0 || ii >= F->nx || jj >= F->ny ||
                    kk >= F->nz)
                  continue; /* folded: coefficient is 0 */
                if (!F->unk[IDX(F, ii, jj, kk)]) continue;
                if (ii / 2 == I && jj / 2 == J && kk / 2 == K)
                  s[0] += A[1 + q]; /* sibling: lands on the coarse diagonal */
                else
                  s[1 + q] += A[1 + q]; /* child of coarse neighbour I+e_q */
              }
            }
        C->unk[cI] = (uint8_t)any;
        for (int q = 0; q < 7; q++) C->A[7 * cI + q] = 0.125 * s[q];
      }
}

orc_hier *orc_create(int nx, int ny, int nz, double h, const int *bc_type,
                     const double *bc_value, const uint8_t *solid,
                     int min_coarse, int max_levels) {
  if (nx <= 0 || ny <= 0 || nz <= 0 || !(h > 0.0)) return NULL;
  if (max_levels <= 0) max_levels = MAXLEV;
  if (max_levels > MAXLEV) max_levels = MAXLEV;
  /* periodic faces come in pairs: an axis is periodic on both sides or on
   * neither ("cyclically extend the domain") */
  int per[3];
  for (int a = 0; a < 3; a++) {
    const int lo = bc_type[2 * a] == ORC_PERIODIC;
    const int hi = bc_type[2 * a + 1] == ORC_PERIODIC;
    if (lo != hi) return NULL;
    per[a] = lo;
  }
  orc_hier *H = (orc_hier *)calloc(1, sizeof(orc_hier));
  H->h = h;
  for (int q = 0; q < 6; q++) {
    H->bct[q] = bc_type[q];
    H->bcv[q] = bc_value[q];
  }
  for (int a = 0; a < 3; a++) H->per[a] = per[a];
  H->nu1 = 2;
  H->nu2 = 2;
  H->alpha = 2.0;
  H->coarse_tol = 1e-12;
  H->coarse_maxit = 1000;
  /* hierarchy (reading c9): coarsen while every dimension is even,
   * the coarse dimensions are again even ("a multiple of two" at the
   * coarsest level) and the smallest dimension exceeds min_coarse. */
  int d[3] = {nx, ny, nz};
  level_alloc(&H->L[0], d[0], d[1], d[2]);
  H->nlev = 1;
  for (int a = 0; a < 3; a++) H->L[0].per[a] = per[a];
  while (H->nlev < max_levels) {
    int ok = 1;
    for (int a = 0; a < 3; a++)
      if (d[a] % 2 != 0 || (d[a] / 2) % 2 != 0) ok = 0;
    int mn = d[0] < d[1] ? d[0] : d[1];
    if (d[2] < mn) mn = d[2];
    if (mn <= min_coarse) ok = 0;
    if (!ok) break;
    for (int a = 0; a < 3; a++) d[a] /= 2;
    level_alloc(&H->L[H->nlev], d[0], d[1], d[2]);
    for (int a = 0; a < 3; a++) H->L[H->nlev].per[a] = per[a];
    H->nlev++;
  }
  level_t *L0 = &H->L[0];
  for (long c = 0; c < L0->n; c++) L0->unk[c] = solid ? (solid[c] ? 0 : 1) : 1;
  assemble_finest(H);
  for (int l = 0; l + 1 < H->nlev; l++) galerkin(H, l);
  return H;
}

void orc_destroy(orc_hier *H) {
  if (!H) return;
  for (int l = 0; l < H->nlev; l++) level_free(&H->L[l]);
  for (int q = 0; q < 6; q++) {
    free(H->fty[q]);
    free(H->fva[q]);
  }
  free(H->eps);
  free(H);
}

/* per-cell values on face q, the face's BC type unchanged (analytic
 * Dirichlet data of the charged-sphere validation) */
int orc_set_face_values(orc_hier *H, int q, const double *values) {
  level_t *L = &H->L[0];
  if (q < 0 || q > 5 || H->per[q / 2]) return -1;
  const int ext[3] = {L->nx, L->ny, L->nz};
  const int ax = q / 2;
  const long n = (long)ext[ax == 0 ? 1 : 0] * ext[ax == 2 ? 1 : 2];
  if (!H->fty[q]) {
    H->fty[q] = (int *)malloc(sizeof(int) * (size_t)n);
    H->fva[q] = (double *)malloc(sizeof(double) * (size_t)n);
    for (long c = 0; c < n; c++) H->fty[q][c] = H->bct[q];
  }
  for (long c = 0; c < n; c++) H->fva[q][c] = values[c];
  return 0;
}

/* Boundary patch (config 5's partial-length electrodes, reading c17): on face
 * q the cells with in-face coordinates a in [a0,a1), b in [b0,b1) get BC
 * (type, value).  Re-assembles the finest stencil and every Galerkin level;
 * the caller re-sets the RHS (its BC adaptation uses the patches). */
int orc_set_bc_patch(orc_hier *H, int q, int a0, int a1, int b0, int b1,
                     int type, double value) {
  level_t *L = &H->L[0];
  if (q < 0 || q > 5 || H->per[q / 2] || type == ORC_PERIODIC) return -1;
  const int ext[3] = {L->nx, L->ny, L->nz};
  const int ax = q / 2;
  const int na = ext[ax == 0 ? 1 : 0], nb = ext[ax == 2 ? 1 : 2];
  if (a0 < 0 || b0 < 0 || a1 > na || b1 > nb || a0 > a1 || b0 > b1) return -1;
  if (!H->fty[q]) {
    H->fty[q] = (int *)malloc(sizeof(int) * (size_t)na * nb);
    H->fva[q] = (double *)malloc(sizeof(double) * (size_t)na * nb);
    for (long c = 0; c < (long)na * nb; c++) {
      H->fty[q][c] = H->bct[q];
      H->fva[q][c] = H->bcv[q];
    }
  }
  for (int a = a0; a < a1; a++)
    for (int b = b0; b < b1; b++) {
      H->fty[q][(long)a * nb + b] = type;
      H->fva[q][(long)a * nb + b] = value;
    }
  assemble_finest(H);
  for (int l = 0; l + 1 < H->nlev; l++) galerkin(H, l);
  return 0;
}

int orc_num_levels(const orc_hier *H) { return H->nlev; }

void orc_level_dims(const orc_hier *H, int l, int *d) {
  d[0] = H->L[l].nx;
  d[1] = H->L[l].ny;
  d[2] = H->L[l].nz;
}

void orc_get_stencil(const orc_hier *H, int l, double *out) {
  memcpy(out, H->L[l].A, sizeof(double) * 7 * H->L[l].n);
}
void orc_get_unknown(const orc_hier *H, int l, uint8_t *out) {
  memcpy(out, H->L[l].unk, H->L[l].n);
}
void orc_get_phi(const orc_hier *H, int l, double *out) {
  memcpy(out, H->L[l].phi, sizeof(double) * H->L[l].n);
}
void orc_set_phi(orc_hier *H, int l, const double *in) {
  memcpy(H->L[l].phi, in, sizeof(double) * H->L[l].n);
}
void orc_get_rhs(const orc_hier *H, int l, double *out) {
  memcpy(out, H->L[l].f, sizeof(double) * H->L[l].n);
}
void orc_set_rhs_raw(orc_hier *H, int l, const double *in) {
  memcpy(H->L[l].f, in, sizeof(double) * H->L[l].n);
}

/* RHS adaptation to the BCs on the finest grid only, per
 * direction in face order x-, x+, y-, y+, z-, z+ (P:726-729).  With alpha the
 * unfolded coefficient toward the boundary (-1/h^2):
 *   Dirichlet g_d:  f <- f - 2 alpha g_d                 (c3)
 *   Neumann   g_n:  f <- f - alpha (h g_n)               (c2:
 *                   Phi_0 - Phi_1 = h g_n, outward normal derivative)      */
void orc_bc_adapt(orc_hier *H) {
  level_t *L = &H->L[0];
  const double inv = 1.0 / (H->h * H->h);
  const double alpha1 = -1.0 * inv;
  for (int i = 0; i < L->nx; i++)
    for (int j = 0; j < L->ny; j++)
      for (int k = 0; k < L->nz; k++) {
        long c = IDX(L, i, j, k);
        if (!L->unk[c]) continue;
        /* variable permittivity (d10): alpha = -eps_c / h^2 */
        const double alpha = H->eps ? -(H->eps[c] * inv) : alpha1;
        int on[6] = {i == 0, i == L->nx - 1, j == 0,
                     j == L->ny - 1, k == 0, k == L->nz - 1};
        for (int q = 0; q < 6; q++) {
          if (!on[q] || H->per[q / 2]) continue; /* periodic: no boundary */
          double g = face_value(H, q, i, j, k);
          if (face_type(H, q, i, j, k) == ORC_DIRICHLET)
            L->f[c] = L->f[c] - 2.0 * alpha * g;
          else
            L->f[c] = L->f[c] - alpha * (H->h * g);
        }
      }
}

void orc_set_rhs(orc_hier *H, const double *f) {
  level_t *L = &H->L[0];
  for (long c = 0; c < L->n; c++) L->f[c] = L->unk[c] ? f[c] : 0.0;
  orc_bc_adapt(H);
}

/* "each cell whose center is overlapped"; cell centres at
 * ((i+1/2)h, (j+1/2)h, (k+1/2)h); inclusive test |x-c|^2 <= R^2 (c13). */
static inline int inside(int i, int j, int k, double h, double cx, double cy,
                         double cz, double R) {
  double dx = ((double)i + 0.5) * h - cx;
  double dy = ((double)j + 0.5) * h - cy;
  double dz = ((double)k + 0.5) * h - cz;
  double d2 = (dx * dx + dy * dy) + dz * dz;
  return d2 <= R * R;
}

static void bbox(int n, double h, double c, double R, int *lo, int *hi) {
  /* every cell whose centre can be within R of c, plus a safety margin */
  int a = (int)floor((c - R) / h - 0.5) - 1;
  int b = (int)ceil((c + R) / h - 0.5) + 1;
  if (a < 0) a = 0;
  if (b > n - 1) b = n - 1;
  *lo = a;
  *hi = b;
}

/* Subsampling (Table 4): "equidistantly subdivides a cell and
 * counts the overlapped subvolumes" -- the s^3 sub-cell centres of cell
 * (i,j,k) are ((i s + a + 1/2) h/s, ...), a = 0..s-1, tested with the same
 * inclusive rule.  s = 1 is the plain centre rule (hs = h exactly). */
static inline int sub_count(int i, int j, int k, int s, double hs, double cx,
                            double cy, double cz, double R) {
  int cnt = 0;
  for (int a = 0; a < s; a++)
    for (int b = 0; b < s; b++)
      for (int c = 0; c < s; c++)
        cnt += inside(i * s + a, j * s + b, k * s + c, hs, cx, cy, cz, R);
  return cnt;
}

/* Periodic images of a sphere (the domain is cyclically
 * extended): centres c + m (n h) with m in {-1, 0, 1} on periodic axes (m = 0
 * leaves the coordinate untouched), in (mx, my, mz) lexicographic order.
 * With 2R + 2h <= n h on every periodic axis (checked by the callers) no
 * cell is reached by two images.  per == NULL: no periodic axis. */
static int sphere_images(const int *per, int nx, int ny, int nz, double h,
                         double cx, double cy, double cz, double img[27][3]) {
  const int px = per ? per[0] : 0, py = per ? per[1] : 0, pz = per ? per[2] : 0;
  int n = 0;
  for (int mx = -px; mx <= px; mx++)
    for (int my = -py; my <= py; my++)
      for (int mz = -pz; mz <= pz; mz++) {
        img[n][0] = mx ? cx + (double)mx * ((double)nx * h) : cx;
        img[n][1] = my ? cy + (double)my * ((double)ny * h) : cy;
        img[n][2] = mz ? cz + (double)mz * ((double)nz * h) : cz;
        n++;
      }
  return n;
}

static long subcount_one(int nx, int ny, int nz, double h, int s, double cx,
                         double cy, double cz, double R) {
  const double hs = h / (double)s;
  int i0, i1, j0, j1, k0, k1;
  bbox(nx, h, cx, R, &i0, &i1);
  bbox(ny, h, cy, R, &j0, &j1);
  bbox(nz, h, cz, R, &k0, &k1);
  long cnt = 0;
  for (int i = i0; i <= i1; i++)
    for (int j = j0; j <= j1; j++)
      for (int k = k0; k <= k1; k++)
        cnt += sub_count(i, j, k, s, hs, cx, cy, cz, R);
  return cnt;
}

/* covered sub-cells of the domain, summed over the periodic images */
static long subcount_per(const int *per, int nx, int ny, int nz, double h,
                         int s, double cx, double cy, double cz, double R) {
  double img[27][3];
  const int ni = sphere_images(per, nx, ny, nz, h, cx, cy, cz, img);
  long cnt = 0;
  for (int m = 0; m < ni; m++)
    cnt += subcount_one(nx, ny, nz, h, s, img[m][0], img[m][1], img[m][2], R);
  return cnt;
}

long orc_sphere_subcount(int nx, int ny, int nz, double h, int s, double cx,
                         double cy, double cz, double R) {
  return subcount_one(nx, ny, nz, h, s, cx, cy, cz, R);
}

long orc_sphere_cell_count(int nx, int ny, int nz, double h, double cx,
                           double cy, double cz, double R) {
  return orc_sphere_subcount(nx, ny, nz, h, 1, cx, cy, cz, R);
}

/* charge density of uniformly charged spheres (c12), subsampling
 * factor s, n_p = number of covered sub-cells of the domain:
 *   PER_CELLS:  cell value = (Q_p cnt) / (n_p h^3)       (charge exact)
 *   PER_VOLUME: cell value = (Q_p / (4/3 pi R^3)) (cnt / s^3)  (the paper's)
 * eps = 1 (c15), so f = rho.  Overlapping spheres add in sphere order. */
static void density_per(const int *per, int nx, int ny, int nz, double h,
                        int s, int n, const double *centers,
                        const double *radii, const double *charges,
                        int normalization, double *out) {
  long N = (long)nx * ny * nz;
  const double hs = h / (double)s;
  for (long c = 0; c < N; c++) out[c] = 0.0;
  for (int p = 0; p < n; p++) {
    double R = radii[p], Q = charges[p];
    double img[27][3];
    const int ni = sphere_images(per, nx, ny, nz, h, centers[3 * p],
                                 centers[3 * p + 1], centers[3 * p + 2], img);
    long np = subcount_per(per, nx, ny, nz, h, s, centers[3 * p],
                           centers[3 * p + 1], centers[3 * p + 2], R);
    if (normalization != ORC_PER_VOLUME && np == 0) continue;
    const double rho0 = Q / ((4.0 / 3.0) * ORC_PI * (R * R * R));
    for (int m = 0; m < ni; m++) {
      const double cx = img[m][0], cy = img[m][1], cz = img[m][2];
      int i0, i1, j0, j1, k0, k1;
      bbox(nx, h, cx, R, &i0, &i1);
      bbox(ny, h, cy, R, &j0, &j1);
      bbox(nz, h, cz, R, &k0, &k1);
      for (int i = i0; i <= i1; i++)
        for (int j = j0; j <= j1; j++)
          for (int k = k0; k <= k1; k++) {
            const int cnt = sub_count(i, j, k, s, hs, cx, cy, cz, R);
            if (!cnt) continue;
            double v;
            if (normalization == ORC_PER_VOLUME)
              v = rho0 * ((double)cnt / (double)(s * s * s));
            else
              v = (Q * (double)cnt) / ((double)np * (h * h * h));
            out[((long)i * ny + j) * nz + k] += v;
          }
    }
  }
}

void orc_sphere_density_sub(int nx, int ny, int nz, double h, int s, int n,
                            const double *centers, const double *radii,
                            const double *charges, int normalization,
                            double *out) {
  density_per(NULL, nx, ny, nz, h, s, n, centers, radii, charges,
              normalization, out);
}

/* spheres on a periodic axis: centre in [0, n h) and 2R + 2h <= n h, so the
 * images are disjoint (sphere_images); 0 or -1 */
static int check_periodic_spheres(const orc_hier *H, int n,
                                  const double *centers, const double *radii) {
  const level_t *L = &H->L[0];
  const int ext[3] = {L->nx, L->ny, L->nz};
  for (int p = 0; p < n; p++)
    for (int a = 0; a < 3; a++) {
      if (!H->per[a]) continue;
      const double len = (double)ext[a] * H->h, c = centers[3 * p + a];
      if (!(c >= 0.0 && c < len) || !(2.0 * radii[p] + 2.0 * H->h <= len))
        return -1;
    }
  return 0;
}

void orc_sphere_density(int nx, int ny, int nz, double h, int n,
                        const double *centers, const double *radii,
                        const double *charges, int normalization,
                        double *out) {
  orc_sphere_density_sub(nx, ny, nz, h, 1, n, centers, radii, charges,
                         normalization, out);
}

int orc_set_rhs_from_spheres_sub(orc_hier *H, int n, const double *centers,
                                 const double *radii, const double *charges,
                                 int normalization, int s) {
  level_t *L = &H->L[0];
  if (s < 1) return -1;
  if (check_periodic_spheres(H, n, centers, radii)) return -1;
  if (normalization == ORC_PER_CELLS)
    for (int p = 0; p < n; p++)
      if (subcount_per(H->per, L->nx, L->ny, L->nz, H->h, s, centers[3 * p],
                       centers[3 * p + 1], centers[3 * p + 2], radii[p]) == 0)
        return -1;
  density_per(H->per, L->nx, L->ny, L->nz, H->h, s, n, centers, radii,
              charges, normalization, L->f);
  for (long c = 0; c < L->n; c++)
    if (!L->unk[c]) L->f[c] = 0.0;
  orc_bc_adapt(H);
  return 0;
}

int orc_set_rhs_from_spheres(orc_hier *H, int n, const double *centers,
                             const double *radii, const double *charges,
                             int normalization) {
  return orc_set_rhs_from_spheres_sub(H, n, centers, radii, charges,
                                      normalization, 1);
}

/* ---- Coulomb force (Eq.14) with the isotropic D3Q19 gradient
 * (Eq.15), §8(f) N2 -------------------------------------------
 * grad Phi(x_b) = (1/w_1) sum_{q=2..19} w_q Phi(x_b + e_q) e_q / dx^2 with the
 * D3Q19 weights w_1 = 1/3, faces 1/18, edges 1/36.  Per component:
 * S = sum_q w_q c_q Phi_q in the fixed order of ORC_Q19 (terms with c_q = 0
 * skipped), g = (3 S) / h.  Reading d6 (the paper only says "where
 * possible"): the D3Q19 stencil is used where all 18 neighbours are fluid
 * cells of the domain; otherwise, per axis, the central difference
 * (Phi_+ - Phi_-) / (2h) if both axis neighbours are, else the one-sided
 * first-order difference toward the valid one, else 0. */
static const int ORC_Q19[18][3] = {
    {1, 0, 0},  {-1, 0, 0}, {0, 1, 0},   {0, -1, 0}, {0, 0, 1},  {0, 0, -1},
    {1, 1, 0},  {-1, -1, 0}, {1, -1, 0}, {-1, 1, 0}, {1, 0, 1},  {-1, 0, -1},
    {1, 0, -1}, {-1, 0, 1}, {0, 1, 1},   {0, -1, -1}, {0, 1, -1}, {0, -1, 1}};

static inline int valid_cell(const level_t *L, int i, int j, int k) {
  i = wrap(i, L->nx, L->per[0]);
  j = wrap(j, L->ny, L->per[1]);
  k = wrap(k, L->nz, L->per[2]);
  return i >= 0 && j >= 0 && k >= 0 && i < L->nx && j < L->ny && k < L->nz &&
         L->unk[IDX(L, i, j, k)];
}

/* phi at a (valid) cell, wrapped on periodic axes */
static inline double phi_w(const level_t *L, const double *phi, int i, int j,
                           int k) {
  return phi[IDX(L, wrap(i, L->nx, L->per[0]), wrap(j, L->ny, L->per[1]),
                 wrap(k, L->nz, L->per[2]))];
}

void orc_gradient(const orc_hier *H, const double *phi, int i, int j, int k,
                  double *g) {
  const level_t *L = &H->L[0];
  const double h = H->h;
  int all = 1;
  for (int q = 0; q < 18; q++)
    if (!valid_cell(L, i + ORC_Q19[q][0], j + ORC_Q19[q][1], k + ORC_Q19[q][2]))
      all = 0;
  if (all) {
    for (int a = 0; a < 3; a++) {
      double S = 0.0;
      for (int q = 0; q < 18; q++) {
        const int c = ORC_Q19[q][a];
        if (c == 0) continue;
        const double w = q < 6 ? 1.0 / 18.0 : 1.0 / 36.0;
        const double v = phi_w(L, phi, i + ORC_Q19[q][0], j + ORC_Q19[q][1],
                               k + ORC_Q19[q][2]);
        S = c > 0 ? S + w * v : S - w * v;
      }
      g[a] = (3.0 * S) / h;
    }
    return;
  }
  for (int a = 0; a < 3; a++) {
    int dp[3] = {0, 0, 0}, dm[3] = {0, 0, 0};
    dp[a] = 1;
    dm[a] = -1;
    const int vp = valid_cell(L, i + dp[0], j + dp[1], k + dp[2]);
    const int vm = valid_cell(L, i + dm[0], j + dm[1], k + dm[2]);
    const double c0 = phi[IDX(L, i, j, k)];
    if (vp && vm)
      g[a] = (phi_w(L, phi, i + dp[0], j + dp[1], k + dp[2]) -
              phi_w(L, phi, i + dm[0], j + dm[1], k + dm[2])) / (2.0 * h);
    else if (vp)
      g[a] = (phi_w(L, phi, i + dp[0], j + dp[1], k + dp[2]) - c0) / h;
    else if (vm)
      g[a] = (c0 - phi_w(L, phi, i + dm[0], j + dm[1], k + dm[2])) / h;
    else
      g[a] = 0.0;
  }
}

/* F_p = -dx^3 sum_b grad Phi(x_b) rho_p(x_b) over the cells of sphere p, rho_p
 * its own (subsampled, s) charge density (the mapping of
 * orc_sphere_density_sub); the sum runs over the bounding box in (i,j,k)
 * order.  forces[3p..3p+2]. */
int orc_coulomb_forces(const orc_hier *H, int n, const double *centers,
                       const double *radii, const double *charges,
                       int normalization, int s, double *forces) {
  const level_t *L = &H->L[0];
  const double h = H->h, hs = h / (double)s;
  if (check_periodic_spheres(H, n, centers, radii)) return -1;
  for (int p = 0; p < n; p++) {
    const double R = radii[p], Q = charges[p];
    double img[27][3];
    const int ni = sphere_images(H->per, L->nx, L->ny, L->nz, h, centers[3 * p],
                                 centers[3 * p + 1], centers[3 * p + 2], img);
    const long np = subcount_per(H->per, L->nx, L->ny, L->nz, h, s,
                                 centers[3 * p], centers[3 * p + 1],
                                 centers[3 * p + 2], R);
    double F[3] = {0.0, 0.0, 0.0};
    if (np > 0 || normalization == ORC_PER_VOLUME) {
      const double rho0 = Q / ((4.0 / 3.0) * ORC_PI * (R * R * R));
      for (int m = 0; m < ni; m++) {
        const double cx = img[m][0], cy = img[m][1], cz = img[m][2];
        int i0, i1, j0, j1, k0, k1;
        bbox(L->nx, h, cx, R, &i0, &i1);
        bbox(L->ny, h, cy, R, &j0, &j1);
        bbox(L->nz, h, cz, R, &k0, &k1);
        for (int i = i0; i <= i1; i++)
          for (int j = j0; j <= j1; j++)
            for (int k = k0; k <= k1; k++) {
              const int cnt = sub_count(i, j, k, s, hs, cx, cy, cz, R);
              if (!cnt || !L->unk[IDX(L, i, j, k)]) continue;
              const double rho =
                  normalization == ORC_PER_VOLUME
                      ? rho0 * ((double)cnt / (double)(s * s * s))
                      : (Q * (double)cnt) / ((double)np * (h * h * h));
              double g[3];
              orc_gradient(H, L->phi, i, j, k, g);
              for (int a = 0; a < 3; a++) F[a] = F[a] + g[a] * rho;
            }
      }
    }
    for (int a = 0; a < 3; a++) forces[3 * p + a] = -(h * h * h) * F[a];
  }
  return 0;
}

/* sum_q a_q phi_q in the fixed direction order x-, x+, y-, y+, z-, z+ */
static inline double offdiag(const level_t *L, const double *a,
                             const double *v, int i, int j, int k) {
  return ((((a[1] * get(L, v, i - 1, j, k) + a[2] * get(L, v, i + 1, j, k)) +
            a[3] * get(L, v, i, j - 1, k)) +
           a[4] * get(L, v, i, j + 1, k)) +
          a[5] * get(L, v, i, j, k - 1)) +
         a[6] * get(L, v, i, j, k + 1);
}

/* Red-black Gauss-Seidel half-sweep (colour order c7): for every
 * unknown cell with (i+j+k)%2 == color,  phi_c <- (f_c - sum_q a_q phi_q)/a_cc */
void orc_smooth_half(orc_hier *H, int l, int color) {
  level_t *L = &H->L[l];
#pragma omp parallel for schedule(static)
  for (int i = 0; i < L->nx; i++)
    for (int j = 0; j < L->ny; j++)
      for (int k = 0; k < L->nz; k++) {
        if (((i + j + k) & 1) != color) continue;
        long c = IDX(L, i, j, k);
        if (!L->unk[c]) continue;
        const double *a = &L->A[7 * c];
        double nb = offdiag(L, a, L->phi, i, j, k);
        L->phi[c] = (L->f[c] - nb) / a[0];
      }
}

/* y = A x on level l (masked cells give 0) */
void orc_apply(const orc_hier *H, int l, const double *x, double *y) {
  const level_t *L = &H->L[l];
#pragma omp parallel for schedule(static)
  for (int i = 0; i < L->nx; i++)
    for (int j = 0; j < L->ny; j++)
      for (int k = 0; k < L->nz; k++) {
        long c = IDX(L, i, j, k);
        if (!L->unk[c]) {
          y[c] = 0.0;
          continue;
        }
        const double *a = &L->A[7 * c];
        y[c] = a[0] * x[c] + offdiag(L, a, x, i, j, k);
      }
}

/* r = f - A phi (unknown cells), 0 on masked cells */
void orc_residual(const orc_hier *H, int l, double *r) {
  const level_t *L = &H->L[l];
#pragma omp parallel for schedule(static)
  for (int i = 0; i < L->nx; i++)
    for (int j = 0; j < L->ny; j++)
      for (int k = 0; k < L->nz; k++) {
        long c = IDX(L, i, j, k);
        if (!L->unk[c]) {
          r[c] = 0.0;
          continue;
        }
        const double *a = &L->A[7 * c];
        double Au = a[0] * L->phi[c] + offdiag(L, a, L->phi, i, j, k);
        r[c] = L->f[c] - Au;
      }
}

/* f_{l+1} = R r_l, R the 8-child average (reading c4).  Summation order
 * is a fixed pairwise tree over child bits (dx,dy,dz), dz fastest. */
void orc_restrict_residual(orc_hier *H, int l) {
  level_t *F = &H->L[l];
  level_t *C = &H->L[l + 1];
  orc_residual(H, l, F->r);
#pragma omp parallel for schedule(static)
  for (int I = 0; I < C->nx; I++)
    for (int J = 0; J < C->ny; J++)
      for (int K = 0; K < C->nz; K++) {
        double r[2][2][2];
        for (int a = 0; a < 2; a++)
          for (int b = 0; b < 2; b++)
            for (int c = 0; c < 2; c++)
              r[a][b][c] = F->r[IDX(F, 2 * I + a, 2 * J + b, 2 * K + c)];
        double s = ((r[0][0][0] + r[0][0][1]) + (r[0][1][0] + r[0][1][1])) +
                   ((r[1][0][0] + r[1][0][1]) + (r[1][1][0] + r[1][1][1]));
        C->f[IDX(C, I, J, K)] = 0.125 * s;
      }
}

/* phi_l += alpha * P e_{l+1}; P = nearest-neighbour prolongation,
 * alpha the magnification of the coarse-grid correction (c6). */
void orc_prolong_correct(orc_hier *H, int l, double alpha) {
  level_t *F = &H->L[l];
  const level_t *C = &H->L[l + 1];
#pragma omp parallel for schedule(static)
  for (int i = 0; i < F->nx; i++)
    for (int j = 0; j < F->ny; j++)
      for (int k = 0; k < F->nz; k++) {
        long c = IDX(F, i, j, k);
        if (!F->unk[c]) continue;
        F->phi[c] = F->phi[c] + alpha * C->phi[IDX(C, i / 2, j / 2, k / 2)];
      }
}

static double dot(const level_t *L, const double *x, const double *y) {
  double s = 0.0;
  for (long c = 0; c < L->n; c++)
    if (L->unk[c]) s += x[c] * y[c];
  return s;
}

/* Coarsest-grid solve by unpreconditioned CG, Hestenes-Stiefel
 * from x = 0; stop when ||r|| <= tol ||b|| or after maxit iterations (c8).
 * Writes the solution into phi of level l; returns the iteration count. */
int orc_cg(orc_hier *H, int l, double tol, int maxit) {
  level_t *L = &H->L[l];
  long n = L->n;
  double *x = L->phi, *b = L->f;
  double *r = (double *)malloc(sizeof(double) * n);
  double *p = (double *)malloc(sizeof(double) * n);
  double *q = (double *)malloc(sizeof(double) * n);
  for (long c = 0; c < n; c++) {
    x[c] = 0.0;
    r[c] = L->unk[c] ? b[c] : 0.0;
    p[c] = r[c];
  }
  double rho = dot(L, r, r);
  double bnorm = sqrt(rho);
  int it = 0;
  if (bnorm > 0.0) {
    while (it < maxit) {
      orc_apply(H, l, p, q);
      double pq = dot(L, p, q);
      double a = rho / pq;
      for (long c = 0; c < n; c++) {
        x[c] = x[c] + a * p[c];
        r[c] = r[c] - a * q[c];
      }
      double rho1 = dot(L, r, r);
      it++;
      if (sqrt(rho1) <= tol * bnorm) break;
      double beta = rho1 / rho;
      for (long c = 0; c < n; c++) p[c] = r[c] + beta * p[c];
      rho = rho1;
    }
  }
  free(r);
  free(p);
  free(q);
  H->last_cg_iters = it;
  return it;
}

int orc_last_cg_iters(const orc_hier *H) { return H->last_cg_iters; }

void orc_set_schedule(orc_hier *H, int nu1, int nu2, double alpha,
                      double coarse_tol, int coarse_maxit) {
  H->nu1 = nu1;
  H->nu2 = nu2;
  H->alpha = alpha;
  H->coarse_tol = coarse_tol;
  H->coarse_maxit = coarse_maxit;
}

/* ||f - A phi||_2 on the finest level, unscaled (c10); serial sum */
double orc_residual_norm(const orc_hier *H) {
  const level_t *L = &H->L[0];
  orc_residual(H, 0, L->r);
  double s = 0.0;
  for (long c = 0; c < L->n; c++) s += L->r[c] * L->r[c];
  return sqrt(s);
}

/* V(nu1,nu2)-cycle: pre-smoothing, residual, restriction, coarse
 * phi = 0, recursion, CG on the coarsest level, prolongation with magnified
 * correction, post-smoothing.  Red then black in every sweep (c7). */
static void vcycle_level(orc_hier *H, int l) {
  if (l == H->nlev - 1) {
    orc_cg(H, l, H->coarse_tol, H->coarse_maxit);
    return;
  }
  for (int s = 0; s < H->nu1; s++) {
    orc_smooth_half(H, l, 0);
    orc_smooth_half(H, l, 1);
  }
  if (l == 0 && H->fused_norm) H->in_cycle_norm = orc_residual_norm(H);
  orc_restrict_residual(H, l);
  level_t *C = &H->L[l + 1];
  for (long c = 0; c < C->n; c++) C->phi[c] = 0.0;
  vcycle_level(H, l + 1);
  orc_prolong_correct(H, l, H->alpha);
  for (int s = 0; s < H->nu2; s++) {
    orc_smooth_half(H, l, 0);
    orc_smooth_half(H, l, 1);
  }
}

/* Alg.1: the cycle's residual norm.  Default: ||f - A phi|| of the
 * new iterate (a separate pass).  fused_norm (c11, "negligible"
 * termination check): the norm of the level-0 residual after this cycle's
 * pre-smoothing, the one restricted to level 1 (a single level has no
 * restriction: post-cycle norm). */
double orc_vcycle(orc_hier *H) {
  vcycle_level(H, 0);
  if (H->fused_norm && H->nlev > 1) return H->in_cycle_norm;
  return orc_residual_norm(H);
}

void orc_set_fused_norm(orc_hier *H, int on) { H->fused_norm = on != 0; }

/* Alg.1: while residual >= tol: V-cycle.  tol is relative to the
 * initial residual (c10).  Divergence: NaN or growth > 10x in one cycle. */
int orc_solve(orc_hier *H, double tol, int max_cycles, int *cycles_out,
              double *hist) {
  double r0 = orc_residual_norm(H);
  double prev = r0;
  if (hist) hist[0] = r0;
  int k = 0;
  int status = 1;
  if (r0 == 0.0) status = 0;
  while (status == 1 && k < max_cycles) {
    double rk = orc_vcycle(H);
    k++;
    if (hist) hist[k] = rk;
    if (!(rk == rk) || rk > 10.0 * prev) {
      status = 2;
      break;
    }
    if (rk <= tol * r0) status = 0;
    prev = rk;
  }
  if (cycles_out) *cycles_out = k;
  return status;
}
