/*
 * oracle/mg_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Interface of the plain CPU fp64 oracle for the cell-centered multigrid
 * Poisson solve of Bartuschat & Ruede (arXiv 1410.6609).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  It shares no code, header or constant with the CUDA product
 * (paper_1410_6609_b200/, include/mg.h); the product never loads it.
 *
 * Layout: natural C order, x slowest, z fastest: idx = (i*ny + j)*nz + k.
 * Stencils are stored per cell as 7 doubles in the order
 *   [centre, x-, x+, y-, y+, z-, z+].
 * Face order everywhere: 0 x-, 1 x+, 2 y-, 3 y+, 4 z-, 5 z+.
 */
#ifndef MG_ORACLE_H
#define MG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_DIRICHLET 0
#define ORC_NEUMANN 1
#define ORC_PERIODIC 2 /* both faces of an axis */

#define ORC_PER_CELLS 0  /* rho = Q / (n_p h^3)      (reading c12, default)  */
#define ORC_PER_VOLUME 1 /* rho = Q / (4/3 pi R^3)   (paper's naive map P:481) */

typedef struct orc_hier orc_hier;

/* Build the level hierarchy and all operators (finest folded stencil, coarse
 * stencils by Galerkin R A P).  solid may be NULL (no mask).  Returns NULL on
 * bad arguments. */
orc_hier *orc_create(int nx, int ny, int nz, double h, const int *bc_type,
                     const double *bc_value, const uint8_t *solid,
                     int min_coarse, int max_levels);
void orc_destroy(orc_hier *H);
/* per-cell values of face q (type unchanged); 0 or -1 */
int orc_set_face_values(orc_hier *H, int face, const double *values);
/* per-face-cell boundary patch; returns 0 or -1 (bad arguments) */
int orc_set_bc_patch(orc_hier *H, int face, int a0, int a1, int b0, int b1,
                     int type, double value);

/* cell permittivity eps[nx*ny*nz] > 0 (natural layout), NULL = constant 1;
 * re-assembles the finest operator and every Galerkin level (N4, d10).
 * Set the RHS afterwards (its BC adaptation uses eps).  0 or -1. */
int orc_set_permittivity(orc_hier *H, const double *eps);

int orc_num_levels(const orc_hier *H);
void orc_level_dims(const orc_hier *H, int l, int *dims3);

/* copies of per-level data, natural layout */
void orc_get_stencil(const orc_hier *H, int l, double *out7n);
void orc_get_unknown(const orc_hier *H, int l, uint8_t *out);
void orc_get_phi(const orc_hier *H, int l, double *out);
void orc_set_phi(orc_hier *H, int l, const double *in);
void orc_get_rhs(const orc_hier *H, int l, double *out);
void orc_set_rhs_raw(orc_hier *H, int l, const double *in); /* no BC adaptation */

/* level-0 RHS: f := given field, then BC adaptation. */
void orc_set_rhs(orc_hier *H, const double *f);
/* level-0 RHS: f := charge density of spheres, then BC adaptation.
 * Returns 0, or -1 if a sphere covers no cell centre with ORC_PER_CELLS. */
int orc_set_rhs_from_spheres(orc_hier *H, int n, const double *centers,
                             const double *radii, const double *charges,
                             int normalization);
/* pure geometry helpers used by the pins */
long orc_sphere_cell_count(int nx, int ny, int nz, double h, double cx,
                           double cy, double cz, double R);
void orc_sphere_density(int nx, int ny, int nz, double h, int n,
                        const double *centers, const double *radii,
                        const double *charges, int normalization, double *out);
void orc_bc_adapt(orc_hier *H);
/* subsampling factor s: s^3 sub-cell centres per cell */
long orc_sphere_subcount(int nx, int ny, int nz, double h, int s, double cx,
                         double cy, double cz, double R);
void orc_sphere_density_sub(int nx, int ny, int nz, double h, int s, int n,
                            const double *centers, const double *radii,
                            const double *charges, int normalization,
                            double *out);
int orc_set_rhs_from_spheres_sub(orc_hier *H, int n, const double *centers,
                                 const double *radii, const double *charges,
                                 int normalization, int s);

/* single steps of the method on level l */
void orc_smooth_half(orc_hier *H, int l, int color);
void orc_residual(const orc_hier *H, int l, double *r_out);   /* f - A phi */
void orc_restrict_residual(orc_hier *H, int l);               /* f_{l+1} = R r_l */
void orc_prolong_correct(orc_hier *H, int l, double alpha);
int orc_cg(orc_hier *H, int l, double tol, int maxit);
void orc_apply(const orc_hier *H, int l, const double *x, double *y); /* y = A x */

/* Coulomb force (Eq.14) with the isotropic D3Q19 gradient (Eq.15) of the
 * current level-0 Phi; gradient g[3] at cell (i,j,k) */
void orc_gradient(const orc_hier *H, const double *phi, int i, int j, int k,
                  double *g);
int orc_coulomb_forces(const orc_hier *H, int n, const double *centers,
                       const double *radii, const double *charges,
                       int normalization, int s, double *forces);

/* whole cycles */
void orc_set_schedule(orc_hier *H, int nu1, int nu2, double alpha,
                      double coarse_tol, int coarse_maxit);
double orc_residual_norm(const orc_hier *H);
double orc_vcycle(orc_hier *H);
/* reading c11: orc_vcycle returns the norm of the residual after the cycle's
 * level-0 pre-smoothing (the restricted one) instead of a post-cycle pass */
void orc_set_fused_norm(orc_hier *H, int on);
/* returns 0 converged, 1 not converged at max_cycles, 2 diverged;
 * hist has room for max_cycles+1 entries (may be NULL). */
int orc_solve(orc_hier *H, double tol, int max_cycles, int *cycles_out,
              double *hist);
int orc_last_cg_iters(const orc_hier *H);

#ifdef __cplusplus
}
#endif
#endif
