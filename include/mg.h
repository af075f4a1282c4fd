/*
 * include/mg.h -- C-ABI of the B200-native cell-centered multigrid Poisson
 * solver (libmg_cuda.so), after Bartuschat & Ruede, arXiv 1410.6609.
 * Citations "P:<line>" refer to the paper's LaTeX source.
 *
 * What is solved (Eq.12; Eq.13):
 *     A Phi = f,   A = -Lap_h (7-point finite-volume stencil, spacing h),
 * on a box of nx*ny*nz cells, unknowns at cell centres, eps = 1, with
 * Dirichlet / Neumann conditions on each face folded into the stencil and the
 * right-hand side.  The solver is the paper's cell-centered
 * geometric multigrid: red-black Gauss-Seidel
 * smoothing, residual + 8-cell averaging restriction, nearest-neighbour
 * prolongation with the coarse correction magnified by alpha = 2, Galerkin
 * coarse operators, CG on the coarsest grid, V(nu1,nu2)-cycles.
 *
 * Conventions
 *  - Arrays exchanged with the caller are fp64 in natural C order with x the
 *    slowest and z the fastest axis: a[(i*ny + j)*nz + k].  Cell (i,j,k) has
 *    its centre at ((i+1/2)h, (j+1/2)h, (k+1/2)h).
 *  - Face order: 0 x-, 1 x+, 2 y-, 3 y+, 4 z-, 5 z+.
 *  - Every int return is MG_OK (0) or a negative MG_ERR_* code; the message
 *    of the last error is returned by mg_last_error().
 *  - A context is not thread-safe.  All device work is enqueued on the
 *    context's stream; calls that return host values synchronise it.
 *  - Multi-GPU (nranks > 1, halo backend NCCL): every call is collective, all
 *    ranks call in the same order.  Rank r owns the x-planes
 *    [r*nx/P, (r+1)*nx/P) of every distributed level; caller arrays are then
 *    the rank's slab (nx/P * ny * nz values).  With the LOOPBACK backend one
 *    process holds all P slabs on one GPU (used to test the decomposition)
 *    and caller arrays cover the whole domain (likewise EMULATE, which also
 *    keeps one copy of the agglomerated levels per emulated rank).
 *  - Pointers marked "where" are host pointers (MG_HOST, any host memory;
 *    pinned memory gives full PCIe bandwidth) or device pointers (MG_DEVICE).
 *    The library never keeps or frees caller pointers.
 */
#ifndef MG_H
#define MG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ------------------------------------------------------ */
#define MG_OK 0
#define MG_ERR_ARG (-1)      /* invalid argument                              */
#define MG_ERR_BC (-2)       /* unsupported / singular boundary conditions    */
#define MG_ERR_COARSEN (-3)  /* dimensions cannot form the required hierarchy */
#define MG_ERR_CUDA (-4)     /* CUDA runtime error (or no device)             */
#define MG_ERR_NCCL (-5)     /* NCCL missing or failed                        */
#define MG_ERR_NOMEM (-6)    /* device memory / workspace too small           */
#define MG_ERR_DIVERGED (-7) /* NaN, or residual grew > 10x in one cycle      */
#define MG_ERR_NOTCONV (-8)  /* max_cycles reached (solution stays valid)     */

/* ---- boundary conditions ------------------------------------ */
#define MG_DIRICHLET 0 /* Phi = value on the face:   centre +1, f += 2 g/h^2  */
#define MG_NEUMANN 1   /* dPhi/dn = value (outward): centre -1, f += g/h      */
#define MG_PERIODIC 2  /* P:441-443 "cyclically extend the domain": both
                          faces of an axis; centre and RHS untouched, the
                          neighbour is the opposite side's cell            */

typedef struct {
  int type;     /* MG_DIRICHLET, MG_NEUMANN or MG_PERIODIC                */
  double value; /* g_d (potential) or g_n (outward normal derivative);
                   ignored on periodic faces                              */
} mg_bc;

#define MG_HOST 0
#define MG_DEVICE 1

#define MG_CHARGE_PER_CELLS 0  /* rho = Q/(n_p h^3): charge exact (default)    */
#define MG_CHARGE_PER_VOLUME 1 /* rho = Q/(4/3 pi R^3): the paper's P:481-482  */

#define MG_FIELD_PHI 0 /* solution / coarse-grid correction of a level        */
#define MG_FIELD_RHS 1 /* right-hand side of a level (level 0: BC-adapted)    */

#define MG_HALO_NONE 0     /* single slab (nranks must be 1)                  */
#define MG_HALO_NCCL 1     /* one process per GPU, NCCL send/recv over NVLink */
#define MG_HALO_LOOPBACK 2 /* all nranks slabs in this process on one GPU     */
#define MG_HALO_EMULATE 3  /* all nranks ranks in this process on one GPU with
                              NCCL's data layout: one copy of every
                              agglomerated level per rank, the halo schedule
                              (mg_halo_schedule) and the all-gathers executed
                              as device copies with NCCL's matching and
                              indexing -- tests the NCCL layout on one GPU  */

typedef struct {
  int nu1, nu2;       /* pre/post RBGS sweeps (default 2, 2)      */
  double alpha;       /* coarse-correction magnification (default 2.0) */
  int min_coarse;     /* stop coarsening when min dim <= this (default 4)    */
  int max_levels;     /* 0 = as many as the coarsening rule allows           */
  long long agglomerate_below; /* local cells/GPU below which the remaining
                                  levels are gathered (default 64^3)         */
  double coarse_tol;  /* CG relative tolerance (default 1e-12)               */
  int coarse_maxit;   /* CG iteration cap (default 1000)                     */
  int max_cycles;     /* mg_solve cycle cap (default 100)                    */
  int device;         /* CUDA device ordinal (default 0)                     */
  void *stream;       /* cudaStream_t to enqueue on; NULL = own stream       */
  int rank, nranks;   /* this process's rank / number of slabs (default 0,1) */
  int halo_backend;   /* MG_HALO_* (default NONE)                            */
  unsigned char nccl_id[128]; /* ncclUniqueId from mg_nccl_unique_id (rank 0) */
  void *workspace;    /* optional caller-owned device memory (e.g. a torch
                         uint8 tensor) of >= mg_workspace_bytes(); NULL = the
                         library allocates and frees its own                 */
  size_t workspace_bytes;
  int use_graph;      /* capture one V-cycle as a CUDA graph (default 1)     */
  int fused_norm;     /* reading c11 (Alg.1):
                         0 (default) = mg_vcycle returns ||f - A Phi|| of the
                         new iterate (4, 12 or 16 B/cell of extra traffic:
                         look-ahead sweep, split norm, full pass);
                         1 = it returns the norm of the level-0 residual the
                         cycle computes after pre-smoothing for the
                         restriction (no extra pass).  mg_solve's r_0 is a
                         separate pass in both modes; a single-level
                         hierarchy always reports the post-cycle norm.  The
                         iterates are identical in both modes.              */
  int disable;        /* bitmask of MG_OFF_* (default 0: every fast path the
                         grid allows).  Each bit selects an equivalent slower
                         path -- used to test that the paths agree: the
                         per-cell arithmetic is identical, so iterates are
                         bitwise equal; only reductions may round
                         differently.  Which paths a recorded V-cycle took is
                         reported by mg_cycle_paths().                      */
  int nccl_timeout_ms; /* NCCL contexts: a synchronising call that sees no
                         progress for this long, or an asynchronous NCCL
                         error, aborts the communicator and returns
                         MG_ERR_NCCL (default 600000; 0 = wait forever)     */
  long long tail_cells; /* the coarse end of each V-cycle -- every level from
                         the first one held whole with at most this many
                         cells, down to the coarsest solve and back -- runs
                         as ONE persistent thread-block-cluster kernel
                         instead of a launch per step (box / periodic grids
                         whose coarsest solve is the single-CTA CG; 0 =
                         default 32768 = 32^3; MG_OFF_TAIL disables it)     */
} mg_opts;

/* mg_opts.disable bits */
#define MG_OFF_MARCH 1       /* TMA plane-marching kernels -> direct loads    */
#define MG_OFF_OVERLAP 2     /* multi-slab halo / interior overlap -> serial  */
#define MG_OFF_SPLIT_NORM 4  /* split cycle-end norm -> one full norm pass    */
#define MG_OFF_CG_CLUSTER 8  /* 8-CTA cluster CG -> single-CTA CG             */
#define MG_OFF_MASK_CODES 16 /* masked levels: byte codes -> float records    */
#define MG_OFF_TAIL 32       /* persistent tail kernel -> a launch per step   */
#define MG_OFF_RED0 64       /* restriction + next level's first red sweep
                                (from Phi = 0) -> two kernels               */
#define MG_OFF_LOOKAHEAD 128 /* look-ahead red sweep (the cycle-end norm's red
                                residuals from the next cycle's first red
                                half-sweep) -> a red residual pass          */

/* mg_cycle_paths() bits: the paths the last recorded V-cycle took */
#define MG_PATH_MARCH 1          /* level 0 smoothed by the marching kernel   */
#define MG_PATH_OVERLAP 2        /* halo exchange overlapped with interiors   */
#define MG_PATH_SPLIT_NORM 4     /* norm split over the last black sweep      */
#define MG_PATH_CG_CLUSTER 8     /* coarsest CG on a thread-block cluster     */
#define MG_PATH_CG_VAR 16        /* variable-coefficient coarsest CG          */
#define MG_PATH_PROLONG_FUSED 32 /* prolongation fused with the red sweep     */
#define MG_PATH_FUSED_NORM 64    /* norm from the in-cycle residual (c11)     */
#define MG_PATH_TAIL 128         /* coarse levels in the persistent tail      */
#define MG_PATH_RED0 256         /* a restriction did the next red sweep      */
#define MG_PATH_LOOKAHEAD 512    /* the cycle ended with the look-ahead sweep */

typedef struct mg_ctx mg_ctx;

/* Fill *o with the defaults listed above. */
void mg_default_opts(mg_opts *o);

/* Level plan for (nx,ny,nz,o) without touching a GPU.  Levels follow P:502-507
 * (reading c9): coarsen while every dimension is even, the coarse dimensions
 * are again even and min(dims) > min_coarse.  Fills dims[l][3] (global),
 * local_nx[l] (planes per rank, 0 on levels held whole), *nlevels and
 * *agg_level (first level held whole on every rank; nlevels when nranks==1
 * means "no agglomeration").  Arrays must hold 32 entries.  Returns MG_OK or
 * MG_ERR_ARG / MG_ERR_COARSEN. */
int mg_plan(int nx, int ny, int nz, const mg_opts *o, int *nlevels,
            int *agg_level, int dims[][3], int *local_nx);

/* Device bytes the context needs for (nx,ny,nz,o); 0 on invalid arguments. */
size_t mg_workspace_bytes(int nx, int ny, int nz, const mg_opts *o);

/* Create a solver for nx*ny*nz global cells of spacing h; bc[6] per face.
 * Requires even nx, ny, nz (the coarsest level is "a multiple of two",
 * P:506-507) and at least one Dirichlet face (otherwise A is singular).
 * Periodic faces come in pairs (both faces of an axis, else
 * MG_ERR_BC); every level keeps the periodicity (the Galerkin operator of a
 * periodic grid is again periodic), the ghost layers of periodic axes hold
 * the opposite side's cells, and with nranks > 1 a periodic x axis makes
 * the first and last ranks halo neighbours.  A solid mask or boundary
 * patches cannot be combined with periodic faces (MG_ERR_BC).
 * Returns NULL on error (message in mg_last_error(NULL)). */
mg_ctx *mg_create(int nx, int ny, int nz, double h, const mg_bc *bc);
mg_ctx *mg_create_ex(int nx, int ny, int nz, double h, const mg_bc *bc,
                     const mg_opts *o);
/* Frees library-owned device memory, the stream and the NCCL communicator
 * it created; never the caller's workspace or stream. */
void mg_destroy(mg_ctx *ctx);

/* Thread-local message / code of the last failing call (ctx may be NULL);
 * mg_last_error_code() gives the MG_ERR_* of a failed mg_create(_ex). */
const char *mg_last_error(const mg_ctx *ctx);
int mg_last_error_code(void);
const char *mg_strerror(int code);

/* Writes a fresh ncclUniqueId (128 bytes) for mg_opts.nccl_id; call on rank
 * 0 and broadcast (e.g. with torch.distributed).  MG_ERR_NCCL if libnccl
 * cannot be loaded.  Needs no GPU. */
int mg_nccl_unique_id(unsigned char out[128]);

/* Ghost-plane exchange schedule of one colour array on a distributed level
 * (periodic x: "processes are configured in a periodic
 * arrangement"): the ordered point-to-point operations rank
 * `rank` of `nranks` posts in one NCCL group.  ops[k] = {MG_OP_SEND or
 * MG_OP_RECV, peer rank, plane} with plane one of MG_PLANE_FIRST / _LAST
 * (first / last own x-plane) or MG_GHOST_LO / _HI (ghost plane before /
 * after the slab).  Every rank posts (send last -> right, recv lo-ghost <-
 * left, send first -> left, recv hi-ghost <- right), so that repeated peers
 * (2 ranks with periodic x) match message by message.  Returns the number
 * of operations (0..4) or MG_ERR_ARG.  Pure host logic, no GPU. */
#define MG_OP_SEND 0
#define MG_OP_RECV 1
#define MG_PLANE_FIRST 1
#define MG_PLANE_LAST 2
#define MG_GHOST_LO 3
#define MG_GHOST_HI 4
int mg_halo_schedule(int nranks, int rank, int periodic_x, int ops[4][3]);

/* ---- solid mask (config 5) -------------------------------------------------- */
/* Mark solid cells (solid[i] != 0), natural layout of the WHOLE domain
 * (nx*ny*nz bytes, every rank passes the full array).  Solid cells are not
 * unknowns, their f is 0, and the faces between fluid and solid cells are
 * homogeneous Neumann (reading c19).  Coarse operators are the
 * Galerkin R A P of the masked operator, held in the exact
 * face-transmissibility form.  Switches the context to the
 * variable-coefficient kernels.  solid == NULL removes the mask.  Call before
 * setting the RHS (the RHS is re-zeroed on solid cells). */
int mg_set_mask(mg_ctx *ctx, const uint8_t *solid, int where);
/* Boundary patch (config 5's paper-faithful partial-length electrodes,
 * reading c17): on face `face` the cells with in-face coordinates
 * a in [a0,a1), b in [b0,b1) get BC (type, value).  In-face coordinates are
 * the two other axes in (x,y,z) order (x faces: (y,z); y faces: (x,z);
 * z faces: (x,y)), global indices.  Switches the context to the
 * variable-coefficient kernels (level-0 coefficient records) and rebuilds the
 * Galerkin hierarchy; set the RHS afterwards (its BC adaptation uses the
 * patch values).  MG_ERR_ARG for a rectangle outside the face, MG_ERR_BC for
 * a type other than Dirichlet / Neumann. */
int mg_set_bc_patch(mg_ctx *ctx, int face, int a0, int a1, int b0, int b1,
                    int type, double value);
/* Per-cell boundary values on face `face` (the face's BC type unchanged):
 * values[a*nb + b] for the face cells in the in-face order of
 * mg_set_bc_patch (na x nb = the two other global extents).  For analytic
 * Dirichlet data, e.g. the charged-sphere validation (Eq.18).
 * The operator is unchanged (only the RHS adaptation uses the values); set
 * the RHS afterwards.  MG_ERR_BC on a periodic face (it has no boundary). */
int mg_set_face_values(mg_ctx *ctx, int face, const double *values);
/* Variable (jumping) permittivity (the solver "is extensible
 * for discontinuous dielectricity coefficients ... by Galerkin coarsening",
 * P:513-516): solves -div(eps grad Phi) = rho with eps[i] > 0 per
 * cell (natural layout of the WHOLE domain, every rank passes the full
 * array; NULL = constant 1, the paper's P:386-389).  Reading d10: face flux
 * eps_f (Phi_c - Phi_n)/h^2 with the harmonic mean eps_f = 2 eps_c eps_n /
 * (eps_c + eps_n); boundary faces use eps_c (Dirichlet: centre + 2 eps_c/h^2,
 * f += 2 eps_c g/h^2; Neumann: f += eps_c g/h); coarse levels are the
 * Galerkin R A P.  Combines with mg_set_mask / mg_set_bc_patch; not with
 * periodic faces (MG_ERR_BC).  eps <= 0 -> MG_ERR_ARG.  Switches the context
 * to the variable-coefficient kernels (fp64 records, 64 B per cell and
 * level); set the RHS afterwards. */
int mg_set_permittivity(mg_ctx *ctx, const double *eps, int where);
/* The operator of level l as 7 coefficients per cell [centre, x-, x+, y-, y+,
 * z-, z+] (natural layout, the caller's part as mg_get_field), zeros on solid
 * cells.  For tests against the oracle's Galerkin stencils. */
int mg_get_stencil(mg_ctx *ctx, int level, double *out, int where);

/* ---- right-hand side ----------------------------------------------------- */
/* f := charge density of n uniformly charged spheres.  On a
 * periodic axis a sphere also covers the cells of its periodic images
 * (centre +- n h); there the centre must lie in [0, n h) and 2R + 2h <= n h
 * (the images then reach disjoint cells), else MG_ERR_ARG.  Each cell
 * is subdivided into s^3 sub-cells (subsampling factor s = `subsample`,
 * 1..16; s = 1 is the plain rule "each cell whose center is
 * overlapped") and cnt = number of sub-cell centres with
 * |x - c_p|^2 <= R_p^2 (inclusive, reading c13).  The cell receives
 * (Q_p cnt)/(n_p h^3) (MG_CHARGE_PER_CELLS, n_p = covered sub-cells of the
 * whole domain: the charge is exact) or (Q_p/(4/3 pi R_p^3)) (cnt/s^3)
 * (PER_VOLUME, the paper's volume-fraction mapping); cells covered by
 * several spheres receive the sum.  Then the finest-grid BC adaptation
 * (P:731-732).  centers[3n] (x,y,z physical), radii[n], charges[n] are host
 * arrays, read before return; every rank passes the full list.
 * Errors: n < 0, R <= 0, subsample outside 1..16, a bad normalization or
 * periodic-axis placement (MG_ERR_ARG before anything is written: f keeps
 * its previous value); a sphere that covers no sub-cell centre with
 * PER_CELLS (MG_ERR_ARG, detected by the mapping itself: f then holds the
 * other spheres' density -- set it again).  Phi is not touched (warm start,
 * P:1321-1322). */
int mg_set_rhs_from_spheres(mg_ctx *ctx, int n, const double *centers,
                            const double *radii, const double *charges,
                            int normalization, int subsample);

/* f := given field (natural layout, the rank's slab), then the BC
 * adaptation: f += 2 g_d/h^2 per Dirichlet face and f += g_n/h per Neumann
 * face the cell touches, in face order. */
int mg_set_rhs(mg_ctx *ctx, const double *f, int where);

/* ---- Coulomb force ------------------------------------------ */
/* Electrostatic force on each of n spheres from the current Phi (Eq.14,
 * P:466-471): F_p = -h^3 sum_b grad Phi(x_b) rho_p(x_b) over the cells of
 * sphere p, rho_p its own charge density with the mapping of
 * mg_set_rhs_from_spheres (normalization, subsample = the force subsampling
 * factor s_F of Table 5), grad Phi the isotropic D3Q19 gradient (Eq.15,
 * P:472-478; central / one-sided differences where a D3Q19 neighbour is
 * outside the domain or solid, reading d6).  Host arrays; forces_out[3n].
 * Collective for NCCL contexts (partial sums all-gathered, summed in rank
 * order).  Errors as mg_set_rhs_from_spheres. */
int mg_coulomb_forces(mg_ctx *ctx, int n, const double *centers,
                      const double *radii, const double *charges,
                      int normalization, int subsample, double *forces_out);

/* ---- time stepping ------------------------------------------- */
/* The potential part of one time step of Alg.1 for spheres at
 * their current positions: f := their charge density (exactly
 * mg_set_rhs_from_spheres(normalization, subsample)); V-cycles from the
 * current Phi (warm start: "later steps only update the previous solution",
 * P:1321-1322) -- exactly `cycles` of them if cycles > 0 (the paper's
 * regime: 5 V(3,3) at the first step, then 1), or, with cycles == 0, while
 * ||f - A Phi||_2 > abs_tol (Alg.1 "while residual >= tol"; an
 * absolute norm, as the paper monitors 1.5e-8), at most
 * max_cycles; then, if forces_out != NULL, the Coulomb forces of the same
 * spheres on the new Phi (mg_coulomb_forces with force_subsample; forces
 * [3n]).  *cycles_out and *res_out (post-step residual norm) may be NULL.
 * With cycles > 0 the RHS, the cycles and the forces are enqueued back to
 * back and the host waits once at the end, so a sphere that covers no cell
 * centre (MG_ERR_ARG) is reported after the step's cycles have run.
 * Returns MG_OK, MG_ERR_NOTCONV (cycles == 0 and max_cycles reached; forces
 * are still computed), or the errors of the calls it makes. */
int mg_timestep(mg_ctx *ctx, int n, const double *centers, const double *radii,
                const double *charges, int normalization, int subsample,
                int cycles, double abs_tol, double *forces_out,
                int force_subsample, int *cycles_out, double *res_out);

/* ---- solve --------------------------------------------------------------- */
/* One V(nu1,nu2)-cycle (Alg.1); *res_norm_out (may be NULL)
 * = ||f - A Phi||_2 over all cells after the cycle (unscaled, reading c10).
 * Synchronises.  MG_ERR_DIVERGED if the norm is NaN or > 10x the previous
 * cycle's.  On one level-0 slab (nu1, nu2 >= 1, no mask, true cycle-end
 * norm) the cycle ends with the look-ahead red sweep: the next cycle's first
 * red half-sweep is computed into a second red buffer together with the red
 * residuals of the new iterate; Phi as seen by every
 * other call is the cycle's iterate.  Any call that changes Phi, f, the BCs
 * or the operator discards the look-ahead (the next cycle recomputes it);
 * MG_OFF_LOOKAHEAD turns it off. */
int mg_vcycle(mg_ctx *ctx, double *res_norm_out);

/* Asynchronous fixed-count solve, for pipelining independent problems:
 * f := the given field (natural layout, the rank's slab; BC adaptation as
 * mg_set_rhs), Phi := 0, `cycles` V-cycles, then Phi copied to phi_out
 * (natural layout; may be NULL).  Returns after enqueueing (no host
 * synchronisation).  Host buffers (MG_HOST, pinned for real overlap) move on
 * two library copy streams through three staging slots, so the upload of the
 * next problem and the download of the previous one overlap this problem's
 * cycles, which stay on the context's stream.  The caller keeps f and
 * phi_out alive until mg_wait; no per-cycle divergence check. */
int mg_solve_async(mg_ctx *ctx, const double *f, int where_f, double *phi_out,
                   int where_phi, int cycles);
/* Copy-out of the current level-0 Phi (natural layout, the rank's slab)
 * without host synchronisation: the conversion from the split layout is
 * enqueued on the context's stream into one of the library's three staging
 * slots and, for where = MG_HOST, the device-to-host copy on the library's
 * copy stream, so that it overlaps the work enqueued next (e.g. the next
 * time step's RHS and cycles).  `out` (pinned host memory for overlap, or
 * device memory) must stay alive and unread until mg_wait.  A fourth call
 * before mg_wait reuses the first call's slot after its copy finished.
 * Errors: null ctx / out, bad `where` (MG_ERR_ARG). */
int mg_get_solution_async(mg_ctx *ctx, double *out, int where);

/* Synchronise the context's streams (compute and copies); *res_norm_out
 * (may be NULL) = the residual norm after the last V-cycle.
 * MG_ERR_DIVERGED if it is NaN. */
int mg_wait(mg_ctx *ctx, double *res_norm_out);

/* r0 = norm of the current Phi; V-cycles while r_k > tol*r0 (Alg.1,
 * P:547-550), at most mg_opts.max_cycles.  *cycles_out and
 * res_hist[0..cycles] (the caller's array of max_cycles+1 doubles) may be
 * NULL.  MG_OK, MG_ERR_NOTCONV at max_cycles, or MG_ERR_DIVERGED. */
int mg_solve(mg_ctx *ctx, double tol, int *cycles_out, double *res_hist);
/* mg_solve with an explicit cycle limit: max_cycles > 0 replaces
 * mg_opts.max_cycles for this call (res_hist: max_cycles+1 doubles); <= 0
 * uses mg_opts.max_cycles. */
int mg_solve_n(mg_ctx *ctx, double tol, int max_cycles, int *cycles_out,
               double *res_hist);

/* ||f - A Phi||_2 for the current Phi on the finest level, unscaled (Alg.1
 * "residual"; reading c10), summed in a fixed order (per-CTA partials,
 * then in CTA and, for NCCL contexts, rank order).  Synchronises the stream.
 * Errors: null ctx / out (MG_ERR_ARG), MG_ERR_CUDA, MG_ERR_NCCL. */
int mg_residual_norm(mg_ctx *ctx, double *out);

/* ---- solution I/O -------------------------------------------------------- */
int mg_get_solution(mg_ctx *ctx, double *out, int where);
int mg_set_solution(mg_ctx *ctx, const double *in, int where);
int mg_zero_solution(mg_ctx *ctx);

/* ---- single steps (parity tests and composition) ------------------------- */
int mg_num_levels(const mg_ctx *ctx);
/* global dims of level l */
int mg_level_dims(const mg_ctx *ctx, int level, int dims[3]);
/* Copy a level's field out / in, natural layout.  Level 0 and distributed
 * levels: the caller's slab (LOOPBACK: whole domain); levels held whole:
 * the whole level. */
int mg_get_field(mg_ctx *ctx, int level, int field, double *out, int where);
int mg_set_field(mg_ctx *ctx, int level, int field, const double *in,
                 int where);
/* One red (color 0: (i+j+k) even in global level indices) or black (1)
 * half-sweep of RBGS on level l, followed by its ghost exchange.
 * from_zero != 0 treats the other colour as 0 (first sweep after the coarse
 * Phi is zeroed). */
int mg_smooth_half(mg_ctx *ctx, int level, int color, int from_zero);
/* f_{l+1} := R (f_l - A_l Phi_l), R the 8-child average. */
int mg_residual_restrict(mg_ctx *ctx, int level);
/* Phi_l += alpha * P Phi_{l+1}, P nearest-neighbour. */
int mg_prolong_correct(mg_ctx *ctx, int level);
/* CG on the coarsest level from 0; *iters may be NULL. */
int mg_coarse_solve(mg_ctx *ctx, int *iters);

/* ---- measurement ---------------------------------------------------------- */
/* Enable (1) / disable (0) CUDA-event timing of the V-cycle's kernels on the
 * context's stream (events are part of the captured graph; re-captures). */
int mg_set_profiling(mg_ctx *ctx, int on);
/* Times of the last profiled mg_vcycle, in milliseconds:
 *   out[0] level-0 RBGS half-sweeps (sum)   out[1] number of them
 *   out[2] level-0 residual+restriction      out[3] level-0 prolongation
 *   out[4] residual norm                      out[5] levels >= 1 incl. CG
 *   out[6] whole cycle (first to last kernel) out[7] kernel launches/cycle
 * MG_ERR_ARG if profiling was off during the last cycle. */
int mg_last_cycle_times(mg_ctx *ctx, double out[8]);
/* As mg_last_cycle_times, n >= 10 outputs, plus
 *   out[8] level-0 smoothing launches timed in out[0]
 *   out[9] level-0 half-sweeps they perform (one per launch)
 * and with n >= 12
 *   out[10] levels >= 1 held whole on every rank (the agglomerated levels;
 *           every level >= 1 of a single slab) incl. the coarsest solve
 *   out[11] the coarsest-grid CG alone
 * (LOOPBACK / NCCL: one copy; EMULATE times every rank's copy). */
int mg_last_cycle_times_ex(mg_ctx *ctx, double *out, int n);
/* Number of kernels one mg_vcycle launches (counted when it is recorded). */
int mg_cycle_launches(const mg_ctx *ctx);
/* MG_PATH_* bits of the kernel paths the last recorded V-cycle took (0
 * before the first cycle); MG_ERR_ARG for a null ctx. */
int mg_cycle_paths(const mg_ctx *ctx);
/* cudaStream_t of the context (for event timing by the caller). */
void *mg_stream(const mg_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* MG_H */
