/*
 * stk.h — C ABI of the B200-native matrix-free Stokes operator and Uzawa
 * multigrid (data-parallel hot path of arXiv:1604.07994, "A symmetric decoupled
 * weak formulation ..." — citations P:L are PAPER.md line numbers).
 *
 * Problem: on the unit cube, uniformly refined into
 * n^3 cubes x 6 Kuhn tetrahedra, with element-wise constant viscosity
 * mu_T, find P1 velocity u and P1 pressure p with
 *
 *     [ A   B^T ] [u]   [f_h]        A : modified viscous form a_tr
 *     [ B   -C  ] [p] = [ g ]        B : b(v,q) = -(div v, q)
 *                                    C : pressure stabilisation (DESIGN R1)
 *
 * A is applied matrix-free: per-class constant Laplacian stencils inside the
 * isoviscous subdomains, full a_tr rows only at the interface Gamma_12 and
 * the traction boundary Gamma_F (eq. equivalence-stencil).
 *
 * Conventions (all calls):
 *  - Every call returns stk_status; no C++ exception crosses the ABI.
 *  - "dev" pointers are CUDA device pointers (e.g. torch tensors' data_ptr);
 *    "host" pointers are CPU memory.  The caller owns every pointer it passes;
 *    setup arrays are copied during the call.  The context owns the level
 *    hierarchy, stencils, interface data, coarse inverse and communicator.
 *  - Device vectors hold 4 fields (u1,u2,u3,p) in the padded z-slab layout
 *    returned by stk_layout (element (f,i,j,k) at
 *    f*field_stride + (k - z0 + 1)*pitch_y + (j + 1)*pitch_x + (i + 1), doubles;
 *    planes k = z0-1 and z0+nz_local are halo planes owned by the neighbours,
 *    column i = -1 and row j = -1 are an unused ghost frame).
 *    Allocate stk_layout(...).vec_len doubles per vector.
 *  - Velocity entries at Dirichlet vertices (closure of Dirichlet faces) are
 *    ignored on input (treated as 0) and written as 0 on output.  On free-slip
 *    faces the normal component is eliminated: it is written as 0 on output and
 *    must be 0 on input (stk_zero_eliminated; every library output keeps it).
 *    Pressure lives at every vertex.
 *  - All device work is stream-ordered on cfg.stream; calls return before the
 *    work completes, except stk_solve and calls that return host data.
 *  - Errors: STK_EINVAL bad argument / size; STK_ESTATE call order violated
 *    (create -> set_viscosity -> assemble -> the rest); STK_ECUDA / STK_ENCCL
 *    a CUDA / NCCL failure (message in stk_last_error); STK_ENOCONV the solve
 *    did not reach rtol (the iterate and history are still written).
 */
#ifndef STK_H
#define STK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct stk_ctx stk_ctx;
/* a group of nranks contexts of ONE process on ONE device (loopback exchanger) */
typedef struct stk_loopback stk_loopback;

typedef enum {
  STK_OK = 0,
  STK_ENOCONV = 1,
  STK_EINVAL = -1,
  STK_ENOMEM = -2,
  STK_ECUDA = -3,
  STK_ENCCL = -4,
  STK_ESTATE = -5,
  STK_EUNSUP = -6
} stk_status;

/* viscous form of the A block: modified a_tr, strain a_sym,
 * gradient (mu grad u, grad v) */
typedef enum { STK_FORM_MOD = 0, STK_FORM_SYM = 1, STK_FORM_GRAD = 2 } stk_form;
/* faces x0,x1,y0,y1,z0,z1: homogeneous Dirichlet u = 0, traction free
 * sigma n = 0, or free-slip u.n = 0, n x sigma n = 0 (the
 * face-normal velocity component is eliminated, the tangential ones are free; every
 * vertex of a free-slip face is an explicit-stencil row).  Dirichlet wins on shared
 * edges/corners; a vertex on free-slip faces of several normals loses each normal.
 * stk_create needs a Dirichlet face or free-slip faces of all three normals (Korn,
 * P:109-111); without traction faces the pressure is fixed by the gauge. */
typedef enum { STK_FACE_DIRICHLET0 = 0, STK_FACE_TRACTION = 1, STK_FACE_FREESLIP = 2 } stk_face;
/* block mask for stk_apply: y_u = [A u] + [B^T p], y_p = [B u] - [C p] */
enum { STK_BLK_A = 1, STK_BLK_BT = 2, STK_BLK_B = 4, STK_BLK_C = 8, STK_BLK_ALL = 15 };
/* where a canonical (non-padded) array lives */
enum { STK_HOST = 0, STK_DEVICE = 1 };

typedef struct {
  int32_t n;          /* finest intervals per direction, power of 2, >= 4 */
  int32_t n_coarse;   /* coarsest level intervals (direct solve), default 4 */
  int32_t form;       /* stk_form */
  int32_t face[6];    /* stk_face per face */
  double delta;       /* stabilisation constant, c(p,q) = sum_T delta h^2/mu_T (grad p, grad q)_T; default 1/12 */
  int32_t nu_pre, nu_post, nu_inc; /* V_var smoothing: nu + nu_inc * level (DESIGN R13) */
  double omega;       /* Schur-complement under-relaxation, 0.3 */
  int32_t ncolors_u;  /* velocity GS colours (i+j+k) mod ncolors_u: 2 (red-black) or 4 */
  int32_t krylov;     /* 0: stk_solve iterates V-cycles; m > 0: right-preconditioned
                         GMRES(m) with one V-cycle as preconditioner */
  int32_t rank, nranks; /* z-slab owner and number of ranks (one GPU each) */
  void* stream;       /* cudaStream_t; NULL = legacy default stream */
  int32_t coarse_mu;  /* coarse-level viscosity of the A block per coarse tet, from its 8 Bey
                         children (DESIGN R15): 0 = default = 1; 1 = arithmetic mean
                         (the coarse A is then the Galerkin product P^T A P); 2 = harmonic mean.
                         The weight 1/mu of C and of the gauge is always the mean of the children's
                         1/mu.  (SURVEY's "centroid" rule is degenerate for Bey refinement: the
                         coarse centroid lies on the diagonal shared by the four inner children.) */
} stk_config;
enum { STK_COARSE_MU_DEFAULT = 0, STK_COARSE_MU_ARITH = 1, STK_COARSE_MU_HARMONIC = 2 };

typedef struct {
  int32_t n;          /* intervals of this level */
  int32_t nx, ny;     /* n+1 vertices in x and y */
  int32_t nz_local;   /* vertex planes owned by this rank */
  int32_t z0;         /* global index of the first owned plane */
  int64_t pitch_x, pitch_y, field_stride; /* in doubles */
  int64_t vec_len;    /* doubles per 4-field vector */
  int64_t n_irregular; /* vertices whose rows use the full (interface/boundary) stencil */
  int64_t n_vertices; /* owned vertices */
} stk_layout_t;

typedef struct {
  int32_t cycles;
  double rho;         /* mean residual reduction factor of the last cycles */
  double rel_res;     /* ||b - K x|| / ||b|| over free DoFs */
  double t_total_s;   /* device time of the solve */
  double res_hist[256];
  double t_level_s[16]; /* device time by level: [0] the finest level (smoothing, residual,
                           transfers to/from level 1, Krylov vector work), [1] levels >= 1
                           together (one CUDA graph per V-cycle, events around it); rest 0 */
  int32_t nan_seen;
} stk_report;

/* NCCL unique id for nranks > 1: call on rank 0, broadcast the 128 bytes
 * (e.g. with torch.distributed), pass to stk_create on every rank. */
stk_status stk_nccl_unique_id(uint8_t id[128]);

/* Create a context on the current CUDA device (n^3 cubes x 6 tets; the
 * V_var hierarchy of P:1236 with levels n, n/2, ..., n_coarse).  Checks n (power
 * of 2, n/nranks divisible by 2 on every distributed level).  id may be NULL when
 * nranks == 1.  *out is set (to a context holding the error message) even on
 * failure; destroy it with stk_destroy. */
stk_status stk_create(const stk_config* cfg, const uint8_t* id, stk_ctx** out);

/* Loopback exchanger: the nranks contexts of one process share one
 * device and ONE stream (cfg.stream must be equal, else STK_EINVAL); each context is
 * driven by its own host thread, and every collective (halo planes, allreduce,
 * coarse agglomeration) is a host rendezvous of the nranks threads followed by one
 * cudaMemcpyAsync per plane / range.  Same results as nranks GPUs over NCCL (the
 * apply and V-cycle bitwise equal to nranks = 1).  The group outlives its contexts. */
stk_status stk_loopback_create(int32_t nranks, stk_loopback** out);
stk_status stk_create_loopback(const stk_config* cfg, stk_loopback* group, stk_ctx** out);
stk_status stk_loopback_destroy(stk_loopback* group);

/* Element viscosity partition.  elem_class: host uint8 array of this
 * rank's cube layers cz in [z0_cubes, z1_cubes) (see stk_cube_range), layout
 * [cz][cj][ci][t], t = Kuhn permutation index; class_mu: nclass
 * (<= 254; ids 0xFE/0xFF are reserved) viscosities > 0.  Both copied.
 * STK_EINVAL if an element class is >= nclass or a viscosity is not > 0. */
stk_status stk_set_viscosity(stk_ctx* ctx, const uint8_t* elem_class, const double* class_mu,
                             int32_t nclass);
/* cube layers [*z0, *z1) this rank must pass to stk_set_viscosity */
stk_status stk_cube_range(const stk_ctx* ctx, int32_t* z0, int32_t* z1);

/* Assemble all levels: coarse element coefficients
 * (DESIGN R15: per coarse tet the arithmetic mean of its 8 Bey children's mu for A
 * -- the coarse A is then the Galerkin product P^T A P -- and the mean of 1/mu for
 * C; the class is the children's common class or MIXED), per-vertex classification
 * (regular row of class k: isoviscous star; else an interface / boundary row with
 * an explicit stencil), constant subdomain stencils per class, and the
 * coarsest-level inverse (P:1245 direct coarse solve). */
stk_status stk_assemble(stk_ctx* ctx);

stk_status stk_layout(const stk_ctx* ctx, int32_t level, stk_layout_t* out);

/* canonical <-> padded device layout.  canon: 4 fields x (n+1)^3 doubles,
 * field-major, vertex v = i + (n+1)(j + (n+1)k) (this rank's owned planes only:
 * 4 x (n+1)^2 x nz_local, planes z0..z0+nz_local-1).  where = STK_HOST/DEVICE. */
stk_status stk_import(stk_ctx* ctx, int32_t level, const double* canon, int32_t where,
                      double* dev_vec);
stk_status stk_export(stk_ctx* ctx, int32_t level, const double* dev_vec, double* canon,
                      int32_t where);
/* The stabilised P1-P0 operator (§3.3-3.4) on the finest
 * level: P1 velocity as above, one pressure per tetrahedron,
 *   y  = A u + B0^T p0          (velocity fields of the device level vectors x, y)
 *   y0 = B0 u - C0 p0           (device arrays of 6 n^3 doubles, element order of the
 *                                classes: e = 6 (i + n (j + n k)) + t)
 * with b(v,q) = -(div v, q) and the facet-jump stabilisation of eq. (stabc)
 * (P:550-557): c(p,q) = gamma sum_i 1/(2 mu_i) sum_{F interior facet of Omega_i}
 * |T1||T2|/(|T1|+|T2|) [p][q] -- no jump penalised across Gamma_12 or on the
 * boundary; gamma = 1 in the paper's experiments.  The pressure field of x
 * is not read.  nranks == 1 only (STK_EUNSUP otherwise); STK_EINVAL for gamma <= 0. */
stk_status stk_p0_apply(stk_ctx* ctx, const double* x, const double* p0, double* y, double* y0, double gamma);
/* The local flux post-process of the P1-P0 scheme: flux[4 e + m] (device,
 * 4 x 6 n^3 doubles) = int_F j_{F;T} over the facet of tet e opposite its local Kuhn
 * vertex m: int_F u_h . n_T plus, on facets interior to one isoviscous subdomain,
 * gamma/(2 mu) |T||T'|/(|T|+|T'|) (p_T - p_T').  For a discrete solution with zero
 * mass rhs every element's four fluxes sum to 0 (exact element-wise conservation). */
stk_status stk_p0_fluxes(stk_ctx* ctx, const double* x, const double* p0, double* flux, double gamma);
/* Solve the P1-P0 system K0 (u, p0) = (b_u, b0) from the given (x_u, x0) (device; b_u,
 * x_u level-0 vectors whose pressure field is ignored, b_u 0 at eliminated DoFs; b0, x0
 * 6 n^3 per-tet values) to ||b - K0 x|| / ||b|| <= rtol: right-preconditioned GMRES(m)
 * (1 <= m <= 31, CGS2) whose preconditioner maps the P0 residual to the P1 pressure
 * (each tet's integral shared by its 4 vertices), applies one V_var cycle of the P1-P1
 * multigrid of this context (same velocity space and form), averages the P1
 * pressure correction per tet and adds the element-local term -(mu_T / 2|T|) r0 (the
 * 1/mu-weighted P0 mass inverse, for the per-tet modes outside the P1 space).  Without traction faces the mean of p0 is removed at
 * the end.  Synchronous; report gets iterations, residual history and device time.
 * nranks == 1 only; STK_ENOCONV (positive, x holds the last iterate) if rtol is not
 * reached within max_its preconditioner applications. */
stk_status stk_p0_solve(stk_ctx* ctx, const double* b_u, const double* b0, double* x_u, double* x0, double gamma,
                        double rtol, int32_t max_its, int32_t m, stk_report* report);
/* Coarsest-level solver, taking effect at the next stk_assemble.  kind 0 (default): the
 * exact solve of the A_tr coarse system by a dense inverse ("a direct coarse grid
 * solver ... is not problematic").  kind 1: the paper's Krylov coarse solver:
 * the strain form A_sym on the coarse level, the momentum right-hand side corrected to
 * r1 + B^T M_L^-1 r2 (DESIGN R25: M_L = diag int phi/mu, the 1/mu-weighted lumped mass),
 * and block-diagonal preconditioned MINRES from zero -- minres_its iterations (stopping
 * early at gamma_{j+1} <= 1e-14 gamma_1, R24), velocity block cg_its steps of
 * Jacobi-preconditioned CG on A_sym, pressure block M_L -- in one thread block
 * (kernels_minres.cuh).  kind 1 needs the coarsest level held whole (nranks == 1 or a
 * replicated level, else STK_EUNSUP at assembly) and supports n_coarse up to 16.
 * STK_EINVAL for kind outside 0..1, minres_its < 1, cg_its < 0. */
stk_status stk_set_coarse_solver(stk_ctx* ctx, int32_t kind, int32_t minres_its, int32_t cg_its);
/* Set the eliminated velocity entries of a device level vector to 0 (all three on
 * Dirichlet faces, the normal one on free-slip faces, P:97 / P:104-105).  Operator
 * inputs (stk_apply, stk_residual, stk_smooth, stk_solve's x) must hold 0 there when a
 * face is free-slip: the constant-stencil kernels read boundary planes as stored
 * (Dirichlet planes are never read).  stk_import does not mask -- a nodal forcing f is
 * imported whole, since its boundary values enter b = M f at interior rows. */
stk_status stk_zero_eliminated(stk_ctx* ctx, int32_t level, double* dev_vec);

/* Right-hand side b = (f_h, 0).  kind 0: nodal f given as a
 * device level vector (padded layout, fields 0..2 = f; halo planes are
 * exchanged by the call), b_u = consistent mass * f.
 * kind 1: element-constant f: f_dev = uint8 forcing class per element (same
 * layout as stk_set_viscosity), table = host 3 x nftab doubles. */
stk_status stk_load_vector(stk_ctx* ctx, int32_t kind, const void* f_dev, const double* table,
                           int32_t nftab, double* b_dev);

/* y = K x restricted to the requested blocks (STK_BLK_*) on level `level`
 * (0 = finest).  The measured hot kernel. */
stk_status stk_apply(stk_ctx* ctx, int32_t level, uint32_t blocks, const double* x, double* y);
/* r = b - K x; if norms != NULL, writes host norms[5] = ||r_u1||^2, ||r_u2||^2,
 * ||r_u3||^2, ||r_p||^2, total (all ranks; synchronises). */
stk_status stk_residual(stk_ctx* ctx, int32_t level, const double* x, const double* b, double* r,
                        double* norms);
/* `steps` Uzawa smoothing steps in place on x. */
stk_status stk_smooth(stk_ctx* ctx, int32_t level, double* x, const double* b, int32_t steps);
/* b_c = R r_f = P^T r_f, coarse level = fine_level + 1 */
stk_status stk_restrict(stk_ctx* ctx, int32_t fine_level, const double* r_f, double* b_c);
/* x_f += P x_c: the "standard" prolongation of P:1243 (DESIGN R14) -- nodal
 * interpolation of the coarse P1 function (fine vertex 2I takes x_c(I), the midpoint
 * of the coarse Kuhn edge (I, I+d) the mean of its ends), all 4 fields; eliminated
 * velocity entries of x_f stay 0.  coarse_level = fine level + 1; x_c needs no halo. */
stk_status stk_prolong_add(stk_ctx* ctx, int32_t coarse_level, const double* x_c, double* x_f);
/* one V_var cycle (nu_pre + nu_inc*l Uzawa steps before and
 * nu_post + nu_inc*l after the coarse correction on level l, restriction R = P^T,
 * coarsest-level solve as stk_set_coarse_solver selects) on the finest level, in
 * place on x; b and x are finest-level device vectors. */
stk_status stk_vcycle(stk_ctx* ctx, const double* b, double* x);
/* Solve K x = b from the given x: V_var cycles (the paper's
 * all-at-once multigrid) or, cfg.krylov = m > 0, right-preconditioned GMRES(m) with
 * one V-cycle from zero as the preconditioner (DESIGN R23), until ||b - Kx||/||b|| <=
 * rtol over the free DoFs; max_cycles bounds the preconditioner applications.  The
 * mu^-1-weighted pressure gauge is applied at the end.  Synchronous; report
 * (may be NULL) gets the residual history, rho, device time and t_level_s.
 * STK_ENOCONV (positive: x holds the last iterate) when rtol is not reached. */
stk_status stk_solve(stk_ctx* ctx, const double* b, double* x, double rtol, int32_t max_cycles,
                     stk_report* report);
/* subtract the mu^-1-weighted mean pressure (Q of P:136); no-op with traction faces */
stk_status stk_gauge(stk_ctx* ctx, int32_t level, double* x);
/* per-field squared norms of a level vector over owned free DoFs (host out[5]) */
stk_status stk_norms(stk_ctx* ctx, int32_t level, const double* x, double* out);

/* Optional: select the kernel implementation for levels >= 64 intervals:
 * 1 = tiled constant-stencil kernels (default), 0 = generic element-row kernels. */
stk_status stk_set_kernel_mode(stk_ctx* ctx, int32_t mode);
/* Optional: inside the V-cycle, levels >= 1 with n_l <= row_n (default 16) run
 * the lean one-thread-per-row kernels: constant stencils on isoviscous rows,
 * explicit 4x4-block stencils (assembled by stk_assemble) on the
 * Gamma_12 / Gamma_F rows.  0 = off (tiled / generic kernels).  Applies to the
 * V-cycle only: stk_apply / stk_residual / stk_smooth keep their kernels.
 * STK_EINVAL for row_n < 0. */
stk_status stk_set_row_n(stk_ctx* ctx, int32_t row_n);
/* First row-kernel level, or -1. */
int32_t stk_row_level(const stk_ctx* ctx);
/* Optional: row levels with n_l <= fuse_n that this rank holds whole run their
 * part of the V-cycle as ONE persistent cooperative kernel with software grid
 * barriers between the phases (default 0 = off: one launch per phase, replayed
 * as a CUDA graph).  STK_EINVAL for fuse_n < 0. */
stk_status stk_set_fuse_n(stk_ctx* ctx, int32_t fuse_n);
/* First fused level, or -1 when the fused V-cycle is not used. */
int32_t stk_fused_level(const stk_ctx* ctx);
/* Diagnostics for integer parity: the element classes (0xFE = MIXED) of the stored
 * cube layers of a level ([cz][cj][ci][t], cz0..cz1 as stk_partition reports) and,
 * if emu_host != NULL, the per-tet (mu_A, 1/mu_C) pairs (2 doubles per tet; zeros on
 * level 0, whose coefficients are the class table); and the per-vertex row codes of
 * the owned vertices (canonical layout x fastest): 0..0x3F regular row of that class,
 * 0x40|k isoviscous traction-face row, 0xFF interface / boundary row (explicit
 * stencil).  Synchronous. */
stk_status stk_export_classes(stk_ctx* ctx, int32_t level, uint8_t* cls_host, double* emu_host);
stk_status stk_export_codes(stk_ctx* ctx, int32_t level, uint8_t* code_host);
/* Number of kernels this context launched so far (evidence counter). */
int64_t stk_launch_count(const stk_ctx* ctx);

/* Event-timed kernel profile.  on = 1: every op brackets its kernel launches
 * with CUDA events on cfg.stream, except that the V-cycle levels >= 1 run as
 * one captured CUDA graph timed as op 10; on = 2: the graph is bypassed and
 * every launch is timed; on = 0: off.  stk_profile_read sums the records of
 * one op (0 apply, 1 residual, 2 velocity colour pass, 3 pressure pass 1,
 * 4 pressure pass 2, 5 restriction, 6 prolongation, 7 coarse solve,
 * 8 reductions, 9 Krylov vector ops, 10 coarse-level graph, 11 fused
 * coarse V-cycle kernel, 12 list-row passes of the smoother (repeat pass / list rows of
 * the fused sweep), 13 fused forward velocity sweep (both colours)) on one level
 * (-1 = all); synchronises.  STK_EINVAL for on outside 0..2. */
stk_status stk_profile_enable(stk_ctx* ctx, int32_t on);
stk_status stk_profile_reset(stk_ctx* ctx);
stk_status stk_profile_read(stk_ctx* ctx, int32_t op, int32_t level, int64_t* launches, double* ms);

/* Host only (no device needed): the z-slab partition of the level hierarchy that
 * stk_create uses for (nranks, rank).  Writes *nlev and, per level l (finest
 * first), out[8 l .. 8 l + 7] = {n_l, z0, nz_local, cz0, cz1, replicated, K0, K1}:
 * owned vertex planes [z0, z0 + nz_local), stored cube layers [cz0, cz1), whether
 * the level is held whole by every rank, and (for the last distributed level)
 * the planes [K0, K1) of the next, replicated level this rank restricts into
 * (-1 otherwise).  out must hold 8 * 16 int32.  STK_EINVAL on bad sizes. */
stk_status stk_partition(int32_t n, int32_t n_coarse, int32_t nranks, int32_t rank, int32_t* nlev, int32_t* out);

const char* stk_last_error(const stk_ctx* ctx);
stk_status stk_destroy(stk_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* STK_H */
