/*
 * hysco.h — C ABI of libhysco.so, the B200 (sm_100a) hot path of PyHySCO's
 * field-map estimation for reversed-gradient-polarity EPI correction
 * (arXiv 2403.10706; PAPER.md cited as P:<line>, readings R<n> in DESIGN.md).
 *
 * The problem: given two images I+ and I- acquired with opposite
 * phase-encoding (PE) direction +-v, find the field map b minimising
 *
 *   J(b) = D(b) + alpha S(b) + beta P(b)                              Eq.(4)/(6)
 *   D    = 1/2 || I+(x + b v)(1 + d_v b) - I-(x - b v)(1 - d_v b) ||^2   Eq.(1)-(2)
 *   S    = (h1 h2 h3 / 2) b^T L b, L the negative Laplacian             Eq.(5)
 *   P    = 1/2 sum phi(d_v b),  phi(z) = z^4/(1 - z^2) on (-1,1)         Eq.(3)
 *
 * with a 1D optimal-transport initial guess per PE column, a
 * Gauss-Newton / Jacobi-PCG solve and a Jacobian-modulation
 * correction.
 *
 * Layout contract (the PE axis is permuted to be last):
 *   images : C-contiguous [batch][n1][n2][n3]     ("cells")
 *   b, q   : C-contiguous [batch][n1][n2][n3+1]   ("nodes", e3-staggered grid)
 *   element type = the context's dtype (float for HYSCO_F32, double for
 *   HYSCO_F64); b is in mm along +v (R2).  Device pointers must be 16-byte
 *   aligned and must not alias each other unless stated.
 *
 * Streams: every call is ordered on the stream given at hysco_create.  Calls
 * that return host scalars (objective_grad, solve, correct*) synchronise that
 * stream before returning.  A context is not thread-safe; distinct contexts
 * are independent.  Ownership: the caller owns all I/O buffers; images are
 * BORROWED by hysco_bind_images and must stay valid and unmodified until the
 * next bind or destroy; the context owns all scratch (allocated at create,
 * never during a solve).
 *
 * Errors: status codes only, nothing is thrown across the ABI; the message of
 * the last failure is returned by hysco_last_error().  A CUDA error poisons
 * the context (every later call returns HYSCO_ERR_CUDA).  Infeasibility
 * (|d_v b| >= 1 somewhere, phi = +inf) is a state, not an error.
 */
#ifndef HYSCO_H
#define HYSCO_H

#include <stdint.h>

#if defined(__GNUC__)
#define HYSCO_API __attribute__((visibility("default")))
#else
#define HYSCO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hysco_ctx_s* hysco_ctx;

typedef enum {
    HYSCO_OK = 0,
    HYSCO_INFEASIBLE = 1,    /* state: some |Db| >= 1, J = +inf (Eq.(3))       */
    HYSCO_ERR_ARG = -1,      /* NULL / misaligned pointer, bad option value     */
    HYSCO_ERR_SHAPE = -2,    /* bad sizes in hysco_config                       */
    HYSCO_ERR_STATE = -3,    /* e.g. hessvec before a feasible objective_grad   */
    HYSCO_ERR_CUDA = -4,     /* CUDA runtime error (context poisoned)           */
    HYSCO_ERR_NCCL = -5,     /* reserved for the multi-GPU slab path            */
    HYSCO_ERR_NOMEM = -6     /* device allocation failed at create              */
} hysco_status;

typedef enum { HYSCO_F32 = 0, HYSCO_F64 = 1 } hysco_dtype;

/* Problem description.  One context holds `batch` independent pairs of the
 * same shape and voxel size (Table 1 shapes; batched DP). */
typedef struct {
    int64_t n1, n2, n3;      /* cells per pair, PE = n3 (last, contiguous); n3 >= 2, n1,n2 >= 1 */
    int64_t batch;           /* pairs, >= 1                                       */
    double h1, h2, h3;       /* voxel size in mm, > 0                             */
    double alpha, beta;      /* weights of S and P; paper: 300 and 1e-4   */
    int32_t dtype;           /* hysco_dtype                                       */
    int32_t device;          /* CUDA device ordinal                               */
} hysco_config;

/* OT initialisation options. */
typedef struct {
    double eps;              /* positivity shift, fraction of the pair's range (R6); default 1e-3 */
    int32_t blur;            /* 1: 3x3x3 Gaussian, sigma = 1 voxel, periodic (R11)          */
    double feas_cap;         /* if max|Db0| >= feas_cap, scale b0 to feas_cap (R10); default 0.95  */
} hysco_ot_opts;

/* GN-PCG options (R14-R16). */
typedef struct {
    int32_t max_gn;          /* Gauss-Newton iterations (fixed mode: exactly this many)   */
    int32_t max_pcg;         /* PCG iterations per GN step, paper: 10             */
    double pcg_rtol;         /* early stop if ||r||/||r0|| < pcg_rtol, paper: 0.1 */
    int32_t fixed_iters;     /* 1: no early stops (parity / timing), 0: paper stop rules  */
    int32_t ls_max;          /* Armijo halvings, default 10 (R15)                          */
    double armijo_c1;        /* Armijo constant, default 1e-4 (R15)                        */
    double tol_grad_rel;     /* stop if ||grad|| <= tol * ||grad(b0)|| (R16), default 1e-2 */
    double tol_dJ_rel;       /* stop if |J_old - J| <= tol * |J_old| (R16), default 1e-4    */
    double tol_db_rel;       /* stop if max|gamma q| <= tol * h3 (R16), default 1e-3        */
    int32_t armijo;          /* 1 (default): Armijo sufficient decrease (R15);
                                0: accept the full step unless infeasible, halving only for
                                feasibility — the parity mode of DESIGN.md R15, which keeps
                                the accept decision free of fp32-vs-fp64 rounding of J      */
    int32_t precond;         /* HYSCO_PRECOND_JACOBI (default): z = r / diag(H_J);
                                HYSCO_PRECOND_PE_BLOCK: z = B^{-1} r with B the per-PE-column
                                tridiagonal blocks of H_J, the block-diagonal preconditioner
                                named in P:200 (R20).  PE_BLOCK runs the streaming
                                PCG kernels (column-local: slabs need no extra exchange)    */
} hysco_solve_opts;

enum { HYSCO_PRECOND_JACOBI = 0, HYSCO_PRECOND_PE_BLOCK = 1 };

enum { HYSCO_STOP_MAXITER = 0, HYSCO_STOP_GRAD = 1, HYSCO_STOP_DJ = 2, HYSCO_STOP_DB = 3,
       HYSCO_STOP_LSFAIL = 4, HYSCO_STOP_INFEASIBLE = 5 };

/* Per-pair result of a solve (OptimizationLogger analogue; T4 counters P:519). */
typedef struct {
    int32_t gn_iters;        /* accepted GN steps                        */
    int32_t f_evals;         /* objective evaluations incl. the first    */
    int32_t h_evals;         /* Hessian matvecs                          */
    int32_t pcg_iters;       /* total PCG iterations                     */
    int32_t stop_reason;     /* HYSCO_STOP_*                             */
    int32_t ls_halvings;     /* total Armijo halvings                    */
    double J, D, S, P;       /* objective parts at the returned b        */
    double grad_norm;        /* ||grad J|| at the returned b             */
    double last_relres;      /* ||r||/||r0|| of the last PCG solve       */
} hysco_report;

/* Fills the defaults named above (R6, R10, R11, R14-R16). */
HYSCO_API void hysco_default_solve_opts(hysco_solve_opts* o);
HYSCO_API void hysco_default_ot_opts(hysco_ot_opts* o);

/* Create a context: validates cfg, allocates all scratch on cfg->device, and
 * binds `cuda_stream` (a cudaStream_t, not the legacy NULL stream: solves are
 * captured into CUDA graphs; NULL = the context creates and owns a
 * non-blocking stream).  Returns HYSCO_ERR_SHAPE / HYSCO_ERR_ARG for invalid
 * cfg, HYSCO_ERR_NOMEM if the scratch does not fit, *out = NULL on failure. */
HYSCO_API hysco_status hysco_create(const hysco_config* cfg, void* cuda_stream, hysco_ctx* out);

/* Borrow the image pair (device, [batch][n1][n2][n3] of dtype). */
HYSCO_API hysco_status hysco_bind_images(hysco_ctx ctx, const void* d_Iplus, const void* d_Iminus);

/* OT initial field map + optional blur + feasibility guard
 * (R10).  d_b_out: device nodes [batch][n1][n2][n3+1].  opts NULL = defaults. */
HYSCO_API hysco_status hysco_ot_init(hysco_ctx ctx, const hysco_ot_opts* opts, void* d_b_out);

/* Objective at b (Eq.(6)); JDSP (host, [batch][4] = J, D, S, P) and, when
 * non-NULL, the gradient (device nodes).  Also stores the GN-Hessian parts at
 * b for hysco_hessvec / hysco_hess_diag.  Returns HYSCO_INFEASIBLE (J = +inf,
 * grad not written) if any pair is infeasible. */
HYSCO_API hysco_status hysco_objective_grad(hysco_ctx ctx, const void* d_b, double* JDSP, void* d_grad);

/* Hq = H_J q: GN data term + alpha hd L + beta barrier'', at the b
 * of the last successful objective_grad (else HYSCO_ERR_STATE).  d_q, d_Hq:
 * device nodes; must not alias. */
HYSCO_API hysco_status hysco_hessvec(hysco_ctx ctx, const void* d_q, void* d_Hq);

/* diag(H_J), the Jacobi preconditioner, device nodes. */
HYSCO_API hysco_status hysco_hess_diag(hysco_ctx ctx, void* d_diag);

/* Preconditioner solve z = M^{-1} r at the b of the last successful
 * objective_grad (else HYSCO_ERR_STATE): kind = HYSCO_PRECOND_JACOBI (M =
 * diag(H_J)) or HYSCO_PRECOND_PE_BLOCK (M = the per-PE-column
 * tridiagonal blocks of H_J; Thomas algorithm per column).  d_r, d_z:
 * device nodes [batch][n1][n2][n3+1]; must not alias.  Not on slab contexts. */
HYSCO_API hysco_status hysco_precond_solve(hysco_ctx ctx, int kind, const void* d_r, void* d_z);

/* Gauss-Newton with Jacobi-PCG and Armijo from b (in/out, device
 * nodes).  reports: host array [batch] (may be NULL).  The whole solve runs as
 * one CUDA graph with device-side control flow.  Returns HYSCO_INFEASIBLE
 * without iterating if some pair's b is infeasible.  Afterwards the Hessian
 * state is at the final b (hysco_hessvec may follow), except after a batch
 * (batch > 1) solve on the on-chip-resident path, which runs the pairs one
 * after another on shared scratch: call hysco_objective_grad first. */
HYSCO_API hysco_status hysco_solve(hysco_ctx ctx, void* d_b_inout, const hysco_solve_opts* opts,
                         hysco_report* reports);

/* ADMM options (readings R21-R26 in DESIGN.md). */
typedef struct {
    int32_t max_iter;        /* ADMM iterations (fixed mode: exactly this many), default 20        */
    int32_t inner;           /* Gauss-Newton steps per b-update (per column), default 2             */
    int32_t ls_max;          /* Armijo tries per column step, default 10                             */
    int32_t fixed_iters;     /* 1: no convergence stop; 0: stop when b, z, u change < tol   */
    double tol;              /* relative change tolerance, default 1e-3 (R26)                       */
    double rho0;             /* initial augmentation; <= 0: alpha (1/h1^2 + 1/h2^2) (R24)          */
    double mu, tau;          /* residual balancing (Boyd et al. 2011 §3.4.1), default 10, 2 (R25)   */
    double armijo_c1;        /* default 1e-4                                                         */
    double col_tol;          /* a column's GN stops when -grad.q <= col_tol |Fc|, default 1e-6 (R23) */
} hysco_admm_opts;

/* Per-pair ADMM result. */
typedef struct {
    int32_t iters;           /* ADMM iterations run                          */
    int32_t converged;       /* 1: stopped on the change tolerance            */
    double rho;              /* final augmentation parameter                  */
    double r_norm, s_norm;   /* last primal / dual residual norms             */
    double J, D, S, P;       /* objective (Eq.(6), Neumann S) at the returned b */
} hysco_admm_report;

HYSCO_API void hysco_default_admm_opts(hysco_admm_opts* o);

/* ADMM field-map solve from d_b_inout (device nodes; e.g. the OT start):
 * b-update = per-column Gauss-Newton with exact tridiagonal solves and
 * per-column Armijo steps (no communication), z-update = periodic in-plane
 * solve by 2-D FFTs (cuFFT) per PE node slice, u-update, residual balancing
 * of rho and the stop test on the device.  Writes the final b.  reports:
 * [batch] or NULL.  On an NCCL slab context: this rank's part of the slab
 * ADMM (transposed z-update, see hysco_group_admm; every rank calls it with
 * its dense slab); on loopback slab contexts HYSCO_ERR_STATE (use
 * hysco_group_admm). */
HYSCO_API hysco_status hysco_admm(hysco_ctx ctx, void* d_b_inout, const hysco_admm_opts* opts,
                                  hysco_admm_report* reports);

/* Jacobian-modulation correction: the two corrected images
 * T[I+, b, v], T[I-, b, -v] (device cells). */
HYSCO_API hysco_status hysco_apply(hysco_ctx ctx, const void* d_b, void* d_Iplus_corr, void* d_Iminus_corr);

/* Distortion simulation: I+ = A+ T, I- = A- T per PE column, A+-
 * the push-forward matrices of b (R27: true cell k moves to k +- (A b)_k/h3 in
 * index units, its unit mass split between the two nearest distorted cells
 * with hat weights, mass leaving the field of view dropped).  d_b: device
 * nodes; d_T, d_Iplus, d_Iminus: device cells (must not alias).  Synchronises
 * the context stream.  Returns HYSCO_INFEASIBLE if some column has |Db| >= 1
 * (its outputs are then undefined).  Column-local: on a slab context every
 * pointer is the rank's dense slab and no data is exchanged. */
HYSCO_API hysco_status hysco_push_forward(hysco_ctx ctx, const void* d_b, const void* d_T, void* d_Iplus,
                                          void* d_Iminus);

/* Least-squares correction options (R28, R29). */
typedef struct {
    double lambda;           /* weight of ||D1 t||^2 (1-D Neumann, index units), default 0.05 (R29) */
    int32_t max_iter;        /* PCG iterations per column, default 200                              */
    double rtol;             /* stop at ||r|| <= rtol ||rhs||; 0 = 1e-6 (f32) / 1e-12 (f64)          */
} hysco_lsq_opts;

/* Per-pair least-squares report. */
typedef struct {
    int32_t max_iters;       /* most PCG iterations any column used            */
    int64_t unconverged;     /* columns that hit max_iter before rtol           */
    int64_t infeasible;      /* columns with |Db| >= 1 (output set to 0)        */
    double max_relres;       /* largest final ||r|| / ||rhs|| over the columns */
} hysco_lsq_report;

HYSCO_API void hysco_default_lsq_opts(hysco_lsq_opts* o);

/* Least-squares correction (R28): one corrected image t per pair,
 * per PE column the solution of (A+^T A+ + A-^T A- + lambda L1) t =
 * A+^T i+ + A-^T i- for the bound pair (i+, i-) and field map b (device
 * nodes), by Jacobi-PCG per column (one warp each).  d_T_out: device cells
 * [batch][n1][n2][n3].  reports: [batch] or NULL.  Synchronises the context
 * stream.  Returns HYSCO_INFEASIBLE if some column has |Db| >= 1.  Column-
 * local: on a slab context it corrects the rank's dense slab with no exchange
 * and the reports describe the rank's columns. */
HYSCO_API hysco_status hysco_lsq_correct(hysco_ctx ctx, const void* d_b, const hysco_lsq_opts* opts,
                                         void* d_T_out, hysco_lsq_report* reports);

/* The whole path in one call on device buffers: OT init (+blur, guard) ->
 * GN-PCG -> apply.  Any output pointer may be NULL. */
HYSCO_API hysco_status hysco_correct(hysco_ctx ctx, const hysco_ot_opts* ot, const hysco_solve_opts* so,
                           void* d_b_out, void* d_Iplus_corr, void* d_Iminus_corr,
                           hysco_report* reports);

/* Same on HOST buffers (pinned for full speed): copies the pair in, runs the
 * path, copies b and the corrected pair out.  The images are copied into
 * context-owned device memory (re-binding the context to it).  Outputs may be
 * NULL. */
HYSCO_API hysco_status hysco_correct_host(hysco_ctx ctx, const void* h_Iplus, const void* h_Iminus,
                                const hysco_ot_opts* ot, const hysco_solve_opts* so,
                                void* h_b_out, void* h_Iplus_corr, void* h_Iminus_corr,
                                hysco_report* reports);

/* A sequence of n_items independent corrections on HOST buffers (pinned for
 * full speed), pipelined: while item k is corrected on the context stream,
 * item k+1's pair is copied in and item k-1's results are copied out on a
 * second, context-owned copy stream (two device staging slots each way), so
 * the PCIe traffic hides behind the compute.  Item k uses h_Iplus[k],
 * h_Iminus[k] ([batch][n1][n2][n3]) and writes h_b_out[k], h_Iplus_corr[k],
 * h_Iminus_corr[k] (each array of pointers may be NULL, or hold NULL
 * entries, to skip that output).  reports: [n_items][batch] or NULL.
 * Each item's correction reads its pair in place from its input staging
 * slot and writes its results in place to its output slot (the two slots'
 * graphs stay cached), and the host does not synchronise between items: the
 * per-item reports are gathered once at the end.  The context is left bound
 * to the last item's input slot.
 * Returns when every copy has completed; the first failing item's status
 * (errors before HYSCO_INFEASIBLE).  Not on slab contexts. */
HYSCO_API hysco_status hysco_correct_host_stream(hysco_ctx ctx, int32_t n_items, const void* const* h_Iplus,
                                                 const void* const* h_Iminus, const hysco_ot_opts* ot,
                                                 const hysco_solve_opts* so, void* const* h_b_out,
                                                 void* const* h_Iplus_corr, void* const* h_Iminus_corr,
                                                 hysco_report* reports);

/* Per-iteration solver history of the last hysco_solve / hysco_correct (or
 * slab group) call (PyHySCO's OptimizationLogger records the loss
 * terms per iteration).  Record 0 is the Gauss-Newton start (the objective at
 * the initial b, gamma = 0); record k >= 1 is taken when the k-th GN step is
 * accepted: the objective parts at the new b, ||grad J||, the
 * accepted Armijo step gamma, that step's PCG iterations and final relative
 * residual, max |gamma q| (mm), and the cumulative objective evaluations and
 * halvings.  Written on the device by the deciding kernels, no host
 * synchronisation during the solve; at most 64 records (GN steps beyond 63
 * are not recorded).  ADMM solves do not write it.
 * pair: 0 <= pair < batch; out (host) receives min(gn_iters + 1, 64,
 * max_records) records, *n_records their count.  Synchronises the context
 * stream.  HYSCO_ERR_ARG for a bad pair / NULL buffer. */
typedef struct {
    int32_t k;               /* 0: GN start; k: after the k-th accepted step */
    int32_t pcg_iters;       /* PCG iterations of step k (0 for k = 0)       */
    int32_t ls_halvings;     /* Armijo halvings so far                        */
    int32_t f_evals;         /* objective evaluations so far                  */
    double J, D, S, P;       /* objective parts at b_k (Eq.(2)-(6))          */
    double grad_norm;        /* ||grad J(b_k)||                               */
    double gamma;            /* accepted step size (R15)                      */
    double relres;           /* ||r|| / ||r0|| of step k's PCG (R14)          */
    double step_max;         /* max |gamma q| of step k, mm (R16)             */
} hysco_iter_record;
HYSCO_API hysco_status hysco_history(hysco_ctx ctx, int32_t pair, hysco_iter_record* out, int32_t max_records,
                                     int32_t* n_records);

/* Number of kernel launches issued by the last solve / correct call (graph
 * nodes executed, counted on the device). */
HYSCO_API int64_t hysco_last_launch_count(hysco_ctx ctx);

/* Which Jacobi-PCG implementation the context's solves use (fixed at create,
 * DESIGN.md §7): 0 streaming kernels, 1 on-chip-resident PCG over 1-D strips
 * of consecutive PE columns per SM, 2 on-chip-resident PCG over 2-D column
 * tiles, 3 L2-resident persistent PCG; -1 for a NULL context.  tile_out
 * (4 int32, may be NULL) receives (TI, TJ, TH, TW) for path 2 -- TI x TJ
 * tiles of TH x TW columns -- else zeros. */
HYSCO_API int32_t hysco_pcg_path(hysco_ctx ctx, int32_t* tile_out);

/* Profiling hook for the roofline figures: after a solve, re-launches each
 * hot kernel `reps` times on the context stream in the solve's launch
 * configuration and on its buffers, timing each launch with CUDA events.
 * avg_ms (host, [HYSCO_NPROF]) receives the mean launch duration of:
 * [0] matvec (A5, PCG mode), [1] pcg_update (A6), [2] pcg_dir, [3] eval (A4),
 * [4] the on-chip-resident PCG (one launch = one GN step's 10-iteration PCG
 * solve per pair; -1 if this context does not use it), [5] trial_init (A7),
 * [6] the resident PCG's synchronisation floor: a launch of the same grid and
 * shared memory running only its per-iteration dependency chain (p-halo
 * acquire, two tagged all-reduces, p-halo release) for 10 iterations, no
 * arithmetic or data movement (-1 without the resident path), [7] the
 * persistent L2-resident PCG (one launch = one GN step's 10-iteration PCG
 * solve per pair, hysco_l2pcg.cuh; -1 if this context does not use it),
 * [8] pcg_dirmv and [9] pcg_upd: the two launches of a streaming PCG
 * iteration in the flat vectorised form (hysco_flat.cuh: direction + deferred
 * x update + matvec + p.Hp; residual update + preconditioner + r.z, r.r);
 * -1 where this context runs the three-kernel form.  With the flat form [5]
 * times its Armijo start (trial_flat_kernel, which also adds the last
 * direction's deferred x update).
 * flush_l2 != 0: a 256 MiB scratch write (> the 126 MB L2) precedes every
 * timed launch (outside the events), i.e. cold-cache HBM-bound timings.
 * Clobbers the PCG scratch (not b, not the images). */
enum { HYSCO_PROF_MATVEC = 0, HYSCO_PROF_UPDATE = 1, HYSCO_PROF_DIR = 2, HYSCO_PROF_EVAL = 3,
       HYSCO_PROF_RESIDENT = 4, HYSCO_PROF_TRIAL = 5, HYSCO_PROF_RES_SYNC = 6, HYSCO_PROF_L2PCG = 7,
       HYSCO_PROF_DIRMV = 8, HYSCO_PROF_UPD = 9, HYSCO_NPROF = 10 };
HYSCO_API hysco_status hysco_profile_kernels(hysco_ctx ctx, int32_t reps, int32_t flush_l2, double* avg_ms);

/* ---- Multi-GPU slab decomposition along dim 1 (north_star:
 * "Large volumes are partitioned ... as slabs along a non-phase-encoding axis",
 * one-plane halo of the in-plane Laplacian over NCCL, allreduced PCG scalars).
 * A slab context owns global planes [i0, i0 + cfg->n1) of n1_global; its
 * images and node arrays are the rank-local slabs ([batch][cfg->n1][n2][...]).
 * Slab contexts run hysco_solve / hysco_correct / hysco_correct_host (every
 * rank calls them collectively); the other per-kernel calls return
 * HYSCO_ERR_STATE on slab contexts.  Results equal the single-GPU solve up to
 * reduction order. */

/* NCCL unique id (rank 0), to be broadcast to the other ranks by the caller. */
HYSCO_API hysco_status hysco_nccl_unique_id(unsigned char id_out[128]);

/* One rank of an NCCL slab group (one process per GPU).  nranks == 1 needs no id. */
HYSCO_API hysco_status hysco_create_slab(const hysco_config* cfg, int32_t rank, int32_t nranks, int64_t n1_global,
                                         int64_t i0, const unsigned char* nccl_id, void* cuda_stream, hysco_ctx* out);

/* Single-GPU loopback group: cfg describes the WHOLE volume; it is split into
 * nranks contiguous slabs (rank r owns planes [n1 r / nranks, n1 (r+1) / nranks)),
 * out[nranks] receives the contexts (one stream, halo exchange by device copies,
 * allreduce by a fixed-order device sum).  For testing the slab path on one GPU. */
HYSCO_API hysco_status hysco_create_loopback(const hysco_config* cfg, int32_t nranks, void* cuda_stream,
                                             hysco_ctx* out);

/* ADMM (hysco_admm, R21-R26) on slabs.  The b-update is column-local on every
 * rank; the u-update's residual norms are allreduced before the (identical)
 * residual-balancing decision; the z-update -- the periodic in-plane 2-D
 * solve (R22), which the split along dim 1 cuts -- runs after a
 * transpose: rank r receives all n1 planes of its range of PE nodes
 * [r P / N, (r + 1) P / N) (P = n3 + 1 >= N), transforms with cuFFT, scales and
 * returns the planes (strided device copies in a loopback group, NCCL send /
 * receive across processes; hysco_admm on an NCCL slab context runs the same
 * path with its communicator).  ctxs: a loopback group in rank order;
 * d_b_inout[r]: rank r's dense slab of nodes [batch][n1_r][n2][n3+1] (device,
 * overwritten).  Reports as hysco_admm (J of the whole volume).  Equal to the
 * single-context ADMM up to FFT summation order. */
HYSCO_API hysco_status hysco_group_admm(hysco_ctx* ctxs, int32_t nranks, void* const* d_b_inout,
                                        const hysco_admm_opts* opts, hysco_admm_report* reports);

/* Run a loopback group (all ranks, in rank order); per-rank device pointers. */
HYSCO_API hysco_status hysco_group_correct(hysco_ctx* ctxs, int32_t nranks, const hysco_ot_opts* ot,
                                           const hysco_solve_opts* so, void* const* d_b_out,
                                           void* const* d_Iplus_corr, void* const* d_Iminus_corr,
                                           hysco_report* reports);
HYSCO_API hysco_status hysco_group_solve(hysco_ctx* ctxs, int32_t nranks, void* const* d_b_inout,
                                         const hysco_solve_opts* so, hysco_report* reports);

HYSCO_API const char* hysco_last_error(hysco_ctx ctx);
HYSCO_API hysco_status hysco_destroy(hysco_ctx ctx);
HYSCO_API int32_t hysco_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HYSCO_H */
