/*
 * cavac_b200.h -- C ABI of the B200-native complex-FP64 Krylov / Schwarz
 * Helmholtz solver (libcavac_b200.so).
 *
 * Plain pointers and sizes only.  Complex arrays are interleaved (re, im)
 * doubles -- the layout of std::complex<double> / CVector, so a reference
 * caller passes values.data() / b.data() straight through.  Index arrays are
 * uint64 like the reference's std::size_t (numkit.hpp:34-35); they are
 * narrowed to int32 on upload with an overflow check.
 *
 * Every entry point returns CVK_OK (0) or a negative CVK_E* code; the message
 * is available from cvk_last_error() (thread-local).  Non-convergence and
 * Krylov breakdowns are NOT errors: they are reported in cvk_report, as the
 * reference reports them in SolveReport (krylov.hpp:25-33).
 *
 * Reference interfaces each entry point replaces (paths relative to the
 * reference tree proj/core/):
 *   cvk_csr_upload        CsrMatrix (include/cavac/numkit.hpp:31-40)
 *   cvk_precond_jacobi    jacobi (src/krylov.cpp:31-55)
 *   cvk_precond_identity  identity_preconditioner (src/krylov.cpp:27-29)
 *   cvk_solve             solve / bicgstab / bicgstab_l / tfqmr
 *                         (include/cavac/krylov.hpp:50-69, src/krylov.cpp:57-403)
 *   cvk_spmv              spmv (src/numkit.cpp:88-111)
 *   cvk_dot, cvk_norm2    dot_hermitian, norm2 (src/numkit.cpp:113-125)
 *   cvk_axpy, cvk_xpay    axpy_inplace, xpay_inplace (src/numkit.cpp:135-159)
 *   cvk_true_relres       true_relative_residual (src/krylov.cpp:17-23)
 *   cvk_set_exec_mode     set_exec_mode (src/numkit.cpp:29-30)
 *   cvk_schwarz_solve     schwarz_solve (include/cavac/schwarz.hpp:54-58,
 *                         src/schwarz.cpp:111-238)
 *   cvk_csr_assemble_cavity  assemble (src/helmholtz.cpp:59-115) values at a
 *                         new omega, evaluated on the device for frequency
 *                         sweeps (driver pattern: bench_solvers,
 *                         src/pipeline.cpp:227-293)
 *   cvk_precond_jacobi_refresh  jacobi (src/krylov.cpp:31-55) on new values
 *   cvk_rowblock_*        bicgstab (src/krylov.cpp:57-138) with the rows split
 *                         over ranks / GPUs (no reference counterpart: its
 *                         solve runs in one address space, krylov.hpp:68-69)
 */
#ifndef CAVAC_B200_H
#define CAVAC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CVK_ABI_VERSION 2

/* status codes */
#define CVK_OK 0
#define CVK_EINVAL -1      /* std::invalid_argument in the reference */
#define CVK_ECUDA -2       /* CUDA runtime / launch failure */
#define CVK_ENOMEM -3      /* device allocation failed */
#define CVK_EOVERFLOW -4   /* index does not fit the device's int32 layout */
#define CVK_EZERODIAG -5   /* jacobi: zero diagonal at row i (invalid_argument) */
#define CVK_ESOLVER -6     /* unknown solver id (invalid_argument) */
#define CVK_ELOGIC -7      /* std::logic_error in the reference */
#define CVK_ETIMEOUT -8    /* device grid barrier timed out (never expected) */

/* solver ids: the reference's SolverId order (krylov.hpp:63) + GMRES, COCG */
#define CVK_BICGSTAB 0
#define CVK_BICGSTAB_L 1
#define CVK_TFQMR 2
#define CVK_GMRES 3 /* beyond reference: restarted GMRES(m) */
#define CVK_COCG 4  /* beyond reference: conjugate orthogonal CG for the
                       complex-symmetric operator (oracle orc_cocg) */

/* arithmetic modes */
#define CVK_MODE_FAST 0     /* double-double reductions, streamed SpMV (the product) */
#define CVK_MODE_REF 1      /* reference order: row-sequential SpMV and sequential
                               dots, each dot summed by one thread in element order
                               (ExecMode::Sequential); bitwise the reference CPU code */
#define CVK_MODE_REF_PAR 2  /* the same sums in the same order (bitwise CVK_MODE_REF),
                               with the element terms formed by all threads of a CTA
                               and one thread running only the dependent adds
                               (ExecMode::Parallel, numkit.hpp:14-18) */

/* breakdown codes (SolveReport.breakdown strings, krylov.cpp) */
#define CVK_BRK_NONE 0
#define CVK_BRK_RHO 1        /* "rho breakdown" */
#define CVK_BRK_SHADOW_V 2   /* "stagnation in <shadow, v>" */
#define CVK_BRK_OMEGA 3      /* "omega breakdown" */
#define CVK_BRK_SHADOW_U 4   /* "stagnation in <shadow, u>" */
#define CVK_BRK_MR 5         /* "degenerate least-squares in MR step" */
#define CVK_BRK_SIGMA 6      /* "sigma breakdown" */
#define CVK_BRK_ARNOLDI 7    /* "arnoldi breakdown" (GMRES) */
#define CVK_BRK_PAP 8        /* "stagnation in <p, A p>" (COCG) */

typedef struct cvk_ctx cvk_ctx;
typedef struct cvk_csr cvk_csr;
typedef struct cvk_prec cvk_prec;

/* SolverOptions (krylov.hpp:13-18) + GMRES restart length m + arithmetic mode */
typedef struct {
    double tol;            /* default 1e-9 */
    int64_t max_iter;      /* default 10000 */
    int64_t l;             /* BiCGSTAB(l) degree, default 8 */
    int64_t m;             /* GMRES restart, default 30 (beyond reference) */
    int32_t record_history;
    int32_t mode;          /* CVK_MODE_FAST / CVK_MODE_REF / CVK_MODE_REF_PAR (< 0: ctx ExecMode) */
    int32_t warm;          /* Schwarz inner BiCGSTAB solves start from the previous sweep's
                              solution (beyond the reference, cvk_schwarz_solve / cvk_ddm_rank_create) */
    int32_t reserved;
} cvk_opts;

/* SolveReport (krylov.hpp:25-33).  history is caller-owned (may be NULL);
 * history_len is the number of entries the solver produced (it may exceed
 * history_cap, in which case only the first history_cap were stored). */
typedef struct {
    int32_t converged;
    int32_t breakdown;     /* CVK_BRK_* */
    int64_t iterations;
    double final_relres;   /* preconditioned, as recurred by the solver */
    double true_relres;    /* ||b - Ax|| / ||b|| recomputed on the device */
    double wall_time_s;    /* host wall time of the call */
    double *history;
    int64_t history_cap;
    int64_t history_len;
    double device_time_s;  /* CUDA-event time of the solve kernel(s) */
    int64_t kernel_launches;
} cvk_report;

/* ---- version / errors ---- */
int cvk_abi_version(void);
const char *cvk_last_error(void);
const char *cvk_breakdown_name(int code);
const char *cvk_solver_name(int solver);
int cvk_solver_from_name(const char *name); /* >= 0 id, or CVK_ESOLVER */

/* ---- context: one device, one stream ---- */
int cvk_ctx_create(int device, cvk_ctx **out);
int cvk_ctx_destroy(cvk_ctx *ctx);
/* the stream all work of this context is issued on (a cudaStream_t) */
void *cvk_ctx_stream(cvk_ctx *ctx);
/* ExecMode (numkit.hpp:14-21): 0 Sequential -> CVK_MODE_REF, 1 Parallel ->
 * CVK_MODE_REF_PAR.  Both give the reference's iterates bit for bit, as the
 * reference promises for its two modes.  Used when cvk_opts.mode < 0 and by
 * the kernel calls with mode < 0; FAST is always an explicit choice. */
int cvk_set_exec_mode(cvk_ctx *ctx, int parallel);
int cvk_get_exec_mode(cvk_ctx *ctx);

/* Execution-path options of a context (measurement and path-parity tests;
 * the defaults are the tuned product choices).  Unknown key -> CVK_EINVAL. */
#define CVK_OPT_PHASED_MIN_N 1     /* rows from which BiCGSTAB / tfQMR / BiCGSTAB(l) run as
                                      phase kernels instead of one persistent kernel (131072) */
#define CVK_OPT_MAX_CTAS 2         /* cap on the persistent / thread-per-row grid, 0 = none */
#define CVK_OPT_STREAM 3           /* 1: TMA-streamed SpMV phases (default), 0: thread-per-row */
#define CVK_OPT_STREAM_FLAVOR 4    /* 0 auto, 2: 2 x 224-row consumer groups, 4: 4 x 128 */
#define CVK_OPT_SPMV_GROUP 5       /* lanes per row of the thread-per-row FAST SpMV, 0 auto
                                      (read at cvk_csr_upload) */
#define CVK_OPT_GMRES_PERSISTENT 6 /* 1: GMRES in one persistent kernel at any size */
#define CVK_OPT_BICGL_PERSISTENT 7 /* 1: BiCGSTAB(l) in one persistent kernel at any size */
#define CVK_OPT_ILU_HOSTLOOP 8     /* 1: ILU(0) BiCGSTAB as a host loop with scalar read-backs */
#define CVK_OPT_DDM_SEQ_MIN 9      /* strip rows from which Schwarz inner solves run one after
                                      another on the single-system path (131072) */
#define CVK_OPT_RB_STREAM_MIN 10   /* own rows from which row-block phases are streamed */
#define CVK_OPT_BICG_FOLD 11       /* 1: streamed BiCGSTAB and COCG fold each reduction in the consuming
                                      kernel (default); 0: in the producer's last CTA */
#define CVK_OPT_GMRES_TILES 12     /* 1: GMRES basis passes on bulk-copied row tiles (default,
                                      m <= 32); 0: element-loop kernels */
#define CVK_OPT_UNIFORM_OFFDIAG 13 /* 1: streamed SpMVs check each solve's matrix for off-diagonal
                                      values that are all bitwise equal (constant-coefficient
                                      stencils) and then stream only the diagonal; 0: off (default:
                                      the phases are consumer-bound, the bytes saved buy ~2.5%).
                                      Takes effect in builds with -DCVK_UNIFORM_OFFDIAG only */
int cvk_ctx_set_option(cvk_ctx *ctx, int key, int64_t value);
int cvk_ctx_get_option(cvk_ctx *ctx, int key, int64_t *value);

/* ---- matrix ---- */
int cvk_csr_upload(cvk_ctx *ctx, int64_t nrows, int64_t ncols, int64_t nnz,
                   const uint64_t *row_offsets, const uint64_t *col_indices,
                   const double *values, cvk_csr **out);
/* replace the values on the same sparsity pattern (frequency sweeps) */
int cvk_csr_set_values(cvk_csr *A, const double *values);
/* copy the device values back (nnz complex) */
int cvk_csr_get_values(const cvk_csr *A, double *values);
int cvk_csr_free(cvk_csr *A);
int64_t cvk_csr_nrows(const cvk_csr *A);
int64_t cvk_csr_nnz(const cvk_csr *A);

/* ---- preconditioners ---- */
/* inv_diag (host, n complex) may be NULL: the inverse diagonal is then
 * computed on the device with the reference's __divdc3 rounding. */
int cvk_precond_jacobi(cvk_csr *A, const double *inv_diag, cvk_prec **out);
int cvk_precond_identity(cvk_ctx *ctx, int64_t n, cvk_prec **out);
int cvk_precond_free(cvk_prec *M);
/* copy the device inverse diagonal back (n complex) */
int cvk_precond_get_diag(const cvk_prec *M, double *inv_diag);
/* ILU(0) (beyond the reference: it has only jacobi / identity,
 * src/krylov.cpp:27-55).  Exact ILU(0) factor on A's pattern (IKJ, host),
 * applied on the device by `sweeps` (>= 0) Jacobi sweeps per triangle.
 * Zero or missing pivot -> CVK_EZERODIAG.  Solves with an ILU(0) M support
 * CVK_BICGSTAB only (the reference's operation order, host-driven loop of
 * device kernels); other solvers return CVK_EINVAL. */
int cvk_precond_ilu0(cvk_csr *A, int sweeps, cvk_prec **out);
/* copy the factor back: L (strict lower) and U (diagonal and above) in A's
 * value slots (nnz complex) */
int cvk_precond_get_ilu0(const cvk_prec *M, double *factor);
/* z_dev = M^-1 r_dev on ctx's stream (any preconditioner kind; device
 * pointers, n complex each, must not alias) */
int cvk_precond_apply_device(const cvk_prec *M, const double *r_dev, double *z_dev);
/* the same with host r / z (staged through ctx's buffers) */
int cvk_precond_apply(const cvk_prec *M, const double *r, double *z);

/* ---- solve ---- */
/* host b / x (x is overwritten; x0 = 0 as in the reference) */
int cvk_solve(cvk_ctx *ctx, int solver, const cvk_csr *A, const cvk_prec *M,
              const cvk_opts *opts, const double *b, double *x, cvk_report *rep);
/* device-resident b / x (pointers into device memory of ctx's device) */
int cvk_solve_device(cvk_ctx *ctx, int solver, const cvk_csr *A, const cvk_prec *M,
                     const cvk_opts *opts, const double *b_dev, double *x_dev,
                     cvk_report *rep);

/* BiCGSTAB from the x0 in x_dev (beyond the reference, whose solvers start
 * from 0): r0 = M^-1 (b - A x0); relative residuals stay measured against
 * ||M^-1 b||.  Used for warm-started Schwarz inner solves. */
int cvk_solve_device_warm(cvk_ctx *ctx, const cvk_csr *A, const cvk_prec *M, const cvk_opts *opts,
                          const double *b_dev, double *x_dev, cvk_report *rep);

/* ---- kernels (parity tests; mode = CVK_MODE_*) ---- */
int cvk_spmv(const cvk_csr *A, const double *x, double *y, int mode);
int cvk_spmv_device(const cvk_csr *A, const double *x_dev, double *y_dev, int mode);
int cvk_dot(cvk_ctx *ctx, int64_t n, const double *x, const double *y, double *out, int mode);
int cvk_norm2(cvk_ctx *ctx, int64_t n, const double *x, double *out, int mode);
int cvk_axpy(cvk_ctx *ctx, int64_t n, const double *alpha, const double *x, double *y);
int cvk_xpay(cvk_ctx *ctx, int64_t n, const double *alpha, double *x, const double *y);
int cvk_true_relres(const cvk_csr *A, const double *b, const double *x, double *out, int mode);

/* ---- Schwarz domain decomposition (schwarz.hpp:16-58) ---- */

/* CavityGrid (helmholtz.hpp:18-39): interior nodes, node = iy * nx + ix */
typedef struct {
    double width, height, h;
    int64_t nx, ny, roof_begin, roof_end;
    double admittance_re, admittance_im;
} cvk_grid;

/* DdmReport (schwarz.hpp:35-40) */
typedef struct {
    int64_t outer_iterations;
    int32_t converged;
    int32_t inner_breakdown;
    double *jump_history;        /* caller-owned, may be NULL */
    int64_t jump_cap;
    int64_t jump_len;
    cvk_report *sub_reports;     /* last sweep's per-subdomain reports (caller-owned) */
    int64_t n_sub_reports;
    int64_t total_inner_iterations; /* last sweep, summed over subdomains */
    double device_time_s;
    double wall_time_s;
    int64_t kernel_launches;
} cvk_ddm_report;

/* partition (schwarz.cpp:93-109): col_begin receives n_sub + 1 entries */
int cvk_partition(int64_t nx, int64_t n_sub, int64_t *col_begin);

/* schwarz_solve (schwarz.cpp:111-238) on one device: host system (the
 * reference's HelmholtzProblem A, b on `grid`), strips col_begin[n_sub+1],
 * Robin coefficients s_left / s_right (complex, 2 doubles each); the inner
 * solves of all strips run batched in one cooperative launch per sweep.
 * inner->mode selects REF (bitwise reference) or FAST arithmetic. */
int cvk_schwarz_solve(cvk_ctx *ctx, const cvk_grid *grid, double c, int64_t n, int64_t nnz,
                      const uint64_t *row_offsets, const uint64_t *col_indices,
                      const double *values, const double *b, int64_t n_sub,
                      const int64_t *col_begin, const double *s_left, const double *s_right,
                      const cvk_opts *inner, double ddm_tol, int64_t max_outer, int inner_solver,
                      double *x, cvk_ddm_report *rep);

/* ---- multi-GPU Schwarz: one rank's strips (schwarz.cpp:111-238 split
 * across devices; the caller moves the interface data between ranks) ----
 *
 * A rank owns global strips [s_begin, s_end) of the n_sub-strip partition
 * col_begin.  Interface slot j = 0..ns (ns = s_end - s_begin) is the cut
 * between global strips s_begin+j-1 and s_begin+j; slot 0 / slot ns are the
 * rank's external cuts (present iff s_begin > 0 / s_end < n_sub).  One call
 * of cvk_ddm_rank_sweep is one outer sweep of the reference for these
 * strips: local rhs with the current interface data, every local inner solve
 * (one batched launch), the Robin trace update on internal cuts, and for the
 * external cuts the local side's new data, returned for the neighbour:
 *   g_out_left  (ny complex): the new g_l of slot 0 (left neighbour's right
 *               edge data), computed from this rank's left edge column;
 *   g_out_right (ny complex): the new g_r of slot ns.
 * The data received from the neighbours is passed to the next sweep as
 * g_in_left (new g_r of slot 0) / g_in_right (new g_l of slot ns); NULL
 * keeps the current values (zero initially).  jump_terms receives
 * 2*(ns+1)*ny doubles [slot][row][side]: |x_new - x_old|^2 of the cut's left
 * column (side 0) and right column (side 1) where that column is local,
 * 0 otherwise -- the caller sums them over all ranks in the reference's
 * order (per cut, per row, left then right, schwarz.cpp:211-220), so the
 * multi-rank interface norm is bitwise the single-process one. */
typedef struct cvk_ddm_rank cvk_ddm_rank;
typedef struct {
    int32_t inner_breakdown;        /* any local inner solve broke down */
    int32_t pad;
    int64_t total_inner_iterations; /* summed over the rank's strips */
    double device_time_s;
    int64_t kernel_launches;
} cvk_ddm_sweep_info;

int cvk_ddm_rank_create(cvk_ctx *ctx, const cvk_grid *grid, double c, int64_t n, int64_t nnz,
                        const uint64_t *row_offsets, const uint64_t *col_indices, const double *values,
                        const double *b, int64_t n_sub, const int64_t *col_begin, int64_t s_begin,
                        int64_t s_end, const double *s_left, const double *s_right, const cvk_opts *inner,
                        int inner_solver, cvk_ddm_rank **out);
int cvk_ddm_rank_sweep(cvk_ddm_rank *rank, const double *g_in_left, const double *g_in_right,
                       double *g_out_left, double *g_out_right, double *jump_terms,
                       cvk_ddm_sweep_info *info);
/* the last sweep's per-strip inner reports (cap entries) */
int cvk_ddm_rank_reports(const cvk_ddm_rank *rank, cvk_report *reps, int64_t cap);
/* the rank's columns col_begin[s_begin] .. col_begin[s_end]-1 of x, row-major
 * (ny rows x width complex) */
int cvk_ddm_rank_solution(cvk_ddm_rank *rank, double *x_cols);
/* the interface traces g_l, g_r of every slot ((n_strips + 1) x ny complex
 * each, slot j = the cut left of local strip j): get / overwrite the state of
 * the outer iteration (Krylov acceleration, paper_2112_00087_b200/ddm_krylov.py) */
int cvk_ddm_rank_get_traces(cvk_ddm_rank *rank, double *g_l, double *g_r);
int cvk_ddm_rank_set_traces(cvk_ddm_rank *rank, const double *g_l, const double *g_r);
/* warm-started inner solves (beyond the reference; BiCGSTAB inner solver):
 * each strip's solve starts from its previous-sweep solution.  The initial
 * value is inner->warm of cvk_ddm_rank_create / cvk_schwarz_solve. */
int cvk_ddm_rank_set_warm(cvk_ddm_rank *rank, int warm);
int cvk_ddm_rank_destroy(cvk_ddm_rank *rank);

/* ---- Schwarz DDM on algebraic subdomains (FEM meshes, METIS-style / RCB
 * partitions; beyond the reference, whose schwarz_solve knows only the FD
 * cavity's strips, schwarz.cpp:29-89) ----
 *
 * part_of_row[i] in [0, n_parts) assigns row i to a subdomain; each
 * subdomain works on its rows grown by `overlap` layers of A's graph, with
 * every coupling that leaves that set folded into the diagonal by the
 * reference's Robin factor (1/h - s/2) / (1/h + s/2) (schwarz.cpp:43-50,
 * s = s_robin complex, h the mesh size).  The preconditioner is restricted
 * additive Schwarz: each subdomain solves its local system (inner solver and
 * options as the reference's inner solves, schwarz.cpp:177) and writes back
 * its owned rows.  cvk_asm_solve: m = 0 iterates the fixed point
 * u <- u + M^-1 (b - A u) (the reference's additive sweep); m > 0 runs
 * FGMRES(m) right-preconditioned by M^-1.  Both stop at ||b - A u|| <= tol
 * ||b||, whose solution is the monodomain one.  Report: outer_iterations =
 * subdomain sweeps, jump_history = relative residuals, total_inner_iterations
 * = the last sweep's inner iterations. */
typedef struct cvk_asm cvk_asm;
int cvk_asm_create(cvk_ctx *ctx, int64_t n, int64_t nnz, const uint64_t *row_offsets,
                   const uint64_t *col_indices, const double *values, int64_t n_parts,
                   const int64_t *part_of_row, int64_t overlap, const double *s_robin, double h,
                   const cvk_opts *inner, int inner_solver, cvk_asm **out);
/* z = M^-1 r, device vectors of length n on ctx's device */
int cvk_asm_apply_device(cvk_asm *S, const double *r_dev, double *z_dev);
int cvk_asm_solve(cvk_asm *S, const double *b, double *x, double tol, int64_t max_outer, int64_t m,
                  cvk_ddm_report *rep);
int64_t cvk_asm_n_parts(const cvk_asm *S);
int cvk_asm_destroy(cvk_asm *S);
/* Several ranks (one device each, north_star's "one or more subdomains per
 * GPU"): rank r of n_ranks builds and solves the subdomains q with
 * q % n_ranks == r; the outer loop runs on every rank.  After its local
 * solves a rank holds M^-1 r on its subdomains' owned rows and zero
 * elsewhere; the reducer must sum z_dev (n complex, device memory of the
 * rank's device; with buf_dev non-null the library stages z through that
 * caller-owned buffer, e.g. a framework tensor) over all ranks, complete
 * before it returns, and sum meta[0] (inner iterations) and max meta[1]
 * (breakdown flag) -- an all-reduce.  Returns 0 on success.  The sum has one nonzero term per entry,
 * so results are bitwise those of one rank. */
typedef int (*cvk_asm_reduce_fn)(void *user, double *z_dev, int64_t n, int64_t *meta);
int cvk_asm_create_rank(cvk_ctx *ctx, int64_t n, int64_t nnz, const uint64_t *row_offsets,
                        const uint64_t *col_indices, const double *values, int64_t n_parts,
                        const int64_t *part_of_row, int64_t overlap, const double *s_robin, double h,
                        const cvk_opts *inner, int inner_solver, int rank, int n_ranks, cvk_asm **out);
int cvk_asm_set_reducer(cvk_asm *S, cvk_asm_reduce_fn fn, void *user, double *buf_dev);

/* ---- frequency sweeps (beyond the reference's single-omega assemble) ---- */

/* Overwrite A's values with the cavity operator at `omega` (assemble,
 * helmholtz.cpp:59-115): off-diagonals -c^2/h^2, diagonal 4c^2/h^2 - omega^2
 * minus (c^2/h^2) w per missing wall neighbour, w = 1/(1 + i omega h beta)
 * (beta = grid admittance; w = 1 for rigid walls), bitwise the reference's
 * values.  A must carry the cavity's 5-point pattern (as uploaded from an
 * assemble() of the same grid); otherwise CVK_EINVAL names the first
 * mismatching row.  The rhs does not depend on omega. */
int cvk_csr_assemble_cavity(cvk_csr *A, const cvk_grid *grid, double omega, double c);
/* recompute M's inverse diagonal from A's current values (jacobi,
 * krylov.cpp:31-55; CVK_EZERODIAG names the row as the reference does) */
int cvk_precond_jacobi_refresh(cvk_prec *M, const cvk_csr *A);

/* FEM operator (beyond the reference's FD cavity; synthetic P1 cavity in
 * paper_2112_00087_b200/fem3d.py): real K, M, C on A's pattern, resident on
 * A's device; cvk_fem_set_omega writes A = K - omega^2 M + i omega C
 * (re = K - (omega*omega) M, im = omega C). */
typedef struct cvk_fem cvk_fem;
int cvk_fem_create(cvk_csr *A, const double *K, const double *M, const double *C, cvk_fem **out);
int cvk_fem_set_omega(cvk_fem *op, double omega);
int cvk_fem_free(cvk_fem *op);

/* ---- row-block global Krylov (SURVEY.md 8(e) mode 1; beyond the reference,
 * whose solve() runs on one address space, krylov.hpp:68-69) ----
 *
 * One rank's contiguous block of rows of the global system.  Local columns
 * are [0, n_own) for own rows and n_own + h for halo entry h (a row of
 * another rank).  Every reduction phase of BiCGSTAB (krylov.cpp:57-138) is
 *   cvk_rowblock_local(ph)  -- the phase's rows; the rank's double-double
 *                              partial sums and the boundary values other
 *                              ranks read go to the rank's exchange slot;
 *   all-gather              -- of every rank's slot into `recv` (caller:
 *                              NCCL over NVLink, gloo, or
 *                              cvk_rowblock_exchange_local for blocks that
 *                              share one device);
 *   cvk_rowblock_post(ph)   -- fold the ranks' partials in rank order, run
 *                              the scalar recurrence, unpack the halo.
 * The reductions are double-double, so iterates are bitwise those of a
 * single-device FAST solve for any number of blocks. */
#define CVK_RB_INIT 0 /* r = M^-1 b, shadow, x = 0; ||r||, <r,r>; r halo */
#define CVK_RB_A 1    /* p, v = M^-1 A p, <shadow, v>; p, v halo */
#define CVK_RB_B 2    /* s, t = M^-1 A s, x += alpha p; ||s||, <t,t>, <t,s> */
#define CVK_RB_C 3    /* x += omega s, r = s - omega t; ||r||, <shadow, r>; r halo */
#define CVK_RB_X 4    /* x halo (before the true residual) */
#define CVK_RB_T 5    /* ||b||, ||b - A x|| -> report */
typedef struct cvk_rowblock cvk_rowblock;
typedef struct {
    int64_t n_own, n_halo, nnz;
    const int64_t *row_offsets; /* n_own + 1, from 0 */
    const int64_t *col_local;   /* nnz, each in [0, n_own + n_halo) */
    const double *values;       /* 2 nnz, interleaved complex */
    const double *inv_diag;     /* 2 n_own (jacobi of the global matrix), NULL = identity */
    const double *b;            /* 2 n_own */
    int64_t n_send;             /* own rows other ranks read */
    const int64_t *send_rows;   /* n_send local rows, in exchange order */
    int64_t n_ranks, max_send;  /* max_send = largest n_send over all ranks */
    const int64_t *halo_src;    /* n_halo: src_rank * max_send + position in src's send list */
    int64_t history_cap;
} cvk_rowblock_desc;
int cvk_rowblock_create(cvk_ctx *ctx, const cvk_rowblock_desc *desc, int solver, const cvk_opts *opts,
                        cvk_rowblock **out);
/* device exchange buffers: send = this rank's slot (slot_doubles), recv =
 * n_ranks slots, slot q at recv + q * slot_doubles */
int cvk_rowblock_exchange(cvk_rowblock *rb, double **send_dev, double **recv_dev, int64_t *slot_doubles);
int cvk_rowblock_local(cvk_rowblock *rb, int phase);
int cvk_rowblock_post(cvk_rowblock *rb, int phase);
/* all-gather for n blocks on one device (stream-ordered device copies) */
int cvk_rowblock_exchange_local(cvk_rowblock *const *rbs, int n);
/* whole solve for n blocks on one device: the phase loop with lazy polling */
int cvk_rowblock_solve_local(cvk_rowblock *const *rbs, int n);
/* whole solve for one block per process over NCCL (the same phase loop,
 * ncclAllGather on the context's stream, captured in CUDA graphs).  Rank 0
 * makes the id (NCCL_UNIQUE_ID_BYTES = 128 bytes) and the caller broadcasts
 * it; every rank attaches with its plan rank.  libnccl.so.2 is resolved at
 * run time. */
int cvk_nccl_unique_id(char *id);
int cvk_rowblock_attach_nccl(cvk_rowblock *rb, const char *id, int rank);
int cvk_rowblock_solve_nccl(cvk_rowblock *rb);
/* peer-to-peer exchange without a collective library: each rank's pack
 * kernel writes its slot into every rank's mailbox (NVLink stores through
 * CUDA IPC mappings) and raises its flag there; the post kernel waits on its
 * local flags (20 s without progress -> CVK_ETIMEOUT).  The handle is a
 * cudaIpcMemHandle_t (64 bytes); `handles` holds all ranks' in rank order.
 * _attach_local wires n blocks of one process together (same device). */
int cvk_rowblock_p2p_handle(cvk_rowblock *rb, void *handle);
int cvk_rowblock_p2p_attach(cvk_rowblock *rb, const void *handles, int rank);
int cvk_rowblock_p2p_attach_local(cvk_rowblock *const *rbs, int n);
/* the phase loop of p2p-attached blocks sharing one stream (one block per
 * process on a multi-GPU node, or n blocks on one device) */
int cvk_rowblock_solve_p2p(cvk_rowblock *const *rbs, int n);
/* synchronises; *done = the solver's stop flag */
int cvk_rowblock_done(cvk_rowblock *rb, int *done);
/* after CVK_RB_X and CVK_RB_T: own rows of x (2 n_own doubles) and the report */
int cvk_rowblock_result(cvk_rowblock *rb, double *x_own, cvk_report *rep);
int cvk_rowblock_destroy(cvk_rowblock *rb);

/* ---- Matrix Market I/O at scale (host; read_matrix_market /
 * write_matrix_market, mmio.cpp:10-63, + csr_from_triplets, numkit.cpp:41-75).
 * The reader parses with nthreads threads (<= 0: all cores) and returns the
 * CSR the reference builds (duplicates summed in input order, columns
 * sorted); arrays are malloc'd, release them with cvk_mm_free.  The writer
 * prints "%.17g" values, byte-identical to the reference's writer. ---- */
typedef struct {
    int64_t nrows, ncols, nnz;
    uint64_t *row_offsets; /* nrows + 1 */
    uint64_t *col_indices; /* nnz, 0-based */
    double *values;        /* 2 nnz, interleaved complex */
} cvk_mm_matrix;
int cvk_mm_read(const char *path, int nthreads, cvk_mm_matrix *out);
void cvk_mm_free(cvk_mm_matrix *m);
int cvk_mm_write(const char *path, const cvk_mm_matrix *m, int nthreads);

/* ---- SpMV timing helper for the bench: `reps` back-to-back launches on
 * device buffers, returns the average kernel time in seconds ---- */
int cvk_spmv_bench(const cvk_csr *A, const double *x_dev, double *y_dev, int mode,
                   int reps, double *avg_s);

#ifdef __cplusplus
}
#endif

#endif /* CAVAC_B200_H */
