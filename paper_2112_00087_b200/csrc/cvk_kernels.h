// cvk_kernels.h -- internal interface between the C ABI (cvk_api.cu) and the
// kernel translation units.  Not installed; the public surface is
// include/cavac_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <string>

// shared error channel of the C ABI (cvk_last_error); returns code
int cvk_fail(int code, const std::string& msg);
// a context's execution-path option (CVK_OPT_*, cvk_ctx_set_option)
struct cvk_ctx;
long long cvk_ctx_knob(cvk_ctx* c, int key);

namespace cvk {

constexpr int kMaxL = 16;     // BiCGSTAB(l): l <= kMaxL

struct Csr;
struct DevReport;

// persistent solver kernels (cvk_krylov.cu)
// batched: k_solve_batched(const KArgs* segs, int nseg) instead of k_solve(KArgs)
const void* solver_kernel(int solver, int S, bool ref, bool batched = false);
int solver_nwork(int solver, int l, int m);
size_t solver_smem(int solver, int m);

// phase-kernel GMRES(m) (cvk_gmres.cu), kThreads threads per CTA
struct GmresKernels {
    const void *init, *x, *spmv, *dd, *up, *true_res;
    const void* spmv_s;  // streamed Arnoldi SpMV: kStreamThreads threads, dynamic smem
    // the basis passes on bulk-copied row tiles, (GArgs, int smem_bytes), m <= 32
    const void *dd_s, *up_s;
};
constexpr int kGmresDdsThreads = 512 + 32, kGmresUpsThreads = 128 + 32;
constexpr int kGmresTileRows = 128;
GmresKernels gmres_kernels();
size_t gmres_state_size();
size_t gmres_args_size();
void gmres_init_state(void* host_state, double tol, long long max_iter, int m, int record, long long hist_cap);
int gmres_state_done_offset();
void gmres_pack_args(void* out, const Csr& A, const double2* dinv, const double2* b, double2* x, double2* work,
                     double2* part, void* st, double* hist, DevReport* rep, int capk, int nst, int pf_rows, int m);
// work vectors of the phase kernels are padded to whole 128-row basis blocks
long long gmres_padded_rows(long long n);
int gmres_tile_stage_max(int m);  // bytes of the largest tile stage, j < m

// phase-kernel BiCGSTAB(l) (cvk_bicgl.cu): one kernel per phase type; the
// right-looking MGS kernel (mgsr) serves l <= kBiclMgsrL, the left-looking
// per-(i, j) kernel larger l
constexpr int kBiclMgsrL = 8;
constexpr int kBiclMgsrW = 4;  // columns per blockIdx.y slice of k_bl_mgsr
struct BiclKernels {
    const void *init, *u, *r, *mgs, *mgsr, *upd, *exit, *true_res;
};
BiclKernels bicgl_kernels();
size_t bicgl_state_size();
size_t bicgl_args_size();
int bicgl_state_done_offset();
void bicgl_init_state(void* host_state, double tol, long long max_iter, int l, int record, long long hist_cap);
void bicgl_pack_args(void* out, const Csr& A, const double2* dinv, const double2* b, double2* x, double2* work,
                     double2* part, void* st, double* hist, DevReport* rep);

// standalone kernels (cvk_blas.cu); all enqueue on `st`
// uniform off-diagonal values (Csr::dg / Csr::uni), checked per solve
cudaError_t launch_uniform_check(int n, const int* rp, const int* ci, const double2* av, double2* dg, double2* uni,
                                 cudaStream_t st);
cudaError_t launch_spmv(int S, bool ref, int n, const int* rp, const int* ci, const double2* av,
                        const double2* x, double2* y, int tile, cudaStream_t st);
// FAST SpMV on the TMA ring; cudaErrorInvalidConfiguration if a chunk does not fit
cudaError_t launch_spmv_stream(int n, const int* rp, const int* ci, const double2* av, const double2* x,
                               double2* y, int capk, int nsm, int optin, cudaStream_t st, const int* skip = nullptr);
// cavity operator values at omega on the cavity's 5-point pattern (cvk_assemble.cu);
// *bad receives the first row whose pattern does not match (INT32_MAX if none)
cudaError_t launch_cavity_values(int nx, int ny, int roof_begin, int roof_end, double k2, double om2,
                                 double kw_re, double kw_im, const int* rp, const int* ci, double2* av,
                                 int* bad, int nsm, cudaStream_t st);
// FEM operator values K - omega^2 M + i omega C (cvk_assemble.cu)
cudaError_t launch_fem_values(long long nnz, const double* K, const double* M, const double* Cd, double omega,
                              double2* av, int nsm, cudaStream_t st);
cudaError_t launch_inv_diag(int n, const int* rp, const int* ci, const double2* av, double2* out,
                            int* bad_row, cudaStream_t st);
// out[0] = sum conj(x) y (mode dot) or sum |x|^2 (norm, y == nullptr); part >= 2048 double2
// (hi and lo partials of 592 CTAs)
cudaError_t launch_dot(bool ref, int n, const double2* x, const double2* y, double2* part,
                       double2* out, cudaStream_t st);
cudaError_t launch_axpy(int n, double2 alpha, const double2* x, double2* y, cudaStream_t st);
cudaError_t launch_xpay(int n, double2 alpha, double2* x, const double2* y, cudaStream_t st);
cudaError_t launch_residual(int S, bool ref, int n, const int* rp, const int* ci, const double2* av,
                            const double2* b, const double2* x, double2* r, cudaStream_t st);

// ILU(0) factor on the device (cvk_ilu.cu): strict L and strict U as CSR,
// d = 1 / u_ii; the apply runs `sweeps` Jacobi sweeps per triangle
struct IluDev {
    int n = 0, sweeps = 2;
    int *lrp = nullptr, *lci = nullptr, *urp = nullptr, *uci = nullptr;
    double2 *lav = nullptr, *uav = nullptr, *dinv = nullptr;
    void* blob = nullptr;  // one allocation behind all of the above
};
// z = M^-1 r; tmp >= 2 n complex; r, z, tmp disjoint; *nl += launches
// skip (optional, device): a stop flag; the launches return at once when it is set
cudaError_t launch_ilu0_apply(const IluDev& M, const double2* r, double2* z, double2* tmp, int* nl,
                              cudaStream_t st, const int* skip = nullptr);

// BiCGSTAB + ILU(0) phase chain (cvk_ilu.cu): device-resident scalars
struct IcState {
    int done, conv, brk_code, no_true, record, pad;
    long long it, iterations, max_iter, hl, hist_cap;
    double bnorm, brk, tol, final_relres;
    double2 rho, alpha, omega, beta;
    unsigned counter;  // last-arrival counter of the fused folds
};
struct IcArgs {
    int n;
    double2 *x, *r, *p, *v, *s, *t, *tmp, *ptmp;  // ptmp: 2 n (ILU sweeps)
    const double2* sh;
    double2* part;  // >= 4 * 592 double2
    IcState* st;
    double* hist;
};
cudaError_t launch_ic_init(const IcArgs& a, cudaStream_t st);
// `iters` iterations; spmv(ctx, in) computes A in -> a.tmp on st
cudaError_t launch_ic_iters(const IcArgs& a, const IluDev& M, int iters,
                            cudaError_t (*spmv)(void*, const double2*), void* ctx, int* nl, cudaStream_t st);

}  // namespace cvk
