// cvk_phased.h -- device state and kernel table of the phase-kernel solvers
// (cvk_phased.cu), shared with the host launcher in cvk_api.cu.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace cvk {

struct Csr;
struct DevReport;

// BiCGSTAB scalars of the consumer-fold kernels (k_bf_*), double-buffered by
// launch parity: a kernel reads scal[par] and its CTA 0 writes scal[par ^ 1].
struct BiScal {
    double2 rho, alpha, omega, beta;
    long long it;
    int cur, first;
};

// tfQMR scalars of the consumer-fold kernels (k_tq_*), double-buffered the
// same way.
struct TfScal {
    double2 rho, alpha, beta, eta;
    double theta, tau;
    long long it;
    int cur, first;
};

// Solver state carried between phase kernels (device memory).  Written only
// by the last-arriving CTA of each phase kernel (CTA 0 for k_bf_*); read by
// the next kernel.
struct PState {
    double2 rho, rho_new, alpha, omega, beta, eta;
    double bnorm, brk, tol, final_relres, tau, theta;
    long long it, iters, max_iter, hist_len, hist_cap;
    int done, conv, brk_code, first, pending_x, cur, record, skip_true;
    int warm;  // BiCGSTAB: start from the x passed in (k_bi_init)
    unsigned counter[4];
    BiScal scal[2];
    TfScal tscal[2];
};

struct PhasedKernels {
    const void *bi_init, *bi_a, *bi_b, *bi_c;
    const void *tf_init, *tf_init2, *tf_w, *tf_e, *tf_o, *tf_fix;
    const void* true_res;  // (PArgs, double2* scratch)
    // streamed SpMV phases (cvk_stream.cuh): kStreamThreads threads, dynamic smem
    const void *bi_a_s, *bi_b_s, *tf_e_s, *tf_o_s;
    // COCG (beyond the reference): init, thread-per-row SpMV phase, elementwise
    // phase, streamed SpMV phase
    const void *cg_init, *cg_a, *cg_b, *cg_a_s;
    // BiCGSTAB with the reductions folded by the consuming kernel (every CTA,
    // redundantly): (PArgs, int parity)
    const void *bf_a_s, *bf_b_s, *bf_c, *bf_init;
    // COCG with consumer-folded reductions (k_cf_*): (PArgs, int parity)
    const void *cf_a_s, *cf_b;
    // tfQMR with consumer-folded reductions (k_tq_*): (PArgs, int parity); seed (PArgs)
    const void *tq_w, *tq_e_s, *tq_o_s, *tq_seed;
};

PhasedKernels phased_kernels();
// CVK_TRACE builds: copy the phase-kernel timestamp buffer (bytes copied, 0 otherwise)
int phased_trace_read(void* out, size_t bytes);
size_t phased_args_size();
void phased_pack_args(void* out, const Csr& A, const double2* dinv, const double2* b, double2* x,
                      double2* work, double2* part, PState* st, double* hist, DevReport* rep,
                      int capk, const int* nst, int pf_rows, const int* gprod = nullptr);

}  // namespace cvk
