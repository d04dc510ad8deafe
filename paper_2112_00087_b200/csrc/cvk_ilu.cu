// cvk_ilu.cu -- ILU(0) preconditioner apply on sm_100a (beyond the reference,
// which has only jacobi / identity_preconditioner, krylov.cpp:27-55;
// SURVEY.md 8(f) rank 4).
//
// The factor is exact ILU(0) on A's pattern (host, cvk_api.cu
// cvk_precond_ilu0 = oracle/cavac_oracle.c orc_ilu0_arrays).  The triangular
// solves are NOT level-scheduled: the 2-D cavity has ~2 (nx + ny) dependent
// levels (~4,200 at 1M DOF), i.e. thousands of grid-wide steps per apply.
// They are sync-free Jacobi sweeps instead, each one fully parallel and one
// HBM pass over a triangle:
//   y_0 = r,          y_k[i] = r[i] - sum_{j<i} l_ij y_{k-1}[j]
//   z_0 = d .* y,     z_k[i] = d[i] (y[i] - sum_{j>i} u_ij z_{k-1}[j]),  d = 1 / u_ii
// The first U sweep forms z_0 = d .* y inside its gathers, so an apply with
// s sweeps per triangle is 2 s launches (s = 0: one elementwise d .* r).
// Sums run in CSR order with one rounding per complex op: the apply is
// bitwise orc_ilu0_apply_arrays.
//
// Bytes per sweep (algorithmic): L or U values + columns (16 + 4 B per
// stored entry) + row pointers (4 B per row) + rhs, gathered vector and
// output (3 x 16 B per row, plus d (16 B) on the U side).
#include <cuda_runtime.h>

#include "cvk_engine.cuh"
#include "cvk_kernels.h"

namespace cvk {

namespace {

constexpr int kIluThreads = 256;

// out[i] = os[i] * (rhs[i] - sum_p av[p] * xs[c] * xin[c]), c = ci[p]; xs / os optional
template <bool XS, bool OS>
__global__ void __launch_bounds__(kIluThreads) k_ilu_sweep(int n, const int* __restrict__ rp,
                                                           const int* __restrict__ ci,
                                                           const double2* __restrict__ av,
                                                           const double2* __restrict__ rhs,
                                                           const double2* __restrict__ xin,
                                                           const double2* __restrict__ xs,
                                                           const double2* __restrict__ os,
                                                           double2* __restrict__ out, const int* skip) {
    if (skip && *(volatile const int*)skip) return;  // the solve already stopped (graph tail)
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int p0 = __ldg(rp + i), p1 = __ldg(rp + i + 1);
    double2 s = __ldg(rhs + i);
    for (int p = p0; p < p1; ++p) {
        const int c = __ldg(ci + p);
        double2 xv = __ldg(xin + c);
        if (XS) xv = cvk_mul(__ldg(xs + c), xv);
        s = cvk_sub(s, cvk_mul(__ldg(av + p), xv));
    }
    if (OS) s = cvk_mul(__ldg(os + i), s);
    out[i] = s;
}

__global__ void __launch_bounds__(kIluThreads) k_ilu_scale(int n, const double2* __restrict__ d,
                                                           const double2* __restrict__ y,
                                                           double2* __restrict__ z, const int* skip) {
    if (skip && *(volatile const int*)skip) return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) z[i] = cvk_mul(__ldg(d + i), __ldg(y + i));
}

int ilu_grid(int n) { return (n + kIluThreads - 1) / kIluThreads; }

}  // namespace

// z = M^-1 r for the ILU(0) factor (see the header comment).  tmp holds 2 n
// complex.  r and z must not alias.  Returns the number of launches in *nl.
cudaError_t launch_ilu0_apply(const IluDev& M, const double2* r, double2* z, double2* tmp, int* nl,
                              cudaStream_t st, const int* skip) {
    const int n = M.n;
    if (n <= 0) return cudaSuccess;
    const int G = ilu_grid(n);
    int launches = 0;
    if (M.sweeps <= 0) {
        k_ilu_scale<<<G, kIluThreads, 0, st>>>(n, M.dinv, r, z, skip);
        if (nl) *nl += 1;
        return cudaGetLastError();
    }
    // L sweeps: ping-pong between tmp[0] and tmp[1]; y_0 = r
    double2* buf[2] = {tmp, tmp + n};
    const double2* y = r;
    for (int k = 0; k < M.sweeps; ++k) {
        double2* o = buf[k & 1];
        k_ilu_sweep<false, false><<<G, kIluThreads, 0, st>>>(n, M.lrp, M.lci, M.lav, r, y, nullptr, nullptr, o, skip);
        ++launches;
        y = o;
    }
    // U sweeps: y stays in its buffer; z ping-pongs between z and the other tmp half
    double2* other = (y == buf[0]) ? buf[1] : buf[0];
    // choose the first output so that the last sweep lands in z
    double2* zb[2] = {(M.sweeps & 1) ? z : other, (M.sweeps & 1) ? other : z};
    const double2* zin = y;
    for (int k = 0; k < M.sweeps; ++k) {
        double2* o = zb[k & 1];
        if (k == 0)
            k_ilu_sweep<true, true><<<G, kIluThreads, 0, st>>>(n, M.urp, M.uci, M.uav, y, zin, M.dinv, M.dinv, o, skip);
        else
            k_ilu_sweep<false, true><<<G, kIluThreads, 0, st>>>(n, M.urp, M.uci, M.uav, y, zin, nullptr, M.dinv, o, skip);
        ++launches;
        zin = o;
    }
    if (nl) *nl += launches;
    return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// BiCGSTAB with the ILU(0) apply, FAST mode, as a chain of phase kernels with
// the scalars on the device (no host round trip per reduction), replayed from
// a CUDA graph.  Operation order = krylov.cpp:57-138 (oracle orc_bicgstab);
// every reduction is the double-double two-stage sum of cvk_blas.cu.  Per
// iteration: k_ic_p, SpMV, 2s sweeps, k_ic_dot<1> + k_ic_fold<1>, k_ic_s +
// k_ic_fold<3>, SpMV, 2s sweeps, k_ic_dot<2> + k_ic_fold<2>, k_ic_xr +
// k_ic_fold<4> (which also takes <sh, r> for the next iteration's rho).
namespace {

constexpr int kIcBlocks = 592;  // 4 x 148, fixed so the FAST sum order is fixed

__device__ __forceinline__ double cabs2(double2 a) { return hypot(a.x, a.y); }

__device__ void ic_hist(IcState* st, double* hist, double v) {
    if (!st->record) return;
    if (st->hl < st->hist_cap) hist[st->hl] = v;
    st->hl++;
}

// rho for iteration it (MODE 0 logic), thread 0 of the fold
__device__ void ic_rho(IcState* st, double2 rho_new) {
    const long long it = st->it + 1;
    if (it > st->max_iter) { st->done = 1; return; }
    if (cabs2(rho_new) < st->brk) { st->brk_code = 1; st->iterations = it - 1; st->done = 1; return; }
    if (it > 1) st->beta = cvk_mul(cvk_cdiv(rho_new, st->rho), cvk_cdiv(st->alpha, st->omega));
    st->rho = rho_new;
    st->it = it;
}

template <int MODE>
__device__ void ic_fold_tail(const IcArgs& a);

// stage 1: MODE 0 init {|r|^2, <r, r>}, 1 <sh, v>, 2 {|t|^2, <t, s>}
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_ic_dot(IcArgs a) {
    if (a.st->done) return;
    CAcc acc[2] = {};
    for_elems(a.n, gridDim.x, blockIdx.x, [&](int i) {
        if (MODE == 0) {
            const double2 ri = a.r[i];
            acc_norm(acc[0], ri);
            acc_dot(acc[1], ri, ri);
        } else if (MODE == 1) {
            acc_dot(acc[0], __ldg(a.sh + i), a.v[i]);
        } else {
            const double2 ti = a.t[i];
            acc_norm(acc[0], ti);
            acc_dot(acc[1], ti, a.s[i]);
        }
    });
    cta_partial<2>(acc, a.part, gridDim.x, blockIdx.x);
}

// p = r (it == 1) or p = beta (p - omega v) + r  (axpy then xpay, krylov.cpp:77-80)
__global__ void __launch_bounds__(kThreads) k_ic_p(IcArgs a) {
    const IcState* st = a.st;
    if (st->done) return;
    const bool first = st->it == 1;
    const double2 nom = make_double2(-st->omega.x, -st->omega.y), beta = st->beta;
    for_elems(a.n, gridDim.x, blockIdx.x, [&](int i) {
        const double2 ri = a.r[i];
        a.p[i] = first ? ri : cvk_add(cvk_mul(beta, cvk_add(a.p[i], cvk_mul(nom, a.v[i]))), ri);
    });
}

// s = r - alpha v; x += alpha p; partial |s|^2
__global__ void __launch_bounds__(kThreads) k_ic_s(IcArgs a) {
    const IcState* st = a.st;
    if (st->done) return;
    const double2 al = st->alpha, nal = make_double2(-al.x, -al.y);
    CAcc acc[2] = {};
    for_elems(a.n, gridDim.x, blockIdx.x, [&](int i) {
        const double2 si = cvk_add(a.r[i], cvk_mul(nal, a.v[i]));
        a.s[i] = si;
        a.x[i] = cvk_add(a.x[i], cvk_mul(al, a.p[i]));
        acc_norm(acc[0], si);
    });
    cta_partial<2>(acc, a.part, gridDim.x, blockIdx.x);
}

// x += omega s; r = s - omega t; partials |r|^2 and <sh, r>
__global__ void __launch_bounds__(kThreads) k_ic_xr(IcArgs a) {
    const IcState* st = a.st;
    if (st->done) return;
    const double2 om = st->omega, nom = make_double2(-om.x, -om.y);
    CAcc acc[2] = {};
    for_elems(a.n, gridDim.x, blockIdx.x, [&](int i) {
        const double2 si = a.s[i];
        a.x[i] = cvk_add(a.x[i], cvk_mul(om, si));
        const double2 ri = cvk_add(si, cvk_mul(nom, a.t[i]));
        a.r[i] = ri;
        acc_norm(acc[0], ri);
        acc_dot(acc[1], __ldg(a.sh + i), ri);
    });
    cta_partial<2>(acc, a.part, gridDim.x, blockIdx.x);
}

// stage 2 + the scalar step.  MODE 0: bnorm and rho_1; 1: gamma -> alpha;
// 2: omega; 3: |s| test; 4: |r| test, then rho for the next iteration.
template <int MODE>
__device__ void ic_fold_tail(const IcArgs& a) {
    IcState* st = a.st;
    double2 v[2];
    fold_partials<2>(v, a.part, kIcBlocks);
    if (threadIdx.x != 0) return;
    if (MODE == 0) {
        st->bnorm = sqrt(v[0].x);
        if (st->bnorm == 0.0) { st->conv = 1; st->no_true = 1; st->done = 1; return; }
        st->brk = 1e-30 * st->bnorm * st->bnorm;
        ic_rho(st, v[1]);
    } else if (MODE == 1) {
        if (cabs2(v[0]) < st->brk) { st->brk_code = 2; st->iterations = st->it - 1; st->done = 1; return; }
        st->alpha = cvk_cdiv(st->rho, v[0]);
    } else if (MODE == 2) {
        const double2 tt = make_double2(v[0].x, 0.0);
        if (cabs2(tt) < st->brk) { st->brk_code = 3; st->iterations = st->it; st->done = 1; return; }
        st->omega = cvk_cdiv(v[1], tt);
    } else if (MODE == 3) {
        const double relres = sqrt(v[0].x) / st->bnorm;
        if (relres <= st->tol) {
            st->conv = 1, st->iterations = st->it, st->final_relres = relres;
            ic_hist(st, a.hist, relres);
            st->done = 1;
        }
    } else {
        const double relres = sqrt(v[0].x) / st->bnorm;
        st->final_relres = relres;
        st->iterations = st->it;
        ic_hist(st, a.hist, relres);
        if (relres <= st->tol) { st->conv = 1; st->done = 1; return; }
        ic_rho(st, v[1]);
    }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads) k_ic_fold(IcArgs a) {
    if (a.st->done) return;
    ic_fold_tail<MODE>(a);
}

int ic_grid(int n) {
    (void)n;
    return kIcBlocks;
}

}  // namespace

cudaError_t launch_ic_init(const IcArgs& a, cudaStream_t st) {
    k_ic_dot<0><<<kIcBlocks, kThreads, 0, st>>>(a);
    k_ic_fold<0><<<1, kThreads, 0, st>>>(a);
    return cudaGetLastError();
}

// one iteration; spmv(in, out) launches A in -> a.tmp; returns launches in *nl
template <class Spmv>
static cudaError_t ic_iter(const IcArgs& a, const IluDev& M, Spmv&& spmv, int* nl, cudaStream_t st) {
    cudaError_t e;
    const int G = ic_grid(a.n);
    k_ic_p<<<G, kThreads, 0, st>>>(a);
    if ((e = spmv(a.p)) != cudaSuccess) return e;
    if ((e = launch_ilu0_apply(M, a.tmp, a.v, a.ptmp, nl, st, &a.st->done)) != cudaSuccess) return e;
    k_ic_dot<1><<<G, kThreads, 0, st>>>(a);
    k_ic_fold<1><<<1, kThreads, 0, st>>>(a);
    k_ic_s<<<G, kThreads, 0, st>>>(a);
    k_ic_fold<3><<<1, kThreads, 0, st>>>(a);
    if ((e = spmv(a.s)) != cudaSuccess) return e;
    if ((e = launch_ilu0_apply(M, a.tmp, a.t, a.ptmp, nl, st, &a.st->done)) != cudaSuccess) return e;
    k_ic_dot<2><<<G, kThreads, 0, st>>>(a);
    k_ic_fold<2><<<1, kThreads, 0, st>>>(a);
    k_ic_xr<<<G, kThreads, 0, st>>>(a);
    k_ic_fold<4><<<1, kThreads, 0, st>>>(a);
    *nl += 12;
    return cudaGetLastError();
}

cudaError_t launch_ic_iters(const IcArgs& a, const IluDev& M, int iters,
                            cudaError_t (*spmv)(void*, const double2*), void* ctx, int* nl, cudaStream_t st) {
    for (int k = 0; k < iters; ++k) {
        cudaError_t e = ic_iter(a, M, [&](const double2* in) { return spmv(ctx, in); }, nl, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace cvk
