// cvk_bicgl.cu -- FAST-mode BiCGSTAB(l) for large systems (krylov.cpp:140-286)
// as one uniform "step" kernel replayed from a CUDA graph.
//
// A BiCGSTAB(l) cycle is 2l + l(l+1)/2 + 1 reduction phases (l u-steps and
// l r-steps with an SpMV each, the l(l+1)/2 modified-Gram-Schmidt steps of
// the minimal-residual part, the polynomial update).  The graph is one
// cycle's phase sequence -- U0 R0 ... U(l-1) R(l-1), the MGS steps, the
// update, an exit node -- each node a kernel specialised to its phase type
// (k_bl_u / k_bl_r / k_bl_mgs / k_bl_upd / k_bl_exit).  The CTA that arrives
// last folds the double-double partials and runs the reference's scalar
// logic (breakdown tests, tau / sigma / gamma', the gamma recurrences,
// convergence), then names the next phase; a node whose phase is not the
// state's returns at once, so an early exit skips to the exit node.  The host
// polls `done` between graphs.  The persistent kernel
// runs these phases with one CTA-wide element per thread and grid barriers
// at 3 CTAs/SM (2.4 ms per l=8 cycle at 1M DOF); here every phase is a
// full-occupancy kernel.
//
// Per-element arithmetic, the slot rotation of u_j / r_j through a spare
// vector, and the pending-update fusion of the MGS loop are those of the
// persistent kernel (cvk_krylov.cu bicgstab_l_body); reductions are
// double-double, so the two FAST paths agree bit for bit.
#include <cuda_runtime.h>

#include <cstddef>

#include "cvk_engine.cuh"
#include "cvk_kernels.h"

namespace cvk {

namespace {

enum { P_U = 0, P_R = 1, P_MGS = 2, P_UPD = 3, P_EXIT = 4, P_MGSR = 5 };

// right-looking MGS passes for l <= kMgsrL (accumulators per pass: l + 1)
constexpr int kMgsrL = 8;

struct BLState {
    int done, conv, brk_code, phase, j, i, exit_mr, skip_true;
    long long cycle, iters, hl, hist_cap, max_iter;
    int record, L;
    double bnorm, brk, tol, final_relres;
    double2 rho_old, alpha, omega, rho_next, beta;
    unsigned counter[2];
    int ri[kMaxL + 2], ui[kMaxL + 2];
    double2 tau[kMaxL * kMaxL], sig[kMaxL], gam[kMaxL], gp[kMaxL], gpp[kMaxL];
};

struct BLArgs {
    Csr A;
    const double2* dinv;
    const double2* b;
    double2* x;
    double2* work;  // shadow, scratch, then 2l + 4 rotating slots
    double2* part;
    BLState* st;
    double* hist;
    DevReport* rep;
};

__device__ __forceinline__ void pdl_enter_b() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ double2* slot(const BLArgs& a, int s) { return a.work + (size_t)(2 + s) * a.A.n; }

__device__ bool arrive_last_b(unsigned* counter) {
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(counter, 1u) == gridDim.x - 1u;
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last != 0;
}

// CTA partials of K dd accumulators -> grid sums in the last CTA (thread 0 reads tot)
template <int K>
__device__ bool reduce_last(const CAcc (&acc)[K], double2* part, unsigned* counter, double2 (&tot)[K]) {
    CAcc v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = acc[k];
    __shared__ CAcc sm[K][32];
    cta_sum_k<K, kThreads>(v, sm);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) cacc_store(part, k, gridDim.x, blockIdx.x, v[k]);
    if (!arrive_last_b(counter)) return false;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < K; ++k) tot[k] = fold_one(part, k, gridDim.x, lane);
    return true;
}

// element loop over the CTA's 256-row chunks (the ownership of for_rows),
// U chunks per trip with every load of a trip issued before its stores:
// the MGS phases are a few vector reads each, latency-bound one element at
// a time (35 us for 48 MB at 1M DOF)
template <int U, class LD, class STF>
__device__ __forceinline__ void elems_batched(int n, int G, int cta, LD&& ld, STF&& stf) {
    using T = decltype(ld(0));
    const long long step = (long long)G * kThreads;
    for (long long base = (long long)cta * kThreads + threadIdx.x; base < n; base += U * step) {
        T v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = base + u * step;
            if (i < n) v[u] = ld((int)i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = base + u * step;
            if (i < n) stf((int)i, v[u]);
        }
    }
}

__device__ __forceinline__ void bhist(const BLArgs& a, BLState* st, double v) {
    if (!st->record) return;
    if (st->hl < st->hist_cap) a.hist[st->hl] = v;
    st->hl++;
}

// ---- scalar transitions (thread 0 of the last CTA) ----------------------

__device__ void to_exit(BLState* st, int mr) {
    st->exit_mr = mr;
    st->phase = P_EXIT;
}

// gamma, gamma', gamma'' (krylov.cpp:251-262), then the update phase
__device__ void finish_mr(BLState* st, int L) {
    // gamma, gamma', gamma'' (krylov.cpp:251-262)
    st->gam[L - 1] = st->gp[L - 1];
    for (int jj = L - 1; jj-- > 0;) {
        double2 gj = st->gp[jj];
        for (int q = jj + 1; q < L; ++q) gj = cvk_sub(gj, cvk_mul(st->tau[jj * L + q], st->gam[q]));
        st->gam[jj] = gj;
    }
    for (int jj = 0; jj + 1 < L; ++jj) {
        double2 gj = st->gam[jj + 1];
        for (int q = jj + 1; q + 1 < L; ++q) gj = cvk_add(gj, cvk_mul(st->tau[jj * L + q], st->gam[q + 1]));
        st->gpp[jj] = gj;
    }
    st->omega = st->gam[L - 1];
    st->phase = P_UPD;
}

// top of BiCG step j (krylov.cpp:175-186)
__device__ void prep_u(BLState* st) {
    const double2 rho = st->rho_next;
    if (cvk_abs(st->rho_old) < st->brk) { st->brk_code = 1; to_exit(st, 0); return; }
    st->beta = cvk_cdiv(cvk_mul(st->alpha, rho), st->rho_old);
    st->rho_old = rho;
    st->phase = P_U;
}

// top of a cycle (krylov.cpp:170-173)
__device__ void start_cycle(BLState* st) {
    if (st->cycle > st->max_iter) { st->done = 1; return; }
    st->rho_old = cvk_mul(cvk_neg(st->omega), st->rho_old);
    st->j = 0;
    prep_u(st);
}

__global__ void __launch_bounds__(kThreads) k_bl_init(BLArgs a) {
    pdl_enter_b();
    BLState* st = a.st;
    const int n = a.A.n, L = st->L;
    __shared__ int ri[kMaxL + 2], ui[kMaxL + 2];
    if (threadIdx.x <= L) { ri[threadIdx.x] = threadIdx.x; ui[threadIdx.x] = L + 1 + threadIdx.x; }
    if (threadIdx.x == 0) { ri[L + 1] = 2 * L + 2; ui[L + 1] = 2 * L + 3; }
    __syncthreads();
    double2* sh = a.work;
    CAcc acc[2] = {};
    for_elems(n, gridDim.x, blockIdx.x, [&](int i) {
        const double2 v0 = prec_apply(a.dinv, i, __ldg(a.b + i));
        slot(a, ri[0])[i] = v0;
        sh[i] = v0;
        a.x[i] = make_double2(0, 0);
        for (int j = 1; j <= L; ++j) slot(a, ri[j])[i] = make_double2(0, 0);
        for (int j = 0; j <= L; ++j) slot(a, ui[j])[i] = make_double2(0, 0);
        acc_norm(acc[0], v0);
        acc_dot(acc[1], v0, v0);
    });
    double2 tot[2];
    if (!reduce_last<2>(acc, a.part, &st->counter[0], tot)) return;
    if (threadIdx.x != 0) return;
    st->counter[0] = 0;
    for (int q = 0; q <= L + 1; ++q) { st->ri[q] = ri[q]; st->ui[q] = ui[q]; }
    st->bnorm = sqrt(tot[0].x);
    if (st->bnorm == 0.0) { st->done = 1; st->conv = 1; st->skip_true = 1; return; }
    st->brk = 1e-30 * st->bnorm * st->bnorm;
    st->rho_old = make_double2(1, 0);
    st->alpha = make_double2(0, 0);
    st->omega = make_double2(1, 0);
    st->rho_next = tot[1];
    st->cycle = 1;
    start_cycle(st);
}

#ifndef CVK_BL_SPMV_BATCH
#define CVK_BL_SPMV_BATCH 5  // gathers in flight per row in the u/r SpMV phases
#endif
#ifndef CVK_BL_BATCH
#define CVK_BL_BATCH 4  // elements in flight per thread in the MGS phases
#endif
// One phase of the cycle; PH is the phase this launch implements: a launch
// whose phase is not the state's current one returns at once (the graph is
// one cycle's static phase sequence, and an early exit skips ahead to the
// cycle's P_EXIT node).
template <int PH>
__device__ __forceinline__ void bl_phase(const BLArgs& a) {
    pdl_enter_b();
    BLState* st = a.st;
    if (st->done || st->phase != PH) return;
    constexpr int phase = PH;
    const int n = a.A.n, L = st->L, j = st->j;
    __shared__ int ri[kMaxL + 2], ui[kMaxL + 2];
    if (threadIdx.x <= L + 1) { ri[threadIdx.x] = st->ri[threadIdx.x]; ui[threadIdx.x] = st->ui[threadIdx.x]; }
    __syncthreads();
    auto R = [&](int q) { return slot(a, ri[q]); };
    auto U = [&](int q) { return slot(a, ui[q]); };
    const double2* sh = a.work;
    const double2* dinv = a.dinv;
    const int G = gridDim.x, cta = blockIdx.x;

    if constexpr (phase == P_U) {
        // u_i = r_i - beta u_i (i <= j, u_j formed in the gathers); u_{j+1} = M^-1 A u_j; <shadow, u_{j+1}>
        const double2 nbeta = cvk_neg(st->beta);
        const double2* uj_old = U(j);
        const double2* rj = R(j);
        double2* uj_new = U(L + 1);  // spare
        double2* uj1 = U(j + 1);
        auto ujv = [&](int c) -> double2 { return cvk_add(cvk_mul(nbeta, uj_old[c]), rj[c]); };
        CAcc acc[1] = {};
        for_rows<1>(n, G, cta, [&](int row, int, bool valid) {
            const double2 y = row_sum<1, decltype(ujv)&, CVK_BL_SPMV_BATCH>(a.A, row, 0, valid, ujv);
            if (valid) {
                const double2 yi = prec_apply(dinv, row, y);
                uj_new[row] = ujv(row);
                uj1[row] = yi;
                acc_dot(acc[0], sh[row], yi);
            }
        });
        __syncthreads();
        // u_q = r_q - beta u_q for q < j: the loads of four q's are issued
        // before their stores (distinct slots), not one load-store chain per q
        for_elems(n, G, cta, [&](int i) {
            for (int q0 = 0; q0 < j; q0 += 4) {
                double2 uv[4], rv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (q0 + u < j) { uv[u] = U(q0 + u)[i]; rv[u] = R(q0 + u)[i]; }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (q0 + u < j) U(q0 + u)[i] = cvk_add(cvk_mul(nbeta, uv[u]), rv[u]);
            }
        });
        double2 tot[1];
        if (!reduce_last<1>(acc, a.part, &st->counter[0], tot)) return;
        if (threadIdx.x != 0) return;
        st->counter[0] = 0;
        const int tmp = st->ui[j]; st->ui[j] = st->ui[L + 1]; st->ui[L + 1] = tmp;
        if (cvk_abs(tot[0]) < st->brk) { st->brk_code = 4; to_exit(st, 0); return; }
        st->alpha = cvk_cdiv(st->rho_old, tot[0]);
        st->phase = P_R;
        return;
    }
    if constexpr (phase == P_R) {
        // r_i -= alpha u_{i+1} (i <= j, r_j formed in the gathers); r_{j+1} = M^-1 A r_j; x += alpha u_0
        const double2 alpha = st->alpha, nal = cvk_neg(st->alpha);
        const double2* rj_old = R(j);
        const double2* uj1 = U(j + 1);
        double2* rj_new = R(L + 1);
        double2* rj1 = R(j + 1);
        auto rjv = [&](int c) -> double2 { return cvk_add(rj_old[c], cvk_mul(nal, uj1[c])); };
        CAcc acc[2] = {};
        for_rows<1>(n, G, cta, [&](int row, int, bool valid) {
            const double2 y = row_sum<1, decltype(rjv)&, CVK_BL_SPMV_BATCH>(a.A, row, 0, valid, rjv);
            if (valid) {
                rj_new[row] = rjv(row);
                rj1[row] = prec_apply(dinv, row, y);
            }
        });
        __syncthreads();
        const double2* u0 = U(0);
        for_elems(n, G, cta, [&](int i) {
            for (int q0 = 0; q0 < j; q0 += 4) {
                double2 rv[4], uv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (q0 + u < j) { rv[u] = R(q0 + u)[i]; uv[u] = U(q0 + u + 1)[i]; }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (q0 + u < j) R(q0 + u)[i] = cvk_add(rv[u], cvk_mul(nal, uv[u]));
            }
            a.x[i] = cvk_add(a.x[i], cvk_mul(alpha, u0[i]));
            const double2 r0i = (j == 0) ? rj_new[i] : R(0)[i];
            acc_norm(acc[0], r0i);
            acc_dot(acc[1], sh[i], rj1[i]);
        });
        double2 tot[2];
        if (!reduce_last<2>(acc, a.part, &st->counter[0], tot)) return;
        if (threadIdx.x != 0) return;
        st->counter[0] = 0;
        const int tmp = st->ri[j]; st->ri[j] = st->ri[L + 1]; st->ri[L + 1] = tmp;
        st->rho_next = tot[1];
        if (sqrt(tot[0].x) <= st->tol * st->bnorm) { to_exit(st, 0); return; }  // krylov.cpp:203-206
        if (j + 1 < L) {
            st->j = j + 1;
            prep_u(st);
        } else {
            st->phase = L <= kMgsrL ? P_MGSR : P_MGS;
            st->j = 0;
            st->i = 0;
        }
        return;
    }
    if constexpr (phase == P_MGS) {
        // pending update r_{j+1} -= tau_{i-1,j} r_i, then <r_{i+1}, r_{j+1}> (i < j)
        // or sigma_j = <r_{j+1}, r_{j+1}>, <r_{j+1}, r_0> (i == j)   (krylov.cpp:224-238)
        const int i = st->i;
        const bool has_upd = i > 0, last = i == j;
        const double2 ntau = has_upd ? cvk_neg(st->tau[(i - 1) * L + j]) : make_double2(0, 0);
        double2* rj1 = R(j + 1);
        const double2* rprev = has_upd ? R(i) : nullptr;
        const double2* ri1 = R(i + 1);
        const double2* r0 = R(0);
        CAcc acc[2] = {};
        const double2* other = last ? r0 : ri1;
        struct L3 { double2 rj, rp, o; };
        elems_batched<CVK_BL_BATCH>(
            n, G, cta,
            [&](int e) { return L3{rj1[e], has_upd ? rprev[e] : make_double2(0.0, 0.0), other[e]}; },
            [&](int e, const L3& l) {
                double2 v = l.rj;
                if (has_upd) { v = cvk_add(v, cvk_mul(ntau, l.rp)); rj1[e] = v; }
                if (!last) acc_dot(acc[0], l.o, v);
                else { acc_dot(acc[0], v, v); acc_dot(acc[1], v, l.o); }
            });
        double2 tot[2];
        if (!reduce_last<2>(acc, a.part, &st->counter[0], tot)) return;
        if (threadIdx.x != 0) return;
        st->counter[0] = 0;
        if (!last) {
            st->tau[i * L + j] = cvk_cdiv(tot[0], st->sig[i]);
            st->i = i + 1;
            return;
        }
        if (cvk_abs(tot[0]) < st->brk) { st->brk_code = 5; to_exit(st, 1); return; }
        st->sig[j] = tot[0];
        st->gp[j] = cvk_cdiv(tot[1], tot[0]);
        if (j + 1 < L) {
            st->j = j + 1;
            st->i = 0;
            return;
        }
        finish_mr(st, L);
        return;
    }
    if constexpr (phase == P_UPD) {
        // updates (krylov.cpp:264-271), per element in the reference's order
        __shared__ double2 gam[kMaxL], gp[kMaxL], gpp[kMaxL];
        if (threadIdx.x < L) { gam[threadIdx.x] = st->gam[threadIdx.x]; gp[threadIdx.x] = st->gp[threadIdx.x]; gpp[threadIdx.x] = st->gpp[threadIdx.x]; }
        __syncthreads();
        double2* r0 = R(0);
        double2* u0 = U(0);
        CAcc acc[2] = {};
        for_elems(n, G, cta, [&](int i) {
            double2 xi = a.x[i], r0i = r0[i], u0i = u0[i];
            xi = cvk_add(xi, cvk_mul(gam[0], r0i));
            r0i = cvk_add(r0i, cvk_mul(cvk_neg(gp[L - 1]), R(L)[i]));
            u0i = cvk_add(u0i, cvk_mul(cvk_neg(gam[L - 1]), U(L)[i]));
            for (int q = 1; q < L; ++q) {
                const double2 rq = R(q)[i];
                u0i = cvk_add(u0i, cvk_mul(cvk_neg(gam[q - 1]), U(q)[i]));
                xi = cvk_add(xi, cvk_mul(gpp[q - 1], rq));
                r0i = cvk_add(r0i, cvk_mul(cvk_neg(gp[q - 1]), rq));
            }
            a.x[i] = xi; r0[i] = r0i; u0[i] = u0i;
            acc_norm(acc[0], r0i);
            acc_dot(acc[1], sh[i], r0i);
        });
        double2 tot[2];
        if (!reduce_last<2>(acc, a.part, &st->counter[0], tot)) return;
        if (threadIdx.x != 0) return;
        st->counter[0] = 0;
        const double relres = sqrt(tot[0].x) / st->bnorm;
        st->final_relres = relres;
        st->iters = st->cycle;
        bhist(a, st, relres);
        st->rho_next = tot[1];
        if (relres <= st->tol) { st->conv = 1; st->done = 1; return; }
        st->cycle++;
        start_cycle(st);
        return;
    }
    if constexpr (phase != P_EXIT) return;
    // P_EXIT: ||r_0|| after a break (krylov.cpp:208-222, 239-249)
    const double2* r0 = R(0);
    CAcc acc[1] = {};
    for_elems(n, G, cta, [&](int i) { acc_norm(acc[0], r0[i]); });
    double2 tot[1];
    if (!reduce_last<1>(acc, a.part, &st->counter[0], tot)) return;
    if (threadIdx.x != 0) return;
    st->counter[0] = 0;
    const double relres = sqrt(tot[0].x) / st->bnorm;
    st->final_relres = relres;
    if (st->exit_mr) {
        st->iters = st->cycle;
        if (relres <= st->tol) { st->conv = 1; st->brk_code = 0; bhist(a, st, relres); }
    } else if (relres <= st->tol) {
        st->conv = 1; st->brk_code = 0; st->iters = st->cycle;
        bhist(a, st, relres);
    } else {
        st->iters = st->cycle - 1;
    }
    st->done = 1;
}

// Right-looking MGS (l <= kMgsrL): pass q makes r_{q+1} the pivot.  It first
// applies the pending update of every later column, r_{jj+1} -= tau_{q-1,jj}
// r_q (jj >= q), then takes sigma_q = <r_{q+1}, r_{q+1}>, <r_{q+1}, r_0> and
// <r_{q+1}, r_{jj+1}> (jj > q) in the same pass.  Every r_{jj+1} receives
// the same updates in the same order as in the reference's column loop
// (krylov.cpp:224-238), and every inner product sees the same operands, so
// tau, sigma and gamma' are those of the left-looking phases; l passes
// replace l(l+1)/2.
//
// The columns of a pass are split over blockIdx.y slices of kMgsrW: slice y
// updates and writes its own columns (the pivot is column 0 of slice 0) and
// takes their inner products with the pivot, which it updates itself (every
// slice re-reads the pivot and r_q), so a thread carries at most kMgsrW + 1
// double-double accumulators.  All slices arrive on one counter; the last
// CTA folds every accumulator from the x-partials of its slice.
constexpr int kMgsrW = 4;
#ifndef CVK_MGSR_U
#define CVK_MGSR_U 2
#endif
constexpr int kMgsrU = CVK_MGSR_U;
__global__ void __launch_bounds__(kThreads, kMgsrU > 1 ? 2 : 3) k_bl_mgsr(BLArgs a) {
    pdl_enter_b();
    BLState* st = a.st;
    if (st->done || st->phase != P_MGSR) return;
    constexpr int KA = kMgsrW + 1;  // slice 0: sigma, gamma', W - 1 dots; slice y > 0: W dots
    const int n = a.A.n, L = st->L, q = st->i;
    const int nc = L - q;  // columns left (pivot included)
    const int y = blockIdx.y, c0 = y * kMgsrW;
    if (c0 >= nc && y > 0) {  // idle slice: still arrives on the counter
        CAcc acc[1] = {};
        double2 tot[1];
        (void)tot;
        __shared__ int s_last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            s_last = atomicAdd(&st->counter[0], 1u) == gridDim.x * gridDim.y - 1u;
        }
        __syncthreads();
        (void)acc;
        if (!s_last) return;
        __threadfence();
        // fall through as the last CTA: nothing of its own to contribute
        goto fold;
    }
    {
        __shared__ const double2* cols[kMgsrW];
        __shared__ double2* outs[kMgsrW];
        __shared__ double2 ntau[kMgsrW];
        __shared__ double2 ntp;  // pivot's pending factor
        __shared__ const double2 *piv, *rq, *r0;
        if (threadIdx.x < kMgsrW) {
            const int jj = q + c0 + (int)threadIdx.x;
            cols[threadIdx.x] = jj < L ? slot(a, st->ri[jj + 1]) : nullptr;
            // the updated pivot goes to the spare slot: the other slices
            // read the pivot as it was before this pass (swapped in by the fold)
            outs[threadIdx.x] = jj < L ? slot(a, st->ri[jj == q ? L + 1 : jj + 1]) : nullptr;
            ntau[threadIdx.x] = (q > 0 && jj < L) ? cvk_neg(st->tau[(q - 1) * L + jj]) : make_double2(0, 0);
        }
        if (threadIdx.x == 0) {
            piv = slot(a, st->ri[q + 1]);
            ntp = q > 0 ? cvk_neg(st->tau[(q - 1) * L + q]) : make_double2(0, 0);
            rq = q > 0 ? slot(a, st->ri[q]) : nullptr;
            r0 = slot(a, st->ri[0]);
        }
        __syncthreads();
        const int ncol = min(kMgsrW, nc - c0);  // this slice's columns
        CAcc acc[KA] = {};
        // kMgsrU elements per thread per trip, every load of a trip issued
        // before its first update (the pass is latency-bound otherwise)
        const long long stride = (long long)gridDim.x * kThreads;
        for (long long i0 = (long long)blockIdx.x * kThreads + threadIdx.x; i0 < n; i0 += stride * kMgsrU) {
            double2 v[kMgsrU][kMgsrW], pv[kMgsrU], o[kMgsrU], p[kMgsrU];
#pragma unroll
            for (int u = 0; u < kMgsrU; ++u) {
                const long long i = i0 + u * stride;
                if (i >= n) continue;
#pragma unroll
                for (int c = 0; c < kMgsrW; ++c)
                    if (c < ncol) v[u][c] = cols[c][i];
                pv[u] = y == 0 ? make_double2(0, 0) : piv[i];
                o[u] = y == 0 ? r0[i] : make_double2(0, 0);
                p[u] = q > 0 ? rq[i] : make_double2(0, 0);
            }
#pragma unroll
            for (int u = 0; u < kMgsrU; ++u) {
                const long long i = i0 + u * stride;
                if (i >= n) continue;
                if (q > 0) {
#pragma unroll
                    for (int c = 0; c < kMgsrW; ++c)
                        if (c < ncol) {
                            v[u][c] = cvk_add(v[u][c], cvk_mul(ntau[c], p[u]));
                            outs[c][i] = v[u][c];
                        }
                    if (y != 0) pv[u] = cvk_add(pv[u], cvk_mul(ntp, p[u]));
                }
                if (y == 0) {
                    const double2 pw = v[u][0];
                    acc_dot(acc[0], pw, pw);
                    acc_dot(acc[1], pw, o[u]);
#pragma unroll
                    for (int c = 1; c < kMgsrW; ++c)
                        if (c < ncol) acc_dot(acc[1 + c], pw, v[u][c]);
                } else {
#pragma unroll
                    for (int c = 0; c < kMgsrW; ++c)
                        if (c < ncol) acc_dot(acc[c], pv[u], v[u][c]);
                }
            }
        }
        // partial slots: 0 sigma, 1 gamma', 1 + c for global column c (pivot = 0)
        __shared__ CAcc sm[KA][32];
        cta_sum_k<KA, kThreads>(acc, sm);
        const int Gx = gridDim.x;
        if (threadIdx.x == 0) {
            if (y == 0) {
                cacc_store(a.part, 0, Gx, blockIdx.x, acc[0]);
                cacc_store(a.part, 1, Gx, blockIdx.x, acc[1]);
                for (int c = 1; c < ncol; ++c) cacc_store(a.part, 1 + c, Gx, blockIdx.x, acc[1 + c]);
            } else {
                for (int c = 0; c < ncol; ++c) cacc_store(a.part, 1 + c0 + c, Gx, blockIdx.x, acc[c]);
            }
        }
        __shared__ int s_last2;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            s_last2 = atomicAdd(&st->counter[0], 1u) == gridDim.x * gridDim.y - 1u;
        }
        __syncthreads();
        if (!s_last2) return;
        __threadfence();
    }
fold:
    {
        // the last CTA: fold sigma, gamma' and the nc - 1 pivot dots (one warp each)
        __shared__ double2 res[kMgsrL + 1];
        const int Gx = gridDim.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int k = warp; k < 1 + nc; k += kThreads / 32) {
            const double2 t = fold_one(a.part, k, Gx, lane);
            if (lane == 0) res[k] = t;
        }
        __syncthreads();
        if (threadIdx.x != 0) return;
        st->counter[0] = 0;
        if (q > 0) { const int tmp = st->ri[q + 1]; st->ri[q + 1] = st->ri[L + 1]; st->ri[L + 1] = tmp; }
        const double2 sig = res[0];
        if (cvk_abs(sig) < st->brk) { st->brk_code = 5; to_exit(st, 1); return; }  // krylov.cpp:231-236
        st->sig[q] = sig;
        st->gp[q] = cvk_cdiv(res[1], sig);
        for (int c = 1; c < nc; ++c) st->tau[q * L + q + c] = cvk_cdiv(res[1 + c], sig);
        if (q + 1 < L) {
            st->i = q + 1;
            return;
        }
        finish_mr(st, L);
    }
}

// The phase kernels.  Each carries only its own phase's registers: the MGS
// and update phases are plain element streams and run at full occupancy with
// four elements' loads in flight per thread; the u / r phases keep the
// thread-per-row SpMV.
__global__ void __launch_bounds__(kThreads, 3) k_bl_u(BLArgs a) { bl_phase<P_U>(a); }
__global__ void __launch_bounds__(kThreads, 3) k_bl_r(BLArgs a) { bl_phase<P_R>(a); }
__global__ void __launch_bounds__(kThreads, 2) k_bl_mgs(BLArgs a) { bl_phase<P_MGS>(a); }
__global__ void __launch_bounds__(kThreads, 3) k_bl_upd(BLArgs a) { bl_phase<P_UPD>(a); }
__global__ void __launch_bounds__(kThreads, 4) k_bl_exit(BLArgs a) { bl_phase<P_EXIT>(a); }

__global__ void __launch_bounds__(kThreads) k_bl_true(BLArgs a) {
    pdl_enter_b();
    BLState* st = a.st;
    const int n = a.A.n;
    const double2* x = a.x;
    auto xat = [&](int c) -> double2 { return x[c]; };
    CAcc acc[2] = {};
    if (!st->skip_true) {
        for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
            const double2 yv = row_sum<1, decltype(xat)&, 5>(a.A, row, 0, valid, xat);
            if (valid) {
                const double2 bi = __ldg(a.b + row);
                acc_norm(acc[0], bi);
                acc_norm(acc[1], cvk_sub(bi, yv));
            }
        });
    }
    double2 tot[2];
    if (!reduce_last<2>(acc, a.part, &st->counter[1], tot)) return;
    if (threadIdx.x != 0) return;
    st->counter[1] = 0;
    double trr = 0.0;
    if (!st->skip_true) {
        const double bn = sqrt(tot[0].x), rn = sqrt(tot[1].x);
        trr = bn > 0 ? rn / bn : rn;
    }
    a.rep->converged = st->conv;
    a.rep->breakdown = st->brk_code;
    a.rep->iterations = st->iters;
    a.rep->final_relres = st->final_relres;
    a.rep->true_relres = trr;
    a.rep->history_len = st->hl;
    a.rep->error = 0;
}

}  // namespace

BiclKernels bicgl_kernels() {
    BiclKernels k;
    k.init = (const void*)k_bl_init;
    k.u = (const void*)k_bl_u;
    k.r = (const void*)k_bl_r;
    k.mgs = (const void*)k_bl_mgs;
    k.mgsr = (const void*)k_bl_mgsr;
    k.upd = (const void*)k_bl_upd;
    k.exit = (const void*)k_bl_exit;
    k.true_res = (const void*)k_bl_true;
    return k;
}
size_t bicgl_state_size() { return sizeof(BLState); }
size_t bicgl_args_size() { return sizeof(BLArgs); }
int bicgl_state_done_offset() { return (int)offsetof(BLState, done); }
void bicgl_init_state(void* host_state, double tol, long long max_iter, int l, int record, long long hist_cap) {
    BLState* s = (BLState*)host_state;
    s->tol = tol;
    s->max_iter = max_iter;
    s->L = l;
    s->record = record;
    s->hist_cap = hist_cap;
}
void bicgl_pack_args(void* out, const Csr& A, const double2* dinv, const double2* b, double2* x, double2* work,
                     double2* part, void* st, double* hist, DevReport* rep) {
    BLArgs* p = (BLArgs*)out;
    p->A = A;
    p->dinv = dinv;
    p->b = b;
    p->x = x;
    p->work = work;
    p->part = part;
    p->st = (BLState*)st;
    p->hist = hist;
    p->rep = rep;
}

}  // namespace cvk
