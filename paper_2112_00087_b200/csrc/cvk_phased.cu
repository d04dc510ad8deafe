// cvk_phased.cu -- FAST-mode Krylov solvers for large systems as a chain of
// small phase kernels, replayed from a CUDA graph.
//
// Why not the persistent kernel here: a single cooperative kernel carries
// the register allocation of its most complex phase, which caps it at 3
// CTAs/SM and leaves the SpMV phases latency-bound at ~1/3 of HBM peak
// (profiles/r01_persistent_bicgstab.txt).  Each phase kernel below only pays
// for its own work (batched gathers, full occupancy).
//
// Scalars never visit the host.  Each phase kernel ends with a deterministic
// "last CTA folds" reduction: every CTA writes its partials, the CTA that
// arrives last at a per-phase counter folds them in a fixed order, runs the
// solver's scalar recurrence (breakdown tests, alpha/beta/omega, convergence,
// iteration count, history) and writes the next state; the following kernel
// reads it.  Once `done` is set every later kernel returns immediately, so
// the host can queue whole graphs of iterations and poll the flag lazily.
//
// Algorithms and per-element roundings are those of the persistent kernels
// (cvk_krylov.cu): bicgstab krylov.cpp:57-138, tfqmr krylov.cpp:288-375.
#include <cuda_runtime.h>

#include <cstring>

#include "cvk_engine.cuh"
#include "cvk_kernels.h"
#include "cvk_phased.h"
#include "cvk_stream.cuh"

namespace cvk {

namespace {

#ifndef CVK_BATCH
#define CVK_BATCH 2  // gathers in flight per row: 1M DOF BiCGSTAB 142.5 (5) -> 138.4 us (2); FEM 293 -> 286
#endif
constexpr int kBatch = CVK_BATCH;  // (value, column) loads issued up front per row (thread per row)

struct PArgs {
    Csr A;
    const double2* dinv;
    const double2* b;
    double2* x;
    double2* work;
    double2* part;  // kMaxSlots x G per phase counter slot
    PState* st;
    double* hist;
    DevReport* rep;
    int capk;           // nnz capacity of a 256-row chunk (streamed kernels)
    int nst[5];         // ring depths of k_bi_a_s, k_bi_b_s, k_tf_e_s, k_tf_o_s, k_cg_a_s
    int pf_rows;        // StreamLayout::pf_rows (L2 prefetch of the forward gather band)
    int gprod[3];       // k_bf_*: grids of the producers of partial regions 0 (C / init), 1 (A), 2 (B)
    int gstride;        // k_bf_*: partial region stride = max grid
};

// ------------------------------------------------------------ tracing --
// CVK_TRACE builds (tools/variant_build.sh trace -DCVK_TRACE) record per-CTA
// globaltimer stamps of the phase kernels: [kernel][iteration % 16][cta][4]
// = entry (after the PDL wait), main loop done (CTA-wide), partial published,
// fold done (last CTA only).  Read with cvk_trace_read().
#ifdef CVK_TRACE
constexpr int kTrK = 4, kTrIt = 16, kTrCta = 1024;
__device__ unsigned long long g_trace[kTrK * kTrIt * kTrCta * 4];
__device__ __forceinline__ unsigned long long tr_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ unsigned long long g_sprof[kTrK * kTrCta * 4];
#define SPROF(kid) (g_sprof + ((size_t)(kid) * kTrCta + (blockIdx.x < kTrCta ? blockIdx.x : 0)) * 4)
#define TR(kid, it, slot) \
    do { if (threadIdx.x == 0 && blockIdx.x < kTrCta) \
        g_trace[((((kid) * kTrIt + ((it) % kTrIt)) * kTrCta) + blockIdx.x) * 4 + (slot)] = tr_now(); } while (0)
#else
#define TR(kid, it, slot) do { } while (0)
#define SPROF(kid) ((unsigned long long*)nullptr)
#endif

constexpr int kPhSlots = 12;  // partial slots per phase: hi + lo for up to 6 reductions

__device__ __forceinline__ double2* partv(const PArgs& a, int k) {
    return a.part + (size_t)k * kPhSlots * gridDim.x;
}

// Publish this CTA's K partials; returns true in the CTA that arrived last,
// with the grid totals in tot (valid in thread 0 -- callers continue with
// thread 0 only).
template <int K, int NT = kThreads>
__device__ bool partial_last(const CAcc (&acc)[K], double2* part, unsigned* counter,
                             double2 (&tot)[K], int kid = -1, long long it = 0) {
    __shared__ CAcc sm[K][32];
    __shared__ int s_last;
    const int G = gridDim.x;
    CAcc v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = acc[k];
    cta_sum_k<K, NT>(v, sm);
    if (kid >= 0) TR(kid, it, 1);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) cacc_store(part, k, G, blockIdx.x, v[k]);
        __threadfence();
        s_last = (atomicAdd(counter, 1u) == (unsigned)G - 1u);
    }
    __syncthreads();
    if (kid >= 0) TR(kid, it, 2);
    if (!s_last) return false;
    __threadfence();
    CAcc s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) s[k] = CAcc{};
#pragma unroll 1
    for (int b = threadIdx.x; b < G; b += NT) {
#pragma unroll
        for (int k = 0; k < K; ++k) cacc_add(s[k], cacc_load(part, k, G, b));
    }
    cta_sum_k<K, NT>(s, sm);
#pragma unroll
    for (int k = 0; k < K; ++k) tot[k] = s[k].hi;
    if (kid >= 0) TR(kid, it, 3);
    if (threadIdx.x == 0) *counter = 0u;
    return true;
}

// Grid-stride element loop with U elements per thread per trip; all loads of
// a trip are issued before its first store (the elementwise phases are
// latency-bound with one 16-byte load per vector in flight; tools/bicg_lab.cu
// phase C: 3.5 vs 2.0 TB/s at 1M DOF).  Launched on a grid of
// kElemCtasPerSm CTAs per SM.
#ifndef CVK_ELEM_BATCH
#define CVK_ELEM_BATCH 4
#endif
constexpr int kElemBatch = CVK_ELEM_BATCH;
template <int U, class LD, class STF>
__device__ __forceinline__ void for_elems_batched(int n, LD&& ld, STF&& stf) {
    using T = decltype(ld(0));
    const long long stride = (long long)gridDim.x * kThreads;
    for (long long base = (long long)blockIdx.x * kThreads + threadIdx.x; base < n; base += stride * U) {
        T v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = base + u * stride;
            if (i < n) v[u] = ld((int)i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = base + u * stride;
            if (i < n) stf((int)i, v[u]);
        }
    }
}

// Programmatic dependent launch: the successor kernel is launched while this
// one drains; it blocks here until this grid has completed and its memory is
// visible, so launch latency and CTA rasterisation overlap the tail.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void st_hist(const PArgs& a, PState* st, double v) {
    if (!st->record) return;
    if (st->hist_len < st->hist_cap) a.hist[st->hist_len] = v;
    st->hist_len++;
}

// ------------------------------------------------------------ BiCGSTAB --
// work: r, shadow, s, t, p[2], v[2]
struct BiVecs {
    double2 *r, *sh, *s, *t, *p0, *p1, *v0, *v1;
    __device__ BiVecs(double2* w, size_t n)
        : r(w), sh(w + n), s(w + 2 * n), t(w + 3 * n), p0(w + 4 * n), p1(w + 5 * n),
          v0(w + 6 * n), v1(w + 7 * n) {}
};

// top of iteration st->it (krylov.cpp:81-96), run by the last CTA
__device__ void bi_top(PState* st) {
    if (st->it > st->max_iter) { st->done = 1; return; }
    if (cvk_abs(st->rho_new) < st->brk) {
        st->done = 1; st->brk_code = 1; st->iters = st->it - 1;
        return;
    }
    if (!st->first) st->beta = cvk_mul(cvk_cdiv(st->rho_new, st->rho), cvk_cdiv(st->alpha, st->omega));
    st->rho = st->rho_new;
}

__global__ void __launch_bounds__(kThreads) k_bi_init(PArgs a) {
    pdl_enter();
    const int n = a.A.n;
    BiVecs V(a.work, (size_t)n);
    CAcc acc[2] = {};
    if (a.st->warm) {  // r = M^-1 (b - A x0), bnorm = ||M^-1 b|| (cvk_krylov.cu bicgstab_body)
        const double2* __restrict__ x = a.x;
        auto xat = [&](int c) -> double2 { return x[c]; };
        for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
            const double2 y = row_sum<1, decltype(xat)&, kBatch>(a.A, row, 0, valid, xat);
            if (valid) {
                const double2 bi = __ldg(a.b + row);
                const double2 ri = prec_apply(a.dinv, row, cvk_sub(bi, y));
                V.r[row] = ri;
                V.sh[row] = ri;
                acc_norm(acc[0], prec_apply(a.dinv, row, bi));
                acc_dot(acc[1], ri, ri);
            }
        });
    } else {
        for_elems(n, gridDim.x, blockIdx.x, [&](int i) {
            const double2 ri = prec_apply(a.dinv, i, __ldg(a.b + i));
            V.r[i] = ri;
            V.sh[i] = ri;
            a.x[i] = make_double2(0.0, 0.0);
            acc_norm(acc[0], ri);
            acc_dot(acc[1], ri, ri);
        });
    }
    double2 tot[2];
    if (!partial_last<2>(acc, partv(a, 0), &a.st->counter[0], tot)) return;
    if (threadIdx.x != 0) return;
    PState* st = a.st;
    st->bnorm = sqrt(tot[0].x);
    if (st->bnorm == 0.0) {  // krylov.cpp:70-74
        st->done = 1; st->conv = 1; st->iters = 0; st->skip_true = 1;
        return;
    }
    st->brk = 1e-30 * st->bnorm * st->bnorm;
    st->rho_new = tot[1];
    st->rho = st->alpha = st->omega = make_double2(1.0, 0.0);
    st->it = 1;
    st->first = 1;
    st->cur = 0;
    bi_top(st);
}

__global__ void __launch_bounds__(kThreads) k_bi_a(PArgs a) {
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n;
    BiVecs V(a.work, (size_t)n);
    const int cur = st->cur;
    const bool first = st->first != 0;
    const double2 beta = st->beta, nom = cvk_neg(st->omega);
    const double2* __restrict__ r = V.r;
    const double2* __restrict__ pc = cur ? V.p1 : V.p0;
    const double2* __restrict__ vc = cur ? V.v1 : V.v0;
    double2* __restrict__ pn = cur ? V.p0 : V.p1;
    double2* __restrict__ vn = cur ? V.v0 : V.v1;
    const double2* __restrict__ sh = V.sh;
    auto pnew = [&](int c) -> double2 {
        const double2 rc = r[c];
        if (first) return rc;
        return cvk_add(cvk_mul(beta, cvk_add(pc[c], cvk_mul(nom, vc[c]))), rc);
    };
    CAcc acc[1] = {};
    for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
        const double2 y = row_sum<1, decltype(pnew)&, kBatch>(a.A, row, 0, valid, pnew);
        if (valid) {
            const double2 vi = prec_apply(a.dinv, row, y);
            pn[row] = pnew(row);
            vn[row] = vi;
            acc_dot(acc[0], sh[row], vi);
        }
    });
    double2 tot[1];
    if (!partial_last<1>(acc, partv(a, 1), &st->counter[1], tot)) return;
    if (threadIdx.x != 0) return;
    if (cvk_abs(tot[0]) < st->brk) {
        st->done = 1; st->brk_code = 2; st->iters = st->it - 1;
        return;
    }
    st->alpha = cvk_cdiv(st->rho, tot[0]);
}

__global__ void __launch_bounds__(kThreads) k_bi_b(PArgs a) {
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n;
    BiVecs V(a.work, (size_t)n);
    const int cur = st->cur;
    const double2 alpha = st->alpha, nal = cvk_neg(st->alpha);
    const double2* __restrict__ r = V.r;
    const double2* __restrict__ pn = cur ? V.p0 : V.p1;
    const double2* __restrict__ vn = cur ? V.v0 : V.v1;
    double2* __restrict__ s = V.s;
    double2* __restrict__ t = V.t;
    double2* __restrict__ x = a.x;
    auto sval = [&](int c) -> double2 { return cvk_add(r[c], cvk_mul(nal, vn[c])); };
    CAcc acc[3] = {};
    for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
        const double2 y = row_sum<1, decltype(sval)&, kBatch>(a.A, row, 0, valid, sval);
        if (valid) {
            const double2 ti = prec_apply(a.dinv, row, y);
            const double2 si = sval(row);
            s[row] = si;
            t[row] = ti;
            x[row] = cvk_add(x[row], cvk_mul(alpha, pn[row]));
            acc_norm(acc[0], si);
            acc_dot(acc[1], ti, ti);
            acc_dot(acc[2], ti, si);
        }
    });
    double2 tot[3];
    if (!partial_last<3>(acc, partv(a, 2), &st->counter[2], tot)) return;
    if (threadIdx.x != 0) return;
    const double relres = sqrt(tot[0].x) / st->bnorm;
    if (relres <= st->tol) {
        st->done = 1; st->conv = 1; st->iters = st->it; st->final_relres = relres;
        st_hist(a, st, relres);
        return;
    }
    if (cvk_abs(tot[1]) < st->brk) {
        st->done = 1; st->brk_code = 3; st->iters = st->it;
        return;
    }
    st->omega = cvk_cdiv(tot[2], tot[1]);
}

__global__ void __launch_bounds__(kThreads) k_bi_c(PArgs a) {
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    TR(0, st->it, 0);
    const int n = a.A.n;
    BiVecs V(a.work, (size_t)n);
    const double2 omega = st->omega, nom = cvk_neg(st->omega);
    CAcc acc[2] = {};
    const double2* __restrict__ s = V.s;
    const double2* __restrict__ t = V.t;
    const double2* __restrict__ sh = V.sh;
    double2* __restrict__ r = V.r;
    double2* __restrict__ x = a.x;
    struct L4 { double2 s, t, sh, x; };
    for_elems_batched<kElemBatch>(
        n, [&](int i) { return L4{s[i], t[i], sh[i], x[i]}; },
        [&](int i, const L4& v) {
            x[i] = cvk_add(v.x, cvk_mul(omega, v.s));
            const double2 ri = cvk_add(v.s, cvk_mul(nom, v.t));
            r[i] = ri;
            acc_norm(acc[0], ri);
            acc_dot(acc[1], v.sh, ri);
        });
    double2 tot[2];
    if (!partial_last<2>(acc, partv(a, 0), &st->counter[0], tot, 0, st->it)) return;
    if (threadIdx.x != 0) return;
    const double relres = sqrt(tot[0].x) / st->bnorm;
    st->final_relres = relres;
    st->iters = st->it;
    st_hist(a, st, relres);
    if (relres <= st->tol) { st->done = 1; st->conv = 1; return; }
    st->rho_new = tot[1];
    st->cur ^= 1;
    st->first = 0;
    st->it++;
    bi_top(st);
}

// ---------------------------------------------------------------- COCG --
// Beyond the reference (cvk_krylov.cu cocg_body, oracle orc_cocg).  Two
// launches per iteration: the SpMV phase (p = z + beta p formed in the
// gathers, q = A p, mu = p^T q) and the elementwise phase (x, r, z updates,
// ||z||^2 and r^T z).  work: r, z, q, p[2]
struct CgVecs {
    double2 *r, *z, *q, *p0, *p1;
    __device__ CgVecs(double2* w, size_t n) : r(w), z(w + n), q(w + 2 * n), p0(w + 3 * n), p1(w + 4 * n) {}
};

// top of iteration st->it: max_iter, rho breakdown, beta (orc_cocg order)
__device__ void cg_top(PState* st) {
    if (st->it > st->max_iter) { st->done = 1; return; }
    if (cvk_abs(st->rho_new) < st->brk) {
        st->done = 1; st->brk_code = 1; st->iters = st->it - 1;
        return;
    }
    if (!st->first) st->beta = cvk_cdiv(st->rho_new, st->rho);
    st->rho = st->rho_new;
}

__global__ void __launch_bounds__(kThreads) k_cg_init(PArgs a) {
    pdl_enter();
    const int n = a.A.n;
    CgVecs V(a.work, (size_t)n);
    CAcc acc[2] = {};
    for_elems(n, gridDim.x, blockIdx.x, [&](int i) {
        const double2 ri = __ldg(a.b + i);
        const double2 zi = prec_apply(a.dinv, i, ri);
        V.r[i] = ri;
        V.z[i] = zi;
        a.x[i] = make_double2(0.0, 0.0);
        acc_norm(acc[0], zi);
        acc_udot(acc[1], ri, zi);
    });
    double2 tot[2];
    if (!partial_last<2>(acc, partv(a, 0), &a.st->counter[0], tot)) return;
    if (threadIdx.x != 0) return;
    PState* st = a.st;
    st->bnorm = sqrt(tot[0].x);
    if (st->bnorm == 0.0) {
        st->done = 1; st->conv = 1; st->iters = 0; st->skip_true = 1;
        return;
    }
    st->brk = 1e-30 * st->bnorm * st->bnorm;
    st->rho_new = tot[1];
    st->it = 1;
    st->first = 1;
    st->cur = 0;
    cg_top(st);
}

// mu breakdown / alpha, last CTA of the SpMV phase
__device__ __forceinline__ void cg_alpha(PState* st, double2 mu) {
    if (cvk_abs(mu) < st->brk) {
        st->done = 1; st->brk_code = 8; st->iters = st->it - 1;
        return;
    }
    st->alpha = cvk_cdiv(st->rho, mu);
}

__global__ void __launch_bounds__(kThreads) k_cg_a(PArgs a) {
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n;
    CgVecs V(a.work, (size_t)n);
    const bool first = st->first != 0;
    const double2 beta = st->beta;
    const double2* __restrict__ z = V.z;
    const double2* __restrict__ pc = st->cur ? V.p1 : V.p0;
    double2* __restrict__ pn = st->cur ? V.p0 : V.p1;
    auto pnew = [&](int c) -> double2 { return first ? z[c] : cvk_add(cvk_mul(beta, pc[c]), z[c]); };
    CAcc acc[1] = {};
    for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
        const double2 y = row_sum<1, decltype(pnew)&, kBatch>(a.A, row, 0, valid, pnew);
        if (valid) {
            const double2 pi = pnew(row);
            pn[row] = pi;
            V.q[row] = y;
            acc_udot(acc[0], pi, y);
        }
    });
    double2 tot[1];
    if (!partial_last<1>(acc, partv(a, 1), &st->counter[1], tot)) return;
    if (threadIdx.x != 0) return;
    cg_alpha(st, tot[0]);
}

__global__ void __launch_bounds__(kThreads) k_cg_b(PArgs a) {
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n;
    CgVecs V(a.work, (size_t)n);
    const double2 alpha = st->alpha, nal = cvk_neg(st->alpha);
    const double2* __restrict__ pn = st->cur ? V.p0 : V.p1;
    const double2* __restrict__ q = V.q;
    double2* __restrict__ r = V.r;
    double2* __restrict__ z = V.z;
    double2* __restrict__ x = a.x;
    const double2* __restrict__ dinv = a.dinv;
    struct L5 { double2 x, p, r, q, d; };
    CAcc acc[2] = {};
    for_elems_batched<kElemBatch>(
        n, [&](int i) { return L5{x[i], pn[i], r[i], q[i], dinv ? __ldg(dinv + i) : make_double2(1.0, 0.0)}; },
        [&](int i, const L5& v) {
            x[i] = cvk_add(v.x, cvk_mul(alpha, v.p));
            const double2 ri = cvk_add(v.r, cvk_mul(nal, v.q));
            const double2 zi = dinv ? cvk_mul(v.d, ri) : ri;
            r[i] = ri;
            z[i] = zi;
            acc_norm(acc[0], zi);
            acc_udot(acc[1], ri, zi);
        });
    double2 tot[2];
    if (!partial_last<2>(acc, partv(a, 2), &st->counter[2], tot)) return;
    if (threadIdx.x != 0) return;
    const double relres = sqrt(tot[0].x) / st->bnorm;
    st->final_relres = relres;
    st->iters = st->it;
    st_hist(a, st, relres);
    if (relres <= st->tol) { st->done = 1; st->conv = 1; return; }
    st->rho_new = tot[1];
    st->cur ^= 1;
    st->first = 0;
    st->it++;
    cg_top(st);
}

// --------------------------------------------------------------- tfQMR --
// work: r, shadow, w, u[2], au, v, d
struct TfVecs {
    double2 *r, *sh, *w, *u0, *u1, *au, *v, *d;
    __device__ TfVecs(double2* wk, size_t n)
        : r(wk), sh(wk + n), w(wk + 2 * n), u0(wk + 3 * n), u1(wk + 4 * n), au(wk + 5 * n),
          v(wk + 6 * n), d(wk + 7 * n) {}
};

// even half-step head (krylov.cpp:319-326), run by the last CTA after sigma
__device__ void tf_even_head(PState* st, double2 sigma) {
    if (st->it > st->max_iter) { st->done = 1; return; }
    if (cvk_abs(sigma) < st->brk) { st->done = 1; st->brk_code = 6; return; }
    st->alpha = cvk_cdiv(st->rho, sigma);
}

__global__ void __launch_bounds__(kThreads) k_tf_init(PArgs a) {
    pdl_enter();
    const int n = a.A.n;
    TfVecs V(a.work, (size_t)n);
    CAcc acc[2] = {};
    for_elems(n, gridDim.x, blockIdx.x, [&](int i) {
        const double2 ri = prec_apply(a.dinv, i, __ldg(a.b + i));
        V.r[i] = ri; V.sh[i] = ri; V.w[i] = ri; V.u0[i] = ri;
        V.d[i] = make_double2(0, 0);
        a.x[i] = make_double2(0, 0);
        acc_norm(acc[0], ri);
        acc_dot(acc[1], ri, ri);
    });
    double2 tot[2];
    if (!partial_last<2>(acc, partv(a, 0), &a.st->counter[0], tot)) return;
    if (threadIdx.x != 0) return;
    PState* st = a.st;
    st->bnorm = sqrt(tot[0].x);
    if (st->bnorm == 0.0) { st->done = 1; st->conv = 1; st->iters = 0; st->skip_true = 1; return; }
    st->brk = 1e-30 * st->bnorm * st->bnorm;
    st->rho = tot[1];
    st->tau = st->bnorm;
    st->theta = 0.0;
    st->eta = make_double2(0, 0);
    st->alpha = make_double2(0, 0);
    st->it = 1;  // even half-step index = 2 (it - 1)
    st->cur = 0;
}

// au = M^{-1} A u0, v = au, sigma = <shadow, v>
__global__ void __launch_bounds__(kThreads) k_tf_init2(PArgs a) {
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n;
    TfVecs V(a.work, (size_t)n);
    const double2* __restrict__ u0 = V.u0;
    auto uat = [&](int c) -> double2 { return u0[c]; };
    CAcc acc[1] = {};
    for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
        const double2 y = row_sum<1, decltype(uat)&, kBatch>(a.A, row, 0, valid, uat);
        if (valid) {
            const double2 ai = prec_apply(a.dinv, row, y);
            V.au[row] = ai;
            V.v[row] = ai;
            acc_dot(acc[0], V.sh[row], ai);
        }
    });
    double2 tot[1];
    if (!partial_last<1>(acc, partv(a, 1), &st->counter[1], tot)) return;
    if (threadIdx.x != 0) return;
    tf_even_head(st, tot[0]);
}

// even half-step body: w -= alpha au; d = coef d + u; ||w||
__global__ void __launch_bounds__(kThreads) k_tf_w(PArgs a) {
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n;
    TfVecs V(a.work, (size_t)n);
    const double2 nal = cvk_neg(st->alpha);
    const double2 coef = cvk_cdiv(cvk_scale(st->theta * st->theta, st->eta), st->alpha);
    const double2* __restrict__ uc = st->cur ? V.u1 : V.u0;
    CAcc acc[1] = {};
    struct L4 { double2 w, au, d, u; };
    for_elems_batched<kElemBatch>(
        n, [&](int i) { return L4{V.w[i], V.au[i], V.d[i], uc[i]}; },
        [&](int i, const L4& v) {
            const double2 wi = cvk_add(v.w, cvk_mul(nal, v.au));
            V.w[i] = wi;
            V.d[i] = cvk_add(cvk_mul(coef, v.d), v.u);
            acc_norm(acc[0], wi);
        });
    double2 tot[1];
    if (!partial_last<1>(acc, partv(a, 2), &st->counter[2], tot)) return;
    if (threadIdx.x != 0) return;
    st->theta = sqrt(tot[0].x) / st->tau;
    const double c = 1.0 / sqrt(1.0 + st->theta * st->theta);
    st->tau = st->tau * st->theta * c;
    st->eta = cvk_scale(c * c, st->alpha);
    st->pending_x = 1;
    const long long hs = 2 * (st->it - 1);
    const double relres = st->tau * sqrt((double)(hs + 2)) / st->bnorm;
    st->final_relres = relres;
    st->iters = hs / 2 + 1;
    if (relres <= st->tol) { st->done = 1; st->conv = 1; }
}

// even tail + odd head: u' = u - alpha v; au = M^{-1} A u'; x += eta d;
// w -= alpha au; d = coef d + u'; ||w||, <shadow, w>
__global__ void __launch_bounds__(kThreads) k_tf_e(PArgs a) {
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n;
    TfVecs V(a.work, (size_t)n);
    const double2 nal = cvk_neg(st->alpha);
    const double2 eta_e = st->eta;
    const double2 coef = cvk_cdiv(cvk_scale(st->theta * st->theta, st->eta), st->alpha);
    const double2* __restrict__ uc = st->cur ? V.u1 : V.u0;
    double2* __restrict__ un = st->cur ? V.u0 : V.u1;
    const double2* __restrict__ vv = V.v;
    auto uval = [&](int c) -> double2 { return cvk_add(uc[c], cvk_mul(nal, vv[c])); };
    CAcc acc[2] = {};
    for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
        const double2 y = row_sum<1, decltype(uval)&, kBatch>(a.A, row, 0, valid, uval);
        if (valid) {
            const double2 ui = uval(row);
            const double2 ai = prec_apply(a.dinv, row, y);
            un[row] = ui;
            V.au[row] = ai;
            const double2 di = V.d[row];
            a.x[row] = cvk_add(a.x[row], cvk_mul(eta_e, di));
            const double2 wi = cvk_add(V.w[row], cvk_mul(nal, ai));
            V.w[row] = wi;
            V.d[row] = cvk_add(cvk_mul(coef, di), ui);
            acc_norm(acc[0], wi);
            acc_dot(acc[1], V.sh[row], wi);
        }
    });
    double2 tot[2];
    if (!partial_last<2>(acc, partv(a, 0), &st->counter[0], tot)) return;
    if (threadIdx.x != 0) return;
    st->cur ^= 1;
    st->theta = sqrt(tot[0].x) / st->tau;
    const double c = 1.0 / sqrt(1.0 + st->theta * st->theta);
    st->tau = st->tau * st->theta * c;
    st->eta = cvk_scale(c * c, st->alpha);
    st->pending_x = 1;
    const long long hs = 2 * (st->it - 1) + 1;
    const double relres = st->tau * sqrt((double)(hs + 2)) / st->bnorm;
    st->final_relres = relres;
    st->iters = hs / 2 + 1;
    st_hist(a, st, relres);
    if (relres <= st->tol) { st->done = 1; st->conv = 1; return; }
    if (cvk_abs(st->rho) < st->brk) { st->done = 1; st->brk_code = 1; return; }
    st->beta = cvk_cdiv(tot[1], st->rho);
    st->rho = tot[1];
}

// odd tail: u_next = w + beta u; au_next = M^{-1} A u_next;
// v = beta (beta v + au) + au_next; x += eta d; sigma = <shadow, v>
__global__ void __launch_bounds__(kThreads) k_tf_o(PArgs a) {
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n;
    TfVecs V(a.work, (size_t)n);
    const double2 beta = st->beta, eta_o = st->eta;
    const double2* __restrict__ uc = st->cur ? V.u1 : V.u0;
    double2* __restrict__ un = st->cur ? V.u0 : V.u1;
    const double2* __restrict__ w = V.w;
    auto unext = [&](int c) -> double2 { return cvk_add(w[c], cvk_mul(beta, uc[c])); };
    CAcc acc[1] = {};
    for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
        const double2 y = row_sum<1, decltype(unext)&, kBatch>(a.A, row, 0, valid, unext);
        if (valid) {
            const double2 un_i = unext(row);
            const double2 an = prec_apply(a.dinv, row, y);
            un[row] = un_i;
            double2 vi = cvk_add(cvk_mul(beta, V.v[row]), V.au[row]);
            vi = cvk_add(cvk_mul(beta, vi), an);
            V.v[row] = vi;
            V.au[row] = an;
            a.x[row] = cvk_add(a.x[row], cvk_mul(eta_o, V.d[row]));
            acc_dot(acc[0], V.sh[row], vi);
        }
    });
    double2 tot[1];
    if (!partial_last<1>(acc, partv(a, 1), &st->counter[1], tot)) return;
    if (threadIdx.x != 0) return;
    st->pending_x = 0;
    st->cur ^= 1;
    st->it++;
    tf_even_head(st, tot[0]);
}

// owed x += eta d after a tfQMR exit (krylov.cpp:335)
__global__ void __launch_bounds__(kThreads) k_tf_fix(PArgs a) {
    pdl_enter();
    PState* st = a.st;
    if (!st->pending_x) return;
    TfVecs V(a.work, (size_t)a.A.n);
    const double2 e = st->eta;
    for_elems(a.A.n, gridDim.x, blockIdx.x, [&](int i) { a.x[i] = cvk_add(a.x[i], cvk_mul(e, V.d[i])); });
}

// ----------------------------------------------- streamed (TMA) variants --
// The SpMV phases of BiCGSTAB and tfQMR on the producer/consumer ring of
// cvk_stream.cuh: same per-element arithmetic and per-row accumulation order
// as the thread-per-row kernels above, one CTA per SM.

// Pre-hook switch (CVK_PRE_HOOK): with it, each chunk row's gathered
// combination is formed once into shared memory behind a group barrier;
// without it, every in-chunk gather forms it from the staged vectors.
#ifndef CVK_PRE_HOOK
#define CVK_PRE_HOOK 1
#endif
constexpr bool kPreHook = CVK_PRE_HOOK != 0;
template <bool ON, class F>
__device__ __forceinline__ auto PreIf(F&& f) {
    if constexpr (ON) return f;
    else return NoPre();
}

__device__ __forceinline__ double2 prec_staged(const PArgs& a, const Chunk& ch, int j, int t, double2 y) {
    return a.dinv ? cvk_mul(ch.v(j, t), y) : y;
}

__global__ void __launch_bounds__(kStreamThreads, 1) k_bi_a_s(PArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    TR(1, st->it, 0);
    const int n = a.A.n;
    BiVecs V(a.work, (size_t)n);
    const int cur = st->cur;
    const bool first = st->first != 0;
    const double2 beta = st->beta, nom = cvk_neg(st->omega);
    const double2* __restrict__ r = V.r;
    const double2* __restrict__ pc = cur ? V.p1 : V.p0;
    const double2* __restrict__ vc = cur ? V.v1 : V.v0;
    double2* __restrict__ pn = cur ? V.p0 : V.p1;
    double2* __restrict__ vn = cur ? V.v0 : V.v1;
    const double2* vecs[5] = {r, pc, vc, V.sh, a.dinv};
    StreamLayout L{a.capk, 5, a.nst[0]};
    L.ngather = 3;
    L.pf_rows = a.pf_rows;
    CAcc acc[1] = {};
    stream_rows(a.A, L, vecs, smem, [&](int t, const Chunk& ch) {
        // slot 0 of the chunk rows holds p_new (pre); band slots hold raw r, p, v
        auto xs = [&](int l) -> double2 {
            const double2 rc = ch.v(0, l);
            if (first || (kPreHook && l < kStreamRows)) return rc;
            return cvk_add(cvk_mul(beta, cvk_add(ch.v(1, l), cvk_mul(nom, ch.v(2, l)))), rc);
        };
        auto xg = [&](int c) -> double2 {
            const double2 rc = r[c];
            if (first) return rc;
            return cvk_add(cvk_mul(beta, cvk_add(pc[c], cvk_mul(nom, vc[c]))), rc);
        };
        const double2 y = chunk_row_sum<kBatch>(ch, t, xs, xg);
        const double2 vi = prec_staged(a, ch, 4, t, y);
        const int row = ch.r0 + t;
        pn[row] = xs(t);
        vn[row] = vi;
        acc_dot(acc[0], ch.v(3, t), vi);
    }, SPROF(1), PreIf<kPreHook>([&](int t, const Chunk& ch) {
        if (!first)
            ch.set(0, t, cvk_add(cvk_mul(beta, cvk_add(ch.v(1, t), cvk_mul(nom, ch.v(2, t)))), ch.v(0, t)));
    }));
    double2 tot[1];
    if (!partial_last<1, kStreamThreads>(acc, partv(a, 1), &st->counter[1], tot, 1, st->it)) return;
    if (threadIdx.x != 0) return;
    if (cvk_abs(tot[0]) < st->brk) {
        st->done = 1; st->brk_code = 2; st->iters = st->it - 1;
        return;
    }
    st->alpha = cvk_cdiv(st->rho, tot[0]);
}

__global__ void __launch_bounds__(kStreamThreads, 1) k_bi_b_s(PArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    TR(2, st->it, 0);
    const int n = a.A.n;
    BiVecs V(a.work, (size_t)n);
    const int cur = st->cur;
    const double2 alpha = st->alpha, nal = cvk_neg(st->alpha);
    const double2* __restrict__ r = V.r;
    const double2* __restrict__ pn = cur ? V.p0 : V.p1;
    const double2* __restrict__ vn = cur ? V.v0 : V.v1;
    double2* __restrict__ s = V.s;
    double2* __restrict__ t_ = V.t;
    double2* __restrict__ x = a.x;
    const double2* vecs[5] = {r, vn, a.dinv, pn, x};
    StreamLayout L{a.capk, 5, a.nst[1]};
    L.ngather = 2;
    L.pf_rows = a.pf_rows;
    CAcc acc[3] = {};
    stream_rows(a.A, L, vecs, smem, [&](int t, const Chunk& ch) {
        auto xs = [&](int l) -> double2 {  // slot 0 of the chunk rows holds s (pre)
            return (kPreHook && l < kStreamRows) ? ch.v(0, l) : cvk_add(ch.v(0, l), cvk_mul(nal, ch.v(1, l)));
        };
        auto xg = [&](int c) -> double2 { return cvk_add(r[c], cvk_mul(nal, vn[c])); };
        const double2 y = chunk_row_sum<kBatch>(ch, t, xs, xg);
        const double2 ti = prec_staged(a, ch, 2, t, y);
        const double2 si = xs(t);
        const int row = ch.r0 + t;
        s[row] = si;
        t_[row] = ti;
        x[row] = cvk_add(ch.v(4, t), cvk_mul(alpha, ch.v(3, t)));
        acc_norm(acc[0], si);
        acc_dot(acc[1], ti, ti);
        acc_dot(acc[2], ti, si);
    }, SPROF(2), PreIf<kPreHook>([&](int t, const Chunk& ch) {
        ch.set(0, t, cvk_add(ch.v(0, t), cvk_mul(nal, ch.v(1, t))));
    }));
    double2 tot[3];
    if (!partial_last<3, kStreamThreads>(acc, partv(a, 2), &st->counter[2], tot, 2, st->it)) return;
    if (threadIdx.x != 0) return;
    const double relres = sqrt(tot[0].x) / st->bnorm;
    if (relres <= st->tol) {
        st->done = 1; st->conv = 1; st->iters = st->it; st->final_relres = relres;
        st_hist(a, st, relres);
        return;
    }
    if (cvk_abs(tot[1]) < st->brk) {
        st->done = 1; st->brk_code = 3; st->iters = st->it;
        return;
    }
    st->omega = cvk_cdiv(tot[2], tot[1]);
}

// COCG SpMV phase (k_cg_a) on the ring: p = z + beta p formed once per chunk
// row in the pre-hook, q = A p, mu = p^T q
__global__ void __launch_bounds__(kStreamThreads, 1) k_cg_a_s(PArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n;
    CgVecs V(a.work, (size_t)n);
    const bool first = st->first != 0;
    const double2 beta = st->beta;
    const double2* __restrict__ z = V.z;
    const double2* __restrict__ pc = st->cur ? V.p1 : V.p0;
    double2* __restrict__ pn = st->cur ? V.p0 : V.p1;
    double2* __restrict__ q = V.q;
    const double2* vecs[2] = {z, first ? nullptr : pc};
    StreamLayout L{a.capk, 2, a.nst[4]};
    L.ngather = 2;
    L.pf_rows = a.pf_rows;
    CAcc acc[1] = {};
    stream_rows(a.A, L, vecs, smem, [&](int t, const Chunk& ch) {
        auto xs = [&](int l) -> double2 { return ch.v(0, l); };  // p (pre)
        auto xg = [&](int c) -> double2 { return first ? z[c] : cvk_add(cvk_mul(beta, pc[c]), z[c]); };
        const double2 y = chunk_row_sum<kBatch>(ch, t, xs, xg);
        const double2 pi = ch.v(0, t);
        const int row = ch.r0 + t;
        pn[row] = pi;
        q[row] = y;
        acc_udot(acc[0], pi, y);
    }, SPROF(1), [&](int t, const Chunk& ch) {
        if (!first) ch.set(0, t, cvk_add(cvk_mul(beta, ch.v(1, t)), ch.v(0, t)));
    });
    double2 tot[1];
    if (!partial_last<1, kStreamThreads>(acc, partv(a, 1), &st->counter[1], tot)) return;
    if (threadIdx.x != 0) return;
    cg_alpha(st, tot[0]);
}

// even tail + odd head of tfQMR (k_tf_e) on the ring
__global__ void __launch_bounds__(kStreamThreads, 1) k_tf_e_s(PArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n;
    TfVecs V(a.work, (size_t)n);
    const double2 nal = cvk_neg(st->alpha);
    const double2 eta_e = st->eta;
    const double2 coef = cvk_cdiv(cvk_scale(st->theta * st->theta, st->eta), st->alpha);
    const double2* __restrict__ uc = st->cur ? V.u1 : V.u0;
    double2* __restrict__ un = st->cur ? V.u0 : V.u1;
    const double2* __restrict__ vv = V.v;
    const double2* vecs[7] = {uc, vv, a.dinv, V.d, a.x, V.w, V.sh};
    StreamLayout L{a.capk, 7, a.nst[2]};
    L.ngather = 2;
    L.pf_rows = a.pf_rows;
    CAcc acc[2] = {};
    stream_rows(a.A, L, vecs, smem, [&](int t, const Chunk& ch) {
        auto xs = [&](int l) -> double2 {  // slot 0 of the chunk rows holds u - alpha v (pre)
            return l < kStreamRows ? ch.v(0, l) : cvk_add(ch.v(0, l), cvk_mul(nal, ch.v(1, l)));
        };
        auto xg = [&](int c) -> double2 { return cvk_add(uc[c], cvk_mul(nal, vv[c])); };
        const double2 y = chunk_row_sum<kBatch>(ch, t, xs, xg);
        const int row = ch.r0 + t;
        const double2 ui = xs(t);
        const double2 ai = prec_staged(a, ch, 2, t, y);
        un[row] = ui;
        V.au[row] = ai;
        const double2 di = ch.v(3, t);
        a.x[row] = cvk_add(ch.v(4, t), cvk_mul(eta_e, di));
        const double2 wi = cvk_add(ch.v(5, t), cvk_mul(nal, ai));
        V.w[row] = wi;
        V.d[row] = cvk_add(cvk_mul(coef, di), ui);
        acc_norm(acc[0], wi);
        acc_dot(acc[1], ch.v(6, t), wi);
    }, SPROF(3), [&](int t, const Chunk& ch) {
        ch.set(0, t, cvk_add(ch.v(0, t), cvk_mul(nal, ch.v(1, t))));
    });
    double2 tot[2];
    if (!partial_last<2, kStreamThreads>(acc, partv(a, 0), &st->counter[0], tot)) return;
    if (threadIdx.x != 0) return;
    st->cur ^= 1;
    st->theta = sqrt(tot[0].x) / st->tau;
    const double c = 1.0 / sqrt(1.0 + st->theta * st->theta);
    st->tau = st->tau * st->theta * c;
    st->eta = cvk_scale(c * c, st->alpha);
    st->pending_x = 1;
    const long long hs = 2 * (st->it - 1) + 1;
    const double relres = st->tau * sqrt((double)(hs + 2)) / st->bnorm;
    st->final_relres = relres;
    st->iters = hs / 2 + 1;
    st_hist(a, st, relres);
    if (relres <= st->tol) { st->done = 1; st->conv = 1; return; }
    if (cvk_abs(st->rho) < st->brk) { st->done = 1; st->brk_code = 1; return; }
    st->beta = cvk_cdiv(tot[1], st->rho);
    st->rho = tot[1];
}

// odd tail of tfQMR (k_tf_o) on the ring
__global__ void __launch_bounds__(kStreamThreads, 1) k_tf_o_s(PArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n;
    TfVecs V(a.work, (size_t)n);
    const double2 beta = st->beta, eta_o = st->eta;
    const double2* __restrict__ uc = st->cur ? V.u1 : V.u0;
    double2* __restrict__ un = st->cur ? V.u0 : V.u1;
    const double2* __restrict__ w = V.w;
    const double2* vecs[8] = {w, uc, a.dinv, V.v, V.au, a.x, V.d, V.sh};
    StreamLayout L{a.capk, 8, a.nst[3]};
    L.ngather = 2;
    L.pf_rows = a.pf_rows;
    CAcc acc[1] = {};
    stream_rows(a.A, L, vecs, smem, [&](int t, const Chunk& ch) {
        auto xs = [&](int l) -> double2 {  // slot 0 of the chunk rows holds w + beta u (pre)
            return l < kStreamRows ? ch.v(0, l) : cvk_add(ch.v(0, l), cvk_mul(beta, ch.v(1, l)));
        };
        auto xg = [&](int c) -> double2 { return cvk_add(w[c], cvk_mul(beta, uc[c])); };
        const double2 y = chunk_row_sum<kBatch>(ch, t, xs, xg);
        const int row = ch.r0 + t;
        const double2 un_i = xs(t);
        const double2 an = prec_staged(a, ch, 2, t, y);
        un[row] = un_i;
        double2 vi = cvk_add(cvk_mul(beta, ch.v(3, t)), ch.v(4, t));
        vi = cvk_add(cvk_mul(beta, vi), an);
        V.v[row] = vi;
        V.au[row] = an;
        a.x[row] = cvk_add(ch.v(5, t), cvk_mul(eta_o, ch.v(6, t)));
        acc_dot(acc[0], ch.v(7, t), vi);
    }, SPROF(3), [&](int t, const Chunk& ch) {
        ch.set(0, t, cvk_add(ch.v(0, t), cvk_mul(beta, ch.v(1, t))));
    });
    double2 tot[1];
    if (!partial_last<1, kStreamThreads>(acc, partv(a, 1), &st->counter[1], tot)) return;
    if (threadIdx.x != 0) return;
    st->pending_x = 0;
    st->cur ^= 1;
    st->it++;
    tf_even_head(st, tot[0]);
}

// ------------------------------- BiCGSTAB with consumer-folded reductions --
// The three streamed BiCGSTAB phases without a last-CTA fold: every CTA
// publishes its double-double partials and exits; the NEXT kernel's CTAs each
// fold them (one warp per reduction, fold_one) and run the scalar recurrence
// redundantly -- the same bits in every CTA, the same order of checks as the
// last-CTA kernels above -- so the fold leaves the critical path of the
// phase boundary, and the consumer's producer warp starts the ring while its
// consumer warps fold.  Scalars are double-buffered by launch parity
// (PState::scal[par] read, scal[par ^ 1] written by CTA 0); `done`,
// the report fields and the history are written by CTA 0 only, and a kernel
// that sets `done` processes no rows in any CTA.

__device__ __forceinline__ double2* bf_part(const PArgs& a, int region) {
    return a.part + (size_t)region * kPhSlots * a.gstride;
}

// CTA partials of K reductions into region (no arrival counting)
template <int K, int NT>
__device__ __forceinline__ void bf_publish(const CAcc (&acc)[K], const PArgs& a, int region) {
    __shared__ CAcc sm[K][32];
    CAcc v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = acc[k];
    cta_sum_k<K, NT>(v, sm);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) cacc_store(bf_part(a, region), k, a.gstride, blockIdx.x, v[k]);
}

// every CTA: fold K reductions of region -> tot (all threads).  The region's
// slots are laid out with stride gstride, and only its producer's gprod CTAs
// wrote partials: fold exactly those (the loads of four partials issued
// before their adds, then the fixed xor tree -- fold_one's order).
template <int K>
__device__ __forceinline__ void bf_fold(const PArgs& a, int region, double2 (&tot)[K]) {
    __shared__ double2 res[K];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = a.gprod[region], stride = a.gstride;
    const double2* part = bf_part(a, region);
    for (int k = warp; k < K; k += (int)(blockDim.x >> 5)) {
        CAcc sacc = {};
        for (int b0 = lane; b0 < g; b0 += 128) {
            CAcc v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = b0 + 32 * u < g ? cacc_load(part, k, stride, b0 + 32 * u) : CAcc{};
#pragma unroll
            for (int u = 0; u < 4; ++u) cacc_add(sacc, v[u]);
        }
        sacc = warp_sum(sacc);
        if (lane == 0) res[k] = sacc.hi;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) tot[k] = res[k];
}

__device__ __forceinline__ void bf_hist(const PArgs& a, PState* st, double v) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st_hist(a, st, v);
}

// A: evaluate the previous C (end of iteration it - 1) and the top of
// iteration it; then p = r + beta (p - omega v), v = M^-1 A p, <shadow, v>
__global__ void __launch_bounds__(kStreamThreads, 1) k_bf_a_s(PArgs a, int par) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    BiScal S = st->scal[par];
    TR(1, S.it + (S.first ? 0 : 1), 0);
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    if (!S.first) {
        double2 tot[2];
        bf_fold<2>(a, 0, tot);
        const double relres = sqrt(tot[0].x) / st->bnorm;  // krylov.cpp:124-132
        if (lead) { st->final_relres = relres; st->iters = S.it; }
        bf_hist(a, st, relres);
        if (relres <= st->tol) { if (lead) { st->done = 1; st->conv = 1; } return; }
        S.it++;
        S.cur ^= 1;
        // top of iteration S.it (krylov.cpp:81-96)
        if (S.it > st->max_iter) { if (lead) st->done = 1; return; }
        if (cvk_abs(tot[1]) < st->brk) {
            if (lead) { st->done = 1; st->brk_code = 1; st->iters = S.it - 1; }
            return;
        }
        S.beta = cvk_mul(cvk_cdiv(tot[1], S.rho), cvk_cdiv(S.alpha, S.omega));
        S.rho = tot[1];
    }
    const bool first = S.first != 0;
    if (lead) { BiScal W = S; W.first = 0; st->scal[par ^ 1] = W; }
    const int n = a.A.n;
    BiVecs V(a.work, (size_t)n);
    const int cur = S.cur;
    const double2 beta = S.beta, nom = cvk_neg(S.omega);
    const double2* __restrict__ r = V.r;
    const double2* __restrict__ pc = cur ? V.p1 : V.p0;
    const double2* __restrict__ vc = cur ? V.v1 : V.v0;
    double2* __restrict__ pn = cur ? V.p0 : V.p1;
    double2* __restrict__ vn = cur ? V.v0 : V.v1;
    const double2* vecs[5] = {r, pc, vc, V.sh, a.dinv};
    StreamLayout L{a.capk, 5, a.nst[0]};
    L.ngather = 3;
    L.pf_rows = a.pf_rows;
    CAcc acc[1] = {};
    stream_rows(a.A, L, vecs, smem, [&](int t, const Chunk& ch) {
        auto xs = [&](int l) -> double2 {
            const double2 rc = ch.v(0, l);
            if (first || (kPreHook && l < kStreamRows)) return rc;
            return cvk_add(cvk_mul(beta, cvk_add(ch.v(1, l), cvk_mul(nom, ch.v(2, l)))), rc);
        };
        auto xg = [&](int c) -> double2 {
            const double2 rc = r[c];
            if (first) return rc;
            return cvk_add(cvk_mul(beta, cvk_add(pc[c], cvk_mul(nom, vc[c]))), rc);
        };
        const double2 y = chunk_row_sum<kBatch>(ch, t, xs, xg);
        const double2 vi = prec_staged(a, ch, 4, t, y);
        const int row = ch.r0 + t;
        pn[row] = xs(t);
        vn[row] = vi;
        acc_dot(acc[0], ch.v(3, t), vi);
    }, SPROF(1), PreIf<kPreHook>([&](int t, const Chunk& ch) {
        if (!first)
            ch.set(0, t, cvk_add(cvk_mul(beta, cvk_add(ch.v(1, t), cvk_mul(nom, ch.v(2, t)))), ch.v(0, t)));
    }));
    TR(1, S.it, 1);
    bf_publish<1, kStreamThreads>(acc, a, 1);
    TR(1, S.it, 2);
}

// B: alpha = rho / <shadow, v>; s = r - alpha v, t = M^-1 A s, x += alpha p;
// ||s||^2, <t,t>, <t,s>
__global__ void __launch_bounds__(kStreamThreads, 1) k_bf_b_s(PArgs a, int par) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    BiScal S = st->scal[par];
    TR(2, S.it, 0);
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    {
        double2 tot[1];
        bf_fold<1>(a, 1, tot);
        if (cvk_abs(tot[0]) < st->brk) {  // krylov.cpp:99-103
            if (lead) { st->done = 1; st->brk_code = 2; st->iters = S.it - 1; }
            return;
        }
        S.alpha = cvk_cdiv(S.rho, tot[0]);
    }
    if (lead) st->scal[par ^ 1] = S;
    const int n = a.A.n;
    BiVecs V(a.work, (size_t)n);
    const int cur = S.cur;
    const double2 alpha = S.alpha, nal = cvk_neg(S.alpha);
    const double2* __restrict__ r = V.r;
    const double2* __restrict__ pn = cur ? V.p0 : V.p1;
    const double2* __restrict__ vn = cur ? V.v0 : V.v1;
    double2* __restrict__ s = V.s;
    double2* __restrict__ t_ = V.t;
    double2* __restrict__ x = a.x;
    const double2* vecs[5] = {r, vn, a.dinv, pn, x};
    StreamLayout L{a.capk, 5, a.nst[1]};
    L.ngather = 2;
    L.pf_rows = a.pf_rows;
    CAcc acc[3] = {};
    stream_rows(a.A, L, vecs, smem, [&](int t, const Chunk& ch) {
        auto xs = [&](int l) -> double2 {
            return (kPreHook && l < kStreamRows) ? ch.v(0, l) : cvk_add(ch.v(0, l), cvk_mul(nal, ch.v(1, l)));
        };
        auto xg = [&](int c) -> double2 { return cvk_add(r[c], cvk_mul(nal, vn[c])); };
        const double2 y = chunk_row_sum<kBatch>(ch, t, xs, xg);
        const double2 ti = prec_staged(a, ch, 2, t, y);
        const double2 si = xs(t);
        const int row = ch.r0 + t;
        s[row] = si;
        t_[row] = ti;
        x[row] = cvk_add(ch.v(4, t), cvk_mul(alpha, ch.v(3, t)));
        acc_norm(acc[0], si);
        acc_dot(acc[1], ti, ti);
        acc_dot(acc[2], ti, si);
    }, SPROF(2), PreIf<kPreHook>([&](int t, const Chunk& ch) {
        ch.set(0, t, cvk_add(ch.v(0, t), cvk_mul(nal, ch.v(1, t))));
    }));
    TR(2, S.it, 1);
    bf_publish<3, kStreamThreads>(acc, a, 2);
    TR(2, S.it, 2);
}

// C: half-step exit / omega breakdown / omega; x += omega s, r = s - omega t;
// ||r||^2, <shadow, r>
#ifndef CVK_BFC_MINB
#define CVK_BFC_MINB 1
#endif
__global__ void __launch_bounds__(kThreads, CVK_BFC_MINB) k_bf_c(PArgs a, int par) {
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    BiScal S = st->scal[par];
    TR(0, S.it, 0);
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    {
        double2 tot[3];
        bf_fold<3>(a, 2, tot);
        const double relres = sqrt(tot[0].x) / st->bnorm;
        if (relres <= st->tol) {  // half-step exit (krylov.cpp:107-114)
            if (lead) { st->done = 1; st->conv = 1; st->iters = S.it; st->final_relres = relres; }
            bf_hist(a, st, relres);
            return;
        }
        if (cvk_abs(tot[1]) < st->brk) {  // krylov.cpp:117-121
            if (lead) { st->done = 1; st->brk_code = 3; st->iters = S.it; }
            return;
        }
        S.omega = cvk_cdiv(tot[2], tot[1]);
    }
    if (lead) st->scal[par ^ 1] = S;
    const int n = a.A.n;
    BiVecs V(a.work, (size_t)n);
    const double2 omega = S.omega, nom = cvk_neg(S.omega);
    CAcc acc[2] = {};
    const double2* __restrict__ s = V.s;
    const double2* __restrict__ t = V.t;
    const double2* __restrict__ sh = V.sh;
    double2* __restrict__ r = V.r;
    double2* __restrict__ x = a.x;
    struct L4 { double2 s, t, sh, x; };
    for_elems_batched<kElemBatch>(
        n, [&](int i) { return L4{s[i], t[i], sh[i], x[i]}; },
        [&](int i, const L4& v) {
            x[i] = cvk_add(v.x, cvk_mul(omega, v.s));
            const double2 ri = cvk_add(v.s, cvk_mul(nom, v.t));
            r[i] = ri;
            acc_norm(acc[0], ri);
            acc_dot(acc[1], v.sh, ri);
        });
    TR(0, S.it, 1);
    bf_publish<2, kThreads>(acc, a, 0);
    TR(0, S.it, 2);
}

// ------------------------------------ COCG with consumer-folded reductions --
// The k_bf_* pattern for COCG (two kernels per iteration, so A always runs
// with parity 0 and B with parity 1): B's partials (||z||^2, r^T z) go to
// region 0 and are folded by the next A, A's (p^T q) to region 1, folded by
// B.  The checks run in the last-CTA kernels' order (k_cg_b's tail then
// cg_top at A, cg_alpha at B); k_bf_init seeds scal[0] from k_cg_init.

// A: evaluate the previous B and the top of iteration it (cg_top); then
// p = z + beta p, q = M^-1... (COCG: q = A p), mu = p^T q
__global__ void __launch_bounds__(kStreamThreads, 1) k_cf_a_s(PArgs a, int par) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    BiScal S = st->scal[par];
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    if (!S.first) {
        double2 tot[2];
        bf_fold<2>(a, 0, tot);
        const double relres = sqrt(tot[0].x) / st->bnorm;
        if (lead) { st->final_relres = relres; st->iters = S.it; }
        bf_hist(a, st, relres);
        if (relres <= st->tol) { if (lead) { st->done = 1; st->conv = 1; } return; }
        S.cur ^= 1;
        S.it++;
        // cg_top
        if (S.it > st->max_iter) { if (lead) st->done = 1; return; }
        if (cvk_abs(tot[1]) < st->brk) {
            if (lead) { st->done = 1; st->brk_code = 1; st->iters = S.it - 1; }
            return;
        }
        S.beta = cvk_cdiv(tot[1], S.rho);
        S.rho = tot[1];
    }
    const bool first = S.first != 0;
    if (lead) { BiScal W = S; W.first = 0; st->scal[par ^ 1] = W; }
    const int n = a.A.n;
    CgVecs V(a.work, (size_t)n);
    const double2 beta = S.beta;
    const double2* __restrict__ z = V.z;
    const double2* __restrict__ pc = S.cur ? V.p1 : V.p0;
    double2* __restrict__ pn = S.cur ? V.p0 : V.p1;
    double2* __restrict__ q = V.q;
    const double2* vecs[2] = {z, first ? nullptr : pc};
    StreamLayout L{a.capk, 2, a.nst[4]};
    L.ngather = 2;
    L.pf_rows = a.pf_rows;
    CAcc acc[1] = {};
    stream_rows(a.A, L, vecs, smem, [&](int t, const Chunk& ch) {
        auto xs = [&](int l) -> double2 { return ch.v(0, l); };  // p (pre)
        auto xg = [&](int c) -> double2 { return first ? z[c] : cvk_add(cvk_mul(beta, pc[c]), z[c]); };
        const double2 y = chunk_row_sum<kBatch>(ch, t, xs, xg);
        const double2 pi = ch.v(0, t);
        const int row = ch.r0 + t;
        pn[row] = pi;
        q[row] = y;
        acc_udot(acc[0], pi, y);
    }, SPROF(1), [&](int t, const Chunk& ch) {
        if (!first) ch.set(0, t, cvk_add(cvk_mul(beta, ch.v(1, t)), ch.v(0, t)));
    });
    bf_publish<1, kStreamThreads>(acc, a, 1);
}

// B: alpha = rho / mu (cg_alpha); x += alpha p, r -= alpha q, z = M^-1 r;
// ||z||^2, r^T z
__global__ void __launch_bounds__(kThreads) k_cf_b(PArgs a, int par) {
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    BiScal S = st->scal[par];
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    {
        double2 tot[1];
        bf_fold<1>(a, 1, tot);
        if (cvk_abs(tot[0]) < st->brk) {
            if (lead) { st->done = 1; st->brk_code = 8; st->iters = S.it - 1; }
            return;
        }
        S.alpha = cvk_cdiv(S.rho, tot[0]);
    }
    if (lead) st->scal[par ^ 1] = S;
    const int n = a.A.n;
    CgVecs V(a.work, (size_t)n);
    const double2 alpha = S.alpha, nal = cvk_neg(S.alpha);
    // S.cur is A's (A flipped it before its SpMV): A wrote the new p into pn
    const double2* __restrict__ pn = S.cur ? V.p0 : V.p1;
    const double2* __restrict__ q = V.q;
    double2* __restrict__ r = V.r;
    double2* __restrict__ z = V.z;
    double2* __restrict__ x = a.x;
    const double2* __restrict__ dinv = a.dinv;
    struct L5 { double2 x, p, r, q, d; };
    CAcc acc[2] = {};
    for_elems_batched<kElemBatch>(
        n, [&](int i) { return L5{x[i], pn[i], r[i], q[i], dinv ? __ldg(dinv + i) : make_double2(1.0, 0.0)}; },
        [&](int i, const L5& v) {
            x[i] = cvk_add(v.x, cvk_mul(alpha, v.p));
            const double2 ri = cvk_add(v.r, cvk_mul(nal, v.q));
            const double2 zi = dinv ? cvk_mul(v.d, ri) : ri;
            r[i] = ri;
            z[i] = zi;
            acc_norm(acc[0], zi);
            acc_udot(acc[1], ri, zi);
        });
    bf_publish<2, kThreads>(acc, a, 0);
}

// ----------------------------------- tfQMR with consumer-folded reductions --
// The k_bf_* pattern for tfQMR (three launches per iteration: W elementwise,
// E and O on the ring).  W's partial (||w||^2) goes to region 0 and is
// folded by E, E's (||w||^2, <shadow, w>) to region 1 for O, O's (sigma) to
// region 2 for the next W; each consumer runs its producer's tail in the
// last-CTA kernels' order, and CTA 0 keeps pending_x / eta in the state for
// k_tf_fix.  k_tq_seed copies k_tf_init2's scalars into tscal[0].

__device__ __forceinline__ void tq_theta(TfScal& S, double ww) {
    S.theta = sqrt(ww) / S.tau;
    const double c = 1.0 / sqrt(1.0 + S.theta * S.theta);
    S.tau = S.tau * S.theta * c;
    S.eta = cvk_scale(c * c, S.alpha);
}

// W: the previous O's tail (cur, it, tf_even_head); w -= alpha au, d = coef d + u; ||w||^2
__global__ void __launch_bounds__(kThreads) k_tq_w(PArgs a, int par) {
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    TfScal S = st->tscal[par];
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    if (!S.first) {
        double2 tot[1];
        bf_fold<1>(a, 2, tot);
        if (lead) st->pending_x = 0;
        S.cur ^= 1;
        S.it++;
        if (S.it > st->max_iter) { if (lead) st->done = 1; return; }
        if (cvk_abs(tot[0]) < st->brk) { if (lead) { st->done = 1; st->brk_code = 6; } return; }
        S.alpha = cvk_cdiv(S.rho, tot[0]);
    }
    if (lead) { TfScal W = S; W.first = 0; st->tscal[par ^ 1] = W; }
    const int n = a.A.n;
    TfVecs V(a.work, (size_t)n);
    const double2 nal = cvk_neg(S.alpha);
    const double2 coef = cvk_cdiv(cvk_scale(S.theta * S.theta, S.eta), S.alpha);
    const double2* __restrict__ uc = S.cur ? V.u1 : V.u0;
    CAcc acc[1] = {};
    struct L4 { double2 w, au, d, u; };
    for_elems_batched<kElemBatch>(
        n, [&](int i) { return L4{V.w[i], V.au[i], V.d[i], uc[i]}; },
        [&](int i, const L4& v) {
            const double2 wi = cvk_add(v.w, cvk_mul(nal, v.au));
            V.w[i] = wi;
            V.d[i] = cvk_add(cvk_mul(coef, v.d), v.u);
            acc_norm(acc[0], wi);
        });
    bf_publish<1, kThreads>(acc, a, 0);
}

// E: W's tail (theta, tau, eta, the even residual estimate); then the even
// tail + odd head of k_tf_e_s
__global__ void __launch_bounds__(kStreamThreads, 1) k_tq_e_s(PArgs a, int par) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    TfScal S = st->tscal[par];
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    {
        double2 tot[1];
        bf_fold<1>(a, 0, tot);
        tq_theta(S, tot[0].x);
        const long long hs = 2 * (S.it - 1);
        const double relres = S.tau * sqrt((double)(hs + 2)) / st->bnorm;
        if (lead) { st->pending_x = 1; st->eta = S.eta; st->final_relres = relres; st->iters = hs / 2 + 1; }
        if (relres <= st->tol) { if (lead) { st->done = 1; st->conv = 1; } return; }
    }
    if (lead) st->tscal[par ^ 1] = S;
    const int n = a.A.n;
    TfVecs V(a.work, (size_t)n);
    const double2 nal = cvk_neg(S.alpha);
    const double2 eta_e = S.eta;
    const double2 coef = cvk_cdiv(cvk_scale(S.theta * S.theta, S.eta), S.alpha);
    const double2* __restrict__ uc = S.cur ? V.u1 : V.u0;
    double2* __restrict__ un = S.cur ? V.u0 : V.u1;
    const double2* __restrict__ vv = V.v;
    const double2* vecs[7] = {uc, vv, a.dinv, V.d, a.x, V.w, V.sh};
    StreamLayout L{a.capk, 7, a.nst[2]};
    L.ngather = 2;
    L.pf_rows = a.pf_rows;
    CAcc acc[2] = {};
    stream_rows(a.A, L, vecs, smem, [&](int t, const Chunk& ch) {
        auto xs = [&](int l) -> double2 {  // slot 0 of the chunk rows holds u - alpha v (pre)
            return l < kStreamRows ? ch.v(0, l) : cvk_add(ch.v(0, l), cvk_mul(nal, ch.v(1, l)));
        };
        auto xg = [&](int c) -> double2 { return cvk_add(uc[c], cvk_mul(nal, vv[c])); };
        const double2 y = chunk_row_sum<kBatch>(ch, t, xs, xg);
        const int row = ch.r0 + t;
        const double2 ui = xs(t);
        const double2 ai = prec_staged(a, ch, 2, t, y);
        un[row] = ui;
        V.au[row] = ai;
        const double2 di = ch.v(3, t);
        a.x[row] = cvk_add(ch.v(4, t), cvk_mul(eta_e, di));
        const double2 wi = cvk_add(ch.v(5, t), cvk_mul(nal, ai));
        V.w[row] = wi;
        V.d[row] = cvk_add(cvk_mul(coef, di), ui);
        acc_norm(acc[0], wi);
        acc_dot(acc[1], ch.v(6, t), wi);
    }, SPROF(3), [&](int t, const Chunk& ch) {
        ch.set(0, t, cvk_add(ch.v(0, t), cvk_mul(nal, ch.v(1, t))));
    });
    bf_publish<2, kStreamThreads>(acc, a, 1);
}

// O: E's tail (cur, theta, tau, eta, the odd residual estimate, rho, beta);
// then the odd tail of k_tf_o_s
__global__ void __launch_bounds__(kStreamThreads, 1) k_tq_o_s(PArgs a, int par) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter();
    PState* st = a.st;
    if (st->done) return;
    TfScal S = st->tscal[par];
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    {
        double2 tot[2];
        bf_fold<2>(a, 1, tot);
        S.cur ^= 1;
        tq_theta(S, tot[0].x);
        const long long hs = 2 * (S.it - 1) + 1;
        const double relres = S.tau * sqrt((double)(hs + 2)) / st->bnorm;
        if (lead) { st->pending_x = 1; st->eta = S.eta; st->final_relres = relres; st->iters = hs / 2 + 1; }
        bf_hist(a, st, relres);
        if (relres <= st->tol) { if (lead) { st->done = 1; st->conv = 1; } return; }
        if (cvk_abs(S.rho) < st->brk) { if (lead) { st->done = 1; st->brk_code = 1; } return; }
        S.beta = cvk_cdiv(tot[1], S.rho);
        S.rho = tot[1];
    }
    if (lead) st->tscal[par ^ 1] = S;
    const int n = a.A.n;
    TfVecs V(a.work, (size_t)n);
    const double2 beta = S.beta, eta_o = S.eta;
    const double2* __restrict__ uc = S.cur ? V.u1 : V.u0;
    double2* __restrict__ un = S.cur ? V.u0 : V.u1;
    const double2* __restrict__ w = V.w;
    const double2* vecs[8] = {w, uc, a.dinv, V.v, V.au, a.x, V.d, V.sh};
    StreamLayout L{a.capk, 8, a.nst[3]};
    L.ngather = 2;
    L.pf_rows = a.pf_rows;
    CAcc acc[1] = {};
    stream_rows(a.A, L, vecs, smem, [&](int t, const Chunk& ch) {
        auto xs = [&](int l) -> double2 {  // slot 0 of the chunk rows holds w + beta u (pre)
            return l < kStreamRows ? ch.v(0, l) : cvk_add(ch.v(0, l), cvk_mul(beta, ch.v(1, l)));
        };
        auto xg = [&](int c) -> double2 { return cvk_add(w[c], cvk_mul(beta, uc[c])); };
        const double2 y = chunk_row_sum<kBatch>(ch, t, xs, xg);
        const int row = ch.r0 + t;
        const double2 un_i = xs(t);
        const double2 an = prec_staged(a, ch, 2, t, y);
        un[row] = un_i;
        double2 vi = cvk_add(cvk_mul(beta, ch.v(3, t)), ch.v(4, t));
        vi = cvk_add(cvk_mul(beta, vi), an);
        V.v[row] = vi;
        V.au[row] = an;
        a.x[row] = cvk_add(ch.v(5, t), cvk_mul(eta_o, ch.v(6, t)));
        acc_dot(acc[0], ch.v(7, t), vi);
    }, SPROF(3), [&](int t, const Chunk& ch) {
        ch.set(0, t, cvk_add(ch.v(0, t), cvk_mul(beta, ch.v(1, t))));
    });
    bf_publish<1, kStreamThreads>(acc, a, 2);
}

__global__ void k_tq_seed(PArgs a) {
    pdl_enter();
    PState* st = a.st;
    TfScal S;
    S.rho = st->rho;
    S.alpha = st->alpha;
    S.beta = st->beta;
    S.eta = st->eta;
    S.theta = st->theta;
    S.tau = st->tau;
    S.it = st->it;
    S.cur = st->cur;
    S.first = 1;
    st->tscal[0] = S;
}

// after k_bi_init (r0, shadow, x0, ||r0||, <r0, r0>, top of iteration 1):
// its scalars into scal[0] for the first k_bf_a_s
__global__ void k_bf_init(PArgs a) {
    pdl_enter();
    PState* st = a.st;
    BiScal S;
    S.rho = st->rho;
    S.alpha = st->alpha;
    S.omega = st->omega;
    S.beta = st->beta;
    S.it = st->it;
    S.first = st->first;
    S.cur = st->cur;
    st->scal[0] = S;
}

// ------------------------------------------------- true residual + report
__global__ void __launch_bounds__(kThreads) k_true(PArgs a, double2* scratch) {
    pdl_enter();
    PState* st = a.st;
    const int n = a.A.n;
    const double2* __restrict__ x = a.x;
    auto xat = [&](int c) -> double2 { return x[c]; };
    CAcc acc[2] = {};
    if (!st->skip_true) {
        for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
            const double2 y = row_sum<1, decltype(xat)&, kBatch>(a.A, row, 0, valid, xat);
            if (valid) {
                const double2 bi = __ldg(a.b + row);
                const double2 d = cvk_sub(bi, y);
                scratch[row] = d;
                acc_norm(acc[0], bi);
                acc_norm(acc[1], d);
            }
        });
    }
    double2 tot[2];
    if (!partial_last<2>(acc, partv(a, 2), &st->counter[3], tot)) return;
    if (threadIdx.x != 0) return;
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
    a.rep->history_len = st->hist_len;
    a.rep->error = 0;
}

PhasedKernels kernels_all() {
    PhasedKernels k;
    k.bi_init = (const void*)k_bi_init;
    k.bi_a = (const void*)k_bi_a;
    k.bi_b = (const void*)k_bi_b;
    k.bi_c = (const void*)k_bi_c;
    k.tf_init = (const void*)k_tf_init;
    k.tf_init2 = (const void*)k_tf_init2;
    k.tf_w = (const void*)k_tf_w;
    k.tf_e = (const void*)k_tf_e;
    k.tf_o = (const void*)k_tf_o;
    k.tf_fix = (const void*)k_tf_fix;
    k.true_res = (const void*)k_true;
    k.bi_a_s = (const void*)k_bi_a_s;
    k.bi_b_s = (const void*)k_bi_b_s;
    k.tf_e_s = (const void*)k_tf_e_s;
    k.tf_o_s = (const void*)k_tf_o_s;
    k.cg_init = (const void*)k_cg_init;
    k.cg_a = (const void*)k_cg_a;
    k.cg_b = (const void*)k_cg_b;
    k.cg_a_s = (const void*)k_cg_a_s;
    k.bf_a_s = (const void*)k_bf_a_s;
    k.bf_b_s = (const void*)k_bf_b_s;
    k.bf_c = (const void*)k_bf_c;
    k.bf_init = (const void*)k_bf_init;
    k.cf_a_s = (const void*)k_cf_a_s;
    k.cf_b = (const void*)k_cf_b;
    k.tq_w = (const void*)k_tq_w;
    k.tq_e_s = (const void*)k_tq_e_s;
    k.tq_o_s = (const void*)k_tq_o_s;
    k.tq_seed = (const void*)k_tq_seed;
    return k;
}

}  // namespace

PhasedKernels phased_kernels() { return kernels_all(); }

int phased_trace_read(void* out, size_t bytes) {
#ifdef CVK_TRACE
    // [g_trace | g_sprof]
    size_t n = sizeof(g_trace) < bytes ? sizeof(g_trace) : bytes;
    if (cudaMemcpyFromSymbol(out, g_trace, n) != cudaSuccess) return -1;
    if (bytes >= sizeof(g_trace) + sizeof(g_sprof)) {
        if (cudaMemcpyFromSymbol((char*)out + sizeof(g_trace), g_sprof, sizeof(g_sprof)) != cudaSuccess) return -1;
        n += sizeof(g_sprof);
    }
    return (int)n;
#else
    (void)out; (void)bytes;
    return 0;
#endif
}

size_t phased_args_size() { return sizeof(PArgs); }

// The consumer shape of this translation unit's ring.  cvk_phased_g4.cu
// compiles this file again (namespace cvk_g4) with 4 groups of 128 rows; the
// host picks a flavor per matrix through these plain-typed entry points.
int flavor_stream_rows() { return kStreamRows; }
int flavor_stream_threads() { return kStreamThreads; }
size_t flavor_stage_bytes(int capk, int nvec, int ngather) {
    StreamLayout L{capk, nvec, 1};
    L.ngather = ngather;
    return L.stage_bytes();
}
size_t flavor_smem_bytes(int capk, int nvec, int ngather, int stages) {
    StreamLayout L{capk, nvec, stages};
    L.ngather = ngather;
    return L.smem_bytes();
}
void flavor_kernels(void* out) {
    const PhasedKernels k = kernels_all();
    memcpy(out, &k, sizeof(k));
}
void flavor_pack_args(void* out, int n, const int* rp, const int* ci, const double2* av, const int* cmax,
                      const double2* dinv, const double2* b, double2* x, double2* work, double2* part, void* st,
                      double* hist, void* rep, int capk, const int* nst, int pf_rows, const int* gprod,
                      const double2* udg) {
    phased_pack_args(out, Csr{n, rp, ci, av, cmax, udg, udg ? udg + n : nullptr}, dinv, b, x, work, part,
                     (PState*)st, hist, (DevReport*)rep, capk, nst, pf_rows, gprod);
}

void phased_pack_args(void* out, const Csr& A, const double2* dinv, const double2* b, double2* x,
                      double2* work, double2* part, PState* st, double* hist, DevReport* rep,
                      int capk, const int* nst, int pf_rows, const int* gprod) {
    PArgs* p = (PArgs*)out;
    p->pf_rows = pf_rows;
    p->gstride = 0;
    for (int i = 0; i < 3; ++i) {
        p->gprod[i] = gprod ? gprod[i] : 0;
        p->gstride = p->gprod[i] > p->gstride ? p->gprod[i] : p->gstride;
    }
    p->capk = capk;
    for (int i = 0; i < 5; ++i) p->nst[i] = nst[i];
    p->A = A;
    p->dinv = dinv;
    p->b = b;
    p->x = x;
    p->work = work;
    p->part = part;
    p->st = st;
    p->hist = hist;
    p->rep = rep;
}

}  // namespace cvk
