// cvk_engine.cuh -- building blocks of the persistent Krylov kernels.
//
// One cooperative grid of G CTAs x 256 threads runs a whole solve.  Rows are
// owned in chunks of 256: CTA b owns chunks b, b+G, b+2G, ...  Element loops
// map chunk row i to thread i; SpMV loops walk the same chunk with S lanes
// per row in S sub-rounds, so both loop kinds touch the same rows per CTA and
// only a __syncthreads separates them.  Phases are separated by a grid
// barrier (monotone 64-bit arrival counter, acquire spin, globaltimer abort).
//
// Reductions are deterministic:
//  * FAST: each thread accumulates in grid-stride order, warps reduce by a
//    fixed xor tree, CTAs write one partial per slot, and after the barrier
//    EVERY CTA folds the G partials in the same fixed order -- all CTAs hold
//    bitwise identical scalars, so the redundant scalar recurrences on every
//    CTA agree without a broadcast phase.
//  * REF: after the barrier thread 0 of every CTA re-reads the vectors and
//    sums them left to right, exactly as dot_hermitian / norm2 do
//    (numkit.cpp:113-125).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "cvk_complex.h"

namespace cvk {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxDots = 64;                // GMRES(m): m <= kMaxDots
constexpr int kMaxSlots = 2 * kMaxDots + 4;  // partial slots per region (hi and lo per reduction)
constexpr int kRegions = 3;
constexpr int kMinCtas = 3;  // persistent solvers: <= 80 registers, 3 CTAs (24 warps) per SM

struct DevReport {
    int32_t converged;
    int32_t breakdown;
    int64_t iterations;
    double final_relres;
    double true_relres;
    int64_t history_len;
    int32_t error;
    int32_t pad;
};

struct Csr {
    int n;
    const int* __restrict__ rp;
    const int* __restrict__ ci;
    const double2* __restrict__ av;
    const int* cmax = nullptr;  // per streamed chunk: largest column index (L2 prefetch window), optional
    // Uniform off-diagonal values (streamed SpMV only, optional): when uni[0].x
    // != 0 every off-diagonal entry equals uni[1] bit for bit and dg holds the
    // diagonal, so a chunk streams 16 B of values per row instead of per
    // entry.  Checked on the device at the start of every solve (k_uniform_*).
    const double2* dg = nullptr;
    const double2* uni = nullptr;
};

// Kernel arguments (passed by value to cudaLaunchCooperativeKernel).
struct KArgs {
    Csr A;
    const double2* dinv;  // nullptr -> identity preconditioner
    const double2* b;
    double2* x;
    double2* work;        // nwork vectors of length n, contiguous
    double2* part;        // kRegions x kMaxSlots x G partials
    unsigned long long* bar;  // [0] arrival counter, [1] abort flag
    DevReport* rep;
    double* hist;
    long long hist_cap;
    double tol;
    long long max_iter;
    int l;
    int m;
    int record;
    int G;
    int cta_base;  // first CTA of this solve in a batched launch
    int warm;      // BiCGSTAB only: x holds x0 (r0 = M^-1 (b - A x0)); 0 = the reference's x0 = 0
    int refpar;    // REF reductions with parallel term formation (CVK_MODE_REF_PAR)
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Grid barrier over the G co-resident CTAs of a cooperative launch.
struct GridBar {
    unsigned long long* bar;
    unsigned long long target;
    unsigned G;

    int cta;  // CTA index within this grid (or within a batched segment)
    int refpar = 0;  // REF reductions: CTA 0 sums with all its threads forming the terms

    __device__ GridBar(unsigned long long* b, int g, int cta_ = -1)
        : bar(b), target(0), G((unsigned)g), cta(cta_ < 0 ? (int)blockIdx.x : cta_) {}

    // returns false if the barrier was aborted (timeout anywhere in the grid)
    __device__ bool sync() {
        __shared__ int s_ok;
        __syncthreads();
        target += G;
        if (threadIdx.x == 0) {
            int ok = 1;
            __threadfence();
            atomicAdd(bar, 1ull);
            const unsigned long long t0 = global_ns();
            unsigned spins = 0;
            while (ld_acquire_u64(bar) < target) {
                if ((++spins & 1023u) == 0) {
                    if (*((volatile unsigned long long*)(bar + 1)) != 0ull) { ok = 0; break; }
                    if (global_ns() - t0 > 30000000000ull) {  // 30 s: never in a sane solve
                        atomicExch(bar + 1, 1ull);
                        ok = 0;
                        break;
                    }
                }
            }
            __threadfence();
            s_ok = ok;
        }
        __syncthreads();
        return s_ok != 0;
    }
};

// Matrix loads: read-only path, L1-allocating.  Adjacent rows share 32-byte
// sectors of the value/column arrays, so L1::no_allocate refetches them from
// L2 and measured 1.9 vs 5.4 TB/s on the 10M-DOF cavity (tools/spmv_lab.cu,
// profiles/r01_spmv_lab.txt).
__device__ __forceinline__ double2 ld_mat(const double2* p) { return __ldg(p); }
__device__ __forceinline__ int ld_mat(const int* p) { return __ldg(p); }

// ---------------------------------------------------------------- loops --

// Element loop over the CTA's chunks: f(i) for every owned row i < n.
template <class F>
__device__ __forceinline__ void for_elems(int n, int G, int cta, F&& f) {
    for (long long base = (long long)cta * kThreads; base < n; base += (long long)G * kThreads) {
        const long long i = base + threadIdx.x;
        if (i < n) f((int)i);
    }
}

// Row loop with S lanes per row over the same chunks.  f(row, lane, valid)
// is called by every thread (valid=false past n) so group shuffles are safe.
template <int S, class F>
__device__ __forceinline__ void for_rows(int n, int G, int cta, F&& f) {
    constexpr int gpb = kThreads / S;
    const int lane = threadIdx.x & (S - 1);
    const int grp = threadIdx.x / S;
    for (long long base = (long long)cta * kThreads; base < n; base += (long long)G * kThreads) {
#pragma unroll 1
        for (int sub = 0; sub < S; ++sub) {
            const long long row = base + (long long)sub * gpb + grp;
            f((int)row, lane, row < n);
        }
    }
}

// Row sum y = sum_k A[row,k] * x(col_k): left to right per lane; for S > 1
// the S lane sums are combined by a fixed xor tree (all lanes get the sum).
// With S == 1 this is exactly the reference's row loop (numkit.cpp:98-103).
//
// With BATCH > 1 each lane first issues up to U = BATCH/S (value, column)
// loads, then the U gathers -- the row_ptr -> col -> x[col] chain is paid
// once per batch instead of once per entry, at a register cost small enough
// to keep full occupancy (the accumulation order per lane is unchanged).
template <int S, class X, int BATCH = 1>
__device__ __forceinline__ double2 row_sum(const Csr& A, int row, int lane, bool valid, X&& xat) {
    constexpr int U = (BATCH / S) > 0 ? (BATCH / S) : 1;
    double2 acc = make_double2(0.0, 0.0);
    if (valid) {
        const int b = __ldg(A.rp + row), e = __ldg(A.rp + row + 1);
        for (int k = b + lane; k < e; k += U * S) {
            double2 a[U];
            int c[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int kk = k + u * S;
                if (kk < e) {
                    a[u] = ld_mat(A.av + kk);
                    c[u] = ld_mat(A.ci + kk);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (k + u * S < e) acc = cvk_add(acc, cvk_mul(a[u], xat(c[u])));
        }
    }
    if (S > 1) {
#pragma unroll
        for (int o = S / 2; o > 0; o >>= 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        }
    }
    return acc;
}

// ----------------------------------------------------------- reductions --
//
// FAST reductions accumulate in double-double (each component carries
// hi + lo, updated with Knuth's TwoSum), combine CTA and grid partials the
// same way, and return the renormalised hi.  The per-element terms are the
// reference's roundings (std::norm, conj(x) * y); their sum is then all but
// exact, so the reduced scalars -- and with them iterates and iteration
// counts -- do not depend on the grid size, the row-to-CTA mapping or which
// FAST path (persistent, phase-kernel, streamed) ran.  REF mode keeps the
// reference's plain sequential double sums (seq_sums).

struct CAcc {  // aggregate: declare as `CAcc a = {};` (zero); no initialisers so __shared__ arrays are legal
    double2 hi, lo;
};

// (hi, lo) += x, renormalised (|lo| <= ulp(hi) / 2)
#ifdef CVK_REDUCE_PLAIN  // measurement variant only (tools/): plain double sums
__device__ __forceinline__ void dd_add1(double& hi, double&, double x) { hi += x; }
#else
__device__ __forceinline__ void dd_add1(double& hi, double& lo, double x) {
    const double s = hi + x;
    const double bb = s - hi;
    double e = (hi - (s - bb)) + (x - bb);
    e += lo;
    hi = s + e;
    lo = e - (hi - s);
}
#endif

// (hi, lo) += (bh, bl)
__device__ __forceinline__ void dd_add2(double& hi, double& lo, double bh, double bl) {
    const double s = hi + bh;
    const double bb = s - hi;
    double e = (hi - (s - bb)) + (bh - bb);
    e += lo + bl;
    hi = s + e;
    lo = e - (hi - s);
}

__device__ __forceinline__ void cacc_add(CAcc& a, const CAcc& b) {
    dd_add2(a.hi.x, a.lo.x, b.hi.x, b.lo.x);
    dd_add2(a.hi.y, a.lo.y, b.hi.y, b.lo.y);
}

__device__ __forceinline__ CAcc warp_sum(CAcc v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        CAcc w;
        w.hi.x = __shfl_xor_sync(0xffffffffu, v.hi.x, o);
        w.hi.y = __shfl_xor_sync(0xffffffffu, v.hi.y, o);
        w.lo.x = __shfl_xor_sync(0xffffffffu, v.lo.x, o);
        w.lo.y = __shfl_xor_sync(0xffffffffu, v.lo.y, o);
        // order the operands so both lanes of a pair compute the same sum
        if (threadIdx.x & o) { CAcc t = v; v = w; w = t; }
        cacc_add(v, w);
    }
    return v;
}

// partial layout: slot 2k holds the hi parts of reduction k, slot 2k+1 the lo parts
__device__ __forceinline__ void cacc_store(double2* part, int k, int G, int cta, const CAcc& v) {
    part[(size_t)(2 * k) * G + cta] = v.hi;
    part[(size_t)(2 * k + 1) * G + cta] = v.lo;
}
__device__ __forceinline__ CAcc cacc_load(const double2* part, int k, int G, int b) {
    CAcc v;
    v.hi = __ldcg(part + (size_t)(2 * k) * G + b);
    v.lo = __ldcg(part + (size_t)(2 * k + 1) * G + b);
    return v;
}

__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    return v;
}

// K-wide double-double butterfly over a warp: every lane ends with the same
// K sums (operands ordered by lane, so the pairs agree bit for bit).  The
// step loop is kept rolled: this epilogue runs once per CTA from a cold
// instruction cache, and the unrolled form (K x 5 steps x 4 shuffles + dd
// adds, plus unrolled cross-warp chains) cost 5 us per reduction in the
// last CTA's fold (tools/trace_phase.py).
template <int K>
__device__ __forceinline__ void warp_sum_k(CAcc (&v)[K]) {
#pragma unroll 1
    for (int o = 16; o > 0; o >>= 1) {
        const bool up = (threadIdx.x & o) != 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            CAcc w;
            w.hi.x = __shfl_xor_sync(0xffffffffu, v[k].hi.x, o);
            w.hi.y = __shfl_xor_sync(0xffffffffu, v[k].hi.y, o);
            w.lo.x = __shfl_xor_sync(0xffffffffu, v[k].lo.x, o);
            w.lo.y = __shfl_xor_sync(0xffffffffu, v[k].lo.y, o);
            CAcc a = up ? w : v[k];
            const CAcc b = up ? v[k] : w;
            cacc_add(a, b);
            v[k] = a;
        }
    }
}

// CTA sum of K accumulators: warp butterflies, then warp 0 combines the
// per-warp sums with a second butterfly.  Result valid in warp 0.
template <int K, int NT>
__device__ __forceinline__ void cta_sum_k(CAcc (&v)[K], CAcc (*sm)[32]) {
    constexpr int NW = NT / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    warp_sum_k<K>(v);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) sm[k][warp] = v[k];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (lane < NW) v[k] = sm[k][lane];
            else v[k] = CAcc{};
        }
        warp_sum_k<K>(v);
    }
}

// FAST: CTA partial of K reductions -> part slots 2k (hi), 2k+1 (lo)
template <int K, int NT = kThreads>
__device__ __forceinline__ void cta_partial(const CAcc (&acc)[K], double2* part, int G, int cta) {
    constexpr int NW = NT / 32;
    __shared__ CAcc sm[K][NW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const CAcc v = warp_sum(acc[k]);
        if (lane == 0) sm[k][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        CAcc s = sm[threadIdx.x][0];
#pragma unroll
        for (int w = 1; w < NW; ++w) cacc_add(s, sm[threadIdx.x][w]);
        cacc_store(part, threadIdx.x, G, cta, s);
    }
}

// FAST: fold the G partials of reduction k (one warp; all lanes get the sum).
// Loads are issued 4 at a time before their adds: a load-add chain over
// G/32 partials serialises G/32 L2 round trips (~4 us per reduction at
// G = 444; the persistent solvers at 50k DOF spent most of an iteration here).
__device__ __forceinline__ double2 fold_one(const double2* part, int k, int G, int lane) {
    CAcc s = {};
    for (int b0 = lane; b0 < G; b0 += 128) {
        CAcc v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = b0 + 32 * u < G ? cacc_load(part, k, G, b0 + 32 * u) : CAcc{};
#pragma unroll
        for (int u = 0; u < 4; ++u) cacc_add(s, v[u]);
    }
    s = warp_sum(s);
    return s.hi;
}

// FAST: after the barrier, every CTA folds the G partials in the same order.
template <int K>
__device__ __forceinline__ void fold_partials(double2 (&out)[K], const double2* part, int G) {
    __shared__ double2 res[K];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int k = warp; k < K; k += (int)(blockDim.x >> 5)) {  // one warp per reduction
        const double2 s = fold_one(part, k, G, lane);
        if (lane == 0) res[k] = s;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = res[k];
}

// REF: thread 0 of every CTA runs the sequential sums; contrib(i, acc)
// adds element i's terms exactly as the reference loop would.
template <int K, class C>
__device__ __forceinline__ void seq_sums(double2 (&out)[K], int n, C&& contrib) {
    __shared__ double2 res[K];
    if (threadIdx.x == 0) {
        double2 acc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = make_double2(0.0, 0.0);
        for (int i = 0; i < n; ++i) contrib(i, acc);
#pragma unroll
        for (int k = 0; k < K; ++k) res[k] = acc[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = res[k];
}

// REF_PAR: the same sequential sums, bit for bit, at the speed of the
// dependent adds.  Warps 1..7 form the element terms contrib(i, 0) -- exactly
// the reference's rounded products conj(x_i) y_i / std::norm(x_i) (0 + t == t,
// and the sign of a zero term cannot change a sum that starts at +0) -- into
// an NB-deep ring of shared-memory blocks; lane 0 of warp 0 adds them left to
// right, loads of a batch of 8 issued before its adds.  Named barriers
// 1..NB (full) and NB+1..2NB (empty) hand the blocks over.
__device__ __forceinline__ void named_sync(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kThreads) : "memory");
}
__device__ __forceinline__ void named_arrive(int id) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(kThreads) : "memory");
}

constexpr int kRefParTerms = 2016;  // one shared-memory ring for every K (32 KB)
__device__ __forceinline__ double2* refpar_ring() {
    __shared__ double2 ring[kRefParTerms];
    return ring;
}

template <int K, class C>
__device__ __forceinline__ void seq_sums_par(double2* out, int n, C&& contrib) {
    constexpr int P = kThreads - 32;  // producer threads
    constexpr int NB = kRefParTerms / (K * P) < 4 ? kRefParTerms / (K * P) : 4;
    static_assert(NB >= 2, "REF_PAR ring too small for K");
    double2 (*buf)[K][P] = reinterpret_cast<double2 (*)[K][P]>(refpar_ring());
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nblk = (n + P - 1) / P;
    if (warp == 0) {
        double2 acc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = make_double2(0.0, 0.0);
        for (int b = 0; b < nblk; ++b) {
            const int s = b % NB;
            named_sync(1 + s);
            if (lane == 0) {
                // full batches unpredicated, then the tail (the clamped,
                // predicated form measured 13.1 vs 7.5 ns per element,
                // tools/refpar_lab.cu)
                const int cnt = min(P, n - b * P);
                const double2* bs = &buf[s][0][0];
                int e0 = 0;
                for (; e0 + 8 <= cnt; e0 += 8) {
                    double2 v[8][K];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
#pragma unroll
                        for (int k = 0; k < K; ++k) v[u][k] = bs[k * P + e0 + u];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
#pragma unroll
                        for (int k = 0; k < K; ++k) acc[k] = cvk_add(acc[k], v[u][k]);
                }
                for (; e0 < cnt; ++e0)
#pragma unroll
                    for (int k = 0; k < K; ++k) acc[k] = cvk_add(acc[k], bs[k * P + e0]);
            }
            __syncwarp();
            named_arrive(1 + NB + s);
        }
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < K; ++k) out[k] = acc[k];
    } else {
        const int t = threadIdx.x - 32;
        for (int b = 0; b < nblk; ++b) {
            const int s = b % NB;
            if (b >= NB) named_sync(1 + NB + s);
            double2 q[K];
#pragma unroll
            for (int k = 0; k < K; ++k) q[k] = make_double2(0.0, 0.0);
            const int i = b * P + t;
            if (i < n) contrib(i, q);
#pragma unroll
            for (int k = 0; k < K; ++k) buf[s][k][t] = q[k];
            named_arrive(1 + s);
        }
        // match the consumer's releases of the last blocks
        for (int b = max(nblk, NB); b < nblk + NB; ++b) named_sync(1 + NB + b % NB);
    }
    __syncthreads();
}

// One reduction phase end: partials/sequential sums + grid barrier.
template <bool REF, int K, class C>
__device__ __forceinline__ bool reduce(GridBar& g, const CAcc (&acc)[K], double2 (&out)[K],
                                       double2* part, int n, C&& contrib) {
    if (REF && g.refpar) {
        // CTA 0 sums, publishes the K results in part[0..K); the second
        // barrier also keeps fast CTAs from rewriting the vectors meanwhile
        if (!g.sync()) return false;
        if (g.cta == 0) seq_sums_par<K>(part, n, contrib);
        if (!g.sync()) return false;
#pragma unroll
        for (int k = 0; k < K; ++k) out[k] = __ldcg(part + k);
    } else if (REF) {
        // thread 0 of every CTA re-reads whole vectors after the barrier; the
        // second barrier keeps fast CTAs from rewriting them meanwhile
        if (!g.sync()) return false;
        seq_sums<K>(out, n, contrib);
        if (!g.sync()) return false;
    } else {
        cta_partial<K>(acc, part, g.G, g.cta);
        if (!g.sync()) return false;
        fold_partials<K>(out, part, g.G);
    }
    return true;
}

// Accumulation helpers used inside the phase loops (FAST) and by the REF
// contrib functors -- the same expression in both, so the per-element terms
// are rounded identically.
__device__ __forceinline__ void acc_norm(double2& a, double2 v) { a.x += cvk_norm(v); }
__device__ __forceinline__ void acc_dot(double2& a, double2 x, double2 y) { a = cvk_add(a, cvk_cmul(x, y)); }
__device__ __forceinline__ void acc_norm(CAcc& a, double2 v) { dd_add1(a.hi.x, a.lo.x, cvk_norm(v)); }
__device__ __forceinline__ void acc_dot(CAcc& a, double2 x, double2 y) {
    const double2 t = cvk_cmul(x, y);
    dd_add1(a.hi.x, a.lo.x, t.x);
    dd_add1(a.hi.y, a.lo.y, t.y);
}

// unconjugated x^T y terms (COCG's bilinear form)
__device__ __forceinline__ void acc_udot(double2& a, double2 x, double2 y) { a = cvk_add(a, cvk_mul(x, y)); }
__device__ __forceinline__ void acc_udot(CAcc& a, double2 x, double2 y) {
    const double2 t = cvk_mul(x, y);
    dd_add1(a.hi.x, a.lo.x, t.x);
    dd_add1(a.hi.y, a.lo.y, t.y);
}

__device__ __forceinline__ double2 prec_apply(const double2* dinv, int i, double2 y) {
    return dinv ? cvk_mul(__ldg(dinv + i), y) : y;
}

// Report / history writers (CTA 0, thread 0).
__device__ __forceinline__ void hist_push(const KArgs& a, int cta, long long& len, double v) {
    if (!a.record) return;
    if (cta == 0 && threadIdx.x == 0 && len < a.hist_cap) a.hist[len] = v;
    ++len;
}

}  // namespace cvk
