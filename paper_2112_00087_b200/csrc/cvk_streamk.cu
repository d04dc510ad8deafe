// cvk_streamk.cu -- persistent TMA-streamed BiCGSTAB (FAST mode, large n).
//
// One cooperative launch per solve, one CTA per SM.  Each CTA keeps its
// producer/consumer ring (cvk_stream.cuh) alive across every phase of every
// iteration, so the per-kernel costs of the phase-kernel path -- launch and
// release gaps, TMA ramp-up, the last-CTA serial fold (2-5 us each, 3 kernels
// per iteration, profiles/r01_phase_timeline.txt) -- become one grid barrier
// per reduction phase.  After each barrier every CTA folds the G partials in
// the same fixed order (double-double, cvk_engine.cuh) and runs the scalar
// recurrence redundantly; no broadcast phase, no host round trip.
//
// Per iteration (krylov.cpp:81-133), as in cvk_phased.cu:
//   A  streamed: p = r + beta (p - omega v) (once per row, pre-hook), v = D^-1 A p, <shadow, v>
//   B  streamed: s = r - alpha v, t = D^-1 A s, x += alpha p, ||s||^2, <t,t>, <t,s>
//   C  element:  x += omega s, r = s - omega t, ||r||^2, <shadow, r>
// and the true residual ||b - A x|| / ||b|| (krylov.cpp:17-23) streamed at the end.
// Per-element arithmetic and per-row order are those of every other FAST
// path, so the iterates are bitwise the phase kernels' and the persistent
// kernel's (tests/test_gpu_parity.py::test_fast_paths_bitwise_identical).
#include <cuda_runtime.h>

#include "cvk_engine.cuh"
#include "cvk_kernels.h"
#include "cvk_stream.cuh"

namespace cvk {

namespace {

constexpr int NT = kStreamThreads;

#ifdef CVK_TRACE
// CTA 0 / CTA 1 timestamps of the last iteration's phase boundaries (globaltimer ns)
__device__ unsigned long long g_sk_trace[2][8];
#define SKT(slot)                                                                   \
    do {                                                                            \
        if (threadIdx.x == 0 && blockIdx.x < 2) {                                   \
            unsigned long long t_;                                                  \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
            g_sk_trace[blockIdx.x][slot] = t_;                                      \
        }                                                                           \
    } while (0)
#else
#define SKT(slot) do { } while (0)
#endif

struct SKArgs {
    Csr A;
    const double2* dinv;  // nullptr: identity
    const double2* b;
    double2* x;
    double2* work;        // r, shadow, s, t, p[2], v[2]
    double2* part;        // kRegions x kMaxSlots x G
    unsigned long long* bar;
    DevReport* rep;
    double* hist;
    long long hist_cap;
    double tol;
    long long max_iter;
    int record;
    StreamLayout L;
};

struct SState {
    double2 rho, rho_new, alpha, omega, beta;
    double bnorm, brk, final_relres;
    long long it, iters, hl;
    int done, conv, brk_code, first, cur;
};

// grid-wide double-double sums of K accumulators; valid in every thread of
// every CTA (same bits everywhere)
template <int K>
__device__ __forceinline__ bool grid_reduce(const CAcc (&acc)[K], double2 (&out)[K], double2* part, GridBar& g,
                                            CAcc (*sm)[32], double2* res) {
    const int G = gridDim.x;
    CAcc v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = acc[k];
    cta_sum_k<K, NT>(v, sm);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) cacc_store(part, k, G, blockIdx.x, v[k]);
    }
    if (!g.sync()) return false;
    CAcc s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) s[k] = CAcc{};
#pragma unroll 1
    for (int b = threadIdx.x; b < G; b += NT) {
#pragma unroll
        for (int k = 0; k < K; ++k) cacc_add(s[k], cacc_load(part, k, G, b));
    }
    cta_sum_k<K, NT>(s, sm);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) res[k] = s[k].hi;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = res[k];
    return true;
}

// element loop over all rows with every thread of the grid, U rows per trip
template <int U, class LD, class STF>
__device__ __forceinline__ void elems(int n, LD&& ld, STF&& stf) {
    using T = decltype(ld(0));
    const long long stride = (long long)gridDim.x * NT;
    for (long long base = (long long)blockIdx.x * NT + threadIdx.x; base < n; base += stride * U) {
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

__device__ __forceinline__ void hist(const SKArgs& a, SState& S, double v) {
    if (!a.record) return;
    if (blockIdx.x == 0 && threadIdx.x == 0 && S.hl < a.hist_cap) a.hist[S.hl] = v;
    ++S.hl;
}

// Each phase is its own (non-inlined) function so that its register
// allocation does not have to coexist with the other phases' live ranges:
// inlined into one kernel, the three bodies spilled ~1 KB per thread and the
// phases ran 1.5-3x slower than as separate kernels.
struct Acc2 { CAcc v[2]; };
struct Acc3 { CAcc v[3]; };

__device__ __noinline__ CAcc phase_a(Csr A, const double2* dinv, StreamLayout L, unsigned char* smem, int base,
                                     int first, double2 beta, double2 nom, const double2* r, const double2* pc,
                                     const double2* vc, double2* pn, double2* vn, const double2* sh) {
    const double2* vecs[5] = {r, pc, vc, sh, dinv};
    CAcc acc = {};
    stream_rows(
        A, L, vecs, smem,
        [&](int t, const Chunk& ch) {
            auto xs = [&](int l) -> double2 {
                const double2 rc = ch.v(0, l);
                if (first || l < kStreamRows) return rc;
                return cvk_add(cvk_mul(beta, cvk_add(ch.v(1, l), cvk_mul(nom, ch.v(2, l)))), rc);
            };
            auto xg = [&](int c) -> double2 {
                const double2 rc = r[c];
                if (first) return rc;
                return cvk_add(cvk_mul(beta, cvk_add(pc[c], cvk_mul(nom, vc[c]))), rc);
            };
            const double2 y = chunk_row_sum<5>(ch, t, xs, xg);
            const double2 vi = dinv ? cvk_mul(ch.v(4, t), y) : y;
            const int row = ch.r0 + t;
            pn[row] = xs(t);
            vn[row] = vi;
            acc_dot(acc, ch.v(3, t), vi);
        },
        nullptr, nullptr,
        [&](int t, const Chunk& ch) {
            if (!first)
                ch.set(0, t, cvk_add(cvk_mul(beta, cvk_add(ch.v(1, t), cvk_mul(nom, ch.v(2, t)))), ch.v(0, t)));
        },
        base, false);
    return acc;
}

__device__ __noinline__ Acc3 phase_b(Csr A, const double2* dinv, StreamLayout L, unsigned char* smem, int base,
                                     double2 alpha, const double2* r, const double2* vn, const double2* pn,
                                     double2* x, double2* sv, double2* tv) {
    const double2 nal = cvk_neg(alpha);
    const double2* vecs[5] = {r, vn, dinv, pn, x};
    Acc3 acc = {};
    stream_rows(
        A, L, vecs, smem,
        [&](int t, const Chunk& ch) {
            auto xs = [&](int l) -> double2 {
                return l < kStreamRows ? ch.v(0, l) : cvk_add(ch.v(0, l), cvk_mul(nal, ch.v(1, l)));
            };
            auto xg = [&](int c) -> double2 { return cvk_add(r[c], cvk_mul(nal, vn[c])); };
            const double2 y = chunk_row_sum<5>(ch, t, xs, xg);
            const double2 ti = dinv ? cvk_mul(ch.v(2, t), y) : y;
            const double2 si = xs(t);
            const int row = ch.r0 + t;
            sv[row] = si;
            tv[row] = ti;
            x[row] = cvk_add(ch.v(4, t), cvk_mul(alpha, ch.v(3, t)));
            acc_norm(acc.v[0], si);
            acc_dot(acc.v[1], ti, ti);
            acc_dot(acc.v[2], ti, si);
        },
        nullptr, nullptr,
        [&](int t, const Chunk& ch) { ch.set(0, t, cvk_add(ch.v(0, t), cvk_mul(nal, ch.v(1, t)))); },
        base, false);
    return acc;
}

__device__ __noinline__ Acc2 phase_c(int n, double2 omega, const double2* sv, const double2* tv, const double2* sh,
                                     double2* x, double2* r) {
    const double2 nomg = cvk_neg(omega);
    Acc2 acc = {};
    struct L4 { double2 s, t, sh, x; };
    elems<4>(n, [&](int i) { return L4{sv[i], tv[i], sh[i], x[i]}; },
             [&](int i, const L4& v) {
                 x[i] = cvk_add(v.x, cvk_mul(omega, v.s));
                 const double2 ri = cvk_add(v.s, cvk_mul(nomg, v.t));
                 r[i] = ri;
                 acc_norm(acc.v[0], ri);
                 acc_dot(acc.v[1], v.sh, ri);
             });
    return acc;
}

__device__ __noinline__ Acc2 phase_true(Csr A, StreamLayout L, unsigned char* smem, int base, const double2* x,
                                        const double2* b) {
    const double2* vecs[5] = {x, b, nullptr, nullptr, nullptr};  // L.nvec = 5: unused slots skipped
    Acc2 acc = {};
    stream_rows(
        A, L, vecs, smem,
        [&](int t, const Chunk& ch) {
            const double2 y = chunk_row_sum<5>(ch, t, [&](int l) { return ch.v(0, l); }, [&](int c) { return x[c]; });
            const double2 bi = ch.v(1, t);
            acc_norm(acc.v[0], bi);
            acc_norm(acc.v[1], cvk_sub(bi, y));
        },
        nullptr, nullptr, NoPre(), base, false);
    return acc;
}

__global__ void __launch_bounds__(NT, 1) k_bicgstab_stream(SKArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ CAcc sm[3][32];
    __shared__ double2 res[3];
    __shared__ SState S;
    const int n = a.A.n;
    const size_t nn = (size_t)n;
    double2* r = a.work;
    double2* sh = a.work + nn;
    double2* sv = a.work + 2 * nn;
    double2* tv = a.work + 3 * nn;
    // p[c] = work + (4 + c) n, v[c] = work + (6 + c) n (no runtime-indexed local arrays: they live on the stack)
    const double2* dinv = a.dinv;
    double2* x = a.x;
    GridBar g(a.bar, gridDim.x);
    int region = 0;
    auto next_part = [&]() {
        double2* p = a.part + (size_t)region * kMaxSlots * gridDim.x;
        region = region + 1 == kRegions ? 0 : region + 1;
        return p;
    };
    const StreamLayout L = a.L;
    stream_init(smem, L);
    const int cnt = stream_chunks_per_cta(n, L);
    int base = 0;
    bool ok = true;

    // ---- init (krylov.cpp:62-79): r = shadow = M^-1 b, x = 0
    {
        CAcc acc[2] = {};
        elems<4>(n, [&](int i) { return __ldg(a.b + i); },
                 [&](int i, double2 bi) {
                     const double2 ri = prec_apply(dinv, i, bi);
                     r[i] = ri;
                     sh[i] = ri;
                     x[i] = make_double2(0.0, 0.0);
                     acc_norm(acc[0], ri);
                     acc_dot(acc[1], ri, ri);
                 });
        double2 tot[2];
        ok = grid_reduce<2>(acc, tot, next_part(), g, sm, res);
        if (ok && threadIdx.x == 0) {
            S.hl = 0;
            S.done = 0; S.conv = 0; S.brk_code = 0; S.iters = 0; S.final_relres = 0.0;
            S.bnorm = sqrt(tot[0].x);
            if (S.bnorm == 0.0) {  // krylov.cpp:70-74
                S.done = 1; S.conv = 1;
            } else {
                S.brk = 1e-30 * S.bnorm * S.bnorm;
                S.rho_new = tot[1];
                S.rho = S.alpha = S.omega = make_double2(1.0, 0.0);
                S.it = 1; S.first = 1; S.cur = 0;
            }
        }
        __syncthreads();
    }
    const bool zero_rhs = ok && S.done;

    while (ok && !S.done) {
        // ---- top of iteration (krylov.cpp:81-96)
        if (threadIdx.x == 0) {
            if (S.it > a.max_iter) {
                S.done = 1;
            } else if (cvk_abs(S.rho_new) < S.brk) {
                S.done = 1; S.brk_code = 1; S.iters = S.it - 1;
            } else {
                if (!S.first) S.beta = cvk_mul(cvk_cdiv(S.rho_new, S.rho), cvk_cdiv(S.alpha, S.omega));
                S.rho = S.rho_new;
            }
        }
        __syncthreads();
        if (S.done) break;
        const int cur = S.cur;
        const bool first = S.first != 0;
        const double2 beta = S.beta, nom = cvk_neg(S.omega);
        const double2* __restrict__ pc = a.work + (size_t)(4 + cur) * nn;
        const double2* __restrict__ vc = a.work + (size_t)(6 + cur) * nn;
        double2* __restrict__ pn = a.work + (size_t)(5 - cur) * nn;
        double2* __restrict__ vn = a.work + (size_t)(7 - cur) * nn;

        // ---- A: p_new on the fly, v = M^-1 A p, <shadow, v>
        SKT(0);
        {
            CAcc acc[1] = {phase_a(a.A, dinv, L, smem, base, first ? 1 : 0, beta, nom, r, pc, vc, pn, vn, sh)};
            base += cnt;
            SKT(1);
            double2 tot[1];
            if (!(ok = grid_reduce<1>(acc, tot, next_part(), g, sm, res))) break;
            SKT(2);
            if (threadIdx.x == 0) {
                if (cvk_abs(tot[0]) < S.brk) {
                    S.done = 1; S.brk_code = 2; S.iters = S.it - 1;
                } else {
                    S.alpha = cvk_cdiv(S.rho, tot[0]);
                }
            }
            __syncthreads();
            if (S.done) break;
        }
        // ---- B: s = r - alpha v on the fly, t = M^-1 A s, x += alpha p
        {
            const Acc3 b3 = phase_b(a.A, dinv, L, smem, base, S.alpha, r, vn, pn, x, sv, tv);
            CAcc acc[3] = {b3.v[0], b3.v[1], b3.v[2]};
            base += cnt;
            SKT(3);
            double2 tot[3];
            if (!(ok = grid_reduce<3>(acc, tot, next_part(), g, sm, res))) break;
            SKT(4);
            if (threadIdx.x == 0) {
                const double relres = sqrt(tot[0].x) / S.bnorm;
                if (relres <= a.tol) {  // krylov.cpp:107-114 half-step exit
                    S.done = 1; S.conv = 1; S.iters = S.it; S.final_relres = relres;
                    hist(a, S, relres);
                } else if (cvk_abs(tot[1]) < S.brk) {
                    S.done = 1; S.brk_code = 3; S.iters = S.it;
                } else {
                    S.omega = cvk_cdiv(tot[2], tot[1]);
                }
            }
            __syncthreads();
            if (S.done) break;
        }
        // ---- C: x += omega s, r = s - omega t, ||r||, <shadow, r>
        {
            const Acc2 c2 = phase_c(n, S.omega, sv, tv, sh, x, r);
            CAcc acc[2] = {c2.v[0], c2.v[1]};
            SKT(5);
            double2 tot[2];
            if (!(ok = grid_reduce<2>(acc, tot, next_part(), g, sm, res))) break;
            SKT(6);
            if (threadIdx.x == 0) {
                const double relres = sqrt(tot[0].x) / S.bnorm;
                S.final_relres = relres;
                S.iters = S.it;
                hist(a, S, relres);
                if (relres <= a.tol) {
                    S.done = 1; S.conv = 1;
                } else {
                    S.rho_new = tot[1];
                    S.cur ^= 1;
                    S.first = 0;
                    S.it++;
                }
            }
            __syncthreads();
        }
    }

    // ---- true residual ||b - A x|| / ||b|| (krylov.cpp:17-23), skipped for b = 0
    double trr = 0.0;
    if (ok && !zero_rhs) {
        const Acc2 t2 = phase_true(a.A, L, smem, base, x, a.b);
        CAcc acc[2] = {t2.v[0], t2.v[1]};
        base += cnt;
        double2 tot[2];
        ok = grid_reduce<2>(acc, tot, next_part(), g, sm, res);
        if (ok) {
            const double bn = sqrt(tot[0].x), rn = sqrt(tot[1].x);
            trr = bn > 0 ? rn / bn : rn;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.rep->converged = ok ? S.conv : 0;
        a.rep->breakdown = S.brk_code;
        a.rep->iterations = S.iters;
        a.rep->final_relres = S.final_relres;
        a.rep->true_relres = trr;
        a.rep->history_len = S.hl;
        a.rep->error = ok ? 0 : 1;
    }
}

}  // namespace

const void* streamk_bicgstab_kernel() { return (const void*)k_bicgstab_stream; }

int streamk_trace_read(unsigned long long* out16) {
#ifdef CVK_TRACE
    return cudaMemcpyFromSymbol(out16, g_sk_trace, sizeof(g_sk_trace)) == cudaSuccess ? 16 : -1;
#else
    (void)out16;
    return 0;
#endif
}

size_t streamk_args_size() { return sizeof(SKArgs); }

void streamk_pack_args(void* out, const Csr& A, const double2* dinv, const double2* b, double2* x, double2* work,
                       double2* part, unsigned long long* bar, DevReport* rep, double* hist, long long hist_cap,
                       double tol, long long max_iter, int record, const StreamLayout& L) {
    SKArgs* p = (SKArgs*)out;
    p->A = A;
    p->dinv = dinv;
    p->b = b;
    p->x = x;
    p->work = work;
    p->part = part;
    p->bar = bar;
    p->rep = rep;
    p->hist = hist;
    p->hist_cap = hist_cap;
    p->tol = tol;
    p->max_iter = max_iter;
    p->record = record;
    p->L = L;
}

}  // namespace cvk
