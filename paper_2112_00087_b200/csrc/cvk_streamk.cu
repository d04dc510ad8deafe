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
    double2* P[2] = {a.work + 4 * nn, a.work + 5 * nn};
    double2* V[2] = {a.work + 6 * nn, a.work + 7 * nn};
    const double2* dinv = a.dinv;
    double2* x = a.x;
    GridBar g(a.bar, gridDim.x);
    double2* part[kRegions];
    for (int q = 0; q < kRegions; ++q) part[q] = a.part + (size_t)q * kMaxSlots * gridDim.x;
    int region = 0;
    auto next_part = [&]() { double2* p = part[region]; region = (region + 1) % kRegions; return p; };
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
        const double2* __restrict__ pc = P[cur];
        const double2* __restrict__ vc = V[cur];
        double2* __restrict__ pn = P[cur ^ 1];
        double2* __restrict__ vn = V[cur ^ 1];

        // ---- A: p_new on the fly, v = M^-1 A p, <shadow, v>
        {
            const double2* vecs[5] = {r, pc, vc, sh, dinv};
            CAcc acc[1] = {};
            stream_rows(
                a.A, L, vecs, smem,
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
                    acc_dot(acc[0], ch.v(3, t), vi);
                },
                nullptr, nullptr,
                [&](int t, const Chunk& ch) {
                    if (!first)
                        ch.set(0, t, cvk_add(cvk_mul(beta, cvk_add(ch.v(1, t), cvk_mul(nom, ch.v(2, t)))), ch.v(0, t)));
                },
                base, false);
            base += cnt;
            double2 tot[1];
            if (!(ok = grid_reduce<1>(acc, tot, next_part(), g, sm, res))) break;
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
            const double2 alpha = S.alpha, nal = cvk_neg(S.alpha);
            const double2* vecs[5] = {r, vn, dinv, pn, x};
            CAcc acc[3] = {};
            stream_rows(
                a.A, L, vecs, smem,
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
                    acc_norm(acc[0], si);
                    acc_dot(acc[1], ti, ti);
                    acc_dot(acc[2], ti, si);
                },
                nullptr, nullptr,
                [&](int t, const Chunk& ch) { ch.set(0, t, cvk_add(ch.v(0, t), cvk_mul(nal, ch.v(1, t)))); },
                base, false);
            base += cnt;
            double2 tot[3];
            if (!(ok = grid_reduce<3>(acc, tot, next_part(), g, sm, res))) break;
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
            const double2 omega = S.omega, nomg = cvk_neg(S.omega);
            CAcc acc[2] = {};
            struct L4 { double2 s, t, sh, x; };
            elems<4>(n, [&](int i) { return L4{sv[i], tv[i], sh[i], x[i]}; },
                     [&](int i, const L4& v) {
                         x[i] = cvk_add(v.x, cvk_mul(omega, v.s));
                         const double2 ri = cvk_add(v.s, cvk_mul(nomg, v.t));
                         r[i] = ri;
                         acc_norm(acc[0], ri);
                         acc_dot(acc[1], v.sh, ri);
                     });
            double2 tot[2];
            if (!(ok = grid_reduce<2>(acc, tot, next_part(), g, sm, res))) break;
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
        const double2* vecs[2] = {x, a.b};
        CAcc acc[2] = {};
        stream_rows(
            a.A, L, vecs, smem,
            [&](int t, const Chunk& ch) {
                const double2 y = chunk_row_sum<5>(ch, t, [&](int l) { return ch.v(0, l); },
                                                   [&](int c) { return x[c]; });
                const double2 bi = ch.v(1, t);
                acc_norm(acc[0], bi);
                acc_norm(acc[1], cvk_sub(bi, y));
            },
            nullptr, nullptr, NoPre(), base, false);
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
