// cvk_gmres.cu -- FAST-mode restarted GMRES(m) for large systems as a chain
// of phase kernels replayed from a CUDA graph (beyond the reference, which
// has no GMRES; operation order = the persistent kernel's gmres_body =
// oracle/cavac_oracle.c orc_gmres: CGS2 Arnoldi, complex Givens).
//
// The persistent kernel keeps every CTA busy with one element at a time and
// folds each of the up-to-2m inner products with its own block reduction;
// at 1M DOF it ran at ~20% of the HBM roofline (450-500 us per Arnoldi
// step).  Here each Arnoldi step is four kernels:
//   k_g_spmv   V_j = src / scale (formed in the gathers), w = M^-1 A V_j
//   k_g_dots   h1 = V^H w               -- warps own basis vectors q, lanes rows
//   k_g_dots   w -= V h1; h2 = V^H w    -- update pass, then dot pass per block
//   k_g_upd2   w -= V h2; ||w||; Hessenberg column, rotations, residual
//              estimate, restart decision (last CTA)
// and a restart is k_g_x (x += V y) + k_g_spmv in residual mode.  Every
// reduction is double-double, so the scalars equal the persistent FAST path's.
#include <cuda_runtime.h>

#include <cstddef>

#include "cvk_engine.cuh"
#include "cvk_kernels.h"
#include "cvk_stream.cuh"

#ifndef CVK_SPMV_BATCH
#define CVK_SPMV_BATCH 5  // (value, column) loads in flight per row in the streamed SpMV
#endif

namespace cvk {

namespace {

constexpr int kGB = kThreads;  // rows per block = threads per CTA

enum GMode { G_ARN = 0, G_RX = 1, G_RR = 2, G_WAIT = 3 };

struct GState {
    int done, conv, brk_code, mode, stop, j, k, wcur, skip_true, pad;
    long long total, hl, hist_cap, max_iter;
    int record, m;
    double bnorm, brk, beta, scale, final_relres, tol, hn;
    unsigned counter[4];
    double2 h1[kMaxDots], h2[kMaxDots], sn[kMaxDots], gv[kMaxDots + 1], yv[kMaxDots];
    double cs[kMaxDots];
    double2 H[(kMaxDots + 1) * kMaxDots];
};

struct GArgs {
    Csr A;
    const double2* dinv;
    const double2* b;
    double2* x;
    double2* work;  // r, W[2], V[0..m]
    double2* part;
    GState* st;
    double* hist;
    DevReport* rep;
    int capk, nst, pf_rows;  // streamed Arnoldi SpMV (k_g_spmv_s); nst = 0: not streamed
};

__device__ __forceinline__ void pdl_enter_g() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ double2* vec(const GArgs& a, int idx) { return a.work + (size_t)idx * a.A.n; }
__device__ __forceinline__ double2* Vq(const GArgs& a, int q) { return vec(a, 3 + q); }

// publish one dd partial per CTA; true in the CTA that arrived last
__device__ bool arrive_last(unsigned* counter) {
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

__device__ __forceinline__ void ghist(const GArgs& a, GState* st, double v) {
    if (!st->record) return;
    if (st->hl < st->hist_cap) a.hist[st->hl] = v;
    st->hl++;
}

// back substitution H y = g (thread 0), then the x update is k_g_x
__device__ void back_subst(GState* st) {
    const int k = st->k, M = st->m;
    for (int i = k; i-- > 0;) {
        double2 s = st->gv[i];
        for (int q = i + 1; q < k; ++q) s = cvk_sub(s, cvk_mul(st->H[i * M + q], st->yv[q]));
        st->yv[i] = cvk_cdiv(s, st->H[i * M + i]);
    }
}

__global__ void __launch_bounds__(kThreads) k_g_init(GArgs a) {
    pdl_enter_g();
    GState* st = a.st;
    const int n = a.A.n;
    double2* r = vec(a, 0);
    CAcc acc = {};
    for_elems(n, gridDim.x, blockIdx.x, [&](int i) {
        const double2 ri = prec_apply(a.dinv, i, __ldg(a.b + i));
        r[i] = ri;
        a.x[i] = make_double2(0.0, 0.0);
        acc_norm(acc, ri);
    });
    CAcc v[1] = {acc};
    __shared__ CAcc sm[1][32];
    cta_sum_k<1, kThreads>(v, sm);
    if (threadIdx.x == 0) cacc_store(a.part, 0, gridDim.x, blockIdx.x, v[0]);
    if (!arrive_last(&st->counter[0])) return;
    const double2 tot = fold_one(a.part, 0, gridDim.x, threadIdx.x & 31);
    if (threadIdx.x != 0) return;
    st->counter[0] = 0;
    st->bnorm = sqrt(tot.x);
    if (st->bnorm == 0.0) { st->done = 1; st->conv = 1; st->skip_true = 1; return; }
    st->brk = 1e-30 * st->bnorm * st->bnorm;
    st->beta = st->bnorm;
    st->total = 0;
    for (int i = 0; i <= st->m; ++i) st->gv[i] = make_double2(0.0, 0.0);
    st->gv[0] = make_double2(st->beta, 0.0);
    st->scale = st->beta;
    st->j = 0;
    st->k = 0;
    st->wcur = 0;
    st->mode = G_ARN;
}

// slot start: restart x update (x += V y), or the wait -> Arnoldi transition
__global__ void __launch_bounds__(kThreads) k_g_x(GArgs a) {
    pdl_enter_g();
    GState* st = a.st;
    if (st->done) return;
    const int mode = st->mode;
    if (mode == G_RX) {
        const int n = a.A.n, k = st->k;
        __shared__ double2 y[kMaxDots];
        for (int q = threadIdx.x; q < k; q += blockDim.x) y[q] = st->yv[q];
        __syncthreads();
        for_elems(n, gridDim.x, blockIdx.x, [&](int i) {
            double2 xi = a.x[i];
            const int cnt = k;
            for (int q0 = 0; q0 < cnt; q0 += 4) {
                    double2 vq4[4];
#pragma unroll
                    for (int u4 = 0; u4 < 4; ++u4)
                        if (q0 + u4 < cnt) vq4[u4] = Vq(a, q0 + u4)[i];
#pragma unroll
                    for (int u4 = 0; u4 < 4; ++u4)
                        if (q0 + u4 < cnt) xi = cvk_add(xi, cvk_mul(y[q0 + u4], vq4[u4]));
                }
            a.x[i] = xi;
        });
    } else if (mode != G_WAIT) {
        return;
    }
    if (!arrive_last(&st->counter[1])) return;
    if (threadIdx.x != 0) return;
    st->counter[1] = 0;
    if (mode == G_WAIT) { st->mode = G_ARN; return; }
    if (st->brk_code == 7 && st->final_relres <= st->tol) { st->conv = 1; st->brk_code = 0; }
    if (st->stop) { st->done = 1; return; }
    st->mode = G_RR;
}

// Arnoldi SpMV (V_j = src / scale, w = M^-1 A V_j) or the restart residual
// r = M^-1 (b - A x) with ||r||
__global__ void __launch_bounds__(kThreads) k_g_spmv(GArgs a) {
    pdl_enter_g();
    GState* st = a.st;
    if (st->done) return;
    const int mode = st->mode;
    if (mode != G_ARN && mode != G_RR) return;
    const int n = a.A.n;
    if (mode == G_ARN) {
        if (a.nst > 0) return;  // the streamed kernel k_g_spmv_s runs the Arnoldi SpMV
        const int j = st->j;
        const double2* src = j == 0 ? vec(a, 0) : vec(a, 1 + (st->wcur ^ 1));
        double2* w = vec(a, 1 + st->wcur);
        double2* vj = Vq(a, j);
        const double sc = st->scale;
        auto vat = [&](int c) -> double2 { return cvk_divr(src[c], sc); };
        for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
            const double2 yv = row_sum<1, decltype(vat)&, 5>(a.A, row, 0, valid, vat);
            if (valid) {
                vj[row] = vat(row);
                w[row] = prec_apply(a.dinv, row, yv);
            }
        });
        return;
    }
    double2* r = vec(a, 0);
    CAcc acc = {};
    const double2* x = a.x;
    auto xat = [&](int c) -> double2 { return x[c]; };
    for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
        const double2 yv = row_sum<1, decltype(xat)&, 5>(a.A, row, 0, valid, xat);
        if (valid) {
            const double2 ri = prec_apply(a.dinv, row, cvk_sub(__ldg(a.b + row), yv));
            r[row] = ri;
            acc_norm(acc, ri);
        }
    });
    CAcc v[1] = {acc};
    __shared__ CAcc sm[1][32];
    cta_sum_k<1, kThreads>(v, sm);
    if (threadIdx.x == 0) cacc_store(a.part, 0, gridDim.x, blockIdx.x, v[0]);
    if (!arrive_last(&st->counter[2])) return;
    const double2 tot = fold_one(a.part, 0, gridDim.x, threadIdx.x & 31);
    if (threadIdx.x != 0) return;
    st->counter[2] = 0;
    st->beta = sqrt(tot.x);
    if (st->beta == 0.0) { st->conv = 1; st->final_relres = 0.0; st->done = 1; return; }
    // top of the restart loop
    st->final_relres = st->beta / st->bnorm;
    if (st->final_relres <= st->tol) { st->conv = 1; st->done = 1; return; }
    for (int i = 0; i <= st->m; ++i) st->gv[i] = make_double2(0.0, 0.0);
    st->gv[0] = make_double2(st->beta, 0.0);
    st->scale = st->beta;
    st->j = 0;
    st->k = 0;
    st->mode = G_WAIT;
}

// The Arnoldi SpMV on the TMA ring (cvk_stream.cuh): V_j = src / scale is
// formed once per chunk row in the pre-hook and by the out-of-chunk gathers,
// w = M^-1 A V_j -- the per-element roundings and per-row order of k_g_spmv.
__global__ void __launch_bounds__(kStreamThreads, 1) k_g_spmv_s(GArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter_g();
    GState* st = a.st;
    if (st->done || st->mode != G_ARN) return;
    const int j = st->j;
    const double2* src = j == 0 ? vec(a, 0) : vec(a, 1 + (st->wcur ^ 1));
    double2* w = vec(a, 1 + st->wcur);
    double2* vj = Vq(a, j);
    const double sc = st->scale;
    const double2* vecs[2] = {src, a.dinv};
    StreamLayout L{a.capk, 2, a.nst};
    L.ngather = 1;
    L.pf_rows = a.pf_rows;
    stream_rows(a.A, L, vecs, smem, [&](int t, const Chunk& ch) {
        auto xs = [&](int l) -> double2 { return ch.v(0, l); };
        auto xg = [&](int c) -> double2 { return cvk_divr(src[c], sc); };
        const double2 y = chunk_row_sum<CVK_SPMV_BATCH>(ch, t, xs, xg);
        const int row = ch.r0 + t;
        vj[row] = xs(t);
        w[row] = a.dinv ? cvk_mul(ch.v(1, t), y) : y;
    }, nullptr, [&](int t, const Chunk& ch) { ch.set(0, t, cvk_divr(ch.v(0, t), sc)); });
}

// h = V^H w over q <= j (UPDATE: first w -= V h1 per row).  Basis vectors are
// owned by warps (q = warp + 8 u), lanes stride the rows of a 256-row block.
template <bool UPDATE>
__global__ void __launch_bounds__(kThreads) k_g_dots(GArgs a) {
    pdl_enter_g();
    GState* st = a.st;
    if (st->done || st->mode != G_ARN) return;
    const int n = a.A.n, j = st->j, cnt = j + 1;
    double2* w = vec(a, 1 + st->wcur);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ double2 hs[kMaxDots];
    if (UPDATE)
        for (int q = threadIdx.x; q < cnt; q += blockDim.x) hs[q] = st->h1[q];
    __syncthreads();
    const int nblk = (n + kGB - 1) / kGB;
    double2* pr = a.part;
    auto update_block = [&](int blk) {  // w -= V h1 on one block (thread per row, 4 basis loads in flight)
        const int i = blk * kGB + threadIdx.x;
        if (i < n) {
            double2 wi = w[i];
            for (int q0 = 0; q0 < cnt; q0 += 4) {
                double2 vq4[4];
#pragma unroll
                for (int u4 = 0; u4 < 4; ++u4)
                    if (q0 + u4 < cnt) vq4[u4] = Vq(a, q0 + u4)[i];
#pragma unroll
                for (int u4 = 0; u4 < 4; ++u4)
                    if (q0 + u4 < cnt) wi = cvk_add(wi, cvk_mul(cvk_neg(hs[q0 + u4]), vq4[u4]));
            }
            w[i] = wi;
        }
    };
    auto dot_block = [&](CAcc& sq, const double2* vq, int blk) {  // one basis vector, one block
        const int r0 = blk * kGB;
#pragma unroll
        for (int e0 = 0; e0 < kGB / 32; e0 += 4) {
            double2 vv[4], wv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = r0 + lane + 32 * (e0 + e);
                if (i < n) { vv[e] = vq[i]; wv[e] = w[i]; }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (r0 + lane + 32 * (e0 + e) < n) acc_dot(sq, vv[e], wv[e]);
        }
    };
    {
        // update every block of this CTA first, then the dots with one
        // accumulator live at a time (measured faster than block-interleaved
        // update+dots, whose 122 registers halve the occupancy)
        if (UPDATE) {
            for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) update_block(blk);
            __syncthreads();  // the dots below read only this CTA's rows
        }
        for (int q = warp; q < cnt; q += kWarps) {
            CAcc sq = {};
            for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) dot_block(sq, Vq(a, q), blk);
            const CAcc t = warp_sum(sq);
            if (lane == 0) {
                cacc_store(pr, q, gridDim.x, blockIdx.x, t);
                __threadfence();
            }
        }
    }
    if (!arrive_last(&st->counter[UPDATE ? 1 : 0])) return;
    double2* out = UPDATE ? st->h2 : st->h1;
    for (int q = warp; q < cnt; q += kWarps) {
        const double2 v = fold_one(pr, q, gridDim.x, lane);
        if (lane == 0) out[q] = v;
    }
    if (threadIdx.x == 0) st->counter[UPDATE ? 1 : 0] = 0;
}

// Second CGS pass in ONE read of the basis: w -= V h1, then h2 = V^H w, on
// row tiles of [w | V_0 .. V_j] streamed into shared memory by TMA (a ring of
// as many stages as fit).  k_g_dots<true> reads V twice (its update pass,
// then its dot pass); at 5M DOF that pass was ~30% of an Arnoldi step.
// Per-row update order is that of k_g_dots<true>; h2 is double-double, so
// the scalars equal it.
constexpr int kTileRows = 128;                          // rows per tile = threads per consumer group
constexpr int kTileGroups = 3;                          // consumer groups
constexpr int kTileThreads = kTileRows * kTileGroups + 32;  // + producer warp
constexpr int kTileWarps = kTileRows / 32;              // warps per group
constexpr int kTileQ = 8;                               // basis vectors per warp: cnt <= 32 (m <= 32)

__global__ void __launch_bounds__(kTileThreads, 1) k_g_ud_s(GArgs a, int smem_bytes) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter_g();
    GState* st = a.st;
    if (st->done || st->mode != G_ARN) return;
    const int n = a.A.n, cnt = st->j + 1;
    double2* w = vec(a, 1 + st->wcur);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    __shared__ double2 hs[kMaxDots];
    __shared__ CAcc red[kTileGroups][kMaxDots];
    for (int q = tid; q < cnt; q += blockDim.x) hs[q] = st->h1[q];
    const size_t vb = (size_t)kTileRows * 16, sb = (size_t)(cnt + 1) * vb;
    const int ST = (int)min((size_t)kStreamMaxStages, ((size_t)smem_bytes - 2 * kStreamMaxStages * 8) / sb);
    uint64_t* full = (uint64_t*)(smem + (size_t)ST * sb);  // sb is a multiple of 2 KB
    uint64_t* empty = full + kStreamMaxStages;
    if (tid == 0) {
        for (int q = 0; q < ST; ++q) {
            mbar_init(full + q, 1);
            mbar_init(empty + q, kTileRows);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int ntiles = (n + kTileRows - 1) / kTileRows, G = gridDim.x;
    const int mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / G + 1 : 0;
    if (tid >= kTileGroups * kTileRows) {  // producer warp (lane 0 issues; the loop is warp-uniform)
        for (int i = 0; i < mine; ++i) {
            const int s = i % ST, r0 = (blockIdx.x + i * G) * kTileRows;
            const uint32_t bytes = (uint32_t)(min(kTileRows, n - r0) * 16);
            if (lane == 0) {
                mbar_wait(empty + s, ((uint32_t)(i / ST) & 1u) ^ 1u);
                mbar_expect_tx(full + s, bytes * (uint32_t)(cnt + 1));
                unsigned char* sp = smem + (size_t)s * sb;
                bulk_g2s(sp, w + r0, bytes, full + s);
                for (int q = 0; q < cnt; ++q) bulk_g2s(sp + (size_t)(q + 1) * vb, Vq(a, q) + r0, bytes, full + s);
            }
            __syncwarp();
        }
    } else {
        const int g = tid / kTileRows, t = tid % kTileRows, wq = (tid % kTileRows) >> 5;
        CAcc acc[kTileQ];
#pragma unroll
        for (int u = 0; u < kTileQ; ++u) acc[u] = CAcc{};
        for (int i = g; i < mine; i += kTileGroups) {
            const int s = i % ST, r0 = (blockIdx.x + i * G) * kTileRows, rows = min(kTileRows, n - r0);
            mbar_wait(full + s, (uint32_t)(i / ST) & 1u);
            double2* W = (double2*)(smem + (size_t)s * sb);
            const double2* V = W + kTileRows;
            if (t < rows) {
                double2 wi = W[t];
                for (int q = 0; q < cnt; ++q) wi = cvk_add(wi, cvk_mul(cvk_neg(hs[q]), V[(size_t)q * kTileRows + t]));
                W[t] = wi;
                w[r0 + t] = wi;
            }
            asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(kTileRows) : "memory");
#pragma unroll
            for (int u = 0; u < kTileQ; ++u) {
                const int q = wq + kTileWarps * u;
                if (q < cnt) {
                    const double2* vq = V + (size_t)q * kTileRows;
#pragma unroll
                    for (int e = 0; e < kTileRows / 32; ++e) {
                        const int row = lane + 32 * e;
                        if (row < rows) acc_dot(acc[u], vq[row], W[row]);
                    }
                }
            }
            mbar_arrive(empty + s);
        }
#pragma unroll
        for (int u = 0; u < kTileQ; ++u) {
            const int q = wq + kTileWarps * u;
            const CAcc tq = warp_sum(acc[u]);
            if (q < cnt && lane == 0) red[g][q] = tq;
        }
    }
    __syncthreads();
    double2* pr = a.part;
    if (tid < cnt) {
        CAcc sq = red[0][tid];
        for (int g = 1; g < kTileGroups; ++g) cacc_add(sq, red[g][tid]);
        cacc_store(pr, tid, G, blockIdx.x, sq);
        __threadfence();
    }
    if (!arrive_last(&st->counter[1])) return;
    for (int q = warp; q < cnt; q += kTileThreads / 32) {
        const double2 v = fold_one(pr, q, G, lane);
        if (lane == 0) st->h2[q] = v;
    }
    if (tid == 0) st->counter[1] = 0;
}

// w -= V h2, ||w||; then (last CTA) the Givens step of the persistent kernel
__global__ void __launch_bounds__(kThreads) k_g_upd2(GArgs a) {
    pdl_enter_g();
    GState* st = a.st;
    if (st->done || st->mode != G_ARN) return;
    const int n = a.A.n, j = st->j, cnt = j + 1;
    double2* w = vec(a, 1 + st->wcur);
    __shared__ double2 hs[kMaxDots];
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) hs[q] = st->h2[q];
    __syncthreads();
    CAcc acc = {};
    for_elems(n, gridDim.x, blockIdx.x, [&](int i) {
        double2 wi = w[i];
        for (int q0 = 0; q0 < cnt; q0 += 4) {
            double2 vq4[4];
#pragma unroll
            for (int u4 = 0; u4 < 4; ++u4)
                if (q0 + u4 < cnt) vq4[u4] = Vq(a, q0 + u4)[i];
#pragma unroll
            for (int u4 = 0; u4 < 4; ++u4)
                if (q0 + u4 < cnt) wi = cvk_add(wi, cvk_mul(cvk_neg(hs[q0 + u4]), vq4[u4]));
        }
        w[i] = wi;
        acc_norm(acc, wi);
    });
    CAcc v[1] = {acc};
    __shared__ CAcc sm[1][32];
    cta_sum_k<1, kThreads>(v, sm);
    if (threadIdx.x == 0) cacc_store(a.part + (size_t)4 * kMaxDots * gridDim.x, 0, gridDim.x, blockIdx.x, v[0]);
    if (!arrive_last(&st->counter[3])) return;
    const double2 tot = fold_one(a.part + (size_t)4 * kMaxDots * gridDim.x, 0, gridDim.x, threadIdx.x & 31);
    if (threadIdx.x != 0) return;
    st->counter[3] = 0;
    const int M = st->m;
    const double hn = sqrt(tot.x);
    st->total++;
    double2* H = st->H;
    for (int i = 0; i <= j; ++i) H[i * M + j] = cvk_add(st->h1[i], st->h2[i]);
    for (int i = 0; i < j; ++i) {
        const double2 a0 = H[i * M + j], c2 = H[(i + 1) * M + j];
        H[i * M + j] = cvk_add(cvk_scale(st->cs[i], a0), cvk_mul(st->sn[i], c2));
        H[(i + 1) * M + j] = cvk_add(cvk_mul(cvk_neg(cvk_conj(st->sn[i])), a0), cvk_scale(st->cs[i], c2));
    }
    const double2 aj = H[j * M + j];
    const double aa = sqrt(aj.x * aj.x + aj.y * aj.y);
    const double nu = sqrt(aa * aa + hn * hn);
    if (aa == 0.0) {
        st->cs[j] = 0.0; st->sn[j] = make_double2(1.0, 0.0); H[j * M + j] = make_double2(hn, 0.0);
    } else {
        st->cs[j] = aa / nu;
        st->sn[j] = cvk_scale(hn / nu, cvk_divr(aj, aa));
        H[j * M + j] = cvk_scale(nu, cvk_divr(aj, aa));
    }
    st->gv[j + 1] = cvk_mul(cvk_neg(cvk_conj(st->sn[j])), st->gv[j]);
    st->gv[j] = cvk_scale(st->cs[j], st->gv[j]);
    const double2 gj1 = st->gv[j + 1];
    const double relres = sqrt(gj1.x * gj1.x + gj1.y * gj1.y) / st->bnorm;
    st->final_relres = relres;
    ghist(a, st, relres);
    st->k = j + 1;
    bool stop = false;
    if (relres <= st->tol) { st->conv = 1; stop = true; }
    else if (hn * hn < st->brk) { st->brk_code = 7; stop = true; }
    else if (st->total >= st->max_iter) { stop = true; }
    if (stop || j + 1 == M) {
        st->stop = stop ? 1 : 0;
        back_subst(st);
        st->mode = G_RX;
        return;
    }
    st->scale = hn;
    st->wcur ^= 1;
    st->j = j + 1;
}

__global__ void __launch_bounds__(kThreads) k_g_true(GArgs a) {
    pdl_enter_g();
    GState* st = a.st;
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
    __shared__ CAcc sm[2][32];
    cta_sum_k<2, kThreads>(acc, sm);
    if (threadIdx.x == 0) {
        cacc_store(a.part, 0, gridDim.x, blockIdx.x, acc[0]);
        cacc_store(a.part, 1, gridDim.x, blockIdx.x, acc[1]);
    }
    if (!arrive_last(&st->counter[0])) return;
    const double2 bb = fold_one(a.part, 0, gridDim.x, threadIdx.x & 31);
    const double2 rr = fold_one(a.part, 1, gridDim.x, threadIdx.x & 31);
    if (threadIdx.x != 0) return;
    st->counter[0] = 0;
    double trr = 0.0;
    if (!st->skip_true) {
        const double bn = sqrt(bb.x), rn = sqrt(rr.x);
        trr = bn > 0 ? rn / bn : rn;
    }
    a.rep->converged = st->conv;
    a.rep->breakdown = st->brk_code;
    a.rep->iterations = st->total;
    a.rep->final_relres = st->final_relres;
    a.rep->true_relres = trr;
    a.rep->history_len = st->hl;
    a.rep->error = 0;
}

}  // namespace

GmresKernels gmres_kernels() {
    GmresKernels k;
    k.init = (const void*)k_g_init;
    k.x = (const void*)k_g_x;
    k.spmv = (const void*)k_g_spmv;
    k.spmv_s = (const void*)k_g_spmv_s;
    k.upd1_s = (const void*)k_g_ud_s;
    k.dots = (const void*)k_g_dots<false>;
    k.upd1 = (const void*)k_g_dots<true>;
    k.upd2 = (const void*)k_g_upd2;
    k.true_res = (const void*)k_g_true;
    return k;
}

size_t gmres_state_size() { return sizeof(GState); }
size_t gmres_args_size() { return sizeof(GArgs); }

// initial state: options (the rest is zero)
void gmres_init_state(void* host_state, double tol, long long max_iter, int m, int record, long long hist_cap) {
    GState* s = (GState*)host_state;
    s->tol = tol;
    s->max_iter = max_iter;
    s->m = m;
    s->record = record;
    s->hist_cap = hist_cap;
}

int gmres_state_done_offset() { return (int)offsetof(GState, done); }

void gmres_pack_args(void* out, const Csr& A, const double2* dinv, const double2* b, double2* x, double2* work,
                     double2* part, void* st, double* hist, DevReport* rep, int capk, int nst, int pf_rows) {
    GArgs* p = (GArgs*)out;
    p->capk = capk;
    p->nst = nst;
    p->pf_rows = pf_rows;
    p->A = A;
    p->dinv = dinv;
    p->b = b;
    p->x = x;
    p->work = work;
    p->part = part;
    p->st = (GState*)st;
    p->hist = hist;
    p->rep = rep;
}

}  // namespace cvk
