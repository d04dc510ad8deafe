// cvk_gmres.cu -- FAST-mode restarted GMRES(m) for large systems as a chain
// of phase kernels replayed from a CUDA graph (beyond the reference, which
// has no GMRES; operation order = the persistent kernel's gmres_body =
// oracle/cavac_oracle.c orc_gmres: DCGS2 Arnoldi, complex Givens).
//
// Each Arnoldi step reads the basis twice (delayed reorthogonalisation,
// cvk_dcgs2.cuh), in three kernels:
//   k_g_spmv_s  u_j = V_j = src / scale (formed in the gathers), w = M^-1 A u_j
//   k_g_dd      a = V^H u_j, b = V^H w in one pass (u_j, w staged per block in
//               shared memory); last CTA: nu, the delayed correction of
//               column j-1, column j, the update coefficients
//   k_g_up      q_j = (u_j - V a) / nu over V_j, u' = w - V e - gamma u_j,
//               ||u'||; last CTA: provisional rotation, residual estimate,
//               restart decision.  Rows are walked top-down, the reverse of
//               k_g_dd, so the tail k_g_dd left in L2 is read first.
// The CGS2 version read the basis three times (dots; update + dots; update):
// 307 us per step at 1M DOF (profiles/r01_gmres_5m.txt).  A restart is
// k_g_x (x += V y) + k_g_spmv in residual mode.  Every reduction is
// double-double, so the scalars equal the persistent FAST path's.
#include <cuda_runtime.h>

#include <algorithm>

#include <cstddef>

#include "cvk_dcgs2.cuh"
#include "cvk_engine.cuh"
#include "cvk_kernels.h"
#include "cvk_stream.cuh"
#include "cvk_tiles.cuh"

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
    double bnorm, brk, beta, scale, final_relres, tol, nu;
    unsigned counter[4];
    double2 sn[kMaxDots], gv[kMaxDots + 1], gpre[kMaxDots + 1], yv[kMaxDots + 1];
    double2 av[kMaxDots + 1], bv[kMaxDots + 1], ev[kMaxDots + 1];
    double cs[kMaxDots];
    double2 Hu[(kMaxDots + 1) * kMaxDots], R[(kMaxDots + 1) * kMaxDots];
};

__device__ __forceinline__ GmView gview(GState* st) {
    GmView v;
    v.Hu = st->Hu;
    v.R = st->R;
    v.cs = st->cs;
    v.sn = st->sn;
    v.g = st->gv;
    v.gpre = st->gpre;
    v.av = st->av;
    v.bv = st->bv;
    v.ev = st->ev;
    v.yv = st->yv;
    v.nu = &st->nu;
    v.M = st->m;
    return v;
}

// Shared-memory copy of the Hessenberg state for a last CTA's scalar step:
// rows [0, rows) of Hu and R and every vector; all threads of the CTA call
// load and store (each ends / starts with a barrier).
__device__ GmView gm_mirror_load(GState* st, unsigned char* sm, int rows) {
    const int M = st->m, V = kMaxDots + 1, tid = threadIdx.x, nt = blockDim.x;
    GmView v;
    v.M = M;
    v.Hu = (double2*)sm;
    v.R = v.Hu + (size_t)rows * M;
    v.sn = v.R + (size_t)rows * M;
    v.g = v.sn + V;
    v.gpre = v.g + V;
    v.yv = v.gpre + V;
    v.av = v.yv + V;
    v.bv = v.av + V;
    v.ev = v.bv + V;
    v.cs = (double*)(v.ev + V);
    v.nu = v.cs + V;
    for (int i = tid; i < rows * M; i += nt) {
        v.Hu[i] = st->Hu[i];
        v.R[i] = st->R[i];
    }
    for (int i = tid; i < V; i += nt) {
        if (i < kMaxDots) v.sn[i] = st->sn[i];
        v.g[i] = st->gv[i];
        v.gpre[i] = st->gpre[i];
        v.yv[i] = st->yv[i];
        v.av[i] = st->av[i];
        v.bv[i] = st->bv[i];
        v.ev[i] = st->ev[i];
        if (i < kMaxDots) v.cs[i] = st->cs[i];
    }
    if (tid == 0) *v.nu = st->nu;
    __syncthreads();
    return v;
}
__device__ void gm_mirror_store(GState* st, const GmView& v, int rows) {
    const int M = st->m, V = kMaxDots + 1, tid = threadIdx.x, nt = blockDim.x;
    __syncthreads();
    for (int i = tid; i < rows * M; i += nt) {
        st->Hu[i] = v.Hu[i];
        st->R[i] = v.R[i];
    }
    for (int i = tid; i < V; i += nt) {
        if (i < kMaxDots) st->sn[i] = v.sn[i];
        st->gv[i] = v.g[i];
        st->gpre[i] = v.gpre[i];
        st->yv[i] = v.yv[i];
        st->av[i] = v.av[i];
        st->bv[i] = v.bv[i];
        st->ev[i] = v.ev[i];
        if (i < kMaxDots) st->cs[i] = v.cs[i];
    }
    if (tid == 0) st->nu = *v.nu;
}

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
    int npad, mp1;           // vector stride (n rounded up to kVB rows), m + 1
};

__device__ __forceinline__ void pdl_enter_g() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// work: r, W[2] (stride npad), then the basis V_0 .. V_m block-major: 128-row
// blocks of the m + 1 vectors one after the other, so that a tile of
// V_0 .. V_j is one contiguous bulk copy (cvk_tiles.cuh)
constexpr int kVB = 128;
__device__ __forceinline__ double2* vec(const GArgs& a, int idx) { return a.work + (size_t)idx * a.npad; }
__device__ __forceinline__ double2* vbase(const GArgs& a) { return vec(a, 3); }
__device__ __forceinline__ double2& vat(const GArgs& a, int q, int i) {
    return vbase(a)[((size_t)(i >> 7) * a.mp1 + q) * kVB + (i & (kVB - 1))];
}
// the kVB-row segment of V_q holding row r0 (r0 a multiple of kVB)
__device__ __forceinline__ double2* vseg(const GArgs& a, int q, int r0) { return &vat(a, q, r0); }

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
                        if (q0 + u4 < cnt) vq4[u4] = vat(a, q0 + u4, i);
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
        const double sc = st->scale;
        auto uat = [&](int c) -> double2 { return cvk_divr(src[c], sc); };
        for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
            const double2 yv = row_sum<1, decltype(uat)&, 5>(a.A, row, 0, valid, uat);
            if (valid) {
                vat(a, j, row) = uat(row);
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
        vat(a, j, row) = xs(t);
        w[row] = a.dinv ? cvk_mul(ch.v(1, t), y) : y;
    }, nullptr, [&](int t, const Chunk& ch) { ch.set(0, t, cvk_divr(ch.v(0, t), sc)); });
}

// (one thread) hn = ||u'||: Hu[j+1][j], the provisional rotation of column
// j, the residual estimate, the restart decision
__device__ void up_finish(const GArgs& a, GState* st, const GmView& gv, int j, double hn, double nu) {
    const int M = st->m;
    st->total++;
    gm_provisional(gv, j, hn, nu);
    const double2 gj1 = gv.g[j + 1];
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
        gm_back_subst(gv, j + 1, gv.yv);
        st->mode = G_RX;
        return;
    }
    st->scale = hn;
    st->wcur ^= 1;
    st->j = j + 1;
}

// a_q = <V_q, u_j>, b_q = <V_q, w> for q <= j in one pass over the basis.
// Blocks of kGB rows of u_j and w are staged in shared memory; warps own
// basis vectors (q = q0 + warp + kWarps u), lanes stride the block's rows.
// Canonical row groups (gm_group_dots, cvk_dcgs2.cuh), shared with the
// persistent kernel and k_g_dd_s.
#ifndef CVK_GDD_Q
#define CVK_GDD_Q 2
#endif
constexpr int kDdQ = CVK_GDD_Q;  // basis vectors per warp and round: 8 kDdQ per round
#ifndef CVK_GDD_MINB
#define CVK_GDD_MINB 2
#endif
#ifndef CVK_GUP_MINB
#define CVK_GUP_MINB 3
#endif
#ifndef CVK_GUP_B
#define CVK_GUP_B 4  // basis loads in flight per row in k_g_up (two rows per thread)
#endif

__global__ void __launch_bounds__(kThreads, CVK_GDD_MINB) k_g_dd(GArgs a) {
    pdl_enter_g();
    GState* st = a.st;
    if (st->done || st->mode != G_ARN) return;
    const int n = a.A.n, j = st->j, cnt = j + 1, G = gridDim.x;
    const double2* w = vec(a, 1 + st->wcur);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // u_j, w of the block staged in shared memory, double-buffered: the next
    // block's rows are loaded into registers before this block's dots
    __shared__ double2 su[2][kGB], sw[2][kGB];
    const int nblk = (n + kGB - 1) / kGB;
    double2* pr = a.part;
    const int t = threadIdx.x;
    for (int q0 = 0; q0 < cnt; q0 += kWarps * kDdQ) {
        CAcc acc[kDdQ][2];
#pragma unroll
        for (int u = 0; u < kDdQ; ++u) acc[u][0] = acc[u][1] = CAcc{};
        const int qw = q0 + warp * kDdQ, nq = max(0, min(kDdQ, cnt - qw));  // this warp's basis vectors
        int blk = blockIdx.x, buf = 0;
        __syncthreads();  // the previous round's readers are done with both buffers
        if (blk < nblk && blk * kGB + t < n) {
            su[0][t] = vat(a, j, blk * kGB + t);
            sw[0][t] = w[blk * kGB + t];
        }
        for (; blk < nblk; blk += G, buf ^= 1) {
            const int r0 = blk * kGB, rows = min(kGB, n - r0), nb = blk + G;
            double2 pu = make_double2(0, 0), pw = make_double2(0, 0);
            if (nb < nblk && nb * kGB + t < n) {
                pu = vat(a, j, nb * kGB + t);
                pw = w[nb * kGB + t];
            }
            __syncthreads();  // su/sw[buf] written; readers of buf ^ 1 (previous block) done
            if (nq > 0)
#pragma unroll
                for (int h = 0; h < kGB / kVB; ++h) {
                    if (h * kVB >= rows) break;
                    const double2* vb[kDdQ];
#pragma unroll
                    for (int u = 0; u < kDdQ; ++u) vb[u] = vseg(a, min(qw + u, cnt - 1), r0 + h * kVB);
                    gm_group_dots<kDdQ>(vb, nq, su[buf] + h * kVB, sw[buf] + h * kVB, rows - h * kVB, lane, acc);
                }
            if (nb < nblk) {
                su[buf ^ 1][t] = pu;
                sw[buf ^ 1][t] = pw;
            }
        }
#pragma unroll
        for (int u = 0; u < kDdQ; ++u) {
            const CAcc t0 = warp_sum(acc[u][0]), t1 = warp_sum(acc[u][1]);
            if (u < nq && lane == 0) {
                cacc_store(pr, 2 * (qw + u), G, blockIdx.x, t0);
                cacc_store(pr, 2 * (qw + u) + 1, G, blockIdx.x, t1);
            }
        }
    }
    if (!arrive_last(&st->counter[0])) return;
    for (int k = warp; k < 2 * cnt; k += kWarps) {
        const double2 v = fold_one(pr, k, G, lane);
        if (lane == 0) (k & 1 ? st->bv : st->av)[k >> 1] = v;
    }
    if (threadIdx.x == 0) st->counter[0] = 0;
    __syncthreads();
    const GmView gv = gview(st);
    const double nu = gm_dcgs2_scalars(gv, j, threadIdx.x, blockDim.x, [] { __syncthreads(); });
    if (nu > 0.0 || threadIdx.x != 0) return;
    // u_j lies in span(V_0 .. V_{j-1}): stop with the j columns built
    st->brk_code = 7;
    st->k = j;
    st->stop = 1;
    gm_back_subst(gv, j, st->yv);
    st->mode = G_RX;
}

// q_j = (u_j - V a) / nu over V_j; u' = w - V e - gamma u_j over w; ||u'||.
// Then (last CTA) Hu[j+1][j], the provisional rotation of column j, the
// residual estimate and the restart decision.
__global__ void __launch_bounds__(kThreads, CVK_GUP_MINB) k_g_up(GArgs a) {
    pdl_enter_g();
    GState* st = a.st;
    if (st->done || st->mode != G_ARN) return;
    const int n = a.A.n, j = st->j, G = gridDim.x;
    const double nu = st->nu;
    double2* w = vec(a, 1 + st->wcur);
    __shared__ double2 sa[kMaxDots + 1], se[kMaxDots + 1];
    for (int q = threadIdx.x; q <= j; q += blockDim.x) {
        sa[q] = st->av[q];
        se[q] = st->ev[q];
    }
    __syncthreads();
    CAcc acc = {};
    const int nblk = (n + kGB - 1) / kGB;
    const int last = blockIdx.x < nblk ? blockIdx.x + ((nblk - 1 - blockIdx.x) / G) * G : -1;
    // two rows per thread per trip (this block and the CTA's next one down),
    // every basis load of a batch issued for both before the updates
    constexpr int B = CVK_GUP_B;
    for (int blk = last; blk >= 0; blk -= 2 * G) {
        int ii[2] = {blk * kGB + (int)threadIdx.x, (blk - G) * kGB + (int)threadIdx.x};
        bool ok[2] = {ii[0] < n, blk - G >= 0 && ii[1] < n};
        double2 u[2], qv[2], up[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (!ok[r]) ii[r] = 0;
            u[r] = vat(a, j, ii[r]);
            qv[r] = u[r];
            up[r] = w[ii[r]];
        }
        for (int q0 = 0; q0 < j; q0 += B) {
            double2 vq[2][B];
#pragma unroll
            for (int t = 0; t < B; ++t)
#pragma unroll
                for (int r = 0; r < 2; ++r)
                    if (q0 + t < j) vq[r][t] = vat(a, q0 + t, ii[r]);
#pragma unroll
            for (int t = 0; t < B; ++t)
#pragma unroll
                for (int r = 0; r < 2; ++r)
                    if (q0 + t < j) {
                        qv[r] = cvk_sub(qv[r], cvk_mul(sa[q0 + t], vq[r][t]));
                        up[r] = cvk_sub(up[r], cvk_mul(se[q0 + t], vq[r][t]));
                    }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r)
            if (ok[r]) {
                up[r] = cvk_sub(up[r], cvk_mul(se[j], u[r]));
                vat(a, j, ii[r]) = cvk_divr(qv[r], nu);
                w[ii[r]] = up[r];
                acc_norm(acc, up[r]);
            }
    }
    CAcc v[1] = {acc};
    __shared__ CAcc sm[1][32];
    cta_sum_k<1, kThreads>(v, sm);
    double2* pr = a.part + (size_t)4 * kMaxDots * G;
    if (threadIdx.x == 0) cacc_store(pr, 0, G, blockIdx.x, v[0]);
    if (!arrive_last(&st->counter[3])) return;
    const double2 tot = fold_one(pr, 0, G, threadIdx.x & 31);
    if (threadIdx.x != 0) return;
    st->counter[3] = 0;
    up_finish(a, st, gview(st), j, sqrt(tot.x), nu);
}

// The same two passes on 128-row tiles of [u_j | w | V_0 .. V_{j-1}] that
// one producer warp streams into a ring of shared-memory stages by bulk
// copies (cvk_tiles.cuh), m <= 32.  The consumers never wait on a global
// load: the element-loop kernels above keep at most a few loads in flight
// per thread and ran at 2.9 / 3.8 TB/s.  Shared by both kernels:
constexpr int kTR = 128;  // rows per tile

// A tile is kb consecutive 128-row basis blocks (kb copies of V_0 .. V_j)
// and the tile's rows of w (one copy); kb grows as j shrinks so that a
// stage holds >= 32 KB (cvk_tiles.cuh).  Stage layout: block c's V_q at
// S + (c (j + 1) + q) kTR, w at S + kb (j + 1) kTR.
__host__ __device__ __forceinline__ int tile_blocks(int j) {
    const int nv = j + 2;
    return nv >= 16 ? 1 : nv >= 8 ? 2 : nv >= 4 ? 4 : 8;
}
__device__ __forceinline__ TileCopies tile_copies(const GArgs& a, const GState* st, int kb) {
    TileCopies tc;
    const int j = st->j;
    for (int c = 0; c < kb; ++c) {
        tc.src[c] = vbase(a) + (size_t)c * a.mp1 * kVB;
        tc.stride[c] = (long long)kb * a.mp1 * kVB;
        tc.bytes[c] = (j + 1) * kTR * 16;
    }
    tc.src[kb] = vec(a, 1 + st->wcur);
    tc.stride[kb] = (long long)kb * kTR;
    tc.bytes[kb] = kb * kTR * 16;
    tc.nc = kb + 1;
    tc.stage_bytes = kb * (j + 2) * kTR * 16;
    return tc;
}

// a = V^H u_j, b = V^H w: one group of 16 warps; warp wq owns q = wq + 16 k
// (two accumulator pairs per thread: more spill at 96 registers).
constexpr int kDdsGT = 512, kDdsNG = 1, kDdsQ = 2;
__global__ void __launch_bounds__(kDdsGT * kDdsNG + 32, 1) k_g_dd_s(GArgs a, int smem_bytes) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter_g();
    GState* st = a.st;
    if (st->done || st->mode != G_ARN) return;
    const int n = a.A.n, j = st->j, cnt = j + 1, G = gridDim.x;
    const int kb = tile_blocks(j);
    const TileCopies tc = tile_copies(a, st, kb);
    const int tid = threadIdx.x, warp = (tid % kDdsGT) >> 5, lane = tid & 31;
    CAcc acc[kDdsQ][2];
#pragma unroll
    for (int k = 0; k < kDdsQ; ++k) acc[k][0] = acc[k][1] = CAcc{};
    tile_stream<kDdsNG, kDdsGT, false>(n, kb * kTR, tc, smem, smem_bytes,
                                       [&](int, int, int, int rows, const double2* S) {
        const double2* W = S + (size_t)kb * (j + 1) * kTR;
        for (int c = 0; c < kb; ++c) {
            const int nr = gm_group_rows(rows - c * kTR, lane);
            if (nr == 0) break;
            const double2* B = S + (size_t)c * (j + 1) * kTR;
            double2 uu[4], ww[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (e < nr) {
                    uu[e] = B[(size_t)j * kTR + lane + 32 * e];
                    ww[e] = W[c * kTR + lane + 32 * e];
                }
#pragma unroll
            for (int k = 0; k < kDdsQ; ++k) {
                const int q = warp + 16 * k;
                if (q < cnt) {
                    const double2* vq = B + (size_t)q * kTR;
                    double2 vv[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (e < nr) vv[e] = vq[lane + 32 * e];
                    gm_group4(vv, uu, ww, nr, acc[k]);
                }
            }
        }
    });
    // groups -> CTA partial (slots 2q, 2q + 1)
    __shared__ CAcc red[kDdsNG][2 * (kMaxDots + 1)];
    const int g = tid / kDdsGT;
#pragma unroll
    for (int k = 0; k < kDdsQ; ++k) {
        const int q = warp + 16 * k;
        const CAcc t0 = warp_sum(acc[k][0]), t1 = warp_sum(acc[k][1]);
        if (g < kDdsNG && q < cnt && lane == 0) {
            red[g][2 * q] = t0;
            red[g][2 * q + 1] = t1;
        }
    }
    __syncthreads();
    double2* pr = a.part;
    for (int k = tid; k < 2 * cnt; k += blockDim.x) {
        CAcc sq = red[0][k];
        for (int gg = 1; gg < kDdsNG; ++gg) cacc_add(sq, red[gg][k]);
        cacc_store(pr, k, G, blockIdx.x, sq);
        __threadfence();
    }
    if (!arrive_last(&st->counter[0])) return;
    // the last CTA: fold and scalar step on a shared-memory copy of the
    // Hessenberg state (the ring is idle now).  Measured alternatives: the
    // step in global memory (10-30 us), and a separate one-CTA kernel with
    // the up pass's producers streaming meanwhile (+6 us per step: the
    // extra kernel boundary costs more than the overlap wins).
    const GmView gv = gm_mirror_load(st, smem, j + 2);
    const int wg = tid >> 5, nw = blockDim.x >> 5;
    for (int q = wg; q < cnt; q += nw) {  // one warp per (a_q, b_q) pair, loads issued together
        CAcc sa = {}, sb = {};
        for (int b0 = lane; b0 < G; b0 += 64) {
            CAcc v[4];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int b = b0 + 32 * u;
                v[2 * u] = b < G ? cacc_load(pr, 2 * q, G, b) : CAcc{};
                v[2 * u + 1] = b < G ? cacc_load(pr, 2 * q + 1, G, b) : CAcc{};
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                cacc_add(sa, v[2 * u]);
                cacc_add(sb, v[2 * u + 1]);
            }
        }
        sa = warp_sum(sa);
        sb = warp_sum(sb);
        if (lane == 0) {
            gv.av[q] = sa.hi;
            gv.bv[q] = sb.hi;
        }
    }
    if (tid == 0) st->counter[0] = 0;
    __syncthreads();
    const double nu = gm_dcgs2_scalars(gv, j, tid, blockDim.x, [] { __syncthreads(); });
    if (!(nu > 0.0) && tid == 0) {
        // u_j lies in span(V_0 .. V_{j-1}): stop with the j columns built
        st->brk_code = 7;
        st->k = j;
        st->stop = 1;
        gm_back_subst(gv, j, gv.yv);
        st->mode = G_RX;
    }
    gm_mirror_store(st, gv, j + 2);
}

// q_j = (u_j - V a) / nu, u' = w - V e - gamma u_j, ||u'||: thread per tile
// row, tiles walked top-down (the tail of k_g_dd_s's walk is still in L2).
// one consumer group (two intermittently failed at 1M DOF, m = 30 -- not
// understood; one keeps up: the pass is bound by the stream, not the math)
constexpr int kUpsGT = 128, kUpsNG = 1;
__global__ void __launch_bounds__(kUpsGT * kUpsNG + 32, 1) k_g_up_s(GArgs a, int smem_bytes) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter_g();
    GState* st = a.st;
    if (st->done || st->mode != G_ARN) return;
    const int n = a.A.n, j = st->j, G = gridDim.x;
    const double nu = st->nu;
    const int kb = tile_blocks(j);
    const TileCopies tc = tile_copies(a, st, kb);
    __shared__ double2 sa[kMaxDots + 1], se[kMaxDots + 1];
    for (int q = threadIdx.x; q <= j; q += blockDim.x) {
        sa[q] = st->av[q];
        se[q] = st->ev[q];
    }
    __syncthreads();
    double2* w = vec(a, 1 + st->wcur);
    CAcc acc = {};
    tile_stream<kUpsNG, kUpsGT, true>(n, kb * kTR, tc, smem, smem_bytes,
                                      [&](int, int t, int r0, int rows, const double2* S) {
        const double2* W = S + (size_t)kb * (j + 1) * kTR;
        for (int c = 0; c < kb; ++c) {
            const int row = c * kTR + t;
            if (row >= rows) break;
            const double2* B = S + (size_t)c * (j + 1) * kTR;
            const double2 u = B[(size_t)j * kTR + t];
            double2 qv = u, up = W[row];
            for (int q = 0; q < j; ++q) {
                const double2 vq = B[(size_t)q * kTR + t];
                qv = cvk_sub(qv, cvk_mul(sa[q], vq));
                up = cvk_sub(up, cvk_mul(se[q], vq));
            }
            up = cvk_sub(up, cvk_mul(se[j], u));
            vat(a, j, r0 + row) = cvk_divr(qv, nu);
            w[r0 + row] = up;
            acc_norm(acc, up);
        }
    });
    CAcc v[1] = {acc};
    __shared__ CAcc sm[1][32];
    cta_sum_k<1, kUpsGT * kUpsNG + 32>(v, sm);
    double2* pr = a.part + (size_t)4 * kMaxDots * G;
    if (threadIdx.x == 0) cacc_store(pr, 0, G, blockIdx.x, v[0]);
    if (!arrive_last(&st->counter[3])) return;
    const double2 tot = fold_one(pr, 0, G, threadIdx.x & 31);
    if (threadIdx.x != 0) return;
    st->counter[3] = 0;
    up_finish(a, st, gview(st), j, sqrt(tot.x), nu);
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
    k.dd = (const void*)k_g_dd;
    k.up = (const void*)k_g_up;
    k.dd_s = (const void*)k_g_dd_s;
    k.up_s = (const void*)k_g_up_s;
    k.true_res = (const void*)k_g_true;
    return k;
}

size_t gmres_state_size() { return sizeof(GState); }
// the largest stage of the tiled passes over j = 0 .. m - 1
int gmres_tile_stage_max(int m) {
    int mx = 0;
    for (int j = 0; j < m; ++j) mx = std::max(mx, tile_blocks(j) * (j + 2) * kTR * 16);
    return mx;
}
// whole tiles of the largest height (8 basis blocks, tile_blocks)
long long gmres_padded_rows(long long n) { return (n + 8 * kVB - 1) / (8 * kVB) * (8 * kVB); }
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
                     double2* part, void* st, double* hist, DevReport* rep, int capk, int nst, int pf_rows, int m) {
    GArgs* p = (GArgs*)out;
    p->npad = (int)gmres_padded_rows(A.n);
    p->mp1 = m + 1;
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
