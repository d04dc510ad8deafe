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

#include <cstddef>

#include "cvk_dcgs2.cuh"
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
    v.nu = &st->nu;
    v.M = st->m;
    return v;
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

// a_q = <V_q, u_j>, b_q = <V_q, w> for q <= j in one pass over the basis.
// Blocks of kGB rows of u_j and w are staged in shared memory; warps own
// basis vectors (q = q0 + warp + kWarps u), lanes stride the block's rows.
constexpr int kDdQ = 4;  // basis vectors per warp and round: 32 per round

__global__ void __launch_bounds__(kThreads) k_g_dd(GArgs a) {
    pdl_enter_g();
    GState* st = a.st;
    if (st->done || st->mode != G_ARN) return;
    const int n = a.A.n, j = st->j, cnt = j + 1, G = gridDim.x;
    const double2* uj = Vq(a, j);
    const double2* w = vec(a, 1 + st->wcur);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ double2 su[kGB], sw[kGB];
    const int nblk = (n + kGB - 1) / kGB;
    double2* pr = a.part;
    for (int q0 = 0; q0 < cnt; q0 += kWarps * kDdQ) {
        CAcc acc[kDdQ][2];
#pragma unroll
        for (int u = 0; u < kDdQ; ++u) acc[u][0] = acc[u][1] = CAcc{};
        for (int blk = blockIdx.x; blk < nblk; blk += G) {
            const int r0 = blk * kGB, rows = min(kGB, n - r0);
            __syncthreads();
            if ((int)threadIdx.x < rows) {
                su[threadIdx.x] = uj[r0 + threadIdx.x];
                sw[threadIdx.x] = w[r0 + threadIdx.x];
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < kDdQ; ++u) {
                const int q = q0 + warp + kWarps * u;
                if (q >= cnt) break;
                const double2* vq = Vq(a, q) + r0;
                double2 vv[kGB / 32];
#pragma unroll
                for (int e = 0; e < kGB / 32; ++e) {
                    const int row = lane + 32 * e;
                    if (row < rows) vv[e] = vq[row];
                }
#pragma unroll
                for (int e = 0; e < kGB / 32; ++e) {
                    const int row = lane + 32 * e;
                    if (row < rows) {
                        acc_dot(acc[u][0], vv[e], su[row]);
                        acc_dot(acc[u][1], vv[e], sw[row]);
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kDdQ; ++u) {
            const int q = q0 + warp + kWarps * u;
            const CAcc t0 = warp_sum(acc[u][0]), t1 = warp_sum(acc[u][1]);
            if (q < cnt && lane == 0) {
                cacc_store(pr, 2 * q, G, blockIdx.x, t0);
                cacc_store(pr, 2 * q + 1, G, blockIdx.x, t1);
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
__global__ void __launch_bounds__(kThreads) k_g_up(GArgs a) {
    pdl_enter_g();
    GState* st = a.st;
    if (st->done || st->mode != G_ARN) return;
    const int n = a.A.n, j = st->j, G = gridDim.x;
    const double nu = st->nu;
    double2* w = vec(a, 1 + st->wcur);
    double2* uj = Vq(a, j);
    __shared__ double2 sa[kMaxDots + 1], se[kMaxDots + 1];
    for (int q = threadIdx.x; q <= j; q += blockDim.x) {
        sa[q] = st->av[q];
        se[q] = st->ev[q];
    }
    __syncthreads();
    CAcc acc = {};
    const int nblk = (n + kGB - 1) / kGB;
    const int last = blockIdx.x < nblk ? blockIdx.x + ((nblk - 1 - blockIdx.x) / G) * G : -1;
    for (int blk = last; blk >= 0; blk -= G) {
        const int i = blk * kGB + threadIdx.x;
        if (i >= n) continue;
        const double2 u = uj[i];
        double2 qv = u, up = w[i];
        constexpr int B = 8;
        for (int q0 = 0; q0 < j; q0 += B) {
            double2 vq[B];
#pragma unroll
            for (int t = 0; t < B; ++t)
                if (q0 + t < j) vq[t] = Vq(a, q0 + t)[i];
#pragma unroll
            for (int t = 0; t < B; ++t)
                if (q0 + t < j) {
                    qv = cvk_sub(qv, cvk_mul(sa[q0 + t], vq[t]));
                    up = cvk_sub(up, cvk_mul(se[q0 + t], vq[t]));
                }
        }
        up = cvk_sub(up, cvk_mul(se[j], u));
        uj[i] = cvk_divr(qv, nu);
        w[i] = up;
        acc_norm(acc, up);
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
    const int M = st->m;
    const double hn = sqrt(tot.x);
    st->total++;
    const GmView gv = gview(st);
    gm_provisional(gv, j, hn, nu);
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
        gm_back_subst(gv, j + 1, st->yv);
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
    k.dd = (const void*)k_g_dd;
    k.up = (const void*)k_g_up;
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
