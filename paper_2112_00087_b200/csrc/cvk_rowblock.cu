// cvk_rowblock.cu -- row-block global BiCGSTAB: one rank's contiguous block
// of rows of the global system (SURVEY.md 8(e) mode 1).
//
// The reference solves on one address space (krylov.cpp:57-138).  Here the
// rows are split over ranks (one per GPU, or several blocks on one device);
// each reduction phase of the fused BiCGSTAB schedule (cvk_phased.cu k_bi_*)
// becomes
//
//   k_rb_<phase>  the phase over the rank's own rows; its last CTA folds the
//                 CTA partials into the rank's double-double totals and
//                 writes them to the rank's exchange slot
//   k_rb_pack     boundary values other ranks gather (r after C, p and v
//                 after A, x before the true residual) into the same slot
//   all-gather    of every rank's slot (NCCL / gloo / device copies)
//   k_rb_post     every rank folds the ranks' totals in rank order and runs
//                 the reference's scalar logic (identical on all ranks), and
//                 unpacks its halo from the gathered slots
//
// so there is exactly one collective per reduction, carrying both the
// reduction and the halo.  The halo needs no extra exchange step because p
// is formed inside the SpMV gathers from r, p_old and v, whose halo values
// arrive with the preceding phases.
//
// Per-row SpMV order, per-element roundings and the double-double reductions
// are those of the single-device FAST kernels, so iterates are bitwise a
// single-device solve for any number of blocks
// (tests/test_gpu_rowblock.py).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cavac_b200.h"
#include "cvk_engine.cuh"
#include "cvk_kernels.h"
#include "cvk_phased.h"
#include "cvk_stream.cuh"

namespace cvk {
namespace {

constexpr int kHdr = 16;   // exchange slot header: up to 4 complex dd totals (hi.x hi.y lo.x lo.y)
constexpr int kRbBatch = 2;  // as cvk_phased.cu CVK_BATCH

struct RBArgs {
    Csr A;               // n = own rows; columns < n_own + n_halo
    long long nv;        // vector stride
    const double2* dinv;
    const double2* b;
    double2* work;       // x r sh s t p0 p1 v0 v1, stride nv
    double2* part;       // CTA partials (cacc_store layout, 3 reductions)
    PState* st;
    double* hist;
    DevReport* rep;
    double* send;        // this rank's exchange slot
    const double* recv;  // nranks slots
    int nranks, slot;    // slot: doubles per rank
    const int* send_rows;
    int n_send, max_send;
    const int* halo_src;
    int n_halo;
    int capk;            // streamed SpMV phases: chunk nnz capacity, ring depths, L2 prefetch window
    int nst[2];
    int pf_rows;
    // peer-to-peer exchange (cvk_rowblock_p2p_*): every rank's pack kernel
    // writes its slot straight into every rank's mailbox (NVLink stores) and
    // raises its flag there; the post kernel waits on the local flags.
    int p2p, rank, flag_bytes;
    unsigned char* const* peers;  // [nranks] mailbox bases (own included)
    unsigned char* mbox;          // own mailbox: [flags | seq | 2 x nranks slots]
    unsigned* pack_ctr;           // CTA arrivals of the pack kernel
};

enum { VX = 0, VR, VSH, VS, VT, VP0, VP1, VV0, VV1, kRbVecs };

__device__ __forceinline__ double2* vec(const RBArgs& a, int k) { return a.work + (size_t)k * a.nv; }

__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// CTA partials -> the rank's double-double totals in send[0 .. 4K) (last CTA)
template <int K, int NT = kThreads>
__device__ void rank_total(const CAcc (&acc)[K], const RBArgs& a, unsigned* counter) {
    __shared__ CAcc sm[K][32];
    __shared__ int s_last;
    const int G = gridDim.x;
    CAcc v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = acc[k];
    cta_sum_k<K, NT>(v, sm);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) cacc_store(a.part, k, G, blockIdx.x, v[k]);
        __threadfence();
        s_last = (atomicAdd(counter, 1u) == (unsigned)G - 1u);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    CAcc s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) s[k] = CAcc{};
#pragma unroll 1
    for (int q = threadIdx.x; q < G; q += NT) {
#pragma unroll
        for (int k = 0; k < K; ++k) cacc_add(s[k], cacc_load(a.part, k, G, q));
    }
    cta_sum_k<K, NT>(s, sm);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            a.send[4 * k + 0] = s[k].hi.x;
            a.send[4 * k + 1] = s[k].hi.y;
            a.send[4 * k + 2] = s[k].lo.x;
            a.send[4 * k + 3] = s[k].lo.y;
        }
        *counter = 0u;
    }
}

// mailbox pieces (p2p mode)
__device__ __forceinline__ unsigned long long* mb_flags(unsigned char* base) { return (unsigned long long*)base; }
__device__ __forceinline__ unsigned long long* mb_seq(const RBArgs& a) {
    return (unsigned long long*)(a.mbox + a.flag_bytes);
}
__device__ __forceinline__ double* mb_data(unsigned char* base, const RBArgs& a, int parity) {
    return (double*)(base + a.flag_bytes + 256) + (size_t)parity * a.nranks * a.slot;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// the ranks' totals of reduction k, folded in rank order
__device__ double2 fold_ranks(const RBArgs& a, int k, const double* recv) {
    CAcc s = {};
    for (int q = 0; q < a.nranks; ++q) {
        const double* p = recv + (size_t)q * a.slot + 4 * k;
        CAcc t;
        t.hi = make_double2(p[0], p[1]);
        t.lo = make_double2(p[2], p[3]);
        cacc_add(s, t);
    }
    return s.hi;
}

__device__ __forceinline__ void rb_hist(const RBArgs& a, PState* st, double v) {
    if (!st->record) return;
    if (st->hist_len < st->hist_cap) a.hist[st->hist_len] = v;
    st->hist_len++;
}

// top of iteration st->it (krylov.cpp:81-96)
__device__ void rb_top(PState* st) {
    if (st->it > st->max_iter) { st->done = 1; return; }
    if (cvk_abs(st->rho_new) < st->brk) {
        st->done = 1; st->brk_code = 1; st->iters = st->it - 1;
        return;
    }
    if (!st->first) st->beta = cvk_mul(cvk_cdiv(st->rho_new, st->rho), cvk_cdiv(st->alpha, st->omega));
    st->rho = st->rho_new;
}

// ------------------------------------------------------------ local phases

__global__ void __launch_bounds__(kThreads) k_rb_init(RBArgs a) {
    pdl_wait();
    const int n = a.A.n;
    double2* r = vec(a, VR);
    double2* sh = vec(a, VSH);
    double2* x = vec(a, VX);
    CAcc acc[2] = {};
    for_elems(n, gridDim.x, blockIdx.x, [&](int i) {
        const double2 ri = prec_apply(a.dinv, i, __ldg(a.b + i));
        r[i] = ri;
        sh[i] = ri;
        x[i] = make_double2(0.0, 0.0);
        acc_norm(acc[0], ri);
        acc_dot(acc[1], ri, ri);
    });
    rank_total<2>(acc, a, &a.st->counter[0]);
}

// p = r + beta (p - omega v) formed in the gathers; v = M^-1 A p; <shadow, v>
__global__ void __launch_bounds__(kThreads) k_rb_a(RBArgs a) {
    pdl_wait();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n, cur = st->cur;
    const bool first = st->first != 0;
    const double2 beta = st->beta, nom = cvk_neg(st->omega);
    const double2* __restrict__ r = vec(a, VR);
    const double2* __restrict__ pc = vec(a, cur ? VP1 : VP0);
    const double2* __restrict__ vc = vec(a, cur ? VV1 : VV0);
    double2* __restrict__ pn = vec(a, cur ? VP0 : VP1);
    double2* __restrict__ vn = vec(a, cur ? VV0 : VV1);
    const double2* __restrict__ sh = vec(a, VSH);
    auto pnew = [&](int c) -> double2 {
        const double2 rc = r[c];
        if (first) return rc;
        return cvk_add(cvk_mul(beta, cvk_add(pc[c], cvk_mul(nom, vc[c]))), rc);
    };
    CAcc acc[1] = {};
    for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
        const double2 y = row_sum<1, decltype(pnew)&, kRbBatch>(a.A, row, 0, valid, pnew);
        if (valid) {
            const double2 vi = prec_apply(a.dinv, row, y);
            pn[row] = pnew(row);
            vn[row] = vi;
            acc_dot(acc[0], sh[row], vi);
        }
    });
    rank_total<1>(acc, a, &st->counter[1]);
}

// s = r - alpha v formed in the gathers; t = M^-1 A s; x += alpha p
__global__ void __launch_bounds__(kThreads) k_rb_b(RBArgs a) {
    pdl_wait();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n, cur = st->cur;
    const double2 alpha = st->alpha, nal = cvk_neg(st->alpha);
    const double2* __restrict__ r = vec(a, VR);
    const double2* __restrict__ pn = vec(a, cur ? VP0 : VP1);
    const double2* __restrict__ vn = vec(a, cur ? VV0 : VV1);
    double2* __restrict__ s = vec(a, VS);
    double2* __restrict__ t = vec(a, VT);
    double2* __restrict__ x = vec(a, VX);
    auto sval = [&](int c) -> double2 { return cvk_add(r[c], cvk_mul(nal, vn[c])); };
    CAcc acc[3] = {};
    for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
        const double2 y = row_sum<1, decltype(sval)&, kRbBatch>(a.A, row, 0, valid, sval);
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
    rank_total<3>(acc, a, &st->counter[2]);
}

// ---- streamed (TMA ring) SpMV phases: cvk_phased.cu k_bi_a_s / k_bi_b_s
// with the rank's totals instead of the scalar logic

__global__ void __launch_bounds__(kStreamThreads, 1) k_rb_a_s(RBArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_wait();
    PState* st = a.st;
    if (st->done) return;
    const int cur = st->cur;
    const bool first = st->first != 0;
    const double2 beta = st->beta, nom = cvk_neg(st->omega);
    const double2* __restrict__ r = vec(a, VR);
    const double2* __restrict__ pc = vec(a, cur ? VP1 : VP0);
    const double2* __restrict__ vc = vec(a, cur ? VV1 : VV0);
    double2* __restrict__ pn = vec(a, cur ? VP0 : VP1);
    double2* __restrict__ vn = vec(a, cur ? VV0 : VV1);
    const double2* vecs[5] = {r, pc, vc, vec(a, VSH), a.dinv};
    StreamLayout L{a.capk, 5, a.nst[0]};
    L.ngather = 3;
    L.pf_rows = a.pf_rows;
    CAcc acc[1] = {};
    stream_rows(a.A, L, vecs, smem, [&](int t, const Chunk& ch) {
        auto xs = [&](int l) -> double2 {  // slot 0 of the chunk rows holds p_new (pre)
            const double2 rc = ch.v(0, l);
            if (first || l < kStreamRows) return rc;
            return cvk_add(cvk_mul(beta, cvk_add(ch.v(1, l), cvk_mul(nom, ch.v(2, l)))), rc);
        };
        auto xg = [&](int c) -> double2 {
            const double2 rc = r[c];
            if (first) return rc;
            return cvk_add(cvk_mul(beta, cvk_add(pc[c], cvk_mul(nom, vc[c]))), rc);
        };
        const double2 y = chunk_row_sum<kRbBatch>(ch, t, xs, xg);
        const double2 vi = a.dinv ? cvk_mul(ch.v(4, t), y) : y;
        const int row = ch.r0 + t;
        pn[row] = xs(t);
        vn[row] = vi;
        acc_dot(acc[0], ch.v(3, t), vi);
    }, nullptr, [&](int t, const Chunk& ch) {
        if (!first)
            ch.set(0, t, cvk_add(cvk_mul(beta, cvk_add(ch.v(1, t), cvk_mul(nom, ch.v(2, t)))), ch.v(0, t)));
    });
    rank_total<1, kStreamThreads>(acc, a, &st->counter[1]);
}

__global__ void __launch_bounds__(kStreamThreads, 1) k_rb_b_s(RBArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_wait();
    PState* st = a.st;
    if (st->done) return;
    const int cur = st->cur;
    const double2 alpha = st->alpha, nal = cvk_neg(st->alpha);
    const double2* __restrict__ r = vec(a, VR);
    const double2* __restrict__ pn = vec(a, cur ? VP0 : VP1);
    const double2* __restrict__ vn = vec(a, cur ? VV0 : VV1);
    double2* __restrict__ s = vec(a, VS);
    double2* __restrict__ t_ = vec(a, VT);
    double2* __restrict__ x = vec(a, VX);
    const double2* vecs[5] = {r, vn, a.dinv, pn, x};
    StreamLayout L{a.capk, 5, a.nst[1]};
    L.ngather = 2;
    L.pf_rows = a.pf_rows;
    CAcc acc[3] = {};
    stream_rows(a.A, L, vecs, smem, [&](int t, const Chunk& ch) {
        auto xs = [&](int l) -> double2 {  // slot 0 of the chunk rows holds s (pre)
            return l < kStreamRows ? ch.v(0, l) : cvk_add(ch.v(0, l), cvk_mul(nal, ch.v(1, l)));
        };
        auto xg = [&](int c) -> double2 { return cvk_add(r[c], cvk_mul(nal, vn[c])); };
        const double2 y = chunk_row_sum<kRbBatch>(ch, t, xs, xg);
        const double2 ti = a.dinv ? cvk_mul(ch.v(2, t), y) : y;
        const double2 si = xs(t);
        const int row = ch.r0 + t;
        s[row] = si;
        t_[row] = ti;
        x[row] = cvk_add(ch.v(4, t), cvk_mul(alpha, ch.v(3, t)));
        acc_norm(acc[0], si);
        acc_dot(acc[1], ti, ti);
        acc_dot(acc[2], ti, si);
    }, nullptr, [&](int t, const Chunk& ch) {
        ch.set(0, t, cvk_add(ch.v(0, t), cvk_mul(nal, ch.v(1, t))));
    });
    rank_total<3, kStreamThreads>(acc, a, &st->counter[2]);
}

// x += omega s; r = s - omega t; ||r||, <shadow, r> -- small grid, 4 elements
// per thread per trip with all loads first (cvk_phased.cu k_bi_c)
__global__ void __launch_bounds__(kThreads) k_rb_c4(RBArgs a) {
    pdl_wait();
    PState* st = a.st;
    if (st->done) return;
    const int n = a.A.n;
    const double2 omega = st->omega, nom = cvk_neg(st->omega);
    const double2* __restrict__ s = vec(a, VS);
    const double2* __restrict__ t = vec(a, VT);
    const double2* __restrict__ sh = vec(a, VSH);
    double2* __restrict__ r = vec(a, VR);
    double2* __restrict__ x = vec(a, VX);
    CAcc acc[2] = {};
    constexpr int U = 4;
    const long long stride = (long long)gridDim.x * kThreads;
    for (long long base = (long long)blockIdx.x * kThreads + threadIdx.x; base < n; base += stride * U) {
        double2 vs[U], vt[U], vh[U], vx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = base + u * stride;
            if (i < n) { vs[u] = s[i]; vt[u] = t[i]; vh[u] = sh[i]; vx[u] = x[i]; }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = base + u * stride;
            if (i < n) {
                x[i] = cvk_add(vx[u], cvk_mul(omega, vs[u]));
                const double2 ri = cvk_add(vs[u], cvk_mul(nom, vt[u]));
                r[i] = ri;
                acc_norm(acc[0], ri);
                acc_dot(acc[1], vh[u], ri);
            }
        }
    }
    rank_total<2>(acc, a, &st->counter[0]);
}

// ||b||^2, ||b - A x||^2 over own rows (x halo from CVK_RB_X); krylov.cpp:17-23
__global__ void __launch_bounds__(kThreads) k_rb_t(RBArgs a) {
    pdl_wait();
    PState* st = a.st;
    const int n = a.A.n;
    const double2* __restrict__ x = vec(a, VX);
    auto xat = [&](int c) -> double2 { return x[c]; };
    CAcc acc[2] = {};
    if (!st->skip_true) {
        for_rows<1>(n, gridDim.x, blockIdx.x, [&](int row, int, bool valid) {
            const double2 y = row_sum<1, decltype(xat)&, kRbBatch>(a.A, row, 0, valid, xat);
            if (valid) {
                const double2 bi = __ldg(a.b + row);
                acc_norm(acc[0], bi);
                acc_norm(acc[1], cvk_sub(bi, y));
            }
        });
    }
    rank_total<2>(acc, a, &st->counter[3]);
}

// ------------------------------------------------------------- exchange --

// values of phase ph's halo vectors (nv_ph of them) for exchange position k
__device__ __forceinline__ int phase_vecs(int ph, int cur, int (&v)[2]) {
    switch (ph) {
        case CVK_RB_INIT: case CVK_RB_C: v[0] = VR; return 1;
        case CVK_RB_A: v[0] = cur ? VP0 : VP1; v[1] = cur ? VV0 : VV1; return 2;
        case CVK_RB_X: v[0] = VX; return 1;
        default: return 0;
    }
}

__global__ void __launch_bounds__(kThreads) k_rb_pack(RBArgs a, int ph) {
    pdl_wait();
    const PState* st = a.st;
    if (a.p2p) {
        // every phase: the header (this rank's totals) and the boundary values
        // go to all mailboxes; the done test is the same on every rank
        if (ph != CVK_RB_X && ph != CVK_RB_T && st->done) return;
        const unsigned long long seq0 = *(volatile unsigned long long*)mb_seq(a);
        const int parity = (int)((seq0 + 1) & 1);
        int vv[2];
        const int nvp = phase_vecs(ph, st->cur, vv);
        const long long items = kHdr / 2 + (long long)a.n_send * nvp;
        for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < items; i += (long long)gridDim.x * kThreads) {
            double2 v;
            if (i < kHdr / 2) {
                v = ((const double2*)a.send)[i];
            } else {
                const long long e = i - kHdr / 2;
                const int k = (int)(e / nvp), j = (int)(e - (long long)k * nvp);
                v = vec(a, vv[j])[__ldg(a.send_rows + k)];
            }
            for (int q = 0; q < a.nranks; ++q)
                ((double2*)(mb_data(a.peers[q], a, parity) + (size_t)a.rank * a.slot))[i] = v;
        }
        __shared__ int s_last;
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(a.pack_ctr, 1u) == gridDim.x - 1u;
        __syncthreads();
        if (!s_last || threadIdx.x != 0) return;
        *a.pack_ctr = 0u;
        __threadfence_system();
        const unsigned long long seq = seq0 + 1;
        *mb_seq(a) = seq;
        for (int q = 0; q < a.nranks; ++q) st_release_sys(mb_flags(a.peers[q]) + a.rank, seq);
        return;
    }
    if (ph != CVK_RB_X && st->done) return;
    int vv[2];
    const int nvp = phase_vecs(ph, st->cur, vv);
    double2* out = (double2*)(a.send + kHdr);
    const long long total = (long long)a.n_send * nvp;
    for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < total; i += (long long)gridDim.x * kThreads) {
        const int k = (int)(i / nvp), j = (int)(i - (long long)k * nvp);
        out[i] = vec(a, vv[j])[__ldg(a.send_rows + k)];
    }
}

// fold + scalar recurrence (CTA 0, thread 0) and halo unpack (all CTAs)
__global__ void __launch_bounds__(kThreads) k_rb_post(RBArgs a, int ph) {
    pdl_wait();
    PState* st = a.st;
    if (ph != CVK_RB_X && ph != CVK_RB_T && st->done) return;
    const double* recv = a.recv;
    if (a.p2p) {
        // wait until every rank has pushed this phase (its flag here reaches
        // our sequence number); 20 s without progress aborts the solve
        const unsigned long long seq = *(volatile unsigned long long*)mb_seq(a);
        __shared__ int s_ok;
        if (threadIdx.x == 0) {
            int ok = 1;
            const unsigned long long t0 = now_ns();
            for (int q = 0; q < a.nranks && ok; ++q)
                while (ld_acquire_sys(mb_flags(a.mbox) + q) < seq)
                    if (now_ns() - t0 > 20000000000ull) { ok = 0; break; }
            s_ok = ok;
        }
        __syncthreads();
        if (!s_ok) {
            if (blockIdx.x == 0 && threadIdx.x == 0) { a.rep->error = 1; st->done = 1; }
            return;
        }
        recv = mb_data(a.mbox, a, (int)(seq & 1));
    }
    int vv[2];
    const int nvp = phase_vecs(ph, st->cur, vv);
    const long long total = (long long)a.n_halo * nvp;
    for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < total; i += (long long)gridDim.x * kThreads) {
        const int h = (int)(i / nvp), j = (int)(i - (long long)h * nvp);
        const int src = __ldg(a.halo_src + h);
        const int q = src / a.max_send, k = src - q * a.max_send;
        const double2* in = (const double2*)(recv + (size_t)q * a.slot + kHdr);
        vec(a, vv[j])[a.A.n + h] = in[(size_t)k * nvp + j];
    }
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    switch (ph) {
        case CVK_RB_INIT: {  // krylov.cpp:62-79
            const double2 nr = fold_ranks(a, 0, recv), rr = fold_ranks(a, 1, recv);
            st->bnorm = sqrt(nr.x);
            if (st->bnorm == 0.0) {
                st->done = 1; st->conv = 1; st->iters = 0; st->skip_true = 1;
                return;
            }
            st->brk = 1e-30 * st->bnorm * st->bnorm;
            st->rho_new = rr;
            st->rho = st->alpha = st->omega = make_double2(1.0, 0.0);
            st->it = 1;
            st->first = 1;
            st->cur = 0;
            rb_top(st);
            return;
        }
        case CVK_RB_A: {  // krylov.cpp:97-103
            const double2 sv = fold_ranks(a, 0, recv);
            if (cvk_abs(sv) < st->brk) {
                st->done = 1; st->brk_code = 2; st->iters = st->it - 1;
                return;
            }
            st->alpha = cvk_cdiv(st->rho, sv);
            return;
        }
        case CVK_RB_B: {  // krylov.cpp:104-122
            const double2 ss = fold_ranks(a, 0, recv), tt = fold_ranks(a, 1, recv), ts = fold_ranks(a, 2, recv);
            const double relres = sqrt(ss.x) / st->bnorm;
            if (relres <= st->tol) {
                st->done = 1; st->conv = 1; st->iters = st->it; st->final_relres = relres;
                rb_hist(a, st, relres);
                return;
            }
            if (cvk_abs(tt) < st->brk) {
                st->done = 1; st->brk_code = 3; st->iters = st->it;
                return;
            }
            st->omega = cvk_cdiv(ts, tt);
            return;
        }
        case CVK_RB_C: {  // krylov.cpp:123-133
            const double2 rn = fold_ranks(a, 0, recv), shr = fold_ranks(a, 1, recv);
            const double relres = sqrt(rn.x) / st->bnorm;
            st->final_relres = relres;
            st->iters = st->it;
            rb_hist(a, st, relres);
            if (relres <= st->tol) { st->done = 1; st->conv = 1; return; }
            st->rho_new = shr;
            st->cur ^= 1;
            st->first = 0;
            st->it++;
            rb_top(st);
            return;
        }
        case CVK_RB_T: {  // krylov.cpp:17-23, 135
            double trr = 0.0;
            if (!st->skip_true) {
                const double bn = sqrt(fold_ranks(a, 0, recv).x), rn = sqrt(fold_ranks(a, 1, recv).x);
                trr = bn > 0 ? rn / bn : rn;
            }
            a.rep->converged = st->conv;
            a.rep->breakdown = st->brk_code;
            a.rep->iterations = st->iters;
            a.rep->final_relres = st->final_relres;
            a.rep->true_relres = trr;
            a.rep->history_len = st->hist_len;  // rep->error: zeroed at CVK_RB_INIT, set by an aborted wait
            return;
        }
        default: return;
    }
}

}  // namespace
}  // namespace cvk

// ---------------------------------------------------------------- host ---

using cvk::PState;

// NCCL resolved at run time from the process's libnccl.so.2 (the one
// torch.distributed already loaded, or the system's): the library has no
// link-time NCCL dependency and single-device users never load it.
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
};

static const NcclApi& nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
        a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(h, "ncclCommInitRank");
        a.all_gather = (decltype(a.all_gather))dlsym(h, "ncclAllGather");
        a.comm_destroy = (decltype(a.comm_destroy))dlsym(h, "ncclCommDestroy");
        a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
        a.ok = a.get_unique_id && a.comm_init_rank && a.all_gather && a.comm_destroy && a.error_string;
        return a;
    }();
    return api;
}

struct cvk_rowblock {
    cvk_ctx* ctx = nullptr;
    cudaStream_t s = nullptr;
    int nsm = 0;
    int64_t n_own = 0, n_halo = 0, nnz = 0, nv = 0;
    int G = 1, Gx = 1, Ge = 1;  // thread-per-row phases; pack/post; elementwise phase
    bool streamed = false;
    size_t smem_a = 0, smem_b = 0;
    std::vector<void*> bufs;
    double* send = nullptr;
    double* recv = nullptr;
    int64_t slot = 0;
    cvk::RBArgs args{};
    int64_t hist_cap = 0;
    long long launches = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    double t_wall0 = 0.0;
    int solver = CVK_BICGSTAB;
    long long max_iter = 0;
    ncclComm_t comm = nullptr;
    int rank = -1;
    PState st0{};  // initial solver state, restored by every CVK_RB_INIT (blocks are reusable)
    unsigned char* mbox = nullptr;  // p2p mailbox (cudaMalloc'd: IPC-exportable)
    size_t mbox_bytes = 0;
    std::vector<void*> ipc_open;    // peers' mailboxes opened through CUDA IPC
    unsigned char** d_peers = nullptr;
    ~cvk_rowblock() {
        if (comm) nccl_api().comm_destroy(comm);
        for (void* p : ipc_open) cudaIpcCloseMemHandle(p);
        for (void* p : bufs) cudaFree(p);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    }
    template <class T>
    cudaError_t alloc(T** p, size_t count) {
        void* q = nullptr;
        cudaError_t e = cudaMalloc(&q, std::max<size_t>(1, count) * sizeof(T));
        if (e == cudaSuccess) {
            bufs.push_back(q);
            *p = (T*)q;
        }
        return e;
    }
};

namespace {

int rbfail(int code, const std::string& m) { return cvk_fail(code, m); }
#define RK(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return rbfail(e_ == cudaErrorMemoryAllocation ? CVK_ENOMEM : CVK_ECUDA,               \
                          std::string(#call) + ": " + cudaGetErrorString(e_));                    \
    } while (0)

double wall_now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

cudaError_t rb_launch(const void* f, int grid, cudaStream_t s, void** args, int threads = cvk::kThreads,
                      size_t smem = 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, f, args);
}

}  // namespace

extern "C" int cvk_rowblock_create(cvk_ctx* ctx, const cvk_rowblock_desc* d, int solver, const cvk_opts* o,
                                   cvk_rowblock** out) {
    if (!ctx || !d || !o || !out) return rbfail(CVK_EINVAL, "cvk_rowblock_create: null argument");
    *out = nullptr;
    if (solver != CVK_BICGSTAB)
        return rbfail(CVK_ESOLVER, "cvk_rowblock_create: the row-block path runs bicgstab");
    if (o->mode == CVK_MODE_REF)
        return rbfail(CVK_EINVAL, "cvk_rowblock_create: REF mode is single-device (sequential sums)");
    if (d->n_own < 0 || d->n_halo < 0 || d->nnz < 0 || d->n_ranks < 1 || d->n_send < 0 || d->max_send < d->n_send)
        return rbfail(CVK_EINVAL, "cvk_rowblock_create: bad sizes");
    if (d->n_own + d->n_halo >= (1LL << 31) || d->nnz >= (1LL << 31) || d->n_ranks * std::max<int64_t>(1, d->max_send) >= (1LL << 31))
        return rbfail(CVK_EOVERFLOW, "cvk_rowblock_create: block does not fit int32 indices");
    const int64_t ncol = d->n_own + d->n_halo;
    if (d->n_own > 0 && (!d->row_offsets || !d->b)) return rbfail(CVK_EINVAL, "cvk_rowblock_create: null rows / rhs");
    if (d->n_own > 0 && (d->row_offsets[0] != 0 || d->row_offsets[d->n_own] != d->nnz))
        return rbfail(CVK_EINVAL, "cvk_rowblock_create: row_offsets must run 0 .. nnz");
    std::vector<int> rp((size_t)d->n_own + 1, 0), ci((size_t)d->nnz), sr((size_t)d->n_send), hs((size_t)d->n_halo);
    for (int64_t i = 0; i < d->n_own; ++i) {
        if (d->row_offsets[i + 1] < d->row_offsets[i]) return rbfail(CVK_EINVAL, "cvk_rowblock_create: row_offsets decrease");
        rp[(size_t)i + 1] = (int)d->row_offsets[i + 1];
    }
    for (int64_t k = 0; k < d->nnz; ++k) {
        if (d->col_local[k] < 0 || d->col_local[k] >= ncol)
            return rbfail(CVK_EINVAL, "cvk_rowblock_create: column " + std::to_string(d->col_local[k]) + " outside the block");
        ci[(size_t)k] = (int)d->col_local[k];
    }
    for (int64_t k = 0; k < d->n_send; ++k) {
        if (d->send_rows[k] < 0 || d->send_rows[k] >= d->n_own) return rbfail(CVK_EINVAL, "cvk_rowblock_create: send row outside the block");
        sr[(size_t)k] = (int)d->send_rows[k];
    }
    for (int64_t h = 0; h < d->n_halo; ++h) {
        if (d->halo_src[h] < 0 || d->halo_src[h] >= d->n_ranks * d->max_send)
            return rbfail(CVK_EINVAL, "cvk_rowblock_create: halo source outside the exchange");
        hs[(size_t)h] = (int)d->halo_src[h];
    }

    cvk_rowblock* R = new cvk_rowblock();
    auto bail = [&](int e) { delete R; return e; };
    R->ctx = ctx;
    R->s = (cudaStream_t)cvk_ctx_stream(ctx);
    R->solver = solver;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&R->nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return bail(rbfail(CVK_ECUDA, "cvk_rowblock_create: no device"));
    R->n_own = d->n_own;
    R->n_halo = d->n_halo;
    R->nnz = d->nnz;
    R->nv = (ncol + 31) / 32 * 32;
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)cvk::k_rb_b, cvk::kThreads, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    const long long chunks = std::max<long long>(1, (d->n_own + cvk::kThreads - 1) / cvk::kThreads);
    R->G = (int)std::min<long long>(chunks, 32LL * per_sm * R->nsm);
    const long long xchunks = std::max<long long>(1, (std::max(d->n_send, d->n_halo) * 2 + cvk::kThreads - 1) / cvk::kThreads);
    R->Gx = (int)std::min<long long>(xchunks, R->nsm);
    R->slot = cvk::kHdr + 4 * std::max<int64_t>(1, d->max_send);
    R->Ge = (int)std::min<long long>(2LL * R->nsm, std::max<long long>(1, (d->n_own + 4LL * cvk::kThreads - 1) / (4LL * cvk::kThreads)));
    // streamed SpMV phases (TMA ring, cvk_stream.cuh) as in the single-device
    // phase kernels: chunk capacity, each chunk's largest own column (L2
    // prefetch of the forward band), ring depth from the shared-memory budget
    const int64_t nch = (d->n_own + cvk::kStreamRows - 1) / cvk::kStreamRows;
    long long mk = 0;
    std::vector<int> cm((size_t)std::max<int64_t>(1, nch), -1);
    for (int64_t q = 0; q < nch; ++q) {
        const int64_t a0 = q * cvk::kStreamRows, a1 = std::min<int64_t>(a0 + cvk::kStreamRows, d->n_own);
        mk = std::max<long long>(mk, (long long)(rp[(size_t)a1] - rp[(size_t)a0]));
        for (int k = rp[(size_t)a0]; k < rp[(size_t)a1]; ++k)
            if (ci[(size_t)k] < d->n_own) cm[(size_t)q] = std::max(cm[(size_t)q], ci[(size_t)k]);
    }
    const int capk = (int)((mk + 3) & ~3LL);
    int optin = 0, nst[2] = {0, 0};
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const int kv[2] = {5, 5}, kg[2] = {3, 2};
    for (int k = 0; k < 2; ++k) {
        cvk::StreamLayout L1{capk, kv[k], 1};
        L1.ngather = kg[k];
        const long long avail = (long long)optin - 8192 - 2 * cvk::kStreamMaxStages * 8 - cvk::kStreamMaxStages * 32;
        nst[k] = (int)std::min<long long>(4, std::max<long long>(0, avail / (long long)L1.stage_bytes()));
    }
    const long long smin = cvk_ctx_knob(ctx, CVK_OPT_RB_STREAM_MIN);
    // the tested ring depth (4; cvk_api.cu kStreamMinStages)
    R->streamed = d->nnz > 0 && d->n_own >= smin && std::min(nst[0], nst[1]) >= 4 && cvk_ctx_knob(ctx, CVK_OPT_STREAM);
    if (R->streamed) {
        for (int k = 0; k < 2; ++k) {
            cvk::StreamLayout L{capk, kv[k], nst[k]};
            L.ngather = kg[k];
            (k ? R->smem_b : R->smem_a) = L.smem_bytes();
        }
        if (cudaFuncSetAttribute((const void*)cvk::k_rb_a_s, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 8192) != cudaSuccess ||
            cudaFuncSetAttribute((const void*)cvk::k_rb_b_s, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 8192) != cudaSuccess)
            return bail(rbfail(CVK_ECUDA, "cvk_rowblock_create: shared-memory opt-in failed"));
    }
    const int Gpart = std::max(std::max(R->G, R->Ge), R->nsm);
    R->hist_cap = o->record_history ? std::max<int64_t>(d->history_cap, 0) : 0;
    R->max_iter = std::max<long long>(0, o->max_iter);

    int *d_rp, *d_ci, *d_sr, *d_hs, *d_cmax;
    double2 *d_av, *d_dinv = nullptr, *d_b, *d_work, *d_part;
    PState* d_st;
    double* d_hist;
    cvk::DevReport* d_rep;
    cudaError_t e = cudaSuccess;
    if ((e = R->alloc(&d_rp, rp.size() + 4)) != cudaSuccess || (e = R->alloc(&d_ci, ci.size() + 8)) != cudaSuccess ||
        (e = R->alloc(&d_cmax, cm.size())) != cudaSuccess ||
        (e = R->alloc(&d_sr, sr.size())) != cudaSuccess || (e = R->alloc(&d_hs, hs.size())) != cudaSuccess ||
        (e = R->alloc(&d_av, (size_t)d->nnz)) != cudaSuccess || (e = R->alloc(&d_b, (size_t)d->n_own)) != cudaSuccess ||
        (e = R->alloc(&d_work, (size_t)cvk::kRbVecs * R->nv)) != cudaSuccess ||
        (e = R->alloc(&d_part, (size_t)6 * Gpart)) != cudaSuccess || (e = R->alloc(&d_st, 1)) != cudaSuccess ||
        (e = R->alloc(&d_hist, (size_t)std::max<int64_t>(1, R->hist_cap))) != cudaSuccess ||
        (e = R->alloc(&d_rep, 1)) != cudaSuccess || (e = R->alloc(&R->send, (size_t)R->slot)) != cudaSuccess ||
        (e = R->alloc(&R->recv, (size_t)R->slot * d->n_ranks)) != cudaSuccess ||
        (d->inv_diag && (e = R->alloc(&d_dinv, (size_t)d->n_own)) != cudaSuccess))
        return bail(rbfail(e == cudaErrorMemoryAllocation ? CVK_ENOMEM : CVK_ECUDA,
                           std::string("cvk_rowblock_create: ") + cudaGetErrorString(e)));
    // p2p mailbox: [flags: nranks u64, 256-B padded | seq u64 | 2 x nranks slots]
    const int flag_bytes = (int)(((d->n_ranks * 8 + 255) / 256) * 256);
    R->mbox_bytes = (size_t)flag_bytes + 256 + sizeof(double) * 2 * (size_t)R->slot * d->n_ranks;
    unsigned* d_pack_ctr = nullptr;
    if ((e = R->alloc(&R->mbox, R->mbox_bytes)) != cudaSuccess || (e = R->alloc(&d_pack_ctr, 1)) != cudaSuccess ||
        (e = R->alloc(&R->d_peers, (size_t)d->n_ranks)) != cudaSuccess ||
        (e = cudaMemsetAsync(R->mbox, 0, R->mbox_bytes, R->s)) != cudaSuccess ||
        (e = cudaMemsetAsync(d_pack_ctr, 0, sizeof(unsigned), R->s)) != cudaSuccess)
        return bail(rbfail(CVK_ECUDA, std::string("cvk_rowblock_create: mailbox: ") + cudaGetErrorString(e)));
    auto h2d = [&](void* dst, const void* src, size_t bytes) {
        return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, R->s) : cudaSuccess;
    };
    if ((e = h2d(d_rp, rp.data(), rp.size() * 4)) != cudaSuccess || (e = h2d(d_ci, ci.data(), ci.size() * 4)) != cudaSuccess ||
        (e = h2d(d_sr, sr.data(), sr.size() * 4)) != cudaSuccess || (e = h2d(d_cmax, cm.data(), cm.size() * 4)) != cudaSuccess || (e = h2d(d_hs, hs.data(), hs.size() * 4)) != cudaSuccess ||
        (e = h2d(d_av, d->values, (size_t)d->nnz * 16)) != cudaSuccess ||
        (e = h2d(d_b, d->b, (size_t)d->n_own * 16)) != cudaSuccess ||
        (d_dinv && (e = h2d(d_dinv, d->inv_diag, (size_t)d->n_own * 16)) != cudaSuccess) ||
        (e = cudaMemsetAsync(d_work, 0, sizeof(double2) * cvk::kRbVecs * R->nv, R->s)) != cudaSuccess ||
        (e = cudaMemsetAsync(R->send, 0, sizeof(double) * R->slot, R->s)) != cudaSuccess ||
        (e = cudaMemsetAsync(R->recv, 0, sizeof(double) * R->slot * d->n_ranks, R->s)) != cudaSuccess)
        return bail(rbfail(CVK_ECUDA, std::string("cvk_rowblock_create: upload: ") + cudaGetErrorString(e)));
    PState hs0;
    std::memset(&hs0, 0, sizeof(hs0));
    hs0.tol = o->tol;
    hs0.max_iter = o->max_iter < 1 ? 0 : o->max_iter;
    hs0.record = R->hist_cap > 0 ? 1 : 0;
    hs0.hist_cap = R->hist_cap;
    R->st0 = hs0;
    if ((e = cudaMemcpyAsync(d_st, &hs0, sizeof(hs0), cudaMemcpyHostToDevice, R->s)) != cudaSuccess ||
        (e = cudaStreamSynchronize(R->s)) != cudaSuccess || (e = cudaEventCreate(&R->e0)) != cudaSuccess ||
        (e = cudaEventCreate(&R->e1)) != cudaSuccess)
        return bail(rbfail(CVK_ECUDA, std::string("cvk_rowblock_create: ") + cudaGetErrorString(e)));

    cvk::RBArgs& a = R->args;
    a.A.n = (int)d->n_own;
    a.A.rp = d_rp;
    a.A.ci = d_ci;
    a.A.av = d_av;
    a.A.cmax = d_cmax;
    a.capk = capk;
    a.nst[0] = nst[0];
    a.nst[1] = nst[1];
    a.pf_rows = 2 * cvk::kStreamRows;
    a.nv = R->nv;
    a.dinv = d_dinv;
    a.b = d_b;
    a.work = d_work;
    a.part = d_part;
    a.st = d_st;
    a.hist = d_hist;
    a.rep = d_rep;
    a.send = R->send;
    a.recv = R->recv;
    a.nranks = (int)d->n_ranks;
    a.slot = (int)R->slot;
    a.send_rows = d_sr;
    a.n_send = (int)d->n_send;
    a.max_send = (int)std::max<int64_t>(1, d->max_send);
    a.halo_src = d_hs;
    a.n_halo = (int)d->n_halo;
    a.p2p = 0;
    a.rank = 0;
    a.flag_bytes = flag_bytes;
    a.peers = R->d_peers;
    a.mbox = R->mbox;
    a.pack_ctr = d_pack_ctr;
    *out = R;
    return CVK_OK;
}

extern "C" int cvk_rowblock_exchange(cvk_rowblock* R, double** send, double** recv, int64_t* slot) {
    if (!R) return rbfail(CVK_EINVAL, "cvk_rowblock_exchange: null block");
    if (send) *send = R->send;
    if (recv) *recv = R->recv;
    if (slot) *slot = R->slot;
    return CVK_OK;
}

extern "C" int cvk_rowblock_local(cvk_rowblock* R, int ph) {
    if (!R) return rbfail(CVK_EINVAL, "cvk_rowblock_local: null block");
    void* args[2] = {&R->args, &ph};
    const void* f = nullptr;
    switch (ph) {
        case CVK_RB_INIT:
            R->t_wall0 = wall_now();
            R->launches = 0;
            RK(cudaMemcpyAsync(R->args.st, &R->st0, sizeof(PState), cudaMemcpyHostToDevice, R->s));
            RK(cudaMemsetAsync(R->args.rep, 0, sizeof(cvk::DevReport), R->s));
            RK(cudaEventRecord(R->e0, R->s));
            f = (const void*)cvk::k_rb_init;
            break;
        case CVK_RB_A:
        case CVK_RB_B:
            if (R->streamed) {
                RK(rb_launch(ph == CVK_RB_A ? (const void*)cvk::k_rb_a_s : (const void*)cvk::k_rb_b_s, R->nsm, R->s,
                             args, cvk::kStreamThreads, ph == CVK_RB_A ? R->smem_a : R->smem_b));
                R->launches++;
            } else {
                f = ph == CVK_RB_A ? (const void*)cvk::k_rb_a : (const void*)cvk::k_rb_b;
            }
            break;
        case CVK_RB_C:
            RK(rb_launch((const void*)cvk::k_rb_c4, R->Ge, R->s, args));
            R->launches++;
            break;
        case CVK_RB_X: break;
        case CVK_RB_T: f = (const void*)cvk::k_rb_t; break;
        default: return rbfail(CVK_EINVAL, "cvk_rowblock_local: unknown phase " + std::to_string(ph));
    }
    if (f) {
        RK(rb_launch(f, R->G, R->s, args));
        R->launches++;
    }
    if (R->args.p2p) {
        RK(rb_launch((const void*)cvk::k_rb_pack, R->Gx, R->s, args));
        R->launches++;
    } else if (ph == CVK_RB_INIT || ph == CVK_RB_A || ph == CVK_RB_C || ph == CVK_RB_X) {
        if (R->args.n_send > 0) {
            RK(rb_launch((const void*)cvk::k_rb_pack, R->Gx, R->s, args));
            R->launches++;
        }
    }
    return CVK_OK;
}

extern "C" int cvk_rowblock_post(cvk_rowblock* R, int ph) {
    if (!R) return rbfail(CVK_EINVAL, "cvk_rowblock_post: null block");
    if (ph < CVK_RB_INIT || ph > CVK_RB_T) return rbfail(CVK_EINVAL, "cvk_rowblock_post: unknown phase " + std::to_string(ph));
    void* args[2] = {&R->args, &ph};
    RK(rb_launch((const void*)cvk::k_rb_post, R->Gx, R->s, args));
    R->launches++;
    if (ph == CVK_RB_T) RK(cudaEventRecord(R->e1, R->s));
    return CVK_OK;
}

extern "C" int cvk_rowblock_exchange_local(cvk_rowblock* const* rbs, int n) {
    if (!rbs || n < 1) return rbfail(CVK_EINVAL, "cvk_rowblock_exchange_local: no blocks");
    for (int q = 0; q < n; ++q)
        if (!rbs[q] || rbs[q]->args.nranks != n || rbs[q]->slot != rbs[0]->slot || rbs[q]->s != rbs[0]->s)
            return rbfail(CVK_EINVAL, "cvk_rowblock_exchange_local: blocks disagree on ranks / slot / stream");
    const size_t bytes = sizeof(double) * rbs[0]->slot;
    for (int dst = 0; dst < n; ++dst)
        for (int q = 0; q < n; ++q)
            RK(cudaMemcpyAsync(rbs[dst]->recv + (size_t)q * rbs[0]->slot, rbs[q]->send, bytes, cudaMemcpyDeviceToDevice,
                               rbs[0]->s));
    return CVK_OK;
}

extern "C" int cvk_rowblock_done(cvk_rowblock* R, int* done) {
    if (!R || !done) return rbfail(CVK_EINVAL, "cvk_rowblock_done: null argument");
    int v = 0;
    RK(cudaMemcpyAsync(&v, &R->args.st->done, sizeof(int), cudaMemcpyDeviceToHost, R->s));
    RK(cudaStreamSynchronize(R->s));
    *done = v;
    return CVK_OK;
}

namespace {
// The solve's phase loop for blocks on one stream: INIT, then kIters
// iterations (A, B, C per block, xchg between local and post) captured once
// and replayed with the stop flag read back lazily (one graph in flight
// behind the poll, as the single-device phase kernels do), then X and T.
template <class Xchg>
int run_phases(cvk_rowblock* const* rbs, int n, Xchg&& xchg) {
    auto phase = [&](int ph) -> int {
        int e;
        for (int q = 0; q < n; ++q)
            if ((e = cvk_rowblock_local(rbs[q], ph)) != CVK_OK) return e;
        if ((e = xchg()) != CVK_OK) return e;
        for (int q = 0; q < n; ++q)
            if ((e = cvk_rowblock_post(rbs[q], ph)) != CVK_OK) return e;
        return CVK_OK;
    };
    int e;
    if ((e = phase(CVK_RB_INIT)) != CVK_OK) return e;
    constexpr int kIters = 8;
    cudaStream_t s = rbs[0]->s;
    std::vector<long long> before(n);
    for (int q = 0; q < n; ++q) before[q] = rbs[q]->launches;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gx = nullptr;
    RK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < kIters && e == CVK_OK; ++k)
        for (int ph : {CVK_RB_A, CVK_RB_B, CVK_RB_C})
            if (e == CVK_OK) e = phase(ph);
    const cudaError_t ce = cudaStreamEndCapture(s, &graph);
    if (e != CVK_OK) {
        if (graph) cudaGraphDestroy(graph);
        return e;
    }
    RK(ce);
    const cudaError_t ie = cudaGraphInstantiate(&gx, graph, 0);
    cudaGraphDestroy(graph);
    RK(ie);
    std::vector<long long> per_graph(n);
    for (int q = 0; q < n; ++q) per_graph[q] = rbs[q]->launches - before[q], rbs[q]->launches = before[q];
    int* h_done = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    auto cleanup = [&]() {
        if (gx) cudaGraphExecDestroy(gx);
        if (h_done) cudaFreeHost(h_done);
        for (cudaEvent_t x : ev)
            if (x) cudaEventDestroy(x);
    };
    if (cudaMallocHost(&h_done, 2 * sizeof(int)) != cudaSuccess || cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming) != cudaSuccess) {
        cleanup();
        return rbfail(CVK_ECUDA, "rowblock solve: host flag / events");
    }
    const long long max_graphs = rbs[0]->max_iter / kIters + 3;
    long long graphs = 0;
    cudaError_t le = cudaSuccess;
    while (graphs < max_graphs && le == cudaSuccess) {
        const int sl = (int)(graphs & 1);
        if ((le = cudaGraphLaunch(gx, s)) != cudaSuccess) break;
        if ((le = cudaMemcpyAsync(&h_done[sl], &rbs[0]->args.st->done, sizeof(int), cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
        if ((le = cudaEventRecord(ev[sl], s)) != cudaSuccess) break;
        ++graphs;
        for (int q = 0; q < n; ++q) rbs[q]->launches += per_graph[q];
        if (graphs >= 2) {
            const int old = (int)((graphs - 2) & 1);
            if ((le = cudaEventSynchronize(ev[old])) != cudaSuccess) break;
            if (h_done[old]) break;
        }
    }
    cleanup();
    RK(le);
    if ((e = phase(CVK_RB_X)) != CVK_OK) return e;
    return phase(CVK_RB_T);
}

}  // namespace

extern "C" int cvk_rowblock_solve_local(cvk_rowblock* const* rbs, int n) {
    if (!rbs || n < 1) return rbfail(CVK_EINVAL, "cvk_rowblock_solve_local: no blocks");
    for (int q = 0; q < n; ++q)
        if (!rbs[q] || rbs[q]->args.nranks != n || rbs[q]->slot != rbs[0]->slot || rbs[q]->s != rbs[0]->s)
            return rbfail(CVK_EINVAL, "cvk_rowblock_solve_local: blocks disagree on ranks / slot / stream");
    // the blocks share one stream, so they can share one gathered buffer:
    // block q writes its slot q in place and every block reads them all --
    // the all-gather costs nothing
    double* shared = nullptr;
    RK(cudaMalloc(&shared, sizeof(double) * rbs[0]->slot * n));
    for (int q = 0; q < n; ++q) {
        rbs[q]->args.send = shared + (size_t)q * rbs[0]->slot;
        rbs[q]->args.recv = shared;
    }
    struct Restore {
        cvk_rowblock* const* rbs;
        int n;
        double* shared;
        ~Restore() {
            cudaStreamSynchronize(rbs[0]->s);
            for (int q = 0; q < n; ++q) {
                rbs[q]->args.send = rbs[q]->send;
                rbs[q]->args.recv = rbs[q]->recv;
            }
            cudaFree(shared);
        }
    } restore{rbs, n, shared};
    return run_phases(rbs, n, [] { return CVK_OK; });
}

extern "C" int cvk_nccl_unique_id(char* id) {
    if (!id) return rbfail(CVK_EINVAL, "cvk_nccl_unique_id: null id");
    const NcclApi& api = nccl_api();
    if (!api.ok) return rbfail(CVK_ECUDA, "cvk_nccl_unique_id: libnccl.so.2 not loadable");
    ncclUniqueId u;
    const ncclResult_t r = api.get_unique_id(&u);
    if (r != ncclSuccess) return rbfail(CVK_ECUDA, std::string("ncclGetUniqueId: ") + api.error_string(r));
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    return CVK_OK;
}

extern "C" int cvk_rowblock_attach_nccl(cvk_rowblock* R, const char* id, int rank) {
    if (!R || !id) return rbfail(CVK_EINVAL, "cvk_rowblock_attach_nccl: null argument");
    if (rank < 0 || rank >= R->args.nranks) return rbfail(CVK_EINVAL, "cvk_rowblock_attach_nccl: rank outside the plan");
    const NcclApi& api = nccl_api();
    if (!api.ok) return rbfail(CVK_ECUDA, "cvk_rowblock_attach_nccl: libnccl.so.2 not loadable");
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    if (R->comm) {
        api.comm_destroy(R->comm);
        R->comm = nullptr;
    }
    const ncclResult_t r = api.comm_init_rank(&R->comm, R->args.nranks, u, rank);
    if (r != ncclSuccess) {
        R->comm = nullptr;
        return rbfail(CVK_ECUDA, std::string("ncclCommInitRank: ") + api.error_string(r));
    }
    R->rank = rank;
    return CVK_OK;
}

extern "C" int cvk_rowblock_solve_nccl(cvk_rowblock* R) {
    if (!R || !R->comm) return rbfail(CVK_EINVAL, "cvk_rowblock_solve_nccl: no NCCL communicator attached");
    const NcclApi& api = nccl_api();
    cvk_rowblock* rbs[1] = {R};
    return run_phases(rbs, 1, [&]() -> int {
        const ncclResult_t r = api.all_gather(R->send, R->recv, (size_t)R->slot, ncclDouble, R->comm, R->s);
        if (r != ncclSuccess) return rbfail(CVK_ECUDA, std::string("ncclAllGather: ") + api.error_string(r));
        return CVK_OK;
    });
}

extern "C" int cvk_rowblock_p2p_handle(cvk_rowblock* R, void* handle) {
    if (!R || !handle) return rbfail(CVK_EINVAL, "cvk_rowblock_p2p_handle: null argument");
    cudaIpcMemHandle_t h;
    RK(cudaIpcGetMemHandle(&h, R->mbox));
    std::memcpy(handle, &h, sizeof(h));
    return CVK_OK;
}

namespace {
int p2p_set(cvk_rowblock* R, const std::vector<unsigned char*>& bases, int rank) {
    RK(cudaMemcpyAsync(R->d_peers, bases.data(), sizeof(unsigned char*) * bases.size(), cudaMemcpyHostToDevice, R->s));
    RK(cudaStreamSynchronize(R->s));
    R->args.p2p = 1;
    R->args.rank = rank;
    return CVK_OK;
}
}  // namespace

extern "C" int cvk_rowblock_p2p_attach(cvk_rowblock* R, const void* handles, int rank) {
    if (!R || !handles) return rbfail(CVK_EINVAL, "cvk_rowblock_p2p_attach: null argument");
    const int n = R->args.nranks;
    if (rank < 0 || rank >= n) return rbfail(CVK_EINVAL, "cvk_rowblock_p2p_attach: rank outside the plan");
    std::vector<unsigned char*> bases((size_t)n, nullptr);
    for (int q = 0; q < n; ++q) {
        if (q == rank) { bases[q] = R->mbox; continue; }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, (const unsigned char*)handles + (size_t)q * sizeof(h), sizeof(h));
        void* p = nullptr;
        RK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        R->ipc_open.push_back(p);
        bases[q] = (unsigned char*)p;
    }
    return p2p_set(R, bases, rank);
}

extern "C" int cvk_rowblock_p2p_attach_local(cvk_rowblock* const* rbs, int n) {
    if (!rbs || n < 1) return rbfail(CVK_EINVAL, "cvk_rowblock_p2p_attach_local: no blocks");
    std::vector<unsigned char*> bases((size_t)n);
    for (int q = 0; q < n; ++q) {
        if (!rbs[q] || rbs[q]->args.nranks != n) return rbfail(CVK_EINVAL, "cvk_rowblock_p2p_attach_local: plan mismatch");
        bases[q] = rbs[q]->mbox;
    }
    for (int q = 0; q < n; ++q) {
        const int e = p2p_set(rbs[q], bases, q);
        if (e != CVK_OK) return e;
    }
    return CVK_OK;
}

extern "C" int cvk_rowblock_solve_p2p(cvk_rowblock* const* rbs, int n) {
    if (!rbs || n < 1) return rbfail(CVK_EINVAL, "cvk_rowblock_solve_p2p: no blocks");
    for (int q = 0; q < n; ++q)
        if (!rbs[q] || !rbs[q]->args.p2p || rbs[q]->s != rbs[0]->s)
            return rbfail(CVK_EINVAL, "cvk_rowblock_solve_p2p: blocks must be p2p-attached and share a stream");
    return run_phases(rbs, n, [] { return CVK_OK; });
}

extern "C" int cvk_rowblock_result(cvk_rowblock* R, double* x_own, cvk_report* rep) {
    if (!R) return rbfail(CVK_EINVAL, "cvk_rowblock_result: null block");
    cvk::DevReport dr;
    RK(cudaMemcpyAsync(&dr, R->args.rep, sizeof(dr), cudaMemcpyDeviceToHost, R->s));
    if (x_own && R->n_own > 0)
        RK(cudaMemcpyAsync(x_own, R->args.work, sizeof(double2) * R->n_own, cudaMemcpyDeviceToHost, R->s));
    RK(cudaStreamSynchronize(R->s));
    if (dr.error) return rbfail(CVK_ETIMEOUT, "row-block solve: a peer stopped answering (p2p exchange wait aborted)");
    if (rep) {
        rep->converged = dr.converged;
        rep->breakdown = dr.breakdown;
        rep->iterations = dr.iterations;
        rep->final_relres = dr.final_relres;
        rep->true_relres = dr.true_relres;
        rep->history_len = dr.history_len;
        if (rep->history && rep->history_cap > 0 && R->hist_cap > 0) {
            const int64_t k = std::min<int64_t>(std::min<int64_t>(rep->history_cap, dr.history_len), R->hist_cap);
            if (k > 0) RK(cudaMemcpy(rep->history, R->args.hist, sizeof(double) * k, cudaMemcpyDeviceToHost));
        }
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, R->e0, R->e1) == cudaSuccess) rep->device_time_s = ms * 1e-3;
        else cudaGetLastError();
        rep->wall_time_s = wall_now() - R->t_wall0;
        rep->kernel_launches = R->launches;
    }
    return CVK_OK;
}

extern "C" int cvk_rowblock_destroy(cvk_rowblock* R) {
    if (R) {
        cudaStreamSynchronize(R->s);
        delete R;
    }
    return CVK_OK;
}
