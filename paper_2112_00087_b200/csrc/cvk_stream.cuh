// cvk_stream.cuh -- TMA-fed row streaming for the phase kernels.
//
// A phase kernel that contains an SpMV walks the matrix in chunks of R
// consecutive rows.  One producer warp streams, per chunk, the row offsets,
// the column/value slab and the chunk's row-local vectors into a ring of
// shared-memory stages with 1-D bulk copies (cp.async.bulk, completion on an
// mbarrier with an expected byte count); NCG consumer groups of R threads
// (thread per row) compute from shared memory and release the stage on a
// second mbarrier.  Bytes in flight per SM are (stages - 1) x stage size,
// independent of registers and occupancy -- the r01 thread-per-row kernels
// were latency-bound at 36-47% warp occupancy (profiles/r02_phase_kernels.txt),
// and tools/bicg_lab.cu measured this shape at 4.2 vs 3.0 TB/s (1M DOF) and
// 5.9 vs 3.7 TB/s (4M DOF) for the BiCGSTAB p-update + SpMV phase.
//
// Gathers x[col]: columns inside the chunk read the staged vectors from
// shared memory; the rest (the +-nx band neighbours of the cavity grid) go to
// global memory through L1/L2.  Accumulation order per row is left to right,
// as in row_sum (cvk_engine.cuh).
//
// Grid: one CTA per SM, chunks assigned grid-stride (chunk = cta + i*G).  The
// producer prefetches the k-ranges of its next 32 chunks with one load per
// lane, so the pointer chase rp -> (ci, av) never stalls the ring.
//
// Alignment: bulk copies need 16-byte aligned addresses and sizes.  Vectors
// are double2 (16 B); row offsets are copied from the chunk start (R is a
// multiple of 4) rounded up to 4 entries, so the row-offset array carries 16
// bytes of padding; columns are copied from floor4(k0) to ceil4(k1), so the
// column array is followed by >= 16 bytes of allocated memory (cvk_api.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "cvk_engine.cuh"

namespace cvk {

// R = 224 rows per chunk: 2 x 7 consumer warps + 1 producer warp = 15 warps
// (allocated as 16), so the register file allows 128 registers per thread;
// 256-row groups (17 warps, allocated as 20) cap the kernels at 96 registers
// with spills, and 240-row groups split a warp between the two groups (that
// warp then serves both rings: 168 vs 114 us per BiCGSTAB iteration, 1M DOF).
// R must be a multiple of 4 (16-byte aligned row-offset copies) and of 32.
#ifndef CVK_STREAM_ROWS
#define CVK_STREAM_ROWS 224
#endif
#ifndef CVK_STREAM_GROUPS
#define CVK_STREAM_GROUPS 2
#endif
constexpr int kStreamRows = CVK_STREAM_ROWS;      // R: rows per chunk = threads per consumer group
constexpr int kStreamGroups = CVK_STREAM_GROUPS;  // NCG consumer groups
constexpr int kStreamThreads = kStreamRows * kStreamGroups + 32;
constexpr int kStreamMaxStages = 8;
constexpr int kStreamMaxVecs = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P1;\n"
        "WAIT%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @P1 bra.uni DONE%=;\n"
        " bra.uni WAIT%=;\n"
        "DONE%=:\n}" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Shared-memory layout of one stage (host and device agree on it).
struct StreamLayout {
    int capk;    // nnz capacity of a chunk (multiple of 4)
    int nvec;    // staged row-local vectors
    int stages;  // ring depth
    int ngather = 0;  // vecs[0..ngather) are also gathered at neighbour columns
    int pf_rows = 0;  // L2-prefetch window (rows) below the chunk's largest column, 0 = off
    __host__ __device__ size_t rp_bytes() const { return (size_t)(kStreamRows + 4) * 4; }
    __host__ __device__ size_t ci_bytes() const { return (size_t)(capk + 8) * 4; }
    __host__ __device__ size_t av_bytes() const { return (size_t)capk * 16; }
    __host__ __device__ size_t vec_bytes() const { return (size_t)kStreamRows * 16; }
    __host__ __device__ size_t stage_bytes() const { return rp_bytes() + ci_bytes() + av_bytes() + (size_t)nvec * vec_bytes(); }
    // stages, then full / empty barriers, then the per-stage header (8 ints)
    __host__ __device__ size_t smem_bytes() const {
        return (size_t)stages * stage_bytes() + 2 * kStreamMaxStages * 8 + kStreamMaxStages * 32;
    }
};

// What a consumer thread sees of its chunk.
struct Chunk {
    const int* rp;      // global row offsets of rows r0 .. r0+rows
    const int* ci;      // columns, index k - k0 + cio
    const double2* av;  // values, index k - k0
    const double2* vec; // staged vectors, R rows each
    int k0, cio, r0, rows;
    int uni;            // uniform off-diagonal: av holds the rows' diagonal, coff the rest
    double2 coff;
    __device__ __forceinline__ double2 v(int j, int l) const { return vec[j * kStreamRows + l]; }
    __device__ __forceinline__ void set(int j, int l, double2 x) const { const_cast<double2*>(vec)[j * kStreamRows + l] = x; }
    // slot of column c in the chunk's staged rows, or -1 (global gather)
    __device__ __forceinline__ int stage_index(int c) const {
        const int l = c - r0;
        return (unsigned)l < (unsigned)rows ? l : -1;
    }
};

// Row sum for row t of the chunk: y = sum_k A[k] * x(col_k), left to right,
// with x read through xs(l) for columns staged in shared memory (the chunk's
// own rows; l = Chunk::stage_index) and xg(c) otherwise.  The (value, column)
// pairs of a batch come from shared memory; the global gathers of a batch are
// all issued before the first product.
template <int BATCH, bool UNI, class XS, class XG>
__device__ __forceinline__ double2 chunk_row_sum_t(const Chunk& ch, int t, XS&& xs, XG&& xg) {
    const int b = ch.rp[t] - ch.k0, e = ch.rp[t + 1] - ch.k0;
    double2 acc = make_double2(0.0, 0.0);
    for (int k = b; k < e; k += BATCH) {
        double2 a[BATCH], xv[BATCH];
        int c[BATCH];
#pragma unroll
        for (int u = 0; u < BATCH; ++u)
            if (k + u < e) {
                c[u] = ch.ci[k + u + ch.cio];
                if (!UNI) a[u] = ch.av[k + u];
            }
        if (UNI) {
#pragma unroll
            for (int u = 0; u < BATCH; ++u)
                if (k + u < e) a[u] = c[u] == ch.r0 + t ? ch.av[t] : ch.coff;
        }
#pragma unroll
        for (int u = 0; u < BATCH; ++u)
            if (k + u < e) {
                const int l = ch.stage_index(c[u]);
                xv[u] = l >= 0 ? xs(l) : xg(c[u]);
            }
#pragma unroll
        for (int u = 0; u < BATCH; ++u)
            if (k + u < e) acc = cvk_add(acc, cvk_mul(a[u], xv[u]));
    }
    return acc;
}

// uniform off-diagonal chunks (Chunk::uni) take their own loop: the general
// one keeps its (value, column) loads independent
template <int BATCH, class XS, class XG>
__device__ __forceinline__ double2 chunk_row_sum(const Chunk& ch, int t, XS&& xs, XG&& xg) {
#ifdef CVK_UNIFORM_OFFDIAG
    if (ch.uni) return chunk_row_sum_t<BATCH, true>(ch, t, xs, xg);
#endif
    return chunk_row_sum_t<BATCH, false>(ch, t, xs, xg);
}

// The producer/consumer ring.  `vecs` lists the row-local vectors to stage
// (nullptr entries are skipped but keep their slot).  body(t, chunk) runs for
// every row t < rows of every chunk in consumer threads.  Must be called by
// all kStreamThreads threads of the CTA; returns when the CTA's chunks are
// done.  Chunks are assigned grid-stride (chunk = cta + i * G).
__device__ __forceinline__ void stream_issue(const Csr& A, const StreamLayout& L, const double2* const* vecs,
                                             unsigned char* sp, uint64_t* bar, int chunk, int k0, int k1,
                                             int cmax, bool uni) {
    const int n = A.n;
    const int r0 = chunk * kStreamRows, rows = min(kStreamRows, n - r0);
    const int a0 = k0 & ~3, a1 = (k1 + 3) & ~3;
    const uint32_t b_rp = (uint32_t)(((rows + 1 + 3) & ~3) * 4);
    const uint32_t b_ci = (uint32_t)((a1 - a0) * 4);
    const uint32_t b_av = (uint32_t)((uni ? rows : k1 - k0) * 16);
    const uint32_t b_v = (uint32_t)(rows * 16);
    uint32_t tx = b_rp + b_ci + b_av;
    for (int j2 = 0; j2 < L.nvec; ++j2)
        if (vecs[j2]) tx += b_v;
    mbar_expect_tx(bar, tx);
    bulk_g2s(sp, A.rp + r0, b_rp, bar);
    unsigned char* q = sp + L.rp_bytes();
    if (b_ci) bulk_g2s(q, A.ci + a0, b_ci, bar);
    q += L.ci_bytes();
    if (b_av) bulk_g2s(q, uni ? A.dg + r0 : A.av + k0, b_av, bar);
    q += L.av_bytes();
    for (int j2 = 0; j2 < L.nvec; ++j2) {
        if (vecs[j2]) bulk_g2s(q, vecs[j2] + r0, b_v, bar);
        q += L.vec_bytes();
    }
    // forward band of the gathered vectors (e.g. the +nx neighbours of the
    // cavity grid): not yet streamed by any CTA, so the consumers' gathers
    // would miss to DRAM -- pull it into L2 now
    if (L.pf_rows > 0 && cmax >= r0 + rows) {
        const int lo = max(r0 + rows, cmax - L.pf_rows + 1), hi = min(cmax, n - 1);
        if (hi >= lo)
            for (int j2 = 0; j2 < L.ngather; ++j2)
                if (vecs[j2]) bulk_prefetch_l2(vecs[j2] + lo, (uint32_t)((hi - lo + 1) * 16));
    }
}

// prof (measurement builds): [0] producer cycles waiting for free stages,
// [1] consumer (thread 0) cycles waiting for full stages, [2] consumer cycles
// in the row body, [3] chunks consumed by thread 0's group
struct NoPre {
    __device__ __forceinline__ void operator()(int, const Chunk&) const {}
};

// pre(t, chunk), when given, runs for every row of the chunk before any
// body() of that chunk (the consumer group syncs on a named barrier in
// between): a phase computes each row's gathered combination once -- e.g.
// p = r + beta (p - omega v) -- into the staged slot of vector 0, so the
// in-chunk gathers read one value instead of recomputing it per entry.
template <class Body, class Pre = NoPre>
__device__ __forceinline__ void stream_rows(const Csr& A, const StreamLayout& L, const double2* const* vecs,
                                            unsigned char* smem, Body&& body, unsigned long long* prof = nullptr,
                                            Pre&& pre = Pre()) {
    constexpr bool kPre = !std::is_same<typename std::decay<Pre>::type, NoPre>::value;
    unsigned long long pw = 0, cw = 0, cb = 0, cn = 0;
    uint64_t* full = (uint64_t*)(smem + (size_t)L.stages * L.stage_bytes());
    uint64_t* empty = full + kStreamMaxStages;
    const int n = A.n;
    const int nchunks = (n + kStreamRows - 1) / kStreamRows;
    const int G = gridDim.x;
    const int tid = threadIdx.x;
    const int ST = L.stages;
    // a group waits on the stage of its next chunk with the parity of that
    // chunk's ring cycle: unambiguous only with at least one stage per group
    // (the launcher guarantees it; a 3-stage ring under the 4-group flavor
    // read stale stages -- found by compute-sanitizer)
    if (ST < kStreamGroups) __trap();
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kStreamRows);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int first = blockIdx.x;
    const int cnt = first < nchunks ? (nchunks - 1 - first) / G + 1 : 0;
    // uniform off-diagonal values (CVK_OPT_UNIFORM_OFFDIAG) only in builds
    // with -DCVK_UNIFORM_OFFDIAG: the second row-sum loop alone cost the
    // default build 2.5 us per BiCGSTAB iteration, and the format bought 2.5%
#ifdef CVK_UNIFORM_OFFDIAG
    const bool uni = A.dg != nullptr && __ldcg(&A.uni[0].x) != 0.0;
#else
    const bool uni = false;
#endif
    const double2 coff = uni ? __ldcg(A.uni + 1) : make_double2(0.0, 0.0);
    if (tid >= kStreamGroups * kStreamRows) {
        const int lane = tid & 31;
        const bool pf = L.pf_rows > 0 && A.cmax != nullptr;
        for (int i0 = 0; i0 < cnt; i0 += 32) {
            const int cj = first + (i0 + lane) * G;
            int k0j = 0, k1j = 0, cmj = -1;
            if (i0 + lane < cnt) {
                k0j = __ldg(A.rp + cj * kStreamRows);
                k1j = __ldg(A.rp + min(cj * kStreamRows + kStreamRows, n));
                if (pf) cmj = __ldg(A.cmax + cj);
            }
            for (int j = 0; j < 32; ++j) {
                if (i0 + j >= cnt) break;
                const int k0 = __shfl_sync(0xffffffffu, k0j, j), k1 = __shfl_sync(0xffffffffu, k1j, j);
                const int cm = __shfl_sync(0xffffffffu, cmj, j);
                if (lane == 0) {
                    const int it = i0 + j, s = it % ST;
                    const long long t0 = prof ? clock64() : 0;
                    mbar_wait(empty + s, ((uint32_t)(it / ST) & 1u) ^ 1u);
                    if (prof) pw += clock64() - t0;
                    stream_issue(A, L, vecs, smem + (size_t)s * L.stage_bytes(), full + s, first + it * G, k0, k1, cm,
                                 uni);
                }
            }
        }
    } else {
        const int g = tid / kStreamRows, t = tid % kStreamRows;
        for (int i = g; i < cnt; i += kStreamGroups) {
            const int s = i % ST;
            const long long t0 = prof ? clock64() : 0;
            mbar_wait(full + s, (uint32_t)(i / ST) & 1u);
            const long long t1 = prof ? clock64() : 0;
            const int chunk = first + i * G;
            const unsigned char* sp = smem + (size_t)s * L.stage_bytes();
            Chunk ch;
            ch.rp = (const int*)sp;
            ch.ci = (const int*)(sp + L.rp_bytes());
            ch.av = (const double2*)(sp + L.rp_bytes() + L.ci_bytes());
            ch.vec = (const double2*)(sp + L.rp_bytes() + L.ci_bytes() + L.av_bytes());
            ch.r0 = chunk * kStreamRows;
            ch.rows = min(kStreamRows, n - ch.r0);
            ch.k0 = ch.rp[0];
            ch.cio = ch.k0 & 3;
            ch.uni = uni;
            ch.coff = coff;
            if (kPre) {
                if (t < ch.rows) pre(t, ch);
                asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(kStreamRows) : "memory");
            }
            if (t < ch.rows) body(t, ch);
            mbar_arrive(empty + s);
            if (prof) {
                const long long t2 = clock64();
                cw += t1 - t0;
                cb += t2 - t1;
                ++cn;
            }
        }
    }
    if (prof) {
        if (tid == kStreamGroups * kStreamRows) prof[0] = pw;
        if (tid == 0) { prof[1] = cw; prof[2] = cb; prof[3] = cn; }
    }
}

}  // namespace cvk
