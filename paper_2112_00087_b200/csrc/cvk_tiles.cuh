// cvk_tiles.cuh -- row tiles streamed into shared memory by bulk copies
// (cp.async.bulk + mbarrier transaction counts) through a ring of stages:
// one producer warp (the CTA's last) and NG consumer groups of GT threads,
// group g taking the CTA's tiles g, g + NG, ...  A CTA's tiles are
// b, b + G, b + 2G, ... (b = blockIdx.x), walked bottom-up or, with DESC,
// top-down.
//
// A tile is nc copies: copy c reads bytes[c] from src[c] + tile * stride[c]
// (double2 units) into the stage, one after the other.  Sources are padded
// to whole tiles, so every tile moves the same bytes; the consumers get the
// tile's row count.  Used by the GMRES basis passes (cvk_gmres.cu), whose
// basis is stored block-major so that a 128-row block of j + 1 vectors is
// ONE copy.  Throughput is set by the bytes per stage, not by the ring depth
// or the copy count (tools/tma_lab.cu on the B200, one CTA per SM, 3+
// stages): 2 KB stages 1.0 TB/s, 4 KB 1.7-2.0, 8 KB 3.4-4.0, 16 KB 4.1-6.2,
// 32 KB and more 6.2-6.4 TB/s -- so the callers size tiles for >= 32 KB.
//
// The ring needs at least NG stages: a group waits on the stage of its next
// tile i with the parity of i's ring cycle, which is unambiguous only if the
// stage's previous tile i - ST was already loaded -- true when i - ST is at
// most the group's last tile i - NG.
#pragma once

#include "cvk_stream.cuh"

namespace cvk {

constexpr int kTileMaxCopies = 10;


struct TileCopies {
    const double2* src[kTileMaxCopies];
    long long stride[kTileMaxCopies];  // double2 per tile
    int bytes[kTileMaxCopies];
    int nc, stage_bytes;               // stage_bytes: sum of bytes, a multiple of 128
};

struct NoTilePre {
    __device__ void operator()() const {}
};

// pre(): run once by the consumer threads before their first tile (e.g. a
// programmatic-dependency wait that the producer skips)
template <int NG, int GT, bool DESC, class Body, class Pre = NoTilePre>
__device__ __forceinline__ void tile_stream(int n, int TR, const TileCopies& tc, unsigned char* smem,
                                            int smem_bytes, Body&& body, Pre&& pre = Pre()) {
    const int tid = threadIdx.x, lane = tid & 31;
    const size_t sb = (size_t)tc.stage_bytes;
    const int ST = (int)min((size_t)kStreamMaxStages, ((size_t)smem_bytes - 2 * kStreamMaxStages * 8) / sb);
    if (ST < NG) __trap();  // the launcher sizes the ring (parity aliasing otherwise)
    uint64_t* full = (uint64_t*)(smem + (size_t)ST * sb);
    uint64_t* empty = full + kStreamMaxStages;
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, GT);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int ntiles = (n + TR - 1) / TR, G = gridDim.x;
    const int mine = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / G + 1 : 0;
    auto tile_of = [&](int i) { return (int)blockIdx.x + (DESC ? mine - 1 - i : i) * G; };
    if (tid >= NG * GT) {  // producer warp: lane 0 issues, the loop is warp-uniform
        for (int i = 0; i < mine; ++i) {
            const int s = i % ST, tile = tile_of(i);
            if (lane == 0) {
                mbar_wait(empty + s, ((uint32_t)(i / ST) & 1u) ^ 1u);
                mbar_expect_tx(full + s, (uint32_t)tc.stage_bytes);
                unsigned char* sp = smem + (size_t)s * sb;
                for (int c = 0; c < tc.nc; ++c) {
                    bulk_g2s(sp, tc.src[c] + (long long)tile * tc.stride[c], (uint32_t)tc.bytes[c], full + s);
                    sp += tc.bytes[c];
                }
            }
            __syncwarp();
        }
    } else {
        const int g = tid / GT, t = tid % GT;
        pre();
        for (int i = g; i < mine; i += NG) {
            const int s = i % ST, r0 = tile_of(i) * TR;
            mbar_wait(full + s, (uint32_t)(i / ST) & 1u);
            body(g, t, r0, min(TR, n - r0), (const double2*)(smem + (size_t)s * sb));
            mbar_arrive(empty + s);
        }
    }
}

}  // namespace cvk
