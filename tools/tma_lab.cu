// tma_lab.cu -- bulk-copy (cp.async.bulk) streaming throughput vs copy size,
// copies per stage and ring depth, one CTA per SM (measurement tool, not
// product).  Each CTA streams its share of a 1 GiB buffer into a ring of
// shared-memory stages; one consumer warp group touches one word per stage.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_lab tools/tma_lab.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mexpect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void marrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t par) {
    asm volatile("{\n .reg .pred P;\nW%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @P bra D%=;\n bra W%=;\nD%=:\n}"
                 ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void bcp(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

// stage = ncopy copies of csize bytes from ncopy separate streams (stream k
// at src + k * stream_stride); tiles round-robin over CTAs
__global__ void __launch_bounds__(160, 1) k_stream(const unsigned char* src, long long stream_bytes, int ncopy,
                                                    int csize, int stages, unsigned long long* sink, long long pitch) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int sb = ncopy * csize;
    uint64_t* full = (uint64_t*)(smem + (size_t)stages * sb);
    uint64_t* empty = full + 16;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < stages; ++s) { minit(full + s, 1); minit(empty + s, 128); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long ntiles = pitch ? stream_bytes / (pitch * ncopy) : stream_bytes / csize;
    const long long mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    unsigned long long acc = 0;
    if (tid >= 128) {
        if (tid == 128)
            for (long long i = 0; i < mine; ++i) {
                const int s = (int)(i % stages);
                const long long tile = blockIdx.x + i * gridDim.x;
                mwait(empty + s, ((uint32_t)(i / stages) & 1u) ^ 1u);
                mexpect(full + s, (uint32_t)sb);
                for (int k = 0; k < ncopy; ++k)
                    bcp(smem + (size_t)s * sb + (size_t)k * csize,
                        pitch ? src + (tile * ncopy + k) * pitch : src + k * stream_bytes + tile * csize, csize, full + s);
            }
    } else {
        for (long long i = 0; i < mine; ++i) {
            const int s = (int)(i % stages);
            mwait(full + s, (uint32_t)(i / stages) & 1u);
            acc += smem[(size_t)s * sb + (tid * 16) % sb];
            marrive(empty + s);
        }
    }
    if (acc == 12345) sink[0] = acc;
}

int main() {
    int nsm = 0, optin = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0));
    const long long total = 1LL << 30;
    unsigned char* buf;
    unsigned long long* sink;
    CK(cudaMalloc(&buf, total));
    CK(cudaMemset(buf, 1, total));
    CK(cudaMalloc(&sink, 8));
    unsigned char* flush;
    CK(cudaMalloc(&flush, 512 << 20));
    CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 4096));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto run = [&](int cs, int nc, int st, long long pitch) {
        const long long sbytes = (long long)cs * nc * st;
        const long long stream_bytes = pitch ? total : total / nc / cs * cs;
        const long long moved = pitch ? (total / (pitch * nc)) * nc * cs : stream_bytes * nc;
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaMemset(flush, rep, 512 << 20));
            CK(cudaEventRecord(e0));
            k_stream<<<nsm, 160, (size_t)sbytes + 512>>>(buf, stream_bytes, nc, cs, st, sink, pitch);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
        }
        printf("%6d %5d %6d %8lld %8.0f %6.0f\n", cs, nc, st, pitch, sbytes / 1024.0 / st, (double)moved / (best * 1e-3) / 1e9);
    };
    printf("csize ncopy stages pitch stage_KB  GB/s\n");
    // GMRES basis blocks: j + 1 slots of 2 KB read from each (m + 1) * 2 KB block (m = 30)
    for (int jj : {0, 1, 2, 4, 8, 14, 29})
        for (int kb : {1, 2, 4, 8}) {
            const int cs = (jj + 1) * 2048;
            if ((long long)cs * kb * 3 + 512 > optin - 4096) continue;
            run(cs, kb, 3, 31 * 2048);
        }
    // the same bytes from dense sources
    for (int cs : {4096, 8192, 16384, 32768}) run(cs, 4, 3, cs);
    for (int cs : {4096, 8192, 16384}) run(cs, 4, 3, 0);
    return 0;
}
