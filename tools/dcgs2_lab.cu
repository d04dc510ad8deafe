// dcgs2_lab.cu -- clock the GMRES scalar step (cvk_dcgs2.cuh) on shared
// memory in one CTA (measurement tool, not product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -Iinclude \
//        -Ipaper_2112_00087_b200/csrc -o tools/_bin/dcgs2_lab tools/dcgs2_lab.cu
#include <cstdio>

#include "cvk_dcgs2.cuh"

using namespace cvk;

__global__ void k_lab(int j, int M, int nt_active, long long* out) {
    extern __shared__ __align__(16) unsigned char sm[];
    GmView v;
    v.M = M;
    v.Hu = (double2*)sm;
    v.R = v.Hu + (M + 1) * M;
    v.sn = v.R + (M + 1) * M;
    v.g = v.sn + M + 1;
    v.gpre = v.g + M + 1;
    v.yv = v.gpre + M + 1;
    v.av = v.yv + M + 1;
    v.bv = v.av + M + 1;
    v.ev = v.bv + M + 1;
    v.cs = (double*)(v.ev + M + 1);
    v.nu = v.cs + M + 1;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < (M + 1) * M; i += nt) {
        v.Hu[i] = make_double2(1.0 / (1 + i), 0.5 / (2 + i));
        v.R[i] = v.Hu[i];
    }
    for (int i = tid; i <= M; i += nt) {
        v.sn[i] = make_double2(0.1, 0.01 * i);
        v.cs[i] = 0.99;
        v.g[i] = make_double2(1, 0);
        v.gpre[i] = make_double2(1, 0);
        v.av[i] = make_double2(i == j ? 1.0 : 1e-9 * i, 1e-10);
        v.bv[i] = make_double2(0.3 + 0.01 * i, 0.1);
    }
    __syncthreads();
    long long t0 = clock64();
    const double nu = gm_dcgs2_scalars(v, j, tid, nt, [] { __syncthreads(); });
    long long t1 = clock64();
    if (tid == 0) gm_provisional(v, j, 0.5, nu);
    __syncthreads();
    long long t2 = clock64();
    if (tid == 0) gm_back_subst(v, j + 1, v.yv);
    __syncthreads();
    long long t3 = clock64();
    if (tid == 0) {
        out[0] = t1 - t0;
        out[1] = t2 - t1;
        out[2] = t3 - t2;
        out[3] = (long long)(v.yv[0].x * 1e6);
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    const int M = 30;
    const size_t smem = 2 * (M + 1) * M * 16 + 8 * (M + 1) * 16 + 2 * (M + 1) * 8;
    cudaFuncSetAttribute(k_lab, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    printf("j threads  scalars provisional back_subst (cycles)\n");
    for (int nt : {32, 544})
        for (int j : {1, 4, 14, 29}) {
            long long h[4];
            for (int rep = 0; rep < 2; ++rep) {
                k_lab<<<1, nt, smem>>>(j, M, nt, d);
                cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
            }
            printf("%2d %4d %8lld %8lld %8lld\n", j, nt, h[0], h[1], h[2]);
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
