// spmv_lab.cu -- standalone SpMV variant sweep (measurement tool, not product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o spmv_lab tools/spmv_lab.cu
// Builds the reference 5-point cavity pattern (nx x ny) and times variants.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ double2 cmul(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

template <int MODE> __device__ __forceinline__ double2 ldv(const double2* p) {
    if (MODE == 0) return __ldg(p);
    double2 v;
    if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    else asm volatile("ld.global.nc.L1::evict_first.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
template <int MODE> __device__ __forceinline__ int ldi(const int* p) {
    if (MODE == 0) return __ldg(p);
    int v;
    if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    else asm volatile("ld.global.nc.L1::evict_first.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// rows: S lanes per row, one row group per thread group, grid covers all rows
template <int S, int MODE, int TPB>
__global__ void __launch_bounds__(TPB) k_rows(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                             const double2* __restrict__ av, const double2* __restrict__ x,
                                             double2* __restrict__ y) {
    const int lane = threadIdx.x % S;
    const long long row = ((long long)blockIdx.x * TPB + threadIdx.x) / S;
    double2 acc = make_double2(0, 0);
    if (row < n) {
        const int b = rp[row], e = rp[row + 1];
        for (int k = b + lane; k < e; k += S) acc = cadd(acc, cmul(ldv<MODE>(av + k), __ldg(x + ldi<MODE>(ci + k))));
    }
#pragma unroll
    for (int o = S / 2; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (row < n && lane == 0) y[row] = acc;
}

// 5-point specialised: thread per row, exactly 5-slot unrolled with guards
template <int MODE, int TPB>
__global__ void __launch_bounds__(TPB) k_rows_u(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                const double2* __restrict__ av, const double2* __restrict__ x,
                                                double2* __restrict__ y) {
    const long long row = (long long)blockIdx.x * TPB + threadIdx.x;
    if (row >= n) return;
    const int b = rp[row], e = rp[row + 1];
    double2 a[5]; int c[5];
#pragma unroll
    for (int u = 0; u < 5; ++u) if (b + u < e) { a[u] = ldv<MODE>(av + b + u); c[u] = ldi<MODE>(ci + b + u); }
    double2 acc = make_double2(0, 0);
#pragma unroll
    for (int u = 0; u < 5; ++u) if (b + u < e) acc = cadd(acc, cmul(a[u], __ldg(x + c[u])));
    for (int k = b + 5; k < e; ++k) acc = cadd(acc, cmul(ldv<MODE>(av + k), __ldg(x + ldi<MODE>(ci + k))));
    y[row] = acc;
}

// tiled: CTA chunk of TPB rows, entries loaded coalesced into smem products
template <int U, int MODE, int TPB>
__global__ void __launch_bounds__(TPB) k_tiled(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                               const double2* __restrict__ av, const double2* __restrict__ x,
                                               double2* __restrict__ y, int tile) {
    extern __shared__ double2 prod[];
    __shared__ int srp[TPB + 1];
    const long long base = (long long)blockIdx.x * TPB;
    const int t = threadIdx.x;
    srp[t] = rp[(base + t < n) ? base + t : n];
    if (t == 0) srp[TPB] = rp[(base + TPB < n) ? base + TPB : n];
    __syncthreads();
    const int k0 = srp[0], cnt = srp[TPB] - k0;
    for (int k = t; k < cnt; k += U * TPB) {
        double2 a[U]; int c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) if (k + u * TPB < cnt) { a[u] = ldv<MODE>(av + k0 + k + u * TPB); c[u] = ldi<MODE>(ci + k0 + k + u * TPB); }
#pragma unroll
        for (int u = 0; u < U; ++u) if (k + u * TPB < cnt) prod[k + u * TPB] = cmul(a[u], __ldg(x + c[u]));
    }
    __syncthreads();
    const long long row = base + t;
    if (row < n) {
        double2 acc = make_double2(0, 0);
        for (int k = srp[t] - k0; k < srp[t + 1] - k0; ++k) acc = cadd(acc, prod[k]);
        y[row] = acc;
    }
}

// stream: read values + cols once (no gather), write y -- bandwidth ceiling
template <int TPB>
__global__ void __launch_bounds__(TPB) k_stream(long long nnz, int n, const int* __restrict__ ci,
                                                const double2* __restrict__ av, double2* __restrict__ y) {
    const long long i0 = (long long)blockIdx.x * TPB + threadIdx.x;
    double2 acc = make_double2(0, 0);
    for (long long k = i0; k < nnz; k += (long long)gridDim.x * TPB) {
        const double2 a = ldv<1>(av + k);
        acc = cadd(acc, make_double2(a.x + ldi<1>(ci + k), a.y));
    }
    if (i0 < n) y[i0] = acc;
}

int main(int argc, char** argv) {
    const int nx = argc > 1 ? atoi(argv[1]) : 1411, ny = argc > 2 ? atoi(argv[2]) : 705;
    const int n = nx * ny;
    std::vector<int> rp(n + 1), ci;
    std::vector<double2> av;
    ci.reserve(5 * (size_t)n);
    av.reserve(5 * (size_t)n);
    for (int iy = 0; iy < ny; ++iy)
        for (int ix = 0; ix < nx; ++ix) {
            const int r = iy * nx + ix;
            auto add = [&](int c, double v) { ci.push_back(c); av.push_back(make_double2(v, 0.1 * v)); };
            if (iy > 0) add(r - nx, -1.0);
            if (ix > 0) add(r - 1, -1.0);
            add(r, 4.1);
            if (ix + 1 < nx) add(r + 1, -1.0);
            if (iy + 1 < ny) add(r + nx, -1.0);
            rp[r + 1] = (int)ci.size();
        }
    const long long nnz = (long long)ci.size();
    int *d_rp, *d_ci;
    double2 *d_av, *d_x, *d_y;
    CK(cudaMalloc(&d_rp, sizeof(int) * (n + 1)));
    CK(cudaMalloc(&d_ci, sizeof(int) * nnz));
    CK(cudaMalloc(&d_av, sizeof(double2) * nnz));
    CK(cudaMalloc(&d_x, sizeof(double2) * n));
    CK(cudaMalloc(&d_y, sizeof(double2) * n));
    CK(cudaMemcpy(d_rp, rp.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_av, av.data(), sizeof(double2) * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_x, 0, sizeof(double2) * n));
    // flush buffer > L2
    void* flush;
    const size_t fb = 512ull << 20;
    CK(cudaMalloc(&flush, fb));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = 20.0 * nnz + 4.0 * (n + 1) + 32.0 * n;
    int maxtile = 0;
    for (int b = 0; b < n; b += 256) maxtile = std::max(maxtile, rp[std::min(b + 256, n)] - rp[b]);
    auto run = [&](const char* name, auto launch) {
        float best = 1e30f, sum = 0.f;
        const int reps = 20;
        for (int r = 0; r < reps + 3; ++r) {
            CK(cudaMemsetAsync(flush, r, fb));
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 3) { best = std::min(best, ms); sum += ms; }
        }
        CK(cudaGetLastError());
        printf("%-28s best %7.2f us  avg %7.2f us  %6.0f GB/s (avg)\n", name, best * 1e3, sum / reps * 1e3, bytes / (sum / reps * 1e-3) / 1e9);
    };
#define ROWS(S, M, T) run("rows S=" #S " mode=" #M " tpb=" #T, [&] { k_rows<S, M, T><<<(int)(((long long)n * S + T - 1) / T), T>>>(n, d_rp, d_ci, d_av, d_x, d_y); })
    ROWS(1, 0, 256); ROWS(1, 1, 256); ROWS(1, 2, 256);
    ROWS(2, 0, 256); ROWS(2, 1, 256); ROWS(2, 2, 256);
    ROWS(4, 0, 256); ROWS(4, 1, 256);
    ROWS(1, 0, 128); ROWS(2, 0, 128); ROWS(2, 0, 512); ROWS(1, 0, 512);
#define ROWSU(M, T) run("rows5 unrolled mode=" #M " tpb=" #T, [&] { k_rows_u<M, T><<<(n + T - 1) / T, T>>>(n, d_rp, d_ci, d_av, d_x, d_y); })
    ROWSU(0, 256); ROWSU(1, 256); ROWSU(0, 128); ROWSU(0, 512);
#define TILED(U, M, T) run("tiled U=" #U " mode=" #M " tpb=" #T, [&] { \
        int tl = 0; for (int b = 0; b < n; b += T) tl = std::max(tl, rp[std::min(b + T, n)] - rp[b]); \
        cudaFuncSetAttribute(k_tiled<U, M, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, tl * 16); \
        k_tiled<U, M, T><<<(n + T - 1) / T, T, tl * 16>>>(n, d_rp, d_ci, d_av, d_x, d_y, tl); })
    TILED(1, 0, 256); TILED(2, 0, 256); TILED(4, 0, 256); TILED(1, 1, 256); TILED(2, 1, 256);
    TILED(1, 0, 128); TILED(2, 0, 128); TILED(1, 0, 512);
    run("stream (A only, no gather)", [&] { k_stream<256><<<148 * 8, 256>>>(nnz, n, d_ci, d_av, d_y); });
    run("cudaMemcpy D2D of A values", [&] { cudaMemcpyAsync(d_av, d_av + nnz / 2, sizeof(double2) * (nnz / 2), cudaMemcpyDeviceToDevice); });
    printf("n=%d nnz=%lld bytes/spmv=%.1f MB maxtile=%d\n", n, nnz, bytes / 1e6, maxtile);
    return 0;
}
