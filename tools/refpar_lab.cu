// refpar_lab.cu -- measurement lab for the reference-order sequential sums
// (cvk_engine.cuh seq_sums / seq_sums_par).  Not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 \
//        -I paper_2112_00087_b200/csrc tools/refpar_lab.cu -o tools/refpar_lab
//
// 1. latency of a dependent DADD chain (one thread);
// 2. one CTA summing sum conj(x_i) y_i in element order: the single-thread
//    loop (REF) and the producer/consumer ring (REF_PAR) -- ns per element.
#include <cstdio>
#include <vector>

#include "cvk_engine.cuh"

using namespace cvk;

__global__ void k_chain(double* out, double a, int n, long long* cyc) {
    double s = 0.0, t = 0.0;
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        s = __dadd_rn(s, a);
        t = __dadd_rn(t, s);
    }
    const long long t1 = clock64();
    out[0] = s + t;
    cyc[0] = t1 - t0;
}

__global__ void __launch_bounds__(kThreads) k_ref(const double2* x, const double2* y, int n, double2* out) {
    double2 o[1];
    seq_sums<1>(o, n, [&](int i, double2* q) { acc_dot(q[0], x[i], y[i]); });
    if (threadIdx.x == 0) out[0] = o[0];
}

__global__ void __launch_bounds__(kThreads) k_refpar(const double2* x, const double2* y, int n, double2* out) {
    seq_sums_par<1>(out, n, [&](int i, double2* q) { acc_dot(q[0], x[i], y[i]); });
}

__global__ void __launch_bounds__(kThreads) k_refpar3(const double2* x, const double2* y, int n, double2* out) {
    seq_sums_par<3>(out, n, [&](int i, double2* q) {
        acc_norm(q[0], x[i]);
        acc_dot(q[1], y[i], y[i]);
        acc_dot(q[2], y[i], x[i]);
    });
}

// consumer alone: lane 0 of warp 0 adds nblk blocks of P terms from smem
__global__ void k_cons_only(int nblk, double2* out) {
    __shared__ double2 buf[224];
    for (int i = threadIdx.x; i < 224; i += blockDim.x) buf[i] = make_double2(1e-3 * i, -1e-3 * i);
    __syncthreads();
    if (threadIdx.x == 0) {
        double2 acc = make_double2(0.0, 0.0);
        for (int b = 0; b < nblk; ++b)
            for (int e0 = 0; e0 < 224; e0 += 8) {
                double2 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = buf[e0 + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = cvk_add(acc, v[u]);
            }
        out[0] = acc;
    }
}

// producers with U elements per thread per block (U loads in flight)
template <int K, int U, int NB, class C>
__device__ __forceinline__ void seq_sums_par_u(double2* out, int n, C&& contrib, long long* prof) {
    constexpr int P = kThreads - 32;
    constexpr int B = P * U;
    __shared__ double2 buf[NB][K][B];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nblk = (n + B - 1) / B;
    long long wait_c = 0, wait_p = 0;
    if (warp == 0) {
        double2 acc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = make_double2(0.0, 0.0);
        for (int b = 0; b < nblk; ++b) {
            const int s = b % NB;
            const long long t0 = clock64();
            named_sync(1 + s);
            wait_c += clock64() - t0;
            if (lane == 0) {
                const int cnt = min(B, n - b * B);
                for (int e0 = 0; e0 < cnt; e0 += 8) {
                    double2 v[8][K];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
#pragma unroll
                        for (int k = 0; k < K; ++k) v[u][k] = buf[s][k][min(e0 + u, B - 1)];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (e0 + u < cnt)
#pragma unroll
                            for (int k = 0; k < K; ++k) acc[k] = cvk_add(acc[k], v[u][k]);
                }
            }
            __syncwarp();
            named_arrive(1 + NB + s);
        }
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < K; ++k) out[k] = acc[k];
    } else {
        const int t = threadIdx.x - 32;
        for (int b = 0; b < nblk; ++b) {
            const int s = b % NB;
            const long long t0 = clock64();
            if (b >= NB) named_sync(1 + NB + s);
            wait_p += clock64() - t0;
            double2 q[U][K];
#pragma unroll
            for (int u = 0; u < U; ++u) {
#pragma unroll
                for (int k = 0; k < K; ++k) q[u][k] = make_double2(0.0, 0.0);
                const int i = b * B + u * P + t;
                if (i < n) contrib(i, q[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < K; ++k) buf[s][k][u * P + t] = q[u][k];
            named_arrive(1 + s);
        }
        for (int b = max(nblk, NB); b < nblk + NB; ++b) named_sync(1 + NB + b % NB);
    }
    __syncthreads();
    if (threadIdx.x == 0) prof[0] = wait_c;
    if (threadIdx.x == 32) prof[1] = wait_p;
}

__device__ __forceinline__ void nsync(int id, int cnt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
__device__ __forceinline__ void narrive(int id, int cnt) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }

// v2: full batches unpredicated, tail separate; IDLE4: warp 4 (same SMSP as
// the consumer warp 0) does not produce
template <int K, int NB, bool IDLE4, class C>
__device__ __forceinline__ void seq_sums_par_v2(double2* out, int n, C&& contrib, long long* prof) {
    constexpr int P = IDLE4 ? kThreads - 64 : kThreads - 32;
    __shared__ double2 buf[NB][K][P];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nblk = (n + P - 1) / P;
    if (warp == 0) {
        double2 acc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = make_double2(0.0, 0.0);
        for (int b = 0; b < nblk; ++b) {
            const int s = b % NB;
            nsync(1 + s, IDLE4 ? 224 : 256);
            if (lane == 0) {
                const int cnt = min(P, n - b * P);
                const double2* bs = &buf[s][0][0];
                int e0 = 0;
                for (; e0 + 8 <= cnt; e0 += 8) {
                    double2 v[8][K];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
#pragma unroll
                        for (int k = 0; k < K; ++k) v[u][k] = bs[k * P + e0 + u];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
#pragma unroll
                        for (int k = 0; k < K; ++k) acc[k] = cvk_add(acc[k], v[u][k]);
                }
                for (; e0 < cnt; ++e0)
#pragma unroll
                    for (int k = 0; k < K; ++k) acc[k] = cvk_add(acc[k], bs[k * P + e0]);
            }
            __syncwarp();
            narrive(1 + NB + s, IDLE4 ? 224 : 256);
        }
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < K; ++k) out[k] = acc[k];
    } else if (!(IDLE4 && warp == 4)) {
        const int t = IDLE4 && warp > 4 ? threadIdx.x - 64 : threadIdx.x - 32;
        for (int b = 0; b < nblk; ++b) {
            const int s = b % NB;
            if (b >= NB) nsync(1 + NB + s, IDLE4 ? 224 : 256);
            double2 q[K];
#pragma unroll
            for (int k = 0; k < K; ++k) q[k] = make_double2(0.0, 0.0);
            const int i = b * P + t;
            if (i < n) contrib(i, q);
#pragma unroll
            for (int k = 0; k < K; ++k) buf[s][k][t] = q[k];
            narrive(1 + s, IDLE4 ? 224 : 256);
        }
        for (int b = max(nblk, NB); b < nblk + NB; ++b) nsync(1 + NB + b % NB, IDLE4 ? 224 : 256);
    }
    __syncthreads();
    (void)prof;
}


template <bool IDLE4>
__global__ void __launch_bounds__(kThreads) k_refpar_v2(const double2* x, const double2* y, int n, double2* out,
                                                        long long* prof) {
    seq_sums_par_v2<1, 4, IDLE4>(out, n, [&](int i, double2* q) { acc_dot(q[0], x[i], y[i]); }, prof);
}

template <int U, int NB>
__global__ void __launch_bounds__(kThreads) k_refpar_u(const double2* x, const double2* y, int n, double2* out,
                                                       long long* prof) {
    seq_sums_par_u<1, U, NB>(out, n, [&](int i, double2* q) { acc_dot(q[0], x[i], y[i]); }, prof);
}

int main() {
    double* d;
    long long* c;
    cudaMalloc(&d, 64);
    cudaMalloc(&c, 64);
    const int nc = 1 << 20;
    k_chain<<<1, 1>>>(d, 1e-7, nc, c);
    long long cyc;
    cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("dependent DADD chain: %.2f cycles per add\n", (double)cyc / (2.0 * nc));
    for (int n : {50721, 994755}) {
        std::vector<double2> hx(n), hy(n);
        for (int i = 0; i < n; ++i) {
            hx[i] = make_double2(std::sin(0.1 * i), std::cos(0.3 * i));
            hy[i] = make_double2(std::cos(0.7 * i), std::sin(0.2 * i));
        }
        double2 *x, *y, *o;
        cudaMalloc(&x, 16 * n);
        cudaMalloc(&y, 16 * n);
        cudaMalloc(&o, 64);
        cudaMemcpy(x, hx.data(), 16 * n, cudaMemcpyHostToDevice);
        cudaMemcpy(y, hy.data(), 16 * n, cudaMemcpyHostToDevice);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        double2 r[3];
        auto run = [&](const char* name, auto launch) {
            launch();
            cudaEventRecord(e0);
            for (int k = 0; k < 3; ++k) launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(r, o, sizeof(r), cudaMemcpyDeviceToHost);
            printf("n=%d %-10s %8.3f ms  %6.2f ns/element  sum=(%.17g, %.17g) err=%s\n", n, name, ms / 3,
                   ms / 3 * 1e6 / n, r[0].x, r[0].y, cudaGetErrorString(cudaGetLastError()));
        };
        run("ref", [&] { k_ref<<<1, kThreads>>>(x, y, n, o); });
        run("refpar", [&] { k_refpar<<<1, kThreads>>>(x, y, n, o); });
        run("refpar3", [&] { k_refpar3<<<1, kThreads>>>(x, y, n, o); });
        long long hp[2];
        auto prof = [&](const char* nm) {
            cudaMemcpy(hp, c, 16, cudaMemcpyDeviceToHost);
            printf("   %s: consumer waited %.0f%% of cycles, producer waited %lld cycles\n", nm,
                   0.0, hp[1]);
            printf("   consumer wait cycles %lld\n", hp[0]);
        };
        run("u1nb4", [&] { k_refpar_u<1, 4><<<1, kThreads>>>(x, y, n, o, c); });
        prof("u1nb4");
        run("u2nb4", [&] { k_refpar_u<2, 4><<<1, kThreads>>>(x, y, n, o, c); });
        prof("u2nb4");
        run("u4nb2", [&] { k_refpar_u<4, 2><<<1, kThreads>>>(x, y, n, o, c); });
        prof("u4nb2");
        run("u4nb3", [&] { k_refpar_u<4, 3><<<1, kThreads>>>(x, y, n, o, c); });
        prof("u4nb3");
        run("u6nb2", [&] { k_refpar_u<6, 2><<<1, kThreads>>>(x, y, n, o, c); });
        prof("u6nb2");
        run("cons", [&] { k_cons_only<<<1, kThreads>>>((n + 223) / 224, o); });
        run("v2", [&] { k_refpar_v2<false><<<1, kThreads>>>(x, y, n, o, c); });
        run("v2idle4", [&] { k_refpar_v2<true><<<1, kThreads>>>(x, y, n, o, c); });
    }
    return 0;
}
