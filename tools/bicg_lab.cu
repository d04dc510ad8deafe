// bicg_lab.cu -- BiCGSTAB phase-kernel variant sweep (measurement tool, not product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -lineinfo -o tools/bicg_lab tools/bicg_lab.cu
// The reference 5-point cavity pattern (nx x ny); phase A (fused p-update in
// the SpMV gathers + Jacobi + <shadow, v>) and phase C (streaming x/r update
// + two reductions) in three shapes each:
//   *0  one 256-row chunk per CTA, thread per row (the r01 product kernels)
//   *1  grid-stride over chunks, row-local loads issued up front
//   *2  TMA bulk-copy pipeline: one producer warp streams each chunk's matrix
//       slab + row-local vectors into a 4-stage shared-memory ring (mbarrier
//       full/empty), two consumer groups of 256 threads compute from it
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ double2 cmul(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cconjmul(double2 a, double2 b) { return cmul(make_double2(a.x, -a.y), b); }

struct Vecs {
    const int* rp; const int* ci; const double2* av;
    const double2 *r, *p, *v, *sh, *dinv;
    double2 *pn, *vn;
    // phase C
    const double2 *s, *t;
    double2 *x, *rr;
    double2* part; unsigned* counter; double2* out;
    double2 beta, nom, omega;
    int n;
};

constexpr int kT = 256;

__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { v.x += __shfl_xor_sync(0xffffffffu, v.x, o); v.y += __shfl_xor_sync(0xffffffffu, v.y, o); }
    return v;
}

// CTA partial (any block size multiple of 32) + last-CTA fold
template <int K>
__device__ void reduce_last(double2 (&acc)[K], const Vecs& a) {
    __shared__ double2 sm[K][32];
    __shared__ int s_last;
    const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int G = gridDim.x;
#pragma unroll
    for (int k = 0; k < K; ++k) { double2 v = warp_sum(acc[k]); if (l == 0) sm[k][w] = v; }
    __syncthreads();
    if (threadIdx.x < K) {
        double2 s = sm[threadIdx.x][0];
        for (int i = 1; i < nw; ++i) s = cadd(s, sm[threadIdx.x][i]);
        a.part[threadIdx.x * G + blockIdx.x] = s;
        __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(a.counter, 1u) == (unsigned)G - 1u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x < 32) {
        for (int k = 0; k < K; ++k) {
            double2 s = make_double2(0, 0);
            for (int b = l; b < G; b += 32) s = cadd(s, __ldcg(a.part + k * G + b));
            s = warp_sum(s);
            if (l == 0) a.out[k] = s;
        }
        if (l == 0) *a.counter = 0;
    }
}

// ------------------------------------------------------------------ A0 ----
__global__ void __launch_bounds__(kT) kA0(Vecs a) {
    const int n = a.n;
    double2 acc[1] = {make_double2(0, 0)};
    for (long long base = (long long)blockIdx.x * kT; base < n; base += (long long)gridDim.x * kT) {
        const int row = (int)(base + threadIdx.x);
        if (row < n) {
            auto pnew = [&](int c) { return cadd(cmul(a.beta, cadd(a.p[c], cmul(a.nom, a.v[c]))), a.r[c]); };
            const int b = __ldg(a.rp + row), e = __ldg(a.rp + row + 1);
            double2 y = make_double2(0, 0);
            for (int k = b; k < e; k += 5) {
                double2 av[5]; int c[5];
#pragma unroll
                for (int u = 0; u < 5; ++u) if (k + u < e) { av[u] = __ldg(a.av + k + u); c[u] = __ldg(a.ci + k + u); }
#pragma unroll
                for (int u = 0; u < 5; ++u) if (k + u < e) y = cadd(y, cmul(av[u], pnew(c[u])));
            }
            const double2 vi = cmul(__ldg(a.dinv + row), y);
            a.pn[row] = pnew(row);
            a.vn[row] = vi;
            acc[0] = cadd(acc[0], cconjmul(a.sh[row], vi));
        }
    }
    reduce_last<1>(acc, a);
}

// ------------------------------------------------------------------ A1 ----
template <int MINB>
__global__ void __launch_bounds__(kT, MINB) kA1(Vecs a) {
    const int n = a.n;
    double2 acc[1] = {make_double2(0, 0)};
    const double2* __restrict__ r = a.r;
    const double2* __restrict__ p = a.p;
    const double2* __restrict__ v = a.v;
    for (long long base = (long long)blockIdx.x * kT; base < n; base += (long long)gridDim.x * kT) {
        const int row = (int)(base + threadIdx.x);
        if (row < n) {
            const int b = __ldg(a.rp + row), e = __ldg(a.rp + row + 1);
            const double2 ri = __ldg(r + row), pi = __ldg(p + row), vi0 = __ldg(v + row);
            const double2 shi = __ldg(a.sh + row), di = __ldg(a.dinv + row);
            auto pnew = [&](int c) { return cadd(cmul(a.beta, cadd(__ldg(p + c), cmul(a.nom, __ldg(v + c)))), __ldg(r + c)); };
            double2 y = make_double2(0, 0);
            for (int k = b; k < e; k += 5) {
                double2 av[5]; int c[5];
#pragma unroll
                for (int u = 0; u < 5; ++u) if (k + u < e) { av[u] = __ldg(a.av + k + u); c[u] = __ldg(a.ci + k + u); }
#pragma unroll
                for (int u = 0; u < 5; ++u) if (k + u < e) y = cadd(y, cmul(av[u], pnew(c[u])));
            }
            const double2 vi = cmul(di, y);
            a.pn[row] = cadd(cmul(a.beta, cadd(pi, cmul(a.nom, vi0))), ri);
            a.vn[row] = vi;
            acc[0] = cadd(acc[0], cconjmul(shi, vi));
        }
    }
    reduce_last<1>(acc, a);
}

// ----------------------------------------------------------- TMA helpers --
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P1;\n"
        "WAIT%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @P1 bra.uni DONE%=;\n"
        " bra.uni WAIT%=;\n"
        "DONE%=:\n}" ::"r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

// TMA phase A: R rows per chunk, NCG consumer groups of R threads, ST stages
template <int R, int NCG, int ST>
struct TmaA {
    static constexpr int kThreads = NCG * R + 32;
    int capK;  // nnz capacity per chunk (multiple of 4)
    __host__ __device__ size_t rp_bytes() const { return (size_t)(R + 4) * 4; }
    __host__ __device__ size_t ci_bytes() const { return (size_t)(capK + 8) * 4; }
    __host__ __device__ size_t av_bytes() const { return (size_t)capK * 16; }
    __host__ __device__ size_t vec_bytes() const { return (size_t)R * 16; }
    __host__ __device__ size_t stage_bytes() const { return rp_bytes() + ci_bytes() + av_bytes() + 5 * vec_bytes(); }
    __host__ __device__ size_t smem() const { return ST * stage_bytes() + 2 * ST * 8 + 16; }
};

// MODE: 0 full, 1 no stores, 2 no global gathers, 3 consumers idle (ring only), 4 no gathers + no stores
template <int R, int NCG, int ST, int MODE = 0>
__global__ void __launch_bounds__(NCG * R + 32, 1) kA2(Vecs a, TmaA<R, NCG, ST> L) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = (uint64_t*)(smem + ST * L.stage_bytes());
    uint64_t* empty = full + ST;
    const int n = a.n;
    const int nchunks = (n + R - 1) / R;
    const int G = gridDim.x;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, R); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto stage_ptr = [&](int s) { return smem + (size_t)s * L.stage_bytes(); };
    double2 acc[1] = {make_double2(0, 0)};
    if (tid >= NCG * R) {
        // producer warp
        const int lane = tid & 31;
        int it = 0;
        for (int c0 = blockIdx.x; c0 < nchunks; c0 += 32 * G) {
            // lane j prefetches the k-range of chunk c0 + j*G
            const int cj = c0 + lane * G;
            int k0j = 0, k1j = 0;
            if (cj < nchunks) {
                k0j = __ldg(a.rp + cj * R);
                k1j = __ldg(a.rp + min(cj * R + R, n));
            }
            for (int j = 0; j < 32; ++j, ++it) {
                const int chunk = c0 + j * G;
                if (chunk >= nchunks) break;
                const int k0 = __shfl_sync(0xffffffffu, k0j, j), k1 = __shfl_sync(0xffffffffu, k1j, j);
                if (lane == 0) {
                    const int s = it % ST;
                    const uint32_t ph = (uint32_t)(it / ST) & 1u;
                    mbar_wait(empty + s, ph ^ 1u);
                    unsigned char* sp = stage_ptr(s);
                    const int r0 = chunk * R, rows = min(R, n - r0);
                    const int a0 = k0 & ~3, a1 = (k1 + 3) & ~3;
                    const uint32_t b_rp = (uint32_t)(((rows + 1 + 3) & ~3) * 4);
                    const uint32_t b_ci = (uint32_t)((a1 - a0) * 4);
                    const uint32_t b_av = (uint32_t)((k1 - k0) * 16);
                    const uint32_t b_v = (uint32_t)(rows * 16);
                    mbar_expect_tx(full + s, b_rp + b_ci + b_av + 5 * b_v);
                    bulk_g2s(sp, a.rp + r0, b_rp, full + s);
                    unsigned char* q = sp + L.rp_bytes();
                    bulk_g2s(q, a.ci + a0, b_ci, full + s);
                    q += L.ci_bytes();
                    if (b_av) bulk_g2s(q, a.av + k0, b_av, full + s);
                    q += L.av_bytes();
                    bulk_g2s(q, a.r + r0, b_v, full + s); q += L.vec_bytes();
                    bulk_g2s(q, a.p + r0, b_v, full + s); q += L.vec_bytes();
                    bulk_g2s(q, a.v + r0, b_v, full + s); q += L.vec_bytes();
                    bulk_g2s(q, a.sh + r0, b_v, full + s); q += L.vec_bytes();
                    bulk_g2s(q, a.dinv + r0, b_v, full + s);
                }
            }
        }
    } else {
        const int g = tid / R, t = tid % R;
        const double2* __restrict__ gr = a.r;
        const double2* __restrict__ gp = a.p;
        const double2* __restrict__ gv = a.v;
        for (int chunk = blockIdx.x + g * G, it = g; chunk < nchunks; chunk += NCG * G, it += NCG) {
            const int s = it % ST;
            const uint32_t ph = (uint32_t)(it / ST) & 1u;
            mbar_wait(full + s, ph);
            const unsigned char* sp = stage_ptr(s);
            const int* srp = (const int*)sp;
            const int* sci = (const int*)(sp + L.rp_bytes());
            const double2* sav = (const double2*)(sp + L.rp_bytes() + L.ci_bytes());
            const double2* sr = (const double2*)(sp + L.rp_bytes() + L.ci_bytes() + L.av_bytes());
            const double2* spp = sr + R;
            const double2* sv = spp + R;
            const double2* ssh = sv + R;
            const double2* sd = ssh + R;
            const int r0 = chunk * R, rows = min(R, n - r0);
            if (MODE != 3 && t < rows) {
                const int k0 = srp[0];
                const int cio = k0 & 3;
                const int b = srp[t] - k0, e = srp[t + 1] - k0;
                auto pn_s = [&](int l) { return cadd(cmul(a.beta, cadd(spp[l], cmul(a.nom, sv[l]))), sr[l]); };
                double2 y = make_double2(0, 0);
                for (int k = b; k < e; k += 5) {
                    double2 av[5], pv[5]; int c[5];
#pragma unroll
                    for (int u = 0; u < 5; ++u) if (k + u < e) { av[u] = sav[k + u]; c[u] = sci[k + u + cio]; }
#pragma unroll
                    for (int u = 0; u < 5; ++u) if (k + u < e) {
                        const unsigned l = (unsigned)(c[u] - r0);
                        if (l < (unsigned)rows || MODE == 2 || MODE == 4) pv[u] = pn_s((int)(l % (unsigned)rows));
                        else pv[u] = cadd(cmul(a.beta, cadd(__ldg(gp + c[u]), cmul(a.nom, __ldg(gv + c[u])))), __ldg(gr + c[u]));
                    }
#pragma unroll
                    for (int u = 0; u < 5; ++u) if (k + u < e) y = cadd(y, cmul(av[u], pv[u]));
                }
                const double2 vi = cmul(sd[t], y);
                if (MODE != 1 && MODE != 4) {
                    a.pn[r0 + t] = pn_s(t);
                    a.vn[r0 + t] = vi;
                }
                acc[0] = cadd(acc[0], cconjmul(ssh[t], vi));
            }
            mbar_arrive(empty + s);
        }
    }
    reduce_last<1>(acc, a);
}

// ------------------------------------------------------------------ C -----
__global__ void __launch_bounds__(kT) kC0(Vecs a) {
    double2 acc[2] = {make_double2(0, 0), make_double2(0, 0)};
    for (long long base = (long long)blockIdx.x * kT; base < a.n; base += (long long)gridDim.x * kT) {
        const int i = (int)(base + threadIdx.x);
        if (i < a.n) {
            const double2 si = a.s[i];
            a.x[i] = cadd(a.x[i], cmul(a.omega, si));
            const double2 ri = cadd(si, cmul(a.nom, a.t[i]));
            a.rr[i] = ri;
            acc[0].x += ri.x * ri.x + ri.y * ri.y;
            acc[1] = cadd(acc[1], cconjmul(a.sh[i], ri));
        }
    }
    reduce_last<2>(acc, a);
}

template <int U>
__global__ void __launch_bounds__(kT) kC1(Vecs a) {
    double2 acc[2] = {make_double2(0, 0), make_double2(0, 0)};
    const long long stride = (long long)gridDim.x * kT;
    for (long long base = (long long)blockIdx.x * kT + threadIdx.x; base < a.n; base += stride * U) {
        double2 s[U], t[U], sh[U], x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = base + u * stride;
            if (i < a.n) { s[u] = __ldcs(a.s + i); t[u] = __ldcs(a.t + i); sh[u] = __ldg(a.sh + i); x[u] = a.x[i]; }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = base + u * stride;
            if (i < a.n) {
                a.x[i] = cadd(x[u], cmul(a.omega, s[u]));
                const double2 ri = cadd(s[u], cmul(a.nom, t[u]));
                a.rr[i] = ri;
                acc[0].x += ri.x * ri.x + ri.y * ri.y;
                acc[1] = cadd(acc[1], cconjmul(sh[u], ri));
            }
        }
    }
    reduce_last<2>(acc, a);
}

__global__ void k_flush(const double4* p, size_t n, double* sink) {
    double acc = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc += p[i].x;
    if (acc == 12345.678) *sink = acc;
}

int main(int argc, char** argv) {
    const int nx = argc > 1 ? atoi(argv[1]) : 1411, ny = argc > 2 ? atoi(argv[2]) : 705;
    const int n = nx * ny;
    std::vector<int> rp(n + 1 + 8, 0), ci;
    std::vector<double2> av;
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
    for (int i = n + 1; i < n + 9; ++i) rp[i] = rp[n];
    const long long nnz = (long long)ci.size();
    for (int i = 0; i < 16; ++i) ci.push_back(0);
    int *d_rp, *d_ci;
    double2* d_av;
    CK(cudaMalloc(&d_rp, sizeof(int) * rp.size()));
    CK(cudaMalloc(&d_ci, sizeof(int) * ci.size()));
    CK(cudaMalloc(&d_av, sizeof(double2) * nnz));
    CK(cudaMemcpy(d_rp, rp.data(), sizeof(int) * rp.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci.data(), sizeof(int) * ci.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_av, av.data(), sizeof(double2) * nnz, cudaMemcpyHostToDevice));
    std::vector<double2> h(n);
    srand(42);
    auto mk = [&]() {
        double2* d;
        CK(cudaMalloc(&d, sizeof(double2) * n));
        for (auto& z : h) z = make_double2(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
        CK(cudaMemcpy(d, h.data(), sizeof(double2) * n, cudaMemcpyHostToDevice));
        return d;
    };
    Vecs a{};
    a.rp = d_rp; a.ci = d_ci; a.av = d_av; a.n = n;
    a.r = mk(); a.p = mk(); a.v = mk(); a.sh = mk(); a.dinv = mk();
    double2* pn = mk(); double2* vn = mk();
    a.pn = pn; a.vn = vn;
    a.s = mk(); a.t = mk(); a.x = mk(); a.rr = mk();
    CK(cudaMalloc(&a.part, sizeof(double2) * 4 * 65536));
    CK(cudaMalloc(&a.counter, 64));
    CK(cudaMemset(a.counter, 0, 64));
    CK(cudaMalloc(&a.out, 64));
    a.beta = make_double2(0.7, 0.1); a.nom = make_double2(-0.3, 0.2); a.omega = make_double2(0.3, -0.2);
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    void* flush;
    const size_t fb = 512ull << 20;
    CK(cudaMalloc(&flush, fb));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytesA = 20.0 * nnz + 4.0 * (n + 1) + 16.0 * n * 7;  // r,p,v,sh,dinv read; pn,vn written
    const double bytesC = 16.0 * n * 6;
    std::vector<double2> ref_vn(n), got(n);
    double2 ref_dot{};
    auto run = [&](const char* name, double bytes, bool isA, auto launch) {
        float sum = 0.f, best = 1e30f;
        const int reps = 20;
        for (int r = 0; r < reps + 3; ++r) {
            k_flush<<<148 * 8, 256>>>((const double4*)flush, fb / sizeof(double4), (double*)flush);
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 3) { sum += ms; best = std::min(best, ms); }
        }
        CK(cudaGetLastError());
        double2 dot;
        CK(cudaMemcpy(&dot, a.out, 16, cudaMemcpyDeviceToHost));
        const char* chk = "";
        if (isA) {
            CK(cudaMemcpy(got.data(), vn, sizeof(double2) * n, cudaMemcpyDeviceToHost));
            if (ref_dot.x == 0 && ref_dot.y == 0) { ref_vn = got; ref_dot = dot; }
            bool same = true;
            for (int i = 0; i < n; ++i) if (got[i].x != ref_vn[i].x || got[i].y != ref_vn[i].y) { same = false; break; }
            chk = same && fabs(dot.x - ref_dot.x) <= 1e-9 * fabs(ref_dot.x) ? "ok" : "MISMATCH";
        }
        printf("%-34s best %7.2f us  avg %7.2f us  %6.0f GB/s (avg) %s\n", name, best * 1e3, sum / reps * 1e3,
               bytes / (sum / reps * 1e-3) / 1e9, chk);
        fflush(stdout);
    };
    const int chunks = (n + 255) / 256;
    run("A0 chunk/CTA", bytesA, true, [&] { kA0<<<chunks, kT>>>(a); });
    int occ1 = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, kA1<1>, kT, 0));
    for (int mult : {1, 2, 4}) {
        char nm[64];
        snprintf(nm, 64, "A1 grid-stride G=%dx%dx148", mult, occ1);
        run(nm, bytesA, true, [&] { kA1<1><<<std::min(chunks, mult * occ1 * nsm), kT>>>(a); });
    }
    int occ4 = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ4, kA1<4>, kT, 0));
    {
        char nm[64];
        snprintf(nm, 64, "A1 minb4 G=%dx148", occ4);
        run(nm, bytesA, true, [&] { kA1<4><<<std::min(chunks, occ4 * nsm), kT>>>(a); });
        run("A1 minb4 chunk/CTA", bytesA, true, [&] { kA1<4><<<chunks, kT>>>(a); });
    }
    // TMA variants
    {
        constexpr int R = 256, NCG = 2, ST = 4;
        TmaA<R, NCG, ST> L;
        int maxk = 0;
        for (int r0 = 0; r0 < n; r0 += R) maxk = std::max(maxk, rp[std::min(r0 + R, n)] - rp[r0]);
        L.capK = (maxk + 3) & ~3;
        const size_t sm = L.smem();
        CK(cudaFuncSetAttribute(kA2<R, NCG, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        char nm[80];
        snprintf(nm, 80, "A2 TMA R=%d NCG=%d ST=%d smem=%zuK", R, NCG, ST, sm / 1024);
        run(nm, bytesA, true, [&] { kA2<R, NCG, ST><<<nsm, TmaA<R, NCG, ST>::kThreads, sm>>>(a, L); });
    }
    {
        constexpr int R = 224, NCG = 2, ST = 4;
        TmaA<R, NCG, ST> L;
        int maxk = 0;
        for (int r0 = 0; r0 < n; r0 += R) maxk = std::max(maxk, rp[std::min(r0 + R, n)] - rp[r0]);
        L.capK = (maxk + 3) & ~3;
        const size_t sm = L.smem();
#define MODEV(M, NAME) \
        CK(cudaFuncSetAttribute(kA2<R, NCG, ST, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
        run(NAME, bytesA, M == 0, [&] { kA2<R, NCG, ST, M><<<nsm, TmaA<R, NCG, ST>::kThreads, sm>>>(a, L); });
        MODEV(0, "A2 R224 full")
        MODEV(1, "A2 R224 no stores")
        MODEV(2, "A2 R224 no global gathers")
        MODEV(4, "A2 R224 no gathers+stores")
        MODEV(3, "A2 R224 ring only (idle consumers)")
    }
    {
        constexpr int R = 128, NCG = 2, ST = 6;
        TmaA<R, NCG, ST> L;
        int maxk = 0;
        for (int r0 = 0; r0 < n; r0 += R) maxk = std::max(maxk, rp[std::min(r0 + R, n)] - rp[r0]);
        L.capK = (maxk + 3) & ~3;
        const size_t sm = L.smem();
        CK(cudaFuncSetAttribute(kA2<R, NCG, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        char nm[80];
        snprintf(nm, 80, "A2 TMA R=%d NCG=%d ST=%d smem=%zuK", R, NCG, ST, sm / 1024);
        run(nm, bytesA, true, [&] { kA2<R, NCG, ST><<<nsm, TmaA<R, NCG, ST>::kThreads, sm>>>(a, L); });
        if (2 * sm <= 227 * 1024)
            run("  same, 2 CTA/SM", bytesA, true, [&] { kA2<R, NCG, ST><<<2 * nsm, TmaA<R, NCG, ST>::kThreads, sm>>>(a, L); });
    }
    {
        constexpr int R = 128, NCG = 4, ST = 8;
        TmaA<R, NCG, ST> L;
        int maxk = 0;
        for (int r0 = 0; r0 < n; r0 += R) maxk = std::max(maxk, rp[std::min(r0 + R, n)] - rp[r0]);
        L.capK = (maxk + 3) & ~3;
        const size_t sm = L.smem();
        CK(cudaFuncSetAttribute(kA2<R, NCG, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        char nm[80];
        snprintf(nm, 80, "A2 TMA R=%d NCG=%d ST=%d smem=%zuK", R, NCG, ST, sm / 1024);
        run(nm, bytesA, true, [&] { kA2<R, NCG, ST><<<nsm, TmaA<R, NCG, ST>::kThreads, sm>>>(a, L); });
    }
    run("C0 chunk/CTA", bytesC, false, [&] { kC0<<<chunks, kT>>>(a); });
    for (int mult : {4, 8}) {
        char nm[64];
        snprintf(nm, 64, "C0 grid-stride G=%dx148", mult);
        run(nm, bytesC, false, [&] { kC0<<<mult * nsm, kT>>>(a); });
    }
    run("C1 U=2 G=8x148", bytesC, false, [&] { kC1<2><<<8 * nsm, kT>>>(a); });
    run("C1 U=4 G=4x148", bytesC, false, [&] { kC1<4><<<4 * nsm, kT>>>(a); });
    run("C1 U=4 G=8x148", bytesC, false, [&] { kC1<4><<<8 * nsm, kT>>>(a); });
    run("C1 U=8 G=4x148", bytesC, false, [&] { kC1<8><<<4 * nsm, kT>>>(a); });
    run("memcpy D2D 6n*16 B", bytesC, false, [&] { cudaMemcpyAsync(a.rr, a.s, sizeof(double2) * n * 1, cudaMemcpyDeviceToDevice); cudaMemcpyAsync(a.x, a.t, sizeof(double2) * n * 1, cudaMemcpyDeviceToDevice); cudaMemcpyAsync(pn, a.sh, sizeof(double2) * n * 1, cudaMemcpyDeviceToDevice); });
    printf("n=%d nnz=%lld bytesA=%.1f MB bytesC=%.1f MB\n", n, nnz, bytesA / 1e6, bytesC / 1e6);
    return 0;
}
