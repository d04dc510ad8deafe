// cvk_ilu.cu -- ILU(0) preconditioner apply on sm_100a (beyond the reference,
// which has only jacobi / identity_preconditioner, krylov.cpp:27-55;
// SURVEY.md 8(f) rank 4).
//
// The factor is exact ILU(0) on A's pattern (host, cvk_api.cu
// cvk_precond_ilu0 = oracle/cavac_oracle.c orc_ilu0_arrays).  The triangular
// solves are NOT level-scheduled: the 2-D cavity has ~2 (nx + ny) dependent
// levels (~4,200 at 1M DOF), i.e. thousands of grid-wide steps per apply.
// They are sync-free Jacobi sweeps instead, each one fully parallel and one
// HBM pass over a triangle:
//   y_0 = r,          y_k[i] = r[i] - sum_{j<i} l_ij y_{k-1}[j]
//   z_0 = d .* y,     z_k[i] = d[i] (y[i] - sum_{j>i} u_ij z_{k-1}[j]),  d = 1 / u_ii
// The first U sweep forms z_0 = d .* y inside its gathers, so an apply with
// s sweeps per triangle is 2 s launches (s = 0: one elementwise d .* r).
// Sums run in CSR order with one rounding per complex op: the apply is
// bitwise orc_ilu0_apply_arrays.
//
// Bytes per sweep (algorithmic): L or U values + columns (16 + 4 B per
// stored entry) + row pointers (4 B per row) + rhs, gathered vector and
// output (3 x 16 B per row, plus d (16 B) on the U side).
#include <cuda_runtime.h>

#include "cvk_engine.cuh"
#include "cvk_kernels.h"

namespace cvk {

namespace {

constexpr int kIluThreads = 256;

// out[i] = os[i] * (rhs[i] - sum_p av[p] * xs[c] * xin[c]), c = ci[p]; xs / os optional
template <bool XS, bool OS>
__global__ void __launch_bounds__(kIluThreads) k_ilu_sweep(int n, const int* __restrict__ rp,
                                                           const int* __restrict__ ci,
                                                           const double2* __restrict__ av,
                                                           const double2* __restrict__ rhs,
                                                           const double2* __restrict__ xin,
                                                           const double2* __restrict__ xs,
                                                           const double2* __restrict__ os,
                                                           double2* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int p0 = __ldg(rp + i), p1 = __ldg(rp + i + 1);
    double2 s = __ldg(rhs + i);
    for (int p = p0; p < p1; ++p) {
        const int c = __ldg(ci + p);
        double2 xv = __ldg(xin + c);
        if (XS) xv = cvk_mul(__ldg(xs + c), xv);
        s = cvk_sub(s, cvk_mul(__ldg(av + p), xv));
    }
    if (OS) s = cvk_mul(__ldg(os + i), s);
    out[i] = s;
}

__global__ void __launch_bounds__(kIluThreads) k_ilu_scale(int n, const double2* __restrict__ d,
                                                           const double2* __restrict__ y,
                                                           double2* __restrict__ z) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) z[i] = cvk_mul(__ldg(d + i), __ldg(y + i));
}

int ilu_grid(int n) { return (n + kIluThreads - 1) / kIluThreads; }

}  // namespace

// z = M^-1 r for the ILU(0) factor (see the header comment).  tmp holds 2 n
// complex.  r and z must not alias.  Returns the number of launches in *nl.
cudaError_t launch_ilu0_apply(const IluDev& M, const double2* r, double2* z, double2* tmp, int* nl,
                              cudaStream_t st) {
    const int n = M.n;
    if (n <= 0) return cudaSuccess;
    const int G = ilu_grid(n);
    int launches = 0;
    if (M.sweeps <= 0) {
        k_ilu_scale<<<G, kIluThreads, 0, st>>>(n, M.dinv, r, z);
        if (nl) *nl += 1;
        return cudaGetLastError();
    }
    // L sweeps: ping-pong between tmp[0] and tmp[1]; y_0 = r
    double2* buf[2] = {tmp, tmp + n};
    const double2* y = r;
    for (int k = 0; k < M.sweeps; ++k) {
        double2* o = buf[k & 1];
        k_ilu_sweep<false, false><<<G, kIluThreads, 0, st>>>(n, M.lrp, M.lci, M.lav, r, y, nullptr, nullptr, o);
        ++launches;
        y = o;
    }
    // U sweeps: y stays in its buffer; z ping-pongs between z and the other tmp half
    double2* other = (y == buf[0]) ? buf[1] : buf[0];
    // choose the first output so that the last sweep lands in z
    double2* zb[2] = {(M.sweeps & 1) ? z : other, (M.sweeps & 1) ? other : z};
    const double2* zin = y;
    for (int k = 0; k < M.sweeps; ++k) {
        double2* o = zb[k & 1];
        if (k == 0)
            k_ilu_sweep<true, true><<<G, kIluThreads, 0, st>>>(n, M.urp, M.uci, M.uav, y, zin, M.dinv, M.dinv, o);
        else
            k_ilu_sweep<false, true><<<G, kIluThreads, 0, st>>>(n, M.urp, M.uci, M.uav, y, zin, nullptr, M.dinv, o);
        ++launches;
        zin = o;
    }
    if (nl) *nl += launches;
    return cudaGetLastError();
}

}  // namespace cvk
