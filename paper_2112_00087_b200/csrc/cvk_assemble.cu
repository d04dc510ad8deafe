// cvk_assemble.cu -- A(omega) on the device for frequency sweeps.
//
// The reference assembles the cavity operator once per frequency on the host
// (helmholtz.cpp:59-115: 5 triplets per node, stable sort, CSR; 1.4 s at 1M
// DOF).  The sparsity pattern does not depend on omega, so a sweep uploads
// the pattern once and rewrites only the values here: off-diagonals -k^2,
// diagonal 4k^2 - omega^2 minus k^2 w for each missing wall neighbour, in
// the reference's order (left, right, below, above-unless-roof), with the
// wall weight w = 1 / (1 + i omega h beta) computed on the host with
// std::complex (libgcc __divdc3) -- so the values are bitwise the
// reference's.  The rhs (k^2 x roof data) does not depend on omega.
//
// The kernel also checks that A carries the cavity's 5-point pattern (row
// counts and columns); a mismatch reports the first bad row.
#include <cuda_runtime.h>

#include <algorithm>

#include "cvk_engine.cuh"
#include "cvk_kernels.h"

namespace cvk {

namespace {

__global__ void __launch_bounds__(kThreads) k_cavity_values(int nx, int ny, int roof_begin, int roof_end,
                                                            double k2, double om2, double kw_re, double kw_im,
                                                            const int* __restrict__ rp, const int* __restrict__ ci,
                                                            double2* __restrict__ av, int* bad) {
    const long long n = (long long)nx * ny;
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < n;
         r += (long long)gridDim.x * blockDim.x) {
        const int row = (int)r;
        const int ix = row % nx, iy = row / nx;
        const bool has[5] = {iy > 0, ix > 0, true, ix + 1 < nx, iy + 1 < ny};
        const int off[5] = {-nx, -1, 0, 1, nx};
        int cnt = 0;
#pragma unroll
        for (int s = 0; s < 5; ++s) cnt += has[s] ? 1 : 0;
        const int k0 = rp[row];
        if (rp[row + 1] - k0 != cnt) {
            atomicMin(bad, row);
            continue;
        }
        // diagonal: Complex(4 k^2 - omega^2) -= k^2 w per wall side (helmholtz.cpp:84-112)
        double dre = 4.0 * k2 - om2, dim = 0.0;
        const bool roof = (iy + 1 == ny) && ix >= roof_begin && ix < roof_end;
        if (ix == 0) { dre = dre - kw_re; dim = dim - kw_im; }
        if (ix + 1 == nx) { dre = dre - kw_re; dim = dim - kw_im; }
        if (iy == 0) { dre = dre - kw_re; dim = dim - kw_im; }
        if (iy + 1 == ny && !roof) { dre = dre - kw_re; dim = dim - kw_im; }
        int k = k0;
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            if (!has[s]) continue;
            if (ci[k] != row + off[s]) atomicMin(bad, row);
            av[k] = s == 2 ? make_double2(dre, dim) : make_double2(-k2, 0.0);
            ++k;
        }
    }
}

// FEM operator A(omega) = K - omega^2 M + i omega C on a fixed pattern
// (paper_2112_00087_b200/fem3d.py): re = K - (omega omega) M, im = omega C
__global__ void __launch_bounds__(kThreads) k_fem_values(long long nnz, const double* __restrict__ K,
                                                         const double* __restrict__ M, const double* __restrict__ Cd,
                                                         double om2, double omega, double2* __restrict__ av) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (long long)gridDim.x * blockDim.x)
        av[k] = make_double2(K[k] - om2 * M[k], omega * Cd[k]);
}

}  // namespace

cudaError_t launch_fem_values(long long nnz, const double* K, const double* M, const double* Cd, double omega,
                              double2* av, int nsm, cudaStream_t st) {
    const long long blocks = std::min<long long>((nnz + kThreads - 1) / kThreads, 8LL * nsm);
    k_fem_values<<<(unsigned)std::max<long long>(1, blocks), kThreads, 0, st>>>(nnz, K, M, Cd, omega * omega, omega, av);
    return cudaGetLastError();
}

cudaError_t launch_cavity_values(int nx, int ny, int roof_begin, int roof_end, double k2, double om2,
                                 double kw_re, double kw_im, const int* rp, const int* ci, double2* av,
                                 int* bad, int nsm, cudaStream_t st) {
    const long long n = (long long)nx * ny;
    const long long blocks = std::min<long long>((n + kThreads - 1) / kThreads, 8LL * nsm);
    k_cavity_values<<<(unsigned)std::max<long long>(1, blocks), kThreads, 0, st>>>(
        nx, ny, roof_begin, roof_end, k2, om2, kw_re, kw_im, rp, ci, av, bad);
    return cudaGetLastError();
}

}  // namespace cvk
