// e2e_shim.cpp -- bench.py's end-to-end leg through the reference-facing C++
// API (BENCH INFRASTRUCTURE, not part of the product).  A reference caller
// holds a host cavac::CsrMatrix and right-hand side and runs
//     Preconditioner M = jacobi(A);  SolveResult r = solve(id, A, b, M, opts);
// (pipeline.cpp:196-202).  e2e_prepare builds that CsrMatrix once (the
// caller already has it); e2e_run is the timed call: jacobi + solve, i.e. the
// upload of A and b, the device solve and the download of x.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>

#include "cavac/krylov.hpp"

namespace {
cavac::CsrMatrix g_A;
cavac::CVector g_b;
}  // namespace

extern "C" int e2e_prepare(int64_t n, int64_t nnz, const uint64_t* rp, const uint64_t* ci, const double* v,
                           const double* b) {
    g_A.nrows = g_A.ncols = (std::size_t)n;
    g_A.row_offsets.assign(rp, rp + n + 1);
    g_A.col_indices.assign(ci, ci + nnz);
    g_A.values.resize((std::size_t)nnz);
    std::memcpy(g_A.values.data(), v, sizeof(double) * 2 * (std::size_t)nnz);
    g_b.resize((std::size_t)n);
    std::memcpy(g_b.data(), b, sizeof(double) * 2 * (std::size_t)n);
    return 0;
}

// out: [wall seconds, device seconds, iterations, converged, true relres]
extern "C" int e2e_run(double tol, int64_t max_iter, int fast, double* x, double* out) {
    try {
        const auto t0 = std::chrono::steady_clock::now();
        cavac::Preconditioner M = cavac::jacobi(g_A);
        cavac::SolverOptions o;
        o.tol = tol;
        o.max_iter = (std::size_t)max_iter;
        o.fast_reductions = fast != 0;
        cavac::SolveResult r = cavac::solve(cavac::SolverId::BiCGStab, g_A, g_b, M, o);
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::memcpy(x, r.x.data(), sizeof(double) * 2 * r.x.size());
        out[0] = wall;
        out[1] = r.report.device_time;
        out[2] = (double)r.report.iterations;
        out[3] = r.report.converged ? 1.0 : 0.0;
        out[4] = r.report.true_relres;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}
