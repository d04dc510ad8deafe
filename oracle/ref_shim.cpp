// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference core
// (compiled from /root/reference/proj/core/src/*.cpp by oracle/Makefile into
// oracle/_ref/libcavac_ref.so).  TEST INFRASTRUCTURE ONLY: used by tests/ to
// validate the C restatement against the reference itself, and by bench.py's
// cpu_baseline / --impl reference legs as the timed CPU baseline.
//
// Wraps cavac::jacobi + cavac::solve (krylov.hpp:39,68-69), cavac::spmv
// (numkit.hpp:50) and cavac::set_exec_mode (numkit.hpp:20).
#include <cstdint>
#include <cstring>
#include <exception>

#include "cavac/helmholtz.hpp"
#include "cavac/krylov.hpp"
#include "cavac/numkit.hpp"
#include "cavac/schwarz.hpp"

#ifdef CAVAC_HAVE_OPENMP
#include <omp.h>
#endif

namespace {

struct Report {
    int32_t converged;
    int32_t breakdown;
    int64_t iterations;
    double final_relres;
    double true_relres;
    double wall_time_s;
    double* history;
    int64_t history_cap;
    int64_t history_len;
};

cavac::CsrMatrix make_csr(int64_t n, int64_t nnz, const int64_t* rp, const int64_t* ci,
                          const double* v) {
    cavac::CsrMatrix A;
    A.nrows = A.ncols = static_cast<std::size_t>(n);
    A.row_offsets.assign(rp, rp + n + 1);
    A.col_indices.assign(ci, ci + nnz);
    A.values.resize(static_cast<std::size_t>(nnz));
    std::memcpy(A.values.data(), v, sizeof(double) * 2 * static_cast<std::size_t>(nnz));
    return A;
}

int breakdown_code(const std::optional<std::string>& b) {
    if (!b) return 0;
    const char* names[] = {"rho breakdown", "stagnation in <shadow, v>", "omega breakdown",
                           "stagnation in <shadow, u>", "degenerate least-squares in MR step",
                           "sigma breakdown"};
    for (int i = 0; i < 6; ++i)
        if (*b == names[i]) return i + 1;
    return 99;
}

}  // namespace

extern "C" {

void ref_set_exec_mode(int parallel) {
    cavac::set_exec_mode(parallel ? cavac::ExecMode::Parallel : cavac::ExecMode::Sequential);
}

int ref_omp_threads(void) {
#ifdef CAVAC_HAVE_OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void ref_spmv(int64_t n, int64_t nnz, const int64_t* rp, const int64_t* ci, const double* v,
              const double* x, double* y) {
    cavac::CsrMatrix A = make_csr(n, nnz, rp, ci, v);
    cavac::CVector xv(static_cast<std::size_t>(n));
    std::memcpy(xv.data(), x, sizeof(double) * 2 * static_cast<std::size_t>(n));
    cavac::CVector yv = cavac::spmv(A, xv);
    std::memcpy(y, yv.data(), sizeof(double) * 2 * static_cast<std::size_t>(n));
}

// solver: 0 bicgstab, 1 bicgstab_l, 2 tfqmr.  Returns 0, or -1 on an exception.
int ref_solve(int solver, int64_t n, int64_t nnz, const int64_t* rp, const int64_t* ci,
              const double* v, const double* b, double tol, int64_t max_iter, int64_t l,
              int record_history, double* x, Report* rep) {
    try {
        cavac::CsrMatrix A = make_csr(n, nnz, rp, ci, v);
        cavac::CVector bv(static_cast<std::size_t>(n));
        std::memcpy(bv.data(), b, sizeof(double) * 2 * static_cast<std::size_t>(n));
        cavac::SolverOptions o;
        o.tol = tol;
        o.max_iter = static_cast<std::size_t>(max_iter);
        o.l = static_cast<std::size_t>(l);
        o.record_history = record_history != 0;
        cavac::Preconditioner M = cavac::jacobi(A);
        cavac::SolverId id = solver == 0   ? cavac::SolverId::BiCGStab
                             : solver == 1 ? cavac::SolverId::BiCGStabL
                                           : cavac::SolverId::TfQmr;
        cavac::SolveResult r = cavac::solve(id, A, bv, M, o);
        std::memcpy(x, r.x.data(), sizeof(double) * 2 * static_cast<std::size_t>(n));
        rep->converged = r.report.converged ? 1 : 0;
        rep->breakdown = breakdown_code(r.report.breakdown);
        rep->iterations = static_cast<int64_t>(r.report.iterations);
        rep->final_relres = r.report.final_relres;
        rep->true_relres = r.report.true_relres;
        rep->wall_time_s = r.report.wall_time;
        rep->history_len = static_cast<int64_t>(r.report.residual_history.size());
        if (rep->history) {
            const int64_t k = rep->history_len < rep->history_cap ? rep->history_len : rep->history_cap;
            for (int64_t i = 0; i < k; ++i) rep->history[i] = r.report.residual_history[i];
        }
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

}  // extern "C"
