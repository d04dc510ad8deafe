// krylov_host.cpp -- cavac Krylov API (reference krylov.cpp) over the C ABI.
// A solve uploads A, recovers the Jacobi inverse diagonal from the
// Preconditioner's callable, and runs one device solve; non-convergence and
// breakdowns come back in the report exactly as the reference reports them.
#include <chrono>

#include "cavac/krylov.hpp"
#include "host_common.hpp"

namespace cavac {

CVector JacobiApply::operator()(const CVector& v) const {
    CVector out(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = inv_diag[i] * v[i];
    return out;
}

Preconditioner identity_preconditioner() { return {IdentityApply{}}; }

// krylov.cpp:31-55: the first col == i entry of each row, inverted with
// std::complex division (libgcc __divdc3, the reference's rounding).  This is
// host setup, one pass over the rows the caller already holds: uploading A
// only to read n values back would double the transfer of a
// jacobi + solve pair (pipeline.cpp:196-202).  The callable keeps the inverse
// diagonal so apply() works as in the reference, and the device solve takes
// it from there (cvk_precond_jacobi with inv_diag).
Preconditioner jacobi(const CsrMatrix& A) {
    if (A.nrows != A.ncols) throw std::invalid_argument("jacobi: matrix must be square");
    JacobiApply f;
    f.inv_diag.assign(A.nrows, Complex(0.0));
    for (std::size_t i = 0; i < A.nrows; ++i) {
        bool found = false;
        for (std::size_t k = A.row_offsets[i]; k < A.row_offsets[i + 1]; ++k)
            if (A.col_indices[k] == i) {
                if (A.values[k] != Complex(0.0)) {
                    f.inv_diag[i] = Complex(1.0) / A.values[k];
                    found = true;
                }
                break;
            }
        if (!found) throw std::invalid_argument("jacobi: zero diagonal at row " + std::to_string(i));
    }
    return {f};
}

namespace {

const char* kBreak[] = {"", "rho breakdown", "stagnation in <shadow, v>", "omega breakdown",
                        "stagnation in <shadow, u>", "degenerate least-squares in MR step", "sigma breakdown",
                        "arnoldi breakdown", "stagnation in <p, A p>"};

SolveResult device_solve(int solver, const char* name, const CsrMatrix& A, const CVector& b,
                         const Preconditioner& M, const SolverOptions& opts) {
    if (A.nrows != A.ncols || A.nrows != b.size()) throw std::invalid_argument(std::string(name) + ": dimension mismatch");
    if (solver == CVK_BICGSTAB_L && opts.l < 1) throw std::invalid_argument("bicgstab_l: l must be >= 1");
    const auto t0 = std::chrono::steady_clock::now();
    SolveResult res;
    res.x.assign(b.size(), Complex(0.0));
    detail::DevCsr d(A);
    cvk_prec* P = nullptr;
    if (const JacobiApply* j = M.apply.target<JacobiApply>()) {
        if (j->inv_diag.size() != A.nrows) throw std::invalid_argument(std::string(name) + ": dimension mismatch");
        detail::check(cvk_precond_jacobi(d.h, reinterpret_cast<const double*>(j->inv_diag.data()), &P));
    } else if (M.apply.target<IdentityApply>()) {
        detail::check(cvk_precond_identity(detail::ctx(), (int64_t)A.nrows, &P));
    } else {
        throw std::invalid_argument(std::string(name) +
                                    ": the device solvers support the jacobi and identity preconditioners");
    }
    cvk_opts o{opts.tol, (int64_t)opts.max_iter, (int64_t)opts.l, (int64_t)opts.m,
               opts.record_history ? 1 : 0, opts.fast_reductions ? CVK_MODE_FAST : detail::device_mode(), 0, 0};
    cvk_report r{};
    std::vector<double> hist;
    if (opts.record_history) {
        hist.assign(2 * opts.max_iter + 8, 0.0);
        r.history = hist.data();
        r.history_cap = (int64_t)hist.size();
    }
    const int e = cvk_solve(detail::ctx(), solver, d.h, P, &o, reinterpret_cast<const double*>(b.data()),
                            reinterpret_cast<double*>(res.x.data()), &r);
    cvk_precond_free(P);
    detail::check(e);
    SolveReport& rep = res.report;
    rep.converged = r.converged != 0;
    rep.iterations = (std::size_t)r.iterations;
    rep.final_relres = r.final_relres;
    rep.true_relres = r.true_relres;
    rep.device_time = r.device_time_s;
    if (opts.record_history)
        rep.residual_history.assign(hist.begin(), hist.begin() + std::min<int64_t>(r.history_len, r.history_cap));
    if (r.breakdown > 0 && r.breakdown < 9) rep.breakdown = kBreak[r.breakdown];
    rep.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return res;
}

}  // namespace

SolveResult bicgstab(const CsrMatrix& A, const CVector& b, const Preconditioner& M, const SolverOptions& o) {
    return device_solve(CVK_BICGSTAB, "bicgstab", A, b, M, o);
}
SolveResult bicgstab_l(const CsrMatrix& A, const CVector& b, const Preconditioner& M, const SolverOptions& o) {
    return device_solve(CVK_BICGSTAB_L, "bicgstab_l", A, b, M, o);
}
SolveResult tfqmr(const CsrMatrix& A, const CVector& b, const Preconditioner& M, const SolverOptions& o) {
    return device_solve(CVK_TFQMR, "tfqmr", A, b, M, o);
}
SolveResult gmres(const CsrMatrix& A, const CVector& b, const Preconditioner& M, const SolverOptions& o) {
    return device_solve(CVK_GMRES, "gmres", A, b, M, o);
}
SolveResult cocg(const CsrMatrix& A, const CVector& b, const Preconditioner& M, const SolverOptions& o) {
    return device_solve(CVK_COCG, "cocg", A, b, M, o);
}

SolverId solver_from_name(const std::string& name) {
    if (name == "bicgstab") return SolverId::BiCGStab;
    if (name == "bicgstab_l") return SolverId::BiCGStabL;
    if (name == "tfqmr") return SolverId::TfQmr;
    throw std::invalid_argument("unknown solver \"" + name + "\" (allowed: bicgstab, bicgstab_l, tfqmr)");
}

std::string solver_name(SolverId id) {
    switch (id) {
        case SolverId::BiCGStab: return "bicgstab";
        case SolverId::BiCGStabL: return "bicgstab_l";
        case SolverId::TfQmr: return "tfqmr";
        case SolverId::GMRES: return "gmres";
        case SolverId::COCG: return "cocg";
    }
    return "?";
}

SolveResult solve(SolverId id, const CsrMatrix& A, const CVector& b, const Preconditioner& M,
                  const SolverOptions& opts) {
    switch (id) {
        case SolverId::BiCGStab: return bicgstab(A, b, M, opts);
        case SolverId::BiCGStabL: return bicgstab_l(A, b, M, opts);
        case SolverId::TfQmr: return tfqmr(A, b, M, opts);
        case SolverId::GMRES: return gmres(A, b, M, opts);
        case SolverId::COCG: return cocg(A, b, M, opts);
    }
    throw std::logic_error("solve: unreachable");
}

}  // namespace cavac
