// schwarz_host.cpp -- cavac Schwarz API (reference schwarz.cpp) over the C ABI
// (cvk_partition / cvk_schwarz_solve); tuning and CSV output on the host.
#include <cstdio>
#include <fstream>

#include "cavac/schwarz.hpp"
#include "host_common.hpp"

namespace cavac {

Partition partition(const CavityGrid& grid, std::size_t n_sub) {
    std::vector<int64_t> cb(n_sub + 1, 0);
    if (n_sub < 1) throw std::invalid_argument("partition: n_sub must be >= 1");
    detail::check(cvk_partition((int64_t)grid.nx, (int64_t)n_sub, cb.data()));
    Partition p;
    p.n_sub = n_sub;
    p.col_begin.assign(cb.begin(), cb.end());
    for (std::size_t s = 1; s < n_sub; ++s) p.cut_columns.push_back(p.col_begin[s]);
    return p;
}

DdmResult schwarz_solve(const HelmholtzProblem& problem, const Partition& part, const TransmissionParams& tp,
                        const SolverOptions& inner, double ddm_tol, std::size_t max_outer, SolverId inner_solver) {
    const CavityGrid& g = problem.grid;
    cvk_grid cg{g.width, g.height, g.h, (int64_t)g.nx, (int64_t)g.ny, (int64_t)g.roof_begin, (int64_t)g.roof_end,
                g.wall_admittance.real(), g.wall_admittance.imag()};
    std::vector<int64_t> cb(part.col_begin.begin(), part.col_begin.end());
    const double sl[2] = {tp.s_left.real(), tp.s_left.imag()};
    const double sr[2] = {tp.s_right.real(), tp.s_right.imag()};
    cvk_opts o{inner.tol, (int64_t)inner.max_iter, (int64_t)inner.l, (int64_t)inner.m, 0,
               inner.fast_reductions ? CVK_MODE_FAST : detail::device_mode(), 0, 0};
    DdmResult res;
    res.x.assign(problem.A.nrows, Complex(0.0));
    std::vector<double> hist(max_outer + 1, 0.0);
    std::vector<cvk_report> subs(std::max<std::size_t>(1, part.n_sub));
    cvk_ddm_report r{};
    r.jump_history = hist.data();
    r.jump_cap = (int64_t)hist.size();
    r.sub_reports = subs.data();
    r.n_sub_reports = (int64_t)subs.size();
    const CsrMatrix& A = problem.A;
    detail::check(cvk_schwarz_solve(detail::ctx(), &cg, problem.c, (int64_t)A.nrows, (int64_t)A.nnz(),
                                    reinterpret_cast<const uint64_t*>(A.row_offsets.data()),
                                    reinterpret_cast<const uint64_t*>(A.col_indices.data()),
                                    reinterpret_cast<const double*>(A.values.data()),
                                    reinterpret_cast<const double*>(problem.b.data()), (int64_t)part.n_sub, cb.data(),
                                    sl, sr, &o, ddm_tol, (int64_t)max_outer, (int)inner_solver,
                                    reinterpret_cast<double*>(res.x.data()), &r));
    static const char* kBreak[] = {"", "rho breakdown", "stagnation in <shadow, v>", "omega breakdown",
                                   "stagnation in <shadow, u>", "degenerate least-squares in MR step",
                                   "sigma breakdown", "arnoldi breakdown"};
    res.report.outer_iterations = (std::size_t)r.outer_iterations;
    res.report.converged = r.converged != 0;
    res.report.interface_residual_history.assign(hist.begin(),
                                                 hist.begin() + std::min<int64_t>(r.jump_len, r.jump_cap));
    for (std::size_t s = 0; s < part.n_sub; ++s) {
        SolveReport sr2;
        sr2.converged = subs[s].converged != 0;
        sr2.iterations = (std::size_t)subs[s].iterations;
        sr2.final_relres = subs[s].final_relres;
        sr2.true_relres = subs[s].true_relres;
        if (subs[s].breakdown > 0 && subs[s].breakdown < 8) sr2.breakdown = kBreak[subs[s].breakdown];
        res.report.per_subdomain_solves.push_back(sr2);
    }
    return res;
}

// schwarz.cpp:240-280
TuneResult tune_parameters(const HelmholtzProblem& problem, const Partition& part,
                           const std::vector<TransmissionParams>& candidates, const SolverOptions& inner,
                           std::size_t budget) {
    if (candidates.empty()) throw std::invalid_argument("tune_parameters: empty candidate grid");
    TuneResult out;
    bool any = false;
    std::size_t best_outer = 0, best_inner = 0;
    for (const TransmissionParams& tp : candidates) {
        DdmResult r = schwarz_solve(problem, part, tp, inner, 1e-6, budget);
        TuneEntry e{tp, r.report.outer_iterations, 0, r.report.converged};
        for (const SolveReport& s : r.report.per_subdomain_solves) e.total_inner_iterations += s.iterations;
        out.table.push_back(e);
        if (!e.converged) continue;
        if (!any || e.outer_iterations < best_outer ||
            (e.outer_iterations == best_outer && e.total_inner_iterations < best_inner)) {
            any = true;
            best_outer = e.outer_iterations;
            best_inner = e.total_inner_iterations;
            out.best = tp;
        }
    }
    if (!any) {
        std::string msg = "tune_parameters: all candidates diverged;";
        for (const TuneEntry& e : out.table)
            msg += " (" + std::to_string(e.params.s_left.real()) + "+" + std::to_string(e.params.s_left.imag()) +
                   "i / " + std::to_string(e.params.s_right.real()) + "+" + std::to_string(e.params.s_right.imag()) +
                   "i: " + std::to_string(e.outer_iterations) + ")";
        throw std::runtime_error(msg);
    }
    return out;
}

// schwarz.cpp:282-301
std::vector<TransmissionParams> default_candidate_grid(double k) {
    std::vector<TransmissionParams> out;
    out.push_back({Complex(0.0, k), Complex(0.0, k)});
    const double re[] = {0.25, 1.0, 4.0, 16.0, 64.0};
    const double im[] = {0.0, 0.25, 1.0, 4.0, 16.0};
    for (double a : re)
        for (double b : im) out.push_back({Complex(a * k, b * k), Complex(a * k, b * k)});
    for (double a : re) {
        const Complex s(a * k, k);
        out.push_back({s, 2.0 * s});
        out.push_back({2.0 * s, s});
    }
    return out;
}

void write_ddm_report_csv(const std::string& path, const Partition& part, const TransmissionParams& tp,
                          const DdmReport& report) {
    std::ofstream os(path);
    if (!os) throw std::runtime_error("cannot open " + path + " for writing");
    char buf[200];
    std::snprintf(buf, sizeof buf, "%zu,%.17g,%.17g,%.17g,%.17g,%zu,%d\n", part.n_sub, tp.s_left.real(),
                  tp.s_left.imag(), tp.s_right.real(), tp.s_right.imag(), report.outer_iterations,
                  report.converged ? 1 : 0);
    os << "n_sub,s_left_re,s_left_im,s_right_re,s_right_im,outer_iters,converged\n" << buf;
}

void write_tune_table_csv(const std::string& path, const std::vector<TuneEntry>& table) {
    std::ofstream os(path);
    if (!os) throw std::runtime_error("cannot open " + path + " for writing");
    os << "s_left_re,s_left_im,s_right_re,s_right_im,outer_iters,total_inner_iters,converged\n";
    char buf[220];
    for (const TuneEntry& e : table) {
        std::snprintf(buf, sizeof buf, "%.17g,%.17g,%.17g,%.17g,%zu,%zu,%d\n", e.params.s_left.real(),
                      e.params.s_left.imag(), e.params.s_right.real(), e.params.s_right.imag(), e.outer_iterations,
                      e.total_inner_iterations, e.converged ? 1 : 0);
        os << buf;
    }
}

}  // namespace cavac
