// C++ host API (libcavac_host.so, namespace cavac) on the device: the
// reference's golden run bitwise in Sequential mode, FAST solves, Schwarz and
// the reference's error conventions.  Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <numbers>
#include <sstream>
#include <string>

#include "cavac/helmholtz.hpp"
#include "cavac/krylov.hpp"
#include "cavac/schwarz.hpp"

using namespace cavac;

static int fails = 0;
#define CHECK(c) do { if (!(c)) { std::printf("FAILED: %s (line %d)\n", #c, __LINE__); ++fails; } } while (0)

static std::string slurp(const std::string& p) {
    std::ifstream is(p);
    std::stringstream ss;
    ss << is.rdbuf();
    return ss.str();
}

int main(int argc, char** argv) {
    const std::string gold = argc > 1 ? argv[1] : "tests/golden";
    const double pi = std::numbers::pi;
    // golden system rebuilt by assemble (rhs read back from rhs.csv)
    CavityGrid g = build_grid(2.4, 1.2, 0.05, 0.4, 0.65);
    HelmholtzProblem p = assemble(g, 2.0 * pi * 74.21875, 340.0, CVector(g.roof_size(), Complex(0.0)));
    {
        std::ifstream is(gold + "/rhs.csv");
        std::string line;
        std::getline(is, line);
        std::size_t i = 0;
        while (std::getline(is, line)) {
            double re, im;
            std::sscanf(line.c_str(), "%*zu,%lf,%lf", &re, &im);
            p.b[i++] = Complex(re, im);
        }
        CHECK(i == p.b.size());
    }
    set_exec_mode(ExecMode::Sequential);
    SolveResult r = bicgstab(p.A, p.b, jacobi(p.A), SolverOptions{});
    CHECK(r.report.converged && r.report.iterations == 246);
    std::string out = "index,re,im\n";
    char buf[96];
    for (std::size_t i = 0; i < r.x.size(); ++i) {
        std::snprintf(buf, sizeof buf, "%zu,%.17g,%.17g\n", i, r.x[i].real(), r.x[i].imag());
        out += buf;
    }
    CHECK(out == slurp(gold + "/solution.csv"));
    std::snprintf(buf, sizeof buf, "%.17g", r.report.true_relres);
    CHECK(std::string(buf) == "8.5608367217167752e-10");

    set_exec_mode(ExecMode::Parallel);
    for (SolverId id : {SolverId::BiCGStab, SolverId::BiCGStabL, SolverId::TfQmr}) {
        SolverOptions o;
        o.tol = 1e-12;
        SolveResult f = solve(id, p.A, p.b, jacobi(p.A), o);
        CHECK(f.report.converged && f.report.final_relres <= 1e-12);
        double num = 0, den = 0;
        for (std::size_t i = 0; i < f.x.size(); ++i) { num += std::norm(f.x[i] - r.x[i]); den += std::norm(r.x[i]); }
        CHECK(std::sqrt(num / den) < 1e-7);  // vs the tol-1e-9 golden solution
    }
    // Schwarz (acceptance.cpp:263-291 at h = 0.1)
    CavityGrid gs = build_grid(2.4, 1.2, 0.1, 0.4, 0.65);
    CVector roof(gs.roof_size());
    for (std::size_t i = 0; i < roof.size(); ++i) roof[i] = Complex(1.0 + 0.1 * double(i), 0.3);
    HelmholtzProblem ps = assemble(gs, 2.0 * pi * 13.0, 340.0, roof);
    SolverOptions inner;
    inner.tol = 1e-10;
    SolveResult mono = bicgstab(ps.A, ps.b, jacobi(ps.A), inner);
    const double k = ps.omega / ps.c;
    DdmResult d = schwarz_solve(ps, partition(gs, 3), {Complex(2.0, k), Complex(2.0, k)}, inner, 1e-8, 300);
    CHECK(d.report.converged && d.report.per_subdomain_solves.size() == 3);
    double num = 0, den = 0;
    for (std::size_t i = 0; i < d.x.size(); ++i) { num += std::norm(d.x[i] - mono.x[i]); den += std::norm(mono.x[i]); }
    CHECK(std::sqrt(num / den) <= 1e-6);
    // error conventions
    bool threw = false;
    try { jacobi(csr_from_triplets({{0, 0, Complex(1.0)}, {1, 0, Complex(1.0)}}, 2, 2)); }
    catch (const std::invalid_argument& e) { threw = std::string(e.what()).find("row 1") != std::string::npos; }
    CHECK(threw);
    threw = false;
    try { solver_from_name("cg"); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    SolverOptions few;
    few.max_iter = 3;
    SolveResult e = bicgstab(p.A, p.b, jacobi(p.A), few);
    CHECK(!e.report.converged && e.report.iterations <= 3);
    std::printf("%s (%d failures)\n", fails ? "FAIL" : "OK", fails);
    return fails ? 1 : 0;
}
