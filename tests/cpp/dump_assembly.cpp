// Dumps cavac::assemble / cavac::manufactured_problem from libcavac_host.so
// as raw little-endian arrays (tests/test_host_assembly.py compares them
// bitwise with helmholtz.py, which is pinned to the golden system).
//   dump_assembly <out_prefix> <h> <freq_hz> <adm_re> <adm_im> <m> <n>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numbers>
#include <string>

#include "cavac/helmholtz.hpp"

template <class T>
static void put(const std::string& path, const T* p, std::size_t n) {
    FILE* f = std::fopen(path.c_str(), "wb");
    std::fwrite(p, sizeof(T), n, f);
    std::fclose(f);
}

static void dump(const std::string& pre, const cavac::CsrMatrix& A, const cavac::CVector& b) {
    std::vector<long long> rp(A.row_offsets.begin(), A.row_offsets.end()), ci(A.col_indices.begin(), A.col_indices.end());
    put(pre + "_rp.bin", rp.data(), rp.size());
    put(pre + "_ci.bin", ci.data(), ci.size());
    put(pre + "_v.bin", A.values.data(), A.values.size());
    put(pre + "_b.bin", b.data(), b.size());
}

int main(int argc, char** argv) {
    if (argc != 8) return 2;
    const std::string pre = argv[1];
    const double h = std::atof(argv[2]), f = std::atof(argv[3]);
    const cavac::Complex adm(std::atof(argv[4]), std::atof(argv[5]));
    const auto g = cavac::build_grid(2.4, 1.2, h, 0.4, 0.65, adm);
    std::printf("%zu %zu %zu %zu\n", g.nx, g.ny, g.roof_begin, g.roof_end);
    const double om = 2 * std::numbers::pi * f;
    cavac::CVector dir(g.roof_size());
    for (std::size_t i = 0; i < dir.size(); ++i) dir[i] = cavac::Complex(1.0 + 0.01 * i, -0.5 * i);
    const auto p = cavac::assemble(g, om, 340.0, dir);
    dump(pre + "_asm", p.A, p.b);
    const auto mp = cavac::manufactured_problem(g, std::atoi(argv[6]), std::atoi(argv[7]), om, 340.0);
    dump(pre + "_man", mp.problem.A, mp.problem.b);
    put(pre + "_man_exact.bin", mp.exact.data(), mp.exact.size());
    return 0;
}
