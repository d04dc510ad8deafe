// cavac/helmholtz.hpp -- matrix-assembly input of the solve path
// (reference: proj/core/include/cavac/helmholtz.hpp).  The grid and the
// 5-point assembly are host setup; the line-sampling / spectrum helpers of
// the reference are declared when the reference's spectra.hpp is on the
// include path (drop-in builds of the full reference pipeline).
#ifndef CAVAC_HELMHOLTZ_HPP
#define CAVAC_HELMHOLTZ_HPP

#include <cstddef>
#include <string>
#include <utility>
#include <vector>

#include "cavac/numkit.hpp"
#if __has_include("cavac/spectra.hpp")
#include "cavac/spectra.hpp"
#define CAVAC_HAVE_SPECTRA 1
#endif

namespace cavac {

struct CavityGrid {
    double width = 2.4;
    double height = 1.2;
    double h = 0.05;
    std::size_t nx = 0;
    std::size_t ny = 0;
    std::size_t roof_begin = 0;
    std::size_t roof_end = 0;
    Complex wall_admittance{0.0, 0.0};

    std::size_t size() const { return nx * ny; }
    std::size_t node(std::size_t ix, std::size_t iy) const { return iy * nx + ix; }
    double x_of(std::size_t ix) const { return static_cast<double>(ix + 1) * h; }
    double y_of(std::size_t iy) const { return static_cast<double>(iy + 1) * h; }
    std::size_t roof_size() const { return roof_end - roof_begin; }
};

struct HelmholtzProblem {
    CavityGrid grid;
    double omega = 0.0;
    double c = 340.0;
    CVector dirichlet;
    CsrMatrix A;
    CVector b;
};

CavityGrid build_grid(double width, double height, double h, double roof_fraction_start,
                      double roof_fraction_end, Complex wall_admittance = Complex(0.0));
HelmholtzProblem assemble(const CavityGrid& grid, double omega, double c, const CVector& dirichlet);

struct ManufacturedProblem {
    HelmholtzProblem problem;
    CVector exact;
};
ManufacturedProblem manufactured_problem(const CavityGrid& grid, std::size_t m, std::size_t n,
                                         double omega, double c);

struct LineSpec {
    bool horizontal;
    double coordinate;
};
struct LineProfile {
    bool horizontal;
    double coordinate;
    std::vector<std::pair<double, double>> samples;
};
// Post-processing, off the solve path: declared for the reference's
// pipeline.cpp, defined by the reference's own helmholtz.cpp (not by
// libcavac_host.so).
std::vector<LineProfile> sample_lines(const HelmholtzProblem& problem, const CVector& solution,
                                      const std::vector<LineSpec>& lines);
void write_profiles_csv(const std::string& path, const std::vector<LineProfile>& profiles);
void write_rhs_csv(const std::string& path, const CVector& b);
#ifdef CAVAC_HAVE_SPECTRA
CVector dirichlet_from_spectrum(const std::vector<Spectrum>& roof_spectra, std::size_t bin);
#endif

}  // namespace cavac

#endif
