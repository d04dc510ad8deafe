// numkit_host.cpp -- cavac numkit (reference numkit.cpp) over the C ABI.
// Host containers in, host containers out; the arithmetic runs on the device.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <numeric>

#include "cavac/numkit.hpp"
#include "host_common.hpp"

namespace cavac {
namespace detail {

namespace {
std::atomic<ExecMode> g_mode{ExecMode::Sequential};
std::once_flag g_once;
cvk_ctx* g_ctx = nullptr;
}  // namespace

cvk_ctx* ctx() {
    std::call_once(g_once, [] {
        const char* env = std::getenv("CVK_DEVICE");
        check(cvk_ctx_create(env ? std::atoi(env) : 0, &g_ctx));
    });
    return g_ctx;
}

// Both ExecModes give the reference's iterates bit for bit, as the reference
// promises (numkit.hpp:14-18); Parallel forms the reduction terms with whole
// CTAs (CVK_MODE_REF_PAR).  The FAST arithmetic is SolverOptions::fast_reductions.
int device_mode() { return g_mode.load() == ExecMode::Sequential ? CVK_MODE_REF : CVK_MODE_REF_PAR; }

}  // namespace detail

void set_exec_mode(ExecMode mode) { detail::g_mode.store(mode); }
ExecMode exec_mode() { return detail::g_mode.load(); }

std::vector<Triplet> CsrMatrix::to_triplets() const {
    std::vector<Triplet> t;
    t.reserve(nnz());
    for (std::size_t i = 0; i < nrows; ++i)
        for (std::size_t k = row_offsets[i]; k < row_offsets[i + 1]; ++k) t.push_back({i, col_indices[k], values[k]});
    return t;
}

// numkit.cpp:41-75 semantics: range check, stable (row, col) order,
// duplicates summed in input order, prefix-summed offsets (host setup).
CsrMatrix csr_from_triplets(const std::vector<Triplet>& triplets, std::size_t nrows, std::size_t ncols) {
    for (const Triplet& t : triplets)
        if (t.row >= nrows || t.col >= ncols)
            throw std::invalid_argument("csr_from_triplets: index out of range at (" + std::to_string(t.row) + ", " +
                                        std::to_string(t.col) + ")");
    std::vector<std::size_t> order(triplets.size());
    std::iota(order.begin(), order.end(), std::size_t(0));
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
        return triplets[a].row != triplets[b].row ? triplets[a].row < triplets[b].row
                                                  : triplets[a].col < triplets[b].col;
    });
    CsrMatrix A;
    A.nrows = nrows;
    A.ncols = ncols;
    A.row_offsets.assign(nrows + 1, 0);
    for (std::size_t p = 0; p < order.size();) {
        const Triplet& head = triplets[order[p]];
        Complex sum = head.value;
        std::size_t q = p + 1;
        while (q < order.size() && triplets[order[q]].row == head.row && triplets[order[q]].col == head.col)
            sum += triplets[order[q++]].value;
        A.col_indices.push_back(head.col);
        A.values.push_back(sum);
        ++A.row_offsets[head.row + 1];
        p = q;
    }
    for (std::size_t i = 0; i < nrows; ++i) A.row_offsets[i + 1] += A.row_offsets[i];
    return A;
}

CsrMatrix csr_identity(std::size_t n) {
    CsrMatrix A;
    A.nrows = A.ncols = n;
    A.row_offsets.resize(n + 1);
    std::iota(A.row_offsets.begin(), A.row_offsets.end(), std::size_t(0));
    A.col_indices.resize(n);
    std::iota(A.col_indices.begin(), A.col_indices.end(), std::size_t(0));
    A.values.assign(n, Complex(1.0, 0.0));
    return A;
}

void spmv(const CsrMatrix& A, const CVector& x, CVector& y) {
    if (A.ncols != x.size()) throw std::invalid_argument("spmv: dimension mismatch");
    y.assign(A.nrows, Complex(0.0));
    if (A.nrows == 0) return;
    detail::DevCsr d(A);
    detail::check(cvk_spmv(d.h, reinterpret_cast<const double*>(x.data()), reinterpret_cast<double*>(y.data()),
                           detail::device_mode()));
}

CVector spmv(const CsrMatrix& A, const CVector& x) {
    CVector y;
    spmv(A, x, y);
    return y;
}

Complex dot_hermitian(const CVector& x, const CVector& y) {
    if (x.size() != y.size()) throw std::invalid_argument("dot_hermitian: length mismatch");
    double out[2] = {0.0, 0.0};
    detail::check(cvk_dot(detail::ctx(), (int64_t)x.size(), reinterpret_cast<const double*>(x.data()),
                          reinterpret_cast<const double*>(y.data()), out, detail::device_mode()));
    return {out[0], out[1]};
}

double norm2(const CVector& x) {
    double out = 0.0;
    detail::check(cvk_norm2(detail::ctx(), (int64_t)x.size(), reinterpret_cast<const double*>(x.data()), &out,
                            detail::device_mode()));
    return out;
}

void axpy_inplace(Complex alpha, const CVector& x, CVector& y) {
    if (x.size() != y.size()) throw std::invalid_argument("axpy: length mismatch");
    const double a[2] = {alpha.real(), alpha.imag()};
    detail::check(cvk_axpy(detail::ctx(), (int64_t)x.size(), a, reinterpret_cast<const double*>(x.data()),
                           reinterpret_cast<double*>(y.data())));
}

CVector axpy(Complex alpha, const CVector& x, const CVector& y) {
    if (x.size() != y.size()) throw std::invalid_argument("axpy: length mismatch");
    CVector z = y;
    axpy_inplace(alpha, x, z);
    return z;
}

void xpay_inplace(Complex alpha, CVector& x, const CVector& y) {
    if (x.size() != y.size()) throw std::invalid_argument("xpay: length mismatch");
    const double a[2] = {alpha.real(), alpha.imag()};
    detail::check(cvk_xpay(detail::ctx(), (int64_t)x.size(), a, reinterpret_cast<double*>(x.data()),
                           reinterpret_cast<const double*>(y.data())));
}

void scale_inplace(Complex alpha, CVector& x) {
    for (Complex& z : x) z *= alpha;  // numkit.cpp:161-163 (host, not on any solve path)
}

}  // namespace cavac
