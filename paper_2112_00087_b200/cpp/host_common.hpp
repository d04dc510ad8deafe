// host_common.hpp -- shared plumbing of the C++ host API (libcavac_host.so):
// the process-wide device context and C-ABI error mapping.
#pragma once

#include <stdexcept>
#include <string>

#include "cavac_b200.h"
#include "cavac/numkit.hpp"

namespace cavac::detail {

// Lazily created context on device $CVK_DEVICE (default 0).
cvk_ctx* ctx();

// ExecMode -> CVK_MODE_REF (Sequential) / CVK_MODE_REF_PAR (Parallel)
int device_mode();

// Map a C-ABI status onto the reference's exception types.
inline void check(int code) {
    if (code == CVK_OK) return;
    const std::string msg = cvk_last_error();
    if (code == CVK_EINVAL || code == CVK_EZERODIAG || code == CVK_ESOLVER || code == CVK_EOVERFLOW)
        throw std::invalid_argument(msg);
    if (code == CVK_ELOGIC) throw std::logic_error(msg);
    throw std::runtime_error("cavac device error: " + msg);
}

// RAII device copy of a host CsrMatrix for one call (size_t indices are
// passed through as uint64 and narrowed on the device side).
struct DevCsr {
    cvk_csr* h = nullptr;
    explicit DevCsr(const CsrMatrix& A) {
        static_assert(sizeof(std::size_t) == sizeof(uint64_t), "size_t must be 64-bit");
        check(cvk_csr_upload(ctx(), (int64_t)A.nrows, (int64_t)A.ncols, (int64_t)A.nnz(),
                             reinterpret_cast<const uint64_t*>(A.row_offsets.data()),
                             reinterpret_cast<const uint64_t*>(A.col_indices.data()),
                             reinterpret_cast<const double*>(A.values.data()), &h));
    }
    ~DevCsr() { cvk_csr_free(h); }
    DevCsr(const DevCsr&) = delete;
    DevCsr& operator=(const DevCsr&) = delete;
};

}  // namespace cavac::detail
