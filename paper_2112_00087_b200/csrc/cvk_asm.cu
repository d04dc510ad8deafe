// cvk_asm.cu -- Schwarz domain decomposition on algebraic (FEM / METIS-style)
// subdomains.  Beyond the reference, whose schwarz_solve only knows the FD
// cavity's vertical strips with a Robin ghost elimination specific to the
// 5-point stencil (schwarz.cpp:29-89, 187-208).
//
// Subdomains come from any partition of the rows (RCB of FEM mesh points,
// rowblock.rcb_partition, or a METIS-style graph partition).  Subdomain q owns
// the rows O_q and works on E_q = O_q grown by `overlap` layers of the matrix
// graph.  Its local operator is the restriction A[E_q, E_q] with the
// reference's Robin transmission term generalised to algebraic couplings:
// every coupling a_ij that leaves E_q is folded back into the diagonal with
// the factor theta = (1/h - s/2) / (1/h + s/2) the reference applies to the
// eliminated ghost column (schwarz.cpp:43-50), s = s_robin (2 + ik is the
// acceptance default, acceptance.cpp:272-280).
//
// The preconditioner is restricted additive Schwarz (ORAS):
//     M^-1 r = sum_q R~_q^T A_q^-1 R_q r,
// R_q gathers E_q, R~_q^T scatters back the owned rows only, so the owned
// sets partition the result and the subdomain solves (device Krylov solves,
// cvk_solve_device) never write the same row.  The outer iteration is
// either the plain fixed point u += M^-1 (b - A u) (the reference's additive
// sweep structure) or FGMRES(m) right-preconditioned by M^-1.  Either way
// the iteration's fixed point is b - A u = 0, so at convergence the DDM
// solution IS the monodomain solution (tests/test_gpu_asm.py pins it to the
// reference's monodomain solve).  Helmholtz with one-level Schwarz and more
// than two subdomains diverges as a fixed point on the FEM cavity
// (tools/asm_probe.py); FGMRES converges in tens of sweeps.
//
// Vector algebra of the outer loop runs on this file's kernels and the
// library's double-double dot (cvk_blas.cu); one scalar read-back per
// Arnoldi dot.
//
// Several ranks (one GPU each): rank r builds and solves only the subdomains
// q with q % n_ranks == r; every other operation of the outer loop runs
// redundantly on every rank on full-length vectors.  After the local solves
// each rank holds M^-1 r on its own subdomains' owned rows and zero
// elsewhere, and a caller-supplied sum over ranks (cvk_asm_set_reducer:
// NCCL / gloo all-reduce of n complex values) completes it -- every entry has
// one nonzero contributor, so the sum is exact and the iterates are bitwise
// those of one rank.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/cavac_b200.h"
#include "cvk_complex.h"
#include "cvk_engine.cuh"
#include "cvk_kernels.h"

using cvk::kThreads;
using Cx = std::complex<double>;

namespace {

int afail(int code, const std::string& msg) { return cvk_fail(code, msg); }

#define AK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return afail(e_ == cudaErrorMemoryAllocation ? CVK_ENOMEM : CVK_ECUDA,            \
                         std::string(#call) + ": " + cudaGetErrorString(e_));                 \
    } while (0)
#define AC(call)                          \
    do {                                  \
        const int rc_ = (call);           \
        if (rc_ != CVK_OK) return rc_;    \
    } while (0)

int grid_for(long long n) { return (int)std::max<long long>(1, std::min<long long>((n + kThreads - 1) / kThreads, 4 * 148)); }

__global__ void k_gather(int m, const int* __restrict__ idx, const double2* __restrict__ src, double2* __restrict__ dst) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) dst[i] = src[idx[i]];
}

// dst[idx[own[k]]] = src[own[k]]
__global__ void k_scatter_own(int m, const int* __restrict__ own, const int* __restrict__ idx,
                              const double2* __restrict__ src, double2* __restrict__ dst) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) {
        const int l = own[k];
        dst[idx[l]] = src[l];
    }
}

// y = alpha x (+ y when acc)
__global__ void k_scale(int n, double2 alpha, const double2* __restrict__ x, double2* __restrict__ y, int acc) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double2 t = cvk_mul(alpha, x[i]);
        y[i] = acc ? cvk_add(y[i], t) : t;
    }
}

// r = b - y
__global__ void k_sub(int n, const double2* __restrict__ b, const double2* __restrict__ y, double2* __restrict__ r) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) r[i] = cvk_sub(b[i], y[i]);
}

struct Sub {
    int q = 0;  // global subdomain id
    cvk_csr* A = nullptr;
    cvk_prec* M = nullptr;
    int n_ext = 0, n_own = 0;
    int* d_idx = nullptr;  // E_q, global rows (ascending)
    int* d_own = nullptr;  // positions in E_q of the owned rows
};

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

struct cvk_asm {
    cvk_ctx* ctx = nullptr;
    cudaStream_t st = nullptr;
    int64_t n = 0;
    cvk_csr* A = nullptr;  // the global operator (residuals)
    std::vector<Sub> subs;
    cvk_opts inner{};
    int inner_solver = CVK_BICGSTAB;
    double2 *d_rl = nullptr, *d_xl = nullptr;  // local rhs / solution (max n_ext)
    double2* d_part = nullptr;                 // dot partials
    double2* d_dot = nullptr;                  // one dot result
    int64_t last_inner = 0;                    // inner iterations of the last application
    int last_brk = 0;
    double inner_device_s = 0.0;
    int rank = 0, n_ranks = 1;
    cvk_asm_reduce_fn reduce = nullptr;        // sum over ranks of the owned-row results
    void* reduce_user = nullptr;
    double* reduce_buf = nullptr;              // caller's device buffer (n complex) or null
};

// ||x||^2 or <x, y> (double-double sums, cvk_blas.cu)
static int dev_dot(cvk_asm* S, int n, const double2* x, const double2* y, double2* out) {
    AK(cvk::launch_dot(false, n, x, y, S->d_part, S->d_dot, S->st));
    AK(cudaMemcpyAsync(out, S->d_dot, sizeof(double2), cudaMemcpyDeviceToHost, S->st));
    AK(cudaStreamSynchronize(S->st));
    return CVK_OK;
}

extern "C" {

int cvk_asm_create_rank(cvk_ctx* ctx, int64_t n, int64_t nnz, const uint64_t* rp, const uint64_t* ci, const double* v,
                        int64_t n_parts, const int64_t* part_of_row, int64_t overlap, const double* s_robin, double h,
                        const cvk_opts* inner, int inner_solver, int rank, int n_ranks, cvk_asm** out) {
    if (!ctx || !rp || !part_of_row || !inner || !out || !s_robin)
        return afail(CVK_EINVAL, "cvk_asm_create: null argument");
    if (n < 1 || n_parts < 1 || overlap < 0 || !(h > 0))
        return afail(CVK_EINVAL, "cvk_asm_create: need n >= 1, n_parts >= 1, overlap >= 0, h > 0");
    if (inner_solver < 0 || inner_solver > 4) return afail(CVK_ESOLVER, "cvk_asm_create: unknown inner solver");
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) return afail(CVK_EINVAL, "cvk_asm_create: bad rank / n_ranks");
    std::vector<std::vector<int64_t>> own((size_t)n_parts);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t q = part_of_row[i];
        if (q < 0 || q >= n_parts) return afail(CVK_EINVAL, "cvk_asm_create: part id out of range at row " + std::to_string(i));
        own[(size_t)q].push_back(i);
    }
    for (int64_t q = 0; q < n_parts; ++q)
        if (own[(size_t)q].empty()) return afail(CVK_EINVAL, "cvk_asm_create: empty subdomain " + std::to_string(q));
    auto S = std::make_unique<cvk_asm>();
    S->ctx = ctx;
    S->st = (cudaStream_t)cvk_ctx_stream(ctx);
    S->n = n;
    S->inner = *inner;
    S->inner.record_history = 0;
    S->inner_solver = inner_solver;
    S->rank = rank;
    S->n_ranks = n_ranks;
    AC(cvk_csr_upload(ctx, n, n, nnz, rp, ci, v, &S->A));
    const Cx s(s_robin[0], s_robin[1]);
    const Cx theta = (Cx(1.0 / h) - 0.5 * s) / (Cx(1.0 / h) + 0.5 * s);  // schwarz.cpp:43-50
    const Cx* vals = reinterpret_cast<const Cx*>(v);
    std::vector<int64_t> loc((size_t)n, -1);
    std::vector<char> mark((size_t)n, 0);
    size_t max_ext = 1;
    for (int64_t q = 0; q < n_parts; ++q) {
        if (q % n_ranks != rank) continue;  // another rank's subdomain
        // E_q: the owned rows grown by `overlap` graph layers
        std::vector<int64_t> ext = own[(size_t)q];
        for (int64_t i : ext) mark[(size_t)i] = 1;
        size_t front = 0;
        for (int64_t layer = 0; layer < overlap; ++layer) {
            const size_t end = ext.size();
            for (size_t k = front; k < end; ++k)
                for (uint64_t p = rp[ext[k]]; p < rp[ext[k] + 1]; ++p) {
                    const int64_t j = (int64_t)ci[p];
                    if (!mark[(size_t)j]) { mark[(size_t)j] = 1; ext.push_back(j); }
                }
            front = end;
        }
        std::sort(ext.begin(), ext.end());
        for (size_t k = 0; k < ext.size(); ++k) loc[(size_t)ext[k]] = (int64_t)k;
        // local CSR: rows of E_q, columns inside E_q; couplings leaving E_q
        // folded into the diagonal with theta
        const int64_t m = (int64_t)ext.size();
        std::vector<uint64_t> lrp((size_t)m + 1, 0), lci;
        std::vector<Cx> lv;
        std::vector<int> own_pos;
        for (int64_t k = 0; k < m; ++k) {
            const int64_t i = ext[(size_t)k];
            if (part_of_row[i] == q) own_pos.push_back((int)k);
            Cx cut(0.0);
            int64_t dpos = -1;
            for (uint64_t p = rp[i]; p < rp[i + 1]; ++p) {
                const int64_t j = (int64_t)ci[p];
                if (loc[(size_t)j] >= 0) {
                    if (j == i && dpos < 0) dpos = (int64_t)lv.size();
                    lci.push_back((uint64_t)loc[(size_t)j]);
                    lv.push_back(vals[p]);
                } else {
                    cut += vals[p];
                }
            }
            if (dpos < 0) return afail(CVK_EZERODIAG, "cvk_asm_create: no diagonal at row " + std::to_string(i));
            lv[(size_t)dpos] += theta * cut;
            lrp[(size_t)k + 1] = lci.size();
        }
        Sub sb;
        sb.q = (int)q;
        sb.n_ext = (int)m;
        sb.n_own = (int)own_pos.size();
        AC(cvk_csr_upload(ctx, m, m, (int64_t)lci.size(), lrp.data(), lci.data(),
                          reinterpret_cast<const double*>(lv.data()), &sb.A));
        AC(cvk_precond_jacobi(sb.A, nullptr, &sb.M));
        std::vector<int> idx32(ext.begin(), ext.end());
        AK(cudaMalloc(&sb.d_idx, sizeof(int) * idx32.size()));
        AK(cudaMalloc(&sb.d_own, sizeof(int) * std::max<size_t>(1, own_pos.size())));
        AK(cudaMemcpy(sb.d_idx, idx32.data(), sizeof(int) * idx32.size(), cudaMemcpyHostToDevice));
        AK(cudaMemcpy(sb.d_own, own_pos.data(), sizeof(int) * own_pos.size(), cudaMemcpyHostToDevice));
        S->subs.push_back(sb);
        max_ext = std::max(max_ext, ext.size());
        for (int64_t i : ext) { loc[(size_t)i] = -1; mark[(size_t)i] = 0; }
    }
    AK(cudaMalloc(&S->d_rl, sizeof(double2) * max_ext));
    AK(cudaMalloc(&S->d_xl, sizeof(double2) * max_ext));
    AK(cudaMalloc(&S->d_part, sizeof(double2) * 2048));
    AK(cudaMalloc(&S->d_dot, sizeof(double2)));
    *out = S.release();
    return CVK_OK;
}

int cvk_asm_create(cvk_ctx* ctx, int64_t n, int64_t nnz, const uint64_t* rp, const uint64_t* ci, const double* v,
                   int64_t n_parts, const int64_t* part_of_row, int64_t overlap, const double* s_robin, double h,
                   const cvk_opts* inner, int inner_solver, cvk_asm** out) {
    return cvk_asm_create_rank(ctx, n, nnz, rp, ci, v, n_parts, part_of_row, overlap, s_robin, h, inner, inner_solver,
                               0, 1, out);
}

int cvk_asm_set_reducer(cvk_asm* S, cvk_asm_reduce_fn fn, void* user, double* buf_dev) {
    if (!S) return afail(CVK_EINVAL, "cvk_asm_set_reducer: null argument");
    S->reduce = fn;
    S->reduce_user = user;
    S->reduce_buf = buf_dev;
    return CVK_OK;
}

int cvk_asm_destroy(cvk_asm* S) {
    if (!S) return CVK_OK;
    for (Sub& sb : S->subs) {
        cvk_precond_free(sb.M);
        cvk_csr_free(sb.A);
        cudaFree(sb.d_idx);
        cudaFree(sb.d_own);
    }
    cvk_csr_free(S->A);
    cudaFree(S->d_rl);
    cudaFree(S->d_xl);
    cudaFree(S->d_part);
    cudaFree(S->d_dot);
    delete S;
    return CVK_OK;
}

int64_t cvk_asm_n_parts(const cvk_asm* S) { return S ? (int64_t)S->subs.size() : -1; }

// z = sum_q R~_q^T A_q^-1 R_q r (device vectors of length n, distinct)
int cvk_asm_apply_device(cvk_asm* S, const double* r_dev, double* z_dev) {
    if (!S || !r_dev || !z_dev) return afail(CVK_EINVAL, "cvk_asm_apply: null argument");
    const double2* r = (const double2*)r_dev;
    double2* z = (double2*)z_dev;
    S->last_inner = 0;
    S->last_brk = 0;
    if (S->n_ranks > 1) AK(cudaMemsetAsync(z, 0, sizeof(double2) * (size_t)S->n, S->st));
    for (Sub& sb : S->subs) {
        k_gather<<<grid_for(sb.n_ext), kThreads, 0, S->st>>>(sb.n_ext, sb.d_idx, r, S->d_rl);
        AK(cudaGetLastError());
        cvk_report rep{};
        AC(cvk_solve_device(S->ctx, S->inner_solver, sb.A, sb.M, &S->inner, (const double*)S->d_rl,
                            (double*)S->d_xl, &rep));
        S->last_inner += rep.iterations;
        S->inner_device_s += rep.device_time_s;
        if (rep.breakdown) S->last_brk = 1;
        k_scatter_own<<<grid_for(sb.n_own), kThreads, 0, S->st>>>(sb.n_own, sb.d_own, sb.d_idx, S->d_xl, z);
        AK(cudaGetLastError());
    }
    if (S->n_ranks > 1) {
        if (!S->reduce) return afail(CVK_EINVAL, "cvk_asm_apply: several ranks need cvk_asm_set_reducer");
        const size_t nb = sizeof(double2) * (size_t)S->n;
        double* zb = S->reduce_buf ? S->reduce_buf : (double*)z;
        if (S->reduce_buf) AK(cudaMemcpyAsync(zb, z, nb, cudaMemcpyDeviceToDevice, S->st));
        AK(cudaStreamSynchronize(S->st));
        int64_t meta[2] = {S->last_inner, S->last_brk};
        const int rc = S->reduce(S->reduce_user, zb, S->n, meta);
        if (rc != 0) return afail(CVK_ECUDA, "cvk_asm_apply: reducer failed");
        if (S->reduce_buf) AK(cudaMemcpyAsync(z, zb, nb, cudaMemcpyDeviceToDevice, S->st));
        S->last_inner = meta[0];
        S->last_brk = (int)meta[1];
    }
    return CVK_OK;
}

// The outer DDM iteration.  m = 0: fixed point u <- u + M^-1 (b - A u)
// (the reference's additive sweep, schwarz.cpp:152-234); m > 0: FGMRES(m)
// with M^-1 on the right.  Stops at ||b - A u|| <= tol ||b||.
// rep->outer_iterations counts preconditioner applications (subdomain sweeps),
// rep->jump_history the relative residual after each.
int cvk_asm_solve(cvk_asm* S, const double* b_host, double* x_host, double tol, int64_t max_outer, int64_t m,
                  cvk_ddm_report* rep) {
    if (!S || !b_host || !x_host || !rep) return afail(CVK_EINVAL, "cvk_asm_solve: null argument");
    if (m < 0 || m > 200) return afail(CVK_EINVAL, "cvk_asm_solve: m must be in [0, 200]");
    const double t0 = now_s();
    const int n = (int)S->n;
    const size_t nb = sizeof(double2) * (size_t)n;
    const int nvec = m > 0 ? (int)(2 * m + 5) : 4;  // b, x, r, t, V (m + 1), Z (m)
    double2* W = nullptr;
    AK(cudaMalloc(&W, nb * (size_t)nvec));
    struct Free { void* p; ~Free() { cudaFree(p); } } guard{W};
    double2* b = W;
    double2* x = W + n;
    double2* r = W + 2 * (size_t)n;
    double2* t = W + 3 * (size_t)n;
    double2* V = m > 0 ? W + 4 * (size_t)n : nullptr;  // m + 1 basis vectors
    double2* Z = m > 0 ? W + (size_t)(m + 5) * n : nullptr;  // m preconditioned vectors (flexible)
    AK(cudaMemcpyAsync(b, b_host, nb, cudaMemcpyHostToDevice, S->st));
    AK(cudaMemsetAsync(x, 0, nb, S->st));
    cudaEvent_t e0, e1;
    AK(cudaEventCreate(&e0));
    AK(cudaEventCreate(&e1));
    AK(cudaEventRecord(e0, S->st));
    S->inner_device_s = 0.0;
    double2 d;
    AC(dev_dot(S, n, b, b, &d));
    const double bn = std::sqrt(d.x);
    int64_t outer = 0, hl = 0;
    int conv = 0, brk = 0;
    auto push = [&](double v) {
        if (rep->jump_history && hl < rep->jump_cap) rep->jump_history[hl] = v;
        ++hl;
    };
    auto residual = [&](double* rel) -> int {  // r = b - A x, rel = ||r|| / ||b||
        AC(cvk_spmv_device(S->A, (const double*)x, (double*)t, CVK_MODE_FAST));
        k_sub<<<grid_for(n), kThreads, 0, S->st>>>(n, b, t, r);
        AK(cudaGetLastError());
        double2 q;
        AC(dev_dot(S, n, r, r, &q));
        *rel = bn > 0 ? std::sqrt(q.x) / bn : std::sqrt(q.x);
        return CVK_OK;
    };
    double rel = 0.0;
    if (bn == 0.0) {
        conv = 1;
    } else if (m == 0) {
        AC(residual(&rel));
        while (rel > tol && outer < max_outer && std::isfinite(rel) && rel < 1e6) {
            AC(cvk_asm_apply_device(S, (const double*)r, (double*)t));
            brk |= S->last_brk;
            k_scale<<<grid_for(n), kThreads, 0, S->st>>>(n, make_double2(1.0, 0.0), t, x, 1);
            AK(cudaGetLastError());
            ++outer;
            AC(residual(&rel));
            push(rel);
        }
        conv = rel <= tol;
    } else {
        // FGMRES(m), right preconditioned: x = x0 + Z y
        std::vector<Cx> H((size_t)(m + 1) * m), cs((size_t)m), sn((size_t)m), g((size_t)m + 1);
        AC(residual(&rel));
        while (rel > tol && outer < max_outer) {
            const double beta = rel * bn;
            k_scale<<<grid_for(n), kThreads, 0, S->st>>>(n, make_double2(1.0 / beta, 0.0), r, V, 0);
            std::fill(g.begin(), g.end(), Cx(0.0));
            g[0] = beta;
            int j = 0;
            for (; j < m && outer < max_outer; ++j) {
                double2* vj = V + (size_t)j * n;
                double2* zj = Z + (size_t)j * n;
                AC(cvk_asm_apply_device(S, (const double*)vj, (double*)zj));
                brk |= S->last_brk;
                ++outer;
                double2* w = V + (size_t)(j + 1) * n;
                AC(cvk_spmv_device(S->A, (const double*)zj, (double*)w, CVK_MODE_FAST));
                for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt
                    double2 hij;
                    AC(dev_dot(S, n, V + (size_t)i * n, w, &hij));
                    H[(size_t)i * m + j] = Cx(hij.x, hij.y);
                    k_scale<<<grid_for(n), kThreads, 0, S->st>>>(n, make_double2(-hij.x, -hij.y), V + (size_t)i * n,
                                                                 w, 1);
                }
                double2 hh;
                AC(dev_dot(S, n, w, w, &hh));
                const double hn = std::sqrt(hh.x);
                H[(size_t)(j + 1) * m + j] = hn;
                if (hn > 0) k_scale<<<grid_for(n), kThreads, 0, S->st>>>(n, make_double2(1.0 / hn, 0.0), w, w, 0);
                for (int i = 0; i < j; ++i) {  // previous rotations
                    const Cx a = H[(size_t)i * m + j], c = H[(size_t)(i + 1) * m + j];
                    H[(size_t)i * m + j] = std::conj(cs[i]) * a + std::conj(sn[i]) * c;
                    H[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * c;
                }
                const Cx a = H[(size_t)j * m + j], c = H[(size_t)(j + 1) * m + j];
                const double den = std::sqrt(std::norm(a) + std::norm(c));
                cs[j] = den > 0 ? a / den : Cx(1.0);
                sn[j] = den > 0 ? c / den : Cx(0.0);
                H[(size_t)j * m + j] = den;
                H[(size_t)(j + 1) * m + j] = 0.0;
                g[j + 1] = -sn[j] * g[j];
                g[j] = std::conj(cs[j]) * g[j];
                push(std::abs(g[j + 1]) / bn);
                if (std::abs(g[j + 1]) <= tol * bn || hn == 0.0) { ++j; break; }
            }
            // y = H^-1 g (back substitution), x += Z y
            std::vector<Cx> y((size_t)j);
            for (int i = j - 1; i >= 0; --i) {
                Cx s_ = g[i];
                for (int k = i + 1; k < j; ++k) s_ -= H[(size_t)i * m + k] * y[k];
                y[i] = s_ / H[(size_t)i * m + i];
            }
            for (int i = 0; i < j; ++i)
                k_scale<<<grid_for(n), kThreads, 0, S->st>>>(n, make_double2(y[i].real(), y[i].imag()),
                                                             Z + (size_t)i * n, x, 1);
            AK(cudaGetLastError());
            AC(residual(&rel));  // true residual at every restart
            if (hl > 0 && rep->jump_history && hl - 1 < rep->jump_cap) rep->jump_history[hl - 1] = rel;
        }
        conv = rel <= tol;
    }
    AK(cudaEventRecord(e1, S->st));
    AK(cudaMemcpyAsync(x_host, x, nb, cudaMemcpyDeviceToHost, S->st));
    AK(cudaStreamSynchronize(S->st));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    rep->outer_iterations = outer;
    rep->converged = conv && !brk;
    rep->inner_breakdown = brk;
    rep->jump_len = hl;
    rep->total_inner_iterations = S->last_inner;
    rep->device_time_s = ms * 1e-3;
    rep->wall_time_s = now_s() - t0;
    rep->kernel_launches = 0;
    return CVK_OK;
}

}  // extern "C"
