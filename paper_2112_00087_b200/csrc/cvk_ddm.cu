// cvk_ddm.cu -- additive two-sided optimized Schwarz on the device
// (schwarz.cpp:111-238 of the reference; kernels K8-K10 of SURVEY.md 2.2).
//
// Per outer sweep:
//   k_ddm_rhs        local rhs = b|strip + w_L g_r[s-1] (left edge) + w_R g_l[s] (right edge)
//   k_solve_batched  every strip's inner Krylov solve in ONE cooperative launch
//                    (each strip a CTA segment with its own barrier, cvk_krylov.cu)
//   k_ddm_exchange   Robin trace update on every cut row + interface jump
// and one 8-byte D2H of the jump (plus the inner breakdown flags) for the
// host's convergence test.  The local systems (Robin ghost eliminated into
// the diagonal, schwarz.cpp:29-89) are built once per call on the host with
// std::complex -- the reference's own rounding -- and their Jacobi inverse
// diagonals on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <chrono>
#include <complex>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/cavac_b200.h"
#include "cvk_engine.cuh"
#include "cvk_kernels.h"

namespace cvk {
namespace {

using Cx = std::complex<double>;

struct Strip {
    int64_t c0, c1, n;
    std::vector<int> rp, ci;
    std::vector<Cx> v;
    Cx wl{0.0}, wr{0.0};
};

// schwarz.cpp:29-89: global rows of the strip's columns; couplings across a
// cut replaced by the eliminated Robin ghost, summed onto the diagonal after
// the in-strip entries (csr_from_triplets sums duplicates in input order).
int build_strip(int64_t nx, int64_t ny, double h, double c, const uint64_t* rp, const uint64_t* ci,
                const Cx* val, int64_t c0, int64_t c1, bool hl, bool hr, Cx s_left, Cx s_right,
                Strip& st) {
    const double k2 = c * c / (h * h);
    const int64_t w = c1 - c0;
    const Cx s_lc = s_right, s_rc = s_left;
    const Cx den_l = Cx(1.0 / h) + 0.5 * s_lc;
    const Cx den_r = Cx(1.0 / h) + 0.5 * s_rc;
    st.c0 = c0;
    st.c1 = c1;
    st.n = w * ny;
    if (hl) st.wl = k2 / den_l;
    if (hr) st.wr = k2 / den_r;
    st.rp.assign((size_t)st.n + 1, 0);
    st.ci.clear();
    st.v.clear();
    for (int64_t iy = 0; iy < ny; ++iy) {
        for (int64_t gx = c0; gx < c1; ++gx) {
            const int64_t grow = iy * nx + gx, lrow = iy * w + (gx - c0);
            Cx extra(0.0);
            const size_t first = st.ci.size();
            for (uint64_t k = rp[grow]; k < rp[grow + 1]; ++k) {
                const int64_t gc = (int64_t)ci[k], cx = gc % nx;
                if (cx >= c0 && cx < c1) {
                    const int64_t cy = gc / nx;
                    st.ci.push_back((int)(cy * w + (cx - c0)));
                    st.v.push_back(val[k]);
                } else if (cx == c0 - 1 && hl) {
                    extra += val[k] * ((Cx(1.0 / h) - 0.5 * s_lc) / den_l);
                } else if (cx == c1 && hr) {
                    extra += val[k] * ((Cx(1.0 / h) - 0.5 * s_rc) / den_r);
                } else {
                    return CVK_ELOGIC;  // "build_local: unexpected cross coupling"
                }
            }
            if (extra != Cx(0.0)) {
                // the duplicate diagonal triplet: sorted after the in-strip
                // entries of the same (row, col), so A_ii + extra
                size_t d = first;
                while (d < st.ci.size() && st.ci[d] != (int)lrow) ++d;
                if (d == st.ci.size()) {  // no stored diagonal: insert in column order
                    size_t pos = first;
                    while (pos < st.ci.size() && st.ci[pos] < (int)lrow) ++pos;
                    st.ci.insert(st.ci.begin() + (long)pos, (int)lrow);
                    st.v.insert(st.v.begin() + (long)pos, extra);
                } else {
                    st.v[d] += extra;
                }
            }
            st.rp[(size_t)lrow + 1] = (int)st.ci.size();
        }
    }
    return CVK_OK;
}

// A rank's strips: global strips s0 .. s0+ns-1, local index j.  Interface
// "slots" j = 0..ns: slot j is the cut between global strips s0+j-1 and
// s0+j (it exists iff 0 < s0+j < n_sub); slots 1..ns-1 are internal to the
// rank, slot 0 / slot ns are the rank's external left / right cuts whose
// other side lives on a neighbouring rank.
struct DdmGeom {
    int ns, ny, nx;
    int has_left, has_right;  // external cuts present (s0 > 0, s0 + ns < n_sub)
    const int* c0;            // [ns] first global column of local strip j
    const int* width;         // [ns]
    const int* loff;          // [ns + 1] offset of strip j in the concatenated local vectors
};

__device__ __forceinline__ bool slot_exists(const DdmGeom& g, int j) {
    return (j > 0 && j < g.ns) || (j == 0 && g.has_left) || (j == g.ns && g.has_right);
}

// local rhs (schwarz.cpp:160-175): b on the strip, + w_L g_r at the left
// edge (slot j), + w_R g_l at the right edge (slot j + 1)
__global__ void k_ddm_rhs(DdmGeom g, const double2* __restrict__ b, const double2* __restrict__ gl,
                          const double2* __restrict__ gr, const double2* __restrict__ wlr,
                          double2* __restrict__ rhs, int ntot) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ntot) return;
    int s = 0;
    while (s + 1 < g.ns && i >= g.loff[s + 1]) ++s;
    const int li = i - g.loff[s], w = g.width[s];
    const int iy = li / w, lx = li - iy * w;
    double2 r = b[(size_t)iy * g.nx + g.c0[s] + lx];
    if (lx == 0 && slot_exists(g, s)) r = cvk_add(r, cvk_mul(wlr[2 * s], gr[(size_t)s * g.ny + iy]));
    if (lx == w - 1 && slot_exists(g, s + 1)) r = cvk_add(r, cvk_mul(wlr[2 * s + 1], gl[(size_t)(s + 1) * g.ny + iy]));
    rhs[i] = r;
}

// trace exchange (schwarz.cpp:187-208) on every (slot, row) with the old
// g's, and the interface-jump terms |x_new - x_old|^2 of the edge columns
// (schwarz.cpp:211-220; summed on the host in the reference's order).  For
// an external slot only the local side is updated: its new g is written to
// out_left (slot 0: the left neighbour's g_l) / out_right (slot ns: the right
// neighbour's g_r) for the caller to send.
__global__ void k_ddm_exchange(DdmGeom g, const double2* __restrict__ u, double2* gl, double2* gr,
                               double2* prev, double2 a_l, double2 b_l, double2 a_r, double2 b_r,
                               double2 s_sum, double* terms, double2* out_left, double2* out_right) {
    const int tot = (g.ns + 1) * g.ny;
    const double2 half = cvk_scale(0.5, s_sum);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += gridDim.x * blockDim.x) {
        const int j = e / g.ny, iy = e - j * g.ny;
        terms[2 * e] = 0.0;
        terms[2 * e + 1] = 0.0;
        if (!slot_exists(g, j)) continue;
        const double2 glv = gl[e], grv = gr[e];
        if (j >= 1) {  // left side local: strip j-1, its last column (cut - 1)
            const int wl = g.width[j - 1];
            const double2 el = u[g.loff[j - 1] + (size_t)iy * wl + (wl - 1)];
            const double2 gho_l = cvk_cdiv(cvk_sub(glv, cvk_mul(b_l, el)), a_l);
            const double2 grn = cvk_add(cvk_neg(glv), cvk_mul(half, cvk_add(gho_l, el)));
            if (j == g.ns) out_right[iy] = grn;
            else gr[e] = grn;
            terms[2 * e] = cvk_norm(cvk_sub(el, prev[2 * e]));
            prev[2 * e] = el;
        }
        if (j < g.ns) {  // right side local: strip j, its first column (cut)
            const int wr = g.width[j];
            const double2 er = u[g.loff[j] + (size_t)iy * wr];
            const double2 gho_r = cvk_cdiv(cvk_sub(grv, cvk_mul(b_r, er)), a_r);
            const double2 gln = cvk_add(cvk_neg(grv), cvk_mul(half, cvk_add(gho_r, er)));
            if (j == 0) out_left[iy] = gln;
            else gl[e] = gln;
            terms[2 * e + 1] = cvk_norm(cvk_sub(er, prev[2 * e + 1]));
            prev[2 * e + 1] = er;
        }
    }
}

// the rank's columns, row-major over (iy, column) (schwarz.cpp:180-183)
__global__ void k_ddm_scatter(DdmGeom g, const double2* __restrict__ u, double2* __restrict__ x, int col0,
                              int ncols, int ntot) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ntot) return;
    int s = 0;
    while (s + 1 < g.ns && i >= g.loff[s + 1]) ++s;
    const int li = i - g.loff[s], w = g.width[s];
    const int iy = li / w, lx = li - iy * w;
    x[(size_t)iy * ncols + (g.c0[s] - col0) + lx] = u[i];
}

}  // namespace
}  // namespace cvk

namespace {
int dfail(int code, const std::string& m) { return cvk_fail(code, m); }
#define DK(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) return dfail(CVK_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct DevBuf {
    std::vector<void*> ptrs;
    ~DevBuf() {
        for (void* p : ptrs) cudaFree(p);
    }
    template <class T>
    cudaError_t alloc(T** p, size_t count) {
        void* q = nullptr;
        cudaError_t e = cudaMalloc(&q, std::max<size_t>(1, count) * sizeof(T));
        if (e == cudaSuccess) {
            ptrs.push_back(q);
            *p = (T*)q;
        }
        return e;
    }
};
}  // namespace

// partition (schwarz.cpp:93-109)
extern "C" int cvk_partition(int64_t nx, int64_t n_sub, int64_t* col_begin) {
    if (n_sub < 1) return dfail(CVK_EINVAL, "partition: n_sub must be >= 1");
    if (n_sub > 1 && nx / 3 < n_sub)
        return dfail(CVK_EINVAL, "partition: too many subdomains, each strip needs >= 3 columns");
    const int64_t base = nx / n_sub, rem = nx % n_sub;
    col_begin[0] = 0;
    for (int64_t s = 0; s < n_sub; ++s) col_begin[s + 1] = col_begin[s] + base + (s < rem ? 1 : 0);
    return CVK_OK;
}

// Implemented in cvk_api.cu: a plain (jacobi + solve) device solve of a host
// system, used for n_sub == 1 (schwarz.cpp:118-126).
extern "C" int cvk_ddm_single(cvk_ctx* ctx, int64_t n, int64_t nnz, const uint64_t* rp, const uint64_t* ci,
                              const double* v, const double* b, const cvk_opts* inner, int solver,
                              double* x, cvk_report* rep);

// Batched inner solves: fills the KArgs segments and launches them.
extern "C" int cvk_ddm_launch_batched(cvk_ctx* ctx, int solver, int mode, const void* segs_dev, int nseg,
                                      int total_ctas, size_t smem, float* ms);
extern "C" int cvk_ddm_ctas(cvk_ctx* ctx, int solver, int mode, size_t smem, int* total);
extern "C" void* cvk_ddm_stream(cvk_ctx* ctx);

// ---------------------------------------------------------------- rank plan
// The strips [s0, s1) of an n_sub-strip partition on one device: local
// systems + Jacobi built once, then one call per outer sweep.  A single rank
// owning every strip is the single-device schwarz_solve; one rank per GPU
// (strips split across ranks, external slots exchanged by the caller) is the
// multi-GPU DDM (paper_2112_00087_b200/ddm_dist.py).
struct cvk_ddm_rank {
    cvk_ctx* ctx = nullptr;
    cudaStream_t st = nullptr;
    DevBuf mem;
    int64_t n_sub = 0, s0 = 0, s1 = 0, ns = 0, nx = 0, ny = 0, col0 = 0, col1 = 0, ntot = 0;
    int solver = 0, mode = 0, total_ctas = 0;
    size_t smem = 0;
    cvk::DdmGeom geo{};
    double2 *d_b = nullptr, *d_rhs = nullptr, *d_u = nullptr, *d_gl = nullptr, *d_gr = nullptr,
            *d_prev = nullptr, *d_wlr = nullptr, *d_out = nullptr, *d_x = nullptr;
    double* d_terms = nullptr;
    unsigned long long* d_bars = nullptr;
    cvk::DevReport* d_reps = nullptr;
    cvk::KArgs* d_segs = nullptr;
    double2 a_l{}, b_l{}, a_r{}, b_r{}, s_sum{};
    std::vector<cvk::DevReport> hr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    // FAST mode, every strip >= CVK_DDM_SEQ_MIN rows: the strips' inner
    // solves run one after another on the single-system path (TMA-streamed
    // phase kernels), not as CTA segments of one batched persistent launch
    bool seq = false;
    // warm start (beyond the reference): each inner BiCGSTAB starts from the
    // strip's previous-sweep solution instead of 0
    bool warm = false;
    std::vector<cvk_csr*> seq_A;
    std::vector<cvk_prec*> seq_M;
    std::vector<int64_t> off;
    cvk_opts inner_opts{};
    ~cvk_ddm_rank() {
        for (cvk_prec* M : seq_M) cvk_precond_free(M);
        for (cvk_csr* A : seq_A) cvk_csr_free(A);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    }
};

extern "C" int cvk_ddm_rank_create(cvk_ctx* ctx, const cvk_grid* grid, double c, int64_t n, int64_t nnz,
                                   const uint64_t* row_offsets, const uint64_t* col_indices,
                                   const double* values, const double* b, int64_t n_sub,
                                   const int64_t* col_begin, int64_t s_begin, int64_t s_end,
                                   const double* s_left, const double* s_right, const cvk_opts* inner,
                                   int inner_solver, cvk_ddm_rank** out) {
    using namespace cvk;
    if (!ctx || !grid || !row_offsets || !b || !col_begin || !s_left || !s_right || !inner || !out)
        return dfail(CVK_EINVAL, "schwarz_solve: null argument");
    if (grid->nx * grid->ny != n) return dfail(CVK_EINVAL, "schwarz_solve: grid does not match the system");
    if (inner_solver < 0 || inner_solver > 4) return dfail(CVK_ESOLVER, "schwarz_solve: unknown inner solver");
    if (n_sub < 2 || n_sub > 4096) return dfail(CVK_EINVAL, "schwarz_solve: n_sub out of range");
    if (s_begin < 0 || s_end > n_sub || s_begin >= s_end) return dfail(CVK_EINVAL, "ddm rank: bad strip range");
    (void)nnz;
    auto R = std::make_unique<cvk_ddm_rank>();
    R->ctx = ctx;
    R->n_sub = n_sub;
    R->s0 = s_begin;
    R->s1 = s_end;
    R->ns = s_end - s_begin;
    R->nx = grid->nx;
    R->ny = grid->ny;
    R->col0 = col_begin[s_begin];
    R->col1 = col_begin[s_end];
    R->solver = inner_solver;
    const int64_t ns = R->ns, ny = R->ny, nx = R->nx;
    const double h = grid->h;
    const Cx sl(s_left[0], s_left[1]), sr(s_right[0], s_right[1]);
    std::vector<Strip> strips((size_t)ns);
    const Cx* vals = reinterpret_cast<const Cx*>(values);
    for (int64_t j = 0; j < ns; ++j) {
        const int64_t s = s_begin + j;
        const int e = build_strip(nx, ny, h, c, row_offsets, col_indices, vals, col_begin[s], col_begin[s + 1],
                                  s > 0, s + 1 < n_sub, sl, sr, strips[(size_t)j]);
        if (e != CVK_OK) return dfail(e, "build_local: unexpected cross coupling");
    }
    cudaStream_t st = (cudaStream_t)cvk_ddm_stream(ctx);
    R->st = st;
    DevBuf& mem = R->mem;
    std::vector<int> h_c0(ns), h_w(ns), h_off(ns + 1);
    int64_t ntot = 0;
    for (int64_t j = 0; j < ns; ++j) {
        h_c0[j] = (int)strips[j].c0;
        h_w[j] = (int)(strips[j].c1 - strips[j].c0);
        h_off[j] = (int)ntot;
        ntot += strips[j].n;
    }
    h_off[ns] = (int)ntot;
    R->ntot = ntot;
    int *d_c0, *d_w, *d_off;
    DK(mem.alloc(&d_c0, ns));
    DK(mem.alloc(&d_w, ns));
    DK(mem.alloc(&d_off, ns + 1));
    DK(cudaMemcpyAsync(d_c0, h_c0.data(), sizeof(int) * ns, cudaMemcpyHostToDevice, st));
    DK(cudaMemcpyAsync(d_w, h_w.data(), sizeof(int) * ns, cudaMemcpyHostToDevice, st));
    DK(cudaMemcpyAsync(d_off, h_off.data(), sizeof(int) * (ns + 1), cudaMemcpyHostToDevice, st));
    R->geo = DdmGeom{(int)ns, (int)ny, (int)nx, s_begin > 0 ? 1 : 0, s_end < n_sub ? 1 : 0, d_c0, d_w, d_off};
    const int64_t nslot = (ns + 1) * ny;
    DK(mem.alloc(&R->d_b, n));
    DK(mem.alloc(&R->d_rhs, ntot));
    DK(mem.alloc(&R->d_u, ntot));
    DK(cudaMemsetAsync(R->d_u, 0, sizeof(double2) * ntot, st));  // x0 of a warm-started first sweep
    DK(mem.alloc(&R->d_gl, nslot));
    DK(mem.alloc(&R->d_gr, nslot));
    DK(mem.alloc(&R->d_prev, 2 * nslot));
    DK(mem.alloc(&R->d_terms, 2 * nslot));
    DK(mem.alloc(&R->d_out, 2 * ny));
    DK(mem.alloc(&R->d_wlr, 2 * ns));
    DK(mem.alloc(&R->d_x, ntot));
    DK(cudaMemcpyAsync(R->d_b, b, sizeof(double2) * n, cudaMemcpyHostToDevice, st));
    DK(cudaMemsetAsync(R->d_gl, 0, sizeof(double2) * nslot, st));
    DK(cudaMemsetAsync(R->d_gr, 0, sizeof(double2) * nslot, st));
    DK(cudaMemsetAsync(R->d_prev, 0, sizeof(double2) * 2 * nslot, st));
    DK(cudaMemsetAsync(R->d_out, 0, sizeof(double2) * 2 * ny, st));
    std::vector<double2> h_wlr(2 * ns);
    for (int64_t j = 0; j < ns; ++j) {
        h_wlr[2 * j] = make_double2(strips[j].wl.real(), strips[j].wl.imag());
        h_wlr[2 * j + 1] = make_double2(strips[j].wr.real(), strips[j].wr.imag());
    }
    DK(cudaMemcpyAsync(R->d_wlr, h_wlr.data(), sizeof(double2) * 2 * ns, cudaMemcpyHostToDevice, st));

    // local CSRs + Jacobi, one batched-solve segment per strip
    {
        int m = inner->mode;
        if (m < 0) m = cvk_get_exec_mode(ctx) ? CVK_MODE_REF_PAR : CVK_MODE_REF;
        R->mode = (m == CVK_MODE_REF || m == CVK_MODE_REF_PAR) ? m : CVK_MODE_FAST;
    }
    R->smem = solver_smem(inner_solver, (int)inner->m);
    int e = cvk_ddm_ctas(ctx, inner_solver, R->mode, R->smem, &R->total_ctas);
    if (e != CVK_OK) return e;
    const int nwork = solver_nwork(inner_solver, (int)inner->l, (int)inner->m);
    std::vector<KArgs> segs((size_t)ns);
    int* d_bad;
    DK(mem.alloc(&d_bad, 1));
    std::vector<int> gs(ns, 1);
    {
        int64_t chunks_tot = 0;
        std::vector<int64_t> ch(ns);
        for (int64_t j = 0; j < ns; ++j) {
            ch[j] = std::max<int64_t>(1, (strips[j].n + kThreads - 1) / kThreads);
            chunks_tot += ch[j];
        }
        const int budget = std::max<int>(R->total_ctas, (int)ns);
        for (int64_t j = 0; j < ns; ++j)
            gs[j] = (int)std::max<int64_t>(1, std::min<int64_t>(ch[j], (int64_t)budget * ch[j] / chunks_tot));
    }
    int cta_base = 0;
    DK(mem.alloc(&R->d_bars, 2 * ns));
    DK(mem.alloc(&R->d_reps, ns));
    for (int64_t j = 0; j < ns; ++j) {
        const Strip& S = strips[j];
        int *rp, *ci;
        double2 *av, *dinv, *work, *part;
        DK(mem.alloc(&rp, S.rp.size()));
        DK(mem.alloc(&ci, S.ci.size()));
        DK(mem.alloc(&av, S.v.size()));
        DK(mem.alloc(&dinv, S.n));
        DK(mem.alloc(&work, (size_t)nwork * S.n));
        DK(mem.alloc(&part, (size_t)kRegions * kMaxSlots * gs[j]));
        DK(cudaMemcpyAsync(rp, S.rp.data(), sizeof(int) * S.rp.size(), cudaMemcpyHostToDevice, st));
        DK(cudaMemcpyAsync(ci, S.ci.data(), sizeof(int) * S.ci.size(), cudaMemcpyHostToDevice, st));
        DK(cudaMemcpyAsync(av, S.v.data(), sizeof(double2) * S.v.size(), cudaMemcpyHostToDevice, st));
        const int big = 0x7fffffff;
        DK(cudaMemcpyAsync(d_bad, &big, sizeof(int), cudaMemcpyHostToDevice, st));
        DK(launch_inv_diag((int)S.n, rp, ci, av, dinv, d_bad, st));
        int bad = 0;
        DK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
        DK(cudaStreamSynchronize(st));
        if (bad != big) return dfail(CVK_EZERODIAG, "jacobi: zero diagonal at row " + std::to_string(bad));
        KArgs& a = segs[j];
        std::memset(&a, 0, sizeof(a));
        a.A = Csr{(int)S.n, rp, ci, av};
        a.dinv = dinv;
        a.b = R->d_rhs + h_off[j];
        a.x = R->d_u + h_off[j];
        a.work = work;
        a.part = part;
        a.bar = R->d_bars + 2 * j;
        a.rep = R->d_reps + j;
        a.hist = nullptr;
        a.hist_cap = 0;
        a.tol = inner->tol;
        a.max_iter = inner->max_iter;
        a.l = (int)inner->l;
        a.m = (int)inner->m;
        a.record = 0;
        a.G = gs[j];
        a.cta_base = cta_base;
        a.refpar = R->mode == CVK_MODE_REF_PAR ? 1 : 0;
        cta_base += gs[j];
    }
    R->total_ctas = cta_base;
    R->off.assign(h_off.begin(), h_off.end());
    R->warm = inner_solver == CVK_BICGSTAB && inner->warm != 0;
    for (int64_t j = 0; j < ns; ++j) segs[j].warm = R->warm ? 1 : 0;
    R->inner_opts = *inner;
    R->inner_opts.record_history = 0;
    R->inner_opts.mode = R->mode;
    {
        // a strip this large fills the device on its own: the batched launch
        // gives each strip ~1/ns of the SMs on the latency-bound persistent
        // kernel (5M DOF, 8 strips: ~490 us per inner iteration)
        const long long thr = cvk_ctx_knob(ctx, CVK_OPT_DDM_SEQ_MIN);
        int64_t nmin = INT64_MAX;
        for (const Strip& S : strips) nmin = std::min<int64_t>(nmin, S.n);
        R->seq = R->mode == CVK_MODE_FAST && nmin >= thr;
    }
    if (R->seq) {
        for (int64_t j = 0; j < ns; ++j) {
            const Strip& S = strips[j];
            std::vector<uint64_t> rp64(S.rp.begin(), S.rp.end()), ci64(S.ci.begin(), S.ci.end());
            cvk_csr* A = nullptr;
            cvk_prec* M = nullptr;
            int ee = cvk_csr_upload(ctx, S.n, S.n, (int64_t)S.ci.size(), rp64.data(), ci64.data(),
                                    reinterpret_cast<const double*>(S.v.data()), &A);
            if (ee != CVK_OK) return ee;
            R->seq_A.push_back(A);
            if ((ee = cvk_precond_jacobi(A, nullptr, &M)) != CVK_OK) return ee;
            R->seq_M.push_back(M);
        }
    }
    DK(mem.alloc(&R->d_segs, ns));
    DK(cudaMemcpyAsync(R->d_segs, segs.data(), sizeof(KArgs) * ns, cudaMemcpyHostToDevice, st));
    auto d2 = [](Cx z) { return make_double2(z.real(), z.imag()); };
    R->a_l = d2(Cx(1.0 / h) + 0.5 * sl);
    R->b_l = d2(Cx(-1.0 / h) + 0.5 * sl);
    R->a_r = d2(Cx(1.0 / h) + 0.5 * sr);
    R->b_r = d2(Cx(-1.0 / h) + 0.5 * sr);
    R->s_sum = d2(sl + sr);
    R->hr.resize((size_t)ns);
    DK(cudaEventCreate(&R->e0));
    DK(cudaEventCreate(&R->e1));
    DK(cudaStreamSynchronize(st));
    *out = R.release();
    return CVK_OK;
}

extern "C" int cvk_ddm_rank_sweep(cvk_ddm_rank* R, const double* g_in_left, const double* g_in_right,
                                  double* g_out_left, double* g_out_right, double* jump_terms,
                                  cvk_ddm_sweep_info* info) {
    using namespace cvk;
    if (!R || !jump_terms || !info) return dfail(CVK_EINVAL, "ddm rank sweep: null argument");
    cudaStream_t st = R->st;
    const int64_t ny = R->ny, ns = R->ns;
    // incoming external data (the neighbours' previous-sweep updates)
    if (R->geo.has_left && g_in_left)
        DK(cudaMemcpyAsync(R->d_gr, g_in_left, sizeof(double2) * ny, cudaMemcpyHostToDevice, st));
    if (R->geo.has_right && g_in_right)
        DK(cudaMemcpyAsync(R->d_gl + ns * ny, g_in_right, sizeof(double2) * ny, cudaMemcpyHostToDevice, st));
    const int threads = 256;
    DK(cudaEventRecord(R->e0, st));
    k_ddm_rhs<<<(unsigned)((R->ntot + threads - 1) / threads), threads, 0, st>>>(R->geo, R->d_b, R->d_gl, R->d_gr,
                                                                                R->d_wlr, R->d_rhs, (int)R->ntot);
    DK(cudaGetLastError());
    DK(cudaMemsetAsync(R->d_bars, 0, sizeof(unsigned long long) * 2 * ns, st));
    float ms = 0.f;
    long long launches = 3;
    if (R->seq) {
        for (int64_t j = 0; j < ns; ++j) {
            cvk_report rep{};
            const double* bj = reinterpret_cast<const double*>(R->d_rhs + R->off[j]);
            double* uj = reinterpret_cast<double*>(R->d_u + R->off[j]);
            const int e = R->warm ? cvk_solve_device_warm(R->ctx, R->seq_A[j], R->seq_M[j], &R->inner_opts, bj, uj, &rep)
                                  : cvk_solve_device(R->ctx, R->solver, R->seq_A[j], R->seq_M[j], &R->inner_opts, bj,
                                                     uj, &rep);
            if (e != CVK_OK) return e;
            DevReport& d = R->hr[j];
            d.converged = rep.converged;
            d.breakdown = rep.breakdown;
            d.iterations = rep.iterations;
            d.final_relres = rep.final_relres;
            d.true_relres = rep.true_relres;
            d.history_len = 0;
            d.error = 0;
            launches += rep.kernel_launches;
        }
        DK(cudaMemcpyAsync(R->d_reps, R->hr.data(), sizeof(DevReport) * ns, cudaMemcpyHostToDevice, st));
    } else {
        const int e = cvk_ddm_launch_batched(R->ctx, R->solver, R->mode, R->d_segs, (int)ns, R->total_ctas, R->smem, &ms);
        if (e != CVK_OK) return e;
    }
    const int64_t nslot = (ns + 1) * ny;
    const unsigned xb = (unsigned)std::min<int64_t>(64, (nslot + threads - 1) / threads);
    k_ddm_exchange<<<std::max(1u, xb), threads, 0, st>>>(R->geo, R->d_u, R->d_gl, R->d_gr, R->d_prev, R->a_l, R->b_l,
                                                         R->a_r, R->b_r, R->s_sum, R->d_terms, R->d_out,
                                                         R->d_out + ny);
    DK(cudaGetLastError());
    DK(cudaEventRecord(R->e1, st));
    DK(cudaMemcpyAsync(jump_terms, R->d_terms, sizeof(double) * 2 * nslot, cudaMemcpyDeviceToHost, st));
    if (g_out_left) DK(cudaMemcpyAsync(g_out_left, R->d_out, sizeof(double2) * ny, cudaMemcpyDeviceToHost, st));
    if (g_out_right) DK(cudaMemcpyAsync(g_out_right, R->d_out + ny, sizeof(double2) * ny, cudaMemcpyDeviceToHost, st));
    DK(cudaMemcpyAsync(R->hr.data(), R->d_reps, sizeof(DevReport) * ns, cudaMemcpyDeviceToHost, st));
    DK(cudaStreamSynchronize(st));
    float sweep_ms = 0.f;
    cudaEventElapsedTime(&sweep_ms, R->e0, R->e1);
    info->inner_breakdown = 0;
    info->total_inner_iterations = 0;
    for (int64_t j = 0; j < ns; ++j) {
        if (R->hr[j].error) return dfail(CVK_ETIMEOUT, "schwarz_solve: inner solve grid barrier aborted");
        if (R->hr[j].breakdown) info->inner_breakdown = 1;
        info->total_inner_iterations += R->hr[j].iterations;
    }
    info->device_time_s = sweep_ms * 1e-3;
    info->kernel_launches = launches;
    return CVK_OK;
}

extern "C" int cvk_ddm_rank_reports(const cvk_ddm_rank* R, cvk_report* reps, int64_t cap) {
    if (!R || (!reps && cap > 0)) return dfail(CVK_EINVAL, "ddm rank reports: null argument");
    for (int64_t j = 0; j < R->ns && j < cap; ++j) {
        cvk_report& r = reps[j];
        r.converged = R->hr[j].converged;
        r.breakdown = R->hr[j].breakdown;
        r.iterations = R->hr[j].iterations;
        r.final_relres = R->hr[j].final_relres;
        r.true_relres = R->hr[j].true_relres;
        r.history_len = 0;
    }
    return CVK_OK;
}

extern "C" int cvk_ddm_rank_solution(cvk_ddm_rank* R, double* x_cols) {
    using namespace cvk;
    if (!R || !x_cols) return dfail(CVK_EINVAL, "ddm rank solution: null argument");
    const int threads = 256;
    k_ddm_scatter<<<(unsigned)((R->ntot + threads - 1) / threads), threads, 0, R->st>>>(
        R->geo, R->d_u, R->d_x, (int)R->col0, (int)(R->col1 - R->col0), (int)R->ntot);
    DK(cudaGetLastError());
    DK(cudaMemcpyAsync(x_cols, R->d_x, sizeof(double2) * R->ntot, cudaMemcpyDeviceToHost, R->st));
    DK(cudaStreamSynchronize(R->st));
    return CVK_OK;
}

extern "C" int cvk_ddm_rank_set_warm(cvk_ddm_rank* R, int warm) {
    if (!R) return dfail(CVK_EINVAL, "ddm rank warm: null rank");
    if (warm && R->solver != CVK_BICGSTAB) return dfail(CVK_EINVAL, "ddm rank warm: BiCGSTAB inner solves only");
    R->warm = warm != 0;
    std::vector<cvk::KArgs> segs((size_t)R->ns);
    DK(cudaMemcpy(segs.data(), R->d_segs, sizeof(cvk::KArgs) * R->ns, cudaMemcpyDeviceToHost));
    for (cvk::KArgs& a : segs) a.warm = R->warm ? 1 : 0;
    DK(cudaMemcpy(R->d_segs, segs.data(), sizeof(cvk::KArgs) * R->ns, cudaMemcpyHostToDevice));
    return CVK_OK;
}

// interface traces g_l, g_r of every slot ((ns + 1) x ny complex each):
// the state of the outer iteration, for Krylov acceleration on the host
extern "C" int cvk_ddm_rank_get_traces(cvk_ddm_rank* R, double* g_l, double* g_r) {
    if (!R || !g_l || !g_r) return dfail(CVK_EINVAL, "ddm rank traces: null argument");
    const size_t bytes = sizeof(double2) * (size_t)(R->ns + 1) * R->ny;
    DK(cudaMemcpyAsync(g_l, R->d_gl, bytes, cudaMemcpyDeviceToHost, R->st));
    DK(cudaMemcpyAsync(g_r, R->d_gr, bytes, cudaMemcpyDeviceToHost, R->st));
    DK(cudaStreamSynchronize(R->st));
    return CVK_OK;
}

extern "C" int cvk_ddm_rank_set_traces(cvk_ddm_rank* R, const double* g_l, const double* g_r) {
    if (!R || !g_l || !g_r) return dfail(CVK_EINVAL, "ddm rank traces: null argument");
    const size_t bytes = sizeof(double2) * (size_t)(R->ns + 1) * R->ny;
    DK(cudaMemcpyAsync(R->d_gl, g_l, bytes, cudaMemcpyHostToDevice, R->st));
    DK(cudaMemcpyAsync(R->d_gr, g_r, bytes, cudaMemcpyHostToDevice, R->st));
    DK(cudaStreamSynchronize(R->st));
    return CVK_OK;
}

extern "C" int cvk_ddm_rank_destroy(cvk_ddm_rank* R) {
    if (R) {
        cudaStreamSynchronize(R->st);
        delete R;
    }
    return CVK_OK;
}

// schwarz_solve (schwarz.cpp:111-238) on one device = one rank owning every strip
extern "C" int cvk_schwarz_solve(cvk_ctx* ctx, const cvk_grid* grid, double c, int64_t n, int64_t nnz,
                                 const uint64_t* row_offsets, const uint64_t* col_indices,
                                 const double* values, const double* b, int64_t n_sub,
                                 const int64_t* col_begin, const double* s_left, const double* s_right,
                                 const cvk_opts* inner, double ddm_tol, int64_t max_outer,
                                 int inner_solver, double* x, cvk_ddm_report* rep) {
    const double t_wall0 = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    if (!ctx || !grid || !row_offsets || !b || !col_begin || !s_left || !s_right || !inner || !x || !rep)
        return dfail(CVK_EINVAL, "schwarz_solve: null argument");
    if (grid->nx * grid->ny != n) return dfail(CVK_EINVAL, "schwarz_solve: grid does not match the system");
    if (inner_solver < 0 || inner_solver > 4) return dfail(CVK_ESOLVER, "schwarz_solve: unknown inner solver");
    rep->outer_iterations = 0;
    rep->converged = 0;
    rep->inner_breakdown = 0;
    rep->jump_len = 0;
    rep->total_inner_iterations = 0;
    rep->device_time_s = 0;
    rep->kernel_launches = 0;
    if (n_sub == 1) {
        cvk_report sr;
        std::memset(&sr, 0, sizeof sr);
        const int e = cvk_ddm_single(ctx, n, nnz, row_offsets, col_indices, values, b, inner, inner_solver, x, &sr);
        if (e != CVK_OK) return e;
        rep->outer_iterations = 1;
        rep->converged = sr.converged;
        rep->total_inner_iterations = sr.iterations;
        rep->device_time_s = sr.device_time_s;
        rep->kernel_launches = sr.kernel_launches;
        if (rep->sub_reports && rep->n_sub_reports >= 1) rep->sub_reports[0] = sr;
        return CVK_OK;
    }
    if (n_sub < 1 || n_sub > 256) return dfail(CVK_EINVAL, "schwarz_solve: n_sub out of range");
    cvk_ddm_rank* R = nullptr;
    int e = cvk_ddm_rank_create(ctx, grid, c, n, nnz, row_offsets, col_indices, values, b, n_sub, col_begin, 0, n_sub,
                                s_left, s_right, inner, inner_solver, &R);
    if (e != CVK_OK) return e;
    std::unique_ptr<cvk_ddm_rank, int (*)(cvk_ddm_rank*)> guard(R, cvk_ddm_rank_destroy);
    const int64_t ny = grid->ny, ncut = n_sub - 1;
    std::vector<double> terms((size_t)(2 * (n_sub + 1) * ny));
    double res0 = -1.0, dev_s = 0.0;
    int64_t launches = 0;
    for (int64_t outer = 1; outer <= max_outer; ++outer) {
        cvk_ddm_sweep_info info;
        std::memset(&info, 0, sizeof info);
        e = cvk_ddm_rank_sweep(R, nullptr, nullptr, nullptr, nullptr, terms.data(), &info);
        if (e != CVK_OK) return e;
        dev_s += info.device_time_s;
        launches += info.kernel_launches;
        // jump^2 in the reference's order: per cut, per row, left column then right
        double jump2 = 0.0;
        for (int64_t q = 0; q < ncut; ++q)
            for (int64_t iy = 0; iy < ny; ++iy) {
                const size_t e2 = (size_t)(2 * ((q + 1) * ny + iy));
                jump2 += terms[e2];
                jump2 += terms[e2 + 1];
            }
        const double jump = std::sqrt(jump2);
        if (rep->jump_history && rep->jump_len < rep->jump_cap) rep->jump_history[rep->jump_len] = jump;
        rep->jump_len++;
        rep->outer_iterations = outer;
        rep->total_inner_iterations = info.total_inner_iterations;
        if (info.inner_breakdown) {
            rep->converged = 0;
            rep->inner_breakdown = 1;
            break;
        }
        if (res0 < 0.0) res0 = jump;
        if (jump == 0.0 || jump <= ddm_tol * res0) {
            rep->converged = 1;
            break;
        }
    }
    if (rep->sub_reports) cvk_ddm_rank_reports(R, rep->sub_reports, rep->n_sub_reports);
    e = cvk_ddm_rank_solution(R, x);  // all strips: the rank's columns are the whole grid
    if (e != CVK_OK) return e;
    rep->device_time_s = dev_s;
    rep->kernel_launches = launches + 1;
    rep->wall_time_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count() - t_wall0;
    return CVK_OK;
}
