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
#include <chrono>
#include <complex>
#include <cstring>
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

struct DdmGeom {
    int n_sub, ny, nx;
    const int* c0;       // [n_sub]
    const int* width;    // [n_sub]
    const int* loff;     // [n_sub] offset of strip s in the concatenated local vectors
};

// local rhs (schwarz.cpp:160-175)
__global__ void k_ddm_rhs(DdmGeom g, const double2* __restrict__ b, const double2* __restrict__ gl,
                          const double2* __restrict__ gr, const double2* __restrict__ wlr,
                          double2* __restrict__ rhs, int ntot) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ntot) return;
    int s = 0;
    while (s + 1 < g.n_sub && i >= g.loff[s + 1]) ++s;
    const int li = i - g.loff[s], w = g.width[s];
    const int iy = li / w, lx = li - iy * w;
    double2 r = b[(size_t)iy * g.nx + g.c0[s] + lx];
    if (s > 0 && lx == 0) r = cvk_add(r, cvk_mul(wlr[2 * s], gr[(size_t)(s - 1) * g.ny + iy]));
    if (s + 1 < g.n_sub && lx == w - 1) r = cvk_add(r, cvk_mul(wlr[2 * s + 1], gl[(size_t)s * g.ny + iy]));
    rhs[i] = r;
}

// trace exchange (schwarz.cpp:187-208) on every (cut, row); then the jump
// (schwarz.cpp:211-220) summed by one thread in the reference's order.
__global__ void k_ddm_exchange(DdmGeom g, const double2* __restrict__ u, double2* gl, double2* gr,
                               double2* prev, double2 a_l, double2 b_l, double2 a_r, double2 b_r,
                               double2 s_sum, double* jump2_out) {
    const int ncut = g.n_sub - 1;
    const int tot = ncut * g.ny;
    extern __shared__ double2 dj[];  // per (cut,row): d_left, d_right
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int q = e / g.ny, iy = e - q * g.ny;
        const int wl = g.width[q], wr = g.width[q + 1];
        const double2 el = u[g.loff[q] + (size_t)iy * wl + (wl - 1)];
        const double2 er = u[g.loff[q + 1] + (size_t)iy * wr];
        const double2 glv = gl[e], grv = gr[e];
        const double2 gho_l = cvk_cdiv(cvk_sub(glv, cvk_mul(b_l, el)), a_l);
        const double2 gho_r = cvk_cdiv(cvk_sub(grv, cvk_mul(b_r, er)), a_r);
        const double2 half = cvk_scale(0.5, s_sum);
        gr[e] = cvk_add(cvk_neg(glv), cvk_mul(half, cvk_add(gho_l, el)));
        gl[e] = cvk_add(cvk_neg(grv), cvk_mul(half, cvk_add(gho_r, er)));
        dj[2 * e] = cvk_sub(el, prev[2 * e]);
        dj[2 * e + 1] = cvk_sub(er, prev[2 * e + 1]);
        prev[2 * e] = el;
        prev[2 * e + 1] = er;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double j2 = 0.0;
        for (int e = 0; e < 2 * tot; ++e) j2 += cvk_norm(dj[e]);
        *jump2_out = j2;
    }
}

// x[global] = u_loc (schwarz.cpp:180-183, last sweep)
__global__ void k_ddm_scatter(DdmGeom g, const double2* __restrict__ u, double2* __restrict__ x, int ntot) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ntot) return;
    int s = 0;
    while (s + 1 < g.n_sub && i >= g.loff[s + 1]) ++s;
    const int li = i - g.loff[s], w = g.width[s];
    const int iy = li / w, lx = li - iy * w;
    x[(size_t)iy * g.nx + g.c0[s] + lx] = u[i];
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

extern "C" int cvk_schwarz_solve(cvk_ctx* ctx, const cvk_grid* grid, double c, int64_t n, int64_t nnz,
                                 const uint64_t* row_offsets, const uint64_t* col_indices,
                                 const double* values, const double* b, int64_t n_sub,
                                 const int64_t* col_begin, const double* s_left, const double* s_right,
                                 const cvk_opts* inner, double ddm_tol, int64_t max_outer,
                                 int inner_solver, double* x, cvk_ddm_report* rep) {
    using namespace cvk;
    const double t_wall0 = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    if (!ctx || !grid || !row_offsets || !b || !col_begin || !s_left || !s_right || !inner || !x || !rep)
        return dfail(CVK_EINVAL, "schwarz_solve: null argument");
    if (grid->nx * grid->ny != n) return dfail(CVK_EINVAL, "schwarz_solve: grid does not match the system");
    if (inner_solver < 0 || inner_solver > 3) return dfail(CVK_ESOLVER, "schwarz_solve: unknown inner solver");
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
    const int64_t nx = grid->nx, ny = grid->ny;
    const double h = grid->h;
    const Cx sl(s_left[0], s_left[1]), sr(s_right[0], s_right[1]);
    std::vector<Strip> strips((size_t)n_sub);
    const Cx* vals = reinterpret_cast<const Cx*>(values);
    for (int64_t s = 0; s < n_sub; ++s) {
        const int e = build_strip(nx, ny, h, c, row_offsets, col_indices, vals, col_begin[s], col_begin[s + 1],
                                  s > 0, s + 1 < n_sub, sl, sr, strips[(size_t)s]);
        if (e != CVK_OK) return dfail(e, "build_local: unexpected cross coupling");
    }
    // ---------------- device state
    cudaStream_t st = (cudaStream_t)cvk_ddm_stream(ctx);
    DevBuf mem;
    std::vector<int> h_c0(n_sub), h_w(n_sub), h_off(n_sub + 1);
    int64_t ntot = 0;
    for (int64_t s = 0; s < n_sub; ++s) {
        h_c0[s] = (int)strips[s].c0;
        h_w[s] = (int)(strips[s].c1 - strips[s].c0);
        h_off[s] = (int)ntot;
        ntot += strips[s].n;
    }
    h_off[n_sub] = (int)ntot;
    int *d_c0, *d_w, *d_off;
    DK(mem.alloc(&d_c0, n_sub));
    DK(mem.alloc(&d_w, n_sub));
    DK(mem.alloc(&d_off, n_sub + 1));
    DK(cudaMemcpyAsync(d_c0, h_c0.data(), sizeof(int) * n_sub, cudaMemcpyHostToDevice, st));
    DK(cudaMemcpyAsync(d_w, h_w.data(), sizeof(int) * n_sub, cudaMemcpyHostToDevice, st));
    DK(cudaMemcpyAsync(d_off, h_off.data(), sizeof(int) * (n_sub + 1), cudaMemcpyHostToDevice, st));
    DdmGeom geo{(int)n_sub, (int)ny, (int)nx, d_c0, d_w, d_off};
    double2 *d_b, *d_rhs, *d_u, *d_gl, *d_gr, *d_prev, *d_wlr, *d_x;
    double* d_jump;
    DK(mem.alloc(&d_b, n));
    DK(mem.alloc(&d_rhs, ntot));
    DK(mem.alloc(&d_u, ntot));
    DK(mem.alloc(&d_gl, (n_sub - 1) * ny));
    DK(mem.alloc(&d_gr, (n_sub - 1) * ny));
    DK(mem.alloc(&d_prev, 2 * (n_sub - 1) * ny));
    DK(mem.alloc(&d_wlr, 2 * n_sub));
    DK(mem.alloc(&d_x, n));
    DK(mem.alloc(&d_jump, 1));
    DK(cudaMemcpyAsync(d_b, b, sizeof(double2) * n, cudaMemcpyHostToDevice, st));
    DK(cudaMemsetAsync(d_gl, 0, sizeof(double2) * (n_sub - 1) * ny, st));
    DK(cudaMemsetAsync(d_gr, 0, sizeof(double2) * (n_sub - 1) * ny, st));
    DK(cudaMemsetAsync(d_prev, 0, sizeof(double2) * 2 * (n_sub - 1) * ny, st));
    std::vector<double2> h_wlr(2 * n_sub);
    for (int64_t s = 0; s < n_sub; ++s) {
        h_wlr[2 * s] = make_double2(strips[s].wl.real(), strips[s].wl.imag());
        h_wlr[2 * s + 1] = make_double2(strips[s].wr.real(), strips[s].wr.imag());
    }
    DK(cudaMemcpyAsync(d_wlr, h_wlr.data(), sizeof(double2) * 2 * n_sub, cudaMemcpyHostToDevice, st));

    // local CSRs + Jacobi
    const int mode = inner->mode == CVK_MODE_REF ? CVK_MODE_REF : CVK_MODE_FAST;
    const size_t smem = solver_smem(inner_solver, (int)inner->m);
    int total_ctas = 0;
    int e = cvk_ddm_ctas(ctx, inner_solver, mode, smem, &total_ctas);
    if (e != CVK_OK) return e;
    const int nwork = solver_nwork(inner_solver, (int)inner->l, (int)inner->m);
    std::vector<KArgs> segs((size_t)n_sub);
    int* d_bad;
    DK(mem.alloc(&d_bad, 1));
    // CTAs per strip proportional to its chunks, at least 1
    std::vector<int> gs(n_sub, 1);
    {
        int64_t chunks_tot = 0;
        std::vector<int64_t> ch(n_sub);
        for (int64_t s = 0; s < n_sub; ++s) {
            ch[s] = std::max<int64_t>(1, (strips[s].n + kThreads - 1) / kThreads);
            chunks_tot += ch[s];
        }
        int budget = std::max<int>(total_ctas, (int)n_sub);
        for (int64_t s = 0; s < n_sub; ++s)
            gs[s] = (int)std::max<int64_t>(1, std::min<int64_t>(ch[s], (int64_t)budget * ch[s] / chunks_tot));
    }
    int cta_base = 0;
    unsigned long long* d_bars;
    DevReport* d_reps;
    DK(mem.alloc(&d_bars, 2 * n_sub));
    DK(mem.alloc(&d_reps, n_sub));
    for (int64_t s = 0; s < n_sub; ++s) {
        const Strip& S = strips[s];
        int *rp, *ci;
        double2 *av, *dinv, *work, *part;
        DK(mem.alloc(&rp, S.rp.size()));
        DK(mem.alloc(&ci, S.ci.size()));
        DK(mem.alloc(&av, S.v.size()));
        DK(mem.alloc(&dinv, S.n));
        DK(mem.alloc(&work, (size_t)nwork * S.n));
        DK(mem.alloc(&part, (size_t)kRegions * kMaxSlots * gs[s]));
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
        KArgs& a = segs[s];
        std::memset(&a, 0, sizeof(a));
        a.A = Csr{(int)S.n, rp, ci, av};
        a.dinv = dinv;
        a.b = d_rhs + h_off[s];
        a.x = d_u + h_off[s];
        a.work = work;
        a.part = part;
        a.bar = d_bars + 2 * s;
        a.rep = d_reps + s;
        a.hist = nullptr;
        a.hist_cap = 0;
        a.tol = inner->tol;
        a.max_iter = inner->max_iter;
        a.l = (int)inner->l;
        a.m = (int)inner->m;
        a.record = 0;
        a.G = gs[s];
        a.cta_base = cta_base;
        cta_base += gs[s];
    }
    KArgs* d_segs;
    DK(mem.alloc(&d_segs, n_sub));
    DK(cudaMemcpyAsync(d_segs, segs.data(), sizeof(KArgs) * n_sub, cudaMemcpyHostToDevice, st));

    const Cx a_l = Cx(1.0 / h) + 0.5 * sl, b_l = Cx(-1.0 / h) + 0.5 * sl;
    const Cx a_r = Cx(1.0 / h) + 0.5 * sr, b_r = Cx(-1.0 / h) + 0.5 * sr;
    const Cx s_sum = sl + sr;
    auto d2 = [](Cx z) { return make_double2(z.real(), z.imag()); };
    const int ncut = (int)n_sub - 1;
    const int threads = 256;
    const size_t xsmem = sizeof(double2) * 2 * (size_t)ncut * ny;
    if (xsmem > 200 * 1024) return dfail(CVK_EINVAL, "schwarz_solve: interface too large for the exchange kernel");
    if (xsmem > 48 * 1024) DK(cudaFuncSetAttribute(k_ddm_exchange, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsmem));
    double res0 = -1.0;
    float dev_ms = 0.f;
    int64_t launches = 0;
    std::vector<DevReport> hr((size_t)n_sub);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int64_t outer = 1; outer <= max_outer; ++outer) {
        DK(cudaEventRecord(e0, st));
        k_ddm_rhs<<<(unsigned)((ntot + threads - 1) / threads), threads, 0, st>>>(geo, d_b, d_gl, d_gr, d_wlr, d_rhs, (int)ntot);
        DK(cudaGetLastError());
        DK(cudaMemsetAsync(d_bars, 0, sizeof(unsigned long long) * 2 * n_sub, st));
        float ms = 0.f;
        e = cvk_ddm_launch_batched(ctx, inner_solver, mode, d_segs, (int)n_sub, cta_base, smem, &ms);
        if (e != CVK_OK) return e;
        k_ddm_exchange<<<1, 256, xsmem, st>>>(geo, d_u, d_gl, d_gr, d_prev, d2(a_l), d2(b_l), d2(a_r), d2(b_r),
                                              d2(s_sum), d_jump);
        DK(cudaGetLastError());
        DK(cudaEventRecord(e1, st));
        launches += 3;
        double jump2 = 0.0;
        DK(cudaMemcpyAsync(&jump2, d_jump, sizeof(double), cudaMemcpyDeviceToHost, st));
        DK(cudaMemcpyAsync(hr.data(), d_reps, sizeof(DevReport) * n_sub, cudaMemcpyDeviceToHost, st));
        DK(cudaStreamSynchronize(st));
        float sweep_ms = 0.f;
        cudaEventElapsedTime(&sweep_ms, e0, e1);
        dev_ms += sweep_ms;
        bool inner_ok = true;
        int64_t inner_total = 0;
        for (int64_t s = 0; s < n_sub; ++s) {
            if (hr[s].error) return dfail(CVK_ETIMEOUT, "schwarz_solve: inner solve grid barrier aborted");
            if (hr[s].breakdown) inner_ok = false;
            inner_total += hr[s].iterations;
        }
        const double jump = std::sqrt(jump2);
        if (rep->jump_history && rep->jump_len < rep->jump_cap) rep->jump_history[rep->jump_len] = jump;
        rep->jump_len++;
        rep->outer_iterations = outer;
        rep->total_inner_iterations = inner_total;
        if (!inner_ok) {
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
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rep->sub_reports) {
        for (int64_t s = 0; s < n_sub && s < rep->n_sub_reports; ++s) {
            cvk_report& r = rep->sub_reports[s];
            r.converged = hr[s].converged;
            r.breakdown = hr[s].breakdown;
            r.iterations = hr[s].iterations;
            r.final_relres = hr[s].final_relres;
            r.true_relres = hr[s].true_relres;
            r.history_len = 0;
        }
    }
    k_ddm_scatter<<<(unsigned)((ntot + threads - 1) / threads), threads, 0, st>>>(geo, d_u, d_x, (int)ntot);
    DK(cudaGetLastError());
    DK(cudaMemcpyAsync(x, d_x, sizeof(double2) * n, cudaMemcpyDeviceToHost, st));
    DK(cudaStreamSynchronize(st));
    rep->device_time_s = dev_ms * 1e-3;
    rep->kernel_launches = launches + 1;
    rep->wall_time_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count() - t_wall0;
    return CVK_OK;
}
