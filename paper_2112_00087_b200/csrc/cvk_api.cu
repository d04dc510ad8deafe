// cvk_api.cu -- the C ABI declared in include/cavac_b200.h.
//
// Host control only: validation with the reference's error conventions
// (krylov.cpp / numkit.cpp invalid_argument cases become CVK_EINVAL with the
// same message text), device memory management, and one cooperative launch
// per solve.  There is no CPU compute path: every numeric result comes from a
// kernel; if the device or the kernel image is unavailable the call fails.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cavac_b200.h"
#include "cvk_engine.cuh"
#include "cvk_kernels.h"
#include "cvk_phased.h"
#include "cvk_stream.cuh"

using cvk::DevReport;

// the phase kernels compiled with 4 x 128-row consumer groups (cvk_phased_g4.cu)
namespace cvk_g4 {
int flavor_stream_rows();
int flavor_stream_threads();
size_t flavor_stage_bytes(int capk, int nvec, int ngather);
size_t flavor_smem_bytes(int capk, int nvec, int ngather, int stages);
void flavor_kernels(void* out);
void flavor_pack_args(void* out, int n, const int* rp, const int* ci, const double2* av, const int* cmax,
                      const double2* dinv, const double2* b, double2* x, double2* work, double2* part, void* st,
                      double* hist, void* rep, int capk, const int* nst, int pf_rows, const int* gprod,
                      const double2* udg);
}  // namespace cvk_g4
namespace cvk {
int flavor_stream_rows();
int flavor_stream_threads();
size_t flavor_stage_bytes(int capk, int nvec, int ngather);
size_t flavor_smem_bytes(int capk, int nvec, int ngather, int stages);
void flavor_kernels(void* out);
void flavor_pack_args(void* out, int n, const int* rp, const int* ci, const double2* av, const int* cmax,
                      const double2* dinv, const double2* b, double2* x, double2* work, double2* part, void* st,
                      double* hist, void* rep, int capk, const int* nst, int pf_rows, const int* gprod,
                      const double2* udg);
}  // namespace cvk

// execution-path options (cvk_ctx_set_option); defaults are the product's
struct CvkKnobs {
    long long phased_min_n = 131072;
    long long max_ctas = 0;
    long long stream = 1;
    long long flavor = 0;
    long long spmv_group = 0;
    long long gmres_persistent = 0;
    long long bicgl_persistent = 0;
    long long ilu_hostloop = 0;
    long long ddm_seq_min = 131072;
    long long rb_stream_min = 65536;
    long long bicg_fold = 1;
    long long gmres_tiles = 1;
    long long uniform = 0;  // measured: 24% fewer bytes per BiCGSTAB iteration, 2.5% less time
};

struct cvk_ctx {
    int device = 0;
    int nsm = 0;
    cudaStream_t stream = nullptr;
    int exec_parallel = 0;  // ExecMode::Sequential, the reference's initial mode (numkit.cpp:16)
    CvkKnobs knob;
    // reusable workspace
    void* work = nullptr;
    size_t work_bytes = 0;
    double2* part = nullptr;
    size_t part_bytes = 0;
    unsigned long long* bar = nullptr;  // [2]
    DevReport* rep = nullptr;
    double* hist = nullptr;
    size_t hist_cap = 0;
    double2* bx = nullptr;  // staging for host b / x
    size_t bx_n = 0;
    int* bad = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    // phase-kernel path
    cvk::PState* st = nullptr;
    int* h_done = nullptr;  // pinned [2]
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaGraphExec_t gexec = nullptr;
    std::vector<unsigned char> gkey;
    int gkind = -1;  // kernel set of gexec (solve_phased): updates only within one set
    // phase-kernel GMRES
    void* gst = nullptr;  // cvk::GState
    cudaGraphExec_t gm_exec = nullptr;
    std::vector<unsigned char> gm_key;
    // phase-kernel BiCGSTAB(l)
    void* bst = nullptr;  // cvk::BLState
    // the next BiCGSTAB solve starts from the x passed in (cvk_solve_device_warm)
    int warm_next = 0;
    cudaGraphExec_t bl_exec = nullptr;
    std::vector<unsigned char> bl_key;
    // device blocks released by cvk_csr_free / cvk_precond_free, reused by
    // the next upload of a similar size: a reference caller runs jacobi +
    // solve per call (pipeline.cpp:196-202), i.e. uploads and frees A each
    // time, and cudaMalloc / cudaFree of ~100 MB cost milliseconds each
    std::vector<std::pair<void*, size_t>> spare;
    size_t spare_bytes = 0;
};

static constexpr size_t kSpareCap = size_t(4) << 30;

static cudaError_t ctx_alloc(cvk_ctx* c, void** p, size_t bytes) {
    int best = -1;
    for (int i = 0; i < (int)c->spare.size(); ++i) {
        const size_t b = c->spare[i].second;
        if (b >= bytes && b - bytes <= bytes / 4 + (size_t(1) << 20) &&
            (best < 0 || b < c->spare[best].second))
            best = i;
    }
    if (best >= 0) {
        *p = c->spare[best].first;
        c->spare_bytes -= c->spare[best].second;
        c->spare.erase(c->spare.begin() + best);
        return cudaSuccess;
    }
    return cudaMalloc(p, bytes);
}

// returns the block's real size through *bytes_out when it came from the cache
static void ctx_release(cvk_ctx* c, void* p, size_t bytes) {
    if (!p) return;
    if (bytes > kSpareCap) { cudaFree(p); return; }
    c->spare.emplace_back(p, bytes);
    c->spare_bytes += bytes;
    while (c->spare_bytes > kSpareCap && !c->spare.empty()) {
        cudaFree(c->spare.front().first);
        c->spare_bytes -= c->spare.front().second;
        c->spare.erase(c->spare.begin());
    }
}

struct cvk_csr {
    cvk_ctx* ctx = nullptr;
    int64_t n = 0, nnz = 0;
    int* rp = nullptr;
    int* ci = nullptr;
    double2* av = nullptr;
    void* blob = nullptr;  // av | ci | rp in one allocation
    size_t blob_bytes = 0;
    int group = 1;  // SpMV lanes per row for FAST mode
    int capk = 0;   // max nnz of a kStreamRows-row chunk, rounded up to 4 (streamed kernels)
    int capk_g4 = 0;  // the same for the 128-row chunks of the cvk_g4 flavor
    int* cmax = nullptr;  // [nchunks] largest column of each streamed chunk (L2 prefetch)
    double2* dg = nullptr;   // [n] diagonal + [2] uniform flag / value (Csr::dg, Csr::uni), allocated at
                             // the first streamed solve, refreshed at every streamed solve
};

// The streamed solves check the matrix for uniform off-diagonal values at the
// start of every solve (the values change between solves: sweeps,
// set_values): uniform_dg allocates (nullptr: the general path), the check
// is enqueued inside the solve's timed region.
static double2* uniform_dg(cvk_ctx* c, cvk_csr* A) {
    if (!c->knob.uniform) return nullptr;
    if (!A->dg && cudaMalloc(&A->dg, sizeof(double2) * ((size_t)std::max<int64_t>(1, A->n) + 2)) != cudaSuccess) {
        A->dg = nullptr;
        cudaGetLastError();
    }
    return A->dg;
}

struct cvk_prec {
    cvk_ctx* ctx = nullptr;
    int64_t n = 0;
    double2* dinv = nullptr;  // nullptr: identity (unless ilu is set)
    cvk::IluDev* ilu = nullptr;  // ILU(0) (cvk_precond_ilu0); dinv stays nullptr
    std::vector<double2> ilu_fac;  // host copy of the factor in A's value slots
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                     \
    do {                                                                             \
        cudaError_t e_ = (call);                                                     \
        if (e_ != cudaSuccess)                                                       \
            return fail(e_ == cudaErrorMemoryAllocation ? CVK_ENOMEM : CVK_ECUDA,    \
                        std::string(#call) + ": " + cudaGetErrorString(e_));         \
    } while (0)

const char* kSolverNames[] = {"bicgstab", "bicgstab_l", "tfqmr", "gmres", "cocg"};

int pick_group(const cvk_ctx* c, double avg_nnz) {
    const long long v = c->knob.spmv_group;
    if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) return (int)v;
    // thread per row with all of a row's loads issued up front wins up to
    // ~16 entries per row (profiles/r01_spmv_lab.txt); lanes per row beyond
    if (avg_nnz <= 16.0) return 1;
    if (avg_nnz <= 48.0) return 4;
    return 8;
}

int ensure(cvk_ctx* c, void** p, size_t* have, size_t need) {
    if (*have >= need && *p) return CVK_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    CK(cudaMalloc(p, need));
    *have = need;
    (void)c;
    return CVK_OK;
}

int resolve_mode(const cvk_ctx* c, int mode) {
    if (mode == CVK_MODE_FAST || mode == CVK_MODE_REF || mode == CVK_MODE_REF_PAR) return mode;
    return c->exec_parallel ? CVK_MODE_REF_PAR : CVK_MODE_REF;
}

bool is_ref(int mode) { return mode == CVK_MODE_REF || mode == CVK_MODE_REF_PAR; }

long long* knob_slot(cvk_ctx* c, int key) {
    switch (key) {
        case CVK_OPT_PHASED_MIN_N: return &c->knob.phased_min_n;
        case CVK_OPT_MAX_CTAS: return &c->knob.max_ctas;
        case CVK_OPT_STREAM: return &c->knob.stream;
        case CVK_OPT_STREAM_FLAVOR: return &c->knob.flavor;
        case CVK_OPT_SPMV_GROUP: return &c->knob.spmv_group;
        case CVK_OPT_GMRES_PERSISTENT: return &c->knob.gmres_persistent;
        case CVK_OPT_BICGL_PERSISTENT: return &c->knob.bicgl_persistent;
        case CVK_OPT_ILU_HOSTLOOP: return &c->knob.ilu_hostloop;
        case CVK_OPT_DDM_SEQ_MIN: return &c->knob.ddm_seq_min;
        case CVK_OPT_RB_STREAM_MIN: return &c->knob.rb_stream_min;
        case CVK_OPT_BICG_FOLD: return &c->knob.bicg_fold;
        case CVK_OPT_GMRES_TILES: return &c->knob.gmres_tiles;
        case CVK_OPT_UNIFORM_OFFDIAG: return &c->knob.uniform;
    }
    return nullptr;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

int cvk_fail(int code, const std::string& msg) { return fail(code, msg); }
long long cvk_ctx_knob(cvk_ctx* c, int key) {
    const long long* p = knob_slot(c, key);
    return p ? *p : 0;
}

extern "C" {

int cvk_abi_version(void) { return CVK_ABI_VERSION; }

// measurement builds only (CVK_TRACE): not part of include/cavac_b200.h
int cvk_trace_read(void* out, size_t bytes) { return cvk::phased_trace_read(out, bytes); }
const char* cvk_last_error(void) { return g_err.c_str(); }

const char* cvk_breakdown_name(int code) {
    switch (code) {
        case CVK_BRK_NONE: return "";
        case CVK_BRK_RHO: return "rho breakdown";
        case CVK_BRK_SHADOW_V: return "stagnation in <shadow, v>";
        case CVK_BRK_OMEGA: return "omega breakdown";
        case CVK_BRK_SHADOW_U: return "stagnation in <shadow, u>";
        case CVK_BRK_MR: return "degenerate least-squares in MR step";
        case CVK_BRK_SIGMA: return "sigma breakdown";
        case CVK_BRK_ARNOLDI: return "arnoldi breakdown";
        case CVK_BRK_PAP: return "stagnation in <p, A p>";
    }
    return "unknown breakdown";
}

const char* cvk_solver_name(int solver) {
    if (solver < 0 || solver > 4) return "?";
    return kSolverNames[solver];
}

int cvk_solver_from_name(const char* name) {
    if (name)
        for (int i = 0; i < 5; ++i)
            if (std::strcmp(name, kSolverNames[i]) == 0) return i;
    return fail(CVK_ESOLVER, std::string("unknown solver \"") + (name ? name : "") +
                                 "\" (allowed: bicgstab, bicgstab_l, tfqmr, gmres, cocg)");
}

int cvk_ctx_create(int device, cvk_ctx** out) {
    if (!out) return fail(CVK_EINVAL, "cvk_ctx_create: null out");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(CVK_EINVAL, "cvk_ctx_create: no such device");
    CK(cudaSetDevice(device));
    cvk_ctx* c = new cvk_ctx();
    c->device = device;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) {
        delete c;
        return fail(CVK_ECUDA, "cvk_ctx_create: device is not sm_100-class (built for sm_100a only)");
    }
    c->nsm = prop.multiProcessorCount;
    int coop = 0;
    CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
    if (!coop) {
        delete c;
        return fail(CVK_ECUDA, "cvk_ctx_create: device lacks cooperative launch");
    }
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaMalloc(&c->bar, 2 * sizeof(unsigned long long)));
    CK(cudaMalloc(&c->rep, sizeof(DevReport)));
    CK(cudaMalloc(&c->bad, sizeof(int)));
    CK(cudaEventCreate(&c->e0));
    CK(cudaEventCreate(&c->e1));
    CK(cudaEventCreateWithFlags(&c->ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev[1], cudaEventDisableTiming));
    CK(cudaMalloc(&c->st, sizeof(cvk::PState)));
    CK(cudaHostAlloc(&c->h_done, 2 * sizeof(int), cudaHostAllocDefault));
    *out = c;
    return CVK_OK;
}

int cvk_ctx_destroy(cvk_ctx* c) {
    if (!c) return CVK_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    cudaFree(c->work);
    cudaFree(c->part);
    cudaFree(c->bar);
    cudaFree(c->rep);
    cudaFree(c->hist);
    cudaFree(c->bx);
    cudaFree(c->bad);
    cudaEventDestroy(c->e0);
    cudaEventDestroy(c->e1);
    cudaEventDestroy(c->ev[0]);
    cudaEventDestroy(c->ev[1]);
    cudaFree(c->st);
    cudaFreeHost(c->h_done);
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    if (c->gm_exec) cudaGraphExecDestroy(c->gm_exec);
    cudaFree(c->gst);
    if (c->bl_exec) cudaGraphExecDestroy(c->bl_exec);
    for (auto& sp : c->spare) cudaFree(sp.first);
    cudaFree(c->bst);
    cudaStreamDestroy(c->stream);
    delete c;
    return CVK_OK;
}

void* cvk_ctx_stream(cvk_ctx* c) { return c ? (void*)c->stream : nullptr; }

int cvk_set_exec_mode(cvk_ctx* c, int parallel) {
    if (!c) return fail(CVK_EINVAL, "null ctx");
    c->exec_parallel = parallel ? 1 : 0;
    return CVK_OK;
}
int cvk_get_exec_mode(cvk_ctx* c) { return c ? c->exec_parallel : 0; }

int cvk_ctx_set_option(cvk_ctx* c, int key, int64_t value) {
    if (!c) return fail(CVK_EINVAL, "null ctx");
    long long* p = knob_slot(c, key);
    if (!p) return fail(CVK_EINVAL, "cvk_ctx_set_option: unknown option " + std::to_string(key));
    *p = value;
    return CVK_OK;
}

int cvk_ctx_get_option(cvk_ctx* c, int key, int64_t* value) {
    if (!c || !value) return fail(CVK_EINVAL, "cvk_ctx_get_option: null argument");
    const long long* p = knob_slot(c, key);
    if (!p) return fail(CVK_EINVAL, "cvk_ctx_get_option: unknown option " + std::to_string(key));
    *value = *p;
    return CVK_OK;
}

int cvk_csr_upload(cvk_ctx* c, int64_t nrows, int64_t ncols, int64_t nnz, const uint64_t* row_offsets,
                   const uint64_t* col_indices, const double* values, cvk_csr** out) {
    if (!c || !out) return fail(CVK_EINVAL, "cvk_csr_upload: null argument");
    if (nrows < 0 || ncols < 0 || nnz < 0) return fail(CVK_EINVAL, "cvk_csr_upload: negative size");
    if (nrows != ncols) return fail(CVK_EINVAL, "cvk_csr_upload: matrix must be square");
    if (nrows >= INT32_MAX || nnz >= INT32_MAX)
        return fail(CVK_EOVERFLOW, "cvk_csr_upload: size exceeds the int32 device index range");
    if (!row_offsets || (nnz > 0 && (!col_indices || !values)))
        return fail(CVK_EINVAL, "cvk_csr_upload: null array");
    std::vector<int> rp((size_t)nrows + 1), ci((size_t)nnz);
    if (row_offsets[0] != 0) return fail(CVK_EINVAL, "cvk_csr_upload: row_offsets[0] != 0");
    for (int64_t i = 0; i <= nrows; ++i) {
        if (row_offsets[i] > (uint64_t)nnz || (i > 0 && row_offsets[i] < row_offsets[i - 1]))
            return fail(CVK_EINVAL, "cvk_csr_upload: row_offsets not monotone within [0, nnz]");
        rp[(size_t)i] = (int)row_offsets[i];
    }
    if (row_offsets[nrows] != (uint64_t)nnz) return fail(CVK_EINVAL, "cvk_csr_upload: row_offsets[n] != nnz");
    {
        // narrow the columns on all host cores (5M entries per 1M DOF)
        const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(16, nnz / (1 << 18)));
        std::vector<int64_t> bad((size_t)nt, -1);
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                const int64_t k0 = nnz * t / nt, k1 = nnz * (t + 1) / nt;
                for (int64_t k = k0; k < k1; ++k) {
                    if (col_indices[k] >= (uint64_t)ncols) { bad[(size_t)t] = k; return; }
                    ci[(size_t)k] = (int)col_indices[k];
                }
            });
        for (auto& t : th) t.join();
        for (int64_t k : bad)
            if (k >= 0) return fail(CVK_EINVAL, "cvk_csr_upload: column index out of range at " + std::to_string(k));
    }
    CK(cudaSetDevice(c->device));
    cvk_csr* A = new cvk_csr();
    A->ctx = c;
    A->n = nrows;
    A->nnz = nnz;
    A->group = pick_group(c, nrows ? (double)nnz / (double)nrows : 1.0);

    // one allocation [values | columns | row offsets] so a single L2
    // access-policy window can pin the whole matrix (solve-time persistence)
    const size_t vb = sizeof(double2) * (size_t)std::max<int64_t>(1, nnz);
    const size_t cb = (sizeof(int) * (size_t)std::max<int64_t>(1, nnz) + 255) & ~(size_t)255;
    // 16 bytes of padding: the streamed kernels copy row offsets in 16-byte units
    const size_t rb = sizeof(int) * rp.size() + 16;
    CK(ctx_alloc(c, &A->blob, vb + cb + rb));
    A->blob_bytes = vb + cb + rb;
    A->av = (double2*)A->blob;
    A->ci = (int*)((char*)A->blob + vb);
    A->rp = (int*)((char*)A->blob + vb + cb);
    CK(cudaMemcpyAsync(A->rp, rp.data(), sizeof(int) * rp.size(), cudaMemcpyHostToDevice, c->stream));
    if (nnz) {
        CK(cudaMemcpyAsync(A->ci, ci.data(), sizeof(int) * ci.size(), cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(A->av, values, sizeof(double2) * nnz, cudaMemcpyHostToDevice, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    {
        long long mk = 0;
        for (int64_t r0 = 0; r0 < nrows; r0 += cvk::kStreamRows)
            mk = std::max<long long>(mk, (long long)rp[(size_t)std::min<int64_t>(r0 + cvk::kStreamRows, nrows)] -
                                             (long long)rp[(size_t)r0]);
        A->capk = (int)((mk + 3) & ~3LL);
        long long mk4 = 0;
        const int r4 = cvk_g4::flavor_stream_rows();
        for (int64_t r0 = 0; r0 < nrows; r0 += r4)
            mk4 = std::max<long long>(mk4, (long long)rp[(size_t)std::min<int64_t>(r0 + r4, nrows)] - (long long)rp[(size_t)r0]);
        A->capk_g4 = (int)((mk4 + 3) & ~3LL);
        const int64_t nch = (nrows + cvk::kStreamRows - 1) / cvk::kStreamRows;
        std::vector<int> cm((size_t)std::max<int64_t>(1, nch), -1);
        for (int64_t q = 0; q < nch; ++q) {
            const int64_t r1 = std::min<int64_t>((q + 1) * cvk::kStreamRows, nrows);
            for (int64_t k = rp[(size_t)(q * cvk::kStreamRows)]; k < rp[(size_t)r1]; ++k)
                cm[(size_t)q] = std::max(cm[(size_t)q], ci[(size_t)k]);
        }
        if (cudaMalloc(&A->cmax, sizeof(int) * cm.size()) == cudaSuccess)
            cudaMemcpy(A->cmax, cm.data(), sizeof(int) * cm.size(), cudaMemcpyHostToDevice);
        else
            A->cmax = nullptr;
    }
    *out = A;
    return CVK_OK;
}

int cvk_csr_set_values(cvk_csr* A, const double* values) {
    if (!A || (!values && A->nnz)) return fail(CVK_EINVAL, "cvk_csr_set_values: null argument");
    CK(cudaSetDevice(A->ctx->device));
    if (A->nnz)
        CK(cudaMemcpyAsync(A->av, values, sizeof(double2) * A->nnz, cudaMemcpyHostToDevice, A->ctx->stream));
    CK(cudaStreamSynchronize(A->ctx->stream));
    return CVK_OK;
}

int cvk_csr_get_values(const cvk_csr* A, double* values) {
    if (!A || (!values && A->nnz)) return fail(CVK_EINVAL, "cvk_csr_get_values: null argument");
    CK(cudaSetDevice(A->ctx->device));
    CK(cudaStreamSynchronize(A->ctx->stream));
    if (A->nnz) CK(cudaMemcpy(values, A->av, sizeof(double2) * A->nnz, cudaMemcpyDeviceToHost));
    return CVK_OK;
}

int cvk_csr_free(cvk_csr* A) {
    if (!A) return CVK_OK;
    cudaSetDevice(A->ctx->device);
    cudaStreamSynchronize(A->ctx->stream);
    ctx_release(A->ctx, A->blob, A->blob_bytes);
    if (A->cmax) cudaFree(A->cmax);
    if (A->dg) cudaFree(A->dg);
    delete A;
    return CVK_OK;
}

int64_t cvk_csr_nrows(const cvk_csr* A) { return A ? A->n : -1; }
int64_t cvk_csr_nnz(const cvk_csr* A) { return A ? A->nnz : -1; }

int cvk_precond_jacobi(cvk_csr* A, const double* inv_diag, cvk_prec** out) {
    if (!A || !out) return fail(CVK_EINVAL, "cvk_precond_jacobi: null argument");
    cvk_ctx* c = A->ctx;
    CK(cudaSetDevice(c->device));
    cvk_prec* M = new cvk_prec();
    M->ctx = c;
    M->n = A->n;
    CK(ctx_alloc(c, (void**)&M->dinv, sizeof(double2) * std::max<int64_t>(1, A->n)));
    if (inv_diag) {
        CK(cudaMemcpyAsync(M->dinv, inv_diag, sizeof(double2) * A->n, cudaMemcpyHostToDevice, c->stream));
    } else {
        const int big = INT32_MAX;
        CK(cudaMemcpyAsync(c->bad, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream));
        CK(cvk::launch_inv_diag((int)A->n, A->rp, A->ci, A->av, M->dinv, c->bad, c->stream));
        int bad = 0;
        CK(cudaMemcpyAsync(&bad, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (bad != INT32_MAX) {
            cudaFree(M->dinv);
            delete M;
            return fail(CVK_EZERODIAG, "jacobi: zero diagonal at row " + std::to_string(bad));
        }
    }
    CK(cudaStreamSynchronize(c->stream));
    *out = M;
    return CVK_OK;
}

int cvk_precond_jacobi_refresh(cvk_prec* M, const cvk_csr* A) {
    if (!M || !A) return fail(CVK_EINVAL, "cvk_precond_jacobi_refresh: null argument");
    if (!M->dinv) return fail(CVK_EINVAL, "cvk_precond_jacobi_refresh: identity preconditioner");
    if (M->n != A->n || M->ctx != A->ctx) return fail(CVK_EINVAL, "cvk_precond_jacobi_refresh: dimension mismatch");
    cvk_ctx* c = A->ctx;
    CK(cudaSetDevice(c->device));
    const int big = INT32_MAX;
    CK(cudaMemcpyAsync(c->bad, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CK(cvk::launch_inv_diag((int)A->n, A->rp, A->ci, A->av, M->dinv, c->bad, c->stream));
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (bad != INT32_MAX) return fail(CVK_EZERODIAG, "jacobi: zero diagonal at row " + std::to_string(bad));
    return CVK_OK;
}

int cvk_csr_assemble_cavity(cvk_csr* A, const cvk_grid* g, double omega, double c_sound) {
    if (!A || !g) return fail(CVK_EINVAL, "cvk_csr_assemble_cavity: null argument");
    if (g->nx < 1 || g->ny < 1 || g->nx * g->ny != A->n)
        return fail(CVK_EINVAL, "cvk_csr_assemble_cavity: grid does not match the matrix size");
    cvk_ctx* c = A->ctx;
    // host scalars with std::complex, exactly as helmholtz.cpp:65-73
    using Cx = std::complex<double>;
    const double k2 = c_sound * c_sound / (g->h * g->h);
    const Cx adm(g->admittance_re, g->admittance_im);
    Cx ww(1.0);
    if (adm != Cx(0.0)) ww = 1.0 / (Cx(1.0) + Cx(0.0, omega * g->h) * adm);
    const Cx kw = k2 * ww;
    CK(cudaSetDevice(c->device));
    const int big = INT32_MAX;
    CK(cudaMemcpyAsync(c->bad, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CK(cvk::launch_cavity_values((int)g->nx, (int)g->ny, (int)g->roof_begin, (int)g->roof_end, k2, omega * omega,
                                 kw.real(), kw.imag(), A->rp, A->ci, A->av, c->bad, c->nsm, c->stream));
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (bad != INT32_MAX)
        return fail(CVK_EINVAL, "cvk_csr_assemble_cavity: matrix pattern is not the cavity's 5-point pattern at row " +
                                    std::to_string(bad));
    return CVK_OK;
}

struct cvk_fem {
    cvk_csr* A = nullptr;
    double* kmc = nullptr;  // K | M | C, nnz each
};

int cvk_fem_create(cvk_csr* A, const double* K, const double* M, const double* Cd, cvk_fem** out) {
    if (!A || !K || !M || !Cd || !out) return fail(CVK_EINVAL, "cvk_fem_create: null argument");
    CK(cudaSetDevice(A->ctx->device));
    cvk_fem* F = new cvk_fem();
    F->A = A;
    const size_t nz = (size_t)std::max<int64_t>(1, A->nnz);
    if (cudaMalloc(&F->kmc, 3 * sizeof(double) * nz) != cudaSuccess) {
        delete F;
        return fail(CVK_ENOMEM, "cvk_fem_create: device allocation failed");
    }
    CK(cudaMemcpyAsync(F->kmc, K, sizeof(double) * A->nnz, cudaMemcpyHostToDevice, A->ctx->stream));
    CK(cudaMemcpyAsync(F->kmc + nz, M, sizeof(double) * A->nnz, cudaMemcpyHostToDevice, A->ctx->stream));
    CK(cudaMemcpyAsync(F->kmc + 2 * nz, Cd, sizeof(double) * A->nnz, cudaMemcpyHostToDevice, A->ctx->stream));
    CK(cudaStreamSynchronize(A->ctx->stream));
    *out = F;
    return CVK_OK;
}

int cvk_fem_set_omega(cvk_fem* F, double omega) {
    if (!F) return fail(CVK_EINVAL, "cvk_fem_set_omega: null argument");
    cvk_csr* A = F->A;
    CK(cudaSetDevice(A->ctx->device));
    const size_t nz = (size_t)std::max<int64_t>(1, A->nnz);
    CK(cvk::launch_fem_values(A->nnz, F->kmc, F->kmc + nz, F->kmc + 2 * nz, omega, A->av, A->ctx->nsm, A->ctx->stream));
    CK(cudaStreamSynchronize(A->ctx->stream));
    return CVK_OK;
}

int cvk_fem_free(cvk_fem* F) {
    if (!F) return CVK_OK;
    cudaSetDevice(F->A->ctx->device);
    cudaFree(F->kmc);
    delete F;
    return CVK_OK;
}

int cvk_precond_identity(cvk_ctx* c, int64_t n, cvk_prec** out) {
    if (!c || !out || n < 0) return fail(CVK_EINVAL, "cvk_precond_identity: bad argument");
    cvk_prec* M = new cvk_prec();
    M->ctx = c;
    M->n = n;
    *out = M;
    return CVK_OK;
}

int cvk_precond_free(cvk_prec* M) {
    if (!M) return CVK_OK;
    if (M->dinv) {
        cudaSetDevice(M->ctx->device);
        cudaStreamSynchronize(M->ctx->stream);
        ctx_release(M->ctx, M->dinv, sizeof(double2) * std::max<int64_t>(1, M->n));
    }
    if (M->ilu) {
        cudaSetDevice(M->ctx->device);
        cudaFree(M->ilu->blob);
        delete M->ilu;
    }
    delete M;
    return CVK_OK;
}

int cvk_precond_get_diag(const cvk_prec* M, double* inv_diag) {
    if (!M || !inv_diag) return fail(CVK_EINVAL, "cvk_precond_get_diag: null argument");
    if (!M->dinv) return fail(CVK_EINVAL, M->ilu ? "cvk_precond_get_diag: ILU(0) preconditioner"
                                                 : "cvk_precond_get_diag: identity preconditioner");
    CK(cudaSetDevice(M->ctx->device));
    CK(cudaMemcpy(inv_diag, M->dinv, sizeof(double2) * M->n, cudaMemcpyDeviceToHost));
    return CVK_OK;
}

// ILU(0): exact factor on A's pattern on the host (IKJ; the order and
// roundings of oracle/cavac_oracle.c orc_ilu0_arrays), split into strict L,
// strict U and d = 1 / u_ii for the device sweeps (cvk_ilu.cu).  Beyond the
// reference (krylov.cpp:27-55 has jacobi / identity only).
int cvk_precond_ilu0(cvk_csr* A, int sweeps, cvk_prec** out) {
    if (!A || !out) return fail(CVK_EINVAL, "cvk_precond_ilu0: null argument");
    if (sweeps < 0 || sweeps > 64) return fail(CVK_EINVAL, "cvk_precond_ilu0: sweeps must be in [0, 64]");
    cvk_ctx* c = A->ctx;
    CK(cudaSetDevice(c->device));
    const int64_t n = A->n, nnz = A->nnz;
    std::vector<int> rp(n + 1), ci(std::max<int64_t>(1, nnz));
    std::vector<double2> f(std::max<int64_t>(1, nnz));
    CK(cudaMemcpyAsync(rp.data(), A->rp, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, c->stream));
    if (nnz) {
        CK(cudaMemcpyAsync(ci.data(), A->ci, sizeof(int) * nnz, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(f.data(), A->av, sizeof(double2) * nnz, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    // the IKJ factor below walks each row in column order (L part, then U from
    // the diagonal on): a row with unsorted or repeated columns would get a
    // silently wrong factor, so reject it (csr_from_triplets sorts,
    // numkit.cpp:41-75; a hand-built CsrMatrix need not)
    for (int64_t i = 0; i < n; ++i)
        for (int p = rp[i] + 1; p < rp[i + 1]; ++p)
            if (ci[p] <= ci[p - 1])
                return fail(CVK_EINVAL, "ilu0: columns of row " + std::to_string(i) + " are not strictly increasing");
    std::vector<int64_t> pos(std::max<int64_t>(1, n), -1), dg(std::max<int64_t>(1, n), -1);
    for (int64_t i = 0; i < n; ++i) {
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            pos[ci[p]] = p;
            if (ci[p] == i) dg[i] = p;
        }
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            const int k = ci[p];
            if (k >= i) break;
            f[p] = cvk_cdiv(f[p], f[dg[k]]);
            const double2 lik = f[p];
            for (int q = (int)dg[k] + 1; q < rp[k + 1]; ++q) {
                const int64_t t = pos[ci[q]];
                if (t >= 0) f[t] = cvk_sub(f[t], cvk_mul(lik, f[q]));
            }
        }
        for (int p = rp[i]; p < rp[i + 1]; ++p) pos[ci[p]] = -1;
        if (dg[i] < 0 || (f[dg[i]].x == 0.0 && f[dg[i]].y == 0.0))
            return fail(CVK_EZERODIAG, "ilu0: zero pivot at row " + std::to_string(i));
    }
    // split: L strict lower, U strict upper (CSR order kept), d = 1 / u_ii
    std::vector<int> lrp(n + 1, 0), urp(n + 1, 0), lci, uci;
    std::vector<double2> lav, uav, d(std::max<int64_t>(1, n));
    lci.reserve(nnz / 2 + 1), uci.reserve(nnz / 2 + 1), lav.reserve(nnz / 2 + 1), uav.reserve(nnz / 2 + 1);
    for (int64_t i = 0; i < n; ++i) {
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            if (ci[p] < i) { lci.push_back(ci[p]); lav.push_back(f[p]); }
            else if (ci[p] > i) { uci.push_back(ci[p]); uav.push_back(f[p]); }
        }
        lrp[i + 1] = (int)lci.size();
        urp[i + 1] = (int)uci.size();
        d[i] = cvk_cdiv(make_double2(1.0, 0.0), f[dg[i]]);
    }
    const size_t nl = lci.size(), nu = uci.size();
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t o_lav = 0, o_uav = o_lav + al(16 * nl), o_d = o_uav + al(16 * nu), o_lci = o_d + al(16 * n),
                 o_uci = o_lci + al(4 * nl), o_lrp = o_uci + al(4 * nu), o_urp = o_lrp + al(4 * (n + 1)),
                 total = o_urp + al(4 * (n + 1));
    cvk::IluDev* I = new cvk::IluDev();
    I->n = (int)n;
    I->sweeps = sweeps;
    if (cudaMalloc(&I->blob, total) != cudaSuccess) {
        delete I;
        return fail(CVK_ENOMEM, "ilu0: out of device memory");
    }
    char* b = (char*)I->blob;
    I->lav = (double2*)(b + o_lav), I->uav = (double2*)(b + o_uav), I->dinv = (double2*)(b + o_d);
    I->lci = (int*)(b + o_lci), I->uci = (int*)(b + o_uci), I->lrp = (int*)(b + o_lrp), I->urp = (int*)(b + o_urp);
    cudaStream_t st = c->stream;
    if (nl) CK(cudaMemcpyAsync(I->lav, lav.data(), 16 * nl, cudaMemcpyHostToDevice, st));
    if (nu) CK(cudaMemcpyAsync(I->uav, uav.data(), 16 * nu, cudaMemcpyHostToDevice, st));
    if (nl) CK(cudaMemcpyAsync(I->lci, lci.data(), 4 * nl, cudaMemcpyHostToDevice, st));
    if (nu) CK(cudaMemcpyAsync(I->uci, uci.data(), 4 * nu, cudaMemcpyHostToDevice, st));
    if (n) CK(cudaMemcpyAsync(I->dinv, d.data(), 16 * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(I->lrp, lrp.data(), 4 * (n + 1), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(I->urp, urp.data(), 4 * (n + 1), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    cvk_prec* M = new cvk_prec();
    M->ctx = c;
    M->n = n;
    M->ilu = I;
    f.resize(nnz);
    M->ilu_fac = std::move(f);
    *out = M;
    return CVK_OK;
}

int cvk_precond_get_ilu0(const cvk_prec* M, double* factor) {
    if (!M || !factor) return fail(CVK_EINVAL, "cvk_precond_get_ilu0: null argument");
    if (!M->ilu) return fail(CVK_EINVAL, "cvk_precond_get_ilu0: not an ILU(0) preconditioner");
    if (!M->ilu_fac.empty()) std::memcpy(factor, M->ilu_fac.data(), sizeof(double2) * M->ilu_fac.size());
    return CVK_OK;
}

}  // extern "C"

namespace {
// z = M^-1 r on the device for any preconditioner kind; tmp >= 2 n complex
int prec_apply_dev(const cvk_prec* M, const double2* r, double2* z, double2* tmp, int* nl) {
    cvk_ctx* c = M->ctx;
    const int n = (int)M->n;
    if (n <= 0) return CVK_OK;
    if (M->ilu) {
        CK(cvk::launch_ilu0_apply(*M->ilu, r, z, tmp, nl, c->stream));
    } else if (M->dinv) {
        cvk::IluDev J;  // s = 0: z = d .* r
        J.n = n;
        J.sweeps = 0;
        J.dinv = M->dinv;
        CK(cvk::launch_ilu0_apply(J, r, z, tmp, nl, c->stream));
    } else {
        CK(cudaMemcpyAsync(z, r, sizeof(double2) * n, cudaMemcpyDeviceToDevice, c->stream));
    }
    return CVK_OK;
}
}  // namespace

extern "C" {

int cvk_precond_apply_device(const cvk_prec* M, const double* r_dev, double* z_dev) {
    if (!M || (M->n && (!r_dev || !z_dev))) return fail(CVK_EINVAL, "cvk_precond_apply_device: null argument");
    if (r_dev == z_dev && M->n) return fail(CVK_EINVAL, "cvk_precond_apply_device: r and z alias");
    cvk_ctx* c = M->ctx;
    CK(cudaSetDevice(c->device));
    int e;
    if ((e = ensure(c, &c->work, &c->work_bytes, sizeof(double2) * 2 * std::max<size_t>(1, M->n))) != CVK_OK)
        return e;
    return prec_apply_dev(M, (const double2*)r_dev, (double2*)z_dev, (double2*)c->work, nullptr);
}

static int stage(cvk_ctx* c, size_t n2);

int cvk_precond_apply(const cvk_prec* M, const double* r, double* z) {
    if (!M || (M->n && (!r || !z))) return fail(CVK_EINVAL, "cvk_precond_apply: null argument");
    cvk_ctx* c = M->ctx;
    CK(cudaSetDevice(c->device));
    const size_t n = (size_t)M->n;
    if (!n) return CVK_OK;
    int e;
    if ((e = stage(c, 2 * n)) != CVK_OK) return e;
    double2* rd = c->bx;
    double2* zd = c->bx + n;
    CK(cudaMemcpyAsync(rd, r, sizeof(double2) * n, cudaMemcpyHostToDevice, c->stream));
    if ((e = cvk_precond_apply_device(M, (const double*)rd, (double*)zd)) != CVK_OK) return e;
    CK(cudaMemcpyAsync(z, zd, sizeof(double2) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return CVK_OK;
}

// FAST BiCGSTAB + ILU(0): the cvk_ilu.cu phase chain, scalars on the device,
// kIcPerGraph iterations per CUDA graph, the done flag polled one graph late.
struct IcSpmv {
    const cvk_csr* A;
    double2* out;
    int optin, nsm, streamed;
    cudaStream_t st;
    const int* skip;  // the chain's done flag
};
static cudaError_t ic_spmv(void* ctx, const double2* in) {
    const IcSpmv* q = (const IcSpmv*)ctx;
    const cvk_csr* A = q->A;
    if (q->streamed)
        return cvk::launch_spmv_stream((int)A->n, A->rp, A->ci, A->av, in, q->out, A->capk, q->nsm, q->optin, q->st,
                                       q->skip);
    return cvk::launch_spmv(A->group, false, (int)A->n, A->rp, A->ci, A->av, in, q->out, 0, q->st);
}

static int solve_ilu_chain(cvk_ctx* c, const cvk_csr* A, const cvk_prec* M, const cvk_opts* o,
                           const double2* b, double2* x, cvk_report* rep) {
    constexpr int kIcPerGraph = 8;
    const int n = (int)A->n;
    cudaStream_t st = c->stream;
    int e;
    const size_t nv = (size_t)std::max(1, n);
    if ((e = ensure(c, &c->work, &c->work_bytes, sizeof(double2) * 10 * nv)) != CVK_OK) return e;
    if ((e = ensure(c, (void**)&c->part, &c->part_bytes, sizeof(double2) * 4 * 592)) != CVK_OK) return e;
    double2* w = (double2*)c->work;
    double2* sh = w + 9 * nv;
    cvk::IcArgs a;
    a.n = n, a.x = x, a.r = w, a.p = w + nv, a.v = w + 2 * nv, a.s = w + 3 * nv, a.t = w + 4 * nv;
    a.tmp = w + 5 * nv, a.ptmp = w + 6 * nv, a.sh = sh, a.part = c->part;
    const long long hcap = o->record_history && rep->history ? std::max<long long>(0, rep->history_cap) : 0;
    void* mem = nullptr;
    CK(cudaMalloc(&mem, sizeof(cvk::IcState) + sizeof(double) * std::max<long long>(1, hcap)));
    struct Free { void* p; ~Free() { cudaFree(p); } } guard{mem};
    a.st = (cvk::IcState*)mem;
    a.hist = (double*)((char*)mem + sizeof(cvk::IcState));
    cvk::IcState h0 = {};
    h0.record = o->record_history ? 1 : 0;
    h0.max_iter = o->max_iter, h0.hist_cap = hcap, h0.tol = o->tol;
    h0.rho = h0.alpha = h0.omega = make_double2(1.0, 0.0);
    IcSpmv q{A, a.tmp, 0, c->nsm, 0, st, &a.st->done};
    if (A->n >= 4 * cvk::kStreamRows && A->nnz > 0 && c->knob.stream) {
        CK(cudaDeviceGetAttribute(&q.optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
        q.streamed = 1;
    }
    int nl = 0;
    long long launches = 0;
    CK(cudaEventRecord(c->e0, st));
    CK(cudaMemcpyAsync(a.st, &h0, sizeof(h0), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(x, 0, sizeof(double2) * nv, st));
    CK(cvk::launch_ilu0_apply(*M->ilu, b, a.r, a.ptmp, &nl, st));  // r = M^-1 b
    CK(cudaMemcpyAsync(sh, a.r, sizeof(double2) * n, cudaMemcpyDeviceToDevice, st));
    CK(cvk::launch_ic_init(a, st));
    launches += 2;
    if (q.streamed) {  // first call outside the capture sets the kernel attributes
        const cudaError_t se = ic_spmv(&q, a.r);
        if (se == cudaErrorInvalidConfiguration) {
            (void)cudaGetLastError();
            q.streamed = 0;
        } else {
            CK(se);
            ++launches;
        }
    }
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    int nl_graph = 0;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    const cudaError_t ce = cvk::launch_ic_iters(a, *M->ilu, kIcPerGraph, ic_spmv, &q, &nl_graph, st);
    const cudaError_t ee = cudaStreamEndCapture(st, &graph);
    CK(ce);
    CK(ee);
    CK(cudaGraphInstantiate(&gexec, graph, 0));
    cudaGraphDestroy(graph);
    struct GFree { cudaGraphExec_t g; ~GFree() { cudaGraphExecDestroy(g); } } gguard{gexec};
    long long graphs = 0;
    const long long max_graphs = o->max_iter / kIcPerGraph + 3;
    while (graphs < max_graphs) {
        CK(cudaGraphLaunch(gexec, st));
        const int slot = (int)(graphs & 1);
        CK(cudaMemcpyAsync(&c->h_done[slot], &a.st->done, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(c->ev[slot], st));
        ++graphs;
        launches += nl_graph;
        if (graphs >= 2) {
            const int old = (int)((graphs - 2) & 1);
            CK(cudaEventSynchronize(c->ev[old]));
            if (c->h_done[old]) break;
        }
    }
    cvk::IcState hs;
    CK(cudaMemcpyAsync(&hs, a.st, sizeof(hs), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!hs.done) return fail(CVK_ELOGIC, "bicgstab+ilu0: iteration chain did not finish");
    rep->converged = hs.conv, rep->breakdown = hs.brk_code, rep->iterations = hs.iterations;
    rep->final_relres = hs.final_relres, rep->true_relres = 0.0;
    rep->history_len = o->record_history ? hs.hl : 0;
    if (!hs.no_true) {  // true_relative_residual (krylov.cpp:17-23)
        double2* od = w + 7 * nv;
        CK(cvk::launch_residual(A->group, false, n, A->rp, A->ci, A->av, b, x, a.tmp, st));
        CK(cvk::launch_dot(false, n, b, nullptr, c->part, od, st));
        CK(cvk::launch_dot(false, n, a.tmp, nullptr, c->part, od + 1, st));
        launches += 5;
        double2 hh[2];
        CK(cudaMemcpyAsync(hh, od, sizeof(hh), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const double bn = std::sqrt(hh[0].x), rn = std::sqrt(hh[1].x);
        rep->true_relres = bn > 0 ? rn / bn : rn;
    }
    if (hcap > 0) {
        const long long k = std::min<long long>(hs.hl, hcap);
        if (k > 0) CK(cudaMemcpy(rep->history, a.hist, sizeof(double) * k, cudaMemcpyDeviceToHost));
    }
    CK(cudaEventRecord(c->e1, st));
    CK(cudaEventSynchronize(c->e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
    rep->device_time_s = ms * 1e-3;
    rep->kernel_launches = launches + nl;
    return CVK_OK;
}

// BiCGSTAB with a general preconditioner (ILU(0)): the reference's operation
// order (krylov.cpp:57-138 = oracle orc_bicgstab) as a host loop of device
// kernels -- SpMV, preconditioner sweeps, axpys and double-double dots --
// with one scalar read-back per dependent reduction (4 per iteration; the
// final ||r|| rides with the next rho).  FAST or REF dots per the mode.
static int solve_bicgstab_general(cvk_ctx* c, const cvk_csr* A, const cvk_prec* M, const cvk_opts* o,
                                  const double2* b, double2* x, cvk_report* rep) {
    const int n = (int)A->n;
    const bool ref = is_ref(resolve_mode(c, o->mode));
    if (!ref && M->ilu && n > 0 && !c->knob.ilu_hostloop) return solve_ilu_chain(c, A, M, o, b, x, rep);
    cudaStream_t st = c->stream;
    int e;
    const size_t nv = (size_t)std::max(1, n);
    if ((e = ensure(c, &c->work, &c->work_bytes, sizeof(double2) * (9 * nv + 8))) != CVK_OK) return e;
    if ((e = ensure(c, (void**)&c->part, &c->part_bytes, sizeof(double2) * 2048)) != CVK_OK) return e;
    double2* w = (double2*)c->work;
    double2 *r = w, *sh = w + nv, *p = w + 2 * nv, *v = w + 3 * nv, *s = w + 4 * nv, *t = w + 5 * nv,
            *tmp = w + 6 * nv, *ptmp = w + 7 * nv, *od = w + 9 * nv;
    long long launches = 0;
    int nl = 0;
    auto dot = [&](const double2* xx, const double2* yy, int slot) -> cudaError_t {
        launches += ref ? 1 : 2;
        return cvk::launch_dot(ref, n, xx, yy, c->part, od + slot, st);
    };
    auto fetch = [&](double2* h, int k) -> cudaError_t {
        cudaError_t ce = cudaMemcpyAsync(h, od, sizeof(double2) * k, cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
        return ce;
    };
    auto op = [&](const double2* in, double2* outv) -> int {  // outv = M^-1 (A in)
        int rc = cvk_spmv_device(A, (const double*)in, (double*)tmp, ref ? CVK_MODE_REF : CVK_MODE_FAST);
        if (rc != CVK_OK) return rc;
        ++launches;
        return prec_apply_dev(M, tmp, outv, ptmp, &nl);
    };
    auto hist = [&](double v) {
        if (o->record_history && rep->history && rep->history_len < rep->history_cap) rep->history[rep->history_len] = v;
        if (o->record_history) rep->history_len++;
    };
    rep->converged = 0, rep->breakdown = CVK_BRK_NONE, rep->iterations = 0, rep->final_relres = 0.0;
    rep->true_relres = 0.0, rep->history_len = 0;
    CK(cudaEventRecord(c->e0, st));
    CK(cudaMemsetAsync(x, 0, sizeof(double2) * nv, st));
    if ((e = prec_apply_dev(M, b, r, ptmp, &nl)) != CVK_OK) return e;
    CK(dot(r, nullptr, 0));
    double2 h[2];
    CK(fetch(h, 1));
    const double bnorm = std::sqrt(h[0].x);
    bool have_true = true;
    if (bnorm == 0.0) {
        rep->converged = 1;
        have_true = false;
    } else {
        const double brk = 1e-30 * bnorm * bnorm;
        CK(cudaMemcpyAsync(sh, r, sizeof(double2) * n, cudaMemcpyDeviceToDevice, st));
        double2 rho = make_double2(1.0, 0.0), alpha = rho, omega = rho;
        for (long long it = 1; it <= o->max_iter; ++it) {
            CK(dot(sh, r, 0));
            CK(fetch(h, 1));
            const double2 rho_new = h[0];
            if (std::hypot(rho_new.x, rho_new.y) < brk) { rep->breakdown = CVK_BRK_RHO; rep->iterations = it - 1; break; }
            if (it == 1) {
                CK(cudaMemcpyAsync(p, r, sizeof(double2) * n, cudaMemcpyDeviceToDevice, st));
            } else {
                const double2 beta = cvk_mul(cvk_cdiv(rho_new, rho), cvk_cdiv(alpha, omega));
                CK(cvk::launch_axpy(n, make_double2(-omega.x, -omega.y), v, p, st));
                CK(cvk::launch_xpay(n, beta, p, r, st));
                launches += 2;
            }
            rho = rho_new;
            if ((e = op(p, v)) != CVK_OK) return e;
            CK(dot(sh, v, 0));
            CK(fetch(h, 1));
            const double2 gamma = h[0];
            if (std::hypot(gamma.x, gamma.y) < brk) { rep->breakdown = CVK_BRK_SHADOW_V; rep->iterations = it - 1; break; }
            alpha = cvk_cdiv(rho, gamma);
            CK(cudaMemcpyAsync(s, r, sizeof(double2) * n, cudaMemcpyDeviceToDevice, st));
            CK(cvk::launch_axpy(n, make_double2(-alpha.x, -alpha.y), v, s, st));
            CK(cvk::launch_axpy(n, alpha, p, x, st));
            launches += 2;
            CK(dot(s, nullptr, 0));
            CK(fetch(h, 1));
            double relres = std::sqrt(h[0].x) / bnorm;
            if (relres <= o->tol) {
                rep->converged = 1, rep->iterations = it, rep->final_relres = relres;
                hist(relres);
                break;
            }
            if ((e = op(s, t)) != CVK_OK) return e;
            CK(dot(t, nullptr, 0));
            CK(dot(t, s, 1));
            CK(fetch(h, 2));
            const double tt = h[0].x;  // <t, t> is real
            if (std::fabs(tt) < brk) { rep->breakdown = CVK_BRK_OMEGA; rep->iterations = it; break; }
            omega = cvk_cdiv(h[1], make_double2(tt, 0.0));
            CK(cvk::launch_axpy(n, omega, s, x, st));
            CK(cudaMemcpyAsync(r, s, sizeof(double2) * n, cudaMemcpyDeviceToDevice, st));
            CK(cvk::launch_axpy(n, make_double2(-omega.x, -omega.y), t, r, st));
            launches += 2;
            CK(dot(r, nullptr, 0));
            CK(fetch(h, 1));
            relres = std::sqrt(h[0].x) / bnorm;
            rep->final_relres = relres;
            rep->iterations = it;
            hist(relres);
            if (relres <= o->tol) { rep->converged = 1; break; }
        }
    }
    if (have_true) {  // true_relative_residual (krylov.cpp:17-23)
        CK(cvk::launch_residual(ref ? 1 : A->group, ref, n, A->rp, A->ci, A->av, b, x, tmp, st));
        CK(dot(b, nullptr, 0));
        CK(dot(tmp, nullptr, 1));
        ++launches;
        CK(fetch(h, 2));
        const double bn = std::sqrt(h[0].x), rn = std::sqrt(h[1].x);
        rep->true_relres = bn > 0 ? rn / bn : rn;
    }
    CK(cudaEventRecord(c->e1, st));
    CK(cudaEventSynchronize(c->e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
    rep->device_time_s = ms * 1e-3;
    rep->kernel_launches = launches + nl;
    return CVK_OK;
}

// Phase-kernel FAST path for large systems (cvk_phased.cu): BiCGSTAB and
// tfQMR.  Init kernel(s) -> graph replays of kIterPerGraph iterations with a
// lazily polled device `done` flag -> (tfQMR x fix-up) -> true residual.
static constexpr int kIterPerGraph = 8;

// Install a freshly captured graph as *exec: update the cached executable in
// place when only kernel parameters changed (new matrix / vector pointers of
// the same shapes -- every jacobi + solve of a reference caller uploads A
// anew), instantiate otherwise.  Consumes `graph`.
static cudaError_t install_graph(cudaGraphExec_t* exec, cudaGraph_t graph) {
    cudaError_t e = cudaSuccess;
    if (*exec) {
        cudaGraphExecUpdateResultInfo info;
        if (cudaGraphExecUpdate(*exec, graph, &info) == cudaSuccess) {
            cudaGraphDestroy(graph);
            return cudaSuccess;
        }
        (void)cudaGetLastError();
        cudaGraphExecDestroy(*exec);
        *exec = nullptr;
    }
    e = cudaGraphInstantiate(exec, graph, 0);
    cudaGraphDestroy(graph);
    return e;
}

// ring depth below which the streamed phases are not used (solve_phased,
// the GMRES Arnoldi SpMV): the tested configuration
constexpr int kStreamMinStages = 4;

// cudaLaunchKernel with the programmatic-stream-serialization attribute (PDL)
static cudaError_t launch_pdl(const void* f, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
#ifdef CVK_NO_PDL  // measurement / debugging builds (tools/variant_build.sh)
    cfg.numAttrs = 0;
#else
    cfg.numAttrs = 1;
#endif
    return cudaLaunchKernelExC(&cfg, f, args);
}

static int solve_phased(cvk_ctx* c, int solver, const cvk_csr* A, const cvk_prec* M, const cvk_opts* o,
                        const double2* b_dev, double2* x_dev, cvk_report* rep) {
    const int n = (int)A->n;
    const int S = A->group;
    // consumer shape of the streamed phases: 4 x 128 rows for matrices with
    // many out-of-chunk gathers per row (FEM-3D), 2 x 224 for the 5-point
    // cavity (cvk_phased_g4.cu); CVK_OPT_STREAM_FLAVOR forces one
    bool g4 = A->n > 0 && (double)A->nnz / (double)A->n > 8.0;
#ifndef CVK_STAGES_MAX
#define CVK_STAGES_MAX 4
#endif
    if (g4) {
        // the 4-group flavor needs a ring stage per group (4) in each SpMV
        // phase of the solver; a matrix too wide for that takes 2 x 224
        int optin0 = 0;
        CK(cudaDeviceGetAttribute(&optin0, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
        const long long avail0 = (long long)optin0 - 8192 - 2 * cvk::kStreamMaxStages * 8 - cvk::kStreamMaxStages * 32;
        const int kv[5] = {5, 5, 7, 8, 2}, kg[5] = {3, 2, 2, 2, 2};
        const int k0 = solver == CVK_BICGSTAB ? 0 : solver == CVK_COCG ? 4 : 2;
        const int k1 = solver == CVK_BICGSTAB ? 1 : solver == CVK_COCG ? 4 : 3;
        for (int k = k0; k <= k1; ++k)
            if (std::min<long long>(CVK_STAGES_MAX, avail0 / (long long)cvk_g4::flavor_stage_bytes(A->capk_g4, kv[k], kg[k])) < 4)
                g4 = false;
    }
    if (c->knob.flavor == 2 || c->knob.flavor == 4) g4 = c->knob.flavor == 4;
    cvk::PhasedKernels K;
    if (g4) cvk_g4::flavor_kernels(&K);
    else cvk::flavor_kernels(&K);
    const int sthreads = g4 ? cvk_g4::flavor_stream_threads() : cvk::flavor_stream_threads();
    const int scapk = g4 ? A->capk_g4 : A->capk;
    auto stage_bytes = [&](int nvec, int ngather) {
        return g4 ? cvk_g4::flavor_stage_bytes(scapk, nvec, ngather) : cvk::flavor_stage_bytes(scapk, nvec, ngather);
    };
    const size_t smem = 0;
    const void* heavy = solver == CVK_BICGSTAB ? K.bi_b : K.tf_e;
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, heavy, cvk::kThreads, smem));
    if (per_sm < 1) per_sm = 1;
    const long long chunks = std::max<long long>(1, ((long long)n + cvk::kThreads - 1) / cvk::kThreads);
    // one 256-row chunk per CTA up to kChunkCtasCap CTAs (hardware scheduling
    // keeps the memory pipes full), grid-stride beyond that
    long long G = std::min<long long>(32LL * per_sm * c->nsm, chunks);
    if (c->knob.max_ctas > 0) G = std::min<long long>(G, c->knob.max_ctas);
    int e;
    if ((e = ensure(c, &c->work, &c->work_bytes, sizeof(double2) * 8 * (size_t)std::max(1, n))) != CVK_OK) return e;
    if ((e = ensure(c, (void**)&c->part, &c->part_bytes, sizeof(double2) * cvk::kRegions * cvk::kMaxSlots * (size_t)G)) != CVK_OK)
        return e;
    const long long hcap = o->record_history ? std::max<long long>(2 * o->max_iter + 8, 16) : 0;
    if (hcap > 0 && (size_t)hcap > c->hist_cap) {
        cudaFree(c->hist);
        c->hist = nullptr;
        c->hist_cap = 0;
        CK(cudaMalloc(&c->hist, sizeof(double) * hcap));
        c->hist_cap = (size_t)hcap;
    }
    cvk::PState hs;
    std::memset(&hs, 0, sizeof(hs));
    hs.tol = o->tol;
    hs.max_iter = o->max_iter;
    hs.record = o->record_history ? 1 : 0;
    hs.hist_cap = hcap;
    if (o->max_iter < 1) hs.max_iter = 0;
    hs.warm = (solver == CVK_BICGSTAB && c->warm_next) ? 1 : 0;
    // streamed (TMA ring) SpMV phases when a 256-row chunk fits >= 2 stages
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
    // per kernel: staged vectors, gathered vectors (k_bi_a_s, k_bi_b_s, k_tf_e_s, k_tf_o_s, k_cg_a_s)
    const int kvec[5] = {5, 5, 7, 8, 2}, kgat[5] = {3, 2, 2, 2, 2};
    auto layout_for = [&](int k, int stg) {
        cvk::StreamLayout L{A->capk, kvec[k], stg};
        L.ngather = kgat[k];
        return L;
    };
    auto stage_bytes_k = [&](int k) { return g4 ? stage_bytes(kvec[k], kgat[k]) : layout_for(k, 1).stage_bytes(); };
    int stg[5];
    for (int k = 0; k < 5; ++k) {
        const long long avail = (long long)optin - 8192 - 2 * cvk::kStreamMaxStages * 8 - cvk::kStreamMaxStages * 32;
        stg[k] = (int)std::min<long long>(CVK_STAGES_MAX, std::max<long long>(0, avail / (long long)stage_bytes_k(k)));  // 4: measured best
    }
    // the ring needs a stage per consumer group (cvk_stream.cuh): 2 groups in
    // the 2 x 224 flavor, 4 in the 4 x 128 one.  Streaming also requires the
    // measured-best depth of 4 (kStreamMinStages): a 3-stage COCG ring
    // faulted intermittently on the B200 (2 of 6 runs at 1M DOF; no
    // sanitizer finding), so shallower rings take the thread-per-row phases.
    const int ngroups = (sthreads - 32) / (g4 ? cvk_g4::flavor_stream_rows() : cvk::flavor_stream_rows());
    const int need = std::max(kStreamMinStages, ngroups);
    const bool streamed = c->knob.stream && A->nnz > 0 &&
                          (solver == CVK_BICGSTAB ? std::min(stg[0], stg[1]) >= need
                           : solver == CVK_COCG   ? stg[4] >= need
                                                  : std::min(stg[2], stg[3]) >= need);
    auto smem_for = [&](int k) {
        return g4 ? cvk_g4::flavor_smem_bytes(scapk, kvec[k], kgat[k], stg[k]) : layout_for(k, stg[k]).smem_bytes();
    };
    const void* sk[10] = {K.bi_a_s, K.bi_b_s, K.tf_e_s, K.tf_o_s, K.cg_a_s, K.bf_a_s, K.bf_b_s, K.cf_a_s,
                          K.tq_e_s, K.tq_o_s};
    if (streamed)
        for (const void* f : sk) CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 8192));
    // BiCGSTAB with the reductions folded by the consuming kernel (k_bf_*)
    const bool fold = streamed && c->knob.bicg_fold;  // BiCGSTAB, COCG, tfQMR
    // elementwise phases: grid-stride, 4 elements per thread per trip
#ifndef CVK_EGRID_MUL
#define CVK_EGRID_MUL 2
#endif
    long long Ge = std::min<long long>((long long)CVK_EGRID_MUL * c->nsm,
                                       std::max<long long>(1, (n + 4LL * cvk::kThreads - 1) / (4LL * cvk::kThreads)));
    if (!streamed) Ge = G;
    const long long Gmax = std::max<long long>(std::max<long long>(G, Ge), c->nsm);
    if ((e = ensure(c, (void**)&c->part, &c->part_bytes, sizeof(double2) * cvk::kRegions * cvk::kMaxSlots * (size_t)Gmax)) != CVK_OK)
        return e;
    double2* udg = streamed ? uniform_dg(c, const_cast<cvk_csr*>(A)) : nullptr;
    std::vector<unsigned char> blob(cvk::phased_args_size());
    {
        // the L2 prefetch window reads A->cmax, which is per 224-row chunk
        const int pf = g4 ? 0 : 2 * cvk::kStreamRows;
        // producers of the partial regions of k_bf_*: 0 = k_bf_c, 1 = k_bf_a_s, 2 = k_bf_b_s
        const int gprod[3] = {(int)Ge, c->nsm, c->nsm};
        (g4 ? cvk_g4::flavor_pack_args : cvk::flavor_pack_args)(
            blob.data(), n, A->rp, A->ci, A->av, g4 ? nullptr : A->cmax, M->dinv, b_dev, x_dev, (double2*)c->work,
            c->part, c->st, c->hist, c->rep, scapk, stg, pf, gprod, udg);
    }
    void* args[] = {blob.data()};
    int parity[2] = {0, 1};
    void* pargs[2][2] = {{blob.data(), &parity[0]}, {blob.data(), &parity[1]}};
    double2* scratch = (double2*)c->work;  // r / first work vector, dead after the loop
    void* targs[] = {blob.data(), &scratch};
    const dim3 grid((unsigned)G), block(cvk::kThreads);
    // graph of kIterPerGraph iterations, cached while the arguments are unchanged
    std::vector<unsigned char> key(blob);
    key.push_back((unsigned char)solver);
    key.push_back((unsigned char)S);
    const unsigned char* gp = (const unsigned char*)&G;
    key.insert(key.end(), gp, gp + sizeof(G));
    key.push_back((unsigned char)(streamed ? 1 : 0));
    key.push_back((unsigned char)(g4 ? 1 : 0));
    key.push_back((unsigned char)(fold ? 1 : 0));
    const unsigned char* gep = (const unsigned char*)&Ge;
    key.insert(key.end(), gep, gep + sizeof(Ge));
    if (!c->gexec || c->gkey != key) {
        // a graph of other kernels (another solver, flavor or fold) is never
        // updated in place, only re-instantiated: cudaGraphExecUpdate accepts
        // a same-shaped graph of different kernels (BiCGSTAB -> tfQMR, 24
        // nodes each), and that path faulted intermittently with 3-stage rings
        const int kind = solver | (S << 4) | ((streamed ? 1 : 0) << 12) | ((g4 ? 1 : 0) << 13) | ((fold ? 1 : 0) << 14);
        if (c->gexec && c->gkind != kind) {
            cudaGraphExecDestroy(c->gexec);
            c->gexec = nullptr;
        }
        c->gkind = kind;
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        const dim3 sgrid((unsigned)c->nsm), sblock((unsigned)sthreads), egrid((unsigned)Ge);
        for (int it = 0; it < kIterPerGraph; ++it) {
            if (solver == CVK_COCG && fold) {  // 2 launches per iteration: A parity 0, B parity 1
                launch_pdl(K.cf_a_s, sgrid, sblock, pargs[0], smem_for(4), c->stream);
                launch_pdl(K.cf_b, egrid, block, pargs[1], 0, c->stream);
            } else if (solver == CVK_COCG) {
                if (streamed) launch_pdl(K.cg_a_s, sgrid, sblock, args, smem_for(4), c->stream);
                else launch_pdl(K.cg_a, grid, block, args, smem, c->stream);
                launch_pdl(K.cg_b, egrid, block, args, 0, c->stream);
            } else if (solver == CVK_BICGSTAB && fold) {  // 3 launches per iteration, parity 0 1 0 | 1 0 1 | ...
                const int p0 = (3 * it) & 1;
                launch_pdl(K.bf_a_s, sgrid, sblock, pargs[p0], smem_for(0), c->stream);
                launch_pdl(K.bf_b_s, sgrid, sblock, pargs[p0 ^ 1], smem_for(1), c->stream);
                launch_pdl(K.bf_c, egrid, block, pargs[p0], 0, c->stream);
            } else if (solver == CVK_BICGSTAB) {
                if (streamed) {
                    launch_pdl(K.bi_a_s, sgrid, sblock, args, smem_for(0), c->stream);
                    launch_pdl(K.bi_b_s, sgrid, sblock, args, smem_for(1), c->stream);
                } else {
                    launch_pdl(K.bi_a, grid, block, args, smem, c->stream);
                    launch_pdl(K.bi_b, grid, block, args, smem, c->stream);
                }
                launch_pdl(K.bi_c, egrid, block, args, 0, c->stream);
            } else if (fold) {  // tfQMR, 3 launches per iteration as k_bf_*
                const int p0 = (3 * it) & 1;
                launch_pdl(K.tq_w, egrid, block, pargs[p0], 0, c->stream);
                launch_pdl(K.tq_e_s, sgrid, sblock, pargs[p0 ^ 1], smem_for(2), c->stream);
                launch_pdl(K.tq_o_s, sgrid, sblock, pargs[p0], smem_for(3), c->stream);
            } else {
                launch_pdl(K.tf_w, egrid, block, args, 0, c->stream);
                if (streamed) {
                    launch_pdl(K.tf_e_s, sgrid, sblock, args, smem_for(2), c->stream);
                    launch_pdl(K.tf_o_s, sgrid, sblock, args, smem_for(3), c->stream);
                } else {
                    launch_pdl(K.tf_e, grid, block, args, smem, c->stream);
                    launch_pdl(K.tf_o, grid, block, args, smem, c->stream);
                }
            }
        }
        CK(cudaGetLastError());
        CK(cudaStreamEndCapture(c->stream, &graph));
        CK(install_graph(&c->gexec, graph));
        c->gkey = key;
    }
    CK(cudaMemcpyAsync(c->st, &hs, sizeof(hs), cudaMemcpyHostToDevice, c->stream));
    CK(cudaEventRecord(c->e0, c->stream));
    if (udg) CK(cvk::launch_uniform_check(n, A->rp, A->ci, A->av, udg, udg + n, c->stream));
    long long launches = 0;
    if (solver == CVK_BICGSTAB || solver == CVK_COCG) {
        CK(launch_pdl(solver == CVK_COCG ? K.cg_init : K.bi_init, grid, block, args, 0, c->stream));
        launches += 1;
        if (fold) {
            CK(launch_pdl(K.bf_init, dim3(1), dim3(1), args, 0, c->stream));
            launches += 1;
        }
    } else {
        CK(launch_pdl(K.tf_init, grid, block, args, 0, c->stream));
        CK(launch_pdl(K.tf_init2, grid, block, args, smem, c->stream));
        if (fold) {
            CK(launch_pdl(K.tq_seed, dim3(1), dim3(1), args, 0, c->stream));
            launches += 1;
        }
        launches += 2;
    }
    long long graphs = 0;
    const long long max_graphs = o->max_iter / kIterPerGraph + 3;
    for (;;) {
        if (graphs >= max_graphs) break;
        CK(cudaGraphLaunch(c->gexec, c->stream));
        const int slot = (int)(graphs & 1);
        CK(cudaMemcpyAsync(&c->h_done[slot], &c->st->done, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaEventRecord(c->ev[slot], c->stream));
        ++graphs;
        launches += (solver == CVK_COCG ? 2 : 3) * kIterPerGraph;
        if (graphs >= 2) {
            const int old = (int)((graphs - 2) & 1);
            CK(cudaEventSynchronize(c->ev[old]));
            if (c->h_done[old]) break;
        }
    }
    if (solver == CVK_TFQMR) {
        CK(launch_pdl(K.tf_fix, grid, block, args, 0, c->stream));
        launches += 1;
    }
    CK(launch_pdl(K.true_res, grid, block, targs, smem, c->stream));
    launches += 1;
    CK(cudaEventRecord(c->e1, c->stream));
    cvk::DevReport dr;
    CK(cudaMemcpyAsync(&dr, c->rep, sizeof(dr), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
    rep->converged = dr.converged;
    rep->breakdown = dr.breakdown;
    rep->iterations = dr.iterations;
    rep->final_relres = dr.final_relres;
    rep->true_relres = dr.true_relres;
    rep->history_len = o->record_history ? dr.history_len : 0;
    rep->device_time_s = ms * 1e-3;
    rep->kernel_launches = launches;
    if (o->record_history && rep->history && rep->history_cap > 0) {
        const long long k = std::min<long long>(std::min<long long>(rep->history_len, rep->history_cap), hcap);
        if (k > 0) CK(cudaMemcpy(rep->history, c->hist, sizeof(double) * k, cudaMemcpyDeviceToHost));
    }
    return CVK_OK;
}

static int solve_gmres_phased(cvk_ctx* c, const cvk_csr* A, const cvk_prec* M, const cvk_opts* o,
                              const double2* b_dev, double2* x_dev, cvk_report* rep) {
    const int n = (int)A->n;
    const int m = (int)o->m;
    const cvk::GmresKernels K = cvk::gmres_kernels();
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, K.dd, cvk::kThreads, 0));
    const long long blocks = std::max<long long>(1, ((long long)n + cvk::kThreads - 1) / cvk::kThreads);
    long long G = std::min<long long>(std::max(1, per_sm) * (long long)c->nsm, blocks);
    int e;
    const size_t npad = (size_t)cvk::gmres_padded_rows(std::max(1, n));
    if ((e = ensure(c, &c->work, &c->work_bytes, sizeof(double2) * (size_t)(m + 4) * npad)) != CVK_OK) return e;
    // partials of the G-CTA kernels and of the one-CTA-per-SM streamed ones
    if ((e = ensure(c, (void**)&c->part, &c->part_bytes,
                    sizeof(double2) * cvk::kRegions * cvk::kMaxSlots * (size_t)std::max<long long>(G, c->nsm))) != CVK_OK)
        return e;
    if (!c->gst) CK(cudaMalloc(&c->gst, cvk::gmres_state_size()));
    const long long hcap = o->record_history ? std::max<long long>(2 * o->max_iter + 8, 16) : 0;
    if (hcap > 0 && (size_t)hcap > c->hist_cap) {
        cudaFree(c->hist);
        c->hist = nullptr;
        c->hist_cap = 0;
        CK(cudaMalloc(&c->hist, sizeof(double) * hcap));
        c->hist_cap = (size_t)hcap;
    }
    std::vector<unsigned char> hs(cvk::gmres_state_size(), 0);
    cvk::gmres_init_state(hs.data(), o->tol, o->max_iter < 1 ? 0 : o->max_iter, m, o->record_history ? 1 : 0, hcap);
    // Arnoldi SpMV on the TMA ring when a chunk fits >= 2 stages (as the
    // BiCGSTAB / tfQMR phase kernels; CVK_NO_STREAM=1 keeps thread per row)
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
    cvk::StreamLayout SL{A->capk, 2, 1};
    SL.ngather = 1;
    const long long avail = (long long)optin - 8192 - 2 * cvk::kStreamMaxStages * 8 - cvk::kStreamMaxStages * 32;
    int nst = (int)std::min<long long>(4, std::max<long long>(0, avail / (long long)SL.stage_bytes()));
    if (nst < kStreamMinStages || A->nnz == 0 || !c->knob.stream) nst = 0;
    SL.stages = std::max(1, nst);
    if (nst) CK(cudaFuncSetAttribute(K.spmv_s, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 8192));
    // the basis passes on bulk-copied tiles of the m + 1 vectors (k_g_dd_s /
    // k_g_up_s): at least 2 stages of (m + 1) 128-row vectors
    int tile_smem = optin - 8192 - 4096;
    const int stage_max = cvk::gmres_tile_stage_max(m);
    const bool tiles = c->knob.stream && A->nnz > 0 && m <= 32 && (long long)tile_smem >= 2LL * stage_max + 256 &&
                       c->knob.gmres_tiles;
    if (tiles) {
        CK(cudaFuncSetAttribute(K.dd_s, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem));
        CK(cudaFuncSetAttribute(K.up_s, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem));
    }
    const int pf = 2 * cvk::kStreamRows;
    std::vector<unsigned char> blob(cvk::gmres_args_size());
    double2* udg = nst ? uniform_dg(c, const_cast<cvk_csr*>(A)) : nullptr;
    cvk::gmres_pack_args(blob.data(), cvk::Csr{n, A->rp, A->ci, A->av, A->cmax, udg, udg ? udg + n : nullptr}, M->dinv, b_dev, x_dev,
                         (double2*)c->work, c->part, c->gst, c->hist, c->rep, A->capk, nst, pf, m);
    void* args[] = {blob.data()};
    void* targs[] = {blob.data(), &tile_smem};
    const dim3 grid((unsigned)G), block(cvk::kThreads);
    std::vector<unsigned char> key(blob);
    const unsigned char* gp = (const unsigned char*)&G;
    key.insert(key.end(), gp, gp + sizeof(G));
    key.push_back((unsigned char)(tiles ? 1 : 0));
    if (!c->gm_exec || c->gm_key != key) {
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        for (int it = 0; it < kIterPerGraph; ++it) {
            launch_pdl(K.x, grid, block, args, 0, c->stream);
            launch_pdl(K.spmv, grid, block, args, 0, c->stream);
            if (nst) launch_pdl(K.spmv_s, dim3((unsigned)c->nsm), dim3(cvk::kStreamThreads), args, SL.smem_bytes(), c->stream);
            if (tiles) {
                const dim3 tg((unsigned)c->nsm);
                launch_pdl(K.dd_s, tg, dim3(cvk::kGmresDdsThreads), targs, (size_t)tile_smem, c->stream);
                launch_pdl(K.up_s, tg, dim3(cvk::kGmresUpsThreads), targs, (size_t)tile_smem, c->stream);
            } else {
                launch_pdl(K.dd, grid, block, args, 0, c->stream);
                launch_pdl(K.up, grid, block, args, 0, c->stream);
            }
        }
        CK(cudaGetLastError());
        CK(cudaStreamEndCapture(c->stream, &graph));
        CK(install_graph(&c->gm_exec, graph));
        c->gm_key = key;
    }
    CK(cudaMemcpyAsync(c->gst, hs.data(), hs.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaEventRecord(c->e0, c->stream));
    if (udg) CK(cvk::launch_uniform_check(n, A->rp, A->ci, A->av, udg, udg + n, c->stream));
    CK(launch_pdl(K.init, grid, block, args, 0, c->stream));
    long long launches = 1;
    const int* done_ptr = (const int*)((const char*)c->gst + cvk::gmres_state_done_offset());
    // one Arnoldi step per slot, plus two slots per restart
    const long long max_graphs = (o->max_iter + 2 * (o->max_iter / std::max(1, m) + 1)) / kIterPerGraph + 3;
    long long graphs = 0;
    for (;;) {
        if (graphs >= max_graphs) break;
        CK(cudaGraphLaunch(c->gm_exec, c->stream));
        const int slot = (int)(graphs & 1);
        CK(cudaMemcpyAsync(&c->h_done[slot], done_ptr, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaEventRecord(c->ev[slot], c->stream));
        ++graphs;
        launches += (nst ? 5 : 4) * kIterPerGraph;
        if (graphs >= 2) {
            const int old = (int)((graphs - 2) & 1);
            CK(cudaEventSynchronize(c->ev[old]));
            if (c->h_done[old]) break;
        }
    }
    CK(launch_pdl(K.true_res, grid, block, args, 0, c->stream));
    launches += 1;
    CK(cudaEventRecord(c->e1, c->stream));
    DevReport dr;
    CK(cudaMemcpyAsync(&dr, c->rep, sizeof(dr), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
    rep->converged = dr.converged;
    rep->breakdown = dr.breakdown;
    rep->iterations = dr.iterations;
    rep->final_relres = dr.final_relres;
    rep->true_relres = dr.true_relres;
    rep->history_len = o->record_history ? dr.history_len : 0;
    rep->device_time_s = ms * 1e-3;
    rep->kernel_launches = launches;
    if (o->record_history && rep->history && rep->history_cap > 0) {
        const long long k = std::min<long long>(std::min<long long>(rep->history_len, rep->history_cap), hcap);
        if (k > 0) CK(cudaMemcpy(rep->history, c->hist, sizeof(double) * k, cudaMemcpyDeviceToHost));
    }
    return CVK_OK;
}

// Phase-kernel BiCGSTAB(l) (cvk_bicgl.cu): N identical step launches per graph.
static int solve_bicgl_phased(cvk_ctx* c, const cvk_csr* A, const cvk_prec* M, const cvk_opts* o,
                              const double2* b_dev, double2* x_dev, cvk_report* rep) {
    const int n = (int)A->n;
    const int L = (int)o->l;
    const cvk::BiclKernels K = cvk::bicgl_kernels();
    // grid per kernel: its resident CTAs (the phases are grid-stride)
    const long long chunks = std::max<long long>(1, ((long long)n + cvk::kThreads - 1) / cvk::kThreads);
    auto grid_of = [&](const void* f) -> long long {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, cvk::kThreads, 0);
        return std::min<long long>(std::max(1, per_sm) * (long long)c->nsm, chunks);
    };
    const long long Gu = grid_of(K.u), Gr = grid_of(K.r), Gm = grid_of(K.mgs), Gq = grid_of(K.mgsr),
                    Gp = grid_of(K.upd), Gx = grid_of(K.exit);
    const long long G = std::max(std::max(std::max(Gu, Gr), std::max(Gm, Gp)), std::max(Gx, Gq));
    int e;
    if ((e = ensure(c, &c->work, &c->work_bytes, sizeof(double2) * (size_t)(2 * L + 6) * std::max(1, n))) != CVK_OK)
        return e;
    if ((e = ensure(c, (void**)&c->part, &c->part_bytes, sizeof(double2) * cvk::kRegions * cvk::kMaxSlots * (size_t)G)) != CVK_OK)
        return e;
    if (!c->bst) CK(cudaMalloc(&c->bst, cvk::bicgl_state_size()));
    const long long hcap = o->record_history ? std::max<long long>(2 * o->max_iter + 8, 16) : 0;
    if (hcap > 0 && (size_t)hcap > c->hist_cap) {
        cudaFree(c->hist);
        c->hist = nullptr;
        c->hist_cap = 0;
        CK(cudaMalloc(&c->hist, sizeof(double) * hcap));
        c->hist_cap = (size_t)hcap;
    }
    std::vector<unsigned char> hs(cvk::bicgl_state_size(), 0);
    cvk::bicgl_init_state(hs.data(), o->tol, o->max_iter < 1 ? 0 : o->max_iter, L, o->record_history ? 1 : 0, hcap);
    std::vector<unsigned char> blob(cvk::bicgl_args_size());
    cvk::bicgl_pack_args(blob.data(), cvk::Csr{n, A->rp, A->ci, A->av}, M->dinv, b_dev, x_dev, (double2*)c->work,
                         c->part, c->bst, c->hist, c->rep);
    void* args[] = {blob.data()};
    const dim3 grid((unsigned)G), block(cvk::kThreads);
    // one graph = one cycle's static phase sequence (cvk_bicgl.cu)
    const long long per_cycle = 2LL * L + (L <= cvk::kBiclMgsrL ? L : (long long)L * (L + 1) / 2) + 2;
    std::vector<unsigned char> key(blob);
    const unsigned char* gp = (const unsigned char*)&G;
    key.insert(key.end(), gp, gp + sizeof(G));
    key.push_back((unsigned char)L);
    if (!c->bl_exec || c->bl_key != key) {
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        for (int j = 0; j < L; ++j) {
            launch_pdl(K.u, dim3((unsigned)Gu), block, args, 0, c->stream);
            launch_pdl(K.r, dim3((unsigned)Gr), block, args, 0, c->stream);
        }
        if (L <= cvk::kBiclMgsrL)
            for (int q = 0; q < L; ++q)  // slices of kBiclMgsrW columns (cvk_bicgl.cu k_bl_mgsr)
                launch_pdl(K.mgsr, dim3((unsigned)Gq, (unsigned)((L - q + cvk::kBiclMgsrW - 1) / cvk::kBiclMgsrW)), block,
                           args, 0, c->stream);
        else
            for (int q = 0; q < L * (L + 1) / 2; ++q) launch_pdl(K.mgs, dim3((unsigned)Gm), block, args, 0, c->stream);
        launch_pdl(K.upd, dim3((unsigned)Gp), block, args, 0, c->stream);
        launch_pdl(K.exit, dim3((unsigned)Gx), block, args, 0, c->stream);
        CK(cudaGetLastError());
        CK(cudaStreamEndCapture(c->stream, &graph));
        CK(install_graph(&c->bl_exec, graph));
        c->bl_key = key;
    }
    CK(cudaMemcpyAsync(c->bst, hs.data(), hs.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaEventRecord(c->e0, c->stream));
    CK(launch_pdl(K.init, grid, block, args, 0, c->stream));
    long long launches = 1;
    const int* done_ptr = (const int*)((const char*)c->bst + cvk::bicgl_state_done_offset());
    const long long max_graphs = std::max<long long>(1, o->max_iter) + 3;
    long long graphs = 0;
    for (;;) {
        if (graphs >= max_graphs) break;
        CK(cudaGraphLaunch(c->bl_exec, c->stream));
        const int slot = (int)(graphs & 1);
        CK(cudaMemcpyAsync(&c->h_done[slot], done_ptr, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaEventRecord(c->ev[slot], c->stream));
        ++graphs;
        launches += per_cycle;
        if (graphs >= 2) {
            const int old = (int)((graphs - 2) & 1);
            CK(cudaEventSynchronize(c->ev[old]));
            if (c->h_done[old]) break;
        }
    }
    CK(launch_pdl(K.true_res, grid, block, args, 0, c->stream));
    launches += 1;
    CK(cudaEventRecord(c->e1, c->stream));
    DevReport dr;
    CK(cudaMemcpyAsync(&dr, c->rep, sizeof(dr), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
    rep->converged = dr.converged;
    rep->breakdown = dr.breakdown;
    rep->iterations = dr.iterations;
    rep->final_relres = dr.final_relres;
    rep->true_relres = dr.true_relres;
    rep->history_len = o->record_history ? dr.history_len : 0;
    rep->device_time_s = ms * 1e-3;
    rep->kernel_launches = launches;
    if (o->record_history && rep->history && rep->history_cap > 0) {
        const long long k = std::min<long long>(std::min<long long>(rep->history_len, rep->history_cap), hcap);
        if (k > 0) CK(cudaMemcpy(rep->history, c->hist, sizeof(double) * k, cudaMemcpyDeviceToHost));
    }
    return CVK_OK;
}

static int solve_impl(cvk_ctx* c, int solver, const cvk_csr* A, const cvk_prec* M, const cvk_opts* o,
                      const double2* b_dev, double2* x_dev, cvk_report* rep) {
    if (solver < 0 || solver > 4)
        return fail(CVK_ESOLVER, "unknown solver id " + std::to_string(solver) +
                                     " (allowed: bicgstab, bicgstab_l, tfqmr, gmres, cocg)");
    const char* nm = kSolverNames[solver];
    if (!A || !M || !o || !rep) return fail(CVK_EINVAL, std::string(nm) + ": null argument");
    if (M->n != A->n) return fail(CVK_EINVAL, std::string(nm) + ": dimension mismatch");
    if (solver == CVK_BICGSTAB_L && o->l < 1) return fail(CVK_EINVAL, "bicgstab_l: l must be >= 1");
    if (solver == CVK_BICGSTAB_L && o->l > cvk::kMaxL)
        return fail(CVK_EINVAL, "bicgstab_l: l exceeds the device limit of 16");
    if (solver == CVK_GMRES && (o->m < 1 || o->m > cvk::kMaxDots))
        return fail(CVK_EINVAL, "gmres: m must be in [1, 64]");
    if (o->max_iter < 0) return fail(CVK_EINVAL, std::string(nm) + ": negative max_iter");
    if (M->ilu) {
        if (solver != CVK_BICGSTAB || c->warm_next)
            return fail(CVK_EINVAL, std::string(nm) + ": the ILU(0) preconditioner supports bicgstab (cold start) only");
        CK(cudaSetDevice(c->device));
        return solve_bicgstab_general(c, A, M, o, b_dev, x_dev, rep);
    }
    const int n = (int)A->n;
    const int mode = resolve_mode(c, o->mode);
    const bool ref = is_ref(mode);
    CK(cudaSetDevice(c->device));
    const long long pmin = c->knob.phased_min_n;
    // GMRES phase kernels from 32k rows (50k DOF: 58 vs 63 us per step; BiCGSTAB keeps the persistent kernel there)
    if (!ref && solver == CVK_GMRES && (long long)n >= std::min(pmin, 32768LL) && !c->knob.gmres_persistent)
        return solve_gmres_phased(c, A, M, o, b_dev, x_dev, rep);
    // BiCGSTAB(l) step kernel from 131072 rows (1M DOF, l = 8: 2293 vs 2380 us
    // per cycle on the cavity, 3007 vs 3085 on 3-D FEM)
    if (!ref && solver == CVK_BICGSTAB_L && (long long)n >= pmin && !c->knob.bicgl_persistent)
        return solve_bicgl_phased(c, A, M, o, b_dev, x_dev, rep);
    if (!ref && (solver == CVK_BICGSTAB || solver == CVK_TFQMR || solver == CVK_COCG) && (long long)n >= pmin)
        return solve_phased(c, solver, A, M, o, b_dev, x_dev, rep);
    const int S = ref ? 1 : A->group;
    const void* kern = cvk::solver_kernel(solver, S, ref);
    if (!kern) return fail(CVK_ELOGIC, "no kernel for this configuration");
    const size_t smem = cvk::solver_smem(solver, (int)o->m);
    if (smem > 0) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, cvk::kThreads, smem));
    if (per_sm < 1) return fail(CVK_ECUDA, "solver kernel does not fit on an SM");
    const long long chunks = std::max<long long>(1, ((long long)n + cvk::kThreads - 1) / cvk::kThreads);
    long long G = std::min<long long>((long long)per_sm * c->nsm, chunks);
    if (c->knob.max_ctas > 0) G = std::min<long long>(G, c->knob.max_ctas);
    const int nwork = cvk::solver_nwork(solver, (int)o->l, (int)o->m);
    CK(cudaSetDevice(c->device));
    int e;
    if ((e = ensure(c, &c->work, &c->work_bytes, sizeof(double2) * (size_t)nwork * std::max(1, n))) != CVK_OK)
        return e;
    if ((e = ensure(c, (void**)&c->part, &c->part_bytes, sizeof(double2) * cvk::kRegions * cvk::kMaxSlots * (size_t)G)) != CVK_OK)
        return e;
    const long long hcap = o->record_history ? std::max<long long>(2 * o->max_iter + 8, 16) : 0;
    if (hcap > 0 && (size_t)hcap > c->hist_cap) {
        cudaFree(c->hist);
        c->hist = nullptr;
        c->hist_cap = 0;
        CK(cudaMalloc(&c->hist, sizeof(double) * hcap));
        c->hist_cap = (size_t)hcap;
    }
    CK(cudaMemsetAsync(c->bar, 0, 2 * sizeof(unsigned long long), c->stream));
    cvk::KArgs a;
    a.A = cvk::Csr{n, A->rp, A->ci, A->av};
    a.dinv = M->dinv;
    a.b = b_dev;
    a.x = x_dev;
    a.work = (double2*)c->work;
    a.part = c->part;
    a.bar = c->bar;
    a.rep = c->rep;
    a.hist = c->hist;
    a.hist_cap = hcap;
    a.tol = o->tol;
    a.max_iter = o->max_iter;
    a.l = (int)o->l;
    a.m = (int)o->m;
    a.record = o->record_history ? 1 : 0;
    a.G = (int)G;
    a.cta_base = 0;
    a.warm = (solver == CVK_BICGSTAB && c->warm_next) ? 1 : 0;
    a.refpar = mode == CVK_MODE_REF_PAR ? 1 : 0;
    void* args[] = {&a};
    CK(cudaEventRecord(c->e0, c->stream));
    CK(cudaLaunchCooperativeKernel(kern, dim3((unsigned)G), dim3(cvk::kThreads), args, smem, c->stream));
    CK(cudaEventRecord(c->e1, c->stream));
    DevReport dr;
    CK(cudaMemcpyAsync(&dr, c->rep, sizeof(dr), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
    if (dr.error) return fail(CVK_ETIMEOUT, std::string(nm) + ": device grid barrier aborted");
    rep->converged = dr.converged;
    rep->breakdown = dr.breakdown;
    rep->iterations = dr.iterations;
    rep->final_relres = dr.final_relres;
    rep->true_relres = dr.true_relres;
    rep->history_len = o->record_history ? dr.history_len : 0;
    rep->device_time_s = ms * 1e-3;
    rep->kernel_launches = 1;
    if (o->record_history && rep->history && rep->history_cap > 0) {
        const long long k = std::min<long long>(std::min<long long>(rep->history_len, rep->history_cap), hcap);
        if (k > 0) CK(cudaMemcpy(rep->history, c->hist, sizeof(double) * k, cudaMemcpyDeviceToHost));
    }
    return CVK_OK;
}

int cvk_solve_device(cvk_ctx* c, int solver, const cvk_csr* A, const cvk_prec* M, const cvk_opts* o,
                     const double* b_dev, double* x_dev, cvk_report* rep) {
    if (!c) return fail(CVK_EINVAL, "null ctx");
    const double t0 = now_s();
    const int e = solve_impl(c, solver, A, M, o, (const double2*)b_dev, (double2*)x_dev, rep);
    if (e == CVK_OK) rep->wall_time_s = now_s() - t0;
    return e;
}

int cvk_solve_device_warm(cvk_ctx* c, const cvk_csr* A, const cvk_prec* M, const cvk_opts* o, const double* b_dev,
                          double* x_dev, cvk_report* rep) {
    if (!c) return fail(CVK_EINVAL, "null ctx");
    c->warm_next = 1;
    const int e = cvk_solve_device(c, CVK_BICGSTAB, A, M, o, b_dev, x_dev, rep);
    c->warm_next = 0;
    return e;
}

int cvk_solve(cvk_ctx* c, int solver, const cvk_csr* A, const cvk_prec* M, const cvk_opts* o,
              const double* b, double* x, cvk_report* rep) {
    if (!c || !A || !b || !x) return fail(CVK_EINVAL, "cvk_solve: null argument");
    const double t0 = now_s();
    CK(cudaSetDevice(c->device));
    const size_t n = (size_t)A->n;
    size_t have = c->bx_n * 2 * sizeof(double2);
    int e;
    if ((e = ensure(c, (void**)&c->bx, &have, 2 * sizeof(double2) * std::max<size_t>(1, n))) != CVK_OK) return e;
    c->bx_n = have / (2 * sizeof(double2));
    double2* bd = c->bx;
    double2* xd = c->bx + c->bx_n;
    CK(cudaMemcpyAsync(bd, b, sizeof(double2) * n, cudaMemcpyHostToDevice, c->stream));
    e = solve_impl(c, solver, A, M, o, bd, xd, rep);
    if (e != CVK_OK) return e;
    CK(cudaMemcpyAsync(x, xd, sizeof(double2) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    rep->wall_time_s = now_s() - t0;
    return CVK_OK;
}

// ----------------------------------------------------------------- kernels

static int stage(cvk_ctx* c, size_t n2) {
    size_t have = c->bx_n * 2 * sizeof(double2);
    int e = ensure(c, (void**)&c->bx, &have, std::max<size_t>(2 * sizeof(double2), n2 * sizeof(double2)));
    if (e == CVK_OK) c->bx_n = have / (2 * sizeof(double2));
    return e;
}

int cvk_spmv_device(const cvk_csr* A, const double* x_dev, double* y_dev, int mode) {
    if (!A) return fail(CVK_EINVAL, "spmv: null matrix");
    cvk_ctx* c = A->ctx;
    const bool ref = is_ref(resolve_mode(c, mode));
    CK(cudaSetDevice(c->device));
    if (!ref && A->n >= 4 * cvk::kStreamRows && A->nnz > 0 && c->knob.stream) {
        int optin = 0;
        CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
        const cudaError_t e = cvk::launch_spmv_stream((int)A->n, A->rp, A->ci, A->av, (const double2*)x_dev,
                                                      (double2*)y_dev, A->capk, c->nsm, optin, c->stream);
        if (e == cudaSuccess) return CVK_OK;
        if (e != cudaErrorInvalidConfiguration) CK(e);
        (void)cudaGetLastError();
    }
    CK(cvk::launch_spmv(ref ? 1 : A->group, ref, (int)A->n, A->rp, A->ci, A->av, (const double2*)x_dev,
                        (double2*)y_dev, 0, c->stream));
    return CVK_OK;
}

int cvk_spmv(const cvk_csr* A, const double* x, double* y, int mode) {
    if (!A || !x || !y) return fail(CVK_EINVAL, "spmv: null argument");
    cvk_ctx* c = A->ctx;
    CK(cudaSetDevice(c->device));
    const size_t n = (size_t)A->n;
    int e;
    if ((e = stage(c, 2 * n)) != CVK_OK) return e;
    double2* xd = c->bx;
    double2* yd = c->bx + n;
    CK(cudaMemcpyAsync(xd, x, sizeof(double2) * n, cudaMemcpyHostToDevice, c->stream));
    if ((e = cvk_spmv_device(A, (const double*)xd, (double*)yd, mode)) != CVK_OK) return e;
    CK(cudaMemcpyAsync(y, yd, sizeof(double2) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return CVK_OK;
}

int cvk_spmv_bench(const cvk_csr* A, const double* x_dev, double* y_dev, int mode, int reps, double* avg_s) {
    if (!A || !avg_s || reps < 1) return fail(CVK_EINVAL, "spmv_bench: bad argument");
    cvk_ctx* c = A->ctx;
    CK(cudaSetDevice(c->device));
    int e;
    if ((e = cvk_spmv_device(A, x_dev, y_dev, mode)) != CVK_OK) return e;  // warm-up
    CK(cudaEventRecord(c->e0, c->stream));
    for (int r = 0; r < reps; ++r)
        if ((e = cvk_spmv_device(A, x_dev, y_dev, mode)) != CVK_OK) return e;
    CK(cudaEventRecord(c->e1, c->stream));
    CK(cudaEventSynchronize(c->e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
    *avg_s = (double)ms * 1e-3 / reps;
    return CVK_OK;
}

static int dot_impl(cvk_ctx* c, int64_t n, const double* x, const double* y, double* out, int mode) {
    if (!c || !x || !out || n < 0) return fail(CVK_EINVAL, "dot: bad argument");
    CK(cudaSetDevice(c->device));
    const bool ref = is_ref(resolve_mode(c, mode));
    const size_t nn = (size_t)n;
    int e;
    if ((e = stage(c, 2 * nn + 2)) != CVK_OK) return e;
    double2* xd = c->bx;
    double2* yd = y ? c->bx + nn : nullptr;
    double2* od = c->bx + 2 * nn;
    if ((e = ensure(c, (void**)&c->part, &c->part_bytes, sizeof(double2) * 2048)) != CVK_OK) return e;
    if (nn) CK(cudaMemcpyAsync(xd, x, sizeof(double2) * nn, cudaMemcpyHostToDevice, c->stream));
    if (y && nn) CK(cudaMemcpyAsync(yd, y, sizeof(double2) * nn, cudaMemcpyHostToDevice, c->stream));
    CK(cvk::launch_dot(ref, (int)n, xd, yd, c->part, od, c->stream));
    CK(cudaMemcpyAsync(out, od, sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return CVK_OK;
}

int cvk_dot(cvk_ctx* c, int64_t n, const double* x, const double* y, double* out, int mode) {
    if (!y) return fail(CVK_EINVAL, "dot_hermitian: null argument");
    return dot_impl(c, n, x, y, out, mode);
}

int cvk_norm2(cvk_ctx* c, int64_t n, const double* x, double* out, int mode) {
    double tmp[2];
    const int e = dot_impl(c, n, x, nullptr, tmp, mode);
    if (e == CVK_OK) *out = std::sqrt(tmp[0]);
    return e;
}

static int axpy_like(cvk_ctx* c, int64_t n, const double* alpha, const double* x, double* y, bool xpay) {
    if (!c || !alpha || !x || !y || n < 0) return fail(CVK_EINVAL, "axpy: bad argument");
    CK(cudaSetDevice(c->device));
    const size_t nn = (size_t)n;
    int e;
    if ((e = stage(c, 2 * nn)) != CVK_OK) return e;
    double2* xd = c->bx;
    double2* yd = c->bx + nn;
    const double2 al = make_double2(alpha[0], alpha[1]);
    if (nn) {
        CK(cudaMemcpyAsync(xd, x, sizeof(double2) * nn, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(yd, y, sizeof(double2) * nn, cudaMemcpyHostToDevice, c->stream));
    }
    if (xpay) {
        // x = alpha x + y: result lands in xd, copied back into the caller's x (passed as y here)
        CK(cvk::launch_xpay((int)n, al, xd, yd, c->stream));
        if (nn) CK(cudaMemcpyAsync(y, xd, sizeof(double2) * nn, cudaMemcpyDeviceToHost, c->stream));
    } else {
        CK(cvk::launch_axpy((int)n, al, xd, yd, c->stream));
        if (nn) CK(cudaMemcpyAsync(y, yd, sizeof(double2) * nn, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return CVK_OK;
}

int cvk_axpy(cvk_ctx* c, int64_t n, const double* alpha, const double* x, double* y) {
    return axpy_like(c, n, alpha, x, y, false);
}

int cvk_xpay(cvk_ctx* c, int64_t n, const double* alpha, double* x, const double* y) {
    // axpy_like(xpay) reads "x" from its x argument and "y" from its y argument
    // and writes the result into its y argument: route x there.
    if (!c || !alpha || !x || !y || n < 0) return fail(CVK_EINVAL, "xpay: bad argument");
    CK(cudaSetDevice(c->device));
    const size_t nn = (size_t)n;
    int e;
    if ((e = stage(c, 2 * nn)) != CVK_OK) return e;
    double2* xd = c->bx;
    double2* yd = c->bx + nn;
    if (nn) {
        CK(cudaMemcpyAsync(xd, x, sizeof(double2) * nn, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(yd, y, sizeof(double2) * nn, cudaMemcpyHostToDevice, c->stream));
    }
    CK(cvk::launch_xpay((int)n, make_double2(alpha[0], alpha[1]), xd, yd, c->stream));
    if (nn) CK(cudaMemcpyAsync(x, xd, sizeof(double2) * nn, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return CVK_OK;
}

int cvk_true_relres(const cvk_csr* A, const double* b, const double* x, double* out, int mode) {
    if (!A || !b || !x || !out) return fail(CVK_EINVAL, "true_relres: null argument");
    cvk_ctx* c = A->ctx;
    CK(cudaSetDevice(c->device));
    const size_t n = (size_t)A->n;
    int e;
    if ((e = stage(c, 3 * n + 2)) != CVK_OK) return e;
    double2* bd = c->bx;
    double2* xd = c->bx + n;
    double2* rd = c->bx + 2 * n;
    double2* od = c->bx + 3 * n;
    const bool ref = is_ref(resolve_mode(c, mode));
    if ((e = ensure(c, (void**)&c->part, &c->part_bytes, sizeof(double2) * 2048)) != CVK_OK) return e;
    CK(cudaMemcpyAsync(bd, b, sizeof(double2) * n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(xd, x, sizeof(double2) * n, cudaMemcpyHostToDevice, c->stream));
    CK(cvk::launch_residual(ref ? 1 : A->group, ref, (int)n, A->rp, A->ci, A->av, bd, xd, rd, c->stream));
    CK(cvk::launch_dot(ref, (int)n, bd, nullptr, c->part, od, c->stream));
    CK(cvk::launch_dot(ref, (int)n, rd, nullptr, c->part, od + 1, c->stream));
    double2 h[2];
    CK(cudaMemcpyAsync(h, od, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const double bn = std::sqrt(h[0].x), rn = std::sqrt(h[1].x);
    *out = bn > 0 ? rn / bn : rn;
    return CVK_OK;
}

}  // extern "C"

// ------------------------------------------------- DDM support (cvk_ddm.cu)

extern "C" void* cvk_ddm_stream(cvk_ctx* c) { return c->stream; }

extern "C" int cvk_ddm_ctas(cvk_ctx* c, int solver, int mode, size_t smem, int* total) {
    const void* k = cvk::solver_kernel(solver, 1, is_ref(mode), true);
    if (!k) return fail(CVK_ELOGIC, "no batched kernel");
    CK(cudaSetDevice(c->device));
    if (smem > 0) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, cvk::kThreads, smem));
    *total = per_sm * c->nsm;
    return CVK_OK;
}

extern "C" int cvk_ddm_launch_batched(cvk_ctx* c, int solver, int mode, const void* segs, int nseg,
                                      int total_ctas, size_t smem, float* ms) {
    const void* k = cvk::solver_kernel(solver, 1, is_ref(mode), true);
    void* args[] = {(void*)&segs, &nseg};
    CK(cudaLaunchCooperativeKernel(k, dim3((unsigned)total_ctas), dim3(cvk::kThreads), args, smem, c->stream));
    (void)ms;
    return CVK_OK;
}

extern "C" int cvk_ddm_single(cvk_ctx* c, int64_t n, int64_t nnz, const uint64_t* rp, const uint64_t* ci,
                              const double* v, const double* b, const cvk_opts* inner, int solver, double* x,
                              cvk_report* rep) {
    cvk_csr* A = nullptr;
    int e = cvk_csr_upload(c, n, n, nnz, rp, ci, v, &A);
    if (e != CVK_OK) return e;
    cvk_prec* M = nullptr;
    e = cvk_precond_jacobi(A, nullptr, &M);
    if (e == CVK_OK) e = cvk_solve(c, solver, A, M, inner, b, x, rep);
    cvk_precond_free(M);
    cvk_csr_free(A);
    return e;
}
