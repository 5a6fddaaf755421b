// capi.cu -- the extern "C" boundary (include/samg_b200.h).
//
// Every entry point validates its arguments on the host first (so the
// reference's typed errors surface without touching a GPU), then checks for
// a CUDA device (SAMG_NO_DEVICE otherwise: there is no CPU fallback), then
// runs on the handle's device and stream.  Exceptions become status codes
// plus a thread-local message.
#include <chrono>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "hierarchy.cuh"
#include "problem.cuh"
#include "dist.cuh"

struct samg_bsr3 {
    samgb::Bsr3 own;
    const samgb::Bsr3 *m = nullptr;
    int device = 0;
    samgb::DevBuf<double> xs, ys;  // e2e staging for host-vector spmv
    // batched host-vector spmv: one stream per engine (H2D copies, kernels,
    // D2H copies) over kPipe staging slots, ordered by events only where a
    // slot is reused, so both copy directions stream back to back
    static constexpr int kPipe = 4;
    cudaStream_t bs[3] = {nullptr, nullptr, nullptr};  // h2d, kernel, d2h
    cudaEvent_t ev_h[kPipe] = {}, ev_k[kPipe] = {}, ev_d[kPipe] = {};
    samgb::DevBuf<double> bx[kPipe], by[kPipe];
    ~samg_bsr3() {
        // the staging buffers are stream-ordered on bs[1]: free them first
        for (cudaStream_t &q : bs)
            if (q) cudaStreamSynchronize(q);
        for (int b = 0; b < kPipe; ++b) {
            bx[b].release();
            by[b].release();
            for (cudaEvent_t e : {ev_h[b], ev_k[b], ev_d[b]})
                if (e) cudaEventDestroy(e);
        }
        for (cudaStream_t &q : bs)
            if (q) { cudaStreamSynchronize(q); cudaStreamDestroy(q); }
    }
};

struct samg_hierarchy {
    std::unique_ptr<samgb::Hierarchy> h;
    std::vector<std::unique_ptr<samg_bsr3>> views;
};

namespace samgb {
samg_problem *generate_hex(const samg_problem_params &p);
void generate_hex_device(const samg_problem_params &p, Bsr3 &A, DevBuf<double> &rhs,
                         DevBuf<double> &xyz, DevBuf<double> &B, int64_t &nnodes, cudaStream_t s);
void rigid_body_modes(int64_t nnodes, const double *xyz, double *B);
struct DHierarchy;
DHierarchy *dsetup_all(const unsigned char *id, int nranks, int rank, int64_t nbrows,
                       Bsr3 &&A_rows, const double *B, int64_t b_cols,
                       const int64_t *row_starts, int64_t min_rows, const samg_amg_params &prm,
                       cudaStream_t s, double t0, int pipeline);
void ddelete(DHierarchy *d);
samg_solve_report dcg(DHierarchy *d, const double *f, double *u, const samg_cg_params &cp,
                      bool host);
void dinfo(const DHierarchy *d, int64_t *row0, int64_t *row1, int *nlevels, int *dist_levels,
           double *setup_s);
void nccl_unique_id(unsigned char *out);
int64_t dheld_rows(const DHierarchy *d);
const Bsr3 &dlevel(DHierarchy *d, int level, int which, Bsr3 &tmp);
}

struct samg_dproblem {
    int device = 0;
    samgb::Bsr3 A;
    samgb::DevBuf<double> rhs, xyz, B;
    int64_t nnodes = 0;
    samg_bsr3 view;
};

struct samg_dhierarchy {
    samgb::DHierarchy *d = nullptr;
};


namespace {

using namespace samgb;

thread_local std::string g_err;

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <class F>
int guarded(F f) {
    try {
        f();
        g_err.clear();
        return SAMG_OK;
    } catch (const Error &e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc &) {
        g_err = "host out of memory";
        return SAMG_OUT_OF_MEMORY;
    } catch (const std::exception &e) {
        g_err = e.what();
        return SAMG_ERROR;
    }
}

void require(bool c, int code, const char *msg) {
    if (!c) fail(code, msg);
}

void need_device(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        fail(SAMG_NO_DEVICE, "no CUDA device available (the B200 path has no CPU fallback)");
    }
    require(device >= 0 && device < n, SAMG_INVALID_ARGUMENT, "device ordinal out of range");
    CK(cudaSetDevice(device));
    // keep stream-ordered allocations cached across syncs (setup allocates
    // and frees per level; returning memory to the driver each time costs
    // tens of milliseconds per setup)
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
}

cudaStream_t new_stream() {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    return s;
}

void validate_params(const samg_amg_params *prm, int pipeline) {
    require(prm != nullptr, SAMG_INVALID_ARGUMENT, "setup: params must not be NULL");
    // ns_block, and the hybrids that differ from it only in the Galerkin
    // arithmetic (scalar order, hierarchy.hpp:233-260) and, for ns_hybrid1,
    // in scalar smoothers (ilu0<double> is not on the B200 path)
    // block: no nullspace, block strength / transfer (hierarchy.hpp:340-347)
    // scalar / ns_scalar (hierarchy.hpp:298-330): the scalar-space setup with
    // scalar level matrices -- the same values as 3x3 blocks on the B200
    // (their patterns are whole blocks), reported in scalar CSR accounting
    require(pipeline >= SAMG_PIPELINE_SCALAR && pipeline <= SAMG_PIPELINE_NS_BLOCK,
            SAMG_INVALID_ARGUMENT, "setup: unknown pipeline");
    if ((pipeline == SAMG_PIPELINE_SCALAR || pipeline == SAMG_PIPELINE_NS_SCALAR) && prm &&
        prm->smoother != SAMG_SMOOTHER_JACOBI && prm->smoother != SAMG_SMOOTHER_ILU0)
        fail(SAMG_UNSUPPORTED, "setup: the scalar pipelines take the reference's scalar smoothers "
                               "(damped Jacobi, ilu0<double>)");
    require(prm->smoother >= 0 && prm->smoother <= 3, SAMG_INVALID_ARGUMENT, "setup: unknown smoother");
    require(prm->pre_sweeps >= 0 && prm->post_sweeps >= 0, SAMG_INVALID_ARGUMENT,
            "setup: negative sweep count");
    require(prm->vcycle_precision == SAMG_PRECISION_FP64 || prm->vcycle_precision == SAMG_PRECISION_MIXED,
            SAMG_INVALID_ARGUMENT, "setup: unknown vcycle_precision");
    require(prm->ilu_sweep_order == SAMG_ILU_ORDER_REFERENCE ||
                prm->ilu_sweep_order == SAMG_ILU_ORDER_LATEST_LAST,
            SAMG_INVALID_ARGUMENT, "setup: unknown ilu_sweep_order");
    if (prm->ilu_sweep_order != SAMG_ILU_ORDER_REFERENCE &&
        (prm->smoother != SAMG_SMOOTHER_ILU0 || pipeline == SAMG_PIPELINE_SCALAR ||
         pipeline == SAMG_PIPELINE_NS_SCALAR || pipeline == SAMG_PIPELINE_NS_HYBRID1))
        fail(SAMG_UNSUPPORTED, "setup: ilu_sweep_order applies to the block ILU(0) smoother only");
}

// hierarchy.hpp:267-282 + coarsening.hpp:269-270 checks
void validate_ns(int64_t n, const double *B, int64_t b_rows, int64_t b_cols, int pipeline) {
    require(n >= 0, SAMG_INVALID_ARGUMENT, "setup: negative dimension");
    if (pipeline == SAMG_PIPELINE_BLOCK || pipeline == SAMG_PIPELINE_SCALAR) {  // no nullspace: B ignored
        if (n % 3) fail(SAMG_NOT_DIVISIBLE, "setup: block pipelines require dimension divisible by 3");
        return;
    }
    if (!B) fail(SAMG_BAD_NULLSPACE_SHAPE, "setup: pipeline requires a nullspace basis");
    if (b_rows != n) fail(SAMG_BAD_NULLSPACE_SHAPE, "setup: nullspace rows do not match matrix");
    if (n % 3) fail(SAMG_NOT_DIVISIBLE, "setup: block pipelines require dimension divisible by 3");
    if (b_cols < 1 || b_cols % 3)
        fail(SAMG_NOT_DIVISIBLE, "as_scalar_transfer: coarse dimension not divisible by block size");
    if (b_cols > 12) fail(SAMG_UNSUPPORTED, "setup: at most 12 nullspace vectors");
}

template <class F>
__global__ void k_apply(int64_t n, F f) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        f(i);
}
template <class F>
void apply(int64_t n, F f, cudaStream_t s) {
    if (n <= 0) return;
    int64_t g = (n + 255) / 256;
    if (g > 524280) g = 524280;
    k_apply<<<static_cast<int>(g), 256, 0, s>>>(n, f);
    CK_LAUNCH();
}

// upload a host int64 BSR3 into a device Bsr3 (int32), validating structure
void upload_bsr3(int64_t nrows, int64_t ncols, const int64_t *ptr, const int64_t *col,
                 const double *val, Bsr3 &M, cudaStream_t s) {
    require(ptr && (ptr[nrows] == 0 || (col && val)), SAMG_INVALID_ARGUMENT, "bsr3: NULL array");
    require(ptr[0] == 0, SAMG_INVALID_ARGUMENT, "bsr3: ptr[0] must be 0");
    const int64_t nnz = ptr[nrows];
    M.alloc(nrows, ncols, nnz, s);
    DevBuf<int64_t> p64(nrows + 1, s), c64(nnz, s);
    h2d(p64.p, ptr, sizeof(int64_t) * (nrows + 1), s);
    if (nnz) {
        h2d(c64.p, col, sizeof(int64_t) * nnz, s);
        h2d(M.val.p, val, sizeof(double) * 9 * nnz, s);
    }
    DevBuf<int> bad(1, s);
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    int *mp = M.ptr.p, *mc = M.col.p, *bp = bad.p;
    const int64_t *pp = p64.p, *cp = c64.p;
    apply(nrows + 1, [=] __device__(int64_t i) {
        mp[i] = static_cast<int>(pp[i]);
        if (i > 0 && pp[i] < pp[i - 1]) *bp = 1;
    }, s);
    apply(nrows, [=] __device__(int64_t i) {
        for (int64_t j = pp[i]; j < pp[i + 1]; ++j) {
            const int64_t c = cp[j];
            if (c < 0 || c >= ncols || (j > pp[i] && c <= cp[j - 1])) *bp = 1;
            mc[j] = static_cast<int>(c);
        }
    }, s);
    int hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hbad) fail(SAMG_INVALID_ARGUMENT, "bsr3: ptr must be nondecreasing and each row's columns strictly increasing and in range");
}

samgb::Hierarchy &H(samg_hierarchy *h) {
    if (!h || !h->h) fail(SAMG_INVALID_ARGUMENT, "NULL hierarchy handle");
    CK(cudaSetDevice(h->h->device));
    return *h->h;
}
const samgb::Hierarchy &Hc(const samg_hierarchy *h) {
    if (!h || !h->h) fail(SAMG_INVALID_ARGUMENT, "NULL hierarchy handle");
    return *h->h;
}

const Bsr3 &level_mat(const samgb::Hierarchy &h, int level, int which) {
    if (level < 0 || level >= static_cast<int>(h.levels.size()))
        fail(SAMG_INVALID_ARGUMENT, "level out of range");
    const Level &lv = h.levels[level];
    if (which == 0) return lv.A;
    if (!lv.has_transfer) fail(SAMG_INVALID_ARGUMENT, "coarsest level has no P/R");
    if (which == 1) return lv.P;
    if (which == 2) return lv.R;
    fail(SAMG_INVALID_ARGUMENT, "which must be 0 (A), 1 (P) or 2 (R)");
}

void download_bsr3(const Bsr3 &M, int64_t *ptr, int64_t *col, double *val, cudaStream_t s) {
    std::vector<int> p(M.nrows + 1), c(M.nnzb);
    CK(cudaMemcpyAsync(p.data(), M.ptr.p, sizeof(int) * (M.nrows + 1), cudaMemcpyDeviceToHost, s));
    if (M.nnzb) {
        CK(cudaMemcpyAsync(c.data(), M.col.p, sizeof(int) * M.nnzb, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(val, M.val.p, sizeof(double) * 9 * M.nnzb, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    for (int64_t i = 0; i <= M.nrows; ++i) ptr[i] = p[i];
    for (int64_t i = 0; i < M.nnzb; ++i) col[i] = c[i];
}

samg_hierarchy *finish_setup(Bsr3 &&A0, const double *B, int64_t b_rows, int64_t b_cols,
                             const samg_amg_params &prm, cudaStream_t s, double t0, int pipeline) {
    auto out = std::make_unique<samg_hierarchy>();
    try {
        out->h.reset(setup_hierarchy(std::move(A0), B, b_rows, b_cols, prm, s, t0, pipeline));
    } catch (...) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
        throw;
    }
    return out.release();
}

} // namespace

extern "C" {

SAMG_API void samg_default_amg_params(samg_amg_params *p) {
    if (!p) return;
    p->eps_strong = 0.08;
    p->omega = 2.0 / 3.0;
    p->point_block_size = 3;
    p->smoother = SAMG_SMOOTHER_SPAI0;
    p->smoother_omega = 0.72;
    p->pre_sweeps = 1;
    p->post_sweeps = 1;
    p->coarse_enough = 3000;
    p->stagnation_ratio = 0.8;
    p->verify_galerkin = 0;
    p->device = 0;
    p->vcycle_precision = SAMG_PRECISION_FP64;
    p->ilu_sweep_order = SAMG_ILU_ORDER_REFERENCE;
}

SAMG_API void samg_default_cg_params(samg_cg_params *p) {
    if (!p) return;
    p->tol = 1e-8;
    p->max_iterations = 1000;
}

SAMG_API const char *samg_last_error(void) { return g_err.c_str(); }

SAMG_API const char *samg_status_name(int st) {
    switch (st) {
        case SAMG_OK: return "ok";
        case SAMG_ERROR: return "error";
        case SAMG_DIMENSION_MISMATCH: return "dimension_mismatch";
        case SAMG_NOT_DIVISIBLE: return "not_divisible";
        case SAMG_SINGULAR_BLOCK: return "singular_block";
        case SAMG_MISSING_DIAGONAL: return "missing_diagonal";
        case SAMG_ZERO_DIAGONAL: return "zero_diagonal";
        case SAMG_NON_SQUARE: return "non_square";
        case SAMG_BAD_NULLSPACE_SHAPE: return "bad_nullspace_shape";
        case SAMG_BREAKDOWN_NON_SPD: return "breakdown_non_spd";
        case SAMG_INVALID_MATERIAL: return "invalid_material";
        case SAMG_SHAPE_MISMATCH: return "shape_mismatch";
        case SAMG_CUDA_ERROR: return "cuda_error";
        case SAMG_NCCL_ERROR: return "nccl_error";
        case SAMG_OUT_OF_MEMORY: return "out_of_memory";
        case SAMG_NO_DEVICE: return "no_device";
        case SAMG_UNSUPPORTED: return "unsupported";
        case SAMG_INVALID_ARGUMENT: return "invalid_argument";
        default: return "unknown";
    }
}

SAMG_API int samg_device_count(int *count) {
    return guarded([&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) { cudaGetLastError(); n = 0; }
        *count = n;
    });
}

SAMG_API int samg_setup(int64_t n, const int64_t *ptr, const int64_t *col, const double *val,
                        const double *B, int64_t b_rows, int64_t b_cols, int pipeline,
                        const samg_amg_params *prm, samg_hierarchy **out) {
    return guarded([&] {
        const double t0 = now_s();
        require(out != nullptr, SAMG_INVALID_ARGUMENT, "setup: out must not be NULL");
        *out = nullptr;
        validate_params(prm, pipeline);
        validate_ns(n, B, b_rows, b_cols, pipeline);
        require(ptr && ptr[0] == 0 && (ptr[n] == 0 || (col && val)), SAMG_INVALID_ARGUMENT,
                "setup: malformed CSR arrays");
        need_device(prm->device);
        cudaStream_t s = new_stream();
        static const bool timing = [] {
            const char *e = std::getenv("SAMG_SETUP_TIMING");
            return e && e[0] == '1';
        }();
        double tm = now_s();
        auto tmark = [&](const char *what) {  // SAMG_SETUP_TIMING: the upload's parts
            if (!timing) return;
            CK(cudaStreamSynchronize(s));
            const double t = now_s();
            std::fprintf(stderr, "setup upload %-14s %8.3f ms\n", what, 1e3 * (t - tm));
            tm = t;
        };
        tmark("stream");
        Bsr3 A0;
        try {
            const int64_t nnz = ptr[n];
            DevBuf<int64_t> dp(n + 1, s);
            DevBuf<double> dv(nnz, s);
            tmark("alloc");
            h2d(dp.p, ptr, sizeof(int64_t) * (n + 1), s);
            if (nnz) h2d(dv.p, val, sizeof(double) * nnz, s);
            tmark("h2d values");
            if (n <= INT32_MAX) {
                // column indices narrowed to 32 bits by the staging threads
                // (half the PCIe bytes of the int64 array; range-checked)
                DevBuf<int32_t> dc(nnz, s);
                require(h2d_narrow(dc.p, col, static_cast<size_t>(nnz), n, s), SAMG_INVALID_ARGUMENT,
                        "setup: column index out of range");
                tmark("h2d columns");
                scalar_to_bsr3(n, dp.p, dc.p, dv.p, A0, s);
                tmark("to_block");
            } else {
                DevBuf<int64_t> dc(nnz, s);
                if (nnz) h2d(dc.p, col, sizeof(int64_t) * nnz, s);
                scalar_to_bsr3(n, dp.p, dc.p, dv.p, A0, s);
            }
            // scalar level matrices in the reference (hierarchy.hpp:298-330)
            // and ilu0<double> work on the scalar pattern: the 3x3 storage
            // reproduces them only when every stored block is whole -- a
            // partial block's padding zeros would join the ILU(0) pattern and
            // the footprint.  Refused loudly rather than answered differently.
            const bool scalar_pattern =
                pipeline == SAMG_PIPELINE_SCALAR || pipeline == SAMG_PIPELINE_NS_SCALAR ||
                (pipeline == SAMG_PIPELINE_NS_HYBRID1 && prm->smoother == SAMG_SMOOTHER_ILU0);
            if (scalar_pattern && nnz != 9 * A0.nnzb) {
                { Bsr3 drop = std::move(A0); }  // freed on s before the handler destroys the stream
                fail(SAMG_UNSUPPORTED, "setup: this pipeline keeps the scalar pattern; the input must "
                                       "hold whole 3x3 blocks (all 9 entries of every touched block)");
            }
        } catch (...) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
            throw;
        }
        *out = finish_setup(std::move(A0), B, b_rows, b_cols, *prm, s, t0, pipeline);
    });
}

SAMG_API int samg_setup_bsr3(int64_t nbrows, const int64_t *ptr, const int64_t *col,
                             const double *val, const double *B, int64_t b_rows, int64_t b_cols,
                             int pipeline, const samg_amg_params *prm, samg_hierarchy **out) {
    return guarded([&] {
        const double t0 = now_s();
        require(out != nullptr, SAMG_INVALID_ARGUMENT, "setup: out must not be NULL");
        *out = nullptr;
        validate_params(prm, pipeline);
        validate_ns(3 * nbrows, B, b_rows, b_cols, pipeline);
        need_device(prm->device);
        cudaStream_t s = new_stream();
        Bsr3 A0;
        try {
            upload_bsr3(nbrows, nbrows, ptr, col, val, A0, s);
        } catch (...) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
            throw;
        }
        *out = finish_setup(std::move(A0), B, b_rows, b_cols, *prm, s, t0, pipeline);
    });
}

// setup from a device-resident matrix (copied, the caller keeps its own);
// B may be a host or a device pointer
SAMG_API int samg_setup_device(const samg_bsr3 *A, const double *B, int64_t b_rows, int64_t b_cols,
                               int pipeline, const samg_amg_params *prm, samg_hierarchy **out) {
    return guarded([&] {
        const double t0 = now_s();
        require(out != nullptr && A && A->m, SAMG_INVALID_ARGUMENT, "setup_device: NULL argument");
        *out = nullptr;
        validate_params(prm, pipeline);
        const Bsr3 &M = *A->m;
        if (M.nrows != M.ncols) fail(SAMG_NON_SQUARE, "transfer_operators: matrix must be square");
        validate_ns(3 * M.nrows, B, b_rows, b_cols, pipeline);
        need_device(prm->device);
        require(A->device == prm->device, SAMG_INVALID_ARGUMENT, "setup_device: matrix lives on another device");
        cudaStream_t s = new_stream();
        Bsr3 A0;
        try {
            A0.alloc(M.nrows, M.ncols, M.nnzb, s);
            CK(cudaMemcpyAsync(A0.ptr.p, M.ptr.p, sizeof(int) * (M.nrows + 1), cudaMemcpyDeviceToDevice, s));
            if (M.nnzb) {
                CK(cudaMemcpyAsync(A0.col.p, M.col.p, sizeof(int) * M.nnzb, cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(A0.val.p, M.val.p, sizeof(double) * 9 * M.nnzb, cudaMemcpyDeviceToDevice, s));
            }
        } catch (...) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
            throw;
        }
        *out = finish_setup(std::move(A0), B, b_rows, b_cols, *prm, s, t0, pipeline);
    });
}

SAMG_API int samg_generate_hex_device(const samg_problem_params *p, int device, samg_dproblem **out) {
    return guarded([&] {
        require(p && out, SAMG_INVALID_ARGUMENT, "generate_hex_device: NULL argument");
        *out = nullptr;
        need_device(device);
        auto d = std::make_unique<samg_dproblem>();
        d->device = device;
        cudaStream_t s = nullptr;
        generate_hex_device(*p, d->A, d->rhs, d->xyz, d->B, d->nnodes, s);
        d->view.m = &d->A;
        d->view.device = device;
        *out = d.release();
    });
}

SAMG_API int samg_dproblem_destroy(samg_dproblem *p) {
    return guarded([&] {
        if (!p) return;
        cudaSetDevice(p->device);
        cudaDeviceSynchronize();
        delete p;
    });
}

SAMG_API int samg_dproblem_info(const samg_dproblem *p, int64_t *n, int64_t *nbrows, int64_t *nnzb) {
    return guarded([&] {
        require(p && n && nbrows && nnzb, SAMG_INVALID_ARGUMENT, "dproblem_info: NULL argument");
        *n = 3 * p->nnodes;
        *nbrows = p->A.nrows;
        *nnzb = p->A.nnzb;
    });
}

SAMG_API int samg_dproblem_matrix(const samg_dproblem *p, const samg_bsr3 **A) {
    return guarded([&] {
        require(p && A, SAMG_INVALID_ARGUMENT, "dproblem_matrix: NULL argument");
        *A = &p->view;
    });
}

SAMG_API int samg_dproblem_vectors(const samg_dproblem *p, const double **rhs, const double **B,
                                   const double **xyz) {
    return guarded([&] {
        require(p, SAMG_INVALID_ARGUMENT, "dproblem_vectors: NULL argument");
        if (rhs) *rhs = p->rhs.p;
        if (B) *B = p->B.p;
        if (xyz) *xyz = p->xyz.p;
    });
}

SAMG_API int samg_dproblem_download(const samg_dproblem *p, double *rhs, double *B, double *xyz) {
    return guarded([&] {
        require(p, SAMG_INVALID_ARGUMENT, "dproblem_download: NULL argument");
        CK(cudaSetDevice(p->device));
        const int64_t n = 3 * p->nnodes;
        if (rhs) CK(cudaMemcpy(rhs, p->rhs.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
        if (B) CK(cudaMemcpy(B, p->B.p, sizeof(double) * 6 * n, cudaMemcpyDeviceToHost));
        if (xyz) CK(cudaMemcpy(xyz, p->xyz.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    });
}

SAMG_API int samg_destroy(samg_hierarchy *h) {
    return guarded([&] {
        if (!h) return;
        if (h->h) cudaSetDevice(h->h->device);
        delete h;
    });
}

SAMG_API int samg_cg_solve(samg_hierarchy *hp, const double *f, double *u,
                           const samg_cg_params *prm, samg_solve_report *rep) {
    return guarded([&] {
        require(f && u && prm && rep, SAMG_INVALID_ARGUMENT, "cg_solve: NULL argument");
        samgb::Hierarchy &h = H(hp);
        const double t0 = now_s();
        const int64_t n = h.finest_dim();
        h2d(h.fbuf.p, f, sizeof(double) * n, h.stream);
        *rep = h.cg(h.fbuf.p, h.ubuf.p, *prm);
        CK(cudaMemcpyAsync(u, h.ubuf.p, sizeof(double) * n, cudaMemcpyDeviceToHost, h.stream));
        CK(cudaStreamSynchronize(h.stream));
        rep->solve_seconds = now_s() - t0;
    });
}

SAMG_API int samg_cg_solve_device(samg_hierarchy *hp, const double *d_f, double *d_u,
                                  const samg_cg_params *prm, samg_solve_report *rep) {
    return guarded([&] {
        require(d_f && d_u && prm && rep, SAMG_INVALID_ARGUMENT, "cg_solve: NULL argument");
        samgb::Hierarchy &h = H(hp);
        *rep = h.cg(d_f, d_u, *prm);
    });
}

SAMG_API int samg_vcycle(samg_hierarchy *hp, const double *f, double *u) {
    return guarded([&] {
        require(f && u, SAMG_INVALID_ARGUMENT, "vcycle: NULL argument");
        samgb::Hierarchy &h = H(hp);
        const int64_t n = h.finest_dim();
        h2d(h.fbuf.p, f, sizeof(double) * n, h.stream);
        h2d(h.ubuf.p, u, sizeof(double) * n, h.stream);
        h.vcycle(h.fbuf.p, h.ubuf.p, false);
        CK(cudaMemcpyAsync(u, h.ubuf.p, sizeof(double) * n, cudaMemcpyDeviceToHost, h.stream));
        CK(cudaStreamSynchronize(h.stream));
    });
}

SAMG_API int samg_vcycle_device(samg_hierarchy *hp, const double *d_f, double *d_u) {
    return guarded([&] {
        require(d_f && d_u, SAMG_INVALID_ARGUMENT, "vcycle: NULL argument");
        samgb::Hierarchy &h = H(hp);
        h.vcycle(d_f, d_u, false);
        CK(cudaStreamSynchronize(h.stream));
    });
}

SAMG_API int samg_cg_solve_op(int64_t n, samg_apply_fn apply_A, samg_apply_fn apply_M, void *ctx,
                              const double *d_f, double *d_u, const samg_cg_params *prm, int device,
                              samg_solve_report *rep) {
    return guarded([&] {
        require(n >= 0 && apply_A && d_f && d_u && prm && rep, SAMG_INVALID_ARGUMENT,
                "cg_solve_op: bad arguments");
        need_device(device);
        cudaStream_t s = new_stream();
        try {
            *rep = cg_solve_op(n, apply_A, apply_M, ctx, d_f, d_u, *prm, s);
        } catch (...) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
            throw;
        }
        CK(cudaStreamDestroy(s));
    });
}

SAMG_API int samg_memory_footprint(const samg_hierarchy *h, uint64_t *bytes) {
    return guarded([&] { *bytes = Hc(h).memory_footprint(); });
}
SAMG_API int samg_finest_dim(const samg_hierarchy *h, int64_t *n) {
    return guarded([&] { *n = Hc(h).finest_dim(); });
}
SAMG_API int samg_num_levels(const samg_hierarchy *h, int *nl) {
    return guarded([&] { *nl = static_cast<int>(Hc(h).levels.size()); });
}
SAMG_API int samg_coarse_dim(const samg_hierarchy *h, int64_t *n) {
    return guarded([&] { *n = Hc(h).nc; });
}
SAMG_API int samg_coarse_solver(const samg_hierarchy *h, int *kind) {
    return guarded([&] { *kind = Hc(h).coarse_lu ? 1 : 0; });
}
SAMG_API int samg_setup_seconds(const samg_hierarchy *h, double *sec) {
    return guarded([&] { *sec = Hc(h).setup_seconds; });
}

SAMG_API int samg_level_info(const samg_hierarchy *h, int level, int which, int64_t *nrows,
                             int64_t *ncols, int64_t *nnzb) {
    return guarded([&] {
        const Bsr3 &M = level_mat(Hc(h), level, which);
        *nrows = M.nrows;
        *ncols = M.ncols;
        *nnzb = M.nnzb;
    });
}

SAMG_API int samg_get_level(const samg_hierarchy *hp, int level, int which, int64_t *ptr,
                            int64_t *col, double *val) {
    return guarded([&] {
        const samgb::Hierarchy &h = Hc(hp);
        CK(cudaSetDevice(h.device));
        download_bsr3(level_mat(h, level, which), ptr, col, val, h.stream);
    });
}

SAMG_API int samg_level_matrix(samg_hierarchy *hp, int level, int which, const samg_bsr3 **m) {
    return guarded([&] {
        const samgb::Hierarchy &h = Hc(hp);
        auto v = std::make_unique<samg_bsr3>();
        v->m = &level_mat(h, level, which);
        v->device = h.device;
        *m = v.get();
        hp->views.push_back(std::move(v));
    });
}

SAMG_API int samg_aggregates_info(const samg_hierarchy *hp, int level, int64_t *nnodes,
                                  int64_t *count) {
    return guarded([&] {
        const samgb::Hierarchy &h = Hc(hp);
        if (level < 0 || level + 1 >= static_cast<int>(h.levels.size()))
            fail(SAMG_INVALID_ARGUMENT, "level has no aggregates");
        *nnodes = h.levels[level].nnodes;
        *count = h.levels[level].naggs;
    });
}

SAMG_API int samg_get_aggregates(const samg_hierarchy *hp, int level, int64_t *id) {
    return guarded([&] {
        const samgb::Hierarchy &h = Hc(hp);
        if (level < 0 || level + 1 >= static_cast<int>(h.levels.size()))
            fail(SAMG_INVALID_ARGUMENT, "level has no aggregates");
        CK(cudaSetDevice(h.device));
        const Level &lv = h.levels[level];
        std::vector<int> a(lv.nnodes);
        CK(cudaMemcpyAsync(a.data(), lv.agg.p, sizeof(int) * lv.nnodes, cudaMemcpyDeviceToHost, h.stream));
        CK(cudaStreamSynchronize(h.stream));
        for (int64_t i = 0; i < lv.nnodes; ++i) id[i] = a[i];
    });
}

SAMG_API int samg_smoother_info(const samg_hierarchy *hp, int level, int64_t *len) {
    return guarded([&] {
        const samgb::Hierarchy &h = Hc(hp);
        if (level < 0 || level + 1 >= static_cast<int>(h.levels.size()))
            fail(SAMG_INVALID_ARGUMENT, "level has no smoother");
        const Smoother &M = h.levels[level].M;
        // ILU(0): [factors (9*nnzb) | inverted pivots (9*nrows; ilu0<double>: 3*nrows)]
        *len = M.kind == SM_ILU ? 9 * M.nnzb + (M.scalar ? 3 : 9) * M.nrows : static_cast<int64_t>(M.data.n);
    });
}

SAMG_API int samg_get_smoother(const samg_hierarchy *hp, int level, double *data) {
    return guarded([&] {
        const samgb::Hierarchy &h = Hc(hp);
        if (level < 0 || level + 1 >= static_cast<int>(h.levels.size()))
            fail(SAMG_INVALID_ARGUMENT, "level has no smoother");
        CK(cudaSetDevice(h.device));
        const Smoother &M = h.levels[level].M;
        if (M.kind == SM_ILU) {
            CK(cudaMemcpyAsync(data, M.lu.p, sizeof(double) * 9 * M.nnzb, cudaMemcpyDeviceToHost, h.stream));
            CK(cudaMemcpyAsync(data + 9 * M.nnzb, M.data.p, sizeof(double) * (M.scalar ? 3 : 9) * M.nrows,
                               cudaMemcpyDeviceToHost, h.stream));
        } else {
            CK(cudaMemcpyAsync(data, M.data.p, M.data.bytes(), cudaMemcpyDeviceToHost, h.stream));
        }
        CK(cudaStreamSynchronize(h.stream));
    });
}

SAMG_API int samg_bsr3_create(int64_t nrows, int64_t ncols, const int64_t *ptr, const int64_t *col,
                              const double *val, int device, samg_bsr3 **out) {
    return guarded([&] {
        require(out != nullptr && nrows >= 0 && ncols >= 0, SAMG_INVALID_ARGUMENT, "bsr3_create: bad arguments");
        *out = nullptr;
        need_device(device);
        auto m = std::make_unique<samg_bsr3>();
        m->device = device;
        upload_bsr3(nrows, ncols, ptr, col, val, m->own, nullptr);
        CK(cudaDeviceSynchronize());
        m->m = &m->own;
        *out = m.release();
    });
}

SAMG_API int samg_bsr3_destroy(samg_bsr3 *m) {
    return guarded([&] {
        if (!m) return;
        cudaSetDevice(m->device);
        cudaDeviceSynchronize();
        delete m;
    });
}

SAMG_API int samg_bsr3_info(const samg_bsr3 *m, int64_t *nrows, int64_t *ncols, int64_t *nnzb) {
    return guarded([&] {
        require(m && m->m, SAMG_INVALID_ARGUMENT, "NULL matrix");
        *nrows = m->m->nrows;
        *ncols = m->m->ncols;
        *nnzb = m->m->nnzb;
    });
}

SAMG_API int samg_bsr3_download(const samg_bsr3 *m, int64_t *ptr, int64_t *col, double *val) {
    return guarded([&] {
        require(m && m->m, SAMG_INVALID_ARGUMENT, "NULL matrix");
        CK(cudaSetDevice(m->device));
        CK(cudaDeviceSynchronize());
        download_bsr3(*m->m, ptr, col, val, nullptr);
    });
}

SAMG_API int samg_bsr3_spmv_device(const samg_bsr3 *m, double alpha, const double *d_x,
                                   double beta, double *d_y, void *stream) {
    return guarded([&] {
        require(m && m->m, SAMG_INVALID_ARGUMENT, "NULL matrix");
        require(reinterpret_cast<uintptr_t>(d_x) % 16 == 0, SAMG_INVALID_ARGUMENT,
                "spmv: x must be 16-byte aligned (the kernel gathers x with 16-byte loads)");
        // consecutive standalone SpMVs overlap: the next one's matrix stream
        // starts under the previous one's tail (programmatic dependent
        // launch; x is read only once the previous kernel completed)
        set_spmv_pdl(true);
        try {
            launch_spmv(*m->m, alpha, d_x, beta, d_y, static_cast<cudaStream_t>(stream));
        } catch (...) {
            set_spmv_pdl(false);
            throw;
        }
        set_spmv_pdl(false);
    });
}

SAMG_API int samg_bsr3_spmv(const samg_bsr3 *mc, double alpha, const double *x, double beta,
                            double *y) {
    return guarded([&] {
        require(mc && mc->m && x && y, SAMG_INVALID_ARGUMENT, "spmv: NULL argument");
        auto *m = const_cast<samg_bsr3 *>(mc);
        CK(cudaSetDevice(m->device));
        const Bsr3 &A = *m->m;
        if (m->xs.n < static_cast<size_t>(3 * A.ncols)) m->xs.alloc(3 * A.ncols, nullptr);
        if (m->ys.n < static_cast<size_t>(3 * A.nrows)) m->ys.alloc(3 * A.nrows, nullptr);
        h2d(m->xs.p, x, sizeof(double) * 3 * A.ncols, nullptr);
        if (beta != 0.0)
            h2d(m->ys.p, y, sizeof(double) * 3 * A.nrows, nullptr);
        launch_spmv(A, alpha, m->xs.p, beta, m->ys.p, nullptr);
        CK(cudaMemcpyAsync(y, m->ys.p, sizeof(double) * 3 * A.nrows, cudaMemcpyDeviceToHost, nullptr));
        CK(cudaStreamSynchronize(nullptr));
    });
}

// count independent products y_k = alpha A x_k + beta y_k with host
// vectors (x: count x 3*ncols, y: count x 3*nrows, row-major).  Every
// product still copies its x_k in and its y_k out; three streams with
// triple-buffered device staging overlap the H2D of x_{k+1}, the kernel of
// k and the D2H of y_{k-1} (full-duplex PCIe, separate copy engines): a
// stream's chain H2D -> kernel -> D2H spans ~3 steps, so 3 buffers keep both
// copy directions busy.
// CTAs of the SpMV inside the host-vector pipeline (SAMG_BATCH_CTAS; 0 = one
// per SM).  With the SpMV on every SM the kernel saturates HBM and starves
// the concurrent PCIe DMA in both directions (H2D 116 -> 177 us, the SpMV
// 85 -> 115 us per step, scripts/e2e_timeline.py); on 96 of 148 SMs the
// SpMV still keeps up and the copies run at the duplex PCIe rate: C1 e2e
// 2 900 -> 3 920 GB/s-equivalent (scripts/e2e_sweep.sh).
static int batch_cta_cap() {
    static const int env = [] {
        const char *e = std::getenv("SAMG_BATCH_CTAS");
        return e ? std::atoi(e) : 0;
    }();
    return env ? env : std::max(1, sm_count() * 96 / 148);
}

SAMG_API int samg_bsr3_spmv_batch(const samg_bsr3 *mc, double alpha, const double *x, double beta,
                                  double *y, int64_t count) {
    return guarded([&] {
        require(mc && mc->m && x && y && count >= 0, SAMG_INVALID_ARGUMENT, "spmv_batch: bad argument");
        auto *m = const_cast<samg_bsr3 *>(mc);
        CK(cudaSetDevice(m->device));
        const Bsr3 &A = *m->m;
        const int64_t nx = 3 * A.ncols, ny = 3 * A.nrows;
        constexpr int P = samg_bsr3::kPipe;
        for (cudaStream_t &q : m->bs)
            if (!q) CK(cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking));
        cudaStream_t sh = m->bs[0], sk = m->bs[1], sd = m->bs[2];
        for (int b = 0; b < P; ++b) {
            for (cudaEvent_t *e : {&m->ev_h[b], &m->ev_k[b], &m->ev_d[b]})
                if (!*e) CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
            if (m->bx[b].n < static_cast<size_t>(nx) + 1) m->bx[b].alloc(nx + 1, sk);
            if (m->by[b].n < static_cast<size_t>(ny) + 1) m->by[b].alloc(ny + 1, sk);
        }
        CK(cudaStreamSynchronize(sk));  // staging allocations visible to the copy streams
        for (int64_t k = 0; k < count; ++k) {
            const int b = static_cast<int>(k % P);
            // x slot b: free once kernel k-P has read it
            if (k >= P) CK(cudaStreamWaitEvent(sh, m->ev_k[b], 0));
            CK(cudaMemcpyAsync(m->bx[b].p, x + k * nx, sizeof(double) * nx, cudaMemcpyHostToDevice, sh));
            if (beta != 0.0) {
                // y slot b: step k-P's result must have been copied out first
                if (k >= P) CK(cudaStreamWaitEvent(sh, m->ev_d[b], 0));
                CK(cudaMemcpyAsync(m->by[b].p, y + k * ny, sizeof(double) * ny, cudaMemcpyHostToDevice, sh));
            }
            CK(cudaEventRecord(m->ev_h[b], sh));
            // kernel k: its x has arrived, and y slot b has been copied out (step k-P)
            CK(cudaStreamWaitEvent(sk, m->ev_h[b], 0));
            if (k >= P) CK(cudaStreamWaitEvent(sk, m->ev_d[b], 0));
            set_spmv_cta_cap(batch_cta_cap());
            launch_spmv(A, alpha, m->bx[b].p, beta, m->by[b].p, sk);
            set_spmv_cta_cap(-1);
            CK(cudaEventRecord(m->ev_k[b], sk));
            CK(cudaStreamWaitEvent(sd, m->ev_k[b], 0));
            CK(cudaMemcpyAsync(y + k * ny, m->by[b].p, sizeof(double) * ny, cudaMemcpyDeviceToHost, sd));
            CK(cudaEventRecord(m->ev_d[b], sd));
        }
        for (cudaStream_t q : m->bs) CK(cudaStreamSynchronize(q));
    });
}

SAMG_API int samg_bsr3_galerkin(const samg_bsr3 *R, const samg_bsr3 *A, const samg_bsr3 *P,
                                samg_bsr3 **out) {
    return guarded([&] {
        require(R && A && P && out && R->m && A->m && P->m, SAMG_INVALID_ARGUMENT, "galerkin: NULL argument");
        *out = nullptr;
        if (R->m->ncols != A->m->nrows || A->m->ncols != P->m->nrows)
            fail(SAMG_DIMENSION_MISMATCH, "spgemm: inner dimensions disagree");
        CK(cudaSetDevice(A->device));
        auto c = std::make_unique<samg_bsr3>();
        c->device = A->device;
        Bsr3 RA;
        spgemm(*R->m, *A->m, RA, nullptr);
        spgemm(RA, *P->m, c->own, nullptr);
        CK(cudaDeviceSynchronize());
        c->m = &c->own;
        *out = c.release();
    });
}

SAMG_API int samg_bsr3_dense_inverse(const samg_bsr3 *m, double *inv) {
    return guarded([&] {
        require(m && m->m && inv, SAMG_INVALID_ARGUMENT, "dense_inverse: NULL argument");
        const Bsr3 &A = *m->m;
        if (A.nrows != A.ncols) fail(SAMG_NON_SQUARE, "dense_lu: matrix must be square");
        CK(cudaSetDevice(m->device));
        cudaStream_t s = nullptr;
        DevBuf<DevError> err(1, s);
        CK(cudaMemsetAsync(err.p, 0, sizeof(DevError), s));
        DevBuf<double> Ainv;
        if (!dense_inverse(A, Ainv, err.p, s))
            fail(SAMG_ERROR, "dense_lu: singular coarse matrix (Gauss-Jordan pivot below 1e-300)");
        const int64_t n = 3 * A.nrows, ld = dense_ld(n);
        if (n)
            CK(cudaMemcpy2DAsync(inv, sizeof(double) * n, Ainv.p, sizeof(double) * ld,
                                 sizeof(double) * n, n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    });
}

SAMG_API int samg_bsr3_spmv_bytes(const samg_bsr3 *m, int beta_nonzero, uint64_t *bytes) {
    return guarded([&] {
        require(m && m->m && bytes, SAMG_INVALID_ARGUMENT, "NULL argument");
        const Bsr3 &A = *m->m;
        // nnzb*(72 + 4) + (nrows+1)*4 + x once + y write (+ y read)
        *bytes = static_cast<uint64_t>(A.nnzb) * 76 + static_cast<uint64_t>(A.nrows + 1) * 4 +
                 static_cast<uint64_t>(A.ncols) * 24 + static_cast<uint64_t>(A.nrows) * 24 *
                 (beta_nonzero ? 2 : 1);
    });
}

SAMG_API void samg_default_problem_params(samg_problem_params *p) {
    if (!p) return;
    std::memset(p, 0, sizeof *p);
    p->nx = p->ny = p->nz = 19;
    p->lx = p->ly = p->lz = 1.0;
    p->E = 1.0;
    p->nu = 0.3;
    p->dirichlet = SAMG_DIRICHLET_ELIMINATE;
    p->load = SAMG_LOAD_BODY_FORCE;
    p->seed = 12345;
}

SAMG_API int samg_generate_hex(const samg_problem_params *p, samg_problem **out) {
    return guarded([&] {
        require(p && out, SAMG_INVALID_ARGUMENT, "generate_hex: NULL argument");
        *out = generate_hex(*p);
    });
}

SAMG_API int samg_problem_destroy(samg_problem *p) {
    return guarded([&] { delete p; });
}

SAMG_API int samg_problem_info(const samg_problem *p, int64_t *n, int64_t *nnzb, int64_t *nnodes) {
    return guarded([&] {
        require(p != nullptr, SAMG_INVALID_ARGUMENT, "NULL problem");
        *n = p->n;
        *nnzb = p->ptr.back();
        *nnodes = p->nnodes;
    });
}

SAMG_API int samg_problem_get_bsr3(const samg_problem *p, int64_t *ptr, int64_t *col, double *val) {
    return guarded([&] {
        require(p != nullptr, SAMG_INVALID_ARGUMENT, "NULL problem");
        std::memcpy(ptr, p->ptr.data(), sizeof(int64_t) * p->ptr.size());
        std::memcpy(col, p->col.data(), sizeof(int64_t) * p->col.size());
        std::memcpy(val, p->val.data(), sizeof(double) * p->val.size());
    });
}

SAMG_API int samg_problem_bsr3_view(const samg_problem *p, const int64_t **ptr,
                                    const int64_t **col, const double **val) {
    return guarded([&] {
        require(p != nullptr, SAMG_INVALID_ARGUMENT, "NULL problem");
        *ptr = p->ptr.data();
        *col = p->col.data();
        *val = p->val.data();
    });
}

SAMG_API int samg_problem_get_csr(const samg_problem *p, int64_t *ptr, int64_t *col, double *val) {
    return guarded([&] {
        require(p != nullptr, SAMG_INVALID_ARGUMENT, "NULL problem");
        // to_scalar (csr.hpp:327-353)
        int64_t out = 0;
        ptr[0] = 0;
        const int64_t nb = p->nnodes;
        for (int64_t bi = 0; bi < nb; ++bi)
            for (int r = 0; r < 3; ++r) {
                for (int64_t j = p->ptr[bi]; j < p->ptr[bi + 1]; ++j)
                    for (int c = 0; c < 3; ++c) {
                        col[out] = 3 * p->col[j] + c;
                        val[out] = p->val[9 * j + 3 * r + c];
                        ++out;
                    }
                ptr[3 * bi + r + 1] = out;
            }
    });
}

SAMG_API int samg_problem_get_rhs(const samg_problem *p, double *rhs) {
    return guarded([&] {
        require(p != nullptr, SAMG_INVALID_ARGUMENT, "NULL problem");
        std::memcpy(rhs, p->rhs.data(), sizeof(double) * p->rhs.size());
    });
}

SAMG_API int samg_problem_get_coords(const samg_problem *p, double *xyz) {
    return guarded([&] {
        require(p != nullptr, SAMG_INVALID_ARGUMENT, "NULL problem");
        std::memcpy(xyz, p->xyz.data(), sizeof(double) * p->xyz.size());
    });
}

SAMG_API int samg_rigid_body_modes(int64_t nnodes, const double *xyz, double *B) {
    return guarded([&] {
        require(xyz && B && nnodes >= 0, SAMG_INVALID_ARGUMENT, "rigid_body_modes: bad arguments");
        rigid_body_modes(nnodes, xyz, B);
    });
}

SAMG_API int samg_nccl_unique_id(unsigned char id[128]) {
    return guarded([&] {
        require(id != nullptr, SAMG_INVALID_ARGUMENT, "NULL id");
        nccl_unique_id(id);
    });
}

namespace {
// shared tail of the samg_dsetup* entry points: `rows` are this process's
// input rows (the whole matrix when emulating), B likewise
void dsetup_entry(const unsigned char *id, int nranks, int rank, int64_t nbrows,
                  const std::function<void(Bsr3 &, cudaStream_t)> &rows, const double *B,
                  int64_t b_cols, const int64_t *row_starts, int64_t min_rows, int pipeline,
                  const samg_amg_params *prm, samg_dhierarchy **out, double t0) {
    require(out && nranks >= 1 && rank >= 0 && rank < nranks, SAMG_INVALID_ARGUMENT,
            "dsetup: bad arguments");
    *out = nullptr;
    validate_params(prm, pipeline);
    if (prm->vcycle_precision != SAMG_PRECISION_FP64)
        fail(SAMG_UNSUPPORTED, "dsetup: the mixed-precision V-cycle is single-GPU only");
    need_device(prm->device);
    cudaStream_t s = new_stream();
    try {
        Bsr3 A;
        rows(A, s);
        auto h = std::make_unique<samg_dhierarchy>();
        h->d = dsetup_all(id, nranks, rank, nbrows, std::move(A), B, b_cols, row_starts,
                          min_rows > 0 ? min_rows : 4096, *prm, s, t0, pipeline);
        *out = h.release();
    } catch (...) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
        throw;
    }
}
}  // namespace

SAMG_API int samg_dsetup(const unsigned char id[128], int nranks, int rank, int64_t nbrows,
                         const int64_t *ptr, const int64_t *col, const double *val,
                         const double *B, int64_t b_rows, int64_t b_cols,
                         const int64_t *row_starts, int64_t min_rows, int pipeline,
                         const samg_amg_params *prm, samg_dhierarchy **out) {
    return guarded([&] {
        const double t0 = now_s();
        require(ptr && nranks >= 1 && rank >= 0 && rank < nranks, SAMG_INVALID_ARGUMENT,
                "dsetup: bad arguments");
        validate_ns(3 * nbrows, B, b_rows, b_cols, pipeline);
        // NCCL: only this rank's rows go to the device (the partition is
        // row_starts, or the even split)
        int64_t r0 = 0, r1 = nbrows;
        if (id) {
            r0 = row_starts ? row_starts[rank] : nbrows * rank / nranks;
            r1 = row_starts ? row_starts[rank + 1] : nbrows * (rank + 1) / nranks;
            require(0 <= r0 && r0 <= r1 && r1 <= nbrows, SAMG_INVALID_ARGUMENT, "dsetup: bad row_starts");
        }
        std::vector<int64_t> lp(r1 - r0 + 1);
        for (int64_t i = r0; i <= r1; ++i) lp[i - r0] = ptr[i] - ptr[r0];
        std::vector<double> Bl;
        const double *Bp = B;
        if (id && B && pipeline != SAMG_PIPELINE_BLOCK) {
            const int64_t n3 = 3 * (r1 - r0);
            Bl.resize(n3 * b_cols);
            for (int64_t c = 0; c < b_cols; ++c)
                std::memcpy(Bl.data() + c * n3, B + c * 3 * nbrows + 3 * r0, sizeof(double) * n3);
            Bp = Bl.data();
        }
        dsetup_entry(id, nranks, rank, nbrows, [&](Bsr3 &A, cudaStream_t s) {
            upload_bsr3(r1 - r0, nbrows, lp.data(), col + ptr[r0], val + 9 * ptr[r0], A, s);
        }, Bp, b_cols, row_starts, min_rows, pipeline, prm, out, t0);
    });
}

SAMG_API int samg_dsetup_local(const unsigned char id[128], int nranks, int rank,
                               const int64_t *row_starts, const int64_t *ptr, const int64_t *col,
                               const double *val, const double *B, int64_t b_cols,
                               int64_t min_rows, int pipeline, const samg_amg_params *prm,
                               samg_dhierarchy **out) {
    return guarded([&] {
        const double t0 = now_s();
        require(id && row_starts && ptr && nranks >= 1 && rank >= 0 && rank < nranks,
                SAMG_INVALID_ARGUMENT, "dsetup_local: bad arguments (NCCL id and row_starts required)");
        const int64_t nbrows = row_starts[nranks], nl = row_starts[rank + 1] - row_starts[rank];
        if (pipeline != SAMG_PIPELINE_BLOCK && (!B || b_cols <= 0))
            fail(SAMG_BAD_NULLSPACE_SHAPE, "dsetup_local: the ns pipelines need the nullspace rows");
        dsetup_entry(id, nranks, rank, nbrows, [&](Bsr3 &A, cudaStream_t s) {
            upload_bsr3(nl, nbrows, ptr, col, val, A, s);
        }, B, b_cols, row_starts, min_rows, pipeline, prm, out, t0);
    });
}

SAMG_API int samg_dsetup_device(const unsigned char id[128], int nranks, int rank,
                                const int64_t *row_starts, const samg_bsr3 *A_local,
                                const double *d_B, int64_t b_cols, int64_t min_rows, int pipeline,
                                const samg_amg_params *prm, samg_dhierarchy **out) {
    return guarded([&] {
        const double t0 = now_s();
        require(id && row_starts && A_local && A_local->m && nranks >= 1 && rank >= 0 && rank < nranks,
                SAMG_INVALID_ARGUMENT, "dsetup_device: bad arguments (NCCL id and row_starts required)");
        const int64_t nbrows = row_starts[nranks];
        if (A_local->m->nrows != row_starts[rank + 1] - row_starts[rank] || A_local->m->ncols != nbrows)
            fail(SAMG_DIMENSION_MISMATCH, "dsetup_device: local rows disagree with row_starts");
        if (pipeline != SAMG_PIPELINE_BLOCK && (!d_B || b_cols <= 0))
            fail(SAMG_BAD_NULLSPACE_SHAPE, "dsetup_device: the ns pipelines need the nullspace rows");
        dsetup_entry(id, nranks, rank, nbrows, [&](Bsr3 &A, cudaStream_t s) {
            const Bsr3 &M = *A_local->m;
            A.alloc(M.nrows, M.ncols, M.nnzb, s);
            CK(cudaMemcpyAsync(A.ptr.p, M.ptr.p, sizeof(int) * (M.nrows + 1), cudaMemcpyDeviceToDevice, s));
            if (M.nnzb) {
                CK(cudaMemcpyAsync(A.col.p, M.col.p, sizeof(int) * M.nnzb, cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(A.val.p, M.val.p, sizeof(double) * 9 * M.nnzb, cudaMemcpyDeviceToDevice, s));
            }
        }, d_B, b_cols, row_starts, min_rows, pipeline, prm, out, t0);
    });
}

SAMG_API int samg_ddestroy(samg_dhierarchy *h) {
    return guarded([&] {
        if (!h) return;
        ddelete(h->d);
        delete h;
    });
}

SAMG_API int samg_dinfo(const samg_dhierarchy *h, int64_t *row0, int64_t *row1, int *nlevels,
                        int *dist_levels, double *setup_s) {
    return guarded([&] {
        require(h && h->d, SAMG_INVALID_ARGUMENT, "NULL hierarchy");
        dinfo(h->d, row0, row1, nlevels, dist_levels, setup_s);
    });
}

SAMG_API int samg_dheld_rows(const samg_dhierarchy *h, int64_t *rows) {
    return guarded([&] {
        require(h && h->d && rows, SAMG_INVALID_ARGUMENT, "NULL argument");
        *rows = dheld_rows(h->d);
    });
}

SAMG_API int samg_dlevel_info(const samg_dhierarchy *h, int level, int which, int64_t *nrows,
                              int64_t *ncols, int64_t *nnzb) {
    return guarded([&] {
        require(h && h->d, SAMG_INVALID_ARGUMENT, "NULL hierarchy");
        Bsr3 tmp;
        const Bsr3 &M = dlevel(h->d, level, which, tmp);
        *nrows = M.nrows;
        *ncols = M.ncols;
        *nnzb = M.nnzb;
    });
}

SAMG_API int samg_dget_level(const samg_dhierarchy *h, int level, int which, int64_t *ptr,
                             int64_t *col, double *val) {
    return guarded([&] {
        require(h && h->d, SAMG_INVALID_ARGUMENT, "NULL hierarchy");
        Bsr3 tmp;
        const Bsr3 &M = dlevel(h->d, level, which, tmp);
        download_bsr3(M, ptr, col, val, nullptr);
    });
}

SAMG_API int samg_dcg_solve_device(samg_dhierarchy *h, const double *d_f, double *d_u,
                                   const samg_cg_params *prm, samg_solve_report *rep) {
    return guarded([&] {
        require(h && h->d && d_f && d_u && prm && rep, SAMG_INVALID_ARGUMENT, "dcg: NULL argument");
        *rep = dcg(h->d, d_f, d_u, *prm, false);
    });
}

SAMG_API int samg_dcg_solve(samg_dhierarchy *h, const double *f, double *u,
                            const samg_cg_params *prm, samg_solve_report *rep) {
    return guarded([&] {
        require(h && h->d && f && u && prm && rep, SAMG_INVALID_ARGUMENT, "dcg: NULL argument");
        *rep = dcg(h->d, f, u, *prm, true);
    });
}

SAMG_API int samg_dist_create(int64_t row0, int64_t row1, const int64_t *ptr, const int64_t *col,
                              const double *val, int nranks, const int64_t *row_starts, int rank,
                              samg_dist **out) {
    return guarded([&] {
        require(out && ptr && row_starts && row1 >= row0, SAMG_INVALID_ARGUMENT, "dist_create: bad arguments");
        require(ptr[row1 - row0] == ptr[0] || (col && val), SAMG_INVALID_ARGUMENT, "dist_create: NULL arrays");
        *out = dist_create(row0, row1, ptr, col, val, nranks, row_starts, rank);
    });
}

SAMG_API int samg_dist_destroy(samg_dist *d) {
    return guarded([&] {
        if (d && d->device >= 0) { cudaSetDevice(d->device); cudaDeviceSynchronize(); }
        delete d;
    });
}

SAMG_API int samg_dist_info(const samg_dist *d, int64_t *nloc, int64_t *nghost, int64_t *ninterior,
                            int64_t *nboundary, int *nrecv, int *nsend) {
    return guarded([&] {
        require(d != nullptr, SAMG_INVALID_ARGUMENT, "NULL dist");
        *nloc = d->nloc;
        *nghost = d->nghost;
        *ninterior = static_cast<int64_t>(d->interior.size());
        *nboundary = static_cast<int64_t>(d->boundary.size());
        *nrecv = static_cast<int>(d->recv_peers.size());
        *nsend = static_cast<int>(d->send_peers.size());
    });
}

SAMG_API int samg_dist_recv_plan(const samg_dist *d, int *peers, int64_t *counts, int64_t *offsets) {
    return guarded([&] {
        require(d != nullptr, SAMG_INVALID_ARGUMENT, "NULL dist");
        for (size_t p = 0; p < d->recv_peers.size(); ++p) {
            peers[p] = d->recv_peers[p];
            counts[p] = d->recv_counts[p];
            offsets[p] = d->recv_offsets[p];
        }
    });
}

SAMG_API int samg_dist_ghosts(const samg_dist *d, int64_t *ids) {
    return guarded([&] {
        require(d != nullptr, SAMG_INVALID_ARGUMENT, "NULL dist");
        std::copy(d->ghost.begin(), d->ghost.end(), ids);
    });
}

SAMG_API int samg_dist_set_send(samg_dist *d, int npeers, const int *peers, const int64_t *counts,
                                const int64_t *ids) {
    return guarded([&] {
        require(d != nullptr && npeers >= 0, SAMG_INVALID_ARGUMENT, "dist_set_send: bad arguments");
        dist_set_send(d, npeers, peers, counts, ids);
    });
}

SAMG_API int samg_dist_derive_send(samg_dist *d) {
    return guarded([&] {
        require(d != nullptr, SAMG_INVALID_ARGUMENT, "NULL dist");
        dist_derive_send(d);
    });
}

SAMG_API int samg_dist_send_plan(const samg_dist *d, int *peers, int64_t *counts, int64_t *offsets,
                                 int64_t *local_rows) {
    return guarded([&] {
        require(d != nullptr && d->send_set, SAMG_INVALID_ARGUMENT, "dist: send plan not set");
        for (size_t p = 0; p < d->send_peers.size(); ++p) {
            peers[p] = d->send_peers[p];
            counts[p] = d->send_counts[p];
            offsets[p] = d->send_offsets[p];
        }
        if (local_rows) std::copy(d->send_idx.begin(), d->send_idx.end(), local_rows);
    });
}

SAMG_API int samg_dist_local_matrix(const samg_dist *d, int64_t *ptr, int64_t *col, double *val) {
    return guarded([&] {
        require(d != nullptr, SAMG_INVALID_ARGUMENT, "NULL dist");
        std::copy(d->ptr.begin(), d->ptr.end(), ptr);  // ptr[nloc] = nnzb
        if (col) std::copy(d->col.begin(), d->col.end(), col);
        if (val) std::copy(d->val.begin(), d->val.end(), val);
    });
}

SAMG_API int samg_dist_to_device(samg_dist *d, int device, int group) {
    return guarded([&] {
        require(d != nullptr, SAMG_INVALID_ARGUMENT, "NULL dist");
        require(d->send_set || d->nranks == 1, SAMG_INVALID_ARGUMENT, "dist: set the send plan first");
        need_device(device);
        dist_to_device(d, device, group);
    });
}

SAMG_API int samg_dist_pack(const samg_dist *d, const double *x, double *buf, void *stream) {
    return guarded([&] {
        require(d && d->device >= 0, SAMG_INVALID_ARGUMENT, "dist: not on a device");
        dist_pack(d, x, buf, static_cast<cudaStream_t>(stream));
    });
}

SAMG_API int samg_dist_spmv(const samg_dist *d, int part, double alpha, const double *xext,
                            double beta, double *y, void *stream) {
    return guarded([&] {
        require(d && d->device >= 0, SAMG_INVALID_ARGUMENT, "dist: not on a device");
        require(part >= 0 && part <= 2, SAMG_INVALID_ARGUMENT, "dist: part must be 0, 1 or 2");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (part == 0 || part == 2) dist_spmv(d, 0, alpha, xext, beta, y, s);
        if (part == 1 || part == 2) dist_spmv(d, 1, alpha, xext, beta, y, s);
    });
}

} // extern "C"
