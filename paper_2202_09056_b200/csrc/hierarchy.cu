// hierarchy.cu -- host orchestration of the ns_block setup loop
// (hierarchy.hpp:331-380), the V-cycle (hierarchy.hpp:408-441) and PCG
// (cg.hpp:39-112).  All level data stays in HBM; the host only sequences
// kernels on one stream and reads back sizes and the CG residual.
#include "hierarchy.cuh"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>
#include <utility>

namespace samgb {

int sm_count() {
    static DeviceCache cache;
    return cache.get([] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    });
}

namespace {

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// matrix_bytes (csr.hpp:360-365): 8-byte indices, 72-byte blocks
uint64_t matrix_bytes(const Bsr3 &A) {
    return static_cast<uint64_t>(A.nrows + 1) * 8 + static_cast<uint64_t>(A.nnzb) * 8 +
           static_cast<uint64_t>(A.nnzb) * 72;
}

} // namespace

void choose_coarse_solver(Hierarchy &H, DevError *err, cudaStream_t s, bool inverse_ok);

Hierarchy::~Hierarchy() {
    if (stream) cudaStreamSynchronize(stream);
    levels.clear();
    Ainv.release();
    lu.X.release(); lu.Lt.release(); lu.perm.release();
    r.release(); z.release(); p.release(); q.release();
    fbuf.release(); ubuf.release(); partials.release(); sc.release(); err.release();
    tail_ph.release(); tail_bar.release();
    pinned_small_free(sc_host);
    pinned_small_free(sc_stage);
    if (cg_exec) cudaGraphExecDestroy(cg_exec);
    if (stream && owns_stream) {
        cudaStreamSynchronize(stream);
        cudaStreamDestroy(stream);
    }
}

uint64_t Hierarchy::memory_footprint() const {
    // memory_footprint (hierarchy.hpp:443-458).  The scalar pipelines keep
    // scalar CSR level matrices in the reference (hierarchy.hpp:309-327):
    // their bytes are counted as such -- 9 scalar entries (8-byte index +
    // 8-byte value) per stored 3x3 block, 3 row pointers per block row --
    // although the B200 stores the same values as 3x3 blocks.
    const bool scalar = pipeline == SAMG_PIPELINE_SCALAR || pipeline == SAMG_PIPELINE_NS_SCALAR;
    auto mbytes = [&](const Bsr3 &M) {
        return scalar ? static_cast<uint64_t>(3 * M.nrows + 1) * 8 + static_cast<uint64_t>(M.nnzb) * 9 * 16
                      : matrix_bytes(M);
    };
    // `scalar` with omega 0: P is the indicator tentative operator, one scalar
    // entry per row (the diagonal of each stored block; coarsening.hpp:326)
    const bool diag_transfer = pipeline == SAMG_PIPELINE_SCALAR && prm.omega == 0.0;
    auto tbytes = [&](const Bsr3 &M) {
        return diag_transfer ? static_cast<uint64_t>(3 * M.nrows + 1) * 8 + static_cast<uint64_t>(M.nnzb) * 3 * 16
                             : mbytes(M);
    };
    uint64_t bytes = 0;
    for (const Level &lv : levels) {
        bytes += mbytes(lv.A);
        if (lv.has_transfer) {
            bytes += tbytes(lv.P);
            bytes += tbytes(lv.R);
        }
        if (lv.M.kind == SM_ILU && lv.M.scalar)  // ilu0<double>::bytes: scalar factors + pivots
            bytes += static_cast<uint64_t>(3 * lv.M.nrows + 1) * 8 + static_cast<uint64_t>(lv.M.nnzb) * 9 * 16 +
                     static_cast<uint64_t>(lv.M.nrows) * 24;
        else if (lv.M.kind == SM_ILU)  // ilu0::bytes (relaxation.hpp:93-95)
            bytes += static_cast<uint64_t>(lv.M.nrows + 1) * 8 + static_cast<uint64_t>(lv.M.nnzb) * 80 +
                     static_cast<uint64_t>(lv.M.nrows) * 72;
        else
            bytes += lv.M.data.n * 8;
    }
    bytes += static_cast<uint64_t>(nc) * nc * 8;
    return bytes;
}

Hierarchy *setup_hierarchy(Bsr3 &&A0, const double *B_host, int64_t b_rows, int64_t b_cols,
                           const samg_amg_params &prm, cudaStream_t s, double t_start, int pipeline,
                           GalerkinSlicer *slicer, int first_level) {
    NvtxScope nvtx_scope("samg::setup");
    auto H = std::make_unique<Hierarchy>();
    H->stream = s;
    H->prm = prm;
    H->pipeline = pipeline;
    // the hybrids run the scalar-space setup (hierarchy.hpp:233-260): the
    // same transfer operators, the Galerkin product in scalar arithmetic
    // (and so do the scalar pipelines, hierarchy.hpp:298-330, whose level
    // matrices are the same values in scalar CSR)
    const bool scalar_galerkin =
        pipeline == SAMG_PIPELINE_NS_HYBRID1 || pipeline == SAMG_PIPELINE_NS_HYBRID2 ||
        pipeline == SAMG_PIPELINE_SCALAR || pipeline == SAMG_PIPELINE_NS_SCALAR;
    // `scalar`: no nullspace; the indicator tentative operator with point
    // block size 3 on every level (hierarchy.hpp:284-285, coarsening.hpp:249-266)
    const bool indicator = pipeline == SAMG_PIPELINE_SCALAR;
    CK(cudaGetDevice(&H->device));
    H->err.alloc(1, s);
    CK(cudaMemsetAsync(H->err.p, 0, sizeof(DevError), s));
    DevError *err = H->err.p;

    // SAMG_SETUP_TIMING=1: per-phase wall times on stderr (synchronises
    // after every phase; diagnosis only)
    static const bool timing = [] {
        const char *e = std::getenv("SAMG_SETUP_TIMING");
        return e && e[0] == '1';
    }();
    double t_mark = t_start;
    auto mark = [&](const char *what, size_t level) {
        // an NVTX marker at the end of every setup phase (Nsight timelines:
        // the phases between the markers inside the samg::setup range)
        char nv[64];
        std::snprintf(nv, sizeof nv, "setup L%zu %s done", level, what);
        nvtxMarkA(nv);
        if (!timing) return;
        CK(cudaStreamSynchronize(s));
        const double t = now_s();
        std::fprintf(stderr, "setup L%zu %-12s %8.3f ms\n", level, what, 1e3 * (t - t_mark));
        t_mark = t;
    };
    mark("upload", 0);
    // Grow the stream-ordered pool once to the setup's working set (the
    // level-0 Galerkin intermediate R*A alone is ~1.1x A_0): growing it piece
    // by piece inside the level loop maps fresh physical memory per
    // allocation (C4: 0.1-0.5 s per Galerkin allocation).  The pool keeps it
    // (release threshold = max), so later setups reuse it.
    {
        static const double factor = [] {
            const char *e = std::getenv("SAMG_POOL_RESERVE");
            return e ? std::atof(e) : 2.5;
        }();
        const double a_bytes = static_cast<double>(A0.nnzb) * 76.0 + 4.0 * A0.nrows;
        if (factor > 0.0 && a_bytes * factor > 64.0 * (1 << 20)) {
            cudaMemPool_t pool;
            CK(cudaDeviceGetDefaultMemPool(&pool, H->device));
            uint64_t reserved = 0, used = 0;
            CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
            CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
            size_t free_b = 0, total_b = 0;
            CK(cudaMemGetInfo(&free_b, &total_b));
            const double want = std::min(a_bytes * factor, 0.7 * static_cast<double>(free_b + (reserved - used)));
            if (timing)
                std::fprintf(stderr, "setup pool: reserved %.2f GB used %.2f GB free %.2f GB want %.2f GB\n",
                             reserved / 1e9, used / 1e9, free_b / 1e9, want / 1e9);
            if (want > static_cast<double>(reserved - used)) {
                void *tmp = nullptr;
                if (cudaMallocAsync(&tmp, static_cast<size_t>(want), s) == cudaSuccess)
                    CK(cudaFreeAsync(tmp, s));
                else
                    cudaGetLastError();
            }
        }
        mark("pool", 0);
    }
    const bool block = pipeline == SAMG_PIPELINE_BLOCK;  // no nullspace
    const int k = block ? 0 : (indicator ? 3 : static_cast<int>(b_cols));
    DevBuf<double> B;
    if (!block && !indicator) {
        B.alloc(b_rows * b_cols, s);
        // B may be host (pageable/pinned) or device memory (samg_setup_device)
        CK(cudaMemcpyAsync(B.p, B_host, sizeof(double) * b_rows * b_cols, cudaMemcpyDefault, s));
    }

    H->levels.emplace_back();
    H->levels.back().A = std::move(A0);
    // level loop (hierarchy.hpp:338-363)
    while (3 * H->levels.back().A.nrows > prm.coarse_enough) {
        Level &Li = H->levels.back();
        const size_t lvl = H->levels.size() - 1;
        if (block) {
            // block pipeline (hierarchy.hpp:340-347): Frobenius-norm block
            // strength, block_transfer_operators (coarsening.hpp:471-560)
            Graph G;
            strength_graph(Li.A, 1, prm.eps_strong, G, s, true);
            mark("strength", lvl);
            DevBuf<int> agg;
            DevBuf<int> seedno;
            const int64_t naggs = aggregate(G, agg, s, &seedno);
            mark("aggregate", lvl);
            Bsr3 P;
            block_transfer(Li.A, G, agg, naggs, prm.omega, P, err, s);
            check_dev_error(err, s);
            mark("block_P", lvl);
            if (static_cast<double>(3 * P.ncols) >
                prm.stagnation_ratio * static_cast<double>(3 * Li.A.nrows))
                break;
            Bsr3 R;
            transpose(P, R, s);
            Bsr3 Ac;
            if (!slicer || !slicer->galerkin(lvl, Li.A, seedno.p, G.nnodes, naggs, R, P, Ac, false, s))
                galerkin(R, Li.A, P, Ac, s);
            fix_decoupled_rows(Ac, s);
            mark("galerkin", lvl);
            Li.P = std::move(P);
            Li.R = std::move(R);
            Li.has_transfer = true;
            Li.agg = std::move(agg);
            Li.nnodes = G.nnodes;
            Li.naggs = naggs;
            Li.seedno = std::move(seedno);
            H->levels.emplace_back();
            H->levels.back().A = std::move(Ac);
            continue;
        }
        // ns pipelines force point_block_size = 3 on the fine level
        // (hierarchy.hpp:284-285), then use the nullspace width (:351-353)
        const int pbs = (H->levels.size() == 1 && first_level == 0) || indicator ? 3 : k;
        if (pbs % 3) fail(SAMG_NOT_DIVISIBLE, "ns_block: node size must be a multiple of 3");
        const int h = pbs / 3;
        if (Li.A.nrows % h)
            fail(SAMG_NOT_DIVISIBLE, "strength_graph: rows not divisible by point block size");
        Graph G;
        strength_graph(Li.A, h, prm.eps_strong, G, s);
        mark("strength", lvl);
        DevBuf<int> agg;
        DevBuf<int> seedno;
        const int64_t naggs = aggregate(G, agg, s, &seedno);
        mark("aggregate", lvl);
        DevBuf<double> Pt, Bc;
        if (indicator) tentative_indicator(agg, G.nnodes, naggs, pbs, Pt, s);
        else tentative(agg, G.nnodes, naggs, pbs, B.p, k, Pt, Bc, err, s);
        mark("tentative", lvl);
        Bsr3 P;
        smooth_prolongation(Li.A, G, agg, naggs, pbs, indicator ? 0 : k, Pt.p, prm.omega, P, err, s);
        check_dev_error(err, s);
        mark("smooth_P", lvl);
        // stagnation guard (hierarchy.hpp:355)
        if (static_cast<double>(3 * P.ncols) >
            prm.stagnation_ratio * static_cast<double>(3 * Li.A.nrows))
            break;
        Bsr3 R;
        transpose(P, R, s);
        mark("transpose", lvl);
        // Galerkin (csr.hpp:259-262) + fix_decoupled_rows (hierarchy.hpp:357)
        Bsr3 Ac;
        if (!slicer ||
            !slicer->galerkin(lvl, Li.A, seedno.p, G.nnodes, naggs, R, P, Ac, scalar_galerkin, s))
            galerkin(R, Li.A, P, Ac, s, scalar_galerkin);
        fix_decoupled_rows(Ac, s);
        mark("galerkin", lvl);
        Li.P = std::move(P);
        Li.R = std::move(R);
        Li.has_transfer = true;
        Li.agg = std::move(agg);
        Li.nnodes = G.nnodes;
        Li.naggs = naggs;
        Li.seedno = std::move(seedno);
        B = std::move(Bc);
        b_rows = naggs * k;
        H->levels.emplace_back();
        H->levels.back().A = std::move(Ac);
    }
    B.release();
    const size_t L = H->levels.size();
    // the scalar pipelines and ns_hybrid1 smooth with scalar smoothers
    // (hierarchy.hpp:288-291): ILU(0) is ilu0<double> of the scalar view
    const bool scalar_smoothers = pipeline == SAMG_PIPELINE_SCALAR ||
                                  pipeline == SAMG_PIPELINE_NS_SCALAR ||
                                  pipeline == SAMG_PIPELINE_NS_HYBRID1;
    for (size_t i = 0; i + 1 < L; ++i) {
        if (scalar_smoothers && prm.smoother == SAMG_SMOOTHER_ILU0)
            setup_ilu0_scalar(H->levels[i].A, H->levels[i].M, err, s);
        else
            setup_smoother(H->levels[i].A, prm.smoother, prm.smoother_omega, H->levels[i].M, err, s);
        H->levels[i].M.latest_last = prm.ilu_sweep_order == SAMG_ILU_ORDER_LATEST_LAST;
    }
    check_dev_error(err, s);
    mark("smoothers", L - 1);
    if (prm.vcycle_precision == SAMG_PRECISION_MIXED) {
        // fp32 value copies of every operator the V-cycle streams (A_l, P_l,
        // R_l above the coarsest level); CG's q = A p and the true residual
        // keep reading the fp64 values
        for (size_t i = 0; i + 1 < L; ++i) {
            make_lowp(H->levels[i].A, s);
            make_lowp(H->levels[i].P, s);
            make_lowp(H->levels[i].R, s);
        }
        mark("fp32_copies", L - 1);
    }
    if (prm.verify_galerkin) {
        // hierarchy.hpp:382-401: recompute every A_{i+1} as the scalar
        // Galerkin product of the stored R_i, A_i, P_i (+ fix_decoupled_rows)
        // and compare on the union pattern, relative squared Frobenius 1e-24
        for (size_t i = 0; i + 1 < L; ++i) {
            Bsr3 G;
            galerkin(H->levels[i].R, H->levels[i].A, H->levels[i].P, G, s, true);
            fix_decoupled_rows(G, s);
            double dr[2];
            union_diff(H->levels[i + 1].A, G, dr, s);
            if (dr[0] > 1e-24 * dr[1])
                fail(SAMG_ERROR, "setup: Galerkin consistency check failed on level " +
                                     std::to_string(i));
        }
        mark("verify_galerkin", L - 1);
    }
    // 6x6 node-blocked copies of the operators of levels >= 1 (pbs 6 nodes:
    // rows and columns pair up) for the V-cycle's SpMVs.  Opt-in
    // (SAMG_NODE6=1): measured slower than the 3x3 kernels on C1's levels 1
    // and 2 (35.5 -> 39.9 us and 17.3 -> 28.5 us per residual; DESIGN 5.9)
    if (!block && k == 6) {
        static const bool node6 = [] {
            const char *e = std::getenv("SAMG_NODE6");
            return e && e[0] == '1';
        }();
        for (size_t i = (first_level > 0 ? 0 : 1); node6 && i + 1 < L; ++i) {
            make_node6(H->levels[i].A, s);
            make_node6(H->levels[i].P, s);
            make_node6(H->levels[i].R, s);
        }
        mark("node6", L - 1);
    }
    H->nc = 3 * H->levels.back().A.nrows;
    const bool inverse_ok = dense_inverse(H->levels.back().A, H->Ainv, err, s);
    mark("dense_inv", L - 1);
    choose_coarse_solver(*H, err, s, inverse_ok);
    mark("coarse_check", L - 1);
    // V-cycle / CG workspace
    for (size_t i = 0; i < L; ++i) {
        Level &lv = H->levels[i];
        const int64_t n = 3 * lv.A.nrows;
        lv.f.alloc(n, s); lv.u.alloc(n, s); lv.r.alloc(n, s); lv.t.alloc(n, s);
    }
    const int64_t n0 = H->finest_dim();
    H->r.alloc(n0, s); H->z.alloc(n0, s); H->p.alloc(n0, s); H->q.alloc(n0, s);
    H->fbuf.alloc(n0, s); H->ubuf.alloc(n0, s);
    // one partial per CTA of any fused reduction (<= 148*8 CTAs)
    const int64_t np = 4096;
    H->partials.alloc(np, s);
    H->sc.alloc(1, s);
    CK(cudaMemsetAsync(H->sc.p, 0, sizeof(CgScalars), s));
    H->sc_host = static_cast<CgScalars *>(pinned_small_alloc(sizeof(CgScalars)));
    H->sc_stage = static_cast<CgScalars *>(pinned_small_alloc(sizeof(CgScalars)));
    H->build_tail();
    CK(cudaStreamSynchronize(s));
    mark("workspace", L - 1);
    if (timing) {  // the pool's high-water mark over this setup (SAMG_POOL_RESERVE tuning)
        cudaMemPool_t pool;
        uint64_t high = 0, reserved = 0, used = 0;
        if (cudaDeviceGetDefaultMemPool(&pool, H->device) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &high) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess)
            std::fprintf(stderr, "setup pool after: used %.2f GB (high-water %.2f GB) reserved %.2f GB\n",
                         used / 1e9, high / 1e9, reserved / 1e9);
    }
    H->setup_seconds = now_s() - t_start;
    H->owns_stream = true;
    return H.release();
}

// The explicit inverse is checked once: x random, b = A_c x (the sparse
// coarse operator), e = |Ainv b - x| / |x|.  A well-conditioned coarse
// operator gives e ~ cond * 1e-16; e > 1e-6 means A_c is numerically singular
// and its solve is decided by rounding -- then (n <= kLuMaxN) the coarse
// solve switches to the reference's own LU, bit-exact (coarse_lu.cu).
// SAMG_COARSE_SOLVER=inverse|lu forces either.
void choose_coarse_solver(Hierarchy &H, DevError *err, cudaStream_t s, bool inverse_ok) {
    static const int forced = [] {
        const char *e = std::getenv("SAMG_COARSE_SOLVER");
        if (!e) return 0;
        return std::string(e) == "lu" ? 2 : (std::string(e) == "inverse" ? 1 : 0);
    }();
    const Bsr3 &Ac = H.levels.back().A;
    const int64_t n = H.nc;
    bool use_lu = forced == 2 || !inverse_ok;
    if (!inverse_ok && n > kLuMaxN)
        fail(SAMG_ERROR, "dense coarse solve: Gauss-Jordan pivot below 1e-300 and the coarsest "
                         "level (" + std::to_string(n) + " unknowns) is too large for the LU "
                         "fallback");
    if (!use_lu && forced == 0 && n > 0 && n <= kLuMaxN) {
        std::vector<double> hx(n);
        uint64_t st = 0x9e3779b97f4a7c15ull;
        for (auto &v : hx) {  // xorshift, uniform in [-1, 1)
            st ^= st << 13; st ^= st >> 7; st ^= st << 17;
            v = static_cast<double>(st >> 11) * 0x1.0p-52 - 1.0;
        }
        DevBuf<double> x(n, s), b(n, s), y(n, s);
        CK(cudaMemcpyAsync(x.p, hx.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
        launch_spmv(Ac, 1.0, x.p, 0.0, b.p, s);
        launch_dense_gemv(n, H.Ainv.p, b.p, y.p, s);
        std::vector<double> hy(n);
        CK(cudaMemcpyAsync(hy.data(), y.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double num = 0.0, den = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            num += (hy[i] - hx[i]) * (hy[i] - hx[i]);
            den += hx[i] * hx[i];
        }
        use_lu = !(std::sqrt(num / den) <= 1e-6);
    }
    if (!use_lu || n > kLuMaxN) return;
    dense_lu_ref(Ac, H.lu, err, s);
    H.coarse_lu = true;
    H.Ainv.release();
}

// The V-cycle's small levels as one persistent launch (k_vtail, solve.cu).
// tail_start t = the first level >= 1 whose operator is at most
// SAMG_VTAIL_MB (default 96) MB; the phases replay vcycle_from's level
// loop for levels t..L-1 exactly (same kernels' arithmetic, same buffers,
// same ping-pong), starting with level t-1's restriction and ending with its
// prolongation, whose target (level t-1's current iterate) is passed at
// launch.  Needs block / point smoothers on the tail levels, the explicit
// coarse inverse and the fp64 V-cycle; SAMG_VTAIL=0 disables.
void Hierarchy::build_tail() {
    static const int on = [] {
        const char *e = std::getenv("SAMG_VTAIL");
        return e ? std::atoi(e) : 0;
    }();
    static const double mb = [] {
        const char *e = std::getenv("SAMG_VTAIL_MB");
        return e ? std::atof(e) : 96.0;
    }();
    tail_nph = 0;
    const size_t L = levels.size();
    if (!on || L < 2 || coarse_lu || !Ainv.p || prm.vcycle_precision == SAMG_PRECISION_MIXED) return;
    size_t t = L - 1;
    for (size_t i = 1; i + 1 < L; ++i)
        if (levels[i].A.nnzb * 76.0 <= mb * 1e6) { t = i; break; }
    for (size_t i = t; i + 1 < L; ++i)
        if (levels[i].M.kind != SM_POINT && levels[i].M.kind != SM_BLOCK) return;
    const int64_t ld = dense_ld(nc);
    const size_t smem = static_cast<size_t>(8 * ld) <= 96 * 1024 ? static_cast<size_t>(8 * ld) : 0;
    const int grid = vtail_grid(smem);
    if (grid <= 0) return;
    const int64_t threads = static_cast<int64_t>(grid) * 1024;  // kVtThreads per CTA
    std::vector<VPhase> ph;
    auto mat = [&](int kind, const Bsr3 &A, const double *x) {
        VPhase v{};
        v.kind = kind;
        v.nrows = static_cast<int>(A.nrows);
        v.G = vtail_group(A.nrows, A.nnzb, threads);
        v.ptr = A.ptr.p; v.col = A.col.p; v.val = A.val.p; v.x = x;
        v.alpha = 1.0;
        return v;
    };
    auto restrict_into = [&](size_t i) {  // level i's residual -> level i+1 (+ first sweep)
        Level &lv = levels[i], &nx = levels[i + 1];
        if (i + 2 < L && prm.pre_sweeps > 0) {
            VPhase v = mat(nx.M.kind == SM_BLOCK ? VP_RSMOOTH_B : VP_RSMOOTH_P, lv.R, lv.r.p);
            v.out = nx.f.p; v.out2 = nx.u.p; v.m = nx.M.data.p;
            ph.push_back(v);
            return true;
        }
        VPhase v = mat(VP_SPMV, lv.R, lv.r.p);
        v.out = nx.f.p; v.beta = 0.0;
        ph.push_back(v);
        return false;
    };
    std::vector<double *> cur(L, nullptr);
    bool pre = restrict_into(t - 1);
    for (size_t i = t; i + 1 < L; ++i) {
        Level &lv = levels[i];
        double *a = lv.u.p, *b = lv.t.p;
        int sweeps = prm.pre_sweeps;
        if (sweeps > 0) {
            if (!pre) return;  // (not reached: block / point smoothers fuse it)
            --sweeps;
        } else {
            VPhase v{};
            v.kind = VP_FILL; v.nrows = static_cast<int>(lv.A.nrows); v.out = a; v.alpha = 0.0;
            ph.push_back(v);
        }
        for (; sweeps > 0; --sweeps) {
            VPhase v = mat(lv.M.kind == SM_BLOCK ? VP_SMOOTH_B : VP_SMOOTH_P, lv.A, a);
            v.f = lv.f.p; v.m = lv.M.data.p; v.out = b;
            ph.push_back(v);
            std::swap(a, b);
        }
        VPhase r = mat(VP_RESIDUAL, lv.A, a);
        r.f = lv.f.p; r.out = lv.r.p;
        ph.push_back(r);
        pre = restrict_into(i);
        cur[i] = a;
    }
    {
        VPhase g{};
        g.kind = VP_GEMV; g.nrows = static_cast<int>(nc); g.ld = ld; g.val = Ainv.p;
        g.x = levels[L - 1].f.p; g.out = levels[L - 1].u.p;
        ph.push_back(g);
        cur[L - 1] = levels[L - 1].u.p;
    }
    for (size_t ii = L - 1; ii-- > t;) {
        Level &lv = levels[ii];
        double *a = cur[ii];
        double *b = (a == lv.u.p) ? lv.t.p : lv.u.p;
        VPhase pr = mat(VP_SPMV, lv.P, cur[ii + 1]);
        pr.out = a; pr.beta = 1.0;
        ph.push_back(pr);
        for (int sw = prm.post_sweeps; sw > 0; --sw) {
            VPhase v = mat(lv.M.kind == SM_BLOCK ? VP_SMOOTH_B : VP_SMOOTH_P, lv.A, a);
            v.f = lv.f.p; v.m = lv.M.data.p; v.out = b;
            ph.push_back(v);
            std::swap(a, b);
        }
        cur[ii] = a;
    }
    {
        VPhase pr = mat(VP_SPMV, levels[t - 1].P, cur[t]);
        pr.beta = 1.0; pr.last_out = 1;
        ph.push_back(pr);
    }
    cudaStream_t s = stream;
    tail_ph.alloc(ph.size(), s);
    CK(cudaMemcpyAsync(tail_ph.p, ph.data(), sizeof(VPhase) * ph.size(), cudaMemcpyHostToDevice, s));
    tail_bar.alloc(2, s);
    CK(cudaMemsetAsync(tail_bar.p, 0, 2 * sizeof(unsigned), s));
    CK(cudaStreamSynchronize(s));
    tail_nph = static_cast<int>(ph.size());
    if (std::getenv("SAMG_VTAIL_TRACE")) {
        tail_trace.alloc(2 * ph.size() + 1 + static_cast<size_t>(grid) * (ph.size() + 1), s);
        CK(cudaMemsetAsync(tail_trace.p, 0, tail_trace.bytes(), s));
    }
    tail_grid = grid;
    tail_start = t;
    tail_smem = smem;
}

void Hierarchy::coarse_solve(const double *f, double *u) {
    if (coarse_lu) launch_lu_solve(lu, f, u, stream);
    else launch_dense_gemv(nc, Ainv.p, f, u, stream);
}

// V-cycle (hierarchy.hpp:408-441).  With zero_guess the pre-smoother's first
// sweep needs no SpMV (r = f - A*0 = f exactly), as inside CG (cg.hpp:98-101)
// and on every level > 0 (hierarchy.hpp:426).
// With fuse_rz (inside CG) the last level-0 sweep also forms r.z and
// finishes the CG beta update; returns whether it did.
bool Hierarchy::vcycle(const double *f0, double *u0, bool zero_guess, bool fuse_rz) {
    return vcycle_from(0, f0, u0, zero_guess, fuse_rz);
}

// The V-cycle restricted to levels start..L-1 (f0, u0 live on level
// `start`); the multi-GPU driver runs the replicated coarse levels this way.
bool Hierarchy::vcycle_from(size_t start, const double *f0, double *u0, bool zero_guess,
                            bool fuse_rz, bool presmoothed) {
    cudaStream_t s = stream;
    const size_t L = levels.size();
    const bool lowp = prm.vcycle_precision == SAMG_PRECISION_MIXED;
    if (start + 1 >= L) {
        coarse_solve(f0, u0);
        return false;
    }
    bool fused = false, tail_used = false;
    std::vector<double *> cur(L);
    // pre: the first sweep from a zero guess of this level was fused into
    // the kernel that produced its f (u = M f already in lv.u)
    bool pre = presmoothed && zero_guess && prm.pre_sweeps > 0;
    for (size_t i = start; i + 1 < L; ++i) {
        Level &lv = levels[i];
        const double *fi = i == start ? f0 : lv.f.p;
        double *a = lv.u.p, *b = lv.t.p;
        int sweeps = prm.pre_sweeps;
        const bool zero = (i > start) || zero_guess;
        if (!zero) CK(cudaMemcpyAsync(a, u0, sizeof(double) * 3 * lv.A.nrows, cudaMemcpyDeviceToDevice, s));
        if (zero) {
            if (sweeps > 0) {
                if (!pre) launch_smooth_zero(lv.A.nrows, lv.M, fi, a, s);
                --sweeps;
            } else {
                launch_fill(3 * lv.A.nrows, 0.0, a, s);
            }
        }
        for (; sweeps > 0; --sweeps) {
            launch_smooth(lv.A, lv.M, fi, a, b, s, lowp);
            std::swap(a, b);
        }
        launch_residual(lv.A, fi, a, lv.r.p, s, lowp);
        if (tail_nph && i + 1 == tail_start) {
            // levels i+1 .. L-1 and the prolongation into `a` in one launch
            launch_vtail(tail_ph.p, tail_nph, tail_bar.p, tail_grid, tail_smem, dense_ld(nc), a, s,
                         tail_trace.p);
            cur[i] = a;
            tail_used = true;
            break;
        }
        // restriction, fused with the next level's first sweep from zero
        // when that level has a block-diagonal smoother
        Level &nx = levels[i + 1];
        pre = false;
        if (i + 2 < L && prm.pre_sweeps > 0)
            pre = launch_restrict_smooth(lv.R, lv.r.p, nx.f.p, nx.M, nx.u.p, s, lowp);
        if (!pre) launch_spmv(lv.R, 1.0, lv.r.p, 0.0, nx.f.p, s, lowp);
        cur[i] = a;
    }
    if (!tail_used) {
        coarse_solve(levels[L - 1].f.p, levels[L - 1].u.p);
        cur[L - 1] = levels[L - 1].u.p;
    }
    for (size_t ii = tail_used ? tail_start : L - 1; ii-- > start;) {
        Level &lv = levels[ii];
        const double *fi = ii == start ? f0 : lv.f.p;
        double *a = cur[ii];
        double *b = (a == lv.u.p) ? lv.t.p : lv.u.p;
        if (!(tail_used && ii + 1 == tail_start)) launch_spmv(lv.P, 1.0, cur[ii + 1], 1.0, a, s, lowp);
        for (int sw = prm.post_sweeps; sw > 0; --sw) {
            const bool last0 = ii == start && sw == 1;
            double *out = last0 ? u0 : b;
            if (last0 && fuse_rz) {
                launch_smooth_dot(lv.A, lv.M, fi, a, out, partials.p, sc.p, s, CG_RZ, lowp);
                fused = true;
            } else {
                launch_smooth(lv.A, lv.M, fi, a, out, s, lowp);
            }
            b = a;
            a = out;
        }
        cur[ii] = a;
    }
    if (cur[start] != u0)
        CK(cudaMemcpyAsync(u0, cur[start], sizeof(double) * 3 * levels[start].A.nrows,
                           cudaMemcpyDeviceToDevice, s));
    return fused;
}

// One CG iteration (cg.hpp:63-77) on the internal buffers, as recorded into
// the body of the graph's while node.  The loop condition is set by
// k_finalize_loop right after ||r|| is known; the V-cycle and p update that
// follow in the same pass are then unused on the last pass (u and r are
// final before them).
void Hierarchy::build_cg_graph() {
    cudaStream_t s = stream;
    const int64_t n = finest_dim();
    const Bsr3 &A0 = levels.front().A;
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t wnode;
    CK(cudaGraphAddNode(&wnode, g, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    launch_spmv_dot(A0, p.p, q.p, partials.p, sc.p, s);
    // r -= alpha q, r.r and the loop condition, fused with the V-cycle's
    // first level-0 sweep z0 = M r; u += alpha p is deferred to the p update
    const bool fz = prm.pre_sweeps > 0 && levels.size() > 1 &&
                    launch_cg_update_smooth(A0.nrows, sc.p, q.p, r.p, levels[0].M, levels[0].u.p,
                                            partials.p, CG_RR_LOOP, h, s);
    if (!fz) launch_cg_update(n, sc.p, p.p, q.p, ubuf.p, r.p, partials.p, CG_RR_LOOP, h, s);
    if (!vcycle_from(0, r.p, z.p, true, true, fz)) launch_dot(n, r.p, z.p, partials.p, sc.p, CG_RZ, s);
    if (fz) launch_p_update_u(n, sc.p, z.p, p.p, ubuf.p, s);
    else launch_p_update(n, sc.p, z.p, p.p, s);
    cudaGraph_t captured = body;
    CK(cudaStreamEndCapture(s, &captured));
    CK(cudaGraphInstantiate(&cg_exec, g, 0));
    CK(cudaGraphDestroy(g));
}

// PCG from a zero guess (cg_solve_op, cg.hpp:39-83, and cg_solve(hierarchy),
// cg.hpp:87-112).  alpha/beta stay on the device.  By default the whole
// iteration loop runs as one CUDA graph with a device-side while condition
// (no host round trip per iteration); SAMG_CG_GRAPH=0 selects the host loop
// that reads ||r|| back every iteration.
samg_solve_report Hierarchy::cg(const double *d_f, double *d_u, const samg_cg_params &cp) {
    NvtxScope nvtx_scope("samg::cg_solve");
    static const bool use_graph = [] {
        const char *e = std::getenv("SAMG_CG_GRAPH");
        return !(e && e[0] == '0');
    }();
    cudaStream_t s = stream;
    const double t0 = now_s();
    samg_solve_report rep{};
    rep.variant = pipeline;
    rep.setup_seconds = setup_seconds;
    const int64_t n = finest_dim();
    const Bsr3 &A0 = levels.front().A;
    double *pr = r.p, *pz = z.p, *pp = p.p, *pq = q.p, *pu = ubuf.p;
    CK(cudaMemcpyAsync(pr, d_f, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    launch_fill(n, 0.0, pu, s);
    CK(cudaMemsetAsync(sc.p, 0, sizeof(CgScalars), s));
    launch_dot(n, pr, pr, partials.p, sc.p, CG_RR, s);  // r = f (internal, aligned)
    CK(cudaMemcpyAsync(sc_host, sc.p, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const double norm_f = std::sqrt(sc_host->rr);
    if (norm_f == 0.0) {
        if (pu != d_u)
            CK(cudaMemcpyAsync(d_u, pu, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        CK(cudaStreamSynchronize(s));
        rep.converged = 1;
        rep.relative_residual = 0.0;
        rep.preconditioner_bytes = memory_footprint();
        rep.solve_seconds = now_s() - t0;
        return rep;
    }
    vcycle(pr, pz, true, false);
    launch_dot(n, pr, pz, partials.p, sc.p, CG_RHO, s);
    CK(cudaMemcpyAsync(pp, pz, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    double res_norm = norm_f;
    int iter = 0;
    if (use_graph && norm_f / norm_f > cp.tol && cp.max_iterations > 0) {
        sc_stage->norm_f = norm_f;
        sc_stage->tol = cp.tol;
        sc_stage->breakdown = 0;
        sc_stage->iter = 0;
        sc_stage->max_iter = cp.max_iterations;
        sc_stage->ticket = 0;
        const size_t off = offsetof(CgScalars, norm_f);
        CK(cudaMemcpyAsync(reinterpret_cast<char *>(sc.p) + off,
                           reinterpret_cast<char *>(sc_stage) + off, sizeof(CgScalars) - off,
                           cudaMemcpyHostToDevice, s));
        if (!cg_exec) build_cg_graph();
        CK(cudaGraphLaunch(cg_exec, s));
        CK(cudaMemcpyAsync(sc_host, sc.p, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (sc_host->breakdown)
            fail(SAMG_BREAKDOWN_NON_SPD, "cg: p'Ap <= 0, matrix or preconditioner not SPD");
        iter = sc_host->iter;
        res_norm = std::sqrt(sc_host->rr);
    }
    while (!use_graph && res_norm / norm_f > cp.tol && iter < cp.max_iterations) {
        // the same kernels as the graph body (build_cg_graph)
        launch_spmv_dot(A0, pp, pq, partials.p, sc.p, s);
        const bool fz = prm.pre_sweeps > 0 && levels.size() > 1 &&
                        launch_cg_update_smooth(A0.nrows, sc.p, pq, pr, levels[0].M, levels[0].u.p,
                                                partials.p, CG_RR, 0, s);
        if (!fz) launch_cg_update(n, sc.p, pp, pq, pu, pr, partials.p, CG_RR, 0, s);
        CK(cudaMemcpyAsync(sc_host, sc.p, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (sc_host->breakdown)
            fail(SAMG_BREAKDOWN_NON_SPD, "cg: p'Ap <= 0, matrix or preconditioner not SPD");
        ++iter;
        res_norm = std::sqrt(sc_host->rr);
        if (res_norm / norm_f <= cp.tol || iter >= cp.max_iterations) {
            if (fz) launch_u_update(n, sc.p, pp, pu, s);  // the deferred u += alpha p
            break;
        }
        if (!vcycle_from(0, pr, pz, true, true, fz)) launch_dot(n, pr, pz, partials.p, sc.p, CG_RZ, s);
        if (fz) launch_p_update_u(n, sc.p, pz, pp, pu, s);
        else launch_p_update(n, sc.p, pz, pp, s);
    }
    rep.iterations = iter;
    rep.converged = res_norm / norm_f <= cp.tol;
    // true residual at exit (cg.hpp:105-108)
    launch_residual(A0, d_f, pu, pq, s);
    launch_dot(n, pq, pq, partials.p, sc.p, CG_RR, s);
    CK(cudaMemcpyAsync(sc_host, sc.p, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
    if (pu != d_u)
        CK(cudaMemcpyAsync(d_u, pu, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
    rep.relative_residual = std::sqrt(sc_host->rr) / norm_f;
    rep.preconditioner_bytes = memory_footprint();
    rep.solve_seconds = now_s() - t0;
    if (tail_trace.p) {  // the last tail launch: per phase, CTA 0's end / release and the
                         // spread of the CTAs' phase ends (us from CTA 0's start)
        std::vector<unsigned long long> t(tail_trace.n);
        CK(cudaMemcpy(t.data(), tail_trace.p, tail_trace.bytes(), cudaMemcpyDeviceToHost));
        const int np = tail_nph, g = tail_grid;
        const unsigned long long t0 = t[2 * np];
        const unsigned long long *pe = t.data() + 2 * np + 1;  // [k * g + cta], k = np: start
        std::fprintf(stderr, "vtail trace (%d phases, grid %d)\n", np, g);
        for (int k = 0; k <= np; ++k) {
            std::vector<std::pair<double, int>> v;
            for (int b = 0; b < g; ++b) v.push_back({(static_cast<double>(pe[k * g + b]) - t0) * 1e-3, b});
            std::sort(v.begin(), v.end());
            std::fprintf(stderr, "  %s %d: release %.2f  ends min %.2f med %.2f p90 %.2f max %.2f (cta %d, %d, %d)\n",
                         k < np ? "phase" : "start", k, k < np ? (t[2 * k + 1] - t0) * 1e-3 : 0.0,
                         v[0].first, v[g / 2].first, v[g * 9 / 10].first, v[g - 1].first, v[g - 1].second,
                         v[g - 2].second, v[g - 3].second);
        }
    }
    return rep;
}

} // namespace samgb
