// dsolve.cu -- multi-GPU solve: row-partitioned V-cycle + PCG over NCCL.
//
// One process per GPU (rank).  Every rank builds the same hierarchy with the
// single-GPU setup (deterministic, bit-identical on every rank and to the
// reference), then keeps only its rows of the large levels:
//   * level l (l < Ld) is row-partitioned: fine block rows [f0, f1) of A_l,
//     P_l, the smoother, and coarse block rows [c0, c1) of R_l.  The coarse
//     partition follows the aggregation: aggregate g belongs to the rank that
//     owns its pass-1 seed node, and aggregate ids are numbered in seed order
//     (coarsening.hpp:136-146), so every rank's coarse rows are contiguous;
//   * levels l >= Ld (fewer than min_rows * nranks block rows) are replicated:
//     f_Ld is gathered on every rank (grouped ncclBroadcast) and the coarse
//     V-cycle runs redundantly, so the prolongation into level Ld-1 needs no
//     halo.
// Every local SpMV reads a halo-extended vector: owned entries first, then
// the ghosts sorted by global id (grouped by owner).  Because all ranks hold
// all matrices, each rank derives both sides of every halo plan locally (no
// plan exchange).  A halo exchange is pack kernel + grouped ncclSend/ncclRecv
// on the solve stream.  CG dot products are local fused reductions (the same
// kernels as on one GPU, in STORE mode) + a one-double ncclAllReduce.
#include "nccl_shim.cuh"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <memory>
#include <vector>

#include "hierarchy.cuh"

namespace samgb {

inline void nccl_check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess)
        fail(SAMG_NCCL_ERROR, std::string(what) + " failed: " + nccl().GetErrorString(r));
}
#define NK(x) ::samgb::nccl_check((x), #x)

namespace {

__global__ void k_pack3(int64_t n, const int *idx, const double *x, double *buf) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < 3 * n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k = e / 3;
        buf[e] = x[3 * static_cast<int64_t>(idx[k]) + (e - 3 * k)];
    }
}

std::vector<int> download_int(const DevBuf<int> &b, size_t n, cudaStream_t s) {
    std::vector<int> h(n);
    if (n) CK(cudaMemcpyAsync(h.data(), b.p, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return h;
}

int owner(const std::vector<int64_t> &starts, int64_t g) {
    return static_cast<int>(std::upper_bound(starts.begin(), starts.end(), g) - starts.begin()) - 1;
}

} // namespace

// Halo plan of one local matrix: ghosts of its column space.
struct HaloPlan {
    int64_t nloc = 0, nghost = 0;
    std::vector<int> send_peers, recv_peers;
    std::vector<int64_t> send_counts, send_offsets, recv_counts, recv_offsets;
    DevBuf<int> send_idx;
    DevBuf<double> sendbuf;

    void exchange(double *xext, ncclComm_t comm, cudaStream_t s) const {
        const int64_t ns = send_idx.n;
        if (ns) {
            int64_t g = (3 * ns + 255) / 256;
            if (g > 4096) g = 4096;
            k_pack3<<<static_cast<int>(g), 256, 0, s>>>(ns, send_idx.p, xext, sendbuf.p);
            CK_LAUNCH();
        }
        if (send_peers.empty() && recv_peers.empty()) return;
        NK(nccl().GroupStart());
        for (size_t p = 0; p < send_peers.size(); ++p)
            NK(nccl().Send(sendbuf.p + 3 * send_offsets[p], 3 * send_counts[p], ncclDouble,
                        send_peers[p], comm, s));
        for (size_t p = 0; p < recv_peers.size(); ++p)
            NK(nccl().Recv(xext + 3 * (nloc + recv_offsets[p]), 3 * recv_counts[p], ncclDouble,
                        recv_peers[p], comm, s));
        NK(nccl().GroupEnd());
    }
};

// A row slice of a level matrix with columns renumbered into the
// halo-extended vector of `plan` (or kept global when `global_cols`).
struct LocalMat {
    Bsr3 A;
    HaloPlan plan;
};

// Build rank r's slice of the matrix (host structure hptr/hcol, device
// values dval) whose rows are partitioned by row_starts and whose column
// space is partitioned by col_starts.
void build_local(const std::vector<int> &hptr, const std::vector<int> &hcol, const double *dval,
                 const std::vector<int64_t> &row_starts, const std::vector<int64_t> &col_starts,
                 int rank, bool global_cols, int64_t ncols_global, LocalMat &out, cudaStream_t s) {
    const int nranks = static_cast<int>(row_starts.size()) - 1;
    const int64_t r0 = row_starts[rank], r1 = row_starts[rank + 1];
    const int64_t c0 = col_starts[rank], c1 = col_starts[rank + 1];
    const int64_t nl = r1 - r0, base = hptr[r0], nnz = hptr[r1] - base;
    HaloPlan &pl = out.plan;
    std::vector<int64_t> ghost;
    if (!global_cols) {
        for (int64_t j = base; j < base + nnz; ++j)
            if (hcol[j] < c0 || hcol[j] >= c1) ghost.push_back(hcol[j]);
        std::sort(ghost.begin(), ghost.end());
        ghost.erase(std::unique(ghost.begin(), ghost.end()), ghost.end());
        pl.nloc = c1 - c0;
        pl.nghost = static_cast<int64_t>(ghost.size());
        for (int64_t k = 0; k < pl.nghost;) {
            const int q = owner(col_starts, ghost[k]);
            int64_t e = k;
            while (e < pl.nghost && ghost[e] < col_starts[q + 1]) ++e;
            pl.recv_peers.push_back(q);
            pl.recv_counts.push_back(e - k);
            pl.recv_offsets.push_back(k);
            k = e;
        }
        // send side: what every other rank's slice reads from my columns
        std::vector<int> sidx;
        std::vector<int64_t> need;
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            need.clear();
            for (int64_t j = hptr[row_starts[q]]; j < hptr[row_starts[q + 1]]; ++j)
                if (hcol[j] >= c0 && hcol[j] < c1) need.push_back(hcol[j]);
            if (need.empty()) continue;
            std::sort(need.begin(), need.end());
            need.erase(std::unique(need.begin(), need.end()), need.end());
            pl.send_peers.push_back(q);
            pl.send_counts.push_back(static_cast<int64_t>(need.size()));
            pl.send_offsets.push_back(static_cast<int64_t>(sidx.size()));
            for (int64_t g : need) sidx.push_back(static_cast<int>(g - c0));
        }
        pl.send_idx.alloc(sidx.size(), s);
        if (!sidx.empty())
            CK(cudaMemcpyAsync(pl.send_idx.p, sidx.data(), sizeof(int) * sidx.size(),
                               cudaMemcpyHostToDevice, s));
        pl.sendbuf.alloc(3 * sidx.size() + 3, s);
    } else {
        pl.nloc = ncols_global;
    }
    Bsr3 &A = out.A;
    A.alloc(nl, global_cols ? ncols_global : pl.nloc + pl.nghost, nnz, s);
    std::vector<int> p32(nl + 1), c32(nnz);
    for (int64_t i = 0; i <= nl; ++i) p32[i] = static_cast<int>(hptr[r0 + i] - base);
    for (int64_t j = 0; j < nnz; ++j) {
        const int64_t c = hcol[base + j];
        if (global_cols || (c >= c0 && c < c1)) c32[j] = static_cast<int>(global_cols ? c : c - c0);
        else c32[j] = static_cast<int>(pl.nloc + (std::lower_bound(ghost.begin(), ghost.end(), c) - ghost.begin()));
    }
    CK(cudaMemcpyAsync(A.ptr.p, p32.data(), sizeof(int) * (nl + 1), cudaMemcpyHostToDevice, s));
    if (nnz) {
        CK(cudaMemcpyAsync(A.col.p, c32.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(A.val.p, dval + 9 * base, sizeof(double) * 9 * nnz,
                           cudaMemcpyDeviceToDevice, s));
    }
    CK(cudaStreamSynchronize(s));  // host vectors above go out of scope
}

struct DLevel {
    std::vector<int64_t> fstarts, cstarts;  // partitions of this level and the next
    LocalMat A, R, P;
    bool next_replicated = false;
    Smoother M;
    DevBuf<double> f, uA, rR, t, uP;  // f, t: 3*nloc; uA/rR/uP: halo-extended
};

struct DHierarchy {
    int rank = 0, nranks = 1, device = 0;
    ncclComm_t comm = nullptr;
    std::unique_ptr<Hierarchy> H;
    std::vector<DLevel> dl;
    size_t Ld = 0;
    std::vector<int64_t> ld_starts;     // partition of level Ld (gather pieces)
    DevBuf<double> fLd, uLd;            // replicated level-Ld vectors
    DevBuf<double> r, z, pext, q, u, uext;
    DevBuf<CgScalars> sc;
    CgScalars *sc_host = nullptr;
    DevBuf<double> partials;
    int64_t nloc0 = 0;

    ~DHierarchy() {
        if (H && H->stream) cudaStreamSynchronize(H->stream);
        dl.clear();
        if (sc_host) cudaFreeHost(sc_host);
        if (comm) nccl().CommDestroy(comm);
    }

    cudaStream_t stream() const { return H->stream; }

    // the sum over ranks of sc->tmp, then the CG update `what`
    void allreduce_finish(int what) {
        cudaStream_t s = stream();
        double *t = reinterpret_cast<double *>(reinterpret_cast<char *>(sc.p) + offsetof(CgScalars, tmp));
        NK(nccl().AllReduce(t, t, 1, ncclDouble, ncclSum, comm, s));
        launch_cg_finish(sc.p, what, s);
    }

    void vcycle(const double *f0, double *z0);
    samg_solve_report cg(const double *d_f, double *d_u, const samg_cg_params &cp);
};

// Distributed V-cycle (hierarchy.hpp:408-441) from a zero guess.
void DHierarchy::vcycle(const double *f0, double *z0) {
    cudaStream_t s = stream();
    const int pre = H->prm.pre_sweeps, post = H->prm.post_sweeps;
    for (size_t l = 0; l < Ld; ++l) {
        DLevel &L = dl[l];
        const int64_t nl = L.A.A.nrows;
        const double *f = l == 0 ? f0 : L.f.p;
        if (pre > 0) launch_smooth_zero(nl, L.M, f, L.uA.p, s);
        else launch_fill(3 * nl, 0.0, L.uA.p, s);
        for (int sw = 1; sw < pre; ++sw) {
            L.A.plan.exchange(L.uA.p, comm, s);
            launch_smooth(L.A.A, L.M, f, L.uA.p, L.t.p, s);
            CK(cudaMemcpyAsync(L.uA.p, L.t.p, sizeof(double) * 3 * nl, cudaMemcpyDeviceToDevice, s));
        }
        L.A.plan.exchange(L.uA.p, comm, s);
        launch_residual(L.A.A, f, L.uA.p, L.rR.p, s);
        L.R.plan.exchange(L.rR.p, comm, s);
        double *fc = (l + 1 < Ld) ? dl[l + 1].f.p : fLd.p + 3 * ld_starts[rank];
        launch_spmv(L.R.A, 1.0, L.rR.p, 0.0, fc, s);
    }
    // gather f_Ld on every rank, coarse levels redundantly
    NK(nccl().GroupStart());
    for (int q = 0; q < nranks; ++q) {
        const int64_t o = 3 * ld_starts[q], c = 3 * (ld_starts[q + 1] - ld_starts[q]);
        if (c) NK(nccl().Broadcast(fLd.p + o, fLd.p + o, c, ncclDouble, q, comm, s));
    }
    NK(nccl().GroupEnd());
    H->vcycle_from(Ld, fLd.p, uLd.p, true, false);
    for (size_t l = Ld; l-- > 0;) {
        DLevel &L = dl[l];
        const int64_t nl = L.A.A.nrows;
        const double *f = l == 0 ? f0 : L.f.p;
        const double *uc;
        if (L.next_replicated) {
            uc = uLd.p;
        } else {
            // level l+1's result (in its t or uA) -> local part of uP, then halo
            const DLevel &N = dl[l + 1];
            const double *src = post > 0 ? N.t.p : N.uA.p;
            CK(cudaMemcpyAsync(L.uP.p, src, sizeof(double) * 3 * N.A.A.nrows,
                               cudaMemcpyDeviceToDevice, s));
            L.P.plan.exchange(L.uP.p, comm, s);
            uc = L.uP.p;
        }
        launch_spmv(L.P.A, 1.0, uc, 1.0, L.uA.p, s);
        for (int sw = 0; sw < post; ++sw) {
            L.A.plan.exchange(L.uA.p, comm, s);
            double *out = (l == 0 && sw == post - 1) ? z0 : L.t.p;
            launch_smooth(L.A.A, L.M, f, L.uA.p, out, s);
            if (sw + 1 < post)
                CK(cudaMemcpyAsync(L.uA.p, out, sizeof(double) * 3 * nl, cudaMemcpyDeviceToDevice, s));
        }
        if (l == 0 && post == 0)
            CK(cudaMemcpyAsync(z0, L.uA.p, sizeof(double) * 3 * nl, cudaMemcpyDeviceToDevice, s));
    }
}

// PCG (cg.hpp:39-112) on the row-partitioned fine level; host reads ||r||
// once per iteration (identical decisions on every rank: all-reduced).
samg_solve_report DHierarchy::cg(const double *d_f, double *d_u, const samg_cg_params &cp) {
    cudaStream_t s = stream();
    const auto t0 = std::chrono::steady_clock::now();
    samg_solve_report rep{};
    rep.variant = SAMG_PIPELINE_NS_BLOCK;
    rep.setup_seconds = H->setup_seconds;
    const int64_t n = 3 * nloc0;
    const LocalMat &A0 = dl[0].A;
    CK(cudaMemcpyAsync(r.p, d_f, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    launch_fill(n, 0.0, u.p, s);
    CK(cudaMemsetAsync(sc.p, 0, sizeof(CgScalars), s));
    auto read = [&] {
        CK(cudaMemcpyAsync(sc_host, sc.p, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    };
    launch_dot(n, r.p, r.p, partials.p, sc.p, CG_STORE, s);
    allreduce_finish(CG_RR);
    read();
    const double norm_f = std::sqrt(sc_host->rr);
    auto finish = [&](double res) {
        rep.relative_residual = res;
        rep.preconditioner_bytes = H->memory_footprint();
        rep.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (d_u != u.p)
            CK(cudaMemcpyAsync(d_u, u.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        CK(cudaStreamSynchronize(s));
    };
    if (norm_f == 0.0) {
        rep.converged = 1;
        finish(0.0);
        return rep;
    }
    vcycle(r.p, z.p);
    launch_dot(n, r.p, z.p, partials.p, sc.p, CG_STORE, s);
    allreduce_finish(CG_RHO);
    CK(cudaMemcpyAsync(pext.p, z.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    double res_norm = norm_f;
    int iter = 0;
    while (res_norm / norm_f > cp.tol && iter < cp.max_iterations) {
        A0.plan.exchange(pext.p, comm, s);
        launch_spmv_dot(A0.A, pext.p, q.p, partials.p, sc.p, s, CG_STORE);
        allreduce_finish(CG_PQ);
        launch_cg_update(n, sc.p, pext.p, q.p, u.p, r.p, partials.p, CG_STORE, 0, s);
        allreduce_finish(CG_RR);
        read();
        if (sc_host->breakdown)
            fail(SAMG_BREAKDOWN_NON_SPD, "cg: p'Ap <= 0, matrix or preconditioner not SPD");
        ++iter;
        res_norm = std::sqrt(sc_host->rr);
        if (res_norm / norm_f <= cp.tol) break;
        vcycle(r.p, z.p);
        launch_dot(n, r.p, z.p, partials.p, sc.p, CG_STORE, s);
        allreduce_finish(CG_RZ);
        launch_p_update(n, sc.p, z.p, pext.p, s);
    }
    rep.iterations = iter;
    rep.converged = res_norm / norm_f <= cp.tol;
    // true residual (cg.hpp:105-108)
    CK(cudaMemcpyAsync(uext.p, u.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    A0.plan.exchange(uext.p, comm, s);
    launch_residual(A0.A, d_f, uext.p, q.p, s);
    launch_dot(n, q.p, q.p, partials.p, sc.p, CG_STORE, s);
    allreduce_finish(CG_RR);
    read();
    finish(std::sqrt(sc_host->rr) / norm_f);
    return rep;
}

// Build the distributed hierarchy from a full (redundant) single-GPU one.
DHierarchy *dsetup(std::unique_ptr<Hierarchy> H, ncclComm_t comm, int nranks, int rank,
                   const std::vector<int64_t> &row_starts, int64_t min_rows) {
    auto D = std::make_unique<DHierarchy>();
    D->rank = rank;
    D->nranks = nranks;
    D->comm = comm;
    D->device = H->device;
    cudaStream_t s = H->stream;
    const size_t L = H->levels.size();
    // number of partitioned levels: all levels with a transfer operator that
    // are large enough (the coarsest level is always replicated)
    if (L < 2) fail(SAMG_UNSUPPORTED, "multi-GPU solve needs at least two levels");
    size_t Ld = 0;
    while (Ld + 1 < L && H->levels[Ld].A.nrows >= min_rows * nranks) ++Ld;
    Ld = std::max<size_t>(Ld, 1);  // the fine level is always partitioned
    D->Ld = Ld;
    std::vector<int64_t> fst = row_starts;
    for (size_t l = 0; l < Ld; ++l) {
        Level &lv = H->levels[l];
        DLevel dlv;
        dlv.fstarts = fst;
        // coarse partition through the seeds of the aggregation
        const int h = l == 0 ? 1 : 2;  // block rows per node (pbs 3 / 6)
        const int64_t kb = lv.naggs ? lv.P.ncols / lv.naggs : 2;
        std::vector<int> seedno = download_int(lv.seedno, lv.nnodes + 1, s);
        std::vector<int64_t> cst(nranks + 1);
        for (int q = 0; q <= nranks; ++q) cst[q] = kb * seedno[fst[q] / h];
        dlv.cstarts = cst;
        dlv.next_replicated = l + 1 >= Ld;
        std::vector<int> ap = download_int(lv.A.ptr, lv.A.nrows + 1, s);
        std::vector<int> ac = download_int(lv.A.col, lv.A.nnzb, s);
        build_local(ap, ac, lv.A.val.p, fst, fst, rank, false, lv.A.ncols, dlv.A, s);
        std::vector<int> rp = download_int(lv.R.ptr, lv.R.nrows + 1, s);
        std::vector<int> rc = download_int(lv.R.col, lv.R.nnzb, s);
        build_local(rp, rc, lv.R.val.p, cst, fst, rank, false, lv.R.ncols, dlv.R, s);
        std::vector<int> pp = download_int(lv.P.ptr, lv.P.nrows + 1, s);
        std::vector<int> pc = download_int(lv.P.col, lv.P.nnzb, s);
        build_local(pp, pc, lv.P.val.p, fst, cst, rank, dlv.next_replicated, lv.P.ncols, dlv.P, s);
        // smoother rows
        const int per = lv.M.kind == SM_POINT ? 3 : 9;
        const int64_t f0 = fst[rank], nl = fst[rank + 1] - f0;
        dlv.M.kind = lv.M.kind;
        dlv.M.data.alloc(per * nl + 1, s);
        if (nl)
            CK(cudaMemcpyAsync(dlv.M.data.p, lv.M.data.p + per * f0, sizeof(double) * per * nl,
                               cudaMemcpyDeviceToDevice, s));
        dlv.f.alloc(3 * nl + 3, s);
        dlv.t.alloc(3 * nl + 3, s);
        dlv.uA.alloc(3 * (dlv.A.plan.nloc + dlv.A.plan.nghost) + 3, s);
        dlv.rR.alloc(3 * (dlv.R.plan.nloc + dlv.R.plan.nghost) + 3, s);
        if (!dlv.next_replicated) dlv.uP.alloc(3 * (dlv.P.plan.nloc + dlv.P.plan.nghost) + 3, s);
        D->dl.push_back(std::move(dlv));
        fst = cst;
    }
    D->ld_starts = fst;  // partition of level Ld (from the last partitioned level)
    const int64_t nLd = H->levels[Ld].A.nrows;
    D->fLd.alloc(3 * nLd + 3, s);
    D->uLd.alloc(3 * nLd + 3, s);
    D->nloc0 = row_starts[rank + 1] - row_starts[rank];
    const int64_t n = 3 * D->nloc0;
    const LocalMat &A0 = D->dl[0].A;
    D->r.alloc(n + 3, s);
    D->z.alloc(n + 3, s);
    D->q.alloc(n + 3, s);
    D->u.alloc(n + 3, s);
    D->pext.alloc(3 * (A0.plan.nloc + A0.plan.nghost) + 3, s);
    D->uext.alloc(3 * (A0.plan.nloc + A0.plan.nghost) + 3, s);
    D->partials.alloc(4096, s);
    D->sc.alloc(1, s);
    CK(cudaMallocHost(&D->sc_host, sizeof(CgScalars)));
    CK(cudaStreamSynchronize(s));
    D->H = std::move(H);
    return D.release();
}

} // namespace samgb

// ---- entry points used by capi.cu ------------------------------------------
namespace samgb {

DHierarchy *dsetup_all(const unsigned char *id, int nranks, int rank, Bsr3 &&A0,
                       const double *B, int64_t b_rows, int64_t b_cols,
                       const int64_t *row_starts, int64_t min_rows, const samg_amg_params &prm,
                       cudaStream_t s, double t0) {
    std::unique_ptr<Hierarchy> H(setup_hierarchy(std::move(A0), B, b_rows, b_cols, prm, s, t0));
    const int64_t nb = H->levels.front().A.nrows;
    std::vector<int64_t> st(nranks + 1);
    if (row_starts) {
        st.assign(row_starts, row_starts + nranks + 1);
        if (st[0] != 0 || st[nranks] != nb)
            fail(SAMG_INVALID_ARGUMENT, "dsetup: row_starts must span [0, nbrows]");
        for (int q = 0; q < nranks; ++q)
            if (st[q + 1] < st[q]) fail(SAMG_INVALID_ARGUMENT, "dsetup: row_starts must be nondecreasing");
    } else {
        for (int q = 0; q <= nranks; ++q) st[q] = nb * q / nranks;
    }
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    ncclComm_t comm;
    NK(nccl().CommInitRank(&comm, nranks, uid, rank));
    try {
        return dsetup(std::move(H), comm, nranks, rank, st, min_rows);
    } catch (...) {
        nccl().CommDestroy(comm);
        throw;
    }
}

void ddelete(DHierarchy *d) { delete d; }

samg_solve_report dcg(DHierarchy *d, const double *f, double *u, const samg_cg_params &cp,
                      bool host) {
    CK(cudaSetDevice(d->device));
    if (!host) return d->cg(f, u, cp);
    const auto t0 = std::chrono::steady_clock::now();
    cudaStream_t s = d->stream();
    const int64_t n = 3 * d->nloc0;
    DevBuf<double> df(n + 1, s), du(n + 1, s);
    CK(cudaMemcpyAsync(df.p, f, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    samg_solve_report rep = d->cg(df.p, du.p, cp);
    CK(cudaMemcpyAsync(u, du.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    rep.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rep;
}

void dinfo(const DHierarchy *d, int64_t *row0, int64_t *row1, int *nlevels, int *dist_levels,
           double *setup_s) {
    *row0 = d->dl[0].fstarts[d->rank];
    *row1 = d->dl[0].fstarts[d->rank + 1];
    *nlevels = static_cast<int>(d->H->levels.size());
    *dist_levels = static_cast<int>(d->Ld);
    *setup_s = d->H->setup_seconds;
}

void nccl_unique_id(unsigned char *out) {
    ncclUniqueId uid;
    NK(nccl().GetUniqueId(&uid));
    std::memcpy(out, &uid, sizeof uid);
}

} // namespace samgb
