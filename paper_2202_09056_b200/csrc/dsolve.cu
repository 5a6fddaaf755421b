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
//   * levels l >= Ld (fewer than min_rows * nranks block rows, or a rank
//     would own none) are replicated: f_Ld is gathered on every rank (grouped
//     ncclBroadcast) and the coarse V-cycle runs redundantly, so the
//     prolongation into level Ld-1 needs no halo.
// Every local SpMV reads a halo-extended vector: owned entries first, then
// the ghosts sorted by global id (grouped by owner).  Because all ranks hold
// all matrices, each rank derives both sides of every halo plan locally (no
// plan exchange).  A halo exchange is pack kernel + grouped ncclSend/ncclRecv
// on the solve stream.  CG dot products are local fused reductions (the same
// kernels as on one GPU, in STORE mode) + a one-double ncclAllReduce.
//
// The same code drives an *emulated* group (comm == nullptr): all ranks'
// slices live in one process on one GPU and every communication step is
// carried out, rank by rank in lock step, as device copies with exactly the
// offsets and counts the NCCL calls use.  No kernel waits on another rank;
// this is how the partition and halo plans are verified on a single GPU.
#include "nccl_shim.cuh"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <memory>
#include <vector>

#include <cub/cub.cuh>

#include "hierarchy.cuh"

namespace samgb {

inline void nccl_check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess)
        fail(SAMG_NCCL_ERROR, std::string(what) + " failed: " + nccl().GetErrorString(r));
}
#define NK(x) ::samgb::nccl_check((x), #x)

namespace {

constexpr int kMaxEmulated = 16;

__global__ void k_pack3(int64_t n, const int *idx, const double *x, double *buf) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < 3 * n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k = e / 3;
        buf[e] = x[3 * static_cast<int64_t>(idx[k]) + (e - 3 * k)];
    }
}

struct ScSet {
    CgScalars *p[kMaxEmulated];
    int n;
};

// emulated all-reduce of CgScalars::tmp (sum in rank order)
__global__ void k_sum_tmp(ScSet s) {
    double t = 0;
    for (int i = 0; i < s.n; ++i) t += s.p[i]->tmp;
    for (int i = 0; i < s.n; ++i) s.p[i]->tmp = t;
}



void d2d(double *dst, const double *src, int64_t n, cudaStream_t s) {
    if (n > 0) CK(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
}

} // namespace

// Halo plan of one local matrix: ghosts of its column space.
struct HaloPlan {
    int64_t nloc = 0, nghost = 0;
    std::vector<int> send_peers, recv_peers;
    std::vector<int64_t> send_counts, send_offsets, recv_counts, recv_offsets;
    DevBuf<int> send_idx;
    DevBuf<double> sendbuf;

    void pack(const double *xext, cudaStream_t s) const {
        const int64_t ns = send_idx.n;
        if (!ns) return;
        int64_t g = (3 * ns + 255) / 256;
        if (g > 4096) g = 4096;
        k_pack3<<<static_cast<int>(g), 256, 0, s>>>(ns, send_idx.p, xext, sendbuf.p);
        CK_LAUNCH();
    }

    void post(double *xext, ncclComm_t comm, cudaStream_t s) const {
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
    // [ia, ib): the longest run of rows that read no ghost column; these
    // are multiplied while the halo is in flight (slab partitions: all rows
    // but the first / last node layers)
    int64_t ia = 0, ib = 0;
};

// flag[i] = 1 if row i reads a ghost column (>= nloc)
__global__ void k_ghost_rows(int64_t nrows, const int *ptr, const int *col, int64_t nloc,
                             unsigned char *flag) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nrows;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        unsigned char g = 0;
        for (int e = ptr[i]; e < ptr[i + 1]; ++e) g |= col[e] >= nloc;
        flag[i] = g;
    }
}

// ---- slicing on the device -------------------------------------------------
__global__ void k_rebase(int64_t n, const int *in, int o, int *out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = in[i] + o;
}
void for_each_rebase(int64_t n, const int *in, int o, int *out, cudaStream_t s) {
    if (n <= 0) return;
    k_rebase<<<static_cast<int>(std::min<int64_t>(4096, (n + 255) / 256)), 256, 0, s>>>(n, in, o, out);
    CK_LAUNCH();
}
__global__ void k_gather_ptr(int n, const int64_t *idx, const int *ptr, int *out) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < n) out[q] = ptr[idx[q]];
}
// flag[c - lo] = 1 for every column c of cols[0, n) with (inside ? lo <= c < hi : c outside [lo, hi))
__global__ void k_mark_cols(int64_t n, const int *cols, int64_t lo, int64_t hi, bool inside, int *flag) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t c = cols[j];
        const bool in = c >= lo && c < hi;
        if (in == inside) flag[inside ? c - lo : c] = 1;
    }
}
// out[scan[k]] = k for flagged k (the flagged positions in ascending order)
__global__ void k_compact(int64_t n, const int *flag, const int *scan, int *out) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (flag[k]) out[scan[k]] = static_cast<int>(k);
}
__global__ void k_rebase_ptr(int64_t n, const int *ptr, int base, int *out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = ptr[i] - base;
}
// owned column c -> c - c0; ghost -> nloc + (rank of c among the ghosts)
__global__ void k_renumber(int64_t n, const int *cols, int64_t c0, int64_t c1, int64_t nloc,
                           const int *gscan, bool global_cols, int *out) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t c = cols[j];
        out[j] = static_cast<int>(global_cols ? c : (c >= c0 && c < c1 ? c - c0 : nloc + gscan[c]));
    }
}

int grid_of(int64_t n) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(4096, (n + 255) / 256))); }

// exclusive scan of flag[0, n) into scan[0, n] (scan[n] = total), on s
int64_t scan_flags(const int *flag, int *scan, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flag, scan, n + 1, s));
    DevBuf<char> ws(bytes + 1, s);
    CK(cub::DeviceScan::ExclusiveSum(ws.p, bytes, flag, scan, n + 1, s));
    int total = 0;
    CK(cudaMemcpyAsync(&total, scan + n, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return total;
}

// Rank r's slice of the (device, global) matrix G whose rows are partitioned
// by row_starts and whose column space is partitioned by col_starts: rows
// [r0, r1) with columns renumbered into the halo-extended vector (owned
// first, then the ghosts in ascending global id, i.e. grouped by owner), the
// receive plan (ghost counts per owner) and the send plan (the owned columns
// every other rank's slice reads, ascending).  All on the device: flag
// arrays + scans, O(nnz + ncols) per rank, a few scalars to the host.
void build_local(const Bsr3 &G, const std::vector<int64_t> &row_starts,
                 const std::vector<int64_t> &col_starts, int rank, bool global_cols,
                 LocalMat &out, cudaStream_t s) {
    const int nranks = static_cast<int>(row_starts.size()) - 1;
    // the row bounds of every rank's slice
    std::vector<int> bnd(nranks + 1);
    {
        DevBuf<int64_t> ridx(nranks + 1, s);
        DevBuf<int> rb(nranks + 1, s);
        CK(cudaMemcpyAsync(ridx.p, row_starts.data(), sizeof(int64_t) * (nranks + 1), cudaMemcpyHostToDevice, s));
        k_gather_ptr<<<1, 32, 0, s>>>(nranks + 1, ridx.p, G.ptr.p, rb.p);
        CK(cudaMemcpyAsync(bnd.data(), rb.p, sizeof(int) * (nranks + 1), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    const int64_t r0 = row_starts[rank], r1 = row_starts[rank + 1];
    const int64_t c0 = col_starts[rank], c1 = col_starts[rank + 1];
    const int64_t nl = r1 - r0, base = bnd[rank], nnz = bnd[rank + 1] - base;
    const int64_t ncg = G.ncols;
    HaloPlan &pl = out.plan;
    DevBuf<int> gscan;
    if (!global_cols) {
        pl.nloc = c1 - c0;
        // ghosts: flags over the global column space, scanned
        DevBuf<int> gflag(ncg + 1, s);
        gscan.alloc(ncg + 1, s);
        CK(cudaMemsetAsync(gflag.p, 0, sizeof(int) * (ncg + 1), s));
        if (nnz) k_mark_cols<<<grid_of(nnz), 256, 0, s>>>(nnz, G.col.p + base, c0, c1, false, gflag.p);
        pl.nghost = scan_flags(gflag.p, gscan.p, ncg, s);
        // receive plan: ghosts per owner = scan differences at the owners' bounds
        std::vector<int> at(nranks + 1);
        {
            DevBuf<int64_t> cidx(nranks + 1, s);
            DevBuf<int> cv(nranks + 1, s);
            CK(cudaMemcpyAsync(cidx.p, col_starts.data(), sizeof(int64_t) * (nranks + 1), cudaMemcpyHostToDevice, s));
            k_gather_ptr<<<1, 32, 0, s>>>(nranks + 1, cidx.p, gscan.p, cv.p);
            CK(cudaMemcpyAsync(at.data(), cv.p, sizeof(int) * (nranks + 1), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
        for (int q = 0; q < nranks; ++q)
            if (at[q + 1] > at[q]) {
                pl.recv_peers.push_back(q);
                pl.recv_counts.push_back(at[q + 1] - at[q]);
                pl.recv_offsets.push_back(at[q]);
            }
        // send plan: for every other rank, the owned columns its rows read
        const int64_t nown = c1 - c0;
        DevBuf<int> sflag(nown + 1, s), sscan(nown + 1, s);
        std::vector<DevBuf<int>> parts;
        int64_t total = 0;
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            const int64_t qb = bnd[q], qn = bnd[q + 1] - bnd[q];
            if (!qn || !nown) continue;
            CK(cudaMemsetAsync(sflag.p, 0, sizeof(int) * (nown + 1), s));
            k_mark_cols<<<grid_of(qn), 256, 0, s>>>(qn, G.col.p + qb, c0, c1, true, sflag.p);
            const int64_t cnt = scan_flags(sflag.p, sscan.p, nown, s);
            if (!cnt) continue;
            parts.emplace_back(cnt, s);
            k_compact<<<grid_of(nown), 256, 0, s>>>(nown, sflag.p, sscan.p, parts.back().p);
            pl.send_peers.push_back(q);
            pl.send_counts.push_back(cnt);
            pl.send_offsets.push_back(total);
            total += cnt;
        }
        pl.send_idx.alloc(total, s);
        for (size_t k = 0; k < parts.size(); ++k)
            CK(cudaMemcpyAsync(pl.send_idx.p + pl.send_offsets[k], parts[k].p, sizeof(int) * pl.send_counts[k],
                               cudaMemcpyDeviceToDevice, s));
        pl.sendbuf.alloc(3 * total + 3, s);
    } else {
        pl.nloc = ncg;
    }
    Bsr3 &A = out.A;
    A.alloc(nl, global_cols ? ncg : pl.nloc + pl.nghost, nnz, s);
    k_rebase_ptr<<<grid_of(nl + 1), 256, 0, s>>>(nl + 1, G.ptr.p + r0, static_cast<int>(base), A.ptr.p);
    if (nnz) {
        k_renumber<<<grid_of(nnz), 256, 0, s>>>(nnz, G.col.p + base, c0, c1, pl.nloc, gscan.p, global_cols,
                                               A.col.p);
        CK(cudaMemcpyAsync(A.val.p, G.val.p + 9 * base, sizeof(double) * 9 * nnz, cudaMemcpyDeviceToDevice, s));
    }
    CK_LAUNCH();
    out.ia = out.ib = 0;
    if (!global_cols && nl > 0) {
        DevBuf<unsigned char> gf(nl, s);
        k_ghost_rows<<<grid_of(nl), 256, 0, s>>>(nl, A.ptr.p, A.col.p, pl.nloc, gf.p);
        CK_LAUNCH();
        std::vector<unsigned char> hf(nl);
        CK(cudaMemcpyAsync(hf.data(), gf.p, nl, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        int64_t best = 0, run = 0;
        for (int64_t i = 0; i < nl; ++i) {
            run = hf[i] ? 0 : run + 1;
            if (run > best) { best = run; out.ib = i + 1; out.ia = i + 1 - run; }
        }
    }
    CK(cudaStreamSynchronize(s));  // the temporaries above are freed on s
}

// Rows [r0, r1) of M as a non-owning matrix (ptr offset; col / val shared,
// so the ptr values stay absolute).  Vectors indexed by row (f, u, out, M)
// are offset by the caller.
struct RowView {
    Bsr3 m;
    RowView(const Bsr3 &src, int64_t r0, int64_t r1) {
        m.nrows = r1 - r0;
        m.ncols = src.ncols;
        m.nnzb = src.nnzb;  // bounds of the shared arrays (the TMA path's end checks)
        m.ptr.p = src.ptr.p + r0;
        m.col.p = src.col.p;
        m.val.p = src.val.p;
        m.val32.p = src.val32.p;
    }
    RowView(const RowView &) = delete;
    ~RowView() { m.ptr.p = nullptr; m.col.p = nullptr; m.val.p = nullptr; m.val32.p = nullptr; }
};
struct SmootherView {
    Smoother m;
    SmootherView(const Smoother &src, int64_t r0) {
        m.kind = src.kind;
        m.data.p = src.data.p ? src.data.p + (src.kind == SM_POINT ? 3 : 9) * r0 : nullptr;
    }
    SmootherView(const SmootherView &) = delete;
    ~SmootherView() { m.data.p = nullptr; }
};

struct DLevel {
    LocalMat A, R, P;
    Smoother M;
    DevBuf<double> f, uA, rR, t, uP;  // f, t: 3*nloc; uA/rR/uP: halo-extended
};

// The slices one rank owns.
struct DRank {
    int rank = 0;
    int64_t row0 = 0, nloc0 = 0;
    std::vector<DLevel> dl;
    DevBuf<double> fLd, uLd;  // replicated level-Ld vectors
    DevBuf<double> r, z, pext, q, u, uext;
    DevBuf<CgScalars> sc;
    DevBuf<double> partials;
};

struct DHierarchy {
    int nranks = 1, device = 0;
    ncclComm_t comm = nullptr;   // nullptr: every rank emulated in this process
    std::unique_ptr<Hierarchy> H;
    size_t Ld = 0;
    int sliced_levels = 0;       // levels whose Galerkin product was row-sliced (DistSlicer)
    std::vector<std::vector<int64_t>> starts;  // partition of levels 0..Ld
    std::vector<DRank> ranks;    // the ranks this process drives
    CgScalars *sc_host = nullptr;
    cudaStream_t cs = nullptr;   // halo transfers overlapped with interior rows
    cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;

    ~DHierarchy() {
        if (H && H->stream) cudaStreamSynchronize(H->stream);
        if (cs) cudaStreamSynchronize(cs);
        ranks.clear();
        if (ev_pack) cudaEventDestroy(ev_pack);
        if (ev_halo) cudaEventDestroy(ev_halo);
        if (cs) cudaStreamDestroy(cs);
        pinned_small_free(sc_host);
        if (comm) nccl().CommDestroy(comm);
    }

    cudaStream_t stream() const { return H->stream; }
    bool emulated() const { return comm == nullptr; }

    // Halo exchange of the level-l operator selected by `which` (0 A, 1 R,
    // 2 P) into the extended vector `vec` of every driven rank.
    LocalMat &local(DRank &R, size_t l, int which) {
        DLevel &L = R.dl[l];
        return which == 0 ? L.A : which == 1 ? L.R : L.P;
    }

    // Halo transfer of already packed send buffers into the ghost segments
    // of `vec`, on stream cs (NCCL, or device copies when emulated).
    template <class Vec>
    void transfer(size_t l, int which, Vec vec, cudaStream_t cs) {
        if (!emulated()) {
            local(ranks[0], l, which).plan.post(vec(ranks[0]), comm, cs);
            return;
        }
        for (DRank &R : ranks) {
            const HaloPlan &pl = local(R, l, which).plan;
            double *x = vec(R);
            for (size_t k = 0; k < pl.recv_peers.size(); ++k) {
                const HaloPlan &ql = local(ranks[pl.recv_peers[k]], l, which).plan;
                const auto it = std::find(ql.send_peers.begin(), ql.send_peers.end(), R.rank);
                if (it == ql.send_peers.end()) fail(SAMG_ERROR, "dsolve: unmatched halo receive");
                const size_t i = it - ql.send_peers.begin();
                if (ql.send_counts[i] != pl.recv_counts[k])
                    fail(SAMG_ERROR, "dsolve: halo send/receive counts differ");
                d2d(x + 3 * (pl.nloc + pl.recv_offsets[k]), ql.sendbuf.p + 3 * ql.send_offsets[i],
                    3 * pl.recv_counts[k], cs);
            }
        }
    }

    // Halo exchange of the level-l operator selected by `which` (0 A, 1 R,
    // 2 P) into the extended vector `vec` of every driven rank.
    template <class Vec>
    void exchange(size_t l, int which, Vec vec) {
        cudaStream_t s = stream();
        for (DRank &R : ranks) local(R, l, which).plan.pack(vec(R), s);
        transfer(l, which, vec, s);
    }

    // Exchange overlapped with the rows that read no ghost: pack on the solve
    // stream, the transfer on the comm stream, op(R, r0, r1) on rows [ia, ib)
    // meanwhile, the remaining rows once the halo has arrived.
    template <class Vec, class Op>
    void exchange_overlap(size_t l, int which, Vec vec, Op op) {
        cudaStream_t s = stream();
        for (DRank &R : ranks) local(R, l, which).plan.pack(vec(R), s);
        CK(cudaEventRecord(ev_pack, s));
        CK(cudaStreamWaitEvent(cs, ev_pack, 0));
        transfer(l, which, vec, cs);
        CK(cudaEventRecord(ev_halo, cs));
        for (DRank &R : ranks) {
            const LocalMat &M = local(R, l, which);
            if (M.ib > M.ia) op(R, M.ia, M.ib);
        }
        CK(cudaStreamWaitEvent(s, ev_halo, 0));
        for (DRank &R : ranks) {
            const LocalMat &M = local(R, l, which);
            const int64_t n = M.A.nrows;
            if (M.ib > M.ia) {
                if (M.ia > 0) op(R, 0, M.ia);
                if (n > M.ib) op(R, M.ib, n);
            } else if (n > 0) {
                op(R, 0, n);
            }
        }
    }

    // the sum over ranks of sc->tmp, then the CG update `what`
    void allreduce_finish(int what) {
        cudaStream_t s = stream();
        if (!emulated()) {
            double *t = reinterpret_cast<double *>(reinterpret_cast<char *>(ranks[0].sc.p) +
                                                   offsetof(CgScalars, tmp));
            NK(nccl().AllReduce(t, t, 1, ncclDouble, ncclSum, comm, s));
        } else if (ranks.size() > 1) {
            ScSet set{};
            set.n = static_cast<int>(ranks.size());
            for (int i = 0; i < set.n; ++i) set.p[i] = ranks[i].sc.p;
            k_sum_tmp<<<1, 1, 0, s>>>(set);
            CK_LAUNCH();
        }
        for (DRank &R : ranks) launch_cg_finish(R.sc.p, what, s);
    }

    // every rank's piece of f_Ld to every rank
    void gather_coarse() {
        cudaStream_t s = stream();
        const std::vector<int64_t> &st = starts[Ld];
        if (!emulated()) {
            double *f = ranks[0].fLd.p;
            NK(nccl().GroupStart());
            for (int q = 0; q < nranks; ++q) {
                const int64_t o = 3 * st[q], c = 3 * (st[q + 1] - st[q]);
                if (c) NK(nccl().Broadcast(f + o, f + o, c, ncclDouble, q, comm, s));
            }
            NK(nccl().GroupEnd());
            return;
        }
        for (DRank &R : ranks)
            for (const DRank &Q : ranks)
                if (Q.rank != R.rank)
                    d2d(R.fLd.p + 3 * st[Q.rank], Q.fLd.p + 3 * st[Q.rank],
                        3 * (st[Q.rank + 1] - st[Q.rank]), s);
    }

    void vcycle();
    samg_solve_report cg(const double *d_f, double *d_u, const samg_cg_params &cp);
};

// Distributed V-cycle (hierarchy.hpp:408-441) from a zero guess: z = M^-1 r
// on every driven rank.
void DHierarchy::vcycle() {
    cudaStream_t s = stream();
    const int pre = H->prm.pre_sweeps, post = H->prm.post_sweeps;
    auto fin = [&](DRank &R, size_t l) -> const double * { return l == 0 ? R.r.p : R.dl[l].f.p; };
    for (size_t l = 0; l < Ld; ++l) {
        for (DRank &R : ranks) {
            DLevel &L = R.dl[l];
            if (pre > 0) launch_smooth_zero(L.A.A.nrows, L.M, fin(R, l), L.uA.p, s);
            else launch_fill(3 * L.A.A.nrows, 0.0, L.uA.p, s);
        }
        for (int sw = 1; sw < pre; ++sw) {
            exchange_overlap(l, 0, [&](DRank &R) { return R.dl[l].uA.p; },
                             [&](DRank &R, int64_t a, int64_t b) {
                DLevel &L = R.dl[l];
                RowView v(L.A.A, a, b);
                SmootherView m(L.M, a);
                launch_smooth_split(v.m, m.m, fin(R, l) + 3 * a, L.uA.p, L.uA.p + 3 * a, L.t.p + 3 * a, s);
            });
            for (DRank &R : ranks) d2d(R.dl[l].uA.p, R.dl[l].t.p, 3 * R.dl[l].A.A.nrows, s);
        }
        exchange_overlap(l, 0, [&](DRank &R) { return R.dl[l].uA.p; },
                         [&](DRank &R, int64_t a, int64_t b) {
            DLevel &L = R.dl[l];
            RowView v(L.A.A, a, b);
            launch_residual(v.m, fin(R, l) + 3 * a, L.uA.p, L.rR.p + 3 * a, s);
        });
        exchange_overlap(l, 1, [&](DRank &R) { return R.dl[l].rR.p; },
                         [&](DRank &R, int64_t a, int64_t b) {
            DLevel &L = R.dl[l];
            double *fc = (l + 1 < Ld) ? R.dl[l + 1].f.p : R.fLd.p + 3 * starts[Ld][R.rank];
            RowView v(L.R.A, a, b);
            launch_spmv(v.m, 1.0, L.rR.p, 0.0, fc + 3 * a, s);
        });
    }
    gather_coarse();
    for (DRank &R : ranks) H->vcycle_from(Ld, R.fLd.p, R.uLd.p, true, false);
    for (size_t l = Ld; l-- > 0;) {
        const bool next_replicated = l + 1 == Ld;
        if (!next_replicated) {
            // level l+1's result (in its t or uA) -> local part of uP, then halo
            for (DRank &R : ranks) {
                const DLevel &N = R.dl[l + 1];
                d2d(R.dl[l].uP.p, post > 0 ? N.t.p : N.uA.p, 3 * N.A.A.nrows, s);
            }
            exchange_overlap(l, 2, [&](DRank &R) { return R.dl[l].uP.p; },
                             [&](DRank &R, int64_t a, int64_t b) {
                DLevel &L = R.dl[l];
                RowView v(L.P.A, a, b);
                launch_spmv(v.m, 1.0, L.uP.p, 1.0, L.uA.p + 3 * a, s);
            });
        } else {
            for (DRank &R : ranks) {
                DLevel &L = R.dl[l];
                launch_spmv(L.P.A, 1.0, R.uLd.p, 1.0, L.uA.p, s);
            }
        }
        for (int sw = 0; sw < post; ++sw) {
            auto out_of = [&](DRank &R) { return (l == 0 && sw == post - 1) ? R.z.p : R.dl[l].t.p; };
            exchange_overlap(l, 0, [&](DRank &R) { return R.dl[l].uA.p; },
                             [&](DRank &R, int64_t a, int64_t b) {
                DLevel &L = R.dl[l];
                RowView v(L.A.A, a, b);
                SmootherView m(L.M, a);
                launch_smooth_split(v.m, m.m, fin(R, l) + 3 * a, L.uA.p, L.uA.p + 3 * a,
                                    out_of(R) + 3 * a, s);
            });
            if (sw + 1 < post)
                for (DRank &R : ranks) d2d(R.dl[l].uA.p, out_of(R), 3 * R.dl[l].A.A.nrows, s);
        }
        if (l == 0 && post == 0)
            for (DRank &R : ranks) d2d(R.z.p, R.dl[0].uA.p, 3 * R.nloc0, s);
    }
}

// PCG (cg.hpp:39-112) on the row-partitioned fine level; the host reads the
// (all-reduced, identical on every rank) scalars once per iteration.  d_f /
// d_u are the rank's slices, or the global vectors of an emulated group.
samg_solve_report DHierarchy::cg(const double *d_f, double *d_u, const samg_cg_params &cp) {
    cudaStream_t s = stream();
    const auto t0 = std::chrono::steady_clock::now();
    samg_solve_report rep{};
    rep.variant = H->pipeline;
    rep.setup_seconds = H->setup_seconds;
    const int64_t base0 = emulated() ? ranks[0].row0 : 0;
    auto off = [&](const DRank &R) { return 3 * (R.row0 - base0); };
    for (DRank &R : ranks) {
        d2d(R.r.p, d_f + off(R), 3 * R.nloc0, s);
        launch_fill(3 * R.nloc0, 0.0, R.u.p, s);
        CK(cudaMemsetAsync(R.sc.p, 0, sizeof(CgScalars), s));
    }
    auto read = [&] {
        CK(cudaMemcpyAsync(sc_host, ranks[0].sc.p, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    };
    auto dots = [&](auto x, auto y, int what) {
        for (DRank &R : ranks) launch_dot(3 * R.nloc0, x(R), y(R), R.partials.p, R.sc.p, CG_STORE, s);
        allreduce_finish(what);
    };
    dots([](DRank &R) { return R.r.p; }, [](DRank &R) { return R.r.p; }, CG_RR);
    read();
    const double norm_f = std::sqrt(sc_host->rr);
    auto finish = [&](double res) {
        rep.relative_residual = res;
        rep.preconditioner_bytes = H->memory_footprint();
        rep.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (DRank &R : ranks) d2d(d_u + off(R), R.u.p, 3 * R.nloc0, s);
        CK(cudaStreamSynchronize(s));
    };
    if (norm_f == 0.0) {
        rep.converged = 1;
        finish(0.0);
        return rep;
    }
    auto precondition = [&] {
        vcycle();
        dots([](DRank &R) { return R.r.p; }, [](DRank &R) { return R.z.p; }, CG_RZ);
    };
    vcycle();
    dots([](DRank &R) { return R.r.p; }, [](DRank &R) { return R.z.p; }, CG_RHO);
    for (DRank &R : ranks) d2d(R.pext.p, R.z.p, 3 * R.nloc0, s);
    double res_norm = norm_f;
    int iter = 0;
    while (res_norm / norm_f > cp.tol && iter < cp.max_iterations) {
        // q = A p overlapped with the halo: the first row range stores its
        // partial p.q, the others add to it
        std::vector<int> pieces(ranks.size(), 0);
        exchange_overlap(0, 0, [](DRank &R) { return R.pext.p; },
                         [&](DRank &R, int64_t a, int64_t b) {
            RowView v(R.dl[0].A.A, a, b);
            int &k = pieces[&R - ranks.data()];
            launch_spmv_dot_split(v.m, R.pext.p, R.pext.p + 3 * a, R.q.p + 3 * a, R.partials.p,
                                  R.sc.p, s, k++ == 0 ? CG_STORE : CG_ADD);
        });
        allreduce_finish(CG_PQ);
        for (DRank &R : ranks)
            launch_cg_update(3 * R.nloc0, R.sc.p, R.pext.p, R.q.p, R.u.p, R.r.p, R.partials.p,
                             CG_STORE, 0, s);
        allreduce_finish(CG_RR);
        read();
        if (sc_host->breakdown)
            fail(SAMG_BREAKDOWN_NON_SPD, "cg: p'Ap <= 0, matrix or preconditioner not SPD");
        ++iter;
        res_norm = std::sqrt(sc_host->rr);
        if (res_norm / norm_f <= cp.tol) break;
        precondition();
        for (DRank &R : ranks) launch_p_update(3 * R.nloc0, R.sc.p, R.z.p, R.pext.p, s);
    }
    rep.iterations = iter;
    rep.converged = res_norm / norm_f <= cp.tol;
    // true residual (cg.hpp:105-108)
    for (DRank &R : ranks) d2d(R.uext.p, R.u.p, 3 * R.nloc0, s);
    exchange(0, 0, [](DRank &R) { return R.uext.p; });
    for (DRank &R : ranks) launch_residual(R.dl[0].A.A, d_f + off(R), R.uext.p, R.q.p, s);
    dots([](DRank &R) { return R.q.p; }, [](DRank &R) { return R.q.p; }, CG_RR);
    read();
    finish(std::sqrt(sc_host->rr) / norm_f);
    return rep;
}

// Build the distributed hierarchy from a full (redundant) single-GPU one for
// the ranks `mine` (one rank with NCCL, all of them when emulated).
DHierarchy *dsetup(std::unique_ptr<Hierarchy> H, ncclComm_t comm, int nranks,
                   const std::vector<int> &mine, const std::vector<int64_t> &row_starts,
                   int64_t min_rows) {
    auto D = std::make_unique<DHierarchy>();
    D->nranks = nranks;
    D->device = H->device;
    cudaStream_t s = H->stream;
    const size_t L = H->levels.size();
    if (L < 2) fail(SAMG_UNSUPPORTED, "multi-GPU solve needs at least two levels");
    // partition chain: level l+1's rows follow the seeds of level l's aggregation
    std::vector<std::vector<int64_t>> st{row_starts};
    size_t Ld = 1;  // the fine level is always partitioned
    for (size_t l = 0; l + 1 < L; ++l) {
        const Level &lv = H->levels[l];
        // block rows per node: 1 on the fine level (pbs 3) and in the block
        // pipeline, 2 on ns coarse levels (pbs 6)
        const int64_t h = lv.nnodes ? lv.A.nrows / lv.nnodes : 1;
        const int64_t kb = lv.naggs ? lv.P.ncols / lv.naggs : 2;
        // seedno at the partition bounds only (nranks + 1 values)
        std::vector<int64_t> nidx(nranks + 1);
        for (int q = 0; q <= nranks; ++q) nidx[q] = st[l][q] / h;
        std::vector<int> sn(nranks + 1);
        {
            DevBuf<int64_t> di(nranks + 1, s);
            DevBuf<int> dv(nranks + 1, s);
            CK(cudaMemcpyAsync(di.p, nidx.data(), sizeof(int64_t) * (nranks + 1), cudaMemcpyHostToDevice, s));
            k_gather_ptr<<<1, 32, 0, s>>>(nranks + 1, di.p, lv.seedno.p, dv.p);
            CK(cudaMemcpyAsync(sn.data(), dv.p, sizeof(int) * (nranks + 1), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
        std::vector<int64_t> cst(nranks + 1);
        for (int q = 0; q <= nranks; ++q) cst[q] = kb * sn[q];
        st.push_back(cst);
        // level l+1 is partitioned too if it is not the coarsest, large
        // enough, and gives every rank at least one row
        bool part = l + 2 < L && H->levels[l + 1].A.nrows >= min_rows * nranks;
        for (int q = 0; q < nranks && part; ++q) part = cst[q + 1] > cst[q];
        if (!part) break;
        Ld = l + 2;
    }
    D->Ld = Ld;
    D->starts = st;
    D->ranks.resize(mine.size());
    for (size_t i = 0; i < mine.size(); ++i) {
        DRank &R = D->ranks[i];
        R.rank = mine[i];
        R.row0 = row_starts[R.rank];
        R.nloc0 = row_starts[R.rank + 1] - R.row0;
        R.dl.resize(Ld);
    }
    for (size_t l = 0; l < Ld; ++l) {
        Level &lv = H->levels[l];
        const std::vector<int64_t> &fst = st[l], &cst = st[l + 1];
        const bool next_replicated = l + 1 == Ld;
        const int per = lv.M.kind == SM_POINT ? 3 : 9;
        for (DRank &R : D->ranks) {
            DLevel &dlv = R.dl[l];
            build_local(lv.A, fst, fst, R.rank, false, dlv.A, s);
            build_local(lv.R, cst, fst, R.rank, false, dlv.R, s);
            build_local(lv.P, fst, cst, R.rank, next_replicated, dlv.P, s);
            const int64_t f0 = fst[R.rank], nl = fst[R.rank + 1] - f0;
            dlv.M.kind = lv.M.kind;
            dlv.M.data.alloc(per * nl + 1, s);
            if (nl)
                CK(cudaMemcpyAsync(dlv.M.data.p, lv.M.data.p + per * f0, sizeof(double) * per * nl,
                                   cudaMemcpyDeviceToDevice, s));
            dlv.f.alloc(3 * nl + 3, s);
            dlv.t.alloc(3 * nl + 3, s);
            dlv.uA.alloc(3 * (dlv.A.plan.nloc + dlv.A.plan.nghost) + 3, s);
            dlv.rR.alloc(3 * (dlv.R.plan.nloc + dlv.R.plan.nghost) + 3, s);
            if (!next_replicated) dlv.uP.alloc(3 * (dlv.P.plan.nloc + dlv.P.plan.nghost) + 3, s);
        }
    }
    const int64_t nLd = H->levels[Ld].A.nrows;
    for (DRank &R : D->ranks) {
        const int64_t n = 3 * R.nloc0;
        const LocalMat &A0 = R.dl[0].A;
        R.fLd.alloc(3 * nLd + 3, s);
        R.uLd.alloc(3 * nLd + 3, s);
        R.r.alloc(n + 3, s);
        R.z.alloc(n + 3, s);
        R.q.alloc(n + 3, s);
        R.u.alloc(n + 3, s);
        R.pext.alloc(3 * (A0.plan.nloc + A0.plan.nghost) + 3, s);
        R.uext.alloc(3 * (A0.plan.nloc + A0.plan.nghost) + 3, s);
        R.partials.alloc(4096, s);
        R.sc.alloc(1, s);
    }
    D->sc_host = static_cast<CgScalars *>(pinned_small_alloc(sizeof(CgScalars)));
    CK(cudaStreamCreateWithFlags(&D->cs, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&D->ev_pack, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&D->ev_halo, cudaEventDisableTiming));
    CK(cudaStreamSynchronize(s));
    D->H = std::move(H);
    D->comm = comm;
    return D.release();
}

} // namespace samgb

// ---- entry points used by capi.cu ------------------------------------------
namespace samgb {

// Row-sliced Galerkin product for the multi-GPU setup.  Every rank runs the
// (deterministic) setup on the whole matrix, except for the dominant step:
// rank q forms only the coarse rows it will own, [cst[q], cst[q+1]) -- the
// same partition chain dsetup derives from the aggregation seeds -- as
// (R[cst[q]:cst[q+1]] A) P, and the rows are then assembled on every rank
// (one all-reduce of the block counts, then grouped in-place ncclBroadcasts
// of each rank's ptr / col / val piece).  Every output row is computed by
// exactly the kernels of the single-GPU product, so A_c is bit-identical to
// it.  Levels below min_rows * nranks coarse rows are formed redundantly.
// Emulated group (comm == nullptr): the pieces of all ranks are formed one
// after the other and assembled by device copies (verification on one GPU).
struct DistSlicer : GalerkinSlicer {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    int64_t min_rows = 4096;
    std::vector<int64_t> st;  // fine row starts of the current level
    bool active = true;
    int sliced_levels = 0;

    bool galerkin(size_t, const Bsr3 &A, const int *seedno, int64_t nnodes, int64_t naggs,
                  const Bsr3 &R, const Bsr3 &P, Bsr3 &Ac, bool scalar_order, cudaStream_t s) override {
        if (!active || nnodes == 0 || naggs == 0) return active = false;
        const int64_t h = A.nrows / nnodes, kb = P.ncols / naggs;
        std::vector<int64_t> nidx(nranks + 1);
        for (int q = 0; q <= nranks; ++q) nidx[q] = st[q] / h;
        std::vector<int> sn(nranks + 1);
        {
            DevBuf<int64_t> di(nranks + 1, s);
            DevBuf<int> dv(nranks + 1, s);
            CK(cudaMemcpyAsync(di.p, nidx.data(), sizeof(int64_t) * (nranks + 1), cudaMemcpyHostToDevice, s));
            k_gather_ptr<<<1, 32, 0, s>>>(nranks + 1, di.p, seedno, dv.p);
            CK(cudaMemcpyAsync(sn.data(), dv.p, sizeof(int) * (nranks + 1), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
        std::vector<int64_t> cst(nranks + 1);
        for (int q = 0; q <= nranks; ++q) cst[q] = kb * sn[q];
        bool slice = R.nrows >= min_rows * nranks && cst[nranks] == R.nrows;
        for (int q = 0; q < nranks && slice; ++q) slice = cst[q + 1] > cst[q];
        if (!slice) return active = false;
        st = cst;  // the next level's fine partition
        ++sliced_levels;
        std::vector<int> mine;
        if (comm) mine.push_back(rank);
        else for (int q = 0; q < nranks; ++q) mine.push_back(q);
        // each driven rank's piece
        std::vector<Bsr3> piece(nranks);
        std::vector<int64_t> cnt(nranks, 0);
        for (int q : mine) {
            Bsr3 Rs;
            slice_rows(R, cst[q], cst[q + 1], Rs, s);
            galerkin_rows(Rs, A, P, R, piece[q], s, scalar_order);
            cnt[q] = piece[q].nnzb;
        }
        if (comm) {  // block counts of every rank (an all-gather as a sum)
            DevBuf<int64_t> dc(nranks, s);
            CK(cudaMemcpyAsync(dc.p, cnt.data(), sizeof(int64_t) * nranks, cudaMemcpyHostToDevice, s));
            NK(nccl().AllReduce(dc.p, dc.p, nranks, ncclInt64, ncclSum, comm, s));
            CK(cudaMemcpyAsync(cnt.data(), dc.p, sizeof(int64_t) * nranks, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
        std::vector<int64_t> off(nranks + 1, 0);
        for (int q = 0; q < nranks; ++q) off[q + 1] = off[q] + cnt[q];
        Ac.alloc(R.nrows, P.ncols, off[nranks], s);
        for (int q : mine) {  // own pieces into place, ptr rebased
            const int *pp = piece[q].ptr.p;
            int *ap = Ac.ptr.p + cst[q];
            const int o = static_cast<int>(off[q]);
            const int64_t nr = cst[q + 1] - cst[q] + (q == nranks - 1 ? 1 : 0);
            for_each_rebase(nr, pp, o, ap, s);
            if (cnt[q]) {
                CK(cudaMemcpyAsync(Ac.col.p + off[q], piece[q].col.p, sizeof(int) * cnt[q],
                                   cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(Ac.val.p + 9 * off[q], piece[q].val.p, sizeof(double) * 9 * cnt[q],
                                   cudaMemcpyDeviceToDevice, s));
            }
            piece[q] = Bsr3();
        }
        if (comm) {
            NK(nccl().GroupStart());
            for (int q = 0; q < nranks; ++q) {
                const int64_t nr = cst[q + 1] - cst[q] + (q == nranks - 1 ? 1 : 0);
                int *pq = Ac.ptr.p + cst[q];
                NK(nccl().Broadcast(pq, pq, nr, ncclInt32, q, comm, s));
                if (cnt[q]) {
                    int *cq = Ac.col.p + off[q];
                    double *vq = Ac.val.p + 9 * off[q];
                    NK(nccl().Broadcast(cq, cq, cnt[q], ncclInt32, q, comm, s));
                    NK(nccl().Broadcast(vq, vq, 9 * cnt[q], ncclDouble, q, comm, s));
                }
            }
            NK(nccl().GroupEnd());
        }
        return true;
    }
};

// id == nullptr: emulate all nranks in this process (no NCCL).
DHierarchy *dsetup_all(const unsigned char *id, int nranks, int rank, Bsr3 &&A0,
                       const double *B, int64_t b_rows, int64_t b_cols,
                       const int64_t *row_starts, int64_t min_rows, const samg_amg_params &prm,
                       cudaStream_t s, double t0, int pipeline) {
    if (!id && nranks > kMaxEmulated) fail(SAMG_INVALID_ARGUMENT, "dsetup: at most 16 emulated ranks");
    if (prm.smoother == SAMG_SMOOTHER_ILU0)
        fail(SAMG_UNSUPPORTED, "multi-GPU solve: the ILU(0) sweeps are sequential across row partitions");
    const int64_t nb = A0.nrows;
    std::vector<int64_t> st(nranks + 1);
    if (row_starts) {
        st.assign(row_starts, row_starts + nranks + 1);
        if (st[0] != 0 || st[nranks] != nb)
            fail(SAMG_INVALID_ARGUMENT, "dsetup: row_starts must span [0, nbrows]");
    } else {
        for (int q = 0; q <= nranks; ++q) st[q] = nb * q / nranks;
    }
    for (int q = 0; q < nranks; ++q)
        if (st[q + 1] <= st[q]) fail(SAMG_INVALID_ARGUMENT, "dsetup: every rank needs at least one block row");
    std::vector<int> mine;
    if (id) {
        mine.push_back(rank);
    } else {
        for (int q = 0; q < nranks; ++q) mine.push_back(q);
    }
    ncclComm_t comm = nullptr;
    if (id) {
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        NK(nccl().CommInitRank(&comm, nranks, uid, rank));
    }
    try {
        DistSlicer slicer;
        slicer.comm = comm;
        slicer.nranks = nranks;
        slicer.rank = rank;
        slicer.min_rows = min_rows;
        slicer.st = st;
        static const bool slice_env = [] {
            const char *e = std::getenv("SAMG_DIST_SLICED_GALERKIN");
            return !e || e[0] != '0';
        }();
        std::unique_ptr<Hierarchy> H(setup_hierarchy(std::move(A0), B, b_rows, b_cols, prm, s, t0,
                                                     pipeline, slice_env ? &slicer : nullptr));
        H->owns_stream = false;  // the caller destroys s if anything below throws
        DHierarchy *d = dsetup(std::move(H), comm, nranks, mine, st, min_rows);
        d->sliced_levels = slicer.sliced_levels;
        d->H->owns_stream = true;
        return d;
    } catch (...) {
        if (comm) nccl().CommDestroy(comm);
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
    int64_t n = 0;
    for (const DRank &R : d->ranks) n += 3 * R.nloc0;
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
    *row0 = d->ranks.front().row0;
    *row1 = d->ranks.back().row0 + d->ranks.back().nloc0;
    *nlevels = static_cast<int>(d->H->levels.size());
    *dist_levels = static_cast<int>(d->Ld);
    *setup_s = d->H->setup_seconds;
}

int dsliced_levels(const DHierarchy *d) { return d->sliced_levels; }
const Hierarchy &dfull(const DHierarchy *d) { return *d->H; }

void nccl_unique_id(unsigned char *out) {
    ncclUniqueId uid;
    NK(nccl().GetUniqueId(&uid));
    std::memcpy(out, &uid, sizeof uid);
}

} // namespace samgb
