// dsolve.cu -- multi-GPU solve: row-partitioned V-cycle + PCG over NCCL.
//
// One process per GPU (rank).  The setup is distributed (dsetup.cu): every
// rank builds only its rows of the large levels,
//   * level l (l < Ld) is row-partitioned: fine block rows [f0, f1) of A_l,
//     P_l, the smoother, and coarse block rows [c0, c1) of R_l.  The coarse
//     partition follows the aggregation: aggregate g belongs to the rank that
//     owns its pass-1 seed node, and aggregate ids are numbered in seed order
//     (coarsening.hpp:136-146), so every rank's coarse rows are contiguous;
//   * levels l >= Ld (fewer than min_rows * nranks block rows, or a rank
//     would own none) are gathered once and replicated: f_Ld is gathered on
//     every rank (grouped ncclBroadcast) and the coarse V-cycle runs
//     redundantly, so the prolongation into level Ld-1 needs no halo.
// Every local SpMV reads a halo-extended vector: owned entries first, then
// the ghosts sorted by global id (grouped by owner).  The halo plans are
// derived locally: a rank's ghosts are the columns its rows read outside its
// range, and what it sends to rank p are the owned entries p's rows read --
// the rows of the transposed operator (A for A, P for R, R for P) that hold
// a column in p's row range.  A halo exchange is pack kernel + grouped
// ncclSend/ncclRecv.  CG dot products are local fused reductions (the same
// kernels as on one GPU, in STORE mode) + one ncclAllReduce.
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

#include "dsetup.cuh"
#include "hierarchy.cuh"

namespace samgb {

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

// emulated all-reduce of CgScalars::tmp (and tmp2), sums in rank order
__global__ void k_sum_tmp(ScSet s, int two) {
    double t = 0, t2 = 0;
    for (int i = 0; i < s.n; ++i) { t += s.p[i]->tmp; t2 += s.p[i]->tmp2; }
    for (int i = 0; i < s.n; ++i) {
        s.p[i]->tmp = t;
        if (two) s.p[i]->tmp2 = t2;
    }
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
// flag[x] = 1 if row x of T has a column in [lo, hi)
__global__ void k_rows_reading(int64_t n, const int *ptr, const int *col, int64_t lo, int64_t hi,
                               int *flag) {
    for (int64_t x = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < n;
         x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int f = 0;
        for (int e = ptr[x]; e < ptr[x + 1] && !f; ++e) f = col[e] >= lo && col[e] < hi;
        flag[x] = f;
    }
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

// A rank's local operator from its own rows M (rows [row_starts[rank],
// row_starts[rank+1]) of the row space, global column ids in the column
// space partitioned by col_starts): columns renumbered into the
// halo-extended vector (owned first, then the ghosts in ascending global id,
// i.e. grouped by owner), the receive plan (ghost counts per owner) and the
// send plan.  The send plan comes from T, the rank's rows of the transposed
// operator (its owned column-space entries as rows, global ids of M's row
// space as columns): peer p reads the owned entries whose T row has a column
// in p's row range (pattern(T) = pattern(M^T): A is structurally symmetric,
// R = P^T exactly).  global_cols: keep global columns, no plan (the
// prolongation from a replicated level).  All on the device: flag arrays +
// scans, a few scalars to the host.
void build_local_rows(const Bsr3 &M, const Bsr3 *T, const std::vector<int64_t> &row_starts,
                      const std::vector<int64_t> &col_starts, int rank, bool global_cols,
                      LocalMat &out, cudaStream_t s) {
    const int nranks = static_cast<int>(row_starts.size()) - 1;
    const int64_t c0 = col_starts[rank], c1 = col_starts[rank + 1];
    const int64_t nl = M.nrows, nnz = M.nnzb;
    const int64_t ncg = col_starts[nranks];
    HaloPlan &pl = out.plan;
    DevBuf<int> gscan;
    if (!global_cols) {
        pl.nloc = c1 - c0;
        // ghosts: flags over the global column space, scanned
        DevBuf<int> gflag(ncg + 1, s);
        gscan.alloc(ncg + 1, s);
        CK(cudaMemsetAsync(gflag.p, 0, sizeof(int) * (ncg + 1), s));
        if (nnz) k_mark_cols<<<grid_of(nnz), 256, 0, s>>>(nnz, M.col.p, c0, c1, false, gflag.p);
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
        // send plan: for every other rank, the owned entries whose row of T
        // reads that rank's rows
        const int64_t nown = c1 - c0;
        DevBuf<int> sflag(nown + 1, s), sscan(nown + 1, s);
        std::vector<DevBuf<int>> parts;
        int64_t total = 0;
        for (int q = 0; q < nranks; ++q) {
            if (q == rank || !nown) continue;
            CK(cudaMemsetAsync(sflag.p, 0, sizeof(int) * (nown + 1), s));
            k_rows_reading<<<grid_of(nown), 256, 0, s>>>(nown, T->ptr.p, T->col.p, row_starts[q],
                                                        row_starts[q + 1], sflag.p);
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
    CK(cudaMemcpyAsync(A.ptr.p, M.ptr.p, sizeof(int) * (nl + 1), cudaMemcpyDeviceToDevice, s));
    if (nnz) {
        k_renumber<<<grid_of(nnz), 256, 0, s>>>(nnz, M.col.p, c0, c1, pl.nloc, gscan.p, global_cols,
                                               A.col.p);
        CK(cudaMemcpyAsync(A.val.p, M.val.p, sizeof(double) * 9 * nnz, cudaMemcpyDeviceToDevice, s));
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
    cudaStream_t s = nullptr;    // the solve stream (owned)
    samg_amg_params prm{};
    int pipeline = SAMG_PIPELINE_NS_BLOCK;
    double setup_seconds = 0;
    uint64_t footprint = 0;      // memory_footprint of the global hierarchy
    int64_t held_rows0 = 0;      // A_0 rows the setup held on the first driven rank
    std::unique_ptr<Hierarchy> Hc;  // levels Ld.. (replicated; level Ld = Hc level 0)
    size_t Ld = 0;
    std::vector<std::vector<int64_t>> starts;  // partition of levels 0..Ld
    std::vector<int64_t> nrows;  // global block rows of levels 0..Ld
    std::vector<std::vector<DPiece>> pieces;   // setup rows per level / driven rank (taps)
    std::vector<DRank> ranks;    // the ranks this process drives
    CgScalars *sc_host = nullptr;
    cudaStream_t cs = nullptr;   // halo transfers overlapped with interior rows
    cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
    cudaGraphExec_t cg_exec = nullptr;  // PCG loop body (device-side while)

    ~DHierarchy() {
        if (s) cudaStreamSynchronize(s);
        if (cs) cudaStreamSynchronize(cs);
        if (cg_exec) cudaGraphExecDestroy(cg_exec);
        ranks.clear();
        pieces.clear();
        Hc.reset();
        if (ev_pack) cudaEventDestroy(ev_pack);
        if (ev_halo) cudaEventDestroy(ev_halo);
        if (cs) cudaStreamDestroy(cs);
        if (s) cudaStreamDestroy(s);
        pinned_small_free(sc_host);
        if (comm) nccl().CommDestroy(comm);
    }

    cudaStream_t stream() const { return s; }
    bool emulated() const { return comm == nullptr; }
    Xport xport() const {
        Xport x;
        x.comm = comm;
        x.nranks = nranks;
        for (const DRank &R : ranks) x.mine.push_back(R.rank);
        x.s = s;
        return x;
    }

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

    // the sum over ranks of sc->tmp (count 1) or of (tmp, tmp2) (count 2)
    void allreduce_tmp(int count) {
        static_assert(offsetof(CgScalars, tmp2) == offsetof(CgScalars, tmp) + sizeof(double),
                      "tmp, tmp2 are all-reduced as one 2-double buffer");
        cudaStream_t s = stream();
        if (!emulated()) {
            double *t = reinterpret_cast<double *>(reinterpret_cast<char *>(ranks[0].sc.p) +
                                                   offsetof(CgScalars, tmp));
            NK(nccl().AllReduce(t, t, count, ncclDouble, ncclSum, comm, s));
        } else if (ranks.size() > 1) {
            ScSet set{};
            set.n = static_cast<int>(ranks.size());
            for (int i = 0; i < set.n; ++i) set.p[i] = ranks[i].sc.p;
            k_sum_tmp<<<1, 1, 0, s>>>(set, count == 2 ? 1 : 0);
            CK_LAUNCH();
        }
    }

    // the sum over ranks of sc->tmp, then the CG update `what`
    void allreduce_finish(int what) {
        allreduce_tmp(1);
        for (DRank &R : ranks) launch_cg_finish(R.sc.p, what, stream());
    }

    // one CG iteration after the first preconditioner application
    // (cg.hpp:58-77): q = A p, alpha; u, r update; z = M r; then r.r and
    // r.z in ONE 2-double all-reduce; beta; p = z + beta p.  rr_what:
    // CG_RR (host loop) or CG_RR_LOOP (sets the graph loop condition h).
    void cg_iteration(int rr_what, cudaGraphConditionalHandle h);
    void build_cg_graph();

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

void DHierarchy::cg_iteration(int rr_what, cudaGraphConditionalHandle h) {
    cudaStream_t st = stream();
    // q = A p overlapped with the halo: the first row range stores its
    // partial p.q, the others add to it
    std::vector<int> pieces_done(ranks.size(), 0);
    exchange_overlap(0, 0, [](DRank &R) { return R.pext.p; },
                     [&](DRank &R, int64_t a, int64_t b) {
        RowView v(R.dl[0].A.A, a, b);
        int &k = pieces_done[&R - ranks.data()];
        launch_spmv_dot_split(v.m, R.pext.p, R.pext.p + 3 * a, R.q.p + 3 * a, R.partials.p,
                              R.sc.p, st, k++ == 0 ? CG_STORE : CG_ADD);
    });
    allreduce_finish(CG_PQ);
    for (DRank &R : ranks)
        launch_cg_update(3 * R.nloc0, R.sc.p, R.pext.p, R.q.p, R.u.p, R.r.p, R.partials.p,
                         CG_STORE, 0, st);
    vcycle();
    for (DRank &R : ranks) launch_dot(3 * R.nloc0, R.r.p, R.z.p, R.partials.p, R.sc.p, CG_STORE2, st);
    allreduce_tmp(2);
    for (DRank &R : ranks) launch_cg_finish2(R.sc.p, rr_what, h, st);
    for (DRank &R : ranks) launch_p_update(3 * R.nloc0, R.sc.p, R.z.p, R.pext.p, st);
}

// The PCG loop as one CUDA graph with a device-side while node, as on one
// GPU: the halo sends / receives, the all-reduces and the replicated coarse
// V-cycle are captured with the rest; the loop condition is set on every
// rank from the same all-reduced r.r, so all ranks leave together.
void DHierarchy::build_cg_graph() {
    cudaStream_t st = stream();
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
    CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    cg_iteration(CG_RR_LOOP, h);
    cudaGraph_t captured = body;
    CK(cudaStreamEndCapture(st, &captured));
    CK(cudaGraphInstantiate(&cg_exec, g, 0));
    CK(cudaGraphDestroy(g));
}

// Distributed V-cycle (hierarchy.hpp:408-441) from a zero guess: z = M^-1 r
// on every driven rank.
void DHierarchy::vcycle() {
    cudaStream_t s = stream();
    const int pre = prm.pre_sweeps, post = prm.post_sweeps;
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
    for (DRank &R : ranks) Hc->vcycle_from(0, R.fLd.p, R.uLd.p, true, false);
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
    NvtxScope nvtx_scope("samg::dcg_solve (distributed)");
    cudaStream_t s = stream();
    const auto t0 = std::chrono::steady_clock::now();
    samg_solve_report rep{};
    rep.variant = pipeline;
    rep.setup_seconds = setup_seconds;
    const int64_t base0 = emulated() ? ranks[0].row0 : 0;
    auto off = [&](const DRank &R) { return 3 * (R.row0 - base0); };
    for (DRank &R : ranks) {
        d2d(R.r.p, d_f + off(R), 3 * R.nloc0, s);
        launch_fill(3 * R.nloc0, 0.0, R.u.p, s);
        CK(cudaMemsetAsync(R.sc.p, 0, sizeof(CgScalars), s));
    }
    auto read = [&] {
        CK(cudaMemcpyAsync(sc_host, ranks[0].sc.p, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
        stream_wait(comm, s);  // polls ncclCommGetAsyncError: a dead peer raises, no hang
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
        rep.preconditioner_bytes = footprint;
        rep.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (DRank &R : ranks) d2d(d_u + off(R), R.u.p, 3 * R.nloc0, s);
        CK(cudaStreamSynchronize(s));
    };
    if (norm_f == 0.0) {
        rep.converged = 1;
        finish(0.0);
        return rep;
    }
    static const bool use_graph = [] {
        const char *e = std::getenv("SAMG_CG_GRAPH");
        return !(e && e[0] == '0');
    }();
    vcycle();
    dots([](DRank &R) { return R.r.p; }, [](DRank &R) { return R.z.p; }, CG_RHO);
    for (DRank &R : ranks) d2d(R.pext.p, R.z.p, 3 * R.nloc0, s);
    double res_norm = norm_f;
    int iter = 0;
    if (cp.max_iterations > 0 && res_norm / norm_f > cp.tol) {
        for (DRank &R : ranks) {
            CgScalars *st = sc_host;
            CK(cudaMemcpyAsync(st, R.sc.p, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            st->norm_f = norm_f;
            st->tol = cp.tol;
            st->iter = 0;
            st->max_iter = cp.max_iterations;
            st->breakdown = 0;
            st->ticket = 0;
            CK(cudaMemcpyAsync(R.sc.p, st, sizeof(CgScalars), cudaMemcpyHostToDevice, s));
            CK(cudaStreamSynchronize(s));
        }
        if (use_graph) {
            if (!cg_exec) build_cg_graph();
            CK(cudaGraphLaunch(cg_exec, s));
            read();
            if (sc_host->breakdown)
                fail(SAMG_BREAKDOWN_NON_SPD, "cg: p'Ap <= 0, matrix or preconditioner not SPD");
            iter = sc_host->iter;
            res_norm = std::sqrt(sc_host->rr);
        } else {
            while (res_norm / norm_f > cp.tol && iter < cp.max_iterations) {
                cg_iteration(CG_RR, 0);
                read();
                if (sc_host->breakdown)
                    fail(SAMG_BREAKDOWN_NON_SPD, "cg: p'Ap <= 0, matrix or preconditioner not SPD");
                ++iter;
                res_norm = std::sqrt(sc_host->rr);
            }
        }
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

// The solve-side structures of the distributed hierarchy: every driven
// rank's local operators with their halo plans (from the setup's rows).
DHierarchy *dbuild(DSetup &&S, const Xport &x, const samg_amg_params &prm, int pipeline,
                   double t0) {
    auto D = std::make_unique<DHierarchy>();
    D->nranks = x.nranks;
    CK(cudaGetDevice(&D->device));
    D->s = x.s;
    D->comm = x.comm;
    D->prm = prm;
    D->pipeline = pipeline;
    cudaStream_t s = x.s;
    const size_t Ld = S.Ld();
    D->Ld = Ld;
    D->starts = S.starts;
    D->nrows = S.nrows;
    D->footprint = S.footprint;
    D->held_rows0 = S.held_rows.empty() ? 0 : S.held_rows[0];
    D->ranks.resize(x.mine.size());
    const std::vector<int64_t> &row_starts = S.starts[0];
    for (size_t i = 0; i < x.mine.size(); ++i) {
        DRank &R = D->ranks[i];
        R.rank = x.mine[i];
        R.row0 = row_starts[R.rank];
        R.nloc0 = row_starts[R.rank + 1] - R.row0;
        R.dl.resize(Ld);
    }
    for (size_t l = 0; l < Ld; ++l) {
        const std::vector<int64_t> &fst = S.starts[l], &cst = S.starts[l + 1];
        const bool next_replicated = l + 1 == Ld;
        for (size_t i = 0; i < D->ranks.size(); ++i) {
            DRank &R = D->ranks[i];
            const DPiece &pc = S.lv[l][i];
            DLevel &dlv = R.dl[l];
            build_local_rows(pc.A, &pc.A, fst, fst, R.rank, false, dlv.A, s);
            build_local_rows(pc.R, &pc.P, cst, fst, R.rank, false, dlv.R, s);
            build_local_rows(pc.P, &pc.R, fst, cst, R.rank, next_replicated, dlv.P, s);
            const int64_t nl = fst[R.rank + 1] - fst[R.rank];
            const int per = pc.M.kind == SM_POINT ? 3 : 9;
            dlv.M.kind = pc.M.kind;
            dlv.M.data.alloc(per * nl + 1, s);
            if (nl)
                CK(cudaMemcpyAsync(dlv.M.data.p, pc.M.data.p, sizeof(double) * per * nl,
                                   cudaMemcpyDeviceToDevice, s));
            dlv.f.alloc(3 * nl + 3, s);
            dlv.t.alloc(3 * nl + 3, s);
            dlv.uA.alloc(3 * (dlv.A.plan.nloc + dlv.A.plan.nghost) + 3, s);
            dlv.rR.alloc(3 * (dlv.R.plan.nloc + dlv.R.plan.nghost) + 3, s);
            if (!next_replicated) dlv.uP.alloc(3 * (dlv.P.plan.nloc + dlv.P.plan.nghost) + 3, s);
        }
    }
    const int64_t nLd = S.nrows[Ld];
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
    D->Hc = std::move(S.coarse);
    D->pieces = std::move(S.lv);
    D->setup_seconds = std::chrono::duration<double>(
        std::chrono::steady_clock::now().time_since_epoch()).count() - t0;
    return D.release();
}

} // namespace samgb

// ---- entry points used by capi.cu ------------------------------------------
namespace samgb {

// Distributed setup.  NCCL (id != nullptr): this process is `rank` and
// passes only its own rows -- block rows [row_starts[rank],
// row_starts[rank+1]) as (nloc, ptr from 0, global column ids, values) and
// its nullspace rows (3*nloc x b_cols, column-major).  Emulated (id ==
// nullptr): every rank in this process, the rows and nullspace given for
// the whole matrix and cut here.
DHierarchy *dsetup_all(const unsigned char *id, int nranks, int rank, int64_t nbrows,
                       Bsr3 &&A_rows, const double *B, int64_t b_cols,
                       const int64_t *row_starts, int64_t min_rows, const samg_amg_params &prm,
                       cudaStream_t s, double t0, int pipeline) {
    if (!id && nranks > kMaxEmulated) fail(SAMG_INVALID_ARGUMENT, "dsetup: at most 16 emulated ranks");
    if (prm.smoother == SAMG_SMOOTHER_ILU0)
        fail(SAMG_UNSUPPORTED, "multi-GPU solve: the ILU(0) sweeps are sequential across row partitions");
    if (pipeline == SAMG_PIPELINE_SCALAR || pipeline == SAMG_PIPELINE_NS_SCALAR)
        fail(SAMG_UNSUPPORTED, "multi-GPU solve: the scalar pipelines are single-GPU");
    std::vector<int64_t> st(nranks + 1);
    if (row_starts) {
        st.assign(row_starts, row_starts + nranks + 1);
        if (st[0] != 0 || st[nranks] != nbrows)
            fail(SAMG_INVALID_ARGUMENT, "dsetup: row_starts must span [0, nbrows]");
    } else {
        for (int q = 0; q <= nranks; ++q) st[q] = nbrows * q / nranks;
    }
    for (int q = 0; q < nranks; ++q)
        if (st[q + 1] <= st[q]) fail(SAMG_INVALID_ARGUMENT, "dsetup: every rank needs at least one block row");
    Xport x;
    x.nranks = nranks;
    x.s = s;
    if (id) x.mine.push_back(rank);
    else for (int q = 0; q < nranks; ++q) x.mine.push_back(q);
    const bool block = pipeline == SAMG_PIPELINE_BLOCK;
    std::vector<Bsr3> A_own(x.mine.size());
    std::vector<DevBuf<double>> B_own(x.mine.size());
    if (id) {
        if (A_rows.nrows != st[rank + 1] - st[rank])
            fail(SAMG_DIMENSION_MISMATCH, "dsetup: local rows disagree with row_starts");
        A_own[0] = std::move(A_rows);
        if (!block) {
            const int64_t n3 = 3 * A_own[0].nrows;
            B_own[0].alloc(n3 * b_cols + 1, s);
            CK(cudaMemcpyAsync(B_own[0].p, B, sizeof(double) * n3 * b_cols, cudaMemcpyDefault, s));
        }
    } else {
        // cut the global input
        for (int q = 0; q < nranks; ++q) {
            slice_rows(A_rows, st[q], st[q + 1], A_own[q], s);
            if (!block) {
                const int64_t n3 = 3 * (st[q + 1] - st[q]), N3 = 3 * nbrows;
                B_own[q].alloc(n3 * b_cols + 1, s);
                CK(cudaMemcpy2DAsync(B_own[q].p, sizeof(double) * n3, B + 3 * st[q], sizeof(double) * N3,
                                     sizeof(double) * n3, b_cols, cudaMemcpyDefault, s));
            }
        }
        A_rows = Bsr3();
    }
    ncclComm_t comm = nullptr;
    if (id) {
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        NK(nccl().CommInitRank(&comm, nranks, uid, rank));
    }
    x.comm = comm;
    try {
        DSetup S = dist_setup(x, std::move(A_own), std::move(B_own), b_cols, st, min_rows, prm,
                              pipeline, t0);
        return dbuild(std::move(S), x, prm, pipeline, t0);
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
    *nlevels = static_cast<int>(d->Ld + d->Hc->levels.size());
    *dist_levels = static_cast<int>(d->Ld);
    *setup_s = d->setup_seconds;
}

int64_t dheld_rows(const DHierarchy *d) { return d->held_rows0; }

// Parity tap: level `level`'s A (0), P (1) or R (2) as the global matrix --
// assembled from every rank's rows for a distributed level (a collective
// over the communicator), the replicated matrix otherwise.
const Bsr3 &dlevel(DHierarchy *d, int level, int which, Bsr3 &tmp) {
    if (level < 0) fail(SAMG_INVALID_ARGUMENT, "level out of range");
    if (static_cast<size_t>(level) >= d->Ld) {
        const size_t l = level - d->Ld;
        if (l >= d->Hc->levels.size()) fail(SAMG_INVALID_ARGUMENT, "level out of range");
        const Level &lv = d->Hc->levels[l];
        if (which != 0 && !lv.has_transfer) fail(SAMG_INVALID_ARGUMENT, "no transfer operators on the coarsest level");
        return which == 0 ? lv.A : which == 1 ? lv.P : lv.R;
    }
    if (which < 0 || which > 2) fail(SAMG_INVALID_ARGUMENT, "which must be 0, 1 or 2");
    CK(cudaSetDevice(d->device));
    const Xport x = d->xport();
    std::vector<const Bsr3 *> own;
    for (const DPiece &pc : d->pieces[level]) own.push_back(which == 0 ? &pc.A : which == 1 ? &pc.P : &pc.R);
    const std::vector<int64_t> &rows = which == 2 ? d->starts[level + 1] : d->starts[level];
    const int64_t ncols = which == 1 ? d->nrows[level + 1] : d->nrows[level];
    gather_matrix(x, own, rows, ncols, tmp);
    return tmp;
}

void nccl_unique_id(unsigned char *out) {
    ncclUniqueId uid;
    NK(nccl().GetUniqueId(&uid));
    std::memcpy(out, &uid, sizeof uid);
}

} // namespace samgb
