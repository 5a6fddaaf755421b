// dsetup.cu -- distributed setup of the multi-GPU hierarchy.
//
// Every rank owns a contiguous block-row range of each large level and
// builds only those rows; nothing global is formed except the node graph of
// the strength test (0.6 GB at C4), which every rank holds so that the
// aggregation -- order dependent, coarsening.hpp:131-160 -- runs the very
// kernels of the single-GPU setup and yields the reference's aggregates.
// Per level l (rank q owns block rows [f0, f1), nodes [n0, n1)):
//
//  1. A halo: the rows of the other ranks that q's rows reference (one
//     layer; structurally symmetric A, so the owner knows which to send).
//  2. strength_graph on q's rows + halo (coarsening.hpp:52-123): q's node
//     rows of G are exact (the union test of an edge needs both rows).
//  3. G gathered on every rank; aggregate() (coarsening.hpp:131-160) on it:
//     identical ids everywhere.  Ownership rule: aggregate g belongs to the
//     rank owning its pass-1 seed; ids are numbered in seed order, so q owns
//     the contiguous aggregates [seedno[n0], seedno[n1]) -- the coarse rows
//     of level l+1.
//  4. ns pipelines: the nullspace rows of the nodes of q's aggregates are
//     fetched from their owners, q runs the thin QR of its own aggregates
//     only (coarsening.hpp:238-312) -> P_tent rows of their nodes and the
//     coarse nullspace rows q owns; the P_tent rows of q's nodes and their
//     strong neighbours are then fetched from the aggregates' owners and q
//     smooths its own rows of P (coarsening.hpp:319-416).  block pipeline:
//     q forms its rows of the block transfer (coarsening.hpp:471-560).
//  5. Galerkin: q forms its coarse rows A_c[c0:c1) = (R[c0:c1) A) P with
//     the kernels of the single-GPU product (bit-identical rows) from the
//     rows of A and P it needs -- S1 = the fine rows in its rows of R, S2 =
//     S1 and their A-neighbours -- fetched from the owners (each owner
//     decides from the global G and aggregates which of its rows a rank
//     needs; the receiver learns the counts in one all-to-all).
//
// The exchange plans are all derived locally from data every rank holds
// (G, aggregates, the partitions, the rank's own rows); the only collective
// besides the data itself is the small all-to-all of row / block counts.
// Every step runs for the ranks this process drives: one rank over NCCL,
// or all of them emulated in lock step on one GPU (comm == nullptr, each
// exchange a device copy with the offsets and counts of the NCCL calls).
#include "dsetup.cuh"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <numeric>

#include <cub/cub.cuh>

namespace samgb {

namespace {

int gridn(int64_t n) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8192, (n + 255) / 256))); }

template <class F>
__global__ void k_each(int64_t n, F f) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        f(i);
}
template <class F>
void each(int64_t n, F f, cudaStream_t s) {
    if (n <= 0) return;
    k_each<<<gridn(n), 256, 0, s>>>(n, f);
    CK_LAUNCH();
}

// rank q with st[q] <= x < st[q+1]
__device__ __forceinline__ int owner_of(int64_t x, const int64_t *st, int nr) {
    int lo = 0, hi = nr - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (st[mid] <= x) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// exclusive scan of c[0, n) (int) into o[0, n] (int), o[n] = total
int64_t exscan(const int *c, int *o, int64_t n, cudaStream_t s) {
    DevBuf<int64_t> t(n + 1, s);
    int64_t *tp = t.p;
    each(n, [=] __device__(int64_t i) { tp[i] = c[i]; }, s);
    CK(cudaMemsetAsync(tp + n, 0, sizeof(int64_t), s));
    size_t bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, tp, tp, n + 1, s));
    DevBuf<char> ws(bytes + 1, s);
    CK(cub::DeviceScan::ExclusiveSum(ws.p, bytes, tp, tp, n + 1, s));
    int64_t total = 0;
    CK(cudaMemcpyAsync(&total, tp + n, sizeof total, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (total > INT32_MAX) fail(SAMG_UNSUPPORTED, "dsetup: more than 2^31-1 entries");
    each(n + 1, [=] __device__(int64_t i) { o[i] = static_cast<int>(tp[i]); }, s);
    return total;
}

// indices i in [0, n) with flag[i] != 0, ascending
void compact(const int *flag, int64_t n, DevBuf<int> &out, cudaStream_t s) {
    DevBuf<int> off(n + 1, s);
    const int64_t m = exscan(flag, off.p, n, s);
    out.alloc(m + 1, s);
    out.n = m;
    int *o = out.p;
    const int *op = off.p;
    each(n, [=] __device__(int64_t i) { if (flag[i]) o[op[i]] = static_cast<int>(i); }, s);
    CK(cudaStreamSynchronize(s));  // off is freed on s
}

template <class T>
DevBuf<T> to_dev(const std::vector<T> &h, cudaStream_t s) {
    DevBuf<T> d(h.size() + 1, s);
    if (!h.empty()) CK(cudaMemcpyAsync(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, s));
    return d;
}

int read_int(const int *p, cudaStream_t s) {
    int v = 0;
    CK(cudaMemcpyAsync(&v, p, sizeof v, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return v;
}

// ---- matrix rows in transit -------------------------------------------------
// Received rows of a matrix: global row ids, lengths, then the columns and
// values of all rows back to back (in the order of ids).
struct RowsIn {
    int64_t nr = 0, nb = 0;
    DevBuf<int> ids, lens, col;
    DevBuf<double> val;
};

// Driven rank i sends, to every peer p, the rows lists[i][p] (local row
// indices of M[i], ascending) of its matrix M[i] whose local row 0 is the
// global row gid0[i].  Returns what every driven rank received.
std::vector<RowsIn> exchange_rows(const Xport &x, const std::vector<const Bsr3 *> &M,
                                  const std::vector<int64_t> &gid0,
                                  const std::vector<std::vector<DevBuf<int>>> &lists) {
    const int nr = x.nranks;
    const size_t nd = x.mine.size();
    cudaStream_t s = x.s;
    // per driven rank: concatenated send rows (peer order), their lengths and
    // the block offsets
    std::vector<std::vector<int64_t>> cnt(nd, std::vector<int64_t>(2 * nr, 0));
    std::vector<DevBuf<int>> rows(nd), lens(nd), boff(nd);
    std::vector<std::vector<int64_t>> rbase(nd, std::vector<int64_t>(nr + 1, 0));
    for (size_t i = 0; i < nd; ++i) {
        for (int p = 0; p < nr; ++p)
            rbase[i][p + 1] = rbase[i][p] + static_cast<int64_t>(lists[i][p].n);
        const int64_t tot = rbase[i][nr];
        rows[i].alloc(tot + 1, s);
        for (int p = 0; p < nr; ++p)
            if (lists[i][p].n)
                CK(cudaMemcpyAsync(rows[i].p + rbase[i][p], lists[i][p].p, sizeof(int) * lists[i][p].n,
                                   cudaMemcpyDeviceToDevice, s));
        lens[i].alloc(tot + 1, s);
        boff[i].alloc(tot + 1, s);
        const int *rp = rows[i].p, *mp = M[i]->ptr.p;
        int *lp = lens[i].p;
        each(tot, [=] __device__(int64_t t) { lp[t] = mp[rp[t] + 1] - mp[rp[t]]; }, s);
        exscan(lens[i].p, boff[i].p, tot, s);
        std::vector<int> hb(nr + 1);
        for (int p = 0; p <= nr; ++p)
            CK(cudaMemcpyAsync(&hb[p], boff[i].p + rbase[i][p], sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (int p = 0; p < nr; ++p) {
            cnt[i][2 * p] = rbase[i][p + 1] - rbase[i][p];
            cnt[i][2 * p + 1] = hb[p + 1] - hb[p];
        }
    }
    const auto rc = alltoall_counts(x, cnt, 2);
    // int segment per peer: [ids (nr) | lens (nr) | cols (nb)]; val segment: 9 nb
    std::vector<std::vector<int64_t>> sio(nd), svo(nd), rio(nd), rvo(nd);
    std::vector<DevBuf<int>> sint(nd), rint(nd);
    std::vector<DevBuf<double>> sval(nd);
    std::vector<RowsIn> in(nd);
    for (size_t i = 0; i < nd; ++i) {
        sio[i].assign(nr + 1, 0); svo[i].assign(nr + 1, 0); rio[i].assign(nr + 1, 0); rvo[i].assign(nr + 1, 0);
        for (int p = 0; p < nr; ++p) {
            sio[i][p + 1] = sio[i][p] + 2 * cnt[i][2 * p] + cnt[i][2 * p + 1];
            svo[i][p + 1] = svo[i][p] + 9 * cnt[i][2 * p + 1];
            rio[i][p + 1] = rio[i][p] + 2 * rc[i][2 * p] + rc[i][2 * p + 1];
            rvo[i][p + 1] = rvo[i][p] + 9 * rc[i][2 * p + 1];
        }
        sint[i].alloc(sio[i][nr] + 1, s);
        sval[i].alloc(svo[i][nr] + 1, s);
        // pack: row t of peer p
        std::vector<int64_t> meta;  // per peer: rbase, nrows, int offset, block base
        for (int p = 0; p < nr; ++p) {
            meta.push_back(rbase[i][p]);
            meta.push_back(cnt[i][2 * p]);
            meta.push_back(sio[i][p]);
        }
        meta.push_back(rbase[i][nr]);
        DevBuf<int64_t> dm = to_dev(meta, s);
        const int64_t tot = rbase[i][nr];
        const int *rp = rows[i].p, *lp = lens[i].p, *bo = boff[i].p, *mp = M[i]->ptr.p, *mc = M[i]->col.p;
        const double *mv = M[i]->val.p;
        const int64_t *md = dm.p;
        int *si = sint[i].p;
        double *sv = sval[i].p;
        const int g0 = static_cast<int>(gid0[i]);
        const int nrk = nr;
        // one warp per row
        each(tot * 32, [=] __device__(int64_t w) {
            const int64_t t = w >> 5;
            const int lane = static_cast<int>(w & 31);
            int p = 0;
            while (p + 1 < nrk && md[3 * (p + 1)] <= t) ++p;
            const int64_t k = t - md[3 * p], npr = md[3 * p + 1], io = md[3 * p + 2];
            const int64_t b0p = bo[md[3 * p]];       // first block of peer p
            const int64_t bt = bo[t] - b0p;           // row t's blocks within the segment
            const int r = rp[t], len = lp[t], src = mp[r];
            if (lane == 0) {
                si[io + k] = g0 + r;
                si[io + npr + k] = len;
            }
            for (int e = lane; e < len; e += 32) si[io + 2 * npr + bt + e] = mc[src + e];
            for (int e = lane; e < 9 * len; e += 32)
                sv[9 * (b0p + bt) + e] = mv[9 * static_cast<int64_t>(src) + e];
        }, s);
        in[i].nr = 0;
        in[i].nb = 0;
        for (int p = 0; p < nr; ++p) {
            in[i].nr += rc[i][2 * p];
            in[i].nb += rc[i][2 * p + 1];
        }
        rint[i].alloc(rio[i][nr] + 1, s);
        in[i].val.alloc(9 * in[i].nb + 1, s);
    }
    // bytes
    auto bytes_of = [](const std::vector<int64_t> &o, size_t w) {
        std::vector<int64_t> b(o.size());
        for (size_t k = 0; k < o.size(); ++k) b[k] = o[k] * static_cast<int64_t>(w);
        return b;
    };
    {
        std::vector<const char *> src(nd);
        std::vector<char *> dst(nd);
        std::vector<std::vector<int64_t>> so(nd), ro(nd);
        for (size_t i = 0; i < nd; ++i) {
            src[i] = reinterpret_cast<const char *>(sint[i].p);
            dst[i] = reinterpret_cast<char *>(rint[i].p);
            so[i] = bytes_of(sio[i], sizeof(int));
            ro[i] = bytes_of(rio[i], sizeof(int));
        }
        xchg_bytes(x, src, so, dst, ro);
        for (size_t i = 0; i < nd; ++i) {
            src[i] = reinterpret_cast<const char *>(sval[i].p);
            dst[i] = reinterpret_cast<char *>(in[i].val.p);
            so[i] = bytes_of(svo[i], sizeof(double));
            ro[i] = bytes_of(rvo[i], sizeof(double));
        }
        xchg_bytes(x, src, so, dst, ro);
    }
    // unpack the int segments into contiguous ids / lens / cols
    for (size_t i = 0; i < nd; ++i) {
        RowsIn &R = in[i];
        R.ids.alloc(R.nr + 1, s);
        R.lens.alloc(R.nr + 1, s);
        R.col.alloc(R.nb + 1, s);
        int64_t ro = 0, bo = 0;
        for (int p = 0; p < nr; ++p) {
            const int64_t n1 = rc[i][2 * p], b1 = rc[i][2 * p + 1];
            const int *seg = rint[i].p + rio[i][p];
            if (n1) {
                CK(cudaMemcpyAsync(R.ids.p + ro, seg, sizeof(int) * n1, cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(R.lens.p + ro, seg + n1, sizeof(int) * n1, cudaMemcpyDeviceToDevice, s));
            }
            if (b1) CK(cudaMemcpyAsync(R.col.p + bo, seg + 2 * n1, sizeof(int) * b1, cudaMemcpyDeviceToDevice, s));
            ro += n1;
            bo += b1;
        }
    }
    CK(cudaStreamSynchronize(s));
    return in;
}

// Global-numbered matrix (nrows = N; only the rows of `own` (local row 0 =
// global gid0) and of `in` are non-empty).
void assemble(int64_t N, int64_t ncols, const Bsr3 &own, int64_t gid0, const RowsIn &in, Bsr3 &out,
              cudaStream_t s) {
    DevBuf<int> len(N + 1, s);
    CK(cudaMemsetAsync(len.p, 0, sizeof(int) * (N + 1), s));
    int *lp = len.p;
    const int *op = own.ptr.p, *ii = in.ids.p, *il = in.lens.p;
    const int64_t g0 = gid0;
    each(own.nrows, [=] __device__(int64_t r) { lp[g0 + r] = op[r + 1] - op[r]; }, s);
    each(in.nr, [=] __device__(int64_t t) { lp[ii[t]] = il[t]; }, s);
    out.nrows = N;
    out.ncols = ncols;
    out.ptr.alloc(N + 1, s);
    out.nnzb = exscan(len.p, out.ptr.p, N, s);
    out.col.alloc(out.nnzb + 1, s);
    out.val.alloc(9 * out.nnzb + 1, s);
    const int *pp = out.ptr.p, *oc = own.col.p;
    int *dc = out.col.p;
    const double *ov = own.val.p;
    double *dv = out.val.p;
    each(own.nrows * 32, [=] __device__(int64_t w) {
        const int64_t r = w >> 5;
        const int lane = static_cast<int>(w & 31);
        const int a = op[r], n = op[r + 1] - a, d = pp[g0 + r];
        for (int e = lane; e < n; e += 32) dc[d + e] = oc[a + e];
        for (int e = lane; e < 9 * n; e += 32) dv[9 * static_cast<int64_t>(d) + e] = ov[9 * static_cast<int64_t>(a) + e];
    }, s);
    if (in.nr) {
        DevBuf<int> ioff(in.nr + 1, s);
        exscan(in.lens.p, ioff.p, in.nr, s);
        const int *io = ioff.p, *ic = in.col.p;
        const double *iv = in.val.p;
        each(in.nr * 32, [=] __device__(int64_t w) {
            const int64_t t = w >> 5;
            const int lane = static_cast<int>(w & 31);
            const int a = io[t], n = il[t], d = pp[ii[t]];
            for (int e = lane; e < n; e += 32) dc[d + e] = ic[a + e];
            for (int e = lane; e < 9 * n; e += 32) dv[9 * static_cast<int64_t>(d) + e] = iv[9 * static_cast<int64_t>(a) + e];
        }, s);
        CK(cudaStreamSynchronize(s));
    }
}

// rows of M (local) whose flag kernel f(row) is true, ascending
template <class F>
void rows_where(int64_t n, F f, DevBuf<int> &out, cudaStream_t s) {
    DevBuf<int> flag(n + 1, s);
    int *fl = flag.p;
    each(n, [=] __device__(int64_t r) { fl[r] = f(r) ? 1 : 0; }, s);
    compact(flag.p, n, out, s);
}

// Fixed-width node rows in transit: driven rank i sends lists[i][p] (global
// node ids, ascending) packed by pack(node, t, buf) and the receiver stores
// them with store(node, buf); both sides know the lists.
template <class Pack, class Store>
void exchange_nodes(const Xport &x, const std::vector<std::vector<DevBuf<int>>> &send_lists,
                    const std::vector<std::vector<DevBuf<int>>> &recv_lists, int W,
                    const std::vector<Pack> &pack, const std::vector<Store> &store) {
    const int nr = x.nranks;
    const size_t nd = x.mine.size();
    cudaStream_t s = x.s;
    std::vector<DevBuf<double>> sb(nd), rb(nd);
    std::vector<std::vector<int64_t>> so(nd, std::vector<int64_t>(nr + 1, 0)), ro(nd, std::vector<int64_t>(nr + 1, 0));
    for (size_t i = 0; i < nd; ++i) {
        for (int p = 0; p < nr; ++p) {
            so[i][p + 1] = so[i][p] + static_cast<int64_t>(send_lists[i][p].n) * W * 8;
            ro[i][p + 1] = ro[i][p] + static_cast<int64_t>(recv_lists[i][p].n) * W * 8;
        }
        sb[i].alloc(so[i][nr] / 8 + 1, s);
        rb[i].alloc(ro[i][nr] / 8 + 1, s);
        for (int p = 0; p < nr; ++p) {
            const int64_t m = send_lists[i][p].n;
            if (!m) continue;
            const int *L = send_lists[i][p].p;
            double *b = sb[i].p + so[i][p] / 8;
            const Pack pk = pack[i];
            const int w = W;
            each(m * w, [=] __device__(int64_t e) { const int64_t t = e / w; pk(L[t], static_cast<int>(e - t * w), b + e); }, s);
        }
    }
    std::vector<const char *> src(nd);
    std::vector<char *> dst(nd);
    for (size_t i = 0; i < nd; ++i) {
        src[i] = reinterpret_cast<const char *>(sb[i].p);
        dst[i] = reinterpret_cast<char *>(rb[i].p);
    }
    xchg_bytes(x, src, so, dst, ro);
    for (size_t i = 0; i < nd; ++i)
        for (int p = 0; p < nr; ++p) {
            const int64_t m = recv_lists[i][p].n;
            if (!m) continue;
            const int *L = recv_lists[i][p].p;
            const double *b = rb[i].p + ro[i][p] / 8;
            const Store st = store[i];
            const int w = W;
            each(m * w, [=] __device__(int64_t e) { const int64_t t = e / w; st(L[t], static_cast<int>(e - t * w), b[e]); }, s);
        }
    CK(cudaStreamSynchronize(s));
}

// Variable pieces of every rank, concatenated in rank order into `out`
// (every driven process gets the whole).  counts[q] elements of T from rank q.
template <class T>
void allgatherv(const Xport &x, const std::vector<const T *> &piece, const std::vector<int64_t> &counts,
                T *out) {
    cudaStream_t s = x.s;
    std::vector<int64_t> off(x.nranks + 1, 0);
    for (int q = 0; q < x.nranks; ++q) off[q + 1] = off[q] + counts[q];
    for (size_t i = 0; i < x.mine.size(); ++i) {
        const int q = x.mine[i];
        if (counts[q])
            CK(cudaMemcpyAsync(out + off[q], piece[i], sizeof(T) * counts[q], cudaMemcpyDeviceToDevice, s));
    }
    if (!x.emu()) {
        NK(nccl().GroupStart());
        for (int q = 0; q < x.nranks; ++q)
            if (counts[q])
                NK(nccl().Broadcast(out + off[q], out + off[q], sizeof(T) * counts[q], ncclChar, q,
                                    x.comm, s));
        NK(nccl().GroupEnd());
    }
    CK(cudaStreamSynchronize(s));
}

// what every rank needs of a level, held once per process: the node graph,
// the aggregates and the masks derived from them
struct LvGlobal {
    int64_t N = 0, h = 1, nnodes = 0, naggs = 0, kb = 1;
    std::vector<int64_t> fst, nst, ast;  // block-row / node / aggregate starts per rank
    DevBuf<int64_t> d_nst, d_ast;
    Graph G;
    DevBuf<int> agg, seedno;
};

// pack / store of node rows: the nullspace (owner's local column-major
// rows -> a global column-major array) and P_tent (global node-major rows)
struct PackB {
    const double *b; int64_t nl3, o3; int pbs, k;
    __device__ void operator()(int node, int w, double *out) const {
        const int r = w / k, c = w - r * k;
        *out = b[c * nl3 + (static_cast<int64_t>(node) * pbs + r - o3)];
    }
};
struct StoreB {
    double *bx; int64_t nfine; int pbs, k;
    __device__ void operator()(int node, int w, double v) const {
        const int r = w / k, c = w - r * k;
        bx[c * nfine + static_cast<int64_t>(node) * pbs + r] = v;
    }
};
struct PackP {
    const double *pt; int W;
    __device__ void operator()(int node, int w, double *out) const {
        *out = pt[static_cast<int64_t>(node) * W + w];
    }
};
struct StoreP {
    double *pt; int W;
    __device__ void operator()(int node, int w, double v) const {
        pt[static_cast<int64_t>(node) * W + w] = v;
    }
};

} // namespace

// ---- transport ----------------------------------------------------------------

void xchg_bytes(const Xport &x, const std::vector<const char *> &src,
                const std::vector<std::vector<int64_t>> &soff, const std::vector<char *> &dst,
                const std::vector<std::vector<int64_t>> &roff) {
    const int nr = x.nranks;
    if (!x.emu()) {
        const int me = x.mine[0];
        NK(nccl().GroupStart());
        for (int p = 0; p < nr; ++p) {
            if (p == me) continue;
            const int64_t sn = soff[0][p + 1] - soff[0][p], rn = roff[0][p + 1] - roff[0][p];
            if (sn) NK(nccl().Send(src[0] + soff[0][p], sn, ncclChar, p, x.comm, x.s));
            if (rn) NK(nccl().Recv(dst[0] + roff[0][p], rn, ncclChar, p, x.comm, x.s));
        }
        NK(nccl().GroupEnd());
        return;
    }
    // emulated: driven rank i = rank x.mine[i]; every rank is driven
    for (size_t i = 0; i < x.mine.size(); ++i) {
        const int me = x.mine[i];
        for (size_t j = 0; j < x.mine.size(); ++j) {
            const int p = x.mine[j];
            if (p == me) continue;
            const int64_t rn = roff[i][p + 1] - roff[i][p];
            const int64_t sn = soff[j][me + 1] - soff[j][me];
            if (rn != sn) fail(SAMG_ERROR, "dsetup: exchange sizes disagree between ranks");
            if (rn)
                CK(cudaMemcpyAsync(dst[i] + roff[i][p], src[j] + soff[j][me], rn, cudaMemcpyDeviceToDevice,
                                   x.s));
        }
    }
}

std::vector<std::vector<int64_t>> alltoall_counts(const Xport &x,
                                                  const std::vector<std::vector<int64_t>> &send,
                                                  int W) {
    const int nr = x.nranks;
    const size_t nd = x.mine.size();
    std::vector<std::vector<int64_t>> out(nd, std::vector<int64_t>(static_cast<size_t>(nr) * W, 0));
    if (x.emu()) {
        for (size_t i = 0; i < nd; ++i)
            for (size_t j = 0; j < nd; ++j)
                for (int w = 0; w < W; ++w)
                    out[i][x.mine[j] * W + w] = send[j][x.mine[i] * W + w];
        return out;
    }
    DevBuf<int64_t> d(static_cast<size_t>(nr) * nr * W + 1, x.s);
    const int me = x.mine[0];
    CK(cudaMemcpyAsync(d.p + static_cast<size_t>(me) * nr * W, send[0].data(), sizeof(int64_t) * nr * W,
                       cudaMemcpyHostToDevice, x.s));
    NK(nccl().AllGather(d.p + static_cast<size_t>(me) * nr * W, d.p, static_cast<size_t>(nr) * W, ncclInt64,
                        x.comm, x.s));
    std::vector<int64_t> all(static_cast<size_t>(nr) * nr * W);
    CK(cudaMemcpyAsync(all.data(), d.p, sizeof(int64_t) * all.size(), cudaMemcpyDeviceToHost, x.s));
    stream_wait(x.comm, x.s);
    for (int p = 0; p < nr; ++p)
        for (int w = 0; w < W; ++w) out[0][p * W + w] = all[(static_cast<size_t>(p) * nr + me) * W + w];
    return out;
}

std::vector<int64_t> allreduce_sum(const Xport &x, const std::vector<std::vector<int64_t>> &v) {
    const size_t W = v[0].size();
    std::vector<int64_t> out(W, 0);
    if (x.emu()) {
        for (const auto &r : v)
            for (size_t w = 0; w < W; ++w) out[w] += r[w];
        return out;
    }
    DevBuf<int64_t> d(W + 1, x.s);
    CK(cudaMemcpyAsync(d.p, v[0].data(), sizeof(int64_t) * W, cudaMemcpyHostToDevice, x.s));
    NK(nccl().AllReduce(d.p, d.p, W, ncclInt64, ncclSum, x.comm, x.s));
    CK(cudaMemcpyAsync(out.data(), d.p, sizeof(int64_t) * W, cudaMemcpyDeviceToHost, x.s));
    stream_wait(x.comm, x.s);
    return out;
}

void gather_matrix(const Xport &x, const std::vector<const Bsr3 *> &own,
                   const std::vector<int64_t> &row_starts, int64_t ncols, Bsr3 &out) {
    cudaStream_t s = x.s;
    const int nr = x.nranks;
    const int64_t N = row_starts[nr];
    std::vector<std::vector<int64_t>> nb(own.size(), std::vector<int64_t>(nr, 0));
    for (size_t i = 0; i < own.size(); ++i) nb[i][x.mine[i]] = own[i]->nnzb;
    const std::vector<int64_t> cnt = allreduce_sum(x, nb);
    // row lengths, then columns and values, concatenated in rank order
    DevBuf<int> len(N + 1, s);
    std::vector<DevBuf<int>> lp(own.size());
    std::vector<const int *> lpp(own.size()), cpp(own.size());
    std::vector<const double *> vpp(own.size());
    std::vector<int64_t> rc(nr);
    for (int q = 0; q < nr; ++q) rc[q] = row_starts[q + 1] - row_starts[q];
    for (size_t i = 0; i < own.size(); ++i) {
        lp[i].alloc(own[i]->nrows + 1, s);
        int *l = lp[i].p;
        const int *p = own[i]->ptr.p;
        each(own[i]->nrows, [=] __device__(int64_t r) { l[r] = p[r + 1] - p[r]; }, s);
        lpp[i] = lp[i].p;
        cpp[i] = own[i]->col.p;
        vpp[i] = own[i]->val.p;
    }
    allgatherv<int>(x, lpp, rc, len.p);
    out.nrows = N;
    out.ncols = ncols;
    out.ptr.alloc(N + 1, s);
    out.nnzb = exscan(len.p, out.ptr.p, N, s);
    out.col.alloc(out.nnzb + 1, s);
    out.val.alloc(9 * out.nnzb + 1, s);
    allgatherv<int>(x, cpp, cnt, out.col.p);
    std::vector<int64_t> vc(nr);
    for (int q = 0; q < nr; ++q) vc[q] = 9 * cnt[q];
    allgatherv<double>(x, vpp, vc, out.val.p);
}

// ---- the distributed setup ------------------------------------------------------

DSetup dist_setup(const Xport &x, std::vector<Bsr3> &&A_own, std::vector<DevBuf<double>> &&B_own,
                  int64_t b_cols, const std::vector<int64_t> &row_starts, int64_t min_rows,
                  const samg_amg_params &prm, int pipeline, double t_start) {
    NvtxScope nvtx_scope("samg::dsetup (distributed)");
    cudaStream_t s = x.s;
    const int nr = x.nranks;
    const size_t nd = x.mine.size();
    if (nr > 32) fail(SAMG_UNSUPPORTED, "dsetup: at most 32 ranks (rank masks)");
    const bool block = pipeline == SAMG_PIPELINE_BLOCK;
    const bool scalar_galerkin =
        pipeline == SAMG_PIPELINE_NS_HYBRID1 || pipeline == SAMG_PIPELINE_NS_HYBRID2;
    const int k = block ? 0 : static_cast<int>(b_cols);
    DSetup D;
    D.held_rows.assign(nd, 0);
    std::vector<int64_t> fst = row_starts;
    int64_t N = row_starts[nr];
    D.a0_nnzb = 0;
    {
        std::vector<std::vector<int64_t>> v(nd, std::vector<int64_t>(1, 0));
        for (size_t i = 0; i < nd; ++i) v[i][0] = A_own[i].nnzb;
        D.a0_nnzb = allreduce_sum(x, v)[0];
    }
    DevBuf<DevError> err(1, s);
    CK(cudaMemsetAsync(err.p, 0, sizeof(DevError), s));
    static const bool timing = [] {
        const char *e = std::getenv("SAMG_SETUP_TIMING");
        return e && e[0] == '1';
    }();
    double t_mark = t_start;
    auto mark = [&](const char *what, size_t level) {
        char nv[64];
        std::snprintf(nv, sizeof nv, "dsetup L%zu %s done", level, what);
        nvtxMarkA(nv);
        if (!timing) return;
        CK(cudaStreamSynchronize(s));
        const double t = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
        std::fprintf(stderr, "dsetup L%zu %-12s %8.3f ms\n", level, what, 1e3 * (t - t_mark));
        t_mark = t;
    };
    auto driven = [&](size_t i) { return x.mine[i]; };
    bool distributed = 3 * N > prm.coarse_enough;  // the fine level is partitioned unless coarsest
    while (distributed) {
        const size_t lvl = D.lv.size();
        LvGlobal L;
        L.N = N;
        L.fst = fst;
        const int pbs = block ? 3 : (lvl == 0 ? 3 : k);
        if (pbs % 3) fail(SAMG_NOT_DIVISIBLE, "ns_block: node size must be a multiple of 3");
        L.h = pbs / 3;
        if (N % L.h) fail(SAMG_NOT_DIVISIBLE, "strength_graph: rows not divisible by point block size");
        L.nnodes = N / L.h;
        L.nst.resize(nr + 1);
        for (int q = 0; q <= nr; ++q) {
            if (fst[q] % L.h) fail(SAMG_ERROR, "dsetup: partition splits a node");
            L.nst[q] = fst[q] / L.h;
        }
        L.d_nst = to_dev(L.nst, s);
        // 1. one layer of halo rows of A (for the strength test)
        std::vector<Bsr3> Aext(nd);
        {
            std::vector<std::vector<DevBuf<int>>> lists(nd);
            std::vector<const Bsr3 *> M(nd);
            std::vector<int64_t> g0(nd);
            for (size_t i = 0; i < nd; ++i) {
                lists[i].resize(nr);
                M[i] = &A_own[i];
                g0[i] = fst[driven(i)];
                const int *ap = A_own[i].ptr.p, *ac = A_own[i].col.p;
                const int64_t hh = L.h;
                for (int p = 0; p < nr; ++p) {
                    if (p == driven(i)) continue;
                    const int64_t lo = fst[p], hi = fst[p + 1];
                    // whole nodes: the strength weight of a node tile needs
                    // all its block rows (partition bounds are node-aligned)
                    rows_where(A_own[i].nrows, [=] __device__(int64_t r) {
                        const int64_t b0 = (r / hh) * hh;
                        for (int64_t rr = b0; rr < b0 + hh; ++rr)
                            for (int e = ap[rr]; e < ap[rr + 1]; ++e)
                                if (ac[e] >= lo && ac[e] < hi) return true;
                        return false;
                    }, lists[i][p], s);
                }
            }
            std::vector<RowsIn> in = exchange_rows(x, M, g0, lists);
            for (size_t i = 0; i < nd; ++i) {
                assemble(N, N, A_own[i], fst[driven(i)], in[i], Aext[i], s);
                if (lvl == 0) D.held_rows[i] = std::max<int64_t>(D.held_rows[i], A_own[i].nrows + in[i].nr);
            }
        }
        mark("halo_A", lvl);
        // 2. strength graph; 3. own node rows of G gathered on every rank
        {
            std::vector<Graph> Gx(nd);
            std::vector<std::vector<int64_t>> ecnt(nd, std::vector<int64_t>(nr, 0));
            std::vector<DevBuf<int>> glen(nd);
            std::vector<const int *> lenp(nd), colp(nd);
            for (size_t i = 0; i < nd; ++i) {
                strength_graph(Aext[i], static_cast<int>(L.h), prm.eps_strong, Gx[i], s, block);
                const int64_t a = L.nst[driven(i)], b = L.nst[driven(i) + 1];
                int e0 = 0, e1 = 0;
                CK(cudaMemcpyAsync(&e0, Gx[i].ptr.p + a, sizeof(int), cudaMemcpyDeviceToHost, s));
                CK(cudaMemcpyAsync(&e1, Gx[i].ptr.p + b, sizeof(int), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                ecnt[i][driven(i)] = e1 - e0;
                glen[i].alloc(b - a + 1, s);
                int *gl = glen[i].p;
                const int *gp = Gx[i].ptr.p + a;
                each(b - a, [=] __device__(int64_t t) { gl[t] = gp[t + 1] - gp[t]; }, s);
                lenp[i] = glen[i].p;
                colp[i] = Gx[i].col.p + e0;
            }
            const std::vector<int64_t> ec = allreduce_sum(x, ecnt);
            std::vector<int64_t> nc(nr);
            for (int q = 0; q < nr; ++q) nc[q] = L.nst[q + 1] - L.nst[q];
            DevBuf<int> len(L.nnodes + 1, s);
            allgatherv<int>(x, lenp, nc, len.p);
            L.G.nnodes = L.nnodes;
            L.G.ptr.alloc(L.nnodes + 1, s);
            L.G.nedges = exscan(len.p, L.G.ptr.p, L.nnodes, s);
            L.G.col.alloc(L.G.nedges + 1, s);
            allgatherv<int>(x, colp, ec, L.G.col.p);
        }
        mark("strength", lvl);
        // 4. aggregation on the global graph (identical on every rank)
        L.naggs = aggregate(L.G, L.agg, s, &L.seedno);
        L.ast.resize(nr + 1);
        for (int q = 0; q < nr; ++q) L.ast[q] = read_int(L.seedno.p + L.nst[q], s);
        L.ast[nr] = L.naggs;
        L.d_ast = to_dev(L.ast, s);
        L.kb = block ? 1 : k / 3;
        mark("aggregate", lvl);
        // stagnation guard (hierarchy.hpp:355): P would have naggs*kb block columns
        if (static_cast<double>(3 * L.naggs * L.kb) > prm.stagnation_ratio * static_cast<double>(3 * N))
            break;
        std::vector<int64_t> cst(nr + 1);
        for (int q = 0; q <= nr; ++q) cst[q] = L.kb * L.ast[q];
        const int64_t Nc = L.naggs * L.kb;
        const int *agg = L.agg.p;
        const int64_t *dast = L.d_ast.p, *dnst = L.d_nst.p;
        const int h = static_cast<int>(L.h);
        // m1[node] = ranks owning an aggregate the node's row of P touches
        // (agg(node) and agg of its strong neighbours, k_psm_touch)
        DevBuf<unsigned> m1(L.nnodes + 1, s);
        {
            unsigned *m = m1.p;
            const int *gp = L.G.ptr.p, *gc = L.G.col.p;
            each(L.nnodes, [=] __device__(int64_t i) {
                unsigned b = 1u << owner_of(agg[i], dast, nr);
                for (int e = gp[i]; e < gp[i + 1]; ++e) b |= 1u << owner_of(agg[gc[e]], dast, nr);
                m[i] = b;
            }, s);
        }
        // 5. transfer operator rows
        std::vector<Bsr3> P_own(nd);
        std::vector<DevBuf<double>> Bc_own(nd);
        if (block) {
            for (size_t i = 0; i < nd; ++i)
                block_transfer(Aext[i], L.G, L.agg, L.naggs, prm.omega, P_own[i], err.p, s,
                               fst[driven(i)], fst[driven(i) + 1]);
        } else {
            const int64_t nfine = 3 * N;  // scalar rows
            // (a) nullspace rows of the nodes of own aggregates
            std::vector<DevBuf<double>> Bx(nd);
            std::vector<std::vector<DevBuf<int>>> sl(nd), rl(nd);
            for (size_t i = 0; i < nd; ++i) {
                const int q = driven(i);
                Bx[i].alloc(nfine * k + 1, s);
                // own rows: local column-major (3 nloc x k) -> global column-major
                const int64_t nl3 = 3 * (fst[q + 1] - fst[q]), o3 = 3 * fst[q];
                const double *bo = B_own[i].p;
                double *bx = Bx[i].p;
                const int kk = k;
                each(nl3 * kk, [=] __device__(int64_t e) {
                    const int64_t c = e / nl3, r = e - c * nl3;
                    bx[c * nfine + o3 + r] = bo[e];
                }, s);
                sl[i].resize(nr);
                rl[i].resize(nr);
                for (int p = 0; p < nr; ++p) {
                    if (p == q) continue;
                    // send: my nodes in p's aggregates; receive: p's nodes in mine
                    const int64_t a = L.nst[q], b = L.nst[q + 1];
                    DevBuf<int> tmp;
                    rows_where(b - a, [=] __device__(int64_t t) {
                        return owner_of(agg[a + t], dast, nr) == p;
                    }, tmp, s);
                    sl[i][p].alloc(tmp.n + 1, s);
                    sl[i][p].n = tmp.n;
                    int *o = sl[i][p].p;
                    const int *tp = tmp.p;
                    each(tmp.n, [=] __device__(int64_t t) { o[t] = static_cast<int>(a + tp[t]); }, s);
                    const int64_t a2 = L.nst[p], b2 = L.nst[p + 1];
                    DevBuf<int> tmp2;
                    rows_where(b2 - a2, [=] __device__(int64_t t) {
                        return owner_of(agg[a2 + t], dast, nr) == q;
                    }, tmp2, s);
                    rl[i][p].alloc(tmp2.n + 1, s);
                    rl[i][p].n = tmp2.n;
                    int *o2 = rl[i][p].p;
                    const int *tp2 = tmp2.p;
                    each(tmp2.n, [=] __device__(int64_t t) { o2[t] = static_cast<int>(a2 + tp2[t]); }, s);
                    CK(cudaStreamSynchronize(s));
                }
            }
            {
                std::vector<PackB> pk(nd);
                std::vector<StoreB> st(nd);
                for (size_t i = 0; i < nd; ++i) {
                    const int q = driven(i);
                    pk[i] = PackB{B_own[i].p, 3 * (fst[q + 1] - fst[q]), 3 * fst[q], pbs, k};
                    st[i] = StoreB{Bx[i].p, nfine, pbs, k};
                }
                exchange_nodes(x, sl, rl, pbs * k, pk, st);
            }
            mark("halo_B", lvl);
            // (b) thin QR of the own aggregates
            std::vector<DevBuf<double>> Pt(nd);
            for (size_t i = 0; i < nd; ++i) {
                const int q = driven(i);
                DevBuf<double> Bc;
                tentative(L.agg, L.nnodes, L.naggs, pbs, Bx[i].p, k, Pt[i], Bc, err.p, s, L.ast[q],
                          L.ast[q + 1]);
                // own coarse nullspace rows [ast*k, ..) of the global column-major Bc
                const int64_t bcn = L.naggs * k, r0 = L.ast[q] * k, nl = (L.ast[q + 1] - L.ast[q]) * k;
                Bc_own[i].alloc(nl * k + 1, s);
                double *d = Bc_own[i].p;
                const double *src = Bc.p;
                each(nl * k, [=] __device__(int64_t e) {
                    const int64_t c = e / nl, r = e - c * nl;
                    d[e] = src[c * bcn + r0 + r];
                }, s);
                CK(cudaStreamSynchronize(s));
                Bx[i].release();
            }
            mark("tentative", lvl);
            // (c) P_tent rows of my nodes and their strong neighbours from the
            //     owners of their aggregates.  nbm[j] = ranks whose node
            //     range contains j or one of j's strong neighbours
            DevBuf<unsigned> nbm(L.nnodes + 1, s);
            {
                unsigned *m = nbm.p;
                const int *gp = L.G.ptr.p, *gc = L.G.col.p;
                each(L.nnodes, [=] __device__(int64_t j) {
                    unsigned b = 1u << owner_of(j, dnst, nr);
                    for (int e = gp[j]; e < gp[j + 1]; ++e) b |= 1u << owner_of(gc[e], dnst, nr);
                    m[j] = b;
                }, s);
            }
            for (size_t i = 0; i < nd; ++i) {
                const int q = driven(i);
                const unsigned *m = nbm.p;
                for (int p = 0; p < nr; ++p) {
                    sl[i][p] = DevBuf<int>();
                    rl[i][p] = DevBuf<int>();
                    if (p == q) continue;
                    // send: nodes of my aggregates that p reads; receive: nodes
                    // of p's aggregates that I read
                    rows_where(L.nnodes, [=] __device__(int64_t j) {
                        return owner_of(agg[j], dast, nr) == q && ((m[j] >> p) & 1u);
                    }, sl[i][p], s);
                    rows_where(L.nnodes, [=] __device__(int64_t j) {
                        return owner_of(agg[j], dast, nr) == p && ((m[j] >> q) & 1u);
                    }, rl[i][p], s);
                }
            }
            {
                const int W = pbs * k;
                std::vector<PackP> pk(nd);
                std::vector<StoreP> st(nd);
                for (size_t i = 0; i < nd; ++i) {
                    pk[i] = PackP{Pt[i].p, W};
                    st[i] = StoreP{Pt[i].p, W};
                }
                exchange_nodes(x, sl, rl, W, pk, st);
            }
            mark("halo_Pt", lvl);
            // (d) smoothed rows of P (global aggregate columns)
            for (size_t i = 0; i < nd; ++i) {
                const int q = driven(i);
                smooth_prolongation(Aext[i], L.G, L.agg, L.naggs, pbs, k, Pt[i].p, prm.omega, P_own[i],
                                    err.p, s, L.nst[q], L.nst[q + 1]);
                Pt[i].release();
            }
        }
        check_dev_error(err.p, s);
        mark("smooth_P", lvl);
        // 6. rows of A and P the Galerkin rows of each rank read: S1 = fine
        //    rows in its rows of R, S2 = S1 + their A-neighbours
        std::vector<Bsr3> A2(nd), Px(nd);
        {
            std::vector<std::vector<DevBuf<int>>> lists(nd);
            std::vector<const Bsr3 *> MA(nd), MP(nd);
            std::vector<int64_t> g0(nd);
            for (size_t i = 0; i < nd; ++i) {
                const int q = driven(i);
                lists[i].resize(nr);
                MA[i] = &A_own[i];
                MP[i] = &P_own[i];
                g0[i] = fst[q];
                DevBuf<unsigned> rm(A_own[i].nrows + 1, s);
                unsigned *rmp = rm.p;
                const unsigned *m = m1.p;
                const int *ap = A_own[i].ptr.p, *ac = A_own[i].col.p;
                const int64_t f0 = fst[q];
                each(A_own[i].nrows, [=] __device__(int64_t r) {
                    unsigned b = m[(f0 + r) / h];
                    for (int e = ap[r]; e < ap[r + 1]; ++e) b |= m[ac[e] / h];
                    rmp[r] = b;
                }, s);
                for (int p = 0; p < nr; ++p) {
                    if (p == q) continue;
                    rows_where(A_own[i].nrows, [=] __device__(int64_t r) { return ((rmp[r] >> p) & 1u) != 0; },
                               lists[i][p], s);
                }
                CK(cudaStreamSynchronize(s));
            }
            std::vector<RowsIn> inA = exchange_rows(x, MA, g0, lists);
            std::vector<RowsIn> inP = exchange_rows(x, MP, g0, lists);
            for (size_t i = 0; i < nd; ++i) {
                const int q = driven(i);
                Aext[i] = Bsr3();
                assemble(N, N, A_own[i], fst[q], inA[i], A2[i], s);
                assemble(N, Nc, P_own[i], fst[q], inP[i], Px[i], s);
                if (lvl == 0) D.held_rows[i] = std::max<int64_t>(D.held_rows[i], A_own[i].nrows + inA[i].nr);
            }
        }
        mark("halo_S2", lvl);
        // 7. R = P^T (own coarse rows complete: every fine row of theirs is held)
        // 8. own coarse rows of the Galerkin product
        std::vector<DPiece> pieces(nd);
        std::vector<Bsr3> Ac_own(nd);
        for (size_t i = 0; i < nd; ++i) {
            const int q = driven(i);
            Bsr3 Rx;
            transpose(Px[i], Rx, s);
            slice_rows(Rx, cst[q], cst[q + 1], pieces[i].R, s);
            galerkin_rows(pieces[i].R, A2[i], Px[i], Rx, Ac_own[i], s, scalar_galerkin, true);
            fix_decoupled_rows(Ac_own[i], s, cst[q]);
            CK(cudaStreamSynchronize(s));
            A2[i] = Bsr3();
            Px[i] = Bsr3();
        }
        mark("galerkin", lvl);
        // 9. smoother of the own rows
        for (size_t i = 0; i < nd; ++i)
            setup_smoother(A_own[i], prm.smoother, prm.smoother_omega, pieces[i].M, err.p, s,
                           fst[driven(i)]);
        check_dev_error(err.p, s);
        for (size_t i = 0; i < nd; ++i) {
            pieces[i].A = std::move(A_own[i]);
            pieces[i].P = std::move(P_own[i]);
            A_own[i] = std::move(Ac_own[i]);
            if (!block) B_own[i] = std::move(Bc_own[i]);
        }
        D.starts.push_back(fst);
        D.nrows.push_back(N);
        D.lv.push_back(std::move(pieces));
        fst = cst;
        N = Nc;
        distributed = 3 * N > prm.coarse_enough && N >= min_rows * nr;
        for (int q = 0; q < nr && distributed; ++q) distributed = fst[q + 1] > fst[q];
        mark("smoother", lvl);
    }
    if (D.lv.empty())
        fail(SAMG_UNSUPPORTED, "multi-GPU solve needs at least two levels (the fine level is the coarsest)");
    // level Ld gathered on every rank; the rest of the setup is redundant
    const size_t Ld = D.lv.size();
    D.starts.push_back(fst);
    D.nrows.push_back(N);
    Bsr3 A_Ld;
    {
        std::vector<const Bsr3 *> own(nd);
        for (size_t i = 0; i < nd; ++i) own[i] = &A_own[i];
        gather_matrix(x, own, fst, N, A_Ld);
    }
    DevBuf<double> B_Ld;
    if (!block) {
        // own rows (column-major 3 nloc x k) -> row-major, gathered, -> column-major
        std::vector<DevBuf<double>> rm(nd);
        std::vector<const double *> pp(nd);
        for (size_t i = 0; i < nd; ++i) {
            const int q = driven(i);
            const int64_t nl3 = 3 * (fst[q + 1] - fst[q]);
            rm[i].alloc(nl3 * k + 1, s);
            double *d = rm[i].p;
            const double *b = B_own[i].p;
            const int kk = k;
            each(nl3 * kk, [=] __device__(int64_t e) {
                const int64_t c = e / nl3, r = e - c * nl3;
                d[r * kk + c] = b[e];
            }, s);
            pp[i] = rm[i].p;
        }
        std::vector<int64_t> cnt(nr);
        for (int q = 0; q < nr; ++q) cnt[q] = 3 * (fst[q + 1] - fst[q]) * k;
        DevBuf<double> g(3 * N * k + 1, s);
        allgatherv<double>(x, pp, cnt, g.p);
        B_Ld.alloc(3 * N * k + 1, s);
        double *d = B_Ld.p;
        const double *gp = g.p;
        const int64_t n3 = 3 * N;
        const int kk = k;
        each(n3 * kk, [=] __device__(int64_t e) {
            const int64_t c = e / n3, r = e - c * n3;
            d[e] = gp[r * kk + c];
        }, s);
        CK(cudaStreamSynchronize(s));
    }
    for (auto &a : A_own) a = Bsr3();
    D.coarse.reset(setup_hierarchy(std::move(A_Ld), block ? nullptr : B_Ld.p, 3 * N, k, prm, s, t_start,
                                   pipeline, nullptr, static_cast<int>(Ld)));
    D.coarse->owns_stream = false;
    // footprint: the global matrices of the distributed levels + the rest
    {
        std::vector<std::vector<int64_t>> v(nd, std::vector<int64_t>(4 * Ld, 0));
        for (size_t i = 0; i < nd; ++i)
            for (size_t l = 0; l < Ld; ++l) {
                const DPiece &pc = D.lv[l][i];
                v[i][4 * l] = pc.A.nnzb;
                v[i][4 * l + 1] = pc.P.nnzb;
                v[i][4 * l + 2] = pc.R.nnzb;
                v[i][4 * l + 3] = static_cast<int64_t>(pc.M.data.n);
            }
        const std::vector<int64_t> g = allreduce_sum(x, v);
        uint64_t bytes = 0;
        for (size_t l = 0; l < Ld; ++l) {
            const int64_t n = D.nrows[l], nc = D.nrows[l + 1];
            bytes += static_cast<uint64_t>(n + 1) * 8 + static_cast<uint64_t>(g[4 * l]) * 80;
            bytes += static_cast<uint64_t>(n + 1) * 8 + static_cast<uint64_t>(g[4 * l + 1]) * 80;
            bytes += static_cast<uint64_t>(nc + 1) * 8 + static_cast<uint64_t>(g[4 * l + 2]) * 80;
            bytes += static_cast<uint64_t>(g[4 * l + 3]) * 8;
        }
        D.footprint = bytes + D.coarse->memory_footprint();
    }
    mark("coarse", Ld);
    return D;
}

} // namespace samgb
