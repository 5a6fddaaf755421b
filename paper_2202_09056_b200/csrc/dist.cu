// dist.cu -- row-partitioned BSR3 operator for multi-GPU runs.
//
// One process per GPU.  Rank r owns the contiguous block rows
// [row_starts[r], row_starts[r+1]) of a global matrix.  Its local matrix keeps
// the rows' block order (so y is bit-identical to the single-GPU SpMV) with
// columns renumbered: owned columns -> [0, nloc), remote columns -> nloc + g
// where g indexes the sorted ghost list (ghosts are therefore grouped by
// owner rank, one contiguous segment per peer).  The halo plan:
//   recv side: per peer, the segment of the ghost array it fills;
//   send side: per peer, the owned block rows it needs (set from the peers'
//              ghost lists, exchanged by the caller's transport).
// The transport (NCCL via torch.distributed in bench.py, gloo in the CPU
// tests) is the caller's; this file provides the plan (host, testable
// without a GPU) and the device pieces: pack, and the SpMV split into
// interior rows (no ghost column; run while the halo is in flight) and
// boundary rows.
#include <algorithm>
#include <memory>
#include <vector>

#include "dist.cuh"


namespace samgb {

void launch_spmv_rows(const Bsr3 &A, const int *rows, int64_t nrows, int group, double alpha,
                      const double *x, double beta, double *y, cudaStream_t s);

namespace {

__global__ void k_pack(int64_t n, const int *idx, const double *x, double *buf) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < 3 * n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k = e / 3;
        buf[e] = x[3 * static_cast<int64_t>(idx[k]) + (e - 3 * k)];
    }
}

int owner_of(const std::vector<int64_t> &starts, int64_t g) {
    return static_cast<int>(std::upper_bound(starts.begin(), starts.end(), g) - starts.begin()) - 1;
}

} // namespace

samg_dist *dist_create(int64_t row0, int64_t row1, const int64_t *ptr, const int64_t *col,
                       const double *val, int nranks, const int64_t *row_starts, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(SAMG_INVALID_ARGUMENT, "dist: bad rank");
    if (row_starts[rank] != row0 || row_starts[rank + 1] != row1)
        fail(SAMG_INVALID_ARGUMENT, "dist: row range does not match row_starts[rank]");
    for (int q = 0; q < nranks; ++q)
        if (row_starts[q + 1] < row_starts[q]) fail(SAMG_INVALID_ARGUMENT, "dist: row_starts must be nondecreasing");
    auto d = std::make_unique<samg_dist>();
    d->rank = rank;
    d->nranks = nranks;
    d->row0 = row0;
    d->row1 = row1;
    d->nloc = row1 - row0;
    d->row_starts.assign(row_starts, row_starts + nranks + 1);
    const int64_t nl = d->nloc;
    const int64_t base = ptr[0];
    const int64_t nnz = ptr[nl] - base;
    d->ptr.resize(nl + 1);
    for (int64_t i = 0; i <= nl; ++i) d->ptr[i] = ptr[i] - base;
    const int64_t gmax = row_starts[nranks];
    std::vector<int64_t> g;
    for (int64_t j = 0; j < nnz; ++j) {
        const int64_t c = col[base + j];
        if (c < 0 || c >= gmax) fail(SAMG_INVALID_ARGUMENT, "dist: column out of range");
        if (c < row0 || c >= row1) g.push_back(c);
    }
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    d->ghost = g;
    d->nghost = static_cast<int64_t>(g.size());
    d->col.resize(nnz);
    for (int64_t i = 0; i < nl; ++i) {
        bool bnd = false;
        for (int64_t j = d->ptr[i]; j < d->ptr[i + 1]; ++j) {
            const int64_t c = col[base + j];
            if (c >= row0 && c < row1) {
                d->col[j] = c - row0;
            } else {
                d->col[j] = nl + (std::lower_bound(g.begin(), g.end(), c) - g.begin());
                bnd = true;
            }
        }
        (bnd ? d->boundary : d->interior).push_back(static_cast<int>(i));
    }
    d->val.assign(val + 9 * base, val + 9 * (base + nnz));
    // the longest run of interior rows (slab partitions: all but the first
    // and last node layers): one contiguous row view, so it streams through
    // the TMA-fed SpMV like a whole matrix
    {
        std::vector<unsigned char> isb(nl, 0);
        for (int b : d->boundary) isb[b] = 1;
        int64_t best = 0, run = 0;
        for (int64_t i = 0; i < nl; ++i) {
            run = isb[i] ? 0 : run + 1;
            if (run > best) { best = run; d->ib = i + 1; d->ia = i + 1 - run; }
        }
    }
    // recv plan: ghosts grouped by owner (sorted ids + contiguous ranges)
    int64_t k = 0;
    while (k < d->nghost) {
        const int q = owner_of(d->row_starts, g[k]);
        if (q == rank) fail(SAMG_ERROR, "dist: ghost owned by self");
        int64_t e = k;
        while (e < d->nghost && g[e] < row_starts[q + 1]) ++e;
        d->recv_peers.push_back(q);
        d->recv_counts.push_back(e - k);
        d->recv_offsets.push_back(k);
        k = e;
    }
    return d.release();
}

void dist_set_send(samg_dist *d, int npeers, const int *peers, const int64_t *counts,
                   const int64_t *ids) {
    d->send_peers.assign(peers, peers + npeers);
    d->send_counts.assign(counts, counts + npeers);
    d->send_offsets.assign(npeers, 0);
    d->send_idx.clear();
    int64_t off = 0;
    for (int p = 0; p < npeers; ++p) {
        if (peers[p] < 0 || peers[p] >= d->nranks || peers[p] == d->rank)
            fail(SAMG_INVALID_ARGUMENT, "dist: bad send peer");
        d->send_offsets[p] = off;
        for (int64_t k = 0; k < counts[p]; ++k) {
            const int64_t gid = ids[off + k];
            if (gid < d->row0 || gid >= d->row1)
                fail(SAMG_INVALID_ARGUMENT, "dist: requested row is not owned by this rank");
            d->send_idx.push_back(gid - d->row0);
        }
        off += counts[p];
    }
    d->send_set = true;
}

// Peer q reads our row i iff row i of q holds column i, i.e. (structural
// symmetry) iff our row i holds a column in q's range: the owner derives
// the plan from its own rows, ascending global ids per peer -- the order of
// the receiver's sorted ghost segment.
void dist_derive_send(samg_dist *d) {
    std::vector<int> peers;
    std::vector<int64_t> counts, ids;
    const int64_t nl = d->nloc;
    // columns are renumbered: ghosts nl + g -> global d->ghost[g]
    for (int q = 0; q < d->nranks; ++q) {
        if (q == d->rank) continue;
        const int64_t lo = d->row_starts[q], hi = d->row_starts[q + 1];
        int64_t c = 0;
        for (int64_t i = 0; i < nl; ++i) {
            bool hit = false;
            for (int64_t j = d->ptr[i]; j < d->ptr[i + 1] && !hit; ++j) {
                const int64_t lc = d->col[j];
                if (lc < nl) continue;
                const int64_t g = d->ghost[lc - nl];
                hit = g >= lo && g < hi;
            }
            if (hit) { ids.push_back(d->row0 + i); ++c; }
        }
        if (c) { peers.push_back(q); counts.push_back(c); }
    }
    dist_set_send(d, static_cast<int>(peers.size()), peers.data(), counts.data(), ids.data());
}

void dist_to_device(samg_dist *d, int device, int group) {
    CK(cudaSetDevice(device));
    d->device = device;
    const int64_t nl = d->nloc, nnz = d->ptr[nl];
    Bsr3 &A = d->A;
    A.alloc(nl, nl + d->nghost, nnz, nullptr);
    std::vector<int> p32(nl + 1), c32(nnz);
    for (int64_t i = 0; i <= nl; ++i) p32[i] = static_cast<int>(d->ptr[i]);
    for (int64_t j = 0; j < nnz; ++j) c32[j] = static_cast<int>(d->col[j]);
    CK(cudaMemcpy(A.ptr.p, p32.data(), sizeof(int) * (nl + 1), cudaMemcpyHostToDevice));
    if (nnz) {
        CK(cudaMemcpy(A.col.p, c32.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(A.val.p, d->val.data(), sizeof(double) * 9 * nnz, cudaMemcpyHostToDevice));
    }
    auto up = [](DevBuf<int> &b, const std::vector<int> &v) {
        b.alloc(v.size(), nullptr);
        if (!v.empty()) CK(cudaMemcpy(b.p, v.data(), sizeof(int) * v.size(), cudaMemcpyHostToDevice));
    };
    up(d->d_interior, d->interior);
    up(d->d_boundary, d->boundary);
    std::vector<int> si(d->send_idx.begin(), d->send_idx.end());
    up(d->d_send_idx, si);
    d->group = group;
    CK(cudaDeviceSynchronize());
}

void dist_pack(const samg_dist *d, const double *x, double *buf, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(d->send_idx.size());
    if (n == 0) return;
    int64_t g = (3 * n + 255) / 256;
    if (g > 4096) g = 4096;
    k_pack<<<static_cast<int>(g), 256, 0, s>>>(n, d->d_send_idx.p, x, buf);
    CK_LAUNCH();
}

// part 0: the interior run [ia, ib) (reads no ghost: runs while the halo is
// in flight); part 1: the other rows [0, ia) and [ib, nloc).  Row views of
// the local matrix: the same per-row arithmetic as one launch over all rows.
void dist_spmv(const samg_dist *d, int part, double alpha, const double *xext, double beta,
               double *y, cudaStream_t s) {
    auto run = [&](int64_t a, int64_t b) {
        if (b <= a) return;
        RowView v(d->A, a, b);
        launch_spmv(v.m, alpha, xext, beta, y + 3 * a, s);
    };
    if (part == 0) {
        run(d->ia, d->ib);
    } else {
        run(0, d->ia);
        run(d->ib, d->nloc);
    }
}

} // namespace samgb
