// dsetup.cuh -- the distributed (row-partitioned) ns_block / block setup:
// every rank builds only its rows of each large level (dsetup.cu), the
// small coarse levels are replicated (dsolve.cu drives the solve).
#pragma once

#include <memory>
#include <vector>

#include "hierarchy.cuh"
#include "nccl_shim.cuh"

namespace samgb {

// The ranks this process drives and how they talk: one rank with NCCL, or
// all of them emulated in lock step (comm == nullptr: every exchange is a
// device copy with exactly the offsets and counts of the NCCL calls).
struct Xport {
    ncclComm_t comm = nullptr;
    int nranks = 1;
    std::vector<int> mine;  // driven ranks, ascending
    cudaStream_t s = nullptr;
    bool emu() const { return comm == nullptr; }
};

// Exchange of byte segments: driven rank i sends src[i] + soff[i][p] ..
// soff[i][p+1] to peer p and receives into dst[i] + roff[i][p] .. roff[i][p+1]
// (offsets in bytes, size nranks + 1, the own segment empty).
void xchg_bytes(const Xport &x, const std::vector<const char *> &src,
                const std::vector<std::vector<int64_t>> &soff, const std::vector<char *> &dst,
                const std::vector<std::vector<int64_t>> &roff);
// All-to-all of W int64 per (sender, receiver): send[i][p*W + w] is what
// driven rank i sends to p; returns recv[i][p*W + w] = what p sends to it.
std::vector<std::vector<int64_t>> alltoall_counts(const Xport &x,
                                                  const std::vector<std::vector<int64_t>> &send,
                                                  int W);
// Sum over all ranks of per-driven-rank values (host in / host out).
std::vector<int64_t> allreduce_sum(const Xport &x, const std::vector<std::vector<int64_t>> &v);

// One rank's rows of a distributed level (global column ids throughout).
struct DPiece {
    Bsr3 A;   // block rows [f0, f1) of A_l
    Bsr3 P;   // block rows [f0, f1) of P_l (coarse columns)
    Bsr3 R;   // coarse block rows [c0, c1) of R_l = P_l^T (fine columns)
    Smoother M;
};

struct DSetup {
    // starts[l]: block-row partition of level l (l = 0 .. Ld; the coarse
    // partition of l+1 follows the seeds of l's aggregation)
    std::vector<std::vector<int64_t>> starts;
    std::vector<int64_t> nrows;            // global block rows, levels 0 .. Ld
    std::vector<std::vector<DPiece>> lv;   // lv[l][i]: driven rank i's rows of level l < Ld
    std::vector<int64_t> held_rows;        // per driven rank: max A rows held in any level-0 step
    std::unique_ptr<Hierarchy> coarse;     // levels Ld .. (gathered, replicated)
    uint64_t footprint = 0;                // memory_footprint (hierarchy.hpp:443-458), global
    int64_t a0_nnzb = 0;
    size_t Ld() const { return lv.size(); }
};

// Distributed setup from each driven rank's own fine rows (global column
// ids) and own nullspace rows (3*nloc x b_cols, column-major; unused for the
// block pipeline).  row_starts: the fine partition.  Levels are distributed
// while they have >= min_rows * nranks block rows (and every rank owns one);
// the first level below is gathered and the rest set up redundantly.
DSetup dist_setup(const Xport &x, std::vector<Bsr3> &&A_own, std::vector<DevBuf<double>> &&B_own,
                  int64_t b_cols, const std::vector<int64_t> &row_starts, int64_t min_rows,
                  const samg_amg_params &prm, int pipeline, double t_start);

// rows of every rank assembled into the global matrix (parity taps)
void gather_matrix(const Xport &x, const std::vector<const Bsr3 *> &own,
                   const std::vector<int64_t> &row_starts, int64_t ncols, Bsr3 &out);

} // namespace samgb
