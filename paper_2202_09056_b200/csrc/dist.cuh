// dist.cuh -- a rank's partition of a row-partitioned BSR3 matrix and its
// halo plan (samg_dist of the C-ABI); see dist.cu.
#pragma once

#include <vector>

#include "kernels.cuh"

struct samg_dist {
    int rank = 0, nranks = 1, device = -1, group = 0;
    int64_t row0 = 0, row1 = 0, nloc = 0, nghost = 0;
    std::vector<int64_t> row_starts;
    std::vector<int64_t> ptr, col;   // local matrix, renumbered columns
    std::vector<double> val;
    std::vector<int64_t> ghost;      // global ids, sorted (grouped by owner)
    std::vector<int> recv_peers, send_peers;
    std::vector<int64_t> recv_counts, recv_offsets, send_counts, send_offsets;
    std::vector<int64_t> send_idx;   // local block rows, per send peer in order
    std::vector<int> interior, boundary;
    int64_t ia = 0, ib = 0;          // longest run of interior rows (multiplied
                                     // by one contiguous launch while the halo flies)
    bool send_set = false;
    samgb::Bsr3 A;
    samgb::DevBuf<int> d_interior, d_boundary, d_send_idx;
};

namespace samgb {
samg_dist *dist_create(int64_t row0, int64_t row1, const int64_t *ptr, const int64_t *col,
                       const double *val, int nranks, const int64_t *row_starts, int rank);
void dist_set_send(samg_dist *d, int npeers, const int *peers, const int64_t *counts,
                   const int64_t *ids);
// the send plan from the rank's own rows (structurally symmetric matrix)
void dist_derive_send(samg_dist *d);
void dist_to_device(samg_dist *d, int device, int group);
void dist_pack(const samg_dist *d, const double *x, double *buf, cudaStream_t s);
void dist_spmv(const samg_dist *d, int part, double alpha, const double *xext, double beta,
               double *y, cudaStream_t s);
} // namespace samgb
