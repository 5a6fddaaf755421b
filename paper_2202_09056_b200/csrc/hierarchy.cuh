// hierarchy.cuh -- the device-resident AMG hierarchy (hierarchy.hpp:78-148)
// and its setup / V-cycle / CG drivers.
#pragma once

#include <vector>

#include "kernels.cuh"

namespace samgb {

struct Level {
    Bsr3 A, P, R;              // P, R empty on the coarsest level
    bool has_transfer = false;
    Smoother M;                // absent on the coarsest level
    DevBuf<int> agg;           // aggregate id per node (parity tap)
    DevBuf<int> seedno;        // #pass-1 seeds before each node (nnodes+1):
                               // aggregate ids are assigned in seed order
    int64_t nnodes = 0, naggs = 0;
    DevBuf<double> f, u, r, t; // V-cycle workspace (vcycle_workspace, hierarchy.hpp:152-163)
};

struct Hierarchy {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool owns_stream = false;  // set once setup succeeded
    samg_amg_params prm{};
    int pipeline = SAMG_PIPELINE_NS_BLOCK;
    std::vector<Level> levels;
    DevBuf<double> Ainv;       // coarsest inverse, row-major nc x nc
    int64_t nc = 0;
    bool coarse_lu = false;    // coarse solve by the reference's LU (coarse_lu.cu)
    CoarseLu lu;
    void coarse_solve(const double *f, double *u);
    double setup_seconds = 0;
    DevBuf<DevError> err;
    // CG workspace (cg.hpp:46-47)
    DevBuf<double> r, z, p, q, fbuf, ubuf, partials;
    DevBuf<CgScalars> sc;
    CgScalars *sc_host = nullptr;  // pinned mirror
    CgScalars *sc_stage = nullptr; // pinned staging for loop parameters
    cudaGraphExec_t cg_exec = nullptr;  // device-resident CG loop (while node)
    void build_cg_graph();
    // V-cycle tail (solve.cu k_vtail): the levels >= tail_start, the coarse
    // solve and the prolongation into level tail_start - 1 in one
    // cooperative launch (tail_nph == 0: not used)
    DevBuf<VPhase> tail_ph;
    DevBuf<unsigned> tail_bar;
    int tail_nph = 0, tail_grid = 0;
    size_t tail_start = 0, tail_smem = 0;
    DevBuf<unsigned long long> tail_trace;  // SAMG_VTAIL_TRACE=1: per-phase timestamps
    void build_tail();

    ~Hierarchy();
    int64_t finest_dim() const { return 3 * levels.front().A.nrows; }
    uint64_t memory_footprint() const;

    bool vcycle(const double *f, double *u, bool zero_guess, bool fuse_rz = false);
    // presmoothed: the first sweep of level `start` from a zero guess is
    // already in levels[start].u (fused into the kernel that produced f)
    bool vcycle_from(size_t start, const double *f, double *u, bool zero_guess,
                     bool fuse_rz = false, bool presmoothed = false);
    samg_solve_report cg(const double *d_f, double *d_u, const samg_cg_params &prm);
};

// Hook for the multi-GPU setup (dsolve.cu): forms A_c = R A P of level `lvl`
// row-sliced across ranks and returns true, or returns false to let the
// setup form the plain product.  seedno = the aggregation's seed numbering.
struct GalerkinSlicer {
    virtual ~GalerkinSlicer() = default;
    virtual bool galerkin(size_t lvl, const Bsr3 &A, const int *seedno, int64_t nnodes,
                          int64_t naggs, const Bsr3 &R, const Bsr3 &P, Bsr3 &Ac, bool scalar_order,
                          cudaStream_t s) = 0;
};

// Setup from a device BSR3 fine matrix (consumed) and a host nullspace.
// pipeline: ns_block, or ns_hybrid1/2 (Galerkin in scalar order)
// first_level: the global index of A0's level (the multi-GPU setup hands in
// a gathered coarse level: its nodes are k-row tiles, not 3-row ones)
Hierarchy *setup_hierarchy(Bsr3 &&A0, const double *B_host, int64_t b_rows, int64_t b_cols,
                           const samg_amg_params &prm, cudaStream_t stream, double t_start,
                           int pipeline = SAMG_PIPELINE_NS_BLOCK, GalerkinSlicer *slicer = nullptr,
                           int first_level = 0);

} // namespace samgb
