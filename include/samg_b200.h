/*
 * samg_b200.h -- C-ABI of the B200-native SA-AMG "NS Block" solver.
 *
 * This is the drop-in boundary for the reference's ns_block hot path
 * (/root/reference/proj/include/samg).  The reference has no FFI of its own;
 * each entry point below names the reference interface it replaces.  Plain
 * pointers and sizes only; every call returns an int status whose values
 * map 1:1 onto the reference's exception classes (common.hpp:12-28), plus
 * CUDA failures.  Calls on one handle are not thread-safe (the reference's
 * hierarchy is likewise single-threaded); distinct handles are independent.
 *
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns SAMG_NO_DEVICE.
 */
#ifndef SAMG_B200_H
#define SAMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SAMG_API __attribute__((visibility("default")))
#else
#define SAMG_API
#endif

/* Status codes; 1..14 mirror samg::error subclasses (common.hpp:12-28). */
enum samg_status {
    SAMG_OK = 0,
    SAMG_ERROR = 1,                /* samg::error                        */
    SAMG_DIMENSION_MISMATCH = 2,   /* samg::dimension_mismatch           */
    SAMG_NOT_DIVISIBLE = 3,        /* samg::not_divisible                */
    SAMG_SINGULAR_BLOCK = 4,       /* samg::singular_block               */
    SAMG_MISSING_DIAGONAL = 5,     /* samg::missing_diagonal             */
    SAMG_ZERO_DIAGONAL = 6,        /* samg::zero_diagonal                */
    SAMG_NON_SQUARE = 7,           /* samg::non_square                   */
    SAMG_BAD_NULLSPACE_SHAPE = 8,  /* samg::bad_nullspace_shape          */
    SAMG_BREAKDOWN_NON_SPD = 9,    /* samg::breakdown_non_spd            */
    SAMG_INVALID_MATERIAL = 10,    /* samg::invalid_material             */
    SAMG_SHAPE_MISMATCH = 11,      /* samg::shape_mismatch               */
    SAMG_CUDA_ERROR = 100,
    SAMG_NCCL_ERROR = 101,
    SAMG_OUT_OF_MEMORY = 102,
    SAMG_NO_DEVICE = 103,
    SAMG_UNSUPPORTED = 104,        /* pipeline / smoother not on this path */
    SAMG_INVALID_ARGUMENT = 105
};

/* samg::pipeline (hierarchy.hpp:30).  SAMG_PIPELINE_NS_BLOCK is the B200
 * hot path; NS_HYBRID2 and NS_HYBRID1 (scalar-space Galerkin, block storage,
 * hierarchy.hpp:233-330) are supported with the same bit-exact parity, and
 * so is BLOCK (no nullspace: B may be NULL and is ignored,
 * hierarchy.hpp:340-347).  SCALAR (no nullspace: aggregate indicator with
 * 3-unknown points, B ignored) and NS_SCALAR (hierarchy.hpp:298-330) keep
 * scalar CSR levels in the reference: here the same values as 3x3 blocks
 * (their patterns are whole blocks for matrices with full 3x3 blocks),
 * memory_footprint in the reference's scalar accounting, the reference's
 * scalar smoothers (damped Jacobi, ilu0<double>).  ILU0 with SCALAR,
 * NS_SCALAR and NS_HYBRID1 is the scalar ilu0<double> of the level matrix
 * (hierarchy.hpp:288-291), bit-identical.  The scalar pipelines and ILU(0)
 * are single-GPU. */
enum samg_pipeline {
    SAMG_PIPELINE_SCALAR = 0,
    SAMG_PIPELINE_BLOCK = 1,
    SAMG_PIPELINE_NS_SCALAR = 2,
    SAMG_PIPELINE_NS_HYBRID1 = 3,
    SAMG_PIPELINE_NS_HYBRID2 = 4,
    SAMG_PIPELINE_NS_BLOCK = 5
};

/* Smoothers.  JACOBI = the reference's point damped_jacobi
 * (relaxation.hpp:141-180, omega default 0.72).  SPAI0 and BLOCK_JACOBI are
 * 3x3 block smoothers.  ILU0 = the reference's default
 * ilu0<block3> (relaxation.hpp:20-139; ilu0<double> for the scalar-smoother
 * pipelines), bit-identical factors and sweeps
 * (single GPU; the partitioned solver returns SAMG_UNSUPPORTED). */
enum samg_smoother {
    SAMG_SMOOTHER_JACOBI = 0,
    SAMG_SMOOTHER_SPAI0 = 1,
    SAMG_SMOOTHER_BLOCK_JACOBI = 2,
    SAMG_SMOOTHER_ILU0 = 3
};

/* Storage precision of the operators the V-cycle streams (an extension: the
 * reference is fp64 throughout).  FP64 (default) reproduces the reference.
 * MIXED keeps fp32 copies of A_l, P_l, R_l for the V-cycle's sweeps,
 * residuals and transfers (vectors, arithmetic, smoother data, the coarse
 * inverse and CG itself stay fp64; CG's A p and the exit residual read the
 * fp64 matrix): about half the bytes per V-cycle, a preconditioner that
 * differs from the fp64 one at fp32 rounding level. */
enum samg_precision {
    SAMG_PRECISION_FP64 = 0,
    SAMG_PRECISION_MIXED = 1
};

/* Order of the subtraction chain in the block ILU(0) backward sweep (an
 * extension).  REFERENCE (default): ascending columns, as relaxation.hpp:
 * 73-88 -- every application is bit-identical to the reference's.
 * LATEST_LAST: descending columns, so the dependency that completes last
 * (row i + 1) is the chain's last term instead of its first and only a few
 * subtractions follow the hand-off; the same factors and the same sums up to
 * rounding (C1: the same 38 iterations, backward sweeps 1.19 -> 0.57 ms,
 * solve 0.42 -> 0.28 s).  Block ILU(0) only. */
enum samg_ilu_order {
    SAMG_ILU_ORDER_REFERENCE = 0,
    SAMG_ILU_ORDER_LATEST_LAST = 1
};

/* amg_params (hierarchy.hpp:50-58) + coarsening_params (coarsening.hpp:26-31)
 * + the smoother selector and device placement. */
typedef struct {
    double eps_strong;        /* 0.08 */
    double omega;             /* prolongator damping, 2/3 */
    int point_block_size;     /* forced to 3 for ns pipelines (hierarchy.hpp:284) */
    int smoother;             /* samg_smoother, default SPAI0 */
    double smoother_omega;    /* Jacobi / block-Jacobi damping, 0.72 */
    int pre_sweeps;           /* 1 */
    int post_sweeps;          /* 1 */
    int64_t coarse_enough;    /* 3000 scalar unknowns */
    double stagnation_ratio;  /* 0.8 */
    int verify_galerkin;      /* 0; 1: recompute every coarse operator as the
                                 scalar R A P and fail with SAMG_ERROR on a
                                 mismatch (hierarchy.hpp:382-401) */
    int device;               /* CUDA device ordinal, default 0 */
    int vcycle_precision;     /* samg_precision, default FP64 */
    int ilu_sweep_order;      /* samg_ilu_order, default REFERENCE */
} samg_amg_params;

/* cg_params (cg.hpp:32-35) */
typedef struct {
    double tol;               /* 1e-8 */
    int max_iterations;       /* 1000 */
} samg_cg_params;

/* solve_report (cg.hpp:22-30) */
typedef struct {
    int iterations;
    double relative_residual;     /* true residual at exit (cg.hpp:105-108) */
    double setup_seconds;
    double solve_seconds;
    uint64_t preconditioner_bytes; /* memory_footprint (hierarchy.hpp:443-458) */
    int variant;                  /* samg_pipeline */
    int converged;
} samg_solve_report;

typedef struct samg_hierarchy samg_hierarchy;  /* owns all level data on the GPU */
typedef struct samg_bsr3 samg_bsr3;            /* a device-resident 3x3 BSR matrix */
typedef struct samg_problem samg_problem;      /* host-side synthetic problem */

SAMG_API void samg_default_amg_params(samg_amg_params *p);
SAMG_API void samg_default_cg_params(samg_cg_params *p);
SAMG_API const char *samg_last_error(void);     /* thread-local message */
SAMG_API const char *samg_status_name(int status);
SAMG_API int samg_device_count(int *count);

/* ---- setup: replaces samg::setup (hierarchy.hpp:263-405) ----------------
 * Scalar CSR input (int64 ptr/col, fp64 val, n rows), exactly the
 * reference's csr<double> (csr.hpp:26-40).  B is the column-major
 * b_rows-by-b_cols near-nullspace (dense_columns, csr.hpp:46-55) or NULL.
 * Partly stored 3x3 blocks are padded with zeros like to_block<3>
 * (csr.hpp:268-324); the pipelines that keep the scalar pattern (scalar,
 * ns_scalar, ns_hybrid1 with ilu0<double>) return SAMG_UNSUPPORTED for such
 * an input, since the padding would change their ILU(0) pattern and
 * footprint. */
SAMG_API int samg_setup(int64_t n, const int64_t *ptr, const int64_t *col,
        const double *val, const double *B, int64_t b_rows, int64_t b_cols,
        int pipeline, const samg_amg_params *prm, samg_hierarchy **out);
/* Same, from 3x3 block CSR (nbrows block rows, blocks row-major 9 doubles),
 * i.e. the result of to_block<3> (csr.hpp:268-324) without the host pass. */
SAMG_API int samg_setup_bsr3(int64_t nbrows, const int64_t *ptr,
        const int64_t *col, const double *val, const double *B, int64_t b_rows,
        int64_t b_cols, int pipeline, const samg_amg_params *prm,
        samg_hierarchy **out);
SAMG_API int samg_destroy(samg_hierarchy *h);

/* ---- solve: replaces samg::cg_solve (cg.hpp:87-112) --------------------
 * f, u host pointers of length finest_dim; u is overwritten (zero start). */
SAMG_API int samg_cg_solve(samg_hierarchy *h, const double *f, double *u,
        const samg_cg_params *prm, samg_solve_report *rep);
/* Same with device pointers on the hierarchy's device. */
SAMG_API int samg_cg_solve_device(samg_hierarchy *h, const double *d_f,
        double *d_u, const samg_cg_params *prm, samg_solve_report *rep);

/* ---- preconditioner: replaces samg::vcycle (hierarchy.hpp:408-441) ------
 * u is the initial approximation and the result (host / device pointers). */
SAMG_API int samg_vcycle(samg_hierarchy *h, const double *f, double *u);
/* The generic driver cg_solve_op(n, apply_A, apply_M, f, u, prm)
 * (cg.hpp:39-83) with caller operators on DEVICE vectors of n doubles:
 * fn(ctx, in, out, stream) computes out = A in (apply_A) or out = M in
 * (apply_M; NULL = identity) and returns 0 or a samg_status; it sees its
 * input complete and must finish its work before returning or enqueue it on
 * `stream` (a cudaStream_t).  u is zeroed first; the CG vector work runs on
 * the device (deterministic reductions); relative_residual is the
 * recurrence's ||r||/||f|| (cg_solve_op computes no true residual).  E.g.
 * apply_A = samg_bsr3_spmv_device, apply_M = zero z + samg_vcycle_device. */
typedef int (*samg_apply_fn)(void *ctx, const double *d_in, double *d_out, void *stream);
SAMG_API int samg_cg_solve_op(int64_t n, samg_apply_fn apply_A, samg_apply_fn apply_M,
        void *ctx, const double *d_f, double *d_u, const samg_cg_params *prm, int device,
        samg_solve_report *rep);
SAMG_API int samg_vcycle_device(samg_hierarchy *h, const double *d_f,
        double *d_u);

/* ---- introspection / parity taps ---------------------------------------- */
SAMG_API int samg_memory_footprint(const samg_hierarchy *h, uint64_t *bytes);
SAMG_API int samg_finest_dim(const samg_hierarchy *h, int64_t *n);
SAMG_API int samg_num_levels(const samg_hierarchy *h, int *nlevels);
SAMG_API int samg_coarse_dim(const samg_hierarchy *h, int64_t *n);
/* coarse solve in use: 0 = explicit inverse (GEMV), 1 = the reference's
 * dense LU, bit-exact (chosen when the inverse fails its accuracy check,
 * i.e. for a numerically singular coarse operator) */
SAMG_API int samg_coarse_solver(const samg_hierarchy *h, int *kind);
SAMG_API int samg_setup_seconds(const samg_hierarchy *h, double *seconds);
/* which: 0 = A, 1 = P, 2 = R of `level`; sizes in 3x3 blocks */
SAMG_API int samg_level_info(const samg_hierarchy *h, int level, int which,
        int64_t *nrows, int64_t *ncols, int64_t *nnzb);
/* copies into host buffers sized by samg_level_info: ptr[nrows+1],
 * col[nnzb], val[9*nnzb] */
SAMG_API int samg_get_level(const samg_hierarchy *h, int level, int which,
        int64_t *ptr, int64_t *col, double *val);
/* borrow a level matrix as a device BSR3 (owned by the hierarchy) */
SAMG_API int samg_level_matrix(samg_hierarchy *h, int level, int which,
        const samg_bsr3 **m);
/* aggregate ids of the level's nodes (node = point_block_size scalar rows) */
SAMG_API int samg_aggregates_info(const samg_hierarchy *h, int level,
        int64_t *nnodes, int64_t *count);
SAMG_API int samg_get_aggregates(const samg_hierarchy *h, int level,
        int64_t *id);
/* smoother data: 3 per block row (point Jacobi 1/a_ii) or 9 (block M_i) */
SAMG_API int samg_smoother_info(const samg_hierarchy *h, int level,
        int64_t *len);
SAMG_API int samg_get_smoother(const samg_hierarchy *h, int level,
        double *data);

/* ---- device BSR3 matrices: spmv<static_block<3>> (csr.hpp:129-160) ------ */
SAMG_API int samg_bsr3_create(int64_t nrows, int64_t ncols, const int64_t *ptr,
        const int64_t *col, const double *val, int device, samg_bsr3 **out);
SAMG_API int samg_bsr3_destroy(samg_bsr3 *m);
SAMG_API int samg_bsr3_info(const samg_bsr3 *m, int64_t *nrows, int64_t *ncols,
        int64_t *nnzb);
SAMG_API int samg_bsr3_download(const samg_bsr3 *m, int64_t *ptr, int64_t *col,
        double *val);
/* y = alpha*A*x + beta*y with device vectors on `stream` (cudaStream_t or
 * NULL for the legacy stream); asynchronous. */
SAMG_API int samg_bsr3_spmv_device(const samg_bsr3 *m, double alpha,
        const double *d_x, double beta, double *d_y, void *stream);
/* same with host vectors: H2D x (and y if beta != 0), kernel, D2H y */
SAMG_API int samg_bsr3_spmv(const samg_bsr3 *m, double alpha, const double *x,
        double beta, double *y);
/* Galerkin product R*A*P (csr.hpp:259-262) in the reference's summation
 * order; result is a new device matrix. */
/* count products y_k = alpha*A*x_k + beta*y_k with host vectors
 * (x: count x 3*ncols, y: count x 3*nrows, row-major); each product copies
 * its own x_k in and y_k out, pipelined over three streams so the copies of
 * neighbouring products overlap the kernel.  Pinned host memory gives full
 * PCIe bandwidth (pageable memory is copied correctly, more slowly). */
SAMG_API int samg_bsr3_spmv_batch(const samg_bsr3 *m, double alpha,
        const double *x, double beta, double *y, int64_t count);
SAMG_API int samg_bsr3_galerkin(const samg_bsr3 *R, const samg_bsr3 *A,
        const samg_bsr3 *P, samg_bsr3 **out);
/* algorithmic bytes of one spmv */
/* coarsest-level direct solver on its own: inv (host, n x n row-major,
 * n = 3*nrows) = A^-1 by the device's in-place blocked Gauss-Jordan with the
 * reference's partial pivoting (dense_lu, hierarchy.hpp:86-129); a pivot
 * below 1e-300 returns SAMG_ERROR ("singular"). */
SAMG_API int samg_bsr3_dense_inverse(const samg_bsr3 *m, double *inv);
SAMG_API int samg_bsr3_spmv_bytes(const samg_bsr3 *m, int beta_nonzero,
        uint64_t *bytes);

/* ---- row-partitioned operator for multi-GPU runs ---
 * One process per GPU; rank r owns block rows [row_starts[r], row_starts[r+1])
 * of a global BSR3 matrix.  The halo plan is built on the host (no GPU
 * needed); the caller's transport (NCCL / gloo) moves the data:
 *   1. samg_dist_create with the rank's rows (global column ids);
 *   2. send every recv peer the global ids of its ghost segment
 *      (samg_dist_recv_plan + samg_dist_ghosts), receive the peers' lists
 *      and hand them to samg_dist_set_send;
 *   3. per SpMV: samg_dist_pack(x) -> send buffers to the send peers,
 *      receive into x_ext[3*nloc + 3*offset ...], samg_dist_spmv(interior)
 *      may run while the halo is in flight, then samg_dist_spmv(boundary).
 * y equals the single-GPU spmv bit-for-bit (same per-row block order). */
typedef struct samg_dist samg_dist;
SAMG_API int samg_dist_create(int64_t row0, int64_t row1, const int64_t *ptr,
        const int64_t *col, const double *val, int nranks,
        const int64_t *row_starts, int rank, samg_dist **out);
SAMG_API int samg_dist_destroy(samg_dist *d);
SAMG_API int samg_dist_info(const samg_dist *d, int64_t *nloc, int64_t *nghost,
        int64_t *ninterior, int64_t *nboundary, int *nrecv_peers,
        int *nsend_peers);
SAMG_API int samg_dist_recv_plan(const samg_dist *d, int *peers,
        int64_t *counts, int64_t *offsets);
SAMG_API int samg_dist_ghosts(const samg_dist *d, int64_t *global_ids);
SAMG_API int samg_dist_set_send(samg_dist *d, int npeers, const int *peers,
        const int64_t *counts, const int64_t *global_ids);
SAMG_API int samg_dist_send_plan(const samg_dist *d, int *peers,
        int64_t *counts, int64_t *offsets, int64_t *local_rows);
/* Step 2 without the transport: the send plan derived from the rank's own
 * rows -- for a structurally symmetric matrix, peer q reads exactly the
 * owned rows that hold a column in q's range (the rule the distributed
 * setup and solve use for every operator, dsolve.cu build_local_rows). */
SAMG_API int samg_dist_derive_send(samg_dist *d);
/* the renumbered local matrix (columns: owned [0,nloc), ghosts nloc+g) */
SAMG_API int samg_dist_local_matrix(const samg_dist *d, int64_t *ptr,
        int64_t *col, double *val);
/* upload to `device`; group = lanes per row (0 = auto, or 4/8/16/32 to match
 * the single-GPU kernel exactly) */
SAMG_API int samg_dist_to_device(samg_dist *d, int device, int group);
SAMG_API int samg_dist_pack(const samg_dist *d, const double *d_x,
        double *d_sendbuf, void *stream);
/* part: 0 = interior rows, 1 = boundary rows, 2 = all rows */
SAMG_API int samg_dist_spmv(const samg_dist *d, int part, double alpha,
        const double *d_xext, double beta, double *d_y, void *stream);

/* ---- multi-GPU setup + solve (one process per GPU, NCCL; DESIGN.md s.6) --
 * The setup is distributed: each rank builds only its rows of the levels
 * with >= min_rows*nranks block rows (fine block rows
 * row_starts[rank]..row_starts[rank+1]; coarse rows follow the aggregates'
 * seeds: an aggregate belongs to the rank owning its seed node), fetching
 * from the owners only the halo rows it needs; the node graph of the
 * strength test is gathered so that every rank aggregates exactly as one
 * GPU (coarsening.hpp:131-160).  The first level below the threshold is
 * gathered and the rest set up and solved redundantly.  Every level is
 * bit-identical to the single-GPU (and reference) hierarchy.  The V-cycle
 * exchanges halos with ncclSend/ncclRecv and CG all-reduces its dot
 * products.  f and u are the rank's rows (3 per block row).  Obtain the
 * NCCL id on rank 0 with samg_nccl_unique_id and broadcast it.
 * samg_dsetup: every rank passes the global matrix (host), only its rows are
 * uploaded.  samg_dsetup_local / samg_dsetup_device: each rank passes only
 * its rows (global column ids; ptr from 0) and its nullspace rows
 * (3*nloc x b_cols, column-major), from host or device memory.
 * id == NULL (samg_dsetup only) emulates all nranks in the calling process
 * on one GPU (no NCCL): every exchange becomes a device copy with the same
 * offsets and counts, and f and u are the global vectors.  This is the
 * single-GPU check of the distributed setup and the halo plans. */
typedef struct samg_dhierarchy samg_dhierarchy;
SAMG_API int samg_nccl_unique_id(unsigned char id[128]);
SAMG_API int samg_dsetup(const unsigned char id[128], int nranks, int rank,
        int64_t nbrows, const int64_t *ptr, const int64_t *col,
        const double *val, const double *B, int64_t b_rows, int64_t b_cols,
        const int64_t *row_starts, int64_t min_rows, int pipeline,
        const samg_amg_params *prm, samg_dhierarchy **out);
SAMG_API int samg_ddestroy(samg_dhierarchy *h);
SAMG_API int samg_dinfo(const samg_dhierarchy *h, int64_t *row0,
        int64_t *row1, int *nlevels, int *dist_levels, double *setup_seconds);
SAMG_API int samg_dsetup_local(const unsigned char id[128], int nranks, int rank,
        const int64_t *row_starts, const int64_t *ptr, const int64_t *col,
        const double *val, const double *B, int64_t b_cols, int64_t min_rows,
        int pipeline, const samg_amg_params *prm, samg_dhierarchy **out);
SAMG_API int samg_dsetup_device(const unsigned char id[128], int nranks, int rank,
        const int64_t *row_starts, const samg_bsr3 *A_local, const double *d_B,
        int64_t b_cols, int64_t min_rows, int pipeline, const samg_amg_params *prm,
        samg_dhierarchy **out);
/* Block rows of A_0 the (first driven) rank held during the setup: its own
 * rows plus the halo rows it fetched.  No reference counterpart. */
SAMG_API int samg_dheld_rows(const samg_dhierarchy *h, int64_t *rows);
/* Parity taps on the distributed hierarchy's level matrices, assembled from
 * every rank's rows (collective over the ranks for a distributed level):
 * as samg_level_info / samg_get_level. */
SAMG_API int samg_dlevel_info(const samg_dhierarchy *h, int level, int which,
        int64_t *nrows, int64_t *ncols, int64_t *nnzb);
SAMG_API int samg_dget_level(const samg_dhierarchy *h, int level, int which,
        int64_t *ptr, int64_t *col, double *val);
SAMG_API int samg_dcg_solve_device(samg_dhierarchy *h, const double *d_f,
        double *d_u, const samg_cg_params *prm, samg_solve_report *rep);
SAMG_API int samg_dcg_solve(samg_dhierarchy *h, const double *f, double *u,
        const samg_cg_params *prm, samg_solve_report *rep);

/* ---- synthetic problems (input tooling; elasticity.hpp:38-213 extended) -- */
enum samg_dirichlet { SAMG_DIRICHLET_NONE = 0, SAMG_DIRICHLET_KEEP_ROWS = 1,
                      SAMG_DIRICHLET_ELIMINATE = 2 };
enum samg_load { SAMG_LOAD_BODY_FORCE = 0, SAMG_LOAD_TRACTION_XEND = 1,
                 SAMG_LOAD_RANDOM = 2 };
typedef struct {
    int64_t nx, ny, nz;       /* elements per axis (nodes = n+1) */
    double lx, ly, lz;        /* domain lengths (unit cube = 1,1,1) */
    double E, nu;             /* homogeneous material */
    int heterogeneous;        /* 1: E_e = exp(N(0,1)), nu_e ~ U[0.25,0.35] */
    int dirichlet;            /* samg_dirichlet on the x=0 face */
    int load;                 /* samg_load */
    double noise;             /* + U[-noise, noise] per DOF */
    uint64_t seed;
    int x_slowest;            /* node numbering: 0 = x fastest (reference) */
    int64_t node_begin;       /* if node_end > node_begin: only the rows of */
    int64_t node_end;         /* nodes [begin, end), global column ids     */
} samg_problem_params;
SAMG_API void samg_default_problem_params(samg_problem_params *p);
SAMG_API int samg_generate_hex(const samg_problem_params *p, samg_problem **out);
SAMG_API int samg_problem_destroy(samg_problem *p);
/* n = scalar DOFs (3 per node kept), nbrows = n/3, nnzb 3x3 blocks */
SAMG_API int samg_problem_info(const samg_problem *p, int64_t *n,
        int64_t *nnzb, int64_t *nnodes);
SAMG_API int samg_problem_get_bsr3(const samg_problem *p, int64_t *ptr,
        int64_t *col, double *val);
/* scalar CSR with every block entry kept (to_scalar, csr.hpp:327-353) */
SAMG_API int samg_problem_get_csr(const samg_problem *p, int64_t *ptr,
        int64_t *col, double *val);
SAMG_API int samg_problem_get_rhs(const samg_problem *p, double *rhs);
/* coordinates of the kept nodes, 3 per node */
SAMG_API int samg_problem_get_coords(const samg_problem *p, double *xyz);
/* rigid body modes (elasticity.hpp:38-52), column-major n-by-6 */
SAMG_API int samg_rigid_body_modes(int64_t nnodes, const double *xyz,
        double *B);
/* borrow the problem's BSR arrays (no copy; valid until destroy) */
SAMG_API int samg_problem_bsr3_view(const samg_problem *p, const int64_t **ptr,
        const int64_t **col, const double **val);

/* ---- on-GPU assembly ----------------------------------------
 * The same problems assembled directly in device memory (bitwise equal to
 * samg_generate_hex): 3x3 BSR matrix, right-hand side, node coordinates and
 * the rigid-body modes (3n x 6, column-major), all device pointers owned by
 * the handle.  samg_setup_device builds a hierarchy from a device matrix
 * (copied) and a host or device nullspace. */
typedef struct samg_dproblem samg_dproblem;
SAMG_API int samg_generate_hex_device(const samg_problem_params *p, int device,
        samg_dproblem **out);
SAMG_API int samg_dproblem_destroy(samg_dproblem *p);
SAMG_API int samg_dproblem_info(const samg_dproblem *p, int64_t *n,
        int64_t *nbrows, int64_t *nnzb);
SAMG_API int samg_dproblem_matrix(const samg_dproblem *p, const samg_bsr3 **A);
SAMG_API int samg_dproblem_vectors(const samg_dproblem *p, const double **d_rhs,
        const double **d_nullspace, const double **d_xyz);
/* host copies of the vectors (any pointer may be NULL) */
SAMG_API int samg_dproblem_download(const samg_dproblem *p, double *rhs,
        double *nullspace, double *xyz);
SAMG_API int samg_setup_device(const samg_bsr3 *A, const double *B,
        int64_t b_rows, int64_t b_cols, int pipeline,
        const samg_amg_params *prm, samg_hierarchy **out);

#ifdef __cplusplus
}
#endif

#endif /* SAMG_B200_H */
