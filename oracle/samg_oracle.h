/*
 * samg_oracle.h -- CPU restatement of the reference SA-AMG "NS Block" path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 product
 * in paper_2202_09056_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * never links, calls or falls back to anything in oracle/.
 *
 * It restates, in plain C, the algorithms of the reference library
 * (/root/reference/proj/include/samg, cited per function as file:line) with
 * the same loop and summation orders, so that on the same inputs the setup
 * phase is bit-identical to the reference (pinned against oracle/_ref and
 * tests/golden).  Compiled with -ffp-contract=off (no FMA), like the
 * reference's header translation units.
 */
#ifndef SAMG_ORACLE_H
#define SAMG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: 1:1 with the samg exception classes (common.hpp:12-28). */
enum {
    ORC_OK = 0,
    ORC_ERROR = 1,
    ORC_DIMENSION_MISMATCH = 2,
    ORC_NOT_DIVISIBLE = 3,
    ORC_SINGULAR_BLOCK = 4,
    ORC_MISSING_DIAGONAL = 5,
    ORC_ZERO_DIAGONAL = 6,
    ORC_NON_SQUARE = 7,
    ORC_BAD_NULLSPACE_SHAPE = 8,
    ORC_BREAKDOWN_NON_SPD = 9,
    ORC_INVALID_MATERIAL = 10
};

/* Smoother kinds.  JACOBI is the reference's point damped Jacobi
 * (relaxation.hpp:141-180); SPAI0 and BLOCK_JACOBI are the 3x3 block
 * smoothers the reference lacks (definitions in DESIGN.md section 4). */
enum { ORC_SM_JACOBI = 0, ORC_SM_SPAI0 = 1, ORC_SM_BLOCK_JACOBI = 2, ORC_SM_ILU0 = 3 };

/* Block CSR, block size b in {1,3}; val holds nnz*b*b doubles, each block
 * row-major (static_block.hpp:19-66, csr.hpp:26-40). */
typedef struct {
    int64_t nrows, ncols; /* in block units */
    int b;
    int64_t *ptr, *col;
    double *val;
} orc_mat;

typedef struct {
    int64_t nnodes;
    int64_t *ptr, *col;
} orc_adj;

typedef struct {
    double eps_strong;       /* coarsening.hpp:27 */
    double omega;            /* coarsening.hpp:28 */
    int smoother;            /* ORC_SM_* */
    double smoother_omega;   /* Jacobi / block-Jacobi damping */
    int pre_sweeps, post_sweeps;
    int64_t coarse_enough;   /* hierarchy.hpp:55 */
    double stagnation_ratio; /* hierarchy.hpp:56 */
    int pipeline;            /* ORC_PIPELINE_NS_BLOCK or _NS_HYBRID1/2 */
} orc_params;

/* samg::pipeline values (hierarchy.hpp:30) handled by orc_setup_ns_block */
enum { ORC_PIPELINE_BLOCK = 1, ORC_PIPELINE_NS_HYBRID1 = 3, ORC_PIPELINE_NS_HYBRID2 = 4,
       ORC_PIPELINE_NS_BLOCK = 5 };

typedef struct {
    int iterations;
    double relative_residual;
    int converged;
} orc_report;

typedef struct orc_hier orc_hier;

const char *orc_last_error(void);

void orc_default_params(orc_params *p);

/* --- generator (elasticity.hpp) ------------------------------------------ */
/* Reference generator restated: unit cube, clamp x=0 with unit rows,
 * body force -z.  Returns status; outputs are malloc'd (free with orc_free). */
int orc_generate_hex(int64_t nx, int64_t ny, int64_t nz, double E, double nu,
        int clamp_x0, int64_t *n_out, int64_t **ptr, int64_t **col,
        double **val, double **rhs, double **coords);
void orc_hex8_stiffness(double hx, double hy, double hz, double E, double nu,
        double *Ke /* 576 */);
void orc_rigid_body_modes(int64_t nnodes, const double *coords, double *B);
void orc_free(void *p);

/* --- sparse kernels (csr.hpp) --------------------------------------------- */
int orc_spmv_bsr3(int64_t nrows, int64_t ncols, const int64_t *ptr,
        const int64_t *col, const double *val, double alpha, const double *x,
        double beta, double *y);

/* Galerkin R*A*P on 3x3 blocks; result malloc'd. */
int orc_galerkin_bsr3(const orc_mat *R, const orc_mat *A, const orc_mat *P,
        orc_mat *C);

/* Strength + aggregation on a scalar CSR (coarsening.hpp:81-160). */
int orc_aggregate_scalar(int64_t n, const int64_t *ptr, const int64_t *col,
        const double *val, double eps, int pbs, int64_t *id, int64_t *count);

/* --- hierarchy (hierarchy.hpp, cg.hpp) ------------------------------------ */
/* Setup of the ns_block pipeline from a scalar CSR input and a column-major
 * n-by-k nullspace B (hierarchy.hpp:263-405). */
int orc_setup_ns_block(int64_t n, const int64_t *ptr, const int64_t *col,
        const double *val, const double *B, int64_t bcols,
        const orc_params *prm, orc_hier **out);
void orc_hier_free(orc_hier *h);
int orc_hier_nlevels(const orc_hier *h);
/* which: 0=A, 1=P, 2=R.  Returns pointers into the hierarchy (block 3x3). */
int orc_hier_matrix(const orc_hier *h, int level, int which, orc_mat *m);
/* aggregates of level (level < nlevels-1); pointers into the hierarchy */
int orc_hier_aggregates(const orc_hier *h, int level, int64_t *nnodes,
        const int64_t **id, int64_t *count);
/* smoother data of a level: n doubles (point) or 9 per block row */
int orc_hier_smoother(const orc_hier *h, int level, int64_t *len,
        const double **data);
int64_t orc_hier_coarse_dim(const orc_hier *h);
uint64_t orc_hier_memory_footprint(const orc_hier *h);
int orc_vcycle(const orc_hier *h, const double *f, double *u);
int orc_cg_solve(const orc_hier *h, const double *f, double *u, double tol,
        int max_iterations, orc_report *rep);

#ifdef __cplusplus
}
#endif

#endif
