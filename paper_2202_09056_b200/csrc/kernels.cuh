// kernels.cuh -- device data layout and kernel launchers.
//
// HBM layout of a level matrix (Bsr3): the reference's csr<static_block<3>>
// (csr.hpp:26-40) with 32-bit indices: ptr[nrows+1], col[nnzb] (int32) and
// val[9*nnzb] fp64, each 3x3 block row-major and the blocks of a row
// contiguous and column-sorted.  Vectors are in scalar layout (3 per block
// row), exactly as the reference's spmv expects (csr.hpp:9-12).
#pragma once

#include "common.cuh"

namespace samgb {

struct Bsr3 {
    int64_t nrows = 0, ncols = 0, nnzb = 0;
    DevBuf<int> ptr, col;
    DevBuf<double> val;
    DevBuf<float> val32;  // optional fp32 copy of val (mixed-precision V-cycle)
    // optional node-blocked copy (make_node6): rows and columns paired into
    // 6x6 blocks -- the operators of levels >= 1 of the ns pipelines, whose
    // nodes are 2 block rows (pbs 6).  One column index and one 48-byte x
    // gather per four 3x3 blocks; used by the V-cycle's SpMV family.
    int64_t nrows6 = 0, nnzb6 = 0;
    DevBuf<int> ptr6, col6;
    DevBuf<double> val6;
    void alloc(int64_t nr, int64_t nc, int64_t nz, cudaStream_t s) {
        if (nz > INT32_MAX || nr > INT32_MAX || nc > INT32_MAX)
            fail(SAMG_UNSUPPORTED, "BSR3: more than 2^31-1 blocks per matrix");
        nrows = nr; ncols = nc; nnzb = nz;
        ptr.alloc(nr + 1, s);
        col.alloc(nz, s);
        val.alloc(9 * nz, s);
    }
};

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
enum SmootherKind { SM_POINT = 0, SM_BLOCK = 1, SM_ILU = 2 };

// Per-level smoother: point (3 doubles per block row: omega / a_rr), block
// (9 doubles per block row: M_i) or block ILU(0) (ilu0<block3>,
// relaxation.hpp:20-139): data = inverted pivots (9 per block row), lu =
// the factors in A's pattern (9 per block), whose ptr/col are A's.
struct Smoother {
    int kind = SM_POINT;
    DevBuf<double> data;
    // ILU(0) only
    DevBuf<double> lu, tmp;      // factors; scratch vector (3 per block row)
    DevBuf<double> sweep;        // sweep outputs y, x (3 per block row each) + row counters
    DevBuf<int> dpos, flags;     // diagonal position per row; factorization flags
    DevBuf<int> order;           // rows in level order: forward (n), backward (n)
    int depth[2] = {1, 1};       // number of forward / backward dependency levels
    const int *ptr = nullptr, *col = nullptr;  // A's pattern
    int64_t nrows = 0, nnzb = 0;
    // ilu0<double> on the scalar view (the scalar pipelines' and
    // ns_hybrid1's smoother): factors in the same 3x3 block layout, data =
    // the inverted scalar pivots (3 per block row)
    bool scalar = false;
    // backward sweep's subtraction chain over descending columns
    // (samg_ilu_order LATEST_LAST; block ILU(0) only)
    bool latest_last = false;
};

// ---- solve phase (solve.cu) -------------------------------------------------
// y = alpha*A*x + beta*y  (csr.hpp:129-160)
// lowp (mixed-precision V-cycle): read A.val32 instead of A.val when present;
// vectors and arithmetic stay fp64
void launch_spmv(const Bsr3 &A, double alpha, const double *x, double beta, double *y,
                 cudaStream_t s, bool lowp = false);
// r = f - A*u  (csr.hpp:163-169)
void launch_residual(const Bsr3 &A, const double *f, const double *u, double *r,
                     cudaStream_t s, bool lowp = false);
// u_out = u + M (f - A u)  (one smoothing sweep, relaxation.hpp:165-173)
void launch_smooth(const Bsr3 &A, const Smoother &M, const double *f, const double *u,
                   double *u_out, cudaStream_t s, bool lowp = false);
// cap on the persistent SpMV's CTAs for this host thread (-1: default /
// SAMG_TMA_CTAS, 0: one per SM)
void set_spmv_cta_cap(int ctas);
// programmatic dependent launch of the TMA-fed SpMV for this host thread
// (back-to-back standalone SpMVs; solve.cu)
void set_spmv_pdl(bool on);
// fp32 copy of the values (A.val32) for the mixed-precision V-cycle
void make_lowp(Bsr3 &A, cudaStream_t s);
// 6x6 node-blocked copy (A.val6) if A's rows and columns pair up (returns
// whether it did)
bool make_node6(Bsr3 &A, cudaStream_t s);
// u = M f  (one sweep from a zero guess: the residual is f exactly)
// launch_smooth with the gathered x apart from the row-indexed u / f / M / out
void launch_smooth_split(const Bsr3 &A, const Smoother &M, const double *f, const double *x,
                         const double *u, double *u_out, cudaStream_t s);
void launch_smooth_zero(int64_t nrows, const Smoother &M, const double *f, double *u,
                        cudaStream_t s);
// leading dimension of the dense coarse inverse (even, for 16-byte loads)
inline int64_t dense_ld(int64_t n) { return (n + 1) & ~static_cast<int64_t>(1); }
// dense coarse solve u = Ainv f (replaces dense_lu::solve, hierarchy.hpp:113-129)
void launch_dense_gemv(int64_t n, const double *Ainv, const double *f, double *u,
                       cudaStream_t s);

// CG device scalars (cg.hpp:39-83).
struct CgScalars {
    double pq, rho, rho_new, rr, alpha, beta;
    double tmp;  // raw local sum (CG_STORE) awaiting a cross-rank allreduce
    double tmp2; // a second one (CG_STORE2), all-reduced together with tmp
    double norm_f, tol;
    int breakdown, iter, max_iter;
    unsigned ticket;  // last-CTA counter of the fused reductions
};
// What a fused reduction finishes (cg.hpp:58-77).  Every reduction writes
// one partial per CTA; the last CTA sums them in index order (deterministic)
// and applies: RR: rr; PQ: pq, alpha = rho/pq, breakdown if pq <= 0;
// RZ: beta = rz/rho, rho = rz; RHO: rho; RR_LOOP: rr, ++iter and the graph
// loop condition ||r||/||f|| > tol && iter < max && !breakdown.
// STORE: only tmp = s (multi-GPU: allreduce tmp, then launch_cg_finish).
enum { CG_RR = 0, CG_PQ = 1, CG_RZ = 2, CG_RHO = 3, CG_RR_LOOP = 4, CG_STORE = 5, CG_ADD = 6,
       CG_STORE2 = 7 };
// q = A x and p.q on a row range (x the whole halo-extended vector)
void launch_spmv_dot_split(const Bsr3 &A, const double *x, const double *p, double *q,
                           double *partials, CgScalars *sc, cudaStream_t s, int what);
// apply `what` to sc->tmp (after the allreduce of the partial sums)
void launch_cg_finish(CgScalars *sc, int what, cudaStream_t s);
// after the allreduce of (tmp, tmp2) = (r.r, r.z): r.r -> `rr_what` (CG_RR,
// or CG_RR_LOOP setting the graph's loop condition h), r.z -> CG_RZ
void launch_cg_finish2(CgScalars *sc, int rr_what, cudaGraphConditionalHandle h, cudaStream_t s);
// CTAs of the vector kernels: 4 x 148 SMs (8 x 148 measured slower for the
// fused CG update, 13.7 -> 17.4 us at C1); fixed => deterministic sums
constexpr int kRedBlocks = 592;
// q = A p fused with p.q (cg.hpp:63-64) -> PQ
void launch_spmv_dot(const Bsr3 &A, const double *p, double *q, double *partials,
                     CgScalars *sc, cudaStream_t s, int what = CG_PQ);
// last post-smoothing sweep of the V-cycle fused with r.z (cg.hpp:73-75) -> RZ
void launch_smooth_dot(const Bsr3 &A, const Smoother &M, const double *f, const double *u,
                       double *u_out, double *partials, CgScalars *sc, cudaStream_t s,
                       int what = CG_RZ, bool lowp = false);
// x.y -> what
void launch_dot(int64_t n, const double *x, const double *y, double *partials, CgScalars *sc,
                int what, cudaStream_t s);
// u += alpha p; r -= alpha q fused with r.r -> RR or RR_LOOP
void launch_cg_update(int64_t n, CgScalars *sc, const double *p, const double *q, double *u,
                      double *r, double *partials, int what, cudaGraphConditionalHandle h,
                      cudaStream_t s);
// p = z + beta p
void launch_p_update(int64_t n, const CgScalars *sc, const double *z, double *p,
                     cudaStream_t s);
// r -= alpha q with r.r -> what, and z0 = M r (the V-cycle's first level-0
// sweep from zero); u's update is deferred to launch_p_update_u.  false
// (nothing launched) for an ILU(0) smoother.
bool launch_cg_update_smooth(int64_t nrows, CgScalars *sc, const double *q, double *r,
                             const Smoother &M, double *z0, double *partials, int what,
                             cudaGraphConditionalHandle h, cudaStream_t s);
// u += alpha p_old; p = z + beta p_old
void launch_p_update_u(int64_t n, const CgScalars *sc, const double *z, double *p, double *u,
                       cudaStream_t s);
// u += alpha p
void launch_u_update(int64_t n, const CgScalars *sc, const double *p, double *u, cudaStream_t s);
// f = R r fused with u = M f (next level's first sweep from zero); false
// (nothing launched) for an ILU(0) smoother
bool launch_restrict_smooth(const Bsr3 &R, const double *r, double *f, const Smoother &M, double *u,
                            cudaStream_t s, bool lowp = false);
void launch_fill(int64_t n, double v, double *x, cudaStream_t s);

// ---- V-cycle tail (solve.cu): the small levels in one persistent launch ----
// One phase = one of the V-cycle's level operations on the small levels
// (hierarchy.hpp:418-440), executed by every CTA of a cooperative grid with a
// grid barrier between consecutive phases.
enum VPhaseKind {
    VP_SPMV = 0,      // out = alpha A x + beta out
    VP_RESIDUAL = 1,  // out = f - A x
    VP_SMOOTH_B = 2,  // out = x + M_row (f - A x)_row   (3x3 M_i)
    VP_SMOOTH_P = 3,  // out = x + m .* (f - A x)        (point)
    VP_RSMOOTH_B = 4, // out = A x (restriction), out2 = M_row out_row (next level's first sweep)
    VP_RSMOOTH_P = 5,
    VP_GEMV = 6,      // out = Ainv x (dense, row-major, leading dimension ld), nrows = n
    VP_FILL = 7,      // out[0 .. 3 nrows) = alpha
};
struct VPhase {
    int kind, G, nrows, last_out;  // last_out: out is the launch's final_out argument
    const int *ptr, *col;
    const double *val, *x, *f, *m;
    double *out, *out2;
    double alpha, beta;
    long long ld;
};
// lanes per block row for a tail phase over `threads` resident threads
int vtail_group(int64_t nrows, int64_t nnzb, int64_t threads);
// resident CTAs of the tail kernel (0: cooperative launch not possible)
int vtail_grid(size_t smem);
void launch_vtail(const VPhase *d_ph, int nph, unsigned *bar, int grid, size_t smem, int64_t gemv_ld,
                  double *final_out, cudaStream_t s, unsigned long long *trace = nullptr);

// generic PCG with caller operators (cgop.cu, cg.hpp:39-83)
samg_solve_report cg_solve_op(int64_t n, samg_apply_fn apply_A, samg_apply_fn apply_M, void *ctx,
                              const double *d_f, double *d_u, const samg_cg_params &prm,
                              cudaStream_t s);

// ---- setup phase (setup.cu, compiled with --fmad=false) ----------------------
struct Graph {  // node adjacency, symmetric, sorted rows (coarsening.hpp:33-38)
    int64_t nnodes = 0, nedges = 0;
    DevBuf<int> ptr, col;
};

// scalar CSR (int64 on host layout) uploaded -> BSR3 (csr.hpp:268-324)
void scalar_to_bsr3(int64_t n, const int64_t *d_ptr, const int64_t *d_col, const double *d_val,
                    Bsr3 &out, cudaStream_t s);
// the same from 32-bit column indices (samg_setup narrows them on upload)
void scalar_to_bsr3(int64_t n, const int64_t *d_ptr, const int32_t *d_col, const double *d_val,
                    Bsr3 &out, cudaStream_t s);
// strength graph on nodes of h block rows (coarsening.hpp:52-123); tile
// weight max|a| of the scalar view, or with fnorm (the block pipeline's
// csr<block3> strength, pbs 1) the block's Frobenius norm
void strength_graph(const Bsr3 &A, int h, double eps_strong, Graph &G, cudaStream_t s,
                    bool fnorm = false);
// aggregation (coarsening.hpp:131-160); returns the aggregate count
// seedno (optional out): #pass-1 seeds before each node, nnodes+1 entries
int64_t aggregate(const Graph &G, DevBuf<int> &agg, cudaStream_t s, DevBuf<int> *seedno = nullptr);
// tentative prolongation with QR of the nullspace (coarsening.hpp:238-312):
// Pt[nfine*k] row values (columns agg*k + c), Bc column-major (naggs*k)-by-k
// [a0, a1): only these aggregates (the distributed setup's own; B must
// hold their nodes' rows); Pt / Bc keep the global layout
void tentative(const DevBuf<int> &agg, int64_t nnodes, int64_t naggs, int pbs, const double *B,
               int k, DevBuf<double> &Pt, DevBuf<double> &Bc, DevError *err, cudaStream_t s,
               int64_t a0 = 0, int64_t a1 = -1);
// smoothed prolongation in scalar semantics, emitted as BSR3
// (coarsening.hpp:319-416 + to_block<3>)
// the `scalar` pipeline's tentative operator (no nullspace): the unit
// aggregate indicator per point-block component, one value per scalar row
// (coarsening.hpp:249-266); smooth it with k = 0
void tentative_indicator(const DevBuf<int> &agg, int64_t nnodes, int64_t naggs, int pbs,
                         DevBuf<double> &Pt1, cudaStream_t s);
// [node0, node1): only these nodes' rows of P (local row numbering; A in
// global numbering holding at least their rows).  k == 0: Pt is the
// indicator of tentative_indicator (pbs 3)
void smooth_prolongation(const Bsr3 &A, const Graph &G, const DevBuf<int> &agg, int64_t naggs,
                         int pbs, int k, const double *Pt, double omega, Bsr3 &P, DevError *err,
                         cudaStream_t s, int64_t node0 = 0, int64_t node1 = -1);
// block pipeline transfer (block_transfer_operators, coarsening.hpp:471-560):
// identity-block tentative scaled by 1/sqrt(|aggregate|), smoothed with the
// inverse of the lumped filtered block diagonal; P is n-by-naggs blocks
void block_transfer(const Bsr3 &A, const Graph &G, const DevBuf<int> &agg, int64_t naggs,
                    double omega, Bsr3 &P, DevError *err, cudaStream_t s, int64_t r0 = 0,
                    int64_t r1 = -1);
// R = P^T with transposed blocks (csr.hpp:173-194)
void transpose(const Bsr3 &P, Bsr3 &R, cudaStream_t s);
// C = A*B in the reference's order (csr.hpp:199-255): block arithmetic
// (csr<block3>), or with scalar_order the scalar product of the full-block
// scalar views (csr<double>: every scalar term added to the accumulator in
// (ja, q) order) -- the hybrids' scalar Galerkin, hierarchy.hpp:233-260
void spgemm(const Bsr3 &A, const Bsr3 &B, Bsr3 &C, cudaStream_t s, bool scalar_order = false);
// A_c = (R A) P with R = P^T exactly (the hierarchy's transfer operators)
void galerkin(const Bsr3 &R, const Bsr3 &A, const Bsr3 &P, Bsr3 &Ac, cudaStream_t s,
              bool scalar_order = false);
// rows of (Rl A) P for a row slice Rl of R (P's columns read through R);
// subset: A / P / R hold only the rows these products touch (global
// numbering, other rows empty; the distributed setup)
void galerkin_rows(const Bsr3 &Rl, const Bsr3 &A, const Bsr3 &P, const Bsr3 &R, Bsr3 &Ac,
                   cudaStream_t s, bool scalar_order = false, bool subset = false);
// rows [r0, r1) of M as a matrix of their own
void slice_rows(const Bsr3 &M, int64_t r0, int64_t r1, Bsr3 &out, cudaStream_t s);
// row0: global id of A's local row 0 (a row slice: the diagonal is row0 + i)
void fix_decoupled_rows(Bsr3 &A, cudaStream_t s, int64_t row0 = 0);
// sum over the union pattern of (A - G)^2 and of G^2 (the Galerkin
// consistency check, hierarchy.hpp:382-401); out[0] = diff, out[1] = ref
void union_diff(const Bsr3 &A, const Bsr3 &G, double out[2], cudaStream_t s);
// smoother setup: kind SAMG_SMOOTHER_*
void setup_smoother(const Bsr3 &A, int kind, double omega, Smoother &M, DevError *err,
                    cudaStream_t s, int64_t row0 = 0);
// block ILU(0) (ilu.cu): factorization, and one smoothing application
// u_out = u_in + (LU)^-1 (f - A u_in)  (u_in == nullptr: zero guess, r = f)
void setup_ilu0(const Bsr3 &A, Smoother &M, DevError *err, cudaStream_t s);
// ilu0<double> (relaxation.hpp:20-139 with V = double) of the scalar view of
// A (whole 3x3 blocks: the scalar pattern is the blocks' entries)
void setup_ilu0_scalar(const Bsr3 &A, Smoother &M, DevError *err, cudaStream_t s);
void launch_ilu_smooth(const Bsr3 *A, const Smoother &M, const double *f, const double *u_in,
                       double *u_out, cudaStream_t s, bool lowp = false);
// coarsest level: dense inverse (row-major n x n), n = 3*A.nrows
// false: a Gauss-Jordan pivot of the equilibrated matrix fell below 1e-300
// (numerically singular; Ainv is then garbage -- fall back to the LU)
bool dense_inverse(const Bsr3 &A, DevBuf<double> &Ainv, DevError *err, cudaStream_t s);
// the reference's dense_lu (hierarchy.hpp:86-129), bit-exact (coarse_lu.cu):
// for numerically singular coarse operators, where the explicit inverse and
// the LU solve disagree
constexpr int64_t kLuMaxN = 2048;
struct CoarseLu {
    int64_t n = 0;
    DevBuf<double> X;        // row-major n x n: unit L below, U on and above the diagonal
    DevBuf<double> Lt;       // L column-major (forward sweep)
    DevBuf<int64_t> perm;    // composed row swaps: (P f)[k] = f[perm[k]]
};
void dense_lu_ref(const Bsr3 &A, CoarseLu &lu, DevError *err, cudaStream_t s);
void launch_lu_solve(const CoarseLu &lu, const double *f, double *u, cudaStream_t s);

// throws the first device-side error, if any (synchronises s)
void check_dev_error(DevError *err, cudaStream_t s);

} // namespace samgb
