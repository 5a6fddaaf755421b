/*
 * samg_oracle.c -- CPU restatement of the reference SA-AMG NS-Block path.
 *
 * TEST INFRASTRUCTURE ONLY (see samg_oracle.h).  Every function names the
 * reference file:line it follows; paths are relative to
 * /root/reference/proj/include/samg/.  Loop orders and the order of every
 * floating-point sum are kept, so the setup is bit-identical to the
 * reference on identical input (pinned by tests/test_oracle_pins.py).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared (oracle/Makefile).
 */
#include "samg_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* error plumbing: typed errors (common.hpp:12-28) via longjmp to the API    */

static char g_err[512];
static jmp_buf *g_jmp;

const char *orc_last_error(void) { return g_err; }

static void fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    longjmp(*g_jmp, code);
}

#define API_BEGIN                       \
    jmp_buf jb__;                       \
    jmp_buf *prev__ = g_jmp;            \
    int code__ = setjmp(jb__);          \
    if (code__) { g_jmp = prev__; return code__; } \
    g_jmp = &jb__; g_err[0] = 0;
#define API_END do { g_jmp = prev__; return ORC_OK; } while (0)

static void *xmalloc(size_t n) {
    void *p = malloc(n ? n : 1);
    if (!p) fail(ORC_ERROR, "oracle: out of memory (%zu bytes)", n);
    return p;
}
static void *xcalloc(size_t n, size_t s) {
    void *p = calloc(n ? n : 1, s ? s : 1);
    if (!p) fail(ORC_ERROR, "oracle: out of memory");
    return p;
}

void orc_free(void *p) { free(p); }

static void mat_free(orc_mat *m) {
    free(m->ptr); free(m->col); free(m->val);
    memset(m, 0, sizeof *m);
}

static int64_t nnz_of(const orc_mat *m) { return m->ptr[m->nrows]; }

void orc_default_params(orc_params *p) {
    p->eps_strong = 0.08;          /* coarsening.hpp:27 */
    p->omega = 2.0 / 3.0;          /* coarsening.hpp:28 */
    p->smoother = ORC_SM_SPAI0;
    p->smoother_omega = 0.72;      /* relaxation.hpp:143 */
    p->pre_sweeps = 1;             /* hierarchy.hpp:53-54 */
    p->post_sweeps = 1;
    p->coarse_enough = 3000;       /* hierarchy.hpp:55 */
    p->stagnation_ratio = 0.8;     /* hierarchy.hpp:56 */
    p->pipeline = ORC_PIPELINE_NS_BLOCK;
}

/* ------------------------------------------------------------------------ */
/* 3x3 block arithmetic (static_block.hpp)                                   */

/* operator* (static_block.hpp:104-113): r = 0; r(i,j) += a(i,k)*b(k,j),
 * loop order i, k, j. */
static void blk_mul(const double *a, const double *b, double *r) {
    for (int e = 0; e < 9; ++e) r[e] = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) {
            const double aik = a[i * 3 + k];
            for (int j = 0; j < 3; ++j) r[i * 3 + j] += aik * b[k * 3 + j];
        }
}

/* inverse (static_block.hpp:155-194): LU with partial pivoting. */
static void blk_inverse(const double *a, double *inv) {
    double lu[9];
    int piv[3];
    memcpy(lu, a, sizeof lu);
    for (int k = 0; k < 3; ++k) {
        int p = k;
        for (int i = k + 1; i < 3; ++i)
            if (fabs(lu[i * 3 + k]) > fabs(lu[p * 3 + k])) p = i;
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < 3; ++j) {
                double t = lu[k * 3 + j]; lu[k * 3 + j] = lu[p * 3 + j]; lu[p * 3 + j] = t;
            }
        if (fabs(lu[k * 3 + k]) < 1e-300)
            fail(ORC_SINGULAR_BLOCK, "singular pivot in block inversion");
        const double d = 1.0 / lu[k * 3 + k];
        for (int i = k + 1; i < 3; ++i) {
            const double l = lu[i * 3 + k] * d;
            lu[i * 3 + k] = l;
            for (int j = k + 1; j < 3; ++j) lu[i * 3 + j] -= l * lu[k * 3 + j];
        }
    }
    for (int c = 0; c < 3; ++c) {
        double x[3] = {0.0, 0.0, 0.0};
        x[c] = 1.0;
        for (int k = 0; k < 3; ++k)
            if (piv[k] != k) { double t = x[k]; x[k] = x[piv[k]]; x[piv[k]] = t; }
        for (int i = 1; i < 3; ++i)
            for (int j = 0; j < i; ++j) x[i] -= lu[i * 3 + j] * x[j];
        for (int i = 2; i >= 0; --i) {
            for (int j = i + 1; j < 3; ++j) x[i] -= lu[i * 3 + j] * x[j];
            x[i] /= lu[i * 3 + i];
        }
        for (int i = 0; i < 3; ++i) inv[i * 3 + c] = x[i];
    }
}

/* ------------------------------------------------------------------------ */
/* level-1 kernels, scalar variant (kernels_scalar.cpp:5-28)                 */

static void axpby(double a, const double *x, double b, double *y, int64_t n) {
    if (b == 0.0) { for (int64_t i = 0; i < n; ++i) y[i] = a * x[i]; }
    else if (b == 1.0) { for (int64_t i = 0; i < n; ++i) y[i] += a * x[i]; }
    else { for (int64_t i = 0; i < n; ++i) y[i] = a * x[i] + b * y[i]; }
}

static double dot(const double *x, const double *y, int64_t n) {
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int64_t i = 0;
    for (; i + 4 <= n; i += 4) {
        s0 += x[i + 0] * y[i + 0];
        s1 += x[i + 1] * y[i + 1];
        s2 += x[i + 2] * y[i + 2];
        s3 += x[i + 3] * y[i + 3];
    }
    for (; i < n; ++i) s0 += x[i] * y[i];
    return (s0 + s1) + (s2 + s3);
}

static double norm2(const double *x, int64_t n) { return sqrt(dot(x, x, n)); }

/* ------------------------------------------------------------------------ */
/* sparse kernels (csr.hpp)                                                  */

/* spmv (csr.hpp:129-160): s[r] += blk(r,c)*x[col*b+c]; y = a*s + (b?b*y:0). */
static void spmv(double alpha, const orc_mat *A, const double *x, double beta,
        double *y) {
    const int b = A->b;
    for (int64_t i = 0; i < A->nrows; ++i) {
        double s[3] = {0.0, 0.0, 0.0};
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) {
            const double *blk = A->val + j * b * b;
            const double *xs = x + A->col[j] * b;
            for (int r = 0; r < b; ++r)
                for (int c = 0; c < b; ++c) s[r] += blk[r * b + c] * xs[c];
        }
        for (int r = 0; r < b; ++r) {
            double *yi = y + i * b + r;
            *yi = alpha * s[r] + (beta == 0.0 ? 0.0 : beta * *yi);
        }
    }
}

/* residual (csr.hpp:163-169) */
static void residual(const orc_mat *A, const double *f, const double *u,
        double *r) {
    memcpy(r, f, sizeof(double) * A->nrows * A->b);
    spmv(-1.0, A, u, 1.0, r);
}

/* transpose (csr.hpp:173-194): counting sort, blocks transposed. */
static orc_mat transpose(const orc_mat *A) {
    const int b = A->b, bb = b * b;
    const int64_t nnz = nnz_of(A);
    orc_mat T = {A->ncols, A->nrows, b, NULL, NULL, NULL};
    T.ptr = xcalloc(T.nrows + 1, sizeof(int64_t));
    T.col = xmalloc(sizeof(int64_t) * nnz);
    T.val = xmalloc(sizeof(double) * nnz * bb);
    for (int64_t k = 0; k < nnz; ++k) T.ptr[A->col[k] + 1]++;
    for (int64_t i = 0; i < T.nrows; ++i) T.ptr[i + 1] += T.ptr[i];
    int64_t *head = xmalloc(sizeof(int64_t) * (T.nrows + 1));
    memcpy(head, T.ptr, sizeof(int64_t) * (T.nrows + 1));
    for (int64_t i = 0; i < A->nrows; ++i)
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) {
            const int64_t p = head[A->col[j]]++;
            T.col[p] = i;
            for (int r = 0; r < b; ++r)
                for (int c = 0; c < b; ++c)
                    T.val[p * bb + c * b + r] = A->val[j * bb + r * b + c];
        }
    free(head);
    return T;
}

static int cmp_i64(const void *a, const void *b) {
    const int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* spgemm (csr.hpp:199-255): symbolic marker pass, numeric pass with a dense
 * accumulator; first touch assigns the product, later touches add it, in
 * (ja ascending, jb ascending) order.  Block products per blk_mul. */
static orc_mat spgemm(const orc_mat *A, const orc_mat *B) {
    if (A->ncols != B->nrows)
        fail(ORC_DIMENSION_MISMATCH, "spgemm: inner dimensions disagree");
    const int b = A->b, bb = b * b;
    orc_mat C = {A->nrows, B->ncols, b, NULL, NULL, NULL};
    C.ptr = xcalloc(C.nrows + 1, sizeof(int64_t));
    int64_t *marker = xmalloc(sizeof(int64_t) * (B->ncols + 1));
    for (int64_t c = 0; c < B->ncols; ++c) marker[c] = -1;
    for (int64_t i = 0; i < A->nrows; ++i) {
        int64_t count = 0;
        for (int64_t ja = A->ptr[i]; ja < A->ptr[i + 1]; ++ja) {
            const int64_t k = A->col[ja];
            for (int64_t jb = B->ptr[k]; jb < B->ptr[k + 1]; ++jb) {
                const int64_t c = B->col[jb];
                if (marker[c] != i) { marker[c] = i; ++count; }
            }
        }
        C.ptr[i + 1] = count;
    }
    for (int64_t i = 0; i < C.nrows; ++i) C.ptr[i + 1] += C.ptr[i];
    const int64_t nnz = C.ptr[C.nrows];
    C.col = xmalloc(sizeof(int64_t) * nnz);
    C.val = xmalloc(sizeof(double) * nnz * bb);
    for (int64_t c = 0; c < B->ncols; ++c) marker[c] = -1;
    double *acc = xcalloc((size_t)B->ncols * bb, sizeof(double));
    double prod[9];
    for (int64_t i = 0; i < A->nrows; ++i) {
        const int64_t row_beg = C.ptr[i];
        int64_t row_end = row_beg;
        for (int64_t ja = A->ptr[i]; ja < A->ptr[i + 1]; ++ja) {
            const int64_t k = A->col[ja];
            const double *av = A->val + ja * bb;
            for (int64_t jb = B->ptr[k]; jb < B->ptr[k + 1]; ++jb) {
                const int64_t c = B->col[jb];
                const double *bv = B->val + jb * bb;
                if (b == 3) blk_mul(av, bv, prod);
                else prod[0] = av[0] * bv[0];
                double *ac = acc + c * bb;
                if (marker[c] < row_beg) {
                    marker[c] = row_end;
                    C.col[row_end] = c;
                    for (int e = 0; e < bb; ++e) ac[e] = prod[e];
                    ++row_end;
                } else {
                    for (int e = 0; e < bb; ++e) ac[e] += prod[e];
                }
            }
        }
        qsort(C.col + row_beg, (size_t)(row_end - row_beg), sizeof(int64_t), cmp_i64);
        for (int64_t j = row_beg; j < row_end; ++j)
            memcpy(C.val + j * bb, acc + C.col[j] * bb, sizeof(double) * bb);
    }
    free(acc);
    free(marker);
    return C;
}

/* galerkin (csr.hpp:259-262) = spgemm(spgemm(R, A), P) */
static orc_mat galerkin(const orc_mat *R, const orc_mat *A, const orc_mat *P) {
    orc_mat RA = spgemm(R, A);
    orc_mat C = spgemm(&RA, P);
    mat_free(&RA);
    return C;
}

/* to_block<3> (csr.hpp:268-324): tiles with any scalar entry become blocks,
 * absent positions zero-filled, block columns sorted. */
static orc_mat to_block3(const orc_mat *A) {
    if (A->nrows % 3 || A->ncols % 3)
        fail(ORC_NOT_DIVISIBLE, "to_block: matrix dimensions not divisible by block size");
    orc_mat R = {A->nrows / 3, A->ncols / 3, 3, NULL, NULL, NULL};
    R.ptr = xcalloc(R.nrows + 1, sizeof(int64_t));
    int64_t *marker = xmalloc(sizeof(int64_t) * (R.ncols + 1));
    for (int64_t c = 0; c < R.ncols; ++c) marker[c] = -1;
    for (int64_t bi = 0; bi < R.nrows; ++bi) {
        int64_t count = 0;
        for (int r = 0; r < 3; ++r) {
            const int64_t i = bi * 3 + r;
            for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) {
                const int64_t bc = A->col[j] / 3;
                if (marker[bc] != bi) { marker[bc] = bi; ++count; }
            }
        }
        R.ptr[bi + 1] = count;
    }
    for (int64_t i = 0; i < R.nrows; ++i) R.ptr[i + 1] += R.ptr[i];
    const int64_t nnz = R.ptr[R.nrows];
    R.col = xmalloc(sizeof(int64_t) * nnz);
    R.val = xcalloc((size_t)nnz * 9, sizeof(double));
    int64_t *pos = xmalloc(sizeof(int64_t) * (R.ncols + 1));
    for (int64_t c = 0; c < R.ncols; ++c) marker[c] = -1;
    for (int64_t bi = 0; bi < R.nrows; ++bi) {
        const int64_t row_beg = R.ptr[bi];
        int64_t row_end = row_beg;
        for (int r = 0; r < 3; ++r) {
            const int64_t i = bi * 3 + r;
            for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) {
                const int64_t bc = A->col[j] / 3;
                if (marker[bc] != bi) { marker[bc] = bi; R.col[row_end++] = bc; }
            }
        }
        qsort(R.col + row_beg, (size_t)(row_end - row_beg), sizeof(int64_t), cmp_i64);
        for (int64_t j = row_beg; j < row_end; ++j) pos[R.col[j]] = j;
        for (int r = 0; r < 3; ++r) {
            const int64_t i = bi * 3 + r;
            for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) {
                const int64_t bc = A->col[j] / 3;
                R.val[pos[bc] * 9 + r * 3 + (A->col[j] % 3)] = A->val[j];
            }
        }
    }
    free(pos);
    free(marker);
    return R;
}

/* to_scalar<3> (csr.hpp:327-353): every block expands to 9 entries. */
static orc_mat to_scalar(const orc_mat *A) {
    const int64_t nnzb = nnz_of(A);
    orc_mat R = {A->nrows * 3, A->ncols * 3, 1, NULL, NULL, NULL};
    R.ptr = xmalloc(sizeof(int64_t) * (R.nrows + 1));
    R.col = xmalloc(sizeof(int64_t) * nnzb * 9);
    R.val = xmalloc(sizeof(double) * nnzb * 9);
    R.ptr[0] = 0;
    int64_t out = 0;
    for (int64_t bi = 0; bi < A->nrows; ++bi)
        for (int r = 0; r < 3; ++r) {
            for (int64_t j = A->ptr[bi]; j < A->ptr[bi + 1]; ++j) {
                const double *blk = A->val + j * 9;
                for (int c = 0; c < 3; ++c) {
                    R.col[out] = A->col[j] * 3 + c;
                    R.val[out] = blk[r * 3 + c];
                    ++out;
                }
            }
            R.ptr[bi * 3 + r + 1] = out;
        }
    return R;
}

/* ------------------------------------------------------------------------ */
/* coarsening (coarsening.hpp)                                               */

typedef struct { int64_t c; double w; } cw_pair;
static int cmp_cw(const void *a, const void *b) {
    const int64_t x = ((const cw_pair *)a)->c, y = ((const cw_pair *)b)->c;
    return (x > y) - (x < y);
}

/* strength_graph for scalar matrices with point-block condensation
 * (coarsening.hpp:52-77 condense_weights, :81-123 strength_graph). */
/* For a block matrix (b = 3, the block pipeline) the node is the block row
 * and the weight the Frobenius norm of the block (condense_weights,
 * coarsening.hpp:55-62; fnorm, static_block.hpp:111-115). */
static orc_adj strength_graph(const orc_mat *A, double eps_strong, int pbs) {
    if (A->nrows != A->ncols)
        fail(ORC_NON_SQUARE, "strength_graph: matrix must be square");
    if (A->b == 3) pbs = 1;
    if (A->nrows % pbs)
        fail(ORC_NOT_DIVISIBLE, "strength_graph: rows not divisible by point block size");
    const int64_t n = A->nrows / pbs;
    const double eps2 = eps_strong * eps_strong;
    /* condensed weights: per node row, sorted (node col, max |a|) */
    int64_t *wptr = xcalloc(n + 1, sizeof(int64_t));
    cw_pair *w = xmalloc(sizeof(cw_pair) * (A->ptr[A->nrows] + 1));
    int64_t nw = 0;
    for (int64_t ni = 0; ni < n; ++ni) {
        const int64_t beg = nw;
        for (int r = 0; r < pbs; ++r) {
            const int64_t i = ni * pbs + r;
            for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) {
                w[nw].c = A->col[j] / pbs;
                if (A->b == 3) {
                    double sq = 0;
                    for (int e = 0; e < 9; ++e) sq += A->val[9 * j + e] * A->val[9 * j + e];
                    w[nw].w = sqrt(sq);
                } else {
                    w[nw].w = fabs(A->val[j]);
                }
                ++nw;
            }
        }
        qsort(w + beg, (size_t)(nw - beg), sizeof(cw_pair), cmp_cw);
        int64_t out = beg;
        for (int64_t k = beg; k < nw; ++k) {
            if (out > beg && w[out - 1].c == w[k].c) {
                if (w[k].w > w[out - 1].w) w[out - 1].w = w[k].w;
            } else {
                w[out++] = w[k];
            }
        }
        nw = out;
        wptr[ni + 1] = nw;
    }
    double *diag = xcalloc(n, sizeof(double));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = wptr[i]; k < wptr[i + 1]; ++k)
            if (w[k].c == i) diag[i] = w[k].w;
    /* edges pushed both ways (union symmetrisation), then sort + unique */
    int64_t *deg = xcalloc(n + 1, sizeof(int64_t));
    int64_t nedge = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = wptr[i]; k < wptr[i + 1]; ++k) {
            const int64_t j = w[k].c;
            if (j == i) continue;
            const double wij = w[k].w;
            if (wij * wij > eps2 * diag[i] * diag[j]) {
                deg[i + 1]++; deg[j + 1]++; nedge += 2;
            }
        }
    for (int64_t i = 0; i < n; ++i) deg[i + 1] += deg[i];
    int64_t *ecol = xmalloc(sizeof(int64_t) * (nedge + 1));
    int64_t *head = xmalloc(sizeof(int64_t) * (n + 1));
    memcpy(head, deg, sizeof(int64_t) * (n + 1));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = wptr[i]; k < wptr[i + 1]; ++k) {
            const int64_t j = w[k].c;
            if (j == i) continue;
            const double wij = w[k].w;
            if (wij * wij > eps2 * diag[i] * diag[j]) {
                ecol[head[i]++] = j;
                ecol[head[j]++] = i;
            }
        }
    orc_adj G = {n, NULL, NULL};
    G.ptr = xcalloc(n + 1, sizeof(int64_t));
    G.col = xmalloc(sizeof(int64_t) * (nedge + 1));
    int64_t out = 0;
    for (int64_t i = 0; i < n; ++i) {
        qsort(ecol + deg[i], (size_t)(deg[i + 1] - deg[i]), sizeof(int64_t), cmp_i64);
        for (int64_t k = deg[i]; k < deg[i + 1]; ++k)
            if (out == G.ptr[i] || G.col[out - 1] != ecol[k]) G.col[out++] = ecol[k];
        G.ptr[i + 1] = out;
    }
    free(head); free(ecol); free(deg); free(diag); free(w); free(wptr);
    return G;
}

/* aggregate (coarsening.hpp:131-160): greedy three-pass. */
static int64_t aggregate(const orc_adj *G, int64_t *id) {
    int64_t count = 0;
    for (int64_t i = 0; i < G->nnodes; ++i) id[i] = -1;
    for (int64_t i = 0; i < G->nnodes; ++i) {
        if (id[i] != -1) continue;
        int all_free = 1;
        for (int64_t j = G->ptr[i]; j < G->ptr[i + 1]; ++j)
            if (id[G->col[j]] != -1) { all_free = 0; break; }
        if (!all_free) continue;
        const int64_t a = count++;
        id[i] = a;
        for (int64_t j = G->ptr[i]; j < G->ptr[i + 1]; ++j) id[G->col[j]] = a;
    }
    for (int64_t i = 0; i < G->nnodes; ++i) {
        if (id[i] != -1) continue;
        for (int64_t j = G->ptr[i]; j < G->ptr[i + 1]; ++j) {
            const int64_t nb = G->col[j];
            if (id[nb] != -1) { id[i] = id[nb]; break; }
        }
    }
    for (int64_t i = 0; i < G->nnodes; ++i)
        if (id[i] == -1) id[i] = count++;
    return count;
}

/* thin_qr (coarsening.hpp:167-229): Householder, column-major m-by-k. */
static void thin_qr(int64_t m, int64_t k, double *A, double *Q, double *R,
        double drop_tol) {
#define a_(i, j) A[(j) * m + (i)]
    double local_max = 0;
    for (int64_t t = 0; t < m * k; ++t)
        if (fabs(A[t]) > local_max) local_max = fabs(A[t]);
    const double tol = 1e-12 * (local_max > 1.0 ? local_max : 1.0);
    double tau[64];
    for (int64_t j = 0; j < k; ++j) tau[j] = 0.0;
    const int64_t steps = m < k ? m : k;
    for (int64_t j = 0; j < steps; ++j) {
        double normx = 0;
        for (int64_t i = j; i < m; ++i) normx += a_(i, j) * a_(i, j);
        normx = sqrt(normx);
        if (normx <= tol) { tau[j] = 0; continue; }
        const double alpha = a_(j, j) >= 0 ? -normx : normx;
        const double v0 = a_(j, j) - alpha;
        for (int64_t i = j + 1; i < m; ++i) a_(i, j) /= v0;
        tau[j] = -v0 / alpha;
        a_(j, j) = alpha;
        for (int64_t c = j + 1; c < k; ++c) {
            double s = a_(j, c);
            for (int64_t i = j + 1; i < m; ++i) s += a_(i, j) * a_(i, c);
            s *= tau[j];
            a_(j, c) -= s;
            for (int64_t i = j + 1; i < m; ++i) a_(i, c) -= s * a_(i, j);
        }
    }
    for (int64_t t = 0; t < k * k; ++t) R[t] = 0.0;
    for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i <= (j < m - 1 ? j : m - 1); ++i) R[j * k + i] = a_(i, j);
    for (int64_t t = 0; t < m * k; ++t) Q[t] = 0.0;
    for (int64_t j = 0; j < (m < k ? m : k); ++j) Q[j * m + j] = 1.0;
    for (int64_t j = steps - 1; j >= 0; --j) {
        if (tau[j] == 0) continue;
        for (int64_t c = 0; c < k; ++c) {
            double s = Q[c * m + j];
            for (int64_t i = j + 1; i < m; ++i) s += a_(i, j) * Q[c * m + i];
            s *= tau[j];
            Q[c * m + j] -= s;
            for (int64_t i = j + 1; i < m; ++i) Q[c * m + i] -= s * a_(i, j);
        }
    }
    const double lm = local_max > 1e-300 ? local_max : 1e-300;
    for (int64_t j = 0; j < k; ++j) {
        const double rjj = (j < m) ? fabs(R[j * k + j]) : 0.0;
        if (rjj <= drop_tol * lm) {
            for (int64_t i = 0; i < m; ++i) Q[j * m + i] = 0.0;
            for (int64_t c = 0; c < k; ++c) R[c * k + j] = 0.0;
        }
    }
#undef a_
}

/* tentative_prolongation with nullspace (coarsening.hpp:238-312). B is
 * column-major nfine-by-k; Bc (out) column-major (count*k)-by-k. */
static orc_mat tentative(const int64_t *id, int64_t nnodes, int64_t count,
        const double *B, int64_t bnrows, int64_t k, int pbs, double **Bc_out) {
    const int64_t nfine = nnodes * pbs;
    if (bnrows != nfine)
        fail(ORC_BAD_NULLSPACE_SHAPE, "tentative_prolongation: nullspace rows do not match level size");
    if (k > 64) fail(ORC_BAD_NULLSPACE_SHAPE, "oracle: at most 64 nullspace columns");
    /* members per aggregate, ascending scalar rows (counting sort, stable) */
    int64_t *mptr = xcalloc(count + 1, sizeof(int64_t));
    for (int64_t n = 0; n < nnodes; ++n) mptr[id[n] + 1] += pbs;
    for (int64_t a = 0; a < count; ++a) mptr[a + 1] += mptr[a];
    int64_t *rows = xmalloc(sizeof(int64_t) * (nfine + 1));
    int64_t *head = xmalloc(sizeof(int64_t) * (count + 1));
    memcpy(head, mptr, sizeof(int64_t) * (count + 1));
    for (int64_t n = 0; n < nnodes; ++n)
        for (int c = 0; c < pbs; ++c) rows[head[id[n]]++] = n * pbs + c;
    orc_mat P = {nfine, count * k, 1, NULL, NULL, NULL};
    P.ptr = xmalloc(sizeof(int64_t) * (nfine + 1));
    P.ptr[0] = 0;
    for (int64_t i = 0; i < nfine; ++i) P.ptr[i + 1] = P.ptr[i] + k;
    P.col = xmalloc(sizeof(int64_t) * nfine * k);
    P.val = xmalloc(sizeof(double) * nfine * k);
    double *Bc = xcalloc((size_t)count * k * k, sizeof(double));
    const int64_t bcn = count * k;
    int64_t maxm = 0;
    for (int64_t a = 0; a < count; ++a)
        if (mptr[a + 1] - mptr[a] > maxm) maxm = mptr[a + 1] - mptr[a];
    double *local = xmalloc(sizeof(double) * maxm * k);
    double *Q = xmalloc(sizeof(double) * maxm * k);
    double R[64 * 64];
    for (int64_t a = 0; a < count; ++a) {
        const int64_t *rw = rows + mptr[a];
        const int64_t m = mptr[a + 1] - mptr[a];
        for (int64_t c = 0; c < k; ++c)
            for (int64_t r = 0; r < m; ++r) local[c * m + r] = B[c * bnrows + rw[r]];
        thin_qr(m, k, local, Q, R, 1e-12);
        for (int64_t r = 0; r < m; ++r) {
            const int64_t base = P.ptr[rw[r]];
            for (int64_t c = 0; c < k; ++c) {
                P.col[base + c] = a * k + c;
                P.val[base + c] = Q[c * m + r];
            }
        }
        for (int64_t i = 0; i < k; ++i)
            for (int64_t c = 0; c < k; ++c) Bc[c * bcn + a * k + i] = R[c * k + i];
    }
    free(Q); free(local); free(head); free(rows); free(mptr);
    *Bc_out = Bc;
    return P;
}

/* smooth_prolongation, scalar value type (coarsening.hpp:319-416). */
static orc_mat smooth_prolongation(const orc_mat *A, const orc_mat *Pt,
        const orc_adj *G, double omega, int pbs) {
    if (omega == 0.0) {
        orc_mat P = *Pt;
        const int64_t nnz = nnz_of(Pt);
        P.ptr = xmalloc(sizeof(int64_t) * (Pt->nrows + 1));
        P.col = xmalloc(sizeof(int64_t) * (nnz + 1));
        P.val = xmalloc(sizeof(double) * (nnz + 1));
        memcpy(P.ptr, Pt->ptr, sizeof(int64_t) * (Pt->nrows + 1));
        memcpy(P.col, Pt->col, sizeof(int64_t) * nnz);
        memcpy(P.val, Pt->val, sizeof(double) * nnz);
        return P;
    }
    const int64_t n = A->nrows;
    int64_t *marker = xmalloc(sizeof(int64_t) * (G->nnodes + 1));
    for (int64_t i = 0; i < G->nnodes; ++i) marker[i] = -1;
    double *diag = xcalloc(n, sizeof(double));
    char *keep = xcalloc(nnz_of(A) + 1, 1);
    for (int64_t node = 0; node < G->nnodes; ++node) {
        for (int64_t j = G->ptr[node]; j < G->ptr[node + 1]; ++j) marker[G->col[j]] = node;
        for (int r = 0; r < pbs; ++r) {
            const int64_t i = node * pbs + r;
            for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) {
                const int64_t cnode = A->col[j] / pbs;
                if (cnode == node) {
                    keep[j] = 1;
                    if (A->col[j] == i) diag[i] += A->val[j];
                } else if (marker[cnode] == node) {
                    keep[j] = 1;
                } else {
                    diag[i] += A->val[j];
                }
            }
        }
    }
    double *inv_diag = xmalloc(sizeof(double) * (n + 1));
    for (int64_t i = 0; i < n; ++i) {
        if (diag[i] == 0.0)
            fail(ORC_ZERO_DIAGONAL, "smooth_prolongation: zero filtered diagonal");
        if (fabs(diag[i]) < 1e-300) fail(ORC_SINGULAR_BLOCK, "singular scalar pivot");
        inv_diag[i] = 1.0 / diag[i];
    }
    orc_mat P = {A->nrows, Pt->ncols, 1, NULL, NULL, NULL};
    P.ptr = xcalloc(P.nrows + 1, sizeof(int64_t));
    int64_t *cmark = xmalloc(sizeof(int64_t) * (P.ncols + 1));
    for (int64_t c = 0; c < P.ncols; ++c) cmark[c] = -1;
    for (int64_t i = 0; i < n; ++i) {
        int64_t count = 0;
        for (int64_t j = Pt->ptr[i]; j < Pt->ptr[i + 1]; ++j)
            if (cmark[Pt->col[j]] != i) { cmark[Pt->col[j]] = i; ++count; }
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) {
            if (!keep[j]) continue;
            const int64_t k = A->col[j];
            for (int64_t l = Pt->ptr[k]; l < Pt->ptr[k + 1]; ++l)
                if (cmark[Pt->col[l]] != i) { cmark[Pt->col[l]] = i; ++count; }
        }
        P.ptr[i + 1] = count;
    }
    for (int64_t i = 0; i < P.nrows; ++i) P.ptr[i + 1] += P.ptr[i];
    const int64_t nnz = P.ptr[P.nrows];
    P.col = xmalloc(sizeof(int64_t) * (nnz + 1));
    P.val = xmalloc(sizeof(double) * (nnz + 1));
    for (int64_t c = 0; c < P.ncols; ++c) cmark[c] = -1;
    double *acc = xcalloc(P.ncols + 1, sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        const int64_t row_beg = P.ptr[i];
        int64_t row_end = row_beg;
        for (int64_t j = Pt->ptr[i]; j < Pt->ptr[i + 1]; ++j) {
            const int64_t c = Pt->col[j];
            cmark[c] = row_end;
            P.col[row_end++] = c;
            acc[c] = Pt->val[j];
        }
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) {
            if (!keep[j]) continue;
            const int64_t k = A->col[j];
            const double coef = (k == i) ? diag[i] : A->val[j];
            double scaled = inv_diag[i] * coef;
            scaled *= -omega;
            for (int64_t l = Pt->ptr[k]; l < Pt->ptr[k + 1]; ++l) {
                const int64_t c = Pt->col[l];
                if (cmark[c] < row_beg) {
                    cmark[c] = row_end;
                    P.col[row_end++] = c;
                    acc[c] = scaled * Pt->val[l];
                } else {
                    acc[c] += scaled * Pt->val[l];
                }
            }
        }
        qsort(P.col + row_beg, (size_t)(row_end - row_beg), sizeof(int64_t), cmp_i64);
        for (int64_t j = row_beg; j < row_end; ++j) P.val[j] = acc[P.col[j]];
    }
    free(acc); free(cmark); free(inv_diag); free(keep); free(diag); free(marker);
    return P;
}

/* ------------------------------------------------------------------------ */
/* hierarchy (hierarchy.hpp)                                                 */

/* fix_decoupled_rows (hierarchy.hpp:172-191), 3x3 blocks */
static void fix_decoupled_rows(orc_mat *A) {
    const int b = A->b, bb = b * b;
    for (int64_t i = 0; i < A->nrows; ++i) {
        int64_t dg = -1;
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j)
            if (A->col[j] == i) { dg = j; break; }
        for (int r = 0; r < b; ++r) {
            int zero_row = 1;
            for (int64_t j = A->ptr[i]; zero_row && j < A->ptr[i + 1]; ++j)
                for (int c = 0; c < b; ++c)
                    if (A->val[j * bb + r * b + c] != 0.0) { zero_row = 0; break; }
            if (zero_row && dg >= 0) A->val[dg * bb + r * b + r] = 1.0;
        }
    }
}

typedef struct {
    orc_mat A, P, R;
    int has_transfer;
    int64_t *agg;      /* aggregates of this level's nodes */
    int64_t nnodes, naggs;
    double *sm;        /* smoother data: 3*nrows (point) or 9*nrows (block) */
    int64_t sm_len;
} orc_level;

struct orc_hier {
    orc_level *lv;
    int nlev;
    orc_params prm;
    int64_t nc;        /* coarsest dimension */
    double *lu;        /* dense LU, row-major */
    int64_t *piv;
};

/* damped_jacobi ctor for block matrices (relaxation.hpp:147-162). */
static void setup_point_jacobi(orc_level *L) {
    const orc_mat *A = &L->A;
    L->sm_len = A->nrows * 3;
    L->sm = xcalloc(L->sm_len, sizeof(double));
    for (int64_t i = 0; i < A->nrows; ++i)
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j)
            if (A->col[j] == i)
                for (int r = 0; r < 3; ++r) {
                    const double d = A->val[j * 9 + r * 3 + r];
                    if (d == 0.0) fail(ORC_ZERO_DIAGONAL, "jacobi: zero diagonal entry");
                    L->sm[i * 3 + r] = 1.0 / d;
                }
}

/* Block smoothers the reference lacks:
 *   SPAI0:        M_i = A_ii / sum_j sum_e A_ij[e]^2  (j, e ascending)
 *   BLOCK_JACOBI: M_i = omega * inverse(A_ii)  (inverse per
 *                 static_block.hpp:155-194). */
static void setup_block_smoother(orc_level *L, int kind, double omega) {
    const orc_mat *A = &L->A;
    L->sm_len = A->nrows * 9;
    L->sm = xcalloc(L->sm_len, sizeof(double));
    for (int64_t i = 0; i < A->nrows; ++i) {
        int64_t dg = -1;
        double den = 0.0;
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) {
            if (A->col[j] == i) dg = j;
            for (int e = 0; e < 9; ++e) den += A->val[j * 9 + e] * A->val[j * 9 + e];
        }
        if (dg < 0) fail(ORC_MISSING_DIAGONAL, "block smoother: structurally zero diagonal");
        double *M = L->sm + i * 9;
        if (kind == ORC_SM_SPAI0) {
            if (den == 0.0) fail(ORC_ZERO_DIAGONAL, "spai0: zero row");
            for (int e = 0; e < 9; ++e) M[e] = A->val[dg * 9 + e] / den;
        } else {
            double inv[9];
            blk_inverse(A->val + dg * 9, inv);
            for (int e = 0; e < 9; ++e) M[e] = omega * inv[e];
        }
    }
}

/* block_transfer_operators (coarsening.hpp:466-499) for the block pipeline:
 * indicator tentative operator with identity blocks scaled by
 * 1/sqrt(|aggregate|), smoothed with block diagonal inverses
 * (smooth_prolongation<block3>, coarsening.hpp:320-411, pbs = 1). */
static orc_mat block_transfer(const orc_mat *A, const orc_adj *G, const int64_t *agg,
                              int64_t naggs, double omega) {
    const int64_t n = A->nrows;
    int64_t *cnt = xcalloc(naggs + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) cnt[agg[i]]++;
    double *pv = xmalloc(sizeof(double) * (naggs + 1));
    for (int64_t g = 0; g < naggs; ++g) pv[g] = 1.0 / sqrt((double)cnt[g]);
    free(cnt);
    /* tentative blocks v*I (operator*(double, block): v*1, v*0) */
    double *ptb = xmalloc(sizeof(double) * 9 * (n + 1));
    for (int64_t i = 0; i < n; ++i)
        for (int e = 0; e < 9; ++e) ptb[9 * i + e] = pv[agg[i]] * ((e % 4 == 0) ? 1.0 : 0.0);
    free(pv);
    orc_mat P = {n, naggs, 3, xcalloc(n + 1, sizeof(int64_t)), NULL, NULL};
    if (omega == 0.0) {  /* return P_tent */
        P.col = xmalloc(sizeof(int64_t) * (n + 1));
        P.val = ptb;
        for (int64_t i = 0; i < n; ++i) { P.ptr[i + 1] = i + 1; P.col[i] = agg[i]; }
        return P;
    }
    int64_t *marker = xmalloc(sizeof(int64_t) * (n + 1));
    for (int64_t i = 0; i < n; ++i) marker[i] = -1;
    const int64_t nnz = A->ptr[n];
    char *keep = xcalloc(nnz + 1, 1);
    double *diag = xcalloc(9 * (n + 1), sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = G->ptr[i]; j < G->ptr[i + 1]; ++j) marker[G->col[j]] = i;
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) {
            const int64_t c = A->col[j];
            if (c == i) {
                keep[j] = 1;
                for (int e = 0; e < 9; ++e) diag[9 * i + e] += A->val[9 * j + e];
            } else if (marker[c] == i) {
                keep[j] = 1;
            } else {
                for (int e = 0; e < 9; ++e) diag[9 * i + e] += A->val[9 * j + e];
            }
        }
    }
    double *inv = xmalloc(sizeof(double) * 9 * (n + 1));
    for (int64_t i = 0; i < n; ++i) {
        int zero = 1;
        for (int e = 0; e < 9; ++e) if (diag[9 * i + e] != 0.0) zero = 0;
        if (zero) fail(ORC_ZERO_DIAGONAL, "smooth_prolongation: zero filtered diagonal");
        blk_inverse(diag + 9 * i, inv + 9 * i);
    }
    /* rows: P_tent column first, then kept entries in order; first touch
     * assigns the product, later touches add it; columns sorted */
    int64_t cap = 0;
    for (int64_t i = 0; i < n; ++i) cap += 1 + (A->ptr[i + 1] - A->ptr[i]);
    P.col = xmalloc(sizeof(int64_t) * (cap + 1));
    P.val = xmalloc(sizeof(double) * 9 * (cap + 1));
    int64_t out = 0;
    int64_t rc[64];
    double racc[64 * 9];
    for (int64_t i = 0; i < n; ++i) {
        int m = 0;
        rc[m] = agg[i];
        memcpy(racc, ptb + 9 * i, sizeof(double) * 9);
        ++m;
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) {
            if (!keep[j]) continue;
            const int64_t k = A->col[j];
            const double *coef = (k == i) ? diag + 9 * i : A->val + 9 * j;
            double scaled[9], prod[9];
            blk_mul(inv + 9 * i, coef, scaled);
            for (int e = 0; e < 9; ++e) scaled[e] *= -omega;
            blk_mul(scaled, ptb + 9 * k, prod);
            const int64_t c = agg[k];
            int at = -1;
            for (int t = 0; t < m; ++t) if (rc[t] == c) { at = t; break; }
            if (at < 0) {
                if (m == 64) fail(ORC_ERROR, "block_transfer: row too long");
                rc[m] = c;
                memcpy(racc + 9 * m, prod, sizeof prod);
                ++m;
            } else {
                for (int e = 0; e < 9; ++e) racc[9 * at + e] += prod[e];
            }
        }
        /* sort the row's columns (insertion sort, <= 64 entries) */
        for (int a = 1; a < m; ++a)
            for (int b2 = a; b2 > 0 && rc[b2 - 1] > rc[b2]; --b2) {
                int64_t t = rc[b2]; rc[b2] = rc[b2 - 1]; rc[b2 - 1] = t;
                double tv[9];
                memcpy(tv, racc + 9 * b2, sizeof tv);
                memcpy(racc + 9 * b2, racc + 9 * (b2 - 1), sizeof tv);
                memcpy(racc + 9 * (b2 - 1), tv, sizeof tv);
            }
        for (int t = 0; t < m; ++t) {
            P.col[out] = rc[t];
            memcpy(P.val + 9 * out, racc + 9 * t, sizeof(double) * 9);
            ++out;
        }
        P.ptr[i + 1] = out;
    }
    free(marker); free(keep); free(diag); free(inv); free(ptb);
    return P;
}

/* ilu0<block3> ctor (relaxation.hpp:103-136): IKJ elimination restricted
 * to A's pattern, L_ik = A_ik * inverse(U_kk), inverted pivots.  The
 * smoother data is [factors (9*nnz) | inverted pivots (9*nrows)]. */
static void setup_ilu0(orc_level *L) {
    const orc_mat *A = &L->A;
    const int64_t n = A->nrows, nnz = A->ptr[n];
    if (A->nrows != A->ncols) fail(ORC_NON_SQUARE, "ilu0: matrix must be square");
    L->sm_len = 9 * (nnz + n);
    L->sm = xcalloc(L->sm_len, sizeof(double));
    double *lu = L->sm, *inv = L->sm + 9 * nnz;
    memcpy(lu, A->val, sizeof(double) * 9 * nnz);
    int64_t *dpos = xmalloc(sizeof(int64_t) * (n + 1)), *pos = xmalloc(sizeof(int64_t) * (n + 1));
    for (int64_t i = 0; i < n; ++i) {
        dpos[i] = -1;
        pos[i] = -1;
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j)
            if (A->col[j] == i) dpos[i] = j;
    }
    for (int64_t i = 0; i < n; ++i)
        if (dpos[i] < 0) fail(ORC_MISSING_DIAGONAL, "ilu0: structurally zero diagonal");
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) pos[A->col[j]] = j;
        for (int64_t j = A->ptr[i]; j < dpos[i]; ++j) {
            const int64_t k = A->col[j];
            double lik[9], prod[9];
            blk_mul(lu + 9 * j, inv + 9 * k, lik);
            memcpy(lu + 9 * j, lik, sizeof lik);
            for (int64_t l = dpos[k] + 1; l < A->ptr[k + 1]; ++l) {
                const int64_t q = pos[A->col[l]];
                if (q < 0) continue;
                blk_mul(lik, lu + 9 * l, prod);
                for (int e = 0; e < 9; ++e) lu[9 * q + e] -= prod[e];
            }
        }
        blk_inverse(lu + 9 * dpos[i], inv + 9 * i);
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j) pos[A->col[j]] = -1;
    }
    free(dpos);
    free(pos);
}

/* ilu0::solve_in_place (relaxation.hpp:44-88): forward with the unit lower
 * factor, backward with the upper factor and the inverted pivots. */
static void ilu0_solve(const orc_level *L, double *r) {
    const orc_mat *A = &L->A;
    const int64_t n = A->nrows, nnz = A->ptr[n];
    const double *lu = L->sm, *inv = L->sm + 9 * nnz;
    for (int64_t i = 0; i < n; ++i) {
        double *ri = r + 3 * i;
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1] && A->col[j] < i; ++j) {
            const double *rj = r + 3 * A->col[j], *b = lu + 9 * j;
            for (int p = 0; p < 3; ++p)
                for (int q = 0; q < 3; ++q) ri[p] -= b[p * 3 + q] * rj[q];
        }
    }
    for (int64_t i = n - 1; i >= 0; --i) {
        double *ri = r + 3 * i;
        int64_t dg = -1;
        for (int64_t j = A->ptr[i]; j < A->ptr[i + 1]; ++j)
            if (A->col[j] == i) dg = j;
        for (int64_t j = dg + 1; j < A->ptr[i + 1]; ++j) {
            const double *rj = r + 3 * A->col[j], *b = lu + 9 * j;
            for (int p = 0; p < 3; ++p)
                for (int q = 0; q < 3; ++q) ri[p] -= b[p * 3 + q] * rj[q];
        }
        const double *d = inv + 9 * i;
        double t[3];
        for (int p = 0; p < 3; ++p) {
            t[p] = 0;
            for (int q = 0; q < 3; ++q) t[p] += d[p * 3 + q] * ri[q];
        }
        for (int p = 0; p < 3; ++p) ri[p] = t[p];
    }
}

/* dense_lu ctor (hierarchy.hpp:90-111) */
static void dense_lu_factor(orc_hier *H, const orc_mat *Ac) {
    orc_mat S = to_scalar(Ac);
    const int64_t n = S.nrows;
    H->nc = n;
    H->lu = xcalloc((size_t)n * n, sizeof(double));
    H->piv = xmalloc(sizeof(int64_t) * (n + 1));
    /* to_dense (csr.hpp:370-382) */
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = S.ptr[i]; j < S.ptr[i + 1]; ++j) H->lu[i * n + S.col[j]] = S.val[j];
    mat_free(&S);
    double *lu = H->lu;
    for (int64_t k = 0; k < n; ++k) {
        int64_t p = k;
        for (int64_t i = k + 1; i < n; ++i)
            if (fabs(lu[i * n + k]) > fabs(lu[p * n + k])) p = i;
        H->piv[k] = p;
        if (p != k)
            for (int64_t j = 0; j < n; ++j) {
                double t = lu[k * n + j]; lu[k * n + j] = lu[p * n + j]; lu[p * n + j] = t;
            }
        const double d = lu[k * n + k];
        if (fabs(d) < 1e-300) fail(ORC_ERROR, "dense_lu: singular coarse matrix");
        const double inv = 1.0 / d;
        for (int64_t i = k + 1; i < n; ++i) {
            const double l = lu[i * n + k] * inv;
            lu[i * n + k] = l;
            const double *rk = lu + k * n;
            double *ri = lu + i * n;
            for (int64_t j = k + 1; j < n; ++j) ri[j] -= l * rk[j];
        }
    }
}

/* dense_lu::solve (hierarchy.hpp:113-129) */
static void dense_lu_solve(const orc_hier *H, const double *f, double *u) {
    const int64_t n = H->nc;
    const double *lu = H->lu;
    memcpy(u, f, sizeof(double) * n);
    for (int64_t k = 0; k < n; ++k)
        if (H->piv[k] != k) { double t = u[k]; u[k] = u[H->piv[k]]; u[H->piv[k]] = t; }
    for (int64_t i = 1; i < n; ++i) {
        double s = u[i];
        const double *ri = lu + i * n;
        for (int64_t j = 0; j < i; ++j) s -= ri[j] * u[j];
        u[i] = s;
    }
    for (int64_t i = n - 1; i >= 0; --i) {
        double s = u[i];
        const double *ri = lu + i * n;
        for (int64_t j = i + 1; j < n; ++j) s -= ri[j] * u[j];
        u[i] = s / ri[i];
    }
}

void orc_hier_free(orc_hier *h) {
    if (!h) return;
    for (int l = 0; l < h->nlev; ++l) {
        mat_free(&h->lv[l].A); mat_free(&h->lv[l].P); mat_free(&h->lv[l].R);
        free(h->lv[l].agg); free(h->lv[l].sm);
    }
    free(h->lv); free(h->lu); free(h->piv); free(h);
}

/* setup, ns_block branch (hierarchy.hpp:263-285, 331-380) with the
 * as_scalar_transfer wrapper (coarsening.hpp:425-464). */
int orc_setup_ns_block(int64_t n, const int64_t *ptr, const int64_t *col,
        const double *val, const double *B, int64_t bcols,
        const orc_params *prm, orc_hier **out) {
    API_BEGIN
    const int blockp = prm->pipeline == ORC_PIPELINE_BLOCK;
    if (!B && !blockp) fail(ORC_BAD_NULLSPACE_SHAPE, "setup: pipeline requires a nullspace basis");
    if (n % 3) fail(ORC_NOT_DIVISIBLE, "setup: block pipelines require dimension divisible by 3");
    orc_hier *H = xcalloc(1, sizeof(orc_hier));
    H->prm = *prm;
    int cap = 4;
    H->lv = xcalloc(cap, sizeof(orc_level));
    orc_mat Ain = {n, n, 1, (int64_t *)ptr, (int64_t *)col, (double *)val};
    H->lv[0].A = to_block3(&Ain);
    H->nlev = 1;
    double *Bi = NULL;
    int64_t bi_rows = n, k = bcols;
    if (!blockp) {
        Bi = xmalloc(sizeof(double) * n * bcols);
        memcpy(Bi, B, sizeof(double) * n * bcols);
    }
    while (H->lv[H->nlev - 1].A.nrows * 3 > prm->coarse_enough) {
        orc_level *Li = &H->lv[H->nlev - 1];
        if (blockp) {
            /* block pipeline (hierarchy.hpp:340-347): block_transfer_operators */
            orc_adj G = strength_graph(&Li->A, prm->eps_strong, 1);
            int64_t *agg = xmalloc(sizeof(int64_t) * (G.nnodes + 1));
            const int64_t naggs = aggregate(&G, agg);
            orc_mat P = block_transfer(&Li->A, &G, agg, naggs, prm->omega);
            orc_mat R = transpose(&P);
            free(G.ptr); free(G.col);
            if ((double)(P.ncols * 3) > prm->stagnation_ratio * (double)(Li->A.nrows * 3)) {
                mat_free(&P); mat_free(&R); free(agg);
                break;
            }
            orc_mat Ac = galerkin(&R, &Li->A, &P);
            fix_decoupled_rows(&Ac);
            Li->P = P; Li->R = R; Li->has_transfer = 1;
            Li->agg = agg; Li->nnodes = G.nnodes; Li->naggs = naggs;
            if (H->nlev == cap) {
                cap *= 2;
                H->lv = realloc(H->lv, sizeof(orc_level) * cap);
                memset(H->lv + H->nlev, 0, sizeof(orc_level) * (cap - H->nlev));
            }
            H->lv[H->nlev].A = Ac;
            H->nlev++;
            continue;
        }
        const int pbs = (H->nlev == 1) ? 3 : (int)k;
        /* as_scalar_transfer: to_scalar -> transfer_operators -> to_block */
        orc_mat As = to_scalar(&Li->A);
        if (As.nrows != As.ncols) fail(ORC_NON_SQUARE, "transfer_operators: matrix must be square");
        orc_adj G = strength_graph(&As, prm->eps_strong, pbs);
        int64_t *agg = xmalloc(sizeof(int64_t) * (G.nnodes + 1));
        const int64_t naggs = aggregate(&G, agg);
        double *Bc = NULL;
        orc_mat Pt = tentative(agg, G.nnodes, naggs, Bi, bi_rows, k, pbs, &Bc);
        orc_mat Ps = smooth_prolongation(&As, &Pt, &G, prm->omega, pbs);
        orc_mat Rs = transpose(&Ps);
        if (Ps.ncols % 3) fail(ORC_NOT_DIVISIBLE, "as_scalar_transfer: coarse dimension not divisible by block size");
        orc_mat P = to_block3(&Ps), R = to_block3(&Rs);
        /* stagnation guard (hierarchy.hpp:355; scalar_setup :246) */
        if ((double)(P.ncols * 3) > prm->stagnation_ratio * (double)(Li->A.nrows * 3)) {
            mat_free(&As); mat_free(&Pt); mat_free(&Ps); mat_free(&Rs);
            free(G.ptr); free(G.col);
            mat_free(&P); mat_free(&R); free(agg); free(Bc);
            break;
        }
        orc_mat Ac;
        if (prm->pipeline == ORC_PIPELINE_NS_HYBRID1 || prm->pipeline == ORC_PIPELINE_NS_HYBRID2) {
            /* scalar_setup (hierarchy.hpp:233-260): Galerkin and
             * fix_decoupled_rows on the scalar matrices, stored as blocks
             * (hierarchy.hpp:318-322) */
            orc_mat Acs = galerkin(&Rs, &As, &Ps);
            fix_decoupled_rows(&Acs);
            Ac = to_block3(&Acs);
            mat_free(&Acs);
        } else {
            Ac = galerkin(&R, &Li->A, &P);
            fix_decoupled_rows(&Ac);
        }
        mat_free(&As); mat_free(&Pt); mat_free(&Ps); mat_free(&Rs);
        free(G.ptr); free(G.col);
        Li->P = P; Li->R = R; Li->has_transfer = 1;
        Li->agg = agg; Li->nnodes = G.nnodes; Li->naggs = naggs;
        if (H->nlev == cap) {
            cap *= 2;
            H->lv = realloc(H->lv, sizeof(orc_level) * cap);
            memset(H->lv + H->nlev, 0, sizeof(orc_level) * (cap - H->nlev));
        }
        H->lv[H->nlev].A = Ac;
        H->nlev++;
        free(Bi);
        Bi = Bc; bi_rows = naggs * k;
    }
    free(Bi);
    for (int l = 0; l + 1 < H->nlev; ++l) {
        if (prm->smoother == ORC_SM_JACOBI) setup_point_jacobi(&H->lv[l]);
        else if (prm->smoother == ORC_SM_ILU0) setup_ilu0(&H->lv[l]);
        else setup_block_smoother(&H->lv[l], prm->smoother, prm->smoother_omega);
    }
    dense_lu_factor(H, &H->lv[H->nlev - 1].A);
    *out = H;
    API_END;
}

int orc_hier_nlevels(const orc_hier *h) { return h->nlev; }
int64_t orc_hier_coarse_dim(const orc_hier *h) { return h->nc; }

int orc_hier_matrix(const orc_hier *h, int level, int which, orc_mat *m) {
    if (level < 0 || level >= h->nlev) return ORC_ERROR;
    const orc_level *L = &h->lv[level];
    if (which != 0 && !L->has_transfer) return ORC_ERROR;
    *m = which == 0 ? L->A : which == 1 ? L->P : L->R;
    return ORC_OK;
}

int orc_hier_aggregates(const orc_hier *h, int level, int64_t *nnodes,
        const int64_t **id, int64_t *count) {
    if (level < 0 || level + 1 >= h->nlev) return ORC_ERROR;
    *nnodes = h->lv[level].nnodes;
    *id = h->lv[level].agg;
    *count = h->lv[level].naggs;
    return ORC_OK;
}

int orc_hier_smoother(const orc_hier *h, int level, int64_t *len,
        const double **data) {
    if (level < 0 || level + 1 >= h->nlev) return ORC_ERROR;
    *len = h->lv[level].sm_len;
    *data = h->lv[level].sm;
    return ORC_OK;
}

/* matrix_bytes (csr.hpp:360-365) */
static uint64_t matrix_bytes(const orc_mat *A) {
    return (uint64_t)(A->nrows + 1) * 8 + (uint64_t)nnz_of(A) * 8 +
           (uint64_t)nnz_of(A) * 8 * A->b * A->b;
}

/* memory_footprint (hierarchy.hpp:443-458) */
uint64_t orc_hier_memory_footprint(const orc_hier *h) {
    uint64_t bytes = 0;
    for (int l = 0; l < h->nlev; ++l) {
        bytes += matrix_bytes(&h->lv[l].A);
        if (h->lv[l].has_transfer) {
            bytes += matrix_bytes(&h->lv[l].P);
            bytes += matrix_bytes(&h->lv[l].R);
        }
        bytes += (uint64_t)h->lv[l].sm_len * 8;
        /* ilu0::bytes (relaxation.hpp:93-95): the factors are a csr, with
         * its ptr and col arrays */
        if (h->prm.smoother == ORC_SM_ILU0 && l + 1 < h->nlev)
            bytes += (uint64_t)(h->lv[l].A.nrows + 1) * 8 + (uint64_t)nnz_of(&h->lv[l].A) * 8;
    }
    bytes += (uint64_t)h->nc * h->nc * 8;
    return bytes;
}

/* apply_smoother (hierarchy.hpp:193-224) for the point / block smoothers */
static void apply_smoother(const orc_hier *H, const orc_level *L,
        const double *f, double *u, double *r, int sweeps) {
    const int64_t n = L->A.nrows * 3;
    for (int s = 0; s < sweeps; ++s) {
        residual(&L->A, f, u, r);
        if (H->prm.smoother == ORC_SM_ILU0) {
            /* hierarchy.hpp:211-220: r = f - A u; LU d = r; u += d */
            ilu0_solve(L, r);
            for (int64_t i = 0; i < n; ++i) u[i] = r[i] + u[i];
        } else if (H->prm.smoother == ORC_SM_JACOBI) {
            /* damped_jacobi::smooth (relaxation.hpp:165-173) */
            const double w = H->prm.smoother_omega;
            for (int64_t i = 0; i < n; ++i) u[i] += w * L->sm[i] * r[i];
        } else {
            for (int64_t i = 0; i < L->A.nrows; ++i) {
                const double *M = L->sm + i * 9;
                double t[3];
                for (int p = 0; p < 3; ++p) {
                    t[p] = 0;
                    for (int q = 0; q < 3; ++q) t[p] += M[p * 3 + q] * r[i * 3 + q];
                }
                for (int p = 0; p < 3; ++p) u[i * 3 + p] += t[p];
            }
        }
    }
}

/* vcycle (hierarchy.hpp:408-441) with vcycle_workspace (:152-163) */
static void vcycle(const orc_hier *H, const double *f, double *u, double **wf,
        double **wu, double **wr) {
    const int L = H->nlev;
    if (L == 1) { dense_lu_solve(H, f, u); return; }
    const int64_t n0 = H->lv[0].A.nrows * 3;
    memcpy(wf[0], f, sizeof(double) * n0);
    memcpy(wu[0], u, sizeof(double) * n0);
    for (int i = 0; i < L - 1; ++i) {
        const orc_level *lv = &H->lv[i];
        if (i > 0) memset(wu[i], 0, sizeof(double) * lv->A.nrows * 3);
        apply_smoother(H, lv, wf[i], wu[i], wr[i], H->prm.pre_sweeps);
        residual(&lv->A, wf[i], wu[i], wr[i]);
        spmv(1.0, &lv->R, wr[i], 0.0, wf[i + 1]);
    }
    dense_lu_solve(H, wf[L - 1], wu[L - 1]);
    for (int i = L - 2; i >= 0; --i) {
        const orc_level *lv = &H->lv[i];
        spmv(1.0, &lv->P, wu[i + 1], 1.0, wu[i]);
        apply_smoother(H, lv, wf[i], wu[i], wr[i], H->prm.post_sweeps);
    }
    memcpy(u, wu[0], sizeof(double) * n0);
}

static void ws_alloc(const orc_hier *H, double ***wf, double ***wu, double ***wr) {
    *wf = xcalloc(H->nlev, sizeof(double *));
    *wu = xcalloc(H->nlev, sizeof(double *));
    *wr = xcalloc(H->nlev, sizeof(double *));
    for (int l = 0; l < H->nlev; ++l) {
        const int64_t n = H->lv[l].A.nrows * 3;
        (*wf)[l] = xcalloc(n, sizeof(double));
        (*wu)[l] = xcalloc(n, sizeof(double));
        (*wr)[l] = xcalloc(n, sizeof(double));
    }
}

static void ws_free(const orc_hier *H, double **wf, double **wu, double **wr) {
    for (int l = 0; l < H->nlev; ++l) { free(wf[l]); free(wu[l]); free(wr[l]); }
    free(wf); free(wu); free(wr);
}

int orc_vcycle(const orc_hier *h, const double *f, double *u) {
    API_BEGIN
    double **wf, **wu, **wr;
    ws_alloc(h, &wf, &wu, &wr);
    vcycle(h, f, u, wf, wu, wr);
    ws_free(h, wf, wu, wr);
    API_END;
}

/* cg_solve_op (cg.hpp:39-83) + cg_solve(hierarchy) (cg.hpp:87-112) */
int orc_cg_solve(const orc_hier *H, const double *f, double *u, double tol,
        int max_iterations, orc_report *rep) {
    API_BEGIN
    const int64_t n = H->lv[0].A.nrows * 3;
    double *r = xmalloc(sizeof(double) * n), *z = xcalloc(n, sizeof(double));
    double *p = xcalloc(n, sizeof(double)), *q = xcalloc(n, sizeof(double));
    double **wf, **wu, **wr;
    ws_alloc(H, &wf, &wu, &wr);
    memcpy(r, f, sizeof(double) * n);
    memset(u, 0, sizeof(double) * n);
    rep->iterations = 0;
    rep->converged = 0;
    rep->relative_residual = 0;
    const double norm_f = norm2(f, n);
    if (norm_f == 0.0) {
        rep->converged = 1;
    } else {
        memset(z, 0, sizeof(double) * n);
        vcycle(H, r, z, wf, wu, wr);
        memcpy(p, z, sizeof(double) * n);
        double rho = dot(r, z, n);
        double res_norm = norm2(r, n);
        int iter = 0;
        while (res_norm / norm_f > tol && iter < max_iterations) {
            spmv(1.0, &H->lv[0].A, p, 0.0, q);
            const double pq = dot(p, q, n);
            if (pq <= 0.0)
                fail(ORC_BREAKDOWN_NON_SPD, "cg: p'Ap <= 0, matrix or preconditioner not SPD");
            const double alpha = rho / pq;
            axpby(alpha, p, 1.0, u, n);
            axpby(-alpha, q, 1.0, r, n);
            ++iter;
            res_norm = norm2(r, n);
            if (res_norm / norm_f <= tol) break;
            memset(z, 0, sizeof(double) * n);
            vcycle(H, r, z, wf, wu, wr);
            const double rho_new = dot(r, z, n);
            const double beta = rho_new / rho;
            rho = rho_new;
            axpby(1.0, z, beta, p, n);
        }
        rep->iterations = iter;
        rep->converged = res_norm / norm_f <= tol;
        /* true residual at exit (cg.hpp:105-108) */
        memcpy(q, f, sizeof(double) * n);
        spmv(-1.0, &H->lv[0].A, u, 1.0, q);
        rep->relative_residual = norm2(q, n) / norm_f;
    }
    ws_free(H, wf, wu, wr);
    free(r); free(z); free(p); free(q);
    API_END;
}

/* ------------------------------------------------------------------------ */
/* standalone kernels for pins                                               */

int orc_spmv_bsr3(int64_t nrows, int64_t ncols, const int64_t *ptr,
        const int64_t *col, const double *val, double alpha, const double *x,
        double beta, double *y) {
    API_BEGIN
    orc_mat A = {nrows, ncols, 3, (int64_t *)ptr, (int64_t *)col, (double *)val};
    spmv(alpha, &A, x, beta, y);
    API_END;
}

int orc_galerkin_bsr3(const orc_mat *R, const orc_mat *A, const orc_mat *P,
        orc_mat *C) {
    API_BEGIN
    *C = galerkin(R, A, P);
    API_END;
}

int orc_aggregate_scalar(int64_t n, const int64_t *ptr, const int64_t *col,
        const double *val, double eps, int pbs, int64_t *id, int64_t *count) {
    API_BEGIN
    orc_mat A = {n, n, 1, (int64_t *)ptr, (int64_t *)col, (double *)val};
    orc_adj G = strength_graph(&A, eps, pbs);
    *count = aggregate(&G, id);
    free(G.ptr); free(G.col);
    API_END;
}

/* ------------------------------------------------------------------------ */
/* generator (elasticity.hpp)                                                */

/* rigid_body_modes (elasticity.hpp:38-52): column-major (3n)-by-6 */
void orc_rigid_body_modes(int64_t nnodes, const double *xyz, double *B) {
    const int64_t nr = 3 * nnodes;
    memset(B, 0, sizeof(double) * nr * 6);
    for (int64_t a = 0; a < nnodes; ++a) {
        const double x = xyz[3 * a], y = xyz[3 * a + 1], z = xyz[3 * a + 2];
        const int64_t r = 3 * a;
        B[0 * nr + r + 0] = 1;
        B[1 * nr + r + 1] = 1;
        B[2 * nr + r + 2] = 1;
        B[3 * nr + r + 0] = -y; B[3 * nr + r + 1] = x;
        B[4 * nr + r + 1] = -z; B[4 * nr + r + 2] = y;
        B[5 * nr + r + 0] = z;  B[5 * nr + r + 2] = -x;
    }
}

/* hex8_stiffness (elasticity.hpp:57-123): 2x2x2 Gauss, isotropic C. */
void orc_hex8_stiffness(double hx, double hy, double hz, double E, double nu,
        double *Ke) {
    const double lambda = E * nu / ((1 + nu) * (1 - 2 * nu));
    const double mu = E / (2 * (1 + nu));
    double C[6][6];
    memset(C, 0, sizeof C);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) C[i][j] = (i == j) ? lambda + 2 * mu : lambda;
    for (int i = 3; i < 6; ++i) C[i][i] = mu;
    const double g = 1.0 / sqrt(3.0);
    const double gp[2] = {-g, g};
    const double jac[3] = {hx / 2, hy / 2, hz / 2};
    const double detJ = jac[0] * jac[1] * jac[2];
    memset(Ke, 0, sizeof(double) * 576);
    for (int qx = 0; qx < 2; ++qx)
    for (int qy = 0; qy < 2; ++qy)
    for (int qz = 0; qz < 2; ++qz) {
        const double xi = gp[qx], eta = gp[qy], zeta = gp[qz];
        double dN[8][3];
        for (int a = 0; a < 8; ++a) {
            const double sx = (a & 1) ? 1.0 : -1.0;
            const double sy = ((a >> 1) & 1) ? 1.0 : -1.0;
            const double sz = ((a >> 2) & 1) ? 1.0 : -1.0;
            dN[a][0] = 0.125 * sx * (1 + sy * eta) * (1 + sz * zeta) / jac[0];
            dN[a][1] = 0.125 * (1 + sx * xi) * sy * (1 + sz * zeta) / jac[1];
            dN[a][2] = 0.125 * (1 + sx * xi) * (1 + sy * eta) * sz / jac[2];
        }
        for (int a = 0; a < 8; ++a)
        for (int b = 0; b < 8; ++b) {
            double Ba[6][3], Bb[6][3];
            memset(Ba, 0, sizeof Ba); memset(Bb, 0, sizeof Bb);
            const double *d1 = dN[a], *d2 = dN[b];
            Ba[0][0] = d1[0]; Ba[1][1] = d1[1]; Ba[2][2] = d1[2];
            Ba[3][0] = d1[1]; Ba[3][1] = d1[0];
            Ba[4][1] = d1[2]; Ba[4][2] = d1[1];
            Ba[5][0] = d1[2]; Ba[5][2] = d1[0];
            Bb[0][0] = d2[0]; Bb[1][1] = d2[1]; Bb[2][2] = d2[2];
            Bb[3][0] = d2[1]; Bb[3][1] = d2[0];
            Bb[4][1] = d2[2]; Bb[4][2] = d2[1];
            Bb[5][0] = d2[2]; Bb[5][2] = d2[0];
            for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                double s = 0;
                for (int p = 0; p < 6; ++p)
                for (int q = 0; q < 6; ++q) s += Ba[p][i] * C[p][q] * Bb[q][j];
                Ke[(3 * a + i) * 24 + (3 * b + j)] += s * detJ;
            }
        }
    }
}

typedef struct { int64_t c; int64_t seq; double v; } trip;
static int cmp_trip(const void *a, const void *b) {
    const trip *x = a, *y = b;
    if (x->c != y->c) return (x->c > y->c) - (x->c < y->c);
    return (x->seq > y->seq) - (x->seq < y->seq);
}

/* generate_hex_elasticity (elasticity.hpp:129-213): unit cube, x-fastest
 * node numbering, interleaved DOFs, clamped DOFs kept as unit rows, unit
 * downward body force.  Duplicates are summed in triplet order (stable). */
int orc_generate_hex(int64_t nx, int64_t ny, int64_t nz, double E, double nu,
        int clamp_x0, int64_t *n_out, int64_t **ptr_out, int64_t **col_out,
        double **val_out, double **rhs_out, double **coords_out) {
    API_BEGIN
    if (nx < 1 || ny < 1 || nz < 1)
        fail(ORC_INVALID_MATERIAL, "generate_hex_elasticity: element counts must be >= 1");
    if (!(E > 0) || !(nu > 0 && nu < 0.5))
        fail(ORC_INVALID_MATERIAL, "generate_hex_elasticity: need E > 0 and 0 < nu < 0.5");
    const int64_t mx = nx + 1, my = ny + 1, mz = nz + 1;
    const int64_t nnodes = mx * my * mz, ndof = 3 * nnodes;
    const double hx = 1.0 / nx, hy = 1.0 / ny, hz = 1.0 / nz;
    double *xyz = xmalloc(sizeof(double) * 3 * nnodes);
    for (int64_t k = 0; k < mz; ++k)
        for (int64_t j = 0; j < my; ++j)
            for (int64_t i = 0; i < mx; ++i) {
                const int64_t nd = i + mx * (j + my * k);
                xyz[3 * nd + 0] = i * hx;
                xyz[3 * nd + 1] = j * hy;
                xyz[3 * nd + 2] = k * hz;
            }
    char *cons = xcalloc(ndof, 1);
    if (clamp_x0)
        for (int64_t k = 0; k < mz; ++k)
            for (int64_t j = 0; j < my; ++j) {
                const int64_t nd = mx * (j + my * k);
                cons[3 * nd] = cons[3 * nd + 1] = cons[3 * nd + 2] = 1;
            }
    double Ke[576];
    orc_hex8_stiffness(hx, hy, hz, E, nu, Ke);
    double *rhs = xcalloc(ndof, sizeof(double));
    const double nodal_force = -hx * hy * hz / 8.0;
    /* count triplets per row, then fill in triplet order */
    int64_t *rcount = xcalloc(ndof + 1, sizeof(int64_t));
    for (int pass = 0; pass < 2; ++pass) {
        trip *T = NULL;
        int64_t *head = NULL;
        if (pass == 1) {
            for (int64_t d = 0; d < ndof; ++d) rcount[d + 1] += rcount[d];
            T = xmalloc(sizeof(trip) * (rcount[ndof] + 1));
            head = xmalloc(sizeof(int64_t) * (ndof + 1));
            memcpy(head, rcount, sizeof(int64_t) * (ndof + 1));
        }
        int64_t seq = 0;
        for (int64_t ez = 0; ez < nz; ++ez)
        for (int64_t ey = 0; ey < ny; ++ey)
        for (int64_t ex = 0; ex < nx; ++ex) {
            int64_t nodes[8];
            for (int a = 0; a < 8; ++a)
                nodes[a] = (ex + (a & 1)) + mx * ((ey + ((a >> 1) & 1)) + my * (ez + ((a >> 2) & 1)));
            for (int a = 0; a < 8; ++a) {
                if (pass == 0) rhs[3 * nodes[a] + 2] += nodal_force;
                for (int b = 0; b < 8; ++b)
                    for (int i = 0; i < 3; ++i)
                        for (int j = 0; j < 3; ++j) {
                            const int64_t gi = 3 * nodes[a] + i, gj = 3 * nodes[b] + j;
                            if (cons[gi] || cons[gj]) continue;
                            if (pass == 0) { rcount[gi + 1]++; continue; }
                            trip *t = &T[head[gi]++];
                            t->c = gj; t->seq = seq++;
                            t->v = Ke[(3 * a + i) * 24 + (3 * b + j)];
                        }
            }
        }
        if (pass == 0) {
            for (int64_t d = 0; d < ndof; ++d)
                if (cons[d]) { rcount[d + 1]++; rhs[d] = 0.0; }
            continue;
        }
        for (int64_t d = 0; d < ndof; ++d)
            if (cons[d]) { trip *t = &T[head[d]++]; t->c = d; t->seq = seq++; t->v = 1.0; }
        int64_t *ptr = xcalloc(ndof + 1, sizeof(int64_t));
        int64_t *col = xmalloc(sizeof(int64_t) * (rcount[ndof] + 1));
        double *val = xmalloc(sizeof(double) * (rcount[ndof] + 1));
        int64_t out = 0;
        for (int64_t d = 0; d < ndof; ++d) {
            const int64_t beg = rcount[d], end = rcount[d + 1];
            qsort(T + beg, (size_t)(end - beg), sizeof(trip), cmp_trip);
            for (int64_t k = beg; k < end; ++k) {
                if (out > ptr[d] && col[out - 1] == T[k].c) val[out - 1] += T[k].v;
                else { col[out] = T[k].c; val[out] = T[k].v; ++out; }
            }
            ptr[d + 1] = out;
        }
        free(T); free(head);
        *ptr_out = ptr; *col_out = col; *val_out = val;
    }
    free(rcount); free(cons);
    *n_out = ndof;
    *rhs_out = rhs;
    *coords_out = xyz;
    API_END;
}
