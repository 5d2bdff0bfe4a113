/*
 * p1_oracle.c -- CPU restatement of the reference's P1 assembly path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file.  Only tests/, __graft_entry__.smoke() (as the checker) and
 * bench.py's cpu_baseline / --impl reference leg may use it.
 *
 * What it restates (reference = /root/reference/pkg/src/simplex_asm):
 *   - compute_volumes      mesh.py:29-43     (numpy det on B_k = edges as
 *                                              columns: LAPACK getrf, then
 *                                              sign*exp(sum log|u_jj|), glibc
 *                                              scalar log/exp, |det|/d!)
 *   - compute_gradients    kernels.py:49-65  (numpy solve(B_k^T, [-1|I]) =
 *                                              OpenBLAS dgesv; the operation
 *                                              order of the OpenBLAS SkylakeX
 *                                              and Haswell kernels is restated
 *                                              per SURVEY.md Appendix A)
 *   - mass_kernel          kernels.py:68-78, MassKernel :281-303
 *   - stiffness_kernel     kernels.py:81-88
 *   - dot_mat_vec_g / elastic_kernel / ElasticKernel  kernels.py:141-172,332-387
 *   - general operator     (absent in the reference; SURVEY.md Appendix B,
 *                           arithmetic order defined in DESIGN.md §3.4)
 *   - assemble_optv2 / assemble_vector_optv2  assembly.py:92-111,188-209
 *     + sparse_from_triplets/_canonicalize    sparse.py:85-133
 *     i.e. element-major triplets, zero inputs skipped, stable sort by
 *     (row, col), left-to-right sums in ascending element order, exact-zero
 *     sums dropped.
 *
 * The assembly is restricted to a contiguous dof-row block [row_begin,
 * row_end): SURVEY.md 8(e) verified that the rows of a row-block optv2 are
 * bitwise the rows of the full optv2 (same triplet order restricted).
 *
 * Compile with -ffp-contract=off: every a*b+c below must round twice unless
 * written as fma().
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define OR_OK 0
#define OR_DEGENERATE 1
#define OR_BAD_ARG 2
#define OR_NOMEM 3
#define OR_INDEX_RANGE 4

enum { CORE_SKYLAKEX = 0, CORE_HASWELL = 1 };
enum { OP_MASS = 0, OP_STIFF = 1, OP_ELASTIC = 2, OP_GENERAL = 3 };

/* ------------------------------------------------------------------------ */
/* LU with partial pivoting, left-looking (OpenBLAS getf2 structure).       */
/* a is d x d row-major, modified in place; perm[i] = source row of row i.  */
/* Returns 0, or 1 if some pivot is exactly 0.0 (LAPACK info > 0).          */
static int lu_left_looking(int d, double *a, int *perm, int core)
{
    for (int i = 0; i < d; ++i) perm[i] = i;
    int singular = 0;
    for (int j = 0; j < d; ++j) {
        /* U part of column j: rows 1..j-1 */
        for (int i = 1; i < j; ++i) {
            double s = 0.0;
            for (int k = 0; k < i; ++k) {
                if (k == 0) s = a[i * d + k] * a[k * d + j];
                else if (core == CORE_SKYLAKEX) s = fma(a[i * d + k], a[k * d + j], s);
                else s = s + a[i * d + k] * a[k * d + j];
            }
            a[i * d + j] = a[i * d + j] - s;
        }
        /* rows j..d-1 */
        for (int i = j; i < d; ++i) {
            if (j == 0) continue;
            double s = 0.0;
            for (int k = 0; k < j; ++k) {
                if (k == 0) s = a[i * d + k] * a[k * d + j];
                else if (core == CORE_SKYLAKEX) s = fma(a[i * d + k], a[k * d + j], s);
                else s = s + a[i * d + k] * a[k * d + j];
            }
            a[i * d + j] = a[i * d + j] - s;
        }
        /* pivot: first index of max |a[i][j]|, i >= j (idamax) */
        int p = j;
        double best = fabs(a[j * d + j]);
        for (int i = j + 1; i < d; ++i) {
            double v = fabs(a[i * d + j]);
            if (v > best) { best = v; p = i; }
        }
        if (p != j) {
            for (int c = 0; c < d; ++c) {
                double t = a[j * d + c]; a[j * d + c] = a[p * d + c]; a[p * d + c] = t;
            }
            int t = perm[j]; perm[j] = perm[p]; perm[p] = t;
        }
        if (a[j * d + j] == 0.0) { singular = 1; continue; }
        double r = 1.0 / a[j * d + j];
        for (int i = j + 1; i < d; ++i) a[i * d + j] = a[i * d + j] * r;
    }
    return singular;
}

/* getrs on the factored a for the rhs columns of [-1 | I_d].
 * x is d x (d+1) row-major on output: x[nu][alpha]. */
static void getrs_ref_gradients(int d, const double *a, const int *perm, int core, double *x)
{
    double r[3];
    for (int j = 0; j < d; ++j) r[j] = 1.0 / a[j * d + j];
    for (int col = 0; col <= d; ++col) {
        double b[3];
        /* rhs column col of [-1 | I], rows permuted: row i takes source perm[i] */
        for (int i = 0; i < d; ++i) {
            int src = perm[i];
            b[i] = (col == 0) ? -1.0 : (src == col - 1 ? 1.0 : 0.0);
        }
        if (d == 1) {
            b[0] = b[0] * r[0];
        } else if (d == 2) {
            double l10 = a[2], u01 = a[1];
            if (core == CORE_SKYLAKEX) b[1] = fma(-l10, b[0], b[1]);
            else b[1] = b[1] - l10 * b[0];
            b[1] = b[1] * r[1];
            if (core == CORE_SKYLAKEX) b[0] = fma(-u01, b[1], b[0]);
            else b[0] = b[0] - u01 * b[1];
            b[0] = b[0] * r[0];
        } else { /* d == 3 */
            double l10 = a[3], l20 = a[6], l21 = a[7];
            double u01 = a[1], u02 = a[2], u12 = a[5];
            if (core == CORE_SKYLAKEX) b[1] = fma(-l10, b[0], b[1]);
            else b[1] = b[1] - l10 * b[0];
            double acc = l20 * b[0];
            acc = fma(l21, b[1], acc);
            b[2] = b[2] - acc;
            b[2] = b[2] * r[2];
            b[0] = b[0] - u02 * b[2];
            b[1] = b[1] - u12 * b[2];
            b[1] = b[1] * r[1];
            if (core == CORE_SKYLAKEX) b[0] = fma(-b[1], u01, b[0]);
            else b[0] = b[0] - u01 * b[1];
            b[0] = b[0] * r[0];
        }
        for (int i = 0; i < d; ++i) x[i * (d + 1) + col] = b[i];
    }
}

/* Edge matrix A = B_k^T: A[r][c] = q[c][me[r+1][k]] - q[c][me[0][k]]. */
static void edge_rows(int d, int64_t nq, int64_t nme, const double *q, const int64_t *me,
                      int64_t k, double *A)
{
    int64_t v0 = me[k];
    for (int r = 0; r < d; ++r) {
        int64_t vr = me[(int64_t)(r + 1) * nme + k];
        for (int c = 0; c < d; ++c) A[r * d + c] = q[(int64_t)c * nq + vr] - q[(int64_t)c * nq + v0];
    }
}

/* numpy det path on B (edges as columns): det = sign * exp(sum log|u_jj|). */
static double det_numpy(int d, const double *A_rows, int core)
{
    double B[9];
    int perm[3];
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) B[i * d + j] = A_rows[j * d + i];
    int sing = lu_left_looking(d, B, perm, core);
    if (sing) return 0.0;
    /* permutation parity */
    int sign = 1;
    int seen[3] = {0, 0, 0};
    for (int i = 0; i < d; ++i) {
        if (seen[i]) continue;
        int len = 0, j = i;
        while (!seen[j]) { seen[j] = 1; j = perm[j]; ++len; }
        if ((len & 1) == 0) sign = -sign;
    }
    double logdet = 0.0;
    for (int i = 0; i < d; ++i) {
        double u = B[i * d + i];
        if (u < 0) { sign = -sign; u = -u; }
        logdet += log(u);
    }
    return sign * exp(logdet);
}

static double factorial_d(int d) { return d == 1 ? 1.0 : d == 2 ? 2.0 : 6.0; }

/* mesh.py:29-43 -- vols[k] = |det B_k| / d!; first degenerate k in *bad. */
int or_volumes(int d, int64_t nq, int64_t nme, const double *q, const int64_t *me, int core,
               double *vols, int64_t *bad)
{
    if (d < 1 || d > 3) return OR_BAD_ARG;
    double A[9];
    for (int64_t k = 0; k < nme; ++k) {
        edge_rows(d, nq, nme, q, me, k, A);
        double det = det_numpy(d, A, core);
        if (det == 0.0) { *bad = k; return OR_DEGENERATE; }
        vols[k] = fabs(det) / factorial_d(d);
    }
    return OR_OK;
}

/* kernels.py:49-65 -- grads[k][alpha][nu]; degenerate check is the numpy det
 * of B (kernels.py:59-62). */
int or_gradients(int d, int64_t nq, int64_t nme, const double *q, const int64_t *me, int core,
                 double *grads, int64_t *bad)
{
    if (d < 1 || d > 3) return OR_BAD_ARG;
    double A[9], x[12];
    int perm[3];
    for (int64_t k = 0; k < nme; ++k) {
        edge_rows(d, nq, nme, q, me, k, A);
        if (det_numpy(d, A, core) == 0.0) { *bad = k; return OR_DEGENERATE; }
    }
    for (int64_t k = 0; k < nme; ++k) {
        edge_rows(d, nq, nme, q, me, k, A);
        lu_left_looking(d, A, perm, core);
        getrs_ref_gradients(d, A, perm, core, x);
        double *g = grads + k * (int64_t)(d + 1) * d;
        for (int a = 0; a <= d; ++a)
            for (int nu = 0; nu < d; ++nu) g[a * d + nu] = x[nu * (d + 1) + a];
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Operator description passed from Python.                                 */
typedef struct {
    int op;           /* OP_* */
    int d;
    int m;            /* unknowns per node: 1 (scalar) or d (elastic) */
    int core;
    const double *w;        /* mass: nodal weight (nq) */
    const double *lamb;     /* elastic: nodal lambda (nq) */
    const double *mu;       /* elastic: nodal mu (nq) */
    const double *tabQ;     /* elastic: Q[n][l] as d*d blocks of d*d: [(n*d+l)*d*d + j*d + i] */
    const double *tabS;
    const double *A;        /* general: nodal A (nq, d, d) row-major */
    const double *b;        /* general: (nq, d) */
    const double *c;        /* general: (nq, d) */
    const double *a0;       /* general: (nq) */
    const double *vols;     /* (nme) mesh volumes (mesh.vols, as the reference kernels use) */
} or_op;

/* Local matrix of element k: loc[(l*(d+1)+alpha) * M + (n*(d+1)+beta)], M = m(d+1). */
static void local_matrix(const or_op *op, int64_t nq, int64_t nme, const double *q,
                         const int64_t *me, int64_t k, double *loc)
{
    const int d = op->d, dp1 = d + 1, m = op->m, M = m * dp1;
    double vol = op->vols[k];
    int64_t v[4] = {0, 0, 0, 0};
    for (int a = 0; a < dp1; ++a) v[a] = me[(int64_t)a * nme + k];
    double G[12];
    if (op->op != OP_MASS) {
        double A[9], x[12];
        int perm[3];
        edge_rows(d, nq, nme, q, me, k, A);
        lu_left_looking(d, A, perm, op->core);
        getrs_ref_gradients(d, A, perm, op->core, x);
        for (int a = 0; a < dp1; ++a)
            for (int nu = 0; nu < d; ++nu) G[a * d + nu] = x[nu * dp1 + a];
    }
    if (op->op == OP_MASS) {
        /* kernels.py:68-78: coef * vols * (wsum + W[alpha] + W[beta]) */
        double W[4], wsum;
        for (int a = 0; a < dp1; ++a) W[a] = op->w[v[a]];
        wsum = W[0];
        for (int a = 1; a < dp1; ++a) wsum = wsum + W[a];
        double den = (double)((d + 1) * (d + 2) * (d + 3));
        for (int a = 0; a < dp1; ++a)
            for (int bb = 0; bb < dp1; ++bb) {
                double coef = (a == bb ? 2.0 : 1.0) / den;
                loc[a * M + bb] = (coef * vol) * ((wsum + W[a]) + W[bb]);
            }
    } else if (op->op == OP_STIFF) {
        /* kernels.py:81-88: acc = 0; acc += G[beta,i]*G[alpha,i]; acc * vols */
        for (int a = 0; a < dp1; ++a)
            for (int bb = 0; bb < dp1; ++bb) {
                double acc = 0.0;
                for (int i = 0; i < d; ++i) acc = acc + G[bb * d + i] * G[a * d + i];
                loc[a * M + bb] = acc * vol;
            }
    } else if (op->op == OP_ELASTIC) {
        /* kernels.py:332-387: lambs = (sum_gamma lamb_gamma) * (vols/(d+1)) */
        double scale = vol / (double)dp1;
        double ls = op->lamb[v[0]], ms = op->mu[v[0]];
        for (int a = 1; a < dp1; ++a) { ls = ls + op->lamb[v[a]]; ms = ms + op->mu[v[a]]; }
        double lambs = ls * scale, mus = ms * scale;
        for (int l = 0; l < m; ++l)
            for (int n = 0; n < m; ++n) {
                const double *Qt = op->tabQ + (int64_t)(n * d + l) * d * d;
                const double *St = op->tabS + (int64_t)(n * d + l) * d * d;
                for (int a = 0; a < dp1; ++a)
                    for (int bb = 0; bb < dp1; ++bb) {
                        /* dot_mat_vec_g: i outer, j inner, skip zero A[j,i] */
                        double xq = 0.0, xs = 0.0;
                        for (int i = 0; i < d; ++i)
                            for (int j = 0; j < d; ++j) {
                                double aq = Qt[j * d + i];
                                if (aq != 0.0) xq = xq + aq * (G[a * d + i] * G[bb * d + j]);
                            }
                        for (int i = 0; i < d; ++i)
                            for (int j = 0; j < d; ++j) {
                                double as = St[j * d + i];
                                if (as != 0.0) xs = xs + as * (G[a * d + i] * G[bb * d + j]);
                            }
                        loc[(l * dp1 + a) * M + (n * dp1 + bb)] = lambs * xq + mus * xs;
                    }
            }
    } else { /* OP_GENERAL -- DESIGN.md 3.4 */
        double As[9], bs[3], cs[3], a0s;
        for (int i = 0; i < d * d; ++i) As[i] = op->A[v[0] * d * d + i];
        for (int i = 0; i < d; ++i) { bs[i] = op->b[v[0] * d + i]; cs[i] = op->c[v[0] * d + i]; }
        a0s = op->a0[v[0]];
        for (int g = 1; g < dp1; ++g) {
            for (int i = 0; i < d * d; ++i) As[i] = As[i] + op->A[v[g] * d * d + i];
            for (int i = 0; i < d; ++i) {
                bs[i] = bs[i] + op->b[v[g] * d + i];
                cs[i] = cs[i] + op->c[v[g] * d + i];
            }
            a0s = a0s + op->a0[v[g]];
        }
        double s1 = vol / (double)dp1;
        double s2 = vol / (double)(dp1 * (d + 2));
        double den = (double)((d + 1) * (d + 2) * (d + 3));
        /* w[beta] = A^s G_beta */
        double AG[12];
        for (int bb = 0; bb < dp1; ++bb)
            for (int i = 0; i < d; ++i) {
                double acc = As[i * d] * G[bb * d];
                for (int j = 1; j < d; ++j) acc = acc + As[i * d + j] * G[bb * d + j];
                AG[bb * d + i] = acc;
            }
        for (int a = 0; a < dp1; ++a)
            for (int bb = 0; bb < dp1; ++bb) {
                double diff = G[a * d] * AG[bb * d];
                for (int i = 1; i < d; ++i) diff = diff + G[a * d + i] * AG[bb * d + i];
                double conv = (bs[0] + op->b[v[bb] * d]) * G[a * d];
                for (int i = 1; i < d; ++i) conv = conv + (bs[i] + op->b[v[bb] * d + i]) * G[a * d + i];
                double tran = (cs[0] + op->c[v[a] * d]) * G[bb * d];
                for (int i = 1; i < d; ++i) tran = tran + (cs[i] + op->c[v[a] * d + i]) * G[bb * d + i];
                /* reaction in exactly the mass_kernel form (kernels.py:76-78) */
                double coef = (a == bb ? 2.0 : 1.0) / den;
                double rea = (coef * vol) * ((a0s + op->a0[v[a]]) + op->a0[v[bb]]);
                loc[a * M + bb] = ((diff * s1 - conv * s2) + tran * s2) + rea;
            }
    }
}

/* ------------------------------------------------------------------------ */
/* optv2 over a row block [row_begin, row_end) of dof rows.                  */
typedef struct {
    int64_t nrows_blk;
    int64_t *row_ptr;   /* (nrows_blk + 1), relative */
    int64_t *col_idx;
    double *vals;
    int64_t nnz;
    int64_t cap;
} or_csr;

/* Two passes over the elements: count triplets per block row, then scatter
 * (col, val) stably, then per row a stable insertion sort by col and a
 * left-to-right fold.  Equivalent to the stable lexsort + bincount of
 * sparse.py:97-111 restricted to the block rows. */
int or_assemble_block(const or_op *op, int64_t nq, int64_t nme, const double *q,
                      const int64_t *me, int64_t row_begin, int64_t row_end,
                      int64_t **out_rowptr, int64_t **out_col, double **out_val, int64_t *out_nnz)
{
    const int d = op->d, dp1 = d + 1, m = op->m, M = m * dp1;
    const int64_t nb = row_end - row_begin;
    int64_t *cnt = calloc((size_t)nb + 1, sizeof(int64_t));
    if (!cnt) return OR_NOMEM;
    /* pass 1: counts (rows only depend on me) */
    for (int64_t k = 0; k < nme; ++k)
        for (int a = 0; a < dp1; ++a) {
            int64_t node = me[(int64_t)a * nme + k];
            for (int l = 0; l < m; ++l) {
                int64_t r = (int64_t)m * node + l;
                if (r >= row_begin && r < row_end) cnt[r - row_begin + 1] += M;
            }
        }
    for (int64_t i = 0; i < nb; ++i) cnt[i + 1] += cnt[i];
    int64_t L = cnt[nb];
    int64_t *tc = malloc((size_t)(L ? L : 1) * sizeof(int64_t));
    double *tv = malloc((size_t)(L ? L : 1) * sizeof(double));
    int64_t *fill = malloc((size_t)(nb ? nb : 1) * sizeof(int64_t));
    double *loc = malloc((size_t)M * M * sizeof(double));
    if (!tc || !tv || !fill || !loc) { free(cnt); free(tc); free(tv); free(fill); free(loc); return OR_NOMEM; }
    memcpy(fill, cnt, (size_t)nb * sizeof(int64_t));
    /* pass 2: element-major, within element the optv2 order (l, n, beta, alpha) */
    for (int64_t k = 0; k < nme; ++k) {
        int touches = 0;
        for (int a = 0; a < dp1 && !touches; ++a) {
            int64_t node = me[(int64_t)a * nme + k];
            if ((int64_t)m * node + m - 1 >= row_begin && (int64_t)m * node < row_end) touches = 1;
        }
        if (!touches) continue;
        local_matrix(op, nq, nme, q, me, k, loc);
        for (int l = 0; l < m; ++l)
            for (int n = 0; n < m; ++n)
                for (int bb = 0; bb < dp1; ++bb)
                    for (int a = 0; a < dp1; ++a) {
                        int64_t r = (int64_t)m * me[(int64_t)a * nme + k] + l;
                        if (r < row_begin || r >= row_end) continue;
                        int64_t c = (int64_t)m * me[(int64_t)bb * nme + k] + n;
                        int64_t p = fill[r - row_begin]++;
                        tc[p] = c;
                        tv[p] = loc[(l * dp1 + a) * M + (n * dp1 + bb)];
                    }
    }
    free(fill);
    free(loc);
    /* per row: drop zero inputs, stable sort by col, fold, drop zero sums */
    int64_t *rp = calloc((size_t)nb + 1, sizeof(int64_t));
    if (!rp) { free(cnt); free(tc); free(tv); return OR_NOMEM; }
    int64_t w = 0;
    for (int64_t i = 0; i < nb; ++i) {
        int64_t s = cnt[i], e = cnt[i + 1];
        int64_t n = 0;
        for (int64_t t = s; t < e; ++t)
            if (tv[t] != 0.0) { tc[s + n] = tc[t]; tv[s + n] = tv[t]; ++n; }
        /* stable insertion sort by column */
        for (int64_t t = 1; t < n; ++t) {
            int64_t cc = tc[s + t];
            double vv = tv[s + t];
            int64_t u = t - 1;
            while (u >= 0 && tc[s + u] > cc) { tc[s + u + 1] = tc[s + u]; tv[s + u + 1] = tv[s + u]; --u; }
            tc[s + u + 1] = cc;
            tv[s + u + 1] = vv;
        }
        int64_t t = 0;
        while (t < n) {
            int64_t cc = tc[s + t];
            double acc = 0.0;
            while (t < n && tc[s + t] == cc) { acc = acc + tv[s + t]; ++t; }
            if (acc != 0.0) { tc[w] = cc; tv[w] = acc; ++w; }
        }
        rp[i + 1] = w;
    }
    free(cnt);
    *out_rowptr = rp;
    *out_col = tc;
    *out_val = tv;
    *out_nnz = w;
    return OR_OK;
}

void or_free(void *p) { free(p); }

/* ------------------------------------------------------------------------ */
/* Multi-threaded full assembly for the CPU baseline: rows split into        */
/* nthreads contiguous blocks, each assembled with or_assemble_block (the    */
/* row-block optv2 is bitwise the full optv2).                  */
typedef struct {
    const or_op *op; int64_t nq, nme; const double *q; const int64_t *me;
    int64_t rb, re; int64_t *rp; int64_t *col; double *val; int64_t nnz; int rc;
} or_job;

static void *or_job_run(void *arg)
{
    or_job *j = (or_job *)arg;
    j->rc = or_assemble_block(j->op, j->nq, j->nme, j->q, j->me, j->rb, j->re, &j->rp, &j->col, &j->val, &j->nnz);
    return NULL;
}

int or_assemble_threaded(const or_op *op, int64_t nq, int64_t nme, const double *q, const int64_t *me,
                         int nthreads, int64_t *out_nnz, int64_t **out_rowptr, int64_t **out_col,
                         double **out_val)
{
    int64_t ndof = (int64_t)op->m * nq;
    if (nthreads < 1) nthreads = 1;
    or_job *jobs = calloc((size_t)nthreads, sizeof(or_job));
    pthread_t *th = calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (or_job){op, nq, nme, q, me, ndof * t / nthreads, ndof * (t + 1) / nthreads, 0, 0, 0, 0, 0};
        pthread_create(&th[t], NULL, or_job_run, &jobs[t]);
    }
    int rc = OR_OK;
    int64_t total = 0;
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        if (jobs[t].rc) rc = jobs[t].rc;
        total += jobs[t].nnz;
    }
    if (rc == OR_OK) {
        int64_t *rp = malloc((size_t)(ndof + 1) * sizeof(int64_t));
        int64_t *col = malloc((size_t)(total ? total : 1) * sizeof(int64_t));
        double *val = malloc((size_t)(total ? total : 1) * sizeof(double));
        int64_t off = 0;
        rp[0] = 0;
        for (int t = 0; t < nthreads; ++t) {
            int64_t nb = jobs[t].re - jobs[t].rb;
            for (int64_t i = 0; i < nb; ++i) rp[jobs[t].rb + i + 1] = off + jobs[t].rp[i + 1];
            memcpy(col + off, jobs[t].col, (size_t)jobs[t].nnz * sizeof(int64_t));
            memcpy(val + off, jobs[t].val, (size_t)jobs[t].nnz * sizeof(double));
            off += jobs[t].nnz;
        }
        *out_rowptr = rp; *out_col = col; *out_val = val; *out_nnz = total;
    }
    for (int t = 0; t < nthreads; ++t) { free(jobs[t].rp); free(jobs[t].col); free(jobs[t].val); }
    free(jobs);
    free(th);
    return rc;
}
