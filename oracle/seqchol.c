/*
 * oracle/seqchol.c -- O1, the sequential block-Cholesky oracle.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing on the product path may link, load or
 * call this file: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it (task contract). It shares no
 * code, header, table or helper with paper_2601_03754_b200/ or include/.
 *
 * What it computes (plain definitions, fp64, plain loops, no BLAS):
 *   - the four elementary block operations of Table 1:
 *       potrf  L L^T = D                      (lower triangle of D is read)
 *       trsm_right  E <- E L^{-T}
 *       trsm_left   E <- L^{-1} E
 *       syrk_down   D <- D - E E^T  or  D - E^T E
 *       gemm_neg    C <- [C] - A B
 *   - Algorithm 1, the sequential factorization Psi = L L^T in natural order
 *     (PAPER.md:144-155): D^_1 = chol(D_1); for i = 2..N:
 *       E^_{i-1} = E_{i-1} D^_{i-1}^{-T};  D^_i = chol(D_i - E^_{i-1} E^_{i-1}^T)
 *   - the standard block forward/backward substitution with that L (the
 *     paper prints no sequential solve; SPEC.md:201-204 names it):
 *       y_1 = D^_1^{-1} b_1;  y_i = D^_i^{-1} (b_i - E^_{i-1} y_{i-1})
 *       x_N = D^_N^{-T} y_N;  x_i = D^_i^{-T} (y_i - E^_i^T x_{i+1})
 *   - a batch driver that runs independent systems on host threads; it is
 *     the timed CPU baseline (SURVEY.md §8(d) "Oracle timed beside it").
 *
 * Layouts: blocks are row-major n x n; D is [N][n][n], E is [N-1][n][n]
 * (E[k-1] is block (k+1, k)), b and x are [N][n][m].
 *
 * Pivot rule: a pivot <= 0 or NaN fails;
 * potrf returns the 1-based failing row, factor routines return the 1-based
 * failing block index; 0 means success.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define AT(a, ld, r, c) ((a)[(size_t)(r) * (ld) + (c)])

/* Cholesky of one n x n block, in place; strict upper triangle set to 0. */
int orc_potrf(int n, double *a)
{
    for (int j = 0; j < n; ++j) {
        double d = AT(a, n, j, j);
        for (int k = 0; k < j; ++k) d -= AT(a, n, j, k) * AT(a, n, j, k);
        if (!(d > 0.0)) return j + 1;
        double ljj = sqrt(d);
        AT(a, n, j, j) = ljj;
        for (int i = j + 1; i < n; ++i) {
            double s = AT(a, n, i, j);
            for (int k = 0; k < j; ++k) s -= AT(a, n, i, k) * AT(a, n, j, k);
            AT(a, n, i, j) = s / ljj;
        }
    }
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) AT(a, n, i, j) = 0.0;
    return 0;
}

/* e (m x n) <- e * l^{-T}, l lower n x n: solve x l^T = e row by row. */
void orc_trsm_right(int m, int n, double *e, const double *l)
{
    for (int r = 0; r < m; ++r)
        for (int j = 0; j < n; ++j) {
            double s = AT(e, n, r, j);
            for (int k = 0; k < j; ++k) s -= AT(e, n, r, k) * AT(l, n, j, k);
            AT(e, n, r, j) = s / AT(l, n, j, j);
        }
}

/* e (n x m) <- l^{-1} e, l lower n x n: forward substitution per column. */
void orc_trsm_left(int n, int m, double *e, const double *l)
{
    for (int c = 0; c < m; ++c)
        for (int i = 0; i < n; ++i) {
            double s = AT(e, m, i, c);
            for (int k = 0; k < i; ++k) s -= AT(l, n, i, k) * AT(e, m, k, c);
            AT(e, m, i, c) = s / AT(l, n, i, i);
        }
}

/* e (n x m) <- l^{-T} e: back substitution with l^T per column. */
void orc_trsm_left_trans(int n, int m, double *e, const double *l)
{
    for (int c = 0; c < m; ++c)
        for (int i = n - 1; i >= 0; --i) {
            double s = AT(e, m, i, c);
            for (int k = i + 1; k < n; ++k) s -= AT(l, n, k, i) * AT(e, m, k, c);
            AT(e, m, i, c) = s / AT(l, n, i, i);
        }
}

/* d (n x n) <- d - e e^T with e n x k (trans = 0), or d - e^T e with e k x n (trans = 1).
 * The full square is updated (d stays symmetric). */
void orc_syrk_down(int n, int k, double *d, const double *e, int trans)
{
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int t = 0; t < k; ++t)
                s += trans ? AT(e, n, t, i) * AT(e, n, t, j) : AT(e, k, i, t) * AT(e, k, j, t);
            AT(d, n, i, j) -= s;
        }
}

/* c (m x p) <- (accumulate ? c : 0) - a b, a m x n, b n x p. */
void orc_gemm_neg(int m, int n, int p, const double *a, const double *b, double *c, int accumulate)
{
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < p; ++j) {
            double s = 0.0;
            for (int t = 0; t < n; ++t) s += AT(a, n, i, t) * AT(b, p, t, j);
            AT(c, p, i, j) = (accumulate ? AT(c, p, i, j) : 0.0) - s;
        }
}

/* Algorithm 1. Dhat [N][n][n], Ehat [N-1][n][n]. */
int orc_seq_factor(int N, int n, const double *D, const double *E, double *Dhat, double *Ehat)
{
    const size_t nn = (size_t)n * n;
    memcpy(Dhat, D, nn * sizeof(double));
    if (orc_potrf(n, Dhat)) return 1;
    for (int i = 1; i < N; ++i) {
        double *Ei = Ehat + (size_t)(i - 1) * nn;
        double *Di = Dhat + (size_t)i * nn;
        memcpy(Ei, E + (size_t)(i - 1) * nn, nn * sizeof(double));
        orc_trsm_right(n, n, Ei, Dhat + (size_t)(i - 1) * nn);      /* trsm  n^3   */
        memcpy(Di, D + (size_t)i * nn, nn * sizeof(double));
        orc_syrk_down(n, n, Di, Ei, 0);                              /* syrk  n^3   */
        if (orc_potrf(n, Di)) return i + 1;                          /* potrf n^3/3 */
    }
    return 0;
}

/* Block forward/backward substitution with the Algorithm-1 factor. */
void orc_seq_solve(int N, int n, int m, const double *Dhat, const double *Ehat, const double *b,
                   double *x)
{
    const size_t nn = (size_t)n * n, nm = (size_t)n * m;
    memcpy(x, b, (size_t)N * nm * sizeof(double));
    /* forward: L y = b */
    for (int i = 0; i < N; ++i) {
        double *xi = x + (size_t)i * nm;
        if (i > 0) orc_gemm_neg(n, n, m, Ehat + (size_t)(i - 1) * nn, x + (size_t)(i - 1) * nm, xi, 1);
        orc_trsm_left(n, m, xi, Dhat + (size_t)i * nn);
    }
    /* backward: L^T x = y */
    double *t = (double *)malloc(nm * sizeof(double));
    for (int i = N - 1; i >= 0; --i) {
        double *xi = x + (size_t)i * nm;
        if (i < N - 1) {
            const double *Ei = Ehat + (size_t)i * nn; /* block (i+1, i) */
            const double *xn = x + (size_t)(i + 1) * nm;
            for (int r = 0; r < n; ++r)
                for (int c = 0; c < m; ++c) {
                    double s = 0.0;
                    for (int k = 0; k < n; ++k) s += AT(Ei, n, k, r) * AT(xn, m, k, c);
                    t[(size_t)r * m + c] = s;
                }
            for (size_t q = 0; q < nm; ++q) xi[q] -= t[q];
        }
        orc_trsm_left_trans(n, m, xi, Dhat + (size_t)i * nn);
    }
    free(t);
}

/* One system: factor + solve; returns info (0 or failing block, 1-based). */
int orc_seq_factor_solve(int N, int n, int m, const double *D, const double *E, const double *b,
                         double *Dhat, double *Ehat, double *x)
{
    int info = orc_seq_factor(N, n, D, E, Dhat, Ehat);
    if (info == 0) orc_seq_solve(N, n, m, Dhat, Ehat, b, x);
    return info;
}

typedef struct {
    int B, N, n, m, nthreads, tid;
    const double *D, *E, *b;
    double *x;
    int *info;
} batch_job;

static void *batch_worker(void *arg)
{
    batch_job *j = (batch_job *)arg;
    const size_t nn = (size_t)j->n * j->n, nm = (size_t)j->n * j->m;
    const size_t sD = (size_t)j->N * nn, sE = (size_t)(j->N > 0 ? j->N - 1 : 0) * nn,
                 sb = (size_t)j->N * nm;
    double *Dhat = (double *)malloc(sD * sizeof(double));
    double *Ehat = (double *)malloc((sE ? sE : 1) * sizeof(double));
    for (int s = j->tid; s < j->B; s += j->nthreads)
        j->info[s] = orc_seq_factor_solve(j->N, j->n, j->m, j->D + s * sD, j->E + s * sE,
                                          j->b + s * sb, Dhat, Ehat, j->x + s * sb);
    free(Dhat);
    free(Ehat);
    return NULL;
}

/* Batch driver: B independent systems round-robin over nthreads host threads. */
int orc_seq_batch(int B, int N, int n, int m, const double *D, const double *E, const double *b,
                  double *x, int *info, int nthreads)
{
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    batch_job *jobs = (batch_job *)malloc(sizeof(batch_job) * nthreads);
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (batch_job){B, N, n, m, nthreads, t, D, E, b, x, info};
        pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    int bad = 0;
    for (int s = 0; s < B; ++s) bad += info[s] != 0;
    return bad;
}
