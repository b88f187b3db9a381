/*
 * sdnn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU evaluation of the sparse-DNN inference
 * that the CUDA path (paper_2004_10908_b200/) accelerates.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  It shares no code, header, table or helper with the
 * CUDA path; the only thing both sides consume is the seeded generator output
 * (sdnngen/), which holds none of the method's arithmetic.
 *
 * What it computes (one layer, every row i, every output neuron j):
 *
 *     Y_{l+1}[i][j] = min(max( sum_k Y_l[i][k] * W_l[k][j]  +  b_l[j], 0), YMAX)
 *
 *   - the formula and YMAX = 32: BASELINE.json north_star ("every layer
 *     computes Y_{l+1} = min(max(Y_l.W_l + b_l, 0), 32)");
 *   - dataset parts (input matrix, per-layer sparse W, bias, truth
 *     categories): PAPER.md:2557-2559 (Sec. 7.4, LSDNN);
 *   - categories = rows still nonzero after the last layer: north_star, and
 *     "Other CPU tasks evaluate the results with a golden reference"
 *     PAPER.md:2570.
 *
 * Readings where the paper is silent:
 *   A5  the sum is evaluated in fp32 as a chain of correctly rounded fmaf in
 *       ASCENDING source index k, starting from +0.0f; the bias is added by a
 *       separate fp32 addition; A6 the clamp is  z > 0 ? fminf(z, ymax) : +0.
 *   A2  the bias is added to every entry (dense), not only to nonzero sums.
 *   A7  category(i) = exists j: Y_L[i][j] > 0 ; with zero layers, Y_0 itself.
 *
 * Why this loop realises A5: W_l arrives as CSR with rows = input neuron k.
 * The loop visits k = 0, 1, ..., N-1 in order and, for each stored (k, j, w),
 * does z[j] = fmaf(Y[i][k], w, z[j]).  Column j therefore receives its terms in
 * ascending k -- exactly the canonical chain -- and the order of entries inside
 * a CSR row is irrelevant (each touches a different j; duplicates are invalid
 * input).
 *
 * skip_zero (optional): a term with Y[i][k] == 0 is skipped.  This is exact:
 * fmaf(+-0, w, z) = z + (+-0) = z for finite w when z != 0, and = +0 when
 * z == +0; z is never -0 because it starts at +0 and an RN sum is -0 only if
 * both addends are -0.  tests/test_oracle_pins.py checks skip/no-skip equality.
 *
 * Compiled with  gcc -O2 -ffp-contract=off  (no -ffast-math), so the compiler
 * neither fuses nor reorders anything beyond the explicit fmaf calls.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- input */

/* Y0 (CSR: rowptr[B+1], idx[nnz], val[nnz] or NULL meaning 1.0f) into the
 * dense row-major Y[B][n] ("a sparse matrix of the input data").
 * Returns 0, or -1 on an out-of-range index / non-monotone rowptr. */
int oracle_densify(int32_t n, int64_t B, const int64_t *rowptr, const int32_t *idx,
                   const float *val, float *Y) {
    memset(Y, 0, sizeof(float) * (size_t)n * (size_t)B);
    for (int64_t i = 0; i < B; ++i) {
        if (rowptr[i + 1] < rowptr[i]) return -1;
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            if (idx[e] < 0 || idx[e] >= n) return -1;
            Y[i * (int64_t)n + idx[e]] = val ? val[e] : 1.0f;
        }
    }
    return 0;
}

/* ---------------------------------------------------------------- layer */

typedef struct {
    int32_t n;
    int64_t r0, r1;
    const float *Yin;
    float *Yout;
    const int64_t *w_rowptr;
    const int32_t *w_colidx;
    const float *w_val;
    float w_uniform;
    const float *bias;
    float ymax;
    int32_t skip_zero;
} layer_job;

static void *layer_rows(void *arg) {
    const layer_job *J = (const layer_job *)arg;
    const int32_t n = J->n;
    for (int64_t i = J->r0; i < J->r1; ++i) {
        const float *y = J->Yin + i * (int64_t)n;
        float *z = J->Yout + i * (int64_t)n;
        for (int32_t j = 0; j < n; ++j) z[j] = 0.0f;              /* chain starts at +0 */
        for (int32_t k = 0; k < n; ++k) {                          /* ascending source k */
            const float yk = y[k];
            if (J->skip_zero && yk == 0.0f) continue;
            for (int64_t e = J->w_rowptr[k]; e < J->w_rowptr[k + 1]; ++e) {
                const int32_t j = J->w_colidx[e];
                const float w = J->w_val ? J->w_val[e] : J->w_uniform;
                z[j] = fmaf(yk, w, z[j]);                          /* one rounding per term */
            }
        }
        for (int32_t j = 0; j < n; ++j) {
            const float s = z[j] + J->bias[j];                     /* separate RN add */
            z[j] = (s > 0.0f) ? fminf(s, J->ymax) : 0.0f;          /* clamp to [0, ymax] */
        }
    }
    return NULL;
}

/* One layer for rows [0, B): Yout = clamp(Yin . W + b).  Yin, Yout are dense
 * row-major [B][n] and must not alias.  nthreads <= 1 runs on the caller. */
int oracle_layer(int32_t n, int64_t B, const float *Yin, float *Yout,
                 const int64_t *w_rowptr, const int32_t *w_colidx, const float *w_val,
                 float w_uniform, const float *bias, float ymax, int32_t skip_zero,
                 int32_t nthreads) {
    if (n < 1 || B < 0 || Yin == Yout) return -1;
    if (w_rowptr[0] != 0) return -1;
    for (int32_t k = 0; k < n; ++k) {
        if (w_rowptr[k + 1] < w_rowptr[k]) return -1;
        for (int64_t e = w_rowptr[k]; e < w_rowptr[k + 1]; ++e)
            if (w_colidx[e] < 0 || w_colidx[e] >= n) return -1;
    }
    if (nthreads < 1) nthreads = 1;
    if (nthreads > B) nthreads = (int32_t)(B > 0 ? B : 1);
    layer_job *jobs = (layer_job *)calloc((size_t)nthreads, sizeof(layer_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return -2; }
    for (int32_t t = 0; t < nthreads; ++t) {
        layer_job *J = &jobs[t];
        J->n = n; J->Yin = Yin; J->Yout = Yout;
        J->w_rowptr = w_rowptr; J->w_colidx = w_colidx; J->w_val = w_val;
        J->w_uniform = w_uniform; J->bias = bias; J->ymax = ymax; J->skip_zero = skip_zero;
        J->r0 = B * t / nthreads;
        J->r1 = B * (t + 1) / nthreads;
    }
    for (int32_t t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, layer_rows, &jobs[t]);
    layer_rows(&jobs[0]);
    for (int32_t t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
    return 0;
}

/* ----------------------------------------------------------- categories */

/* cat[i] = 1 iff some Y[i][j] > 0 (reading A7).  Returns the count. */
int64_t oracle_categories(int32_t n, int64_t B, const float *Y, uint8_t *cat) {
    int64_t c = 0;
    for (int64_t i = 0; i < B; ++i) {
        uint8_t a = 0;
        for (int32_t j = 0; j < n; ++j)
            if (Y[i * (int64_t)n + j] > 0.0f) { a = 1; break; }
        cat[i] = a;
        c += a;
    }
    return c;
}

/* Number of rows with at least one nonzero entry (the survivor profile). */
int64_t oracle_live_rows(int32_t n, int64_t B, const float *Y) {
    int64_t c = 0;
    for (int64_t i = 0; i < B; ++i)
        for (int32_t j = 0; j < n; ++j)
            if (Y[i * (int64_t)n + j] != 0.0f) { ++c; break; }
    return c;
}
