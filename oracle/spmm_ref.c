/* oracle/spmm_ref.c -- O1: the plain definition Y = A X in fp64 on the CPU.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header or constant with the CUDA product path (paper_2402_19364_b200/).
 *
 * What it computes (§2 "Background": "compute the product Y = AX"):
 *     Y[r, :] = sum over stored entries e of row r (in stored column order) of val[e] * X[col[e], :]
 * accumulated in fp64.  The arrow method reaches exactly this result in exact
 * arithmetic because Eq. (1) partitions A's entries ("each edge
 * occurs in exactly one matrix of the decomposition"), so the oracle is
 * the definition itself and never touches a decomposition.
 *
 * Rows are independent; OpenMP parallelises over rows only (no reordering of any
 * row's summation).  X may be fp64 or fp32 (converted exactly to fp64 per load).
 */
#include <stdint.h>
#include <omp.h>

static void row_f64(int64_t r, const int64_t *rp, const int32_t *col, const double *val,
                    const double *X, int64_t k, double *y) {
    for (int64_t j = 0; j < k; ++j) y[j] = 0.0;
    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
        const double a = val[e];
        const double *x = X + (int64_t)col[e] * k;
        for (int64_t j = 0; j < k; ++j) y[j] += a * x[j];
    }
}

static void row_xf32(int64_t r, const int64_t *rp, const int32_t *col, const double *val,
                     const float *X, int64_t k, double *y) {
    for (int64_t j = 0; j < k; ++j) y[j] = 0.0;
    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
        const double a = val[e];
        const float *x = X + (int64_t)col[e] * k;
        for (int64_t j = 0; j < k; ++j) y[j] += a * (double)x[j];
    }
}

int oracle_num_threads(void) { return omp_get_max_threads(); }

/* Y (n x k, fp64) = A X over all rows. nthreads <= 0: OpenMP default. */
void oracle_spmm(int64_t n, const int64_t *rp, const int32_t *col, const double *val,
                 const void *X, int32_t x_is_f32, int64_t k, double *Y, int32_t nthreads) {
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t r = 0; r < n; ++r) {
        if (x_is_f32) row_xf32(r, rp, col, val, (const float *)X, k, Y + r * k);
        else          row_f64(r, rp, col, val, (const double *)X, k, Y + r * k);
    }
}

/* Y rows for a sample of row ids only: Yout[s, :] = (A X)[rows[s], :]. */
void oracle_spmm_rows(const int64_t *rp, const int32_t *col, const double *val,
                      const void *X, int32_t x_is_f32, int64_t k,
                      const int64_t *rows, int64_t nrows, double *Yout, int32_t nthreads) {
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t s = 0; s < nrows; ++s) {
        if (x_is_f32) row_xf32(rows[s], rp, col, val, (const float *)X, k, Yout + s * k);
        else          row_f64(rows[s], rp, col, val, (const double *)X, k, Yout + s * k);
    }
}
