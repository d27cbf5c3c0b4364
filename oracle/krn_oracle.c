/* TEST INFRASTRUCTURE - CPU oracle, not product code.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
 * load the library built from this file.  The product (libkrn_b200.so) never
 * links or calls it.
 *
 * Plain-C restatement of what the reference interpreter computes for the
 * headline objective (programs/laplacian.krn) and for the bulk builtins, at
 * the reference's own statement granularity and in its canonical summation
 * order, so results are bit-comparable with the reference at any size.
 * Parity status: PINNED against tests/golden/ (outputs of the reference run
 * in the build container, see oracle/make_golden.py) and the reference's
 * known-answer tests.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC  (oracle/build.py)
 * -ffp-contract=off matters: the reference contract is IEEE double with no
 * fused multiply-add.
 *
 * Reference locations restated here (paths under /root/reference/pkg):
 *   pairwise tree            src/krn/runtime.py:166-177
 *   gather into a scalar     src/krn/runtime.py:643-651
 *   fill / copy              src/krn/runtime.py:628-641
 *   dst += src, dst += s     src/krn/runtime.py:653-665
 *   deferred atomics order   src/krn/runtime.py:430-447, 615-620
 *   laplacian forward        programs/laplacian.krn:4-21
 *   laplacian gradient       tests/test_adjoint.py:43-94 (golden emitted text)
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#define KRN_OMP_FOR _Pragma("omp parallel for schedule(static) if (n > 65536)")
int krn_oracle_threads(void) { return omp_get_max_threads(); }
#else
#define KRN_OMP_FOR
int krn_oracle_threads(void) { return 1; }
#endif

/* ---- bulk builtins ------------------------------------------------------ */

/* Adjacent-pair tree over v[0..n); a level of odd length is padded with +0.0.
 * scratch must hold n doubles (contents destroyed); v is not modified. */
double krn_oracle_pairwise_sum(const double *v, size_t n, double *scratch)
{
    if (n == 0) return 0.0;
    memcpy(scratch, v, n * sizeof(double));
    size_t m = n;
    while (m > 1) {
        size_t half = m / 2;
        for (size_t i = 0; i < half; ++i) scratch[i] = scratch[2 * i] + scratch[2 * i + 1];
        if (m & 1) { scratch[half] = scratch[m - 1] + 0.0; }
        m = (m + 1) / 2;
    }
    return scratch[0];
}

void krn_oracle_fill(double *v, size_t n, double s) { for (size_t i = 0; i < n; ++i) v[i] = s; }
void krn_oracle_copy(double *dst, const double *src, size_t n) { memcpy(dst, src, n * sizeof(double)); }
void krn_oracle_add_scalar(double *v, size_t n, double s) { for (size_t i = 0; i < n; ++i) v[i] += s; }
void krn_oracle_add_view(double *dst, const double *src, size_t n) { for (size_t i = 0; i < n; ++i) dst[i] += src[i]; }

/* ---- headline objective: normRes1DLaplacianSQ ---------------------------- */

/* forward sweep, statement by statement (two kernels).  y, y2 are the
 * function's local views (n doubles each, zero-initialised by the caller the
 * way DeclView does).  x is scaled in place. */
static void laplacian_forward(double *x, const double *b, double *y, double *y2, size_t n)
{
    /* iterations of a parallel_for are independent: the reference runs them on a thread
     * pool (runtime.py:594-613); here OpenMP plays that role for the order-free loops */
    KRN_OMP_FOR
    for (size_t j0 = 0; j0 < n; ++j0) x[j0] = 3.0 * x[j0];
    KRN_OMP_FOR
    for (size_t j = 0; j < n; ++j) {
        y[j] = 2.0 * x[j] - b[j];
        if (j != 0)     y[j] -= x[j - 1];
        if (j != n - 1) y[j] -= x[j + 1];
        y2[j] = y[j] * y[j];
    }
}

/* Primal: returns f, leaves x scaled.  work must hold 3n doubles. */
double krn_oracle_laplacian_primal(double *x, const double *b, size_t n, double *work)
{
    double *y = work, *y2 = work + n, *scratch = work + 2 * n;
    memset(y, 0, 2 * n * sizeof(double));
    laplacian_forward(x, b, y, y2, n);
    double sum = 0.0 + krn_oracle_pairwise_sum(y2, n, scratch); /* sum = 0.0 + total */
    return sum;
}

/* Gradient function normRes1DLaplacianSQ_grad(x, b, _d_x, _d_b) with seed
 * literal `seed` (1.0 for a plain gradient).  Accumulates into dx, db; leaves x
 * scaled.  work must hold 5n doubles.  Every statement of the emitted text is
 * kept, including the ones that cancel, so non-finite and signed-zero
 * behaviour matches the interpreter bit for bit.  The deferred atomic adds of
 * the reverse stencil kernel are applied by a sequential ascending-j loop,
 * which is exactly the (iteration, program-order) order the reference sorts
 * into; nothing in that kernel reads _d_x, so immediate application is
 * indistinguishable from deferred.  That loop (and the pairwise tree) stay
 * sequential: their order IS the result.  The order-free loops use OpenMP. */
void krn_oracle_laplacian_grad(double *x, const double *b, double *dx, double *db,
                               size_t n, double seed, double *work)
{
    double *d_y = work, *d_y2 = work + n, *y = work + 2 * n, *y2 = work + 3 * n,
           *scratch = work + 4 * n;
    memset(work, 0, 4 * n * sizeof(double));          /* four DeclView zero-fills */
    double d_sum = 0.0;
    laplacian_forward(x, b, y, y2, n);
    double sum = 0.0 + krn_oracle_pairwise_sum(y2, n, scratch); /* dead, kept: the forward is verbatim */
    (void)sum;
    d_sum += seed;
    KRN_OMP_FOR
    for (size_t j = 0; j < n; ++j) d_y2[j] += d_sum;  /* parallel_sum(_d_y2, _d_sum) */

    for (size_t j = 0; j < n; ++j) {                  /* reverse of the stencil kernel */
        double r4 = d_y2[j];
        d_y2[j] -= r4;
        d_y[j] += r4 * y[j];
        d_y[j] += y[j] * r4;
        if (j != n - 1) {
            double r3 = d_y[j];
            d_y[j] -= r3;
            d_y[j] += r3;
            dx[j + 1] += -r3;                         /* atomic_add(_d_x(j + 1), -_r_d3) */
        }
        if (j != 0) {
            double r2 = d_y[j];
            d_y[j] -= r2;
            d_y[j] += r2;
            dx[j - 1] += -r2;                         /* atomic_add(_d_x(j - 1), -_r_d2) */
        }
        double r1 = d_y[j];
        d_y[j] -= r1;
        dx[j] += 2.0 * r1;                            /* atomic_add(_d_x(j), 2.0 * _r_d1) */
        db[j] += -r1;
    }
    KRN_OMP_FOR
    for (size_t j0 = 0; j0 < n; ++j0) {               /* reverse of the scale kernel */
        double r0 = dx[j0];
        dx[j0] -= r0;
        dx[j0] += 3.0 * r0;
    }
}

/* ---- deferred atomic_add queue, applied in order (runtime.py:615-620) -------------------
 * records r = 0..records-1 are already in (iteration, program order); record r adds its
 * `width` values, one after the other, to target[keys[r]].  keys[r] >= target_size marks a
 * site that did not execute. */
void krn_oracle_apply_queue(double *target, size_t target_size, const uint32_t *keys, const double *vals,
                            size_t records, int width)
{
    for (size_t r = 0; r < records; ++r) {
        if (keys[r] >= target_size) continue;
        for (int w = 0; w < width; ++w) target[keys[r]] = target[keys[r]] + vals[r * (size_t)width + w];
    }
}
