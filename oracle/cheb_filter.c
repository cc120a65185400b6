/* Plain-C restatement of the reference Chebyshev filter — TEST INFRASTRUCTURE ONLY.
 *
 * Follows /root/reference/pkg/src/cscluster/filters.py:
 *   apply_filter      filters.py:155-187
 *     shifted(v) = v - s * (A @ v)          filters.py:172-176
 *     out = c0*x; T1 = shifted(x); out = out + c1*T1
 *     T_{j+1} = 2*shifted(T_j) - T_{j-1}; out += c_j*T_{j+1}   filters.py:178-186
 *   _count_from_block filters.py:190-196
 * with SciPy's csr_matvecs row loop (A @ V for a C-order dense block: y
 * zero-initialised, y_i += a_ij * v_j over the stored nonzeros in order)
 * inlined. Compiled with -ffp-contract=off so every multiply and add rounds
 * separately, like the numpy temporaries and the non-FMA SciPy build.
 *
 * Rows are independent within one order, so the pthread row split does not
 * change any result bit. Used by tests (checker) and by bench.py's
 * cpu_baseline / --impl reference legs (timed CPU baseline, "kind": "port").
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

typedef struct {
    int64_t n, d;
    const int32_t *indptr, *indices;
    const double *data;
    const double *x;       /* order 1: input block */
    const double *t_prev;  /* order >= 2 */
    const double *t_cur;   /* gathered block */
    double *t_next, *out;
    double s, c0, c1, cj;
    int first;             /* 1: order 1 epilogue */
    int64_t row_begin, row_end;
} order_job;

/* y = v - s * (A v) for one row; tmp is a d-vector scratch. */
static inline void shifted_row(int64_t i, const order_job *J, const double *v, double *tmp,
                               double *y) {
    const int64_t d = J->d;
    for (int64_t c = 0; c < d; ++c) tmp[c] = 0.0;
    for (int32_t jj = J->indptr[i]; jj < J->indptr[i + 1]; ++jj) {
        const double a = J->data[jj];
        const double *vr = v + (int64_t)J->indices[jj] * d;
        for (int64_t c = 0; c < d; ++c) tmp[c] += a * vr[c];
    }
    const double *vi = v + i * d;
    for (int64_t c = 0; c < d; ++c) y[c] = vi[c] - J->s * tmp[c];
}

static void *run_rows(void *arg) {
    const order_job *J = (const order_job *)arg;
    const int64_t d = J->d;
    double *tmp = (double *)malloc(sizeof(double) * (size_t)d);
    double *sh = (double *)malloc(sizeof(double) * (size_t)d);
    for (int64_t i = J->row_begin; i < J->row_end; ++i) {
        double *oi = J->out + i * d;
        if (J->first) {
            double *t1 = J->t_next + i * d;
            shifted_row(i, J, J->x, tmp, t1);
            const double *xi = J->x + i * d;
            for (int64_t c = 0; c < d; ++c) {
                const double base = J->c0 * xi[c];
                oi[c] = base + J->c1 * t1[c];
            }
        } else {
            shifted_row(i, J, J->t_cur, tmp, sh);
            const double *pi = J->t_prev + i * d;
            double *ni = J->t_next + i * d;
            for (int64_t c = 0; c < d; ++c) {
                const double two = 2.0 * sh[c];
                ni[c] = two - pi[c];
                oi[c] += J->cj * ni[c];
            }
        }
    }
    free(tmp);
    free(sh);
    return NULL;
}

int oracle_num_threads(void) {
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int)c : 1;
}

static void run_order(const order_job *proto, int nthreads) {
    if (nthreads <= 1 || proto->n < 1024) {
        order_job J = *proto;
        J.row_begin = 0;
        J.row_end = proto->n;
        run_rows(&J);
        return;
    }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    order_job *jobs = (order_job *)malloc(sizeof(order_job) * (size_t)nthreads);
    const int64_t chunk = (proto->n + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = *proto;
        jobs[t].row_begin = t * chunk < proto->n ? t * chunk : proto->n;
        jobs[t].row_end = (t + 1) * chunk < proto->n ? (t + 1) * chunk : proto->n;
        pthread_create(&th[t], NULL, run_rows, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
}

/* out = h(L) x.  work must hold 2*n*d doubles.  Returns 0, or -1 on bad args.
 * ncoeffs >= 2; runs ncoeffs-1 SpMM blocks ("orders"), like the reference.
 * nthreads <= 0 means all online cores. */
int oracle_cheb_filter_f64(int64_t n, const int32_t *indptr, const int32_t *indices,
                           const double *data, int64_t d, const double *x,
                           const double *coeffs, int32_t ncoeffs, double lambda_max,
                           double *out, double *work, int32_t nthreads) {
    if (n < 0 || d < 1 || ncoeffs < 2 || lambda_max <= 0.0) return -1;
    if (nthreads <= 0) nthreads = oracle_num_threads();
    order_job J;
    memset(&J, 0, sizeof(J));
    J.n = n;
    J.d = d;
    J.indptr = indptr;
    J.indices = indices;
    J.data = data;
    J.x = x;
    J.s = 2.0 / lambda_max;
    J.out = out;
    double *ta = work, *tb = work + n * d;
    /* order 1: T1 = shifted(x) into ta; out = c0*x + c1*T1 */
    J.first = 1;
    J.c0 = coeffs[0];
    J.c1 = coeffs[1];
    J.t_next = ta;
    run_order(&J, nthreads);
    /* orders 2..: T_{j+1} = 2 shifted(T_j) - T_{j-1}; from order 3 on it
     * overwrites T_{j-1} in place (each row reads its own entries first) */
    const double *t_prev = x;
    double *t_cur = ta, *t_next = tb;
    J.first = 0;
    for (int32_t j = 2; j < ncoeffs; ++j) {
        J.cj = coeffs[j];
        J.t_prev = t_prev;
        J.t_cur = t_cur;
        J.t_next = t_next;
        run_order(&J, nthreads);
        t_prev = t_cur;
        t_cur = t_next;
        t_next = (double *)t_prev;
    }
    return 0;
}

/* plain sequential sum of squares (checker only; decisions are compared with
 * tolerance in the tests, numpy's pairwise order is not reproduced) */
double oracle_sumsq_f64(int64_t count, const double *x) {
    double acc = 0.0;
    for (int64_t i = 0; i < count; ++i) acc += x[i] * x[i];
    return acc;
}
