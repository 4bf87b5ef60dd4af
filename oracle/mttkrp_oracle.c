/* Full-size CPU oracle for the ALTO MTTKRP -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library; the product package (paper_2102_10245_b200/) never does.
 *
 * It restates the reference's coordinate-list oracle
 *   /root/reference/pkg/src/altotensor/mttkrp.py:64-77 (mttkrp_oracle)
 * in plain C so that it finishes at BASELINE.json's full sizes (cfg5: 500M
 * nonzeros) on the GPU box's host cores:
 *
 *   contrib = values[:, None]                       (mttkrp.py:71)
 *   for n != mode, ascending: contrib = contrib * F_n[coords[:, n]]   (:72-74)
 *   np.add.at(out, coords[:, mode], contrib)        (:75, element order)
 *
 * Arithmetic is float64 in exactly that order (value times the factors in
 * ascending mode order, then one add per element into its output row, in
 * input order), compiled with -ffp-contract=off, so the result is bitwise
 * equal to the reference's on the same inputs (pinned against fixtures the
 * reference produced: tests/test_oracle_c.py).  Threads own disjoint output
 * rows (row mod threads, threads a power of two) and each scans the whole coordinate list, so every
 * row still receives its elements in input order: the thread count does not
 * change a single bit.
 *
 * Coordinates come per mode as int32 arrays (column-major (N, M)), values as
 * float32 (fp32 configs: upcast exactly) or float64.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_MAX_ORDER 8

typedef struct {
    int order, mode, rank, val_f32, tid, nthreads;
    int64_t m, dim_out;
    const int32_t* const* coords;
    const void* values;
    const double* const* factors;
    double* out;
} job_t;

static void* mttkrp_worker(void* p) {
    job_t* j = (job_t*)p;
    const int R = j->rank, mode = j->mode, T = j->nthreads, t = j->tid;
    const int32_t* rows = j->coords[mode];
    int ins[ORACLE_MAX_ORDER];
    int nin = 0;
    for (int n = 0; n < j->order; ++n)
        if (n != mode) ins[nin++] = n;
    double c[256];
    for (int64_t e = 0; e < j->m; ++e) {
        const int64_t r = rows[e];
        if ((r & (T - 1)) != t) continue; /* T is a power of two */
        const double v = j->val_f32 ? (double)((const float*)j->values)[e] : ((const double*)j->values)[e];
        for (int k = 0; k < R; ++k) c[k] = v;
        for (int i = 0; i < nin; ++i) {
            const int n = ins[i];
            const double* f = j->factors[n] + (int64_t)j->coords[n][e] * R;
            for (int k = 0; k < R; ++k) c[k] = c[k] * f[k];
        }
        double* o = j->out + r * R;
        for (int k = 0; k < R; ++k) o[k] = o[k] + c[k];
    }
    return NULL;
}

/* out (dim_out, rank) float64 is overwritten.  Returns 0, or 1 on bad
 * arguments, 2 if a coordinate of the output mode is out of range. */
int oracle_mttkrp_coo(int order, int mode, int64_t m, int rank, const int32_t* const* coords, const void* values,
                      int val_f32, const double* const* factors, double* out, int64_t dim_out, int threads) {
    if (order < 1 || order > ORACLE_MAX_ORDER || mode < 0 || mode >= order || rank < 1 || rank > 256 || m < 0)
        return 1;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    while (threads & (threads - 1)) threads &= threads - 1; /* round down to a power of two */
    memset(out, 0, (size_t)dim_out * rank * sizeof(double));
    for (int64_t e = 0; e < m; ++e)
        if (coords[mode][e] < 0 || coords[mode][e] >= dim_out) return 2;
    pthread_t th[256];
    job_t jobs[256];
    for (int t = 0; t < threads; ++t) {
        job_t jb = {order, mode, rank, val_f32, t, threads, m, dim_out, coords, values, factors, out};
        jobs[t] = jb;
    }
    if (threads == 1) {
        mttkrp_worker(&jobs[0]);
        return 0;
    }
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, mttkrp_worker, &jobs[t]);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    return 0;
}

/* ||a - b||_F^2 and ||b||_F^2 in float64 (a: float32 or float64, b float64),
 * for the relative Frobenius error of the reference's tests
 * (pkg/tests/conftest.py:35-38). */
typedef struct {
    const void* a;
    int a_f32;
    const double* b;
    int64_t lo, hi;
    double d2, n2;
} err_job_t;

static void* err_worker(void* p) {
    err_job_t* j = (err_job_t*)p;
    double d2 = 0.0, n2 = 0.0;
    for (int64_t i = j->lo; i < j->hi; ++i) {
        const double x = j->a_f32 ? (double)((const float*)j->a)[i] : ((const double*)j->a)[i];
        const double d = x - j->b[i];
        d2 += d * d;
        n2 += j->b[i] * j->b[i];
    }
    j->d2 = d2;
    j->n2 = n2;
    return NULL;
}

void oracle_diff_norms(const void* a, int a_f32, const double* b, int64_t n, int threads, double* d2_out,
                       double* n2_out) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    err_job_t jobs[256];
    for (int t = 0; t < threads; ++t) {
        err_job_t jb = {a, a_f32, b, n * t / threads, n * (t + 1) / threads, 0.0, 0.0};
        jobs[t] = jb;
        pthread_create(&th[t], NULL, err_worker, &jobs[t]);
    }
    double d2 = 0.0, n2 = 0.0;
    for (int t = 0; t < threads; ++t) {
        pthread_join(th[t], NULL);
        d2 += jobs[t].d2;
        n2 += jobs[t].n2;
    }
    *d2_out = d2;
    *n2_out = n2;
}
