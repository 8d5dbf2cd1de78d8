/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the PentaRAG flat-index scan.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.  The product path never links
 * or calls it.
 *
 * What it restates (reference paths relative to /root/reference/pkg/src/ragcascade):
 *
 *   index.py:173   scores = np.einsum("ij,j->i", self._vectors64[:n], q64)
 *   index.py:176   order  = np.lexsort((np.arange(n), -scores))[:take]
 *   index.py:179-185 self-snap to 1.0 + clamp to [-1, 1]
 *
 * The arithmetic lives in numpy (third-party, pinned only as numpy>=1.24 in
 * pkg/pyproject.toml:11; numpy 2.3.5 in this image).  Its einsum inner loop
 * for "ij,j->i" on float64 is sum_of_products_contig_contig_outstride0_two
 * compiled for the x86-64 baseline (SSE/SSE2/SSE3 — `numpy.show_config()`),
 * i.e. 2-lane vectors, no FMA, 4 vectors unrolled:
 *
 *     for each block of 8 elements:
 *         acc = p0 + (p1 + (p2 + (p3 + acc)))      (pi = i-th 2-lane product)
 *     tail: 2 elements at a time, zero padded:  acc = p + acc
 *     result = 0.0 + (acc.lane0 + acc.lane1)
 *
 * Products of float32 values are exact in float64, so fma(x, q, acc) equals
 * x*q + acc here and either form reproduces einsum bit-for-bit.  The order
 * was verified against np.einsum on d in {4,8,13,16,64,384,768,1000,1001,
 * 1023,1024} (tests/test_oracle.py re-checks it wherever the tests run).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

double oracle_einsum_dot(const float *x, const float *q, int d) {
    double a0 = 0.0, a1 = 0.0;
    int j = 0;
    for (; j + 8 <= d; j += 8) {
        /* lane 0 sees elements 0,2,4,6 ; lane 1 sees 1,3,5,7 */
        double t0 = (double)x[j + 6] * (double)q[j + 6] + a0;
        double t1 = (double)x[j + 7] * (double)q[j + 7] + a1;
        t0 = (double)x[j + 4] * (double)q[j + 4] + t0;
        t1 = (double)x[j + 5] * (double)q[j + 5] + t1;
        t0 = (double)x[j + 2] * (double)q[j + 2] + t0;
        t1 = (double)x[j + 3] * (double)q[j + 3] + t1;
        a0 = (double)x[j + 0] * (double)q[j + 0] + t0;
        a1 = (double)x[j + 1] * (double)q[j + 1] + t1;
    }
    for (; j < d; j += 2) {
        double p0 = (double)x[j] * (double)q[j];
        double p1 = (j + 1 < d) ? (double)x[j + 1] * (double)q[j + 1] : 0.0;
        a0 = p0 + a0;
        a1 = p1 + a1;
    }
    return 0.0 + (a0 + a1);
}

void oracle_scores(const float *X, int64_t n, int d, const float *q, double *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_einsum_dot(X + i * (int64_t)d, q, d);
}

/* top-k by (score desc, row asc); rows arrive in ascending order, so a later
 * row never displaces an equal score (lexsort's secondary key). */
static void topk_push(double s, int64_t r, int k, int *cnt, double *ts, int64_t *tr) {
    int c = *cnt;
    if (c == k && !(s > ts[k - 1])) return;
    int pos = (c < k) ? c : k - 1;
    while (pos > 0 && s > ts[pos - 1]) {
        ts[pos] = ts[pos - 1];
        tr[pos] = tr[pos - 1];
        --pos;
    }
    ts[pos] = s;
    tr[pos] = r;
    if (c < k) *cnt = c + 1;
}

static void search_one(const float *X, int64_t n, int d, const float *q, int k,
                       int64_t *tr, double *ts, double *rep, int32_t *cnt) {
    int c = 0;
    for (int64_t i = 0; i < n; ++i)
        topk_push(oracle_einsum_dot(X + i * (int64_t)d, q, d), i, k, &c, ts, tr);
    for (int j = 0; j < k; ++j) {
        if (j >= c) {
            tr[j] = -1;
            ts[j] = 0.0;
            rep[j] = 0.0;
            continue;
        }
        double s = ts[j];
        if (s > 1.0 - 1e-6) {
            const float *x = X + tr[j] * (int64_t)d;
            int eq = 1; /* np.array_equal: elementwise ==, so -0.0 == 0.0 */
            for (int t = 0; t < d; ++t)
                if (!(x[t] == q[t])) { eq = 0; break; }
            if (eq) s = 1.0;
        }
        rep[j] = s < -1.0 ? -1.0 : (s > 1.0 ? 1.0 : s);
    }
    *cnt = c;
}

typedef struct {
    const float *X, *Q;
    int64_t n, b, next;
    int d, k;
    int64_t *rows;
    double *raw, *rep;
    int32_t *count;
    pthread_mutex_t mu;
} search_job;

static void *search_worker(void *arg) {
    search_job *j = (search_job *)arg;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        int64_t qi = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (qi >= j->b) return NULL;
        search_one(j->X, j->n, j->d, j->Q + qi * (int64_t)j->d, j->k, j->rows + qi * j->k,
                   j->raw + qi * j->k, j->rep + qi * j->k, j->count + qi);
    }
}

/*
 * Full FlatIndex.search semantics for a batch of queries over rows [0, n).
 * rows/raw/reported are [b, k]; count[b] = min(k, n).  Unused slots get
 * row -1.  Queries are spread over `nthreads` POSIX threads.  Returns 0, or
 * -1 on bad arguments.
 */
int oracle_search(const float *X, int64_t n, int d, const float *Q, int64_t b, int k,
                  int64_t *rows, double *raw, double *reported, int32_t *count, int nthreads) {
    if (k < 1 || d < 1 || n < 0 || b < 0) return -1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > b) nthreads = (int)(b > 0 ? b : 1);
    search_job job = {X, Q, n, b, 0, d, k, rows, raw, reported, count, PTHREAD_MUTEX_INITIALIZER};
    pthread_t th[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, search_worker, &job);
    search_worker(&job);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    return 0;
}

/* exact scores for an explicit (query, row) candidate list — used by tests
 * that check the device rescoring stage in isolation. */
void oracle_pair_scores(const float *X, int d, const float *Q, const int64_t *qidx,
                        const int64_t *ridx, int64_t m, double *out) {
    for (int64_t i = 0; i < m; ++i)
        out[i] = oracle_einsum_dot(X + ridx[i] * (int64_t)d, Q + qidx[i] * (int64_t)d, d);
}
