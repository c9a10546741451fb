/*
 * oracle/kgc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU brute force of the knowledge-graph
 * completion problem.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant with the CUDA path (paper_2307_12059_b200/).
 *
 * What it computes (citations are PAPER.md line numbers):
 *   Definition 1: all (e_i, r_j, e_k) with dist3(e_i, r_j, e_k) <= eps.
 *   TransE:         dist3(h, r, t) = || h + r - t ||_{L_p},  p in {1, 2}.
 *   Straightforward algorithm (Fig. naive): triple loop, check
 *   dist3 <= eps ("Line 5"), append the triplet.
 *
 * Precision: the paper is silent (reading R8).  Every value is
 * widened to double before use; the sum over k runs in index order in FP64;
 * L2 is the non-squared norm sqrt(sum) (reading R2); the bound is inclusive
 * ("<=", reading R4); self edges are kept (reading R5).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t h, r, t, pad;
    double dist;
} kgco_triplet;

/* dist3(h, r, t) = || h + r - t ||_p, FP64, index order. */
double kgco_dist3(const float *h, const float *r, const float *t, int32_t d, int32_t p)
{
    double s = 0.0;
    for (int32_t k = 0; k < d; ++k) {
        double q = (double)h[k] + (double)r[k];   /* connector1(h, r) = h + r */
        double x = q - (double)t[k];              /* connector2(t, r) = t     */
        if (p == 1)
            s += fabs(x);
        else
            s += x * x;
    }
    return p == 1 ? s : sqrt(s);
}

static int clamp_threads(int32_t nthreads)
{
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    return nthreads;
#else
    (void)nthreads;
    return 1;
#endif
}

/* Threads the last parallel call used (reported as "cores" by the bench). */
static int g_threads_used = 1;
int32_t kgco_threads_used(void) { return g_threads_used; }

/*
 * Distances of selected query rows to every tail.
 *   rows[i] = h * R + r  (or NULL: all N*R rows in h-major order)
 *   out     = nrows x N doubles, row-major.
 */
int32_t kgco_dist_rows(const float *E, const float *Rel, int64_t N, int64_t R, int32_t d,
                       int32_t p, const int64_t *rows, int64_t nrows, double *out,
                       int32_t nthreads)
{
    if (p != 1 && p != 2) return -1;
    int nt = clamp_threads(nthreads);
    g_threads_used = nt;
    if (rows == NULL) nrows = N * R;
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t i = 0; i < nrows; ++i) {
        int64_t row = rows ? rows[i] : i;
        int64_t h = row / R, r = row % R;
        for (int64_t t = 0; t < N; ++t)
            out[i * N + t] = kgco_dist3(E + h * d, Rel + r * d, E + t * d, d, p);
    }
    return 0;
}

/*
 * The join.  Returns the number of triplets (>= 0) and a malloc'ed array in
 * *out (free with kgco_free), ordered by (row order, t): with rows == NULL
 * that is (h, r, t) ascending.  Negative return = error.
 */
int64_t kgco_join(const float *E, const float *Rel, int64_t N, int64_t R, int32_t d, int32_t p,
                  double eps, const int64_t *rows, int64_t nrows, int32_t nthreads,
                  kgco_triplet **out)
{
    *out = NULL;
    if (p != 1 && p != 2) return -1;
    if (rows == NULL) nrows = N * R;
    int nt = clamp_threads(nthreads);
    g_threads_used = nt;

    kgco_triplet **buf = (kgco_triplet **)calloc((size_t)nt, sizeof(*buf));
    int64_t *cnt = (int64_t *)calloc((size_t)nt, sizeof(int64_t));
    int64_t *cap = (int64_t *)calloc((size_t)nt, sizeof(int64_t));
    if (!buf || !cnt || !cap) return -3;
    int failed = 0;

    /* schedule(static) hands each thread one contiguous block of rows, so
     * concatenating the per-thread buffers in thread order keeps row order. */
#pragma omp parallel num_threads(nt)
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
#pragma omp for schedule(static)
        for (int64_t i = 0; i < nrows; ++i) {
            int64_t row = rows ? rows[i] : i;
            int64_t h = row / R, r = row % R;
            for (int64_t t = 0; t < N; ++t) {               /* Fig. naive, "Line 5" */
                double dist = kgco_dist3(E + h * d, Rel + r * d, E + t * d, d, p);
                if (dist <= eps) {
                    if (cnt[tid] == cap[tid]) {
                        int64_t nc = cap[tid] ? 2 * cap[tid] : 1024;
                        kgco_triplet *nb = (kgco_triplet *)realloc(buf[tid], (size_t)nc * sizeof(kgco_triplet));
                        if (!nb) { failed = 1; continue; }
                        buf[tid] = nb;
                        cap[tid] = nc;
                    }
                    kgco_triplet *o = &buf[tid][cnt[tid]++];
                    o->h = (int32_t)h; o->r = (int32_t)r; o->t = (int32_t)t; o->pad = 0;
                    o->dist = dist;
                }
            }
        }
    }
    int64_t total = 0;
    for (int i = 0; i < nt; ++i) total += cnt[i];
    kgco_triplet *res = failed ? NULL : (kgco_triplet *)malloc((size_t)(total ? total : 1) * sizeof(kgco_triplet));
    if (res) {
        int64_t off = 0;
        for (int i = 0; i < nt; ++i) {
            if (cnt[i]) memcpy(res + off, buf[i], (size_t)cnt[i] * sizeof(kgco_triplet));
            off += cnt[i];
        }
    }
    for (int i = 0; i < nt; ++i) free(buf[i]);
    free(buf); free(cnt); free(cap);
    if (!res) return -3;
    *out = res;
    return total;
}

void kgco_free(void *p) { free(p); }
