/*
 * sdnn_gen.c -- seeded synthetic workloads for the BASELINE.json configs.
 *
 * Not on the timed path.  Builds (1) layer weights as the union of `width`
 * random permutation matrices with exactly `width` nonzeros per row and per
 * column, and (2) binary input images with Bernoulli pixels inside a
 * centred square, both from counter-based streams so any layer or row can
 * be produced independently, on any host, with identical bytes (the same
 * property radixnet.py:202-206 gives its permutations).
 *
 * The perm-union construction follows BASELINE.json configs[0..4]: permutation
 * p assigns output column j the input row Q_p(j); a collision (Q_p(j) equal to
 * some Q_q(j), q < p) is resampled by swapping Q_p(j) with Q_p(j') for a
 * seeded random j' that keeps both columns collision-free.
 *
 * Compiled twice: into libsdnn.so (the GPU path's fast uploader) and into the
 * host-only libsdnn_gen.so that the CPU tests and the CPU baseline arm load.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/sdnn_gen.h"

static inline uint64_t mix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

typedef struct { uint64_t s; } gen_rng;

static gen_rng rng_stream(uint64_t seed, uint64_t a, uint64_t b, uint64_t c)
{
    gen_rng r;
    r.s = mix64(seed ^ mix64(a ^ mix64(b ^ mix64(c ^ 0x5D4E4E2A5EEDull))));
    return r;
}

static inline uint64_t rng_next(gen_rng *r)
{
    r->s += 0x9E3779B97F4A7C15ull;
    uint64_t z = r->s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* uniform integer in [0, n) (multiply-high; deterministic everywhere) */
static inline uint32_t rng_below(gen_rng *r, uint32_t n)
{
    return (uint32_t)(((unsigned __int128)rng_next(r) * n) >> 64);
}

/* uniform double in [0, 1) with 53 random bits */
static inline double rng_unit(gen_rng *r)
{
    return (double)(rng_next(r) >> 11) * (1.0 / 9007199254740992.0);
}

#define STREAM_PERM 0x7065726DULL  /* "perm" */
#define STREAM_FIX 0x66697821ULL   /* "fix!" */
#define STREAM_IMG 0x696D6167ULL   /* "imag" */

static int col_has(const int32_t *q, int32_t upto, int32_t v)
{
    for (int32_t i = 0; i < upto; i++)
        if (q[i] == v) return 1;
    return 0;
}

int sdnn_gen_permunion_ell(uint64_t seed, int64_t layer, int32_t n, int32_t width,
                           int32_t *idx_out)
{
    if (n < 1 || width < 0 || width > n) return 2;
    if (width == 0) return 0;
    /* q[j * width + p] = input row feeding output column j through perm p */
    int32_t *q = (int32_t *)malloc((size_t)n * (size_t)width * sizeof(int32_t));
    int32_t *perm = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!q || !perm) { free(q); free(perm); return 3; }
    for (int32_t p = 0; p < width; p++) {
        gen_rng r = rng_stream(seed, STREAM_PERM, (uint64_t)layer, (uint64_t)p);
        for (int32_t j = 0; j < n; j++) perm[j] = j;
        for (int32_t j = n - 1; j > 0; j--) {  /* Fisher-Yates */
            uint32_t t = rng_below(&r, (uint32_t)j + 1);
            int32_t tmp = perm[j]; perm[j] = perm[t]; perm[t] = tmp;
        }
        for (int32_t j = 0; j < n; j++) q[(size_t)j * width + p] = perm[j];
        if (p == 0) continue;
        /* resample collisions of permutation p against permutations 0..p-1 */
        for (int32_t j = 0; j < n; j++) {
            int32_t *qj = q + (size_t)j * width;
            if (!col_has(qj, p, qj[p])) continue;
            gen_rng fr = rng_stream(seed, STREAM_FIX, (uint64_t)layer,
                                    ((uint64_t)p << 32) | (uint32_t)j);
            for (;;) {
                int32_t j2 = (int32_t)rng_below(&fr, (uint32_t)n);
                if (j2 == j) continue;
                int32_t *qk = q + (size_t)j2 * width;
                if (col_has(qj, p, qk[p]) || col_has(qk, p, qj[p])) continue;
                int32_t tmp = qj[p]; qj[p] = qk[p]; qk[p] = tmp;
                break;
            }
        }
    }
    /* ELL by output: each column's inputs in ascending order */
    for (int32_t j = 0; j < n; j++) {
        int32_t *src = q + (size_t)j * width;
        int32_t *dst = idx_out + (size_t)j * width;
        for (int32_t i = 0; i < width; i++) {
            int32_t v = src[i], k = i - 1;
            while (k >= 0 && dst[k] > v) { dst[k + 1] = dst[k]; k--; }
            dst[k + 1] = v;
        }
    }
    free(q);
    free(perm);
    return 0;
}

int sdnn_gen_ell_to_csr(int32_t n_in, int32_t n_out, int32_t width, const int32_t *idx,
                        const double *vals, int64_t *off, int64_t *cols, double *out_vals)
{
    /* transpose ELL-by-output into CSR-by-input; walking outputs in ascending
     * order leaves every input row's columns sorted */
    memset(off, 0, ((size_t)n_in + 1) * sizeof(int64_t));
    for (int64_t s = 0; s < (int64_t)n_out * width; s++) {
        if (idx[s] < 0 || idx[s] >= n_in) return 2;
        off[idx[s] + 1]++;
    }
    for (int32_t i = 0; i < n_in; i++) off[i + 1] += off[i];
    int64_t *fill = (int64_t *)malloc(((size_t)n_in + 1) * sizeof(int64_t));
    if (!fill) return 3;
    memcpy(fill, off, ((size_t)n_in + 1) * sizeof(int64_t));
    for (int32_t j = 0; j < n_out; j++) {
        for (int32_t s = 0; s < width; s++) {
            int64_t e = (int64_t)j * width + s;
            int64_t pos = fill[idx[e]]++;
            cols[pos] = j;
            out_vals[pos] = vals ? vals[e] : 0.0;
        }
    }
    free(fill);
    return 0;
}

/* ---------------------------------------------------------------- images */

typedef struct {
    uint64_t seed;
    int64_t row0;           /* stream index of local row 0 */
    int64_t r0, r1;
    int32_t side, square;
    double p;
    int64_t *row_nnz;       /* count pass */
    const int64_t *off;     /* fill pass */
    int64_t *cols64;
    int32_t *cols32;
    double *vals;
} img_job;

static void *img_work(void *arg)
{
    img_job *jb = (img_job *)arg;
    int32_t o = (jb->side - jb->square) / 2;
    for (int64_t r = jb->r0; r < jb->r1; r++) {
        gen_rng g = rng_stream(jb->seed, STREAM_IMG, 0, (uint64_t)(jb->row0 + r));
        int64_t cnt = 0;
        int64_t pos = jb->off ? jb->off[r] : 0;
        for (int32_t y = o; y < o + jb->square; y++) {
            for (int32_t x = o; x < o + jb->square; x++) {
                if (rng_unit(&g) < jb->p) {
                    if (jb->off) {
                        int64_t c = (int64_t)y * jb->side + x;
                        if (jb->cols64) jb->cols64[pos] = c;
                        if (jb->cols32) jb->cols32[pos] = (int32_t)c;
                        if (jb->vals) jb->vals[pos] = 1.0;
                        pos++;
                    }
                    cnt++;
                }
            }
        }
        if (jb->row_nnz) jb->row_nnz[r] = cnt;
    }
    return NULL;
}

static void run_img(img_job *proto, int64_t n_rows, int threads)
{
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    img_job jobs[256];
    int64_t per = (n_rows + threads - 1) / threads;
    int used = 0;
    for (int t = 0; t < threads; t++) {
        jobs[t] = *proto;
        jobs[t].r0 = (int64_t)t * per;
        jobs[t].r1 = jobs[t].r0 + per < n_rows ? jobs[t].r0 + per : n_rows;
        if (jobs[t].r0 >= jobs[t].r1) break;
        pthread_create(&tid[t], NULL, img_work, &jobs[t]);
        used++;
    }
    for (int t = 0; t < used; t++) pthread_join(tid[t], NULL);
}

int sdnn_gen_images_count(uint64_t seed, int64_t row0, int64_t n_rows, int32_t side,
                          int32_t square, double p, int threads, int64_t *row_nnz)
{
    if (square > side || square < 0 || side < 1 || n_rows < 0 || row0 < 0) return 2;
    img_job jb;
    memset(&jb, 0, sizeof(jb));
    jb.seed = seed; jb.row0 = row0; jb.side = side; jb.square = square; jb.p = p; jb.row_nnz = row_nnz;
    run_img(&jb, n_rows, threads);
    return 0;
}

int sdnn_gen_images_fill(uint64_t seed, int64_t row0, int64_t n_rows, int32_t side,
                         int32_t square, double p, int threads, const int64_t *off,
                         int64_t *cols64, int32_t *cols32, double *vals)
{
    if (square > side || square < 0 || side < 1 || n_rows < 0 || row0 < 0) return 2;
    img_job jb;
    memset(&jb, 0, sizeof(jb));
    jb.seed = seed; jb.row0 = row0; jb.side = side; jb.square = square; jb.p = p;
    jb.off = off; jb.cols64 = cols64; jb.cols32 = cols32; jb.vals = vals;
    run_img(&jb, n_rows, threads);
    return 0;
}

/* ------------------------------------------------------- parallel layers */

typedef struct {
    uint64_t seed;
    int64_t first, count;
    int32_t n, width;
    int32_t *idx;      /* [count][n][width] */
    int status;
    int64_t next;      /* shared cursor (guarded by mu) */
    pthread_mutex_t *mu;
} lay_job;

static void *lay_work(void *arg)
{
    lay_job *jb = (lay_job *)arg;
    for (;;) {
        pthread_mutex_lock(jb->mu);
        int64_t l = jb->next++;
        pthread_mutex_unlock(jb->mu);
        if (l >= jb->count) break;
        int rc = sdnn_gen_permunion_ell(jb->seed, jb->first + l, jb->n, jb->width,
                                        jb->idx + (size_t)l * jb->n * jb->width);
        if (rc) jb->status = rc;
    }
    return NULL;
}

int sdnn_gen_permunion_ell_layers(uint64_t seed, int64_t first_layer, int64_t count,
                                  int32_t n, int32_t width, int threads, int32_t *idx_out)
{
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_mutex_t mu;
    pthread_mutex_init(&mu, NULL);
    lay_job shared;
    memset(&shared, 0, sizeof(shared));
    shared.seed = seed; shared.first = first_layer; shared.count = count;
    shared.n = n; shared.width = width; shared.idx = idx_out; shared.mu = &mu;
    pthread_t tid[256];
    int used = threads < count ? threads : (int)count;
    for (int t = 0; t < used; t++) pthread_create(&tid[t], NULL, lay_work, &shared);
    for (int t = 0; t < used; t++) pthread_join(tid[t], NULL);
    pthread_mutex_destroy(&mu);
    return shared.status;
}
