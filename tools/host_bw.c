// Host memory bandwidth probe: pure AVX2 read of an int64+float64 CSR-sized
// buffer pair with T threads vs sdnn_host_narrow16 on the same data.
// gcc -O3 -mavx2 -fopenmp tools/host_bw.c paper_1909_05631_b200/csrc/sdnn_host.c -o /tmp/host_bw
#include <immintrin.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
void sdnn_host_narrow16(const int64_t*, const double*, uint16_t*, int64_t, int64_t, int*, int*);
int main(int argc, char** argv) {
    const int64_t m = argc > 1 ? atoll(argv[1]) : 537600000LL;  // C4 Y0 entries
    int64_t* c = aligned_alloc(64, m * 8);
    double* v = aligned_alloc(64, m * 8);
    uint16_t* d = aligned_alloc(64, m * 2 + 64);
#pragma omp parallel for
    for (int64_t i = 0; i < m; ++i) { c[i] = i & 65535; v[i] = 1.0; }
    for (int rep = 0; rep < 3; ++rep) {
        double t0 = omp_get_wtime();
        __m256i acc = _mm256_setzero_si256();
        int64_t s = 0;
#pragma omp parallel reduction(+ : s)
        {
            __m256i a = _mm256_setzero_si256();
#pragma omp for
            for (int64_t i = 0; i < m; i += 4) {
                a = _mm256_add_epi64(a, _mm256_load_si256((const __m256i*)(c + i)));
                a = _mm256_add_epi64(a, _mm256_castpd_si256(_mm256_load_pd(v + i)));
            }
            int64_t x[4];
            _mm256_storeu_si256((__m256i*)x, a);
            s += x[0] + x[1] + x[2] + x[3];
        }
        double t1 = omp_get_wtime();
        int bad = 0, bin = 1;
        sdnn_host_narrow16(c, v, d, m, 65536, &bad, &bin);
        double t2 = omp_get_wtime();
        printf("threads %d: read %.1f GB/s (%.1f ms), narrow %.1f GB/s (%.1f ms) [%lld %d %d]\n", omp_get_max_threads(),
               m * 16.0 / (t1 - t0) / 1e9, (t1 - t0) * 1e3, m * 16.0 / (t2 - t1) / 1e9, (t2 - t1) * 1e3,
               (long long)(s & 1), bad, bin);
        (void)acc;
    }
    return 0;
}
