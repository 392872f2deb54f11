// sdnn_host.c -- host-side narrowing of the reference's Y0 columns for the
// upload (engine.infer's end-to-end path, sdnn.cu upload_csr).
//
// The reference's FeatureBatch carries int64 columns and float64 values
// (model.py:165-177).  The upload sends uint16 columns (N <= 65536) and no
// values when every value is 1.0.  This pass reads 16 bytes per entry and
// writes 2, so it is bound by host memory bandwidth: the staging writes use
// non-temporal stores (no read-for-ownership of the pinned buffer, and the
// DMA reads it right after), the validation (column range) and the binary
// check ride along in the same registers.
#include <immintrin.h>
#include <omp.h>
#include <stdint.h>

// d16 must be 32-byte aligned.  *bad |= some column outside [0, ncols);
// *bin &= every value == 1.0.  Uses the calling thread's OpenMP team.
void sdnn_host_narrow16(const int64_t* cc, const double* vv, uint16_t* d16, int64_t m, int64_t ncols, int* bad,
                        int* bin) {
    int bad_all = 0, bin_all = 1;
#pragma omp parallel reduction(| : bad_all) reduction(& : bin_all)
    {
        const int nt = omp_get_num_threads(), id = omp_get_thread_num();
        const int64_t blocks = m / 16;  // 16 entries = one 32-byte store
        const int64_t b0 = blocks * id / nt, b1 = blocks * (id + 1) / nt;
        const __m256i nm1 = _mm256_set1_epi64x(ncols - 1), zero = _mm256_setzero_si256();
        const __m256i lo32 = _mm256_setr_epi32(0, 2, 4, 6, 0, 2, 4, 6);
        const __m256d one = _mm256_set1_pd(1.0);
        __m256i badv = zero;
        __m256d nbin = _mm256_setzero_pd();
        for (int64_t b = b0; b < b1; ++b) {
            const int64_t p = b * 16;
            __m256i c[4];
            for (int i = 0; i < 4; ++i) {
                c[i] = _mm256_loadu_si256((const __m256i*)(cc + p + 4 * i));
                badv = _mm256_or_si256(badv, _mm256_or_si256(_mm256_cmpgt_epi64(c[i], nm1),
                                                             _mm256_cmpgt_epi64(zero, c[i])));
                nbin = _mm256_or_pd(nbin, _mm256_cmp_pd(_mm256_loadu_pd(vv + p + 4 * i), one, _CMP_NEQ_UQ));
            }
            // low 32 bits of each int64 -> 8 int32 per pair of vectors
            const __m128i a0 = _mm256_castsi256_si128(_mm256_permutevar8x32_epi32(c[0], lo32));
            const __m128i a1 = _mm256_castsi256_si128(_mm256_permutevar8x32_epi32(c[1], lo32));
            const __m128i a2 = _mm256_castsi256_si128(_mm256_permutevar8x32_epi32(c[2], lo32));
            const __m128i a3 = _mm256_castsi256_si128(_mm256_permutevar8x32_epi32(c[3], lo32));
            const __m256i A = _mm256_set_m128i(a1, a0), B = _mm256_set_m128i(a3, a2);
            // 32 -> 16 (in-range columns fit; out-of-range ones are flagged),
            // then undo packus' per-128-bit-lane interleave
            const __m256i r = _mm256_permute4x64_epi64(_mm256_packus_epi32(A, B), 0xD8);
            _mm256_stream_si256((__m256i*)(d16 + p), r);
        }
        // the tail (fewer than 16 entries) on the last thread
        if (id == nt - 1)
            for (int64_t p = blocks * 16; p < m; ++p) {
                bad_all |= (uint64_t)cc[p] >= (uint64_t)ncols;
                bin_all &= vv[p] == 1.0;
                d16[p] = (uint16_t)cc[p];
            }
        _mm_sfence();  // streaming stores visible before the copy engine reads the buffer
        bad_all |= !_mm256_testz_si256(badv, badv);
        bin_all &= _mm256_movemask_pd(nbin) == 0;
    }
    *bad |= bad_all;
    *bin &= bin_all;
}
