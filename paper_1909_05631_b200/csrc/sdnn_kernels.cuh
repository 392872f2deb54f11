// sdnn_kernels.cuh -- sm_100a kernels of the Sparse DNN inference loop.
//
// Reference semantics (sdnnbench/engine.py):
//   _spmm_kernel (engine.py:64-116): z[j] = sum over the row's stored k, in
//     ascending k, of y[k] * W[k][j]; separately rounded multiply and add;
//     exact zeros are not stored.
//   _bias_relu_clamp_kernel (engine.py:119-137): v = z + bias on stored
//     entries only; keep v > 0; v > ymax -> ymax.
//   categorize (challenge.py:60-67): rows that still hold an entry.
//
// B200 formulation: activations are dense rows (a stored entry is exactly a
// nonzero), weights are ELL by output column with each column's inputs in
// ascending order, so every output is ONE sequential chain
//     acc = ((0 + y[k0]*w0) + y[k1]*w1) + ...      (k0 < k1 < ...)
// owned by one thread.  Adding y*w for an unstored y (= 0) adds a signed
// zero, which leaves any nonzero chain unchanged and cannot turn a zero
// chain nonzero, so the dense gather reproduces the Gustavson result bit
// for bit in float64 (and the same algorithm in float32).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sdnn {

template <typename T> struct Arith;
template <> struct Arith<float> {
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};
template <> struct Arith<double> {
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};

// engine.py:129-133 applied to one dense position; a zero position is an
// unstored entry and receives no bias (SPEC entry-masked bias).
template <typename T>
__device__ __forceinline__ T bias_relu_clamp(T acc, T bias, T ymax) {
    if (acc != T(0)) {
        T v = Arith<T>::add(acc, bias);
        if (v > T(0)) return v > ymax ? ymax : v;
    }
    return T(0);
}

// engine.py:129-133 on one STORED entry (CSR path: stored means present,
// whatever its value).
template <typename T>
__device__ __forceinline__ T bias_relu_clamp_stored(T z, T bias, T ymax) {
    T v = Arith<T>::add(z, bias);
    if (v > T(0)) return v > ymax ? ymax : v;
    return T(0);
}

template <typename T>
struct LayerArgs {
    int n_in, n_out;
    int width;                        // ELL slots per output (padded)
    int ld;                           // leading dimension of idx/val/bnd (>= n_out)
    const int32_t* __restrict__ idx;  // [width][ld] input index, ascending per output
    const T* __restrict__ val;        // [width][ld]
    const uint16_t* __restrict__ bnd; // [(n_chunks+1)][ld] first slot of each input chunk
                                      // (last row = degree); null: all width slots real
    int n_chunks, chunk_len;          // input neurons staged per pass
    T bias, ymax;
    int epilogue;                     // 1: bias/ReLU/clamp + live-row list; 0: raw Z
    // input: dense rows (y_in, indexed row - row_base) or CSR (csr_off != nullptr)
    const T* __restrict__ y_in;
    const int64_t* __restrict__ csr_off;
    const int32_t* __restrict__ csr_cols;
    const T* __restrict__ csr_vals;
    T* __restrict__ y_out;            // dense rows, indexed row - row_base
    int64_t row_base;
    const int32_t* __restrict__ rows_in;   // live rows entering this layer
    const int32_t* __restrict__ count_in;
    int32_t* __restrict__ rows_out;        // live rows leaving it
    int32_t* __restrict__ count_out;
};

// Stage chunk [k0, k0+klen) of the group's rows into shared memory.
template <typename T, int R>
__device__ __forceinline__ void stage_rows(const LayerArgs<T>& a, T* ys, const int (&rows)[R],
                                           int k0, int klen) {
    const int tid = threadIdx.x, nt = blockDim.x;
    if (a.csr_off) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (rows[r] < 0) continue;
            T* dst = ys + r * a.chunk_len;
            for (int k = tid; k < klen; k += nt) dst[k] = T(0);
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (rows[r] < 0) continue;
            T* dst = ys + r * a.chunk_len;
            const int64_t p0 = a.csr_off[rows[r]], p1 = a.csr_off[rows[r] + 1];
            for (int64_t p = p0 + tid; p < p1; p += nt) {
                const int k = a.csr_cols[p] - k0;
                if (k >= 0 && k < klen) dst[k] = a.csr_vals[p];
            }
        }
        return;
    }
    const bool vec = ((a.n_in * sizeof(T)) % 16 == 0) && ((k0 * sizeof(T)) % 16 == 0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (rows[r] < 0) continue;
        T* dst = ys + r * a.chunk_len;
        const T* src = a.y_in + (rows[r] - a.row_base) * (int64_t)a.n_in + k0;
        if (vec) {
            constexpr int V = 16 / sizeof(T);
            const int nv = klen / V;
            const int4* s4 = reinterpret_cast<const int4*>(src);
            int4* d4 = reinterpret_cast<int4*>(dst);
            for (int v = tid; v < nv; v += nt) d4[v] = __ldg(s4 + v);
            for (int k = nv * V + tid; k < klen; k += nt) dst[k] = src[k];
        } else {
            for (int k = tid; k < klen; k += nt) dst[k] = src[k];
        }
    }
}

// One layer for the rows of a live-row list.  Persistent grid: CTA b takes
// groups b, b + grid, ... of R rows; each group's rows sit in shared memory
// (one input chunk at a time) and every thread owns output columns
// j = tid, tid + blockDim, ... for all R rows, reusing each weight slot it
// loads across the R rows.  With more than one chunk the partial sums are
// parked in y_out between chunks: chunk c continues exactly the chain chunk
// c-1 left, so the accumulation order is unchanged.
template <typename T, int R>
__global__ void __launch_bounds__(256) layer_kernel(LayerArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* ys = reinterpret_cast<T*>(smem_raw);
    __shared__ int s_rows[R];
    __shared__ int s_alive[R];
    using A = Arith<T>;
    const int count = *a.count_in;
    const int n_groups = (count + R - 1) / R;
    const int tid = threadIdx.x, nt = blockDim.x;

    for (int g = blockIdx.x; g < n_groups; g += gridDim.x) {
        if (tid < R) {
            const int i = g * R + tid;
            s_rows[tid] = i < count ? a.rows_in[i] : -1;
            s_alive[tid] = 0;
        }
        __syncthreads();
        int rows[R];
#pragma unroll
        for (int r = 0; r < R; ++r) rows[r] = s_rows[r];
        unsigned alive = 0;

        for (int c = 0; c < a.n_chunks; ++c) {
            const int k0 = c * a.chunk_len;
            const int klen = min(a.chunk_len, a.n_in - k0);
            stage_rows<T, R>(a, ys, rows, k0, klen);
            __syncthreads();
            const bool last = (c == a.n_chunks - 1);
            for (int j = tid; j < a.n_out; j += nt) {
                T acc[R];
#pragma unroll
                for (int r = 0; r < R; ++r)
                    acc[r] = (c == 0 || rows[r] < 0)
                                 ? T(0)
                                 : a.y_out[(rows[r] - a.row_base) * (int64_t)a.n_out + j];
                int s0 = 0, s1 = a.width;
                if (a.bnd) {
                    s0 = a.bnd[(size_t)c * a.ld + j];
                    s1 = a.bnd[(size_t)(c + 1) * a.ld + j];
                }
                const int32_t* ip = a.idx + j;
                const T* vp = a.val + j;
                for (int s = s0; s < s1; ++s) {
                    const int k = __ldg(ip + (size_t)s * a.ld) - k0;
                    const T w = __ldg(vp + (size_t)s * a.ld);
#pragma unroll
                    for (int r = 0; r < R; ++r) acc[r] = A::add(acc[r], A::mul(ys[r * a.chunk_len + k], w));
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (rows[r] < 0) continue;
                    T v = acc[r];
                    if (last && a.epilogue) {
                        v = bias_relu_clamp(v, a.bias, a.ymax);
                        alive |= (v != T(0)) ? (1u << r) : 0u;
                    }
                    a.y_out[(rows[r] - a.row_base) * (int64_t)a.n_out + j] = v;
                }
            }
            __syncthreads();
        }
        if (a.epilogue) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (__any_sync(0xffffffffu, (alive >> r) & 1u) && (tid & 31) == 0) s_alive[r] = 1;
            }
            __syncthreads();
            if (tid == 0) {
                int n = 0;
#pragma unroll
                for (int r = 0; r < R; ++r) n += (rows[r] >= 0 && s_alive[r]) ? 1 : 0;
                if (n) {
                    int pos = atomicAdd(a.count_out, n);
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        if (rows[r] >= 0 && s_alive[r]) a.rows_out[pos++] = rows[r];
                }
            }
        }
        __syncthreads();
    }
}

// Live rows of the input batch: rows [r0, r1) with at least one stored entry
// (an empty row stays empty through every layer, test_engine.py:138-146).
// With all_rows set every row is listed (used by the per-step spmm entry).
__global__ void init_rows_kernel(const int64_t* __restrict__ off, int64_t r0, int64_t r1,
                                 int all_rows, int32_t* __restrict__ rows, int32_t* __restrict__ count);

// ---------------------------------------------------------------- compaction
// Ordered dense-row -> CSR compaction for the rows of a list: pass 1 counts
// nonzeros per listed row, pass 2 writes (column, value) in ascending column
// order at the offsets the host scanned from pass 1.

template <typename T>
__global__ void dense_count_kernel(const T* __restrict__ y, int64_t row_base, int n_cols,
                                   const int32_t* __restrict__ rows, int n_rows,
                                   int32_t* __restrict__ counts) {
    __shared__ int s_sum[32];
    for (int i = blockIdx.x; i < n_rows; i += gridDim.x) {
        const T* src = y + (rows[i] - row_base) * (int64_t)n_cols;
        int c = 0;
        for (int k = threadIdx.x; k < n_cols; k += blockDim.x) c += (src[k] != T(0));
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x < 32) {
            int v = threadIdx.x < (blockDim.x >> 5) ? s_sum[threadIdx.x] : 0;
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (threadIdx.x == 0) counts[i] = v;
        }
        __syncthreads();
    }
}

// Block-wide exclusive prefix of a 0/1 flag in thread order; returns the
// position and sets *total.  blockDim.x must be a multiple of 32 (<= 1024).
__device__ __forceinline__ int block_prefix(bool flag, int* s_warp, int* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const unsigned b = __ballot_sync(0xffffffffu, flag);
    const int in_warp = __popc(b & ((1u << lane) - 1u));
    if (lane == 0) s_warp[w] = __popc(b);
    __syncthreads();
    if (w == 0) {
        int v = lane < nw ? s_warp[lane] : 0;
        int incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane < nw) s_warp[lane] = incl - v;
        if (lane == 31) s_warp[32] = incl;
    }
    __syncthreads();
    const int pos = s_warp[w] + in_warp;
    *total = s_warp[32];
    __syncthreads();
    return pos;
}

template <typename T>
__global__ void dense_write_kernel(const T* __restrict__ y, int64_t row_base, int n_cols,
                                   const int32_t* __restrict__ rows, int n_rows,
                                   const int64_t* __restrict__ pos,
                                   int32_t* __restrict__ cols_out, T* __restrict__ vals_out) {
    __shared__ int s_warp[33];
    for (int i = blockIdx.x; i < n_rows; i += gridDim.x) {
        const T* src = y + (rows[i] - row_base) * (int64_t)n_cols;
        int64_t base = pos[i];
        for (int k0 = 0; k0 < n_cols; k0 += blockDim.x) {
            const int k = k0 + threadIdx.x;
            const T v = k < n_cols ? src[k] : T(0);
            int total;
            const int p = block_prefix(v != T(0), s_warp, &total);
            if (v != T(0)) {
                cols_out[base + p] = k;
                vals_out[base + p] = v;
            }
            base += total;
        }
    }
}

// engine.apply_bias_relu_clamp on CSR values: count then ordered write.
template <typename T>
__global__ void csr_brc_count_kernel(const int64_t* __restrict__ off, const T* __restrict__ vals,
                                     int64_t n_rows, T bias, T ymax, int32_t* __restrict__ counts) {
    __shared__ int s_sum[32];
    for (int64_t i = blockIdx.x; i < n_rows; i += gridDim.x) {
        int c = 0;
        for (int64_t p = off[i] + threadIdx.x; p < off[i + 1]; p += blockDim.x)
            c += (bias_relu_clamp_stored(vals[p], bias, ymax) != T(0));
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x < 32) {
            int v = threadIdx.x < (blockDim.x >> 5) ? s_sum[threadIdx.x] : 0;
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (threadIdx.x == 0) counts[i] = v;
        }
        __syncthreads();
    }
}

template <typename T>
__global__ void csr_brc_write_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ cols,
                                     const T* __restrict__ vals, int64_t n_rows, T bias, T ymax,
                                     const int64_t* __restrict__ pos, int32_t* __restrict__ cols_out,
                                     T* __restrict__ vals_out) {
    __shared__ int s_warp[33];
    for (int64_t i = blockIdx.x; i < n_rows; i += gridDim.x) {
        int64_t base = pos[i];
        for (int64_t p0 = off[i]; p0 < off[i + 1]; p0 += blockDim.x) {
            const int64_t p = p0 + threadIdx.x;
            const T v = p < off[i + 1] ? bias_relu_clamp_stored(vals[p], bias, ymax) : T(0);
            int total;
            const int q = block_prefix(v != T(0), s_warp, &total);
            if (v != T(0)) {
                cols_out[base + q] = cols[p];
                vals_out[base + q] = v;
            }
            base += total;
        }
    }
}

}  // namespace sdnn
