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
// B200 formulation
// ----------------
// Weights: ELL by output column, inputs ascending, padded to a multiple of
// 32 slots with index -1.  Every output is ONE sequential chain
//     acc = ((0 + y[k0]*w0) + y[k1]*w1) + ...      (k0 < k1 < ...)
// computed by one lane, so float64 reproduces the reference bit for bit
// (adding y*w for an unstored y = 0 adds a signed zero, which cannot change
// a nonzero chain nor make a zero chain nonzero).
//
// Activations: "tiles" of 32 live rows stored neuron-major, one line of
// 32 values per (tile, neuron): slab[(tile * ld + k) * 32 + lane].  A warp
// owns an output column j of a tile, lane = row: for each slot it gathers one
// whole line (128 B in float32) for its 32 rows, so each weight slot loaded
// serves 32 rows and each gather is a full coalesced line.  A byte mask per
// (tile, neuron) flags which 32-byte sectors of the line hold a nonzero;
// zero sectors are neither stored nor loaded (exact: they contribute +-0).
//
// One cooperative persistent kernel walks all layers: densify Y0 (CSR) into
// tiles, then per layer a work list of (live tile, output block) items, a
// grid barrier between layers, and a per-layer live-tile count so layers
// after the last live row cost a loop iteration.
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
// unstored entry and receives no bias (entry-masked bias).
template <typename T>
__device__ __forceinline__ T bias_relu_clamp(T acc, T bias, T ymax) {
    if (acc != T(0)) {
        T v = Arith<T>::add(acc, bias);
        if (v > T(0)) return v > ymax ? ymax : v;
    }
    return T(0);
}

// engine.py:129-133 on one STORED entry (CSR path: stored means present).
template <typename T>
__device__ __forceinline__ T bias_relu_clamp_stored(T z, T bias, T ymax) {
    T v = Arith<T>::add(z, bias);
    if (v > T(0)) return v > ymax ? ymax : v;
    return T(0);
}

template <typename T>
struct LayerDesc {
    const int32_t* idx;  // [n_out][wp] input index ascending, -1 = padding
    const T* val;        // [n_out][wp]
    int wp;              // slots per output, multiple of 32
    T bias;
};

template <typename T>
struct NetArgs {
    int n_in, n_out;      // input lines per tile, outputs per layer
    int ld;               // per-tile line stride of slabs (>= n_in, n_out)
    int mstride;          // per-tile byte stride of masks (ld rounded to 16)
    int L;
    const LayerDesc<T>* layers;
    T ymax;
    int epilogue;         // 1: bias/ReLU/clamp; 0: raw Z (engine.spmm)
    int n_tiles;
    const int32_t* rowid; // [n_tiles * 32] batch row of each lane, -1 empty
    const int64_t* csr_off;
    const int32_t* csr_cols;
    const T* csr_vals;
    T* slab[2];           // [n_tiles][ld][32]
    uint8_t* mask[2];     // [n_tiles][mstride]
    uint32_t* alive;      // [L + 1][n_tiles] lane bits of rows with an entry
    int32_t* tile_count;  // [L + 1] tiles with any live row
    unsigned* bar;        // grid barrier {count, generation}
    unsigned long long* stamps;  // [L + 1] globaltimer after each layer, or null
    int jb;               // outputs per work item
};

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Sense-reversing grid barrier for a cooperative launch (all CTAs resident).
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned n_blocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == n_blocks - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ float ld_cg(const float* p) { return __ldcg(p); }
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// Rows per 32-byte sector: 8 in float32, 4 in float64.
template <typename T>
__host__ __device__ constexpr int sector_rows() { return 32 / (int)sizeof(T); }

// ------------------------------------------------------------ phase 0
// Build tile t of Y0 from CSR: sector masks, zeroed nonzero lines, values.
template <typename T>
__device__ void densify_tile(const NetArgs<T>& a, int t, uint32_t* smask_w, uint32_t* s_has) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nw32 = (a.n_in + 3) >> 2;
    for (int i = tid; i < nw32; i += kThreads) smask_w[i] = 0u;
    if (tid == 0) *s_has = 0u;
    __syncthreads();
    for (int r = warp; r < 32; r += kWarps) {
        const int row = a.rowid[t * 32 + r];
        if (row < 0) continue;
        const uint32_t bit = 1u << (r / sector_rows<T>());
        const int64_t p0 = a.csr_off[row], p1 = a.csr_off[row + 1];
        for (int64_t p = p0 + lane; p < p1; p += 32) {
            const int k = a.csr_cols[p];
            atomicOr(&smask_w[k >> 2], bit << ((k & 3) * 8));
        }
    }
    __syncthreads();
    const uint8_t* smask = reinterpret_cast<const uint8_t*>(smask_w);
    uint8_t* gmask = a.mask[0] + (size_t)t * a.mstride;
    for (int k = tid; k < a.n_in; k += kThreads) gmask[k] = smask[k];
    // zero every line that will be read (any sector set)
    T* slab = a.slab[0] + (size_t)t * a.ld * 32;
    for (int k = warp; k < a.n_in; k += kWarps)
        if (smask[k]) slab[(size_t)k * 32 + lane] = T(0);
    __syncthreads();
    uint32_t has = 0;
    for (int r = warp; r < 32; r += kWarps) {
        const int row = a.rowid[t * 32 + r];
        if (row < 0) continue;
        const int64_t p0 = a.csr_off[row], p1 = a.csr_off[row + 1];
        if (p1 > p0) has |= 1u << r;
        for (int64_t p = p0 + lane; p < p1; p += 32) {
            const int k = a.csr_cols[p];
            slab[(size_t)k * 32 + r] = a.csr_vals[p];
        }
    }
    if (lane == 0 && has) atomicOr(s_has, has);
    __syncthreads();
    if (tid == 0) {
        a.alive[t] = *s_has;
        if (*s_has) atomicAdd(&a.tile_count[0], 1);
    }
    __syncthreads();
}

// ------------------------------------------------------------ one item
// Output columns [j0, j1) of tile t for layer l: warp per column, lane per row.
template <typename T>
__device__ __forceinline__ void layer_item(const NetArgs<T>& a, const LayerDesc<T>& L, int l, int t,
                                           int j0, int j1, const uint8_t* smask, uint32_t& alive_acc) {
    using A = Arith<T>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sec = lane / sector_rows<T>();
    const T* in = a.slab[l & 1] + (size_t)t * a.ld * 32;
    T* out = a.slab[(l + 1) & 1] + (size_t)t * a.ld * 32;
    uint8_t* omask = a.mask[(l + 1) & 1] + (size_t)t * a.mstride;
    for (int j = j0 + warp; j < j1; j += kWarps) {
        const int32_t* ip = L.idx + (size_t)j * L.wp;
        const T* vp = L.val + (size_t)j * L.wp;
        T acc = T(0);
        for (int s0 = 0; s0 < L.wp; s0 += 32) {
            const int my_k = __ldg(ip + s0 + lane);
            const T my_w = __ldg(vp + s0 + lane);
            T y[32];
#pragma unroll
            for (int s = 0; s < 32; ++s) {
                const int k = __shfl_sync(0xffffffffu, my_k, s);
                bool live = k >= 0;
                if (live) live = (smask[k] >> sec) & 1u;
                y[s] = live ? ld_cg(in + (size_t)k * 32 + lane) : T(0);
            }
#pragma unroll
            for (int s = 0; s < 32; ++s) {
                const int k = __shfl_sync(0xffffffffu, my_k, s);
                const T w = __shfl_sync(0xffffffffu, my_w, s);
                if (k >= 0) acc = A::add(acc, A::mul(y[s], w));
            }
        }
        const T v = a.epilogue ? bias_relu_clamp(acc, L.bias, a.ymax) : acc;
        const unsigned nz = __ballot_sync(0xffffffffu, v != T(0));
        unsigned m = 0;
#pragma unroll
        for (int s = 0; s < 32 / sector_rows<T>(); ++s) {
            const unsigned rows = ((1u << sector_rows<T>()) - 1u) << (s * sector_rows<T>());
            if (nz & rows) m |= 1u << s;
        }
        if ((m >> sec) & 1u) out[(size_t)j * 32 + lane] = v;
        if (lane == 0) omask[j] = (uint8_t)m;
        alive_acc |= nz;
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) net_kernel(NetArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    // [0, mstride): sector mask of the current tile; then the live-tile list
    uint8_t* smask = smem;
    int32_t* tiles = reinterpret_cast<int32_t*>(smem + a.mstride);
    __shared__ int s_count;
    __shared__ int s_scan[kWarps + 1];
    __shared__ uint32_t s_alive;
    const int tid = threadIdx.x;
    const unsigned nb = gridDim.x;

    for (int t = blockIdx.x; t < a.n_tiles; t += gridDim.x)
        densify_tile<T>(a, t, reinterpret_cast<uint32_t*>(smask), &s_alive);
    grid_barrier(a.bar, nb);
    if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[0] = globaltimer();

    bool all_dead = false;
    for (int l = 0; l < a.L; ++l) {
        // zero rows stay zero: once no tile is live every later layer is empty
        if (!all_dead && __ldcg(&a.tile_count[l]) == 0) all_dead = true;
        if (all_dead) continue;
        const uint32_t* alive_in = a.alive + (size_t)l * a.n_tiles;
        uint32_t* alive_out = a.alive + (size_t)(l + 1) * a.n_tiles;
        // ascending live-tile list (block-wide ordered compaction)
        if (tid == 0) s_count = 0;
        __syncthreads();
        for (int base = 0; base < a.n_tiles; base += kThreads) {
            const int t = base + tid;
            const bool live = t < a.n_tiles && __ldcg(&alive_in[t]) != 0u;
            const unsigned b = __ballot_sync(0xffffffffu, live);
            if ((tid & 31) == 0) s_scan[tid >> 5] = __popc(b);
            __syncthreads();
            if (tid == 0) {
                int acc = s_count;
                for (int w = 0; w < kWarps; ++w) {
                    const int c = s_scan[w];
                    s_scan[w] = acc;
                    acc += c;
                }
                s_scan[kWarps] = acc;
            }
            __syncthreads();
            if (live) tiles[s_scan[tid >> 5] + __popc(b & ((1u << (tid & 31)) - 1u))] = t;
            __syncthreads();
            if (tid == 0) s_count = s_scan[kWarps];
            __syncthreads();
        }
        const int count = s_count;
        const LayerDesc<T> L = a.layers[l];
        const int nblk = (a.n_out + a.jb - 1) / a.jb;
        const long long items = (long long)count * nblk;
        int cur = -1;
        if (tid == 0) s_alive = 0u;
        for (long long it = blockIdx.x; it < items; it += gridDim.x) {
            const int t = tiles[it / nblk];
            const int b = (int)(it % nblk);
            if (t != cur) {
                __syncthreads();
                const int4* src = reinterpret_cast<const int4*>(a.mask[l & 1] + (size_t)t * a.mstride);
                int4* dst = reinterpret_cast<int4*>(smask);
                for (int i = tid; i < a.mstride / 16; i += kThreads) dst[i] = __ldcg(src + i);
                __syncthreads();
                cur = t;
            }
            uint32_t alive_acc = 0;
            const int j0 = b * a.jb, j1 = min(a.n_out, j0 + a.jb);
            layer_item<T>(a, L, l, t, j0, j1, smask, alive_acc);
            if ((tid & 31) == 0 && alive_acc) atomicOr(&s_alive, alive_acc);
            __syncthreads();
            if (tid == 0 && s_alive) {
                const uint32_t old = atomicOr(&alive_out[t], s_alive);
                if (old == 0u) atomicAdd(&a.tile_count[l + 1], 1);
                s_alive = 0u;
            }
            __syncthreads();
        }
        grid_barrier(a.bar, nb);
        if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[l + 1] = globaltimer();
    }
}

// Read back the rows of each tile of the final slab, one warp per tile, lane
// per row: pass 1 (pos == null) counts entries, pass 2 writes (column,
// value) in ascending column order at pos[tile * 32 + lane].
template <typename T>
__global__ void extract_kernel(const T* __restrict__ slab, const uint8_t* __restrict__ mask, int ld,
                               int mstride, int n_cols, int n_tiles, const int64_t* __restrict__ pos,
                               int32_t* __restrict__ counts, int32_t* __restrict__ cols_out,
                               T* __restrict__ vals_out) {
    const int lane = threadIdx.x & 31;
    const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int n_warps = (gridDim.x * blockDim.x) >> 5;
    const int sec = lane / sector_rows<T>();
    for (int t = warp_global; t < n_tiles; t += n_warps) {
        const T* s = slab + (size_t)t * ld * 32;
        const uint8_t* m = mask + (size_t)t * mstride;
        int64_t at = pos ? pos[t * 32 + lane] : 0;
        int c = 0;
        for (int k = 0; k < n_cols; ++k) {
            if (!((m[k] >> sec) & 1u)) continue;
            const T v = s[(size_t)k * 32 + lane];
            if (v != T(0)) {
                if (pos) {
                    cols_out[at] = k;
                    vals_out[at] = v;
                    ++at;
                }
                ++c;
            }
        }
        if (!pos) counts[t * 32 + lane] = c;
    }
}

// ---------------------------------------------------- CSR bias/ReLU/clamp
// engine.apply_bias_relu_clamp on CSR values: count, then ordered write.
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
