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
// 32 slots with index -1.  Every (row, output) is ONE sequential chain
//     acc = ((0 + y[k0]*w0) + y[k1]*w1) + ...      (k0 < k1 < ...)
// kept in one register, so float64 reproduces the reference bit for bit
// (adding y*w for an unstored y = 0 adds a signed zero, which cannot change
// a nonzero chain nor make a zero chain nonzero -- so zero lines may be
// skipped or gathered as zeros without changing a bit).
//
// Activations: "tiles" of TR live rows (128 in float32, 64 in float64)
// stored neuron-major: one 512-byte line per (tile, neuron),
//     slab[(tile * ld + k) * TR + r],
// lane l of a warp owns rows l*RPL .. l*RPL+RPL-1 (RPL = 16 B / sizeof(T)).
// A warp computes one output column of a tile: per weight slot it gathers
// one whole line (every lane one 16-byte load), so one weight slot serves
// TR rows.  A byte per (tile, neuron) flags which 64-byte groups (4 lanes)
// of the line hold a nonzero; zero groups are not stored, and their gathers
// read the tile's dedicated zero line (line ld-1) instead; slots whose whole
// line is zero are dropped from the warp's slot list before any gather.
//
// A cooperative persistent kernel walks all layers with one grid barrier per
// live layer and a per-layer live-tile count, so layers after the last live
// row cost a loop iteration.  Y0 (CSR) is expanded into tiles by
// densify_kernel beforehand.
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

// Tile geometry.
constexpr int kLineBytes = 512;  // one (tile, neuron) line: 32 lanes x 16 B
template <typename T>
__host__ __device__ constexpr int rows_per_lane() { return 16 / (int)sizeof(T); }
template <typename T>
__host__ __device__ constexpr int tile_rows() { return 32 * rows_per_lane<T>(); }
// alive words per (layer, tile): one per lane component, plus an "any" flag
template <typename T>
__host__ __device__ constexpr int alive_words() { return rows_per_lane<T>() + 1; }

// 16-byte line piece of one lane <-> its RPL values
__device__ __forceinline__ void ld16(float (&d)[4], const char* p) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
}
__device__ __forceinline__ void ld16(double (&d)[2], const char* p) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    d[0] = v.x; d[1] = v.y;
}
__device__ __forceinline__ void st16(char* p, const float (&d)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(d[0], d[1], d[2], d[3]);
}
__device__ __forceinline__ void st16(char* p, const double (&d)[2]) {
    *reinterpret_cast<double2*>(p) = make_double2(d[0], d[1]);
}

// One live slot of a warp's compacted slot list.
template <typename T>
struct SlotEntry {
    unsigned off;  // line byte offset k * 512 | group mask of that line
    T w;           // weight
};

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
    int ld;               // lines per tile (>= n_in, n_out, plus the zero line)
    int L;
    const LayerDesc<T>* layers;
    T ymax;
    int epilogue;         // 1: bias/ReLU/clamp; 0: raw Z (engine.spmm)
    int n_tiles;
    T* slab[2];           // [n_tiles][ld][TR]
    uint8_t* mask[2];     // [n_tiles][ld] nonzero 64-byte groups of each line
    uint32_t* alive;      // [L + 1][n_tiles][alive_words] live-row bits
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
// The gpu-scope fences make every layer's stores visible to the next layer
// and invalidate this SM's L1, so plain (L1-cached) loads are coherent.
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

// ------------------------------------------------------------ densify
// Expand Y0 (CSR) into tiles: one block per tile.  Builds the group masks,
// zeroes every line that will be read, scatters the values, and records
// the tile's live rows (rows with an entry).
template <typename T>
__global__ void __launch_bounds__(512) densify_kernel(const int64_t* __restrict__ csr_off,
                                                      const int32_t* __restrict__ csr_cols,
                                                      const T* __restrict__ csr_vals,
                                                      const int32_t* __restrict__ rowid, int n_in, int ld,
                                                      int n_tiles, T* slab0, T* slab1, uint8_t* mask0,
                                                      uint32_t* alive0, int32_t* tile_count0) {
    extern __shared__ __align__(16) uint32_t smask_w[];
    __shared__ uint32_t s_alive[alive_words<T>()];
    constexpr int TR = tile_rows<T>(), RPL = rows_per_lane<T>();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        for (int i = tid; i < (n_in + 3) / 4; i += blockDim.x) smask_w[i] = 0u;
        if (tid < alive_words<T>()) s_alive[tid] = 0u;
        __syncthreads();
        for (int r = warp; r < TR; r += nwarp) {
            const int row = rowid[(size_t)t * TR + r];
            if (row < 0) continue;
            const uint32_t bit = 1u << (r / RPL / 4);
            for (int64_t p = csr_off[row] + lane; p < csr_off[row + 1]; p += 32) {
                const int k = csr_cols[p];
                atomicOr(&smask_w[k >> 2], bit << ((k & 3) * 8));
            }
        }
        __syncthreads();
        const uint8_t* smask = reinterpret_cast<const uint8_t*>(smask_w);
        uint8_t* gm = mask0 + (size_t)t * ld;
        for (int k = tid; k < n_in; k += blockDim.x) gm[k] = smask[k];
        char* s0 = reinterpret_cast<char*>(slab0 + (size_t)t * ld * TR);
        char* s1 = reinterpret_cast<char*>(slab1 + (size_t)t * ld * TR);
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int k = warp; k < n_in; k += nwarp)
            if (smask[k]) *reinterpret_cast<float4*>(s0 + (size_t)k * kLineBytes + lane * 16) = z;
        if (warp == 0) {  // the zero line of both buffers
            *reinterpret_cast<float4*>(s0 + (size_t)(ld - 1) * kLineBytes + lane * 16) = z;
            *reinterpret_cast<float4*>(s1 + (size_t)(ld - 1) * kLineBytes + lane * 16) = z;
        }
        __syncthreads();
        T* sl = slab0 + (size_t)t * ld * TR;
        for (int r = warp; r < TR; r += nwarp) {
            const int row = rowid[(size_t)t * TR + r];
            if (row < 0) continue;
            const int64_t p0 = csr_off[row], p1 = csr_off[row + 1];
            if (lane == 0 && p1 > p0) {
                atomicOr(&s_alive[r % RPL], 1u << (r / RPL));
                atomicOr(&s_alive[RPL], 1u);
            }
            for (int64_t p = p0 + lane; p < p1; p += 32) sl[(size_t)csr_cols[p] * TR + r] = csr_vals[p];
        }
        __syncthreads();
        if (tid < alive_words<T>()) alive0[(size_t)t * alive_words<T>() + tid] = s_alive[tid];
        if (tid == 0 && s_alive[RPL]) atomicAdd(tile_count0, 1);
        __syncthreads();
    }
}

// ------------------------------------------------------------ one item
// Output columns [j0, j1) of tile t for layer l: warp per column.
// Per 32-slot batch, lane s resolves slot s (input line offset, its group
// mask, weight); slots whose line is entirely zero are dropped and the rest
// are compacted, in slot order, into the warp's smem list; the list is then
// gathered 8 lines at a time.  Each lane chains its RPL rows separately.
template <typename T>
__device__ __forceinline__ void layer_item(const NetArgs<T>& a, const LayerDesc<T>& L, int l, int t,
                                           int j0, int j1, SlotEntry<T>* wlist, uint32_t (&alive_acc)[4]) {
    using A = Arith<T>;
    constexpr int RPL = rows_per_lane<T>();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned gbit = 1u << (lane >> 2);
    const size_t tile_lines = (size_t)t * a.ld;
    // select, not index: a runtime index into the parameter struct would
    // force a local-memory copy of it
    const bool odd = l & 1;
    const char* in = reinterpret_cast<const char*>(odd ? a.slab[1] : a.slab[0]) + tile_lines * kLineBytes + lane * 16;
    char* out = reinterpret_cast<char*>(odd ? a.slab[0] : a.slab[1]) + tile_lines * kLineBytes + lane * 16;
    const uint8_t* imask = (odd ? a.mask[1] : a.mask[0]) + tile_lines;
    uint8_t* omask = (odd ? a.mask[0] : a.mask[1]) + tile_lines;
    const unsigned zoff = (unsigned)(a.ld - 1) * kLineBytes;
    for (int j = j0 + warp; j < j1; j += kWarps) {
        T acc[RPL];
#pragma unroll
        for (int c = 0; c < RPL; ++c) acc[c] = T(0);
        for (int s0 = 0; s0 < L.wp; s0 += 32) {
            const int k = __ldg(L.idx + (size_t)j * L.wp + s0 + lane);
            const T w = __ldg(L.val + (size_t)j * L.wp + s0 + lane);
            const unsigned m = k >= 0 ? (unsigned)imask[k] : 0u;
            const unsigned live = __ballot_sync(0xffffffffu, m != 0u);
            if (m) {
                SlotEntry<T> e;
                e.off = (unsigned)k * kLineBytes | m;
                e.w = w;
                wlist[__popc(live & ((1u << lane) - 1u))] = e;
            }
            __syncwarp();
            const int n = __popc(live);
            for (int i0 = 0; i0 < n; i0 += 8) {
                T y[8][RPL];
                T wv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (i0 + u < n) {
                        const SlotEntry<T> e = wlist[i0 + u];
                        const unsigned off = (e.off & gbit) ? (e.off & ~(unsigned)(kLineBytes - 1)) : zoff;
                        ld16(y[u], in + off);
                        wv[u] = e.w;
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (i0 + u < n) {
#pragma unroll
                        for (int c = 0; c < RPL; ++c) acc[c] = A::add(acc[c], A::mul(y[u][c], wv[u]));
                    }
                }
            }
            __syncwarp();
        }
        T v[RPL];
        bool any = false;
#pragma unroll
        for (int c = 0; c < RPL; ++c) {
            v[c] = a.epilogue ? bias_relu_clamp(acc[c], L.bias, a.ymax) : acc[c];
            any |= v[c] != T(0);
            alive_acc[c] |= __ballot_sync(0xffffffffu, v[c] != T(0));
        }
        const unsigned lanes = __ballot_sync(0xffffffffu, any);
        unsigned om = 0;
#pragma unroll
        for (int g = 0; g < 8; ++g)
            if ((lanes >> (4 * g)) & 0xFu) om |= 1u << g;
        if (om & gbit) st16(out + (size_t)j * kLineBytes, v);
        if (lane == 0) omask[j] = (uint8_t)om;
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 2) net_kernel(NetArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    int32_t* tiles = reinterpret_cast<int32_t*>(smem);
    __shared__ SlotEntry<T> s_list[kWarps][32];
    __shared__ int s_count;
    __shared__ int s_scan[kWarps + 1];
    __shared__ uint32_t s_alive[4];
    constexpr int RPL = rows_per_lane<T>(), AW = alive_words<T>();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned nb = gridDim.x;
    if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[0] = globaltimer();

    bool all_dead = false;
    for (int l = 0; l < a.L; ++l) {
        // zero rows stay zero: once no tile is live every later layer is empty
        if (!all_dead && __ldcg(&a.tile_count[l]) == 0) all_dead = true;
        if (all_dead) continue;
        const uint32_t* alive_in = a.alive + (size_t)l * a.n_tiles * AW;
        uint32_t* alive_out = a.alive + (size_t)(l + 1) * a.n_tiles * AW;
        // ascending live-tile list (block-wide ordered compaction)
        if (tid == 0) s_count = 0;
        __syncthreads();
        for (int base = 0; base < a.n_tiles; base += kThreads) {
            const int t = base + tid;
            const bool live = t < a.n_tiles && __ldcg(&alive_in[(size_t)t * AW + RPL]) != 0u;
            const unsigned b = __ballot_sync(0xffffffffu, live);
            if (lane == 0) s_scan[warp] = __popc(b);
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
            if (live) tiles[s_scan[warp] + __popc(b & ((1u << lane) - 1u))] = t;
            __syncthreads();
            if (tid == 0) s_count = s_scan[kWarps];
            __syncthreads();
        }
        const int count = s_count;
        const LayerDesc<T> L = a.layers[l];
        const int nblk = (a.n_out + a.jb - 1) / a.jb;
        const long long items = (long long)count * nblk;
        if (tid < 4) s_alive[tid] = 0u;
        __syncthreads();
        for (long long it = blockIdx.x; it < items; it += gridDim.x) {
            const int t = tiles[it / nblk];
            const int b = (int)(it % nblk);
            uint32_t alive_acc[4] = {0u, 0u, 0u, 0u};
            const int j0 = b * a.jb, j1 = min(a.n_out, j0 + a.jb);
            layer_item<T>(a, L, l, t, j0, j1, s_list[warp], alive_acc);
            if (lane == 0) {
#pragma unroll
                for (int c = 0; c < RPL; ++c)
                    if (alive_acc[c]) atomicOr(&s_alive[c], alive_acc[c]);
            }
            __syncthreads();
            if (tid < RPL && s_alive[tid]) atomicOr(&alive_out[(size_t)t * AW + tid], s_alive[tid]);
            if (tid == RPL) {
                bool any = false;
                for (int c = 0; c < RPL; ++c) any |= s_alive[c] != 0u;
                if (any && atomicOr(&alive_out[(size_t)t * AW + RPL], 1u) == 0u) atomicAdd(&a.tile_count[l + 1], 1);
            }
            __syncthreads();
            if (tid < 4) s_alive[tid] = 0u;
            __syncthreads();
        }
        grid_barrier(a.bar, nb);
        if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[l + 1] = globaltimer();
    }
}

// Read back the rows of each tile of the final slab, one warp per tile,
// each lane its RPL rows: pass 1 (pos == null) counts entries, pass 2 writes
// (column, value) in ascending column order at pos[tile * TR + row].
template <typename T>
__global__ void extract_kernel(const T* __restrict__ slab, const uint8_t* __restrict__ mask, int ld,
                               int n_cols, int n_tiles, const int64_t* __restrict__ pos,
                               int32_t* __restrict__ counts, int32_t* __restrict__ cols_out,
                               T* __restrict__ vals_out) {
    constexpr int RPL = rows_per_lane<T>(), TR = tile_rows<T>();
    const int lane = threadIdx.x & 31;
    const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int n_warps = (gridDim.x * blockDim.x) >> 5;
    const unsigned gbit = 1u << (lane >> 2);
    for (int t = warp_global; t < n_tiles; t += n_warps) {
        const T* s = slab + (size_t)t * ld * TR + lane * RPL;
        const uint8_t* m = mask + (size_t)t * ld;
        int64_t at[RPL];
        int c[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
            at[q] = pos ? pos[(size_t)t * TR + lane * RPL + q] : 0;
            c[q] = 0;
        }
        for (int k = 0; k < n_cols; ++k) {
            if (!(m[k] & gbit)) continue;
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const T v = s[(size_t)k * TR + q];
                if (v != T(0)) {
                    if (pos) {
                        cols_out[at[q]] = k;
                        vals_out[at[q]] = v;
                        ++at[q];
                    }
                    ++c[q];
                }
            }
        }
        if (!pos)
#pragma unroll
            for (int q = 0; q < RPL; ++q) counts[(size_t)t * TR + lane * RPL + q] = c[q];
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
