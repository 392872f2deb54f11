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
// TR rows.  16 bits per (tile, neuron) flag which 32-byte sectors (2 lanes)
// of the line hold a nonzero; zero sectors are not stored, and their
// gathers read the tile's dedicated zero line (line ld-1) instead; slots
// whose whole line is zero are dropped from the warp's slot list before any
// gather.
//
// A cooperative persistent kernel walks all layers with one grid barrier per
// live layer and a per-layer live-tile count, so layers after the last live
// row cost a loop iteration.  Y0 (CSR) is expanded into tiles by
// densify_kernel beforehand.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sdnn {

// One accumulation step acc + y*w.  float64 (the parity path) rounds the
// multiply and the add apart, like the reference's mulsd + addsd; float32
// (the throughput path) uses one fused multiply-add per step, which the
// oracle's float instance mirrors with fmaf.
template <typename T> struct Arith;
template <> struct Arith<float> {
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float muladd(float y, float w, float acc) { return __fmaf_rn(y, w, acc); }
};
template <> struct Arith<double> {
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double muladd(double y, double w, double acc) {
        return __dadd_rn(acc, __dmul_rn(y, w));
    }
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
// Output lines are streamed (evict-first): a layer's output is read only in
// the next layer, after the whole slab has been written, so keeping it in L2
// would only push out the input lines still being gathered.
__device__ __forceinline__ void st16(char* p, const float (&d)[4]) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(d[0], d[1], d[2], d[3]));
}
__device__ __forceinline__ void st16(char* p, const double (&d)[2]) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(d[0], d[1]));
}

// One live slot of a warp's compacted slot list (16 bytes).
template <typename T>
struct __align__(16) SlotEntry {
    unsigned off;   // line byte offset k * 512
    unsigned mask;  // nonzero sectors of that line
    T w;            // weight
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
    uint16_t* mask[2];    // [n_tiles][ld] nonzero 32-byte sectors of each line
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

// Sector mask of a line from the lanes holding a nonzero: bit s <- lanes 2s, 2s+1.
__device__ __forceinline__ unsigned sector_mask(unsigned lanes) {
    const unsigned pair = (lanes | (lanes >> 1)) & 0x55555555u;  // bit 2s set if lane 2s or 2s+1
    // compress even bits to the low 16 bits
    unsigned x = pair;
    x = (x | (x >> 1)) & 0x33333333u;
    x = (x | (x >> 2)) & 0x0F0F0F0Fu;
    x = (x | (x >> 4)) & 0x00FF00FFu;
    x = (x | (x >> 8)) & 0x0000FFFFu;
    return x;
}

// ------------------------------------------------------------ densify
// Expand Y0 (CSR) into tiles: one block (8 warps) per tile; warp w owns rows
// w, w+8, ...  Each row keeps a 32-entry window of its (ascending) CSR
// entries in registers, one per lane, and refills it only when every entry
// of the window is consumed, so a row costs one coalesced load per 32
// entries however many chunks it spans.  Chunks of kc input neurons are
// assembled in a shared [kc][TR] staging tile, then written out as whole
// coalesced lines (only lines holding a nonzero) with their sector masks,
// and the staging tile is re-zeroed.  Also records the tile's live rows and
// zeroes the tile's zero line in both slab buffers.
constexpr int kDensifyThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kDensifyThreads) densify_kernel(const int64_t* __restrict__ csr_off,
                                                                  const int32_t* __restrict__ csr_cols,
                                                                  const T* __restrict__ csr_vals,
                                                                  const int32_t* __restrict__ rowid, int n_in,
                                                                  int ld, int n_tiles, int kc, T* slab0, T* slab1,
                                                                  uint16_t* mask0, uint32_t* alive0,
                                                                  int32_t* tile_count0) {
    extern __shared__ __align__(16) unsigned char dsm[];
    constexpr int TR = tile_rows<T>(), RPL = rows_per_lane<T>();
    constexpr int NW = kDensifyThreads / 32, RW = TR / NW;  // rows per warp
    T* stage = reinterpret_cast<T*>(dsm);                  // [kc][TR]
    __shared__ int64_t s_pos[TR], s_end[TR];               // window base, row end
    __shared__ uint32_t s_alive[alive_words<T>()];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    {
        float4* st4 = reinterpret_cast<float4*>(stage);
        for (int i = tid; i < kc * kLineBytes / 16; i += blockDim.x) st4[i] = z;
    }
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        if (tid < alive_words<T>()) s_alive[tid] = 0u;
        __syncthreads();
        if (tid < TR) {
            const int row = rowid[(size_t)t * TR + tid];
            const int64_t p = row >= 0 ? csr_off[row] : 0, e = row >= 0 ? csr_off[row + 1] : 0;
            s_pos[tid] = p;
            s_end[tid] = e;
            if (e > p) {
                atomicOr(&s_alive[tid % RPL], 1u << (tid / RPL));
                atomicOr(&s_alive[RPL], 1u);
            }
        }
        __syncthreads();
        int cb[RW];
        T vb[RW];
#pragma unroll
        for (int i = 0; i < RW; ++i) {
            const int r = warp + i * NW;
            const int64_t q = s_pos[r] + lane;
            cb[i] = q < s_end[r] ? csr_cols[q] : INT32_MAX;
            vb[i] = q < s_end[r] ? csr_vals[q] : T(0);
        }
        char* s0 = reinterpret_cast<char*>(slab0 + (size_t)t * ld * TR);
        char* s1 = reinterpret_cast<char*>(slab1 + (size_t)t * ld * TR);
        if (warp == 0) {
            *reinterpret_cast<float4*>(s0 + (size_t)(ld - 1) * kLineBytes + lane * 16) = z;
            *reinterpret_cast<float4*>(s1 + (size_t)(ld - 1) * kLineBytes + lane * 16) = z;
        }
        uint16_t* gm = mask0 + (size_t)t * ld;
        for (int k0 = 0; k0 < n_in; k0 += kc) {
            const int kn = min(kc, n_in - k0);
            bool mine = false;
#pragma unroll
            for (int i = 0; i < RW; ++i) mine |= cb[i] < k0 + kn;
            if (!__syncthreads_or(mine)) {  // the whole chunk is zero for every row
                for (int k = tid; k < kn; k += blockDim.x) gm[k0 + k] = 0;
                continue;
            }
#pragma unroll
            for (int i = 0; i < RW; ++i) {
                const int r = warp + i * NW;
                while (true) {
                    if (cb[i] < k0 + kn) {
                        stage[(size_t)(cb[i] - k0) * TR + r] = vb[i];
                        cb[i] = INT32_MAX;
                    }
                    if (__ballot_sync(0xffffffffu, cb[i] != INT32_MAX)) break;  // window not used up
                    const int64_t base = s_pos[r] + 32;
                    if (base >= s_end[r]) break;                              // row done
                    __syncwarp();  // every lane has read s_pos[r]
                    if (lane == 0) s_pos[r] = base;
                    __syncwarp();  // the new base is visible to later reads
                    const int64_t q = base + lane;
                    cb[i] = q < s_end[r] ? csr_cols[q] : INT32_MAX;
                    vb[i] = q < s_end[r] ? csr_vals[q] : T(0);
                }
            }
            __syncthreads();
            // write out the chunk's nonzero lines and their sector masks
            for (int k = warp; k < kn; k += NW) {
                char* src = reinterpret_cast<char*>(stage) + (size_t)k * kLineBytes + lane * 16;
                const float4 q = *reinterpret_cast<const float4*>(src);
                const bool any = (q.x != 0.f) | (q.y != 0.f) | (q.z != 0.f) | (q.w != 0.f);
                const unsigned m = sector_mask(__ballot_sync(0xffffffffu, any));
                if (m & (1u << (lane >> 1)))
                    *reinterpret_cast<float4*>(s0 + (size_t)(k0 + k) * kLineBytes + lane * 16) = q;
                if (lane == 0) gm[k0 + k] = (uint16_t)m;
                *reinterpret_cast<float4*>(src) = z;  // re-zero for the next chunk
            }
        }
        __syncthreads();
        if (tid < alive_words<T>()) alive0[(size_t)t * alive_words<T>() + tid] = s_alive[tid];
        if (tid == 0 && s_alive[RPL]) atomicAdd(tile_count0, 1);
    }
}

// ------------------------------------------------------------ one item
// Output columns [j0, j1) of tile t for layer l: warp per column.
// The warp walks its columns' 32-slot batches with a three-stage prefetch
// (slot indices + weights two batches ahead, the lines' group masks one
// batch ahead).  In a batch, lane s holds slot s (input line offset, group
// mask, weight); slots whose line is entirely zero are dropped and the rest
// are compacted, in slot order, into the warp's smem list, which is then
// gathered GB lines at a time.  Each lane chains its RPL rows separately.
// Live-row bits go straight to the tile's alive words (one atomic per word).
template <typename T, int GB>
__device__ __forceinline__ void layer_item(const NetArgs<T>& a, const LayerDesc<T>& L, int l, int t,
                                           int j0, int j1, SlotEntry<T>* wlist) {
    using A = Arith<T>;
    constexpr int RPL = rows_per_lane<T>(), AW = alive_words<T>();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned sbit = 1u << (lane >> 1);
    const size_t tile_lines = (size_t)t * a.ld;
    // select, not index: a runtime index into the parameter struct would
    // force a local-memory copy of it
    const bool odd = l & 1;
    const char* in = reinterpret_cast<const char*>(odd ? a.slab[1] : a.slab[0]) + tile_lines * kLineBytes + lane * 16;
    char* out = reinterpret_cast<char*>(odd ? a.slab[0] : a.slab[1]) + tile_lines * kLineBytes + lane * 16;
    const uint16_t* imask = (odd ? a.mask[1] : a.mask[0]) + tile_lines;
    uint16_t* omask = (odd ? a.mask[0] : a.mask[1]) + tile_lines;
    const unsigned zoff = (unsigned)(a.ld - 1) * kLineBytes;
    const int jw = j0 + warp;
    if (jw >= j1) return;
    const int nb = L.wp / 32;  // batches per column
    const int n_cols = (j1 - jw + kWarps - 1) / kWarps;
    const int total = n_cols * nb;
    if (total == 0) {  // zero-width layer: every output is an empty chain
        for (int j = jw; j < j1; j += kWarps)
            if (lane == 0) omask[j] = 0;
        return;
    }
    auto slot_ptr = [&](int b) {
        const int j = jw + (b / nb) * kWarps;
        return (size_t)j * L.wp + (size_t)(b % nb) * 32 + lane;
    };
    // pipeline registers: (k1, w1) for batch b+1, (k2, w2) for batch b+2
    int k0 = __ldg(L.idx + slot_ptr(0));
    T w0 = __ldg(L.val + slot_ptr(0));
    int k1 = -1, k2 = -1;
    T w1 = T(0), w2 = T(0);
    if (total > 1) {
        k1 = __ldg(L.idx + slot_ptr(1));
        w1 = __ldg(L.val + slot_ptr(1));
    }
    unsigned m0 = k0 >= 0 ? (unsigned)imask[k0] : 0u;
    T acc[RPL];
    uint32_t alive_acc[RPL];
#pragma unroll
    for (int c = 0; c < RPL; ++c) {
        acc[c] = T(0);
        alive_acc[c] = 0u;
    }
    for (int b = 0; b < total; ++b) {
        // issue the next loads before working on batch b
        if (b + 2 < total) {
            k2 = __ldg(L.idx + slot_ptr(b + 2));
            w2 = __ldg(L.val + slot_ptr(b + 2));
        }
        const unsigned m1 = (b + 1 < total && k1 >= 0) ? (unsigned)imask[k1] : 0u;

        const unsigned live = __ballot_sync(0xffffffffu, m0 != 0u);
        if (m0) {
            SlotEntry<T> e;
            e.off = (unsigned)k0 * kLineBytes;
            e.mask = m0;
            e.w = w0;
            wlist[__popc(live & ((1u << lane) - 1u))] = e;
        }
        __syncwarp();
        const int n = __popc(live);
        for (int i0 = 0; i0 < n; i0 += GB) {
            T y[GB][RPL];
#pragma unroll
            for (int u = 0; u < GB; ++u) {
                if (i0 + u < n) {
                    const unsigned off = (wlist[i0 + u].mask & sbit) ? wlist[i0 + u].off : zoff;
                    ld16(y[u], in + off);
                }
            }
#pragma unroll
            for (int u = 0; u < GB; ++u) {
                if (i0 + u < n) {
                    const T w = wlist[i0 + u].w;
#pragma unroll
                    for (int c = 0; c < RPL; ++c) acc[c] = A::muladd(y[u][c], w, acc[c]);
                }
            }
        }
        __syncwarp();
        if (b % nb == nb - 1) {  // column complete: epilogue
            const int j = jw + (b / nb) * kWarps;
            T v[RPL];
            bool any = false;
#pragma unroll
            for (int c = 0; c < RPL; ++c) {
                v[c] = a.epilogue ? bias_relu_clamp(acc[c], L.bias, a.ymax) : acc[c];
                any |= v[c] != T(0);
                alive_acc[c] |= __ballot_sync(0xffffffffu, v[c] != T(0));
                acc[c] = T(0);
            }
            const unsigned om = sector_mask(__ballot_sync(0xffffffffu, any));
            if (om & sbit) st16(out + (size_t)j * kLineBytes, v);
            if (lane == 0) __stcs(reinterpret_cast<unsigned short*>(omask + j), (unsigned short)om);
        }
        k0 = k1;
        w0 = w1;
        m0 = m1;
        k1 = k2;
        w1 = w2;
    }
    // live rows of this warp's columns -> the tile's alive words
    bool any_alive = false;
#pragma unroll
    for (int c = 0; c < RPL; ++c) any_alive |= alive_acc[c] != 0u;
    if (lane == 0 && any_alive) {
        uint32_t* aw = a.alive + ((size_t)(l + 1) * a.n_tiles + t) * AW;
#pragma unroll
        for (int c = 0; c < RPL; ++c)
            if (alive_acc[c]) atomicOr(&aw[c], alive_acc[c]);
        if (atomicOr(&aw[RPL], 1u) == 0u) atomicAdd(&a.tile_count[l + 1], 1);
    }
}

// GB = lines gathered per batch (loads in flight per warp); fewer CTAs per
// SM for the deeper batch so its registers fit.
template <typename T, int GB>
__global__ void __launch_bounds__(kThreads, GB <= 8 ? 3 : 2) net_kernel(NetArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    int32_t* tiles = reinterpret_cast<int32_t*>(smem);
    __shared__ SlotEntry<T> s_list[kWarps][32];
    __shared__ int s_count;
    __shared__ int s_scan[kWarps + 1];
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
        for (long long it = blockIdx.x; it < items; it += gridDim.x) {
            const int t = tiles[it / nblk];
            const int b = (int)(it % nblk);
            const int j0 = b * a.jb, j1 = min(a.n_out, j0 + a.jb);
            layer_item<T, GB>(a, L, l, t, j0, j1, s_list[warp]);
        }
        grid_barrier(a.bar, nb);
        if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[l + 1] = globaltimer();
    }
}

// Read back the rows of each tile of the final slab, one warp per tile,
// each lane its RPL rows: pass 1 (pos == null) counts entries, pass 2 writes
// (column, value) in ascending column order at pos[tile * TR + row].
template <typename T>
__global__ void extract_kernel(const T* __restrict__ slab, const uint16_t* __restrict__ mask, int ld,
                               int n_cols, int n_tiles, const int64_t* __restrict__ pos,
                               int32_t* __restrict__ counts, int32_t* __restrict__ cols_out,
                               T* __restrict__ vals_out) {
    constexpr int RPL = rows_per_lane<T>(), TR = tile_rows<T>();
    const int lane = threadIdx.x & 31;
    const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int n_warps = (gridDim.x * blockDim.x) >> 5;
    const unsigned sbit = 1u << (lane >> 1);
    for (int t = warp_global; t < n_tiles; t += n_warps) {
        const T* s = slab + (size_t)t * ld * TR + lane * RPL;
        const uint16_t* m = mask + (size_t)t * ld;
        int64_t at[RPL];
        int c[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
            at[q] = pos ? pos[(size_t)t * TR + lane * RPL + q] : 0;
            c[q] = 0;
        }
        for (int k = 0; k < n_cols; ++k) {
            if (!(m[k] & sbit)) continue;
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
