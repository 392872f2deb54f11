// sdnn.cu -- host side of libsdnn.so: the C ABI declared in include/sdnn.h.
//
// Owns device memory (weights, activations, live-row lists), launches the
// sm_100a kernels of sdnn_kernels.cuh, and converts between the reference's
// host layouts (CSR int64/float64, model.py:51-125) and the device layouts:
//   weights  ELL by output column, slot-major [width][n] int32 + T, inputs
//            ascending per column (so each output is one ordered chain);
//   Y0       CSR (int64 offsets, int32 columns, T values);
//   Y_l      dense rows [rows][n] of T for live rows, ping-pong buffers;
//   live     int32 row lists + per-layer counts (R_l).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sdnn.h"
#include "sdnn_kernels.cuh"

#include <omp.h>

// csrc/sdnn_host.c: AVX2 narrowing of int64 columns to uint16 with
// non-temporal staging stores
extern "C" void sdnn_host_narrow16(const int64_t* cc, const double* vv, uint16_t* d16, int64_t m, int64_t ncols,
                                   int* bad, int* bin);

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

using namespace sdnn;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return fail(SDNN_ERR_CAPACITY, "%s failed: %s (%s:%d)", #call,              \
                        cudaGetErrorString(e_), __FILE__, __LINE__);                     \
    } while (0)

double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

int host_threads() {
    int n = (int)std::thread::hardware_concurrency();
    n = env_int("SDNN_HOST_THREADS", n);
    return std::max(1, std::min(n, 64));
}

template <typename F>
void parallel_for(int64_t n, F f) {
    int nt = (int)std::min<int64_t>(host_threads(), std::max<int64_t>(1, n / 4096));
    if (nt <= 1) {
        f(0, n);
        return;
    }
    std::vector<std::thread> ts;
    int64_t per = (n + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) {
        int64_t a = t * per, b = std::min(n, a + per);
        if (a >= b) break;
        ts.emplace_back([=] { f(a, b); });
    }
    for (auto& t : ts) t.join();
}

struct DevLayer {
    int width = 0;           // real slots (max column degree)
    int wp = 0;              // padded to a multiple of 32
    int32_t* idx = nullptr;  // [n][wp], -1 = padding
    void* val = nullptr;     // [n][wp] of T
    double bias = 0;
    int64_t bytes = 0;
};

}  // namespace

struct sdnn_net {
    int device = 0;
    int dtype = SDNN_F32;
    int64_t n = 0;
    int elem = 4;
    int sm_count = 0;
    int jb = 256;  // outputs per work item
    std::vector<DevLayer> layers;
    void* descs = nullptr;  // device LayerDesc<T>[layers]
    int64_t descs_n = 0;    // layers mirrored in `descs`
    cudaStream_t stream = nullptr;
    cudaStream_t ustream = nullptr;  // uploads of a streamed infer (producer thread)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t ev_d = nullptr, ev_b = nullptr;  // after densify, after the bit-line layer
    // run scratch, grown on demand
    void* slab[2] = {nullptr, nullptr};
    uint2* meta[2] = {nullptr, nullptr};
    void* zero = nullptr;  // one all-zero 32-byte sector
    int64_t tcap = 0;  // tiles per buffer
    int64_t tcap_lines = 0;
    int32_t* rowid = nullptr;
    int32_t* rowlist = nullptr;
    int64_t rcap = 0;
    uint32_t* alive = nullptr;
    int64_t acap = 0;
    int32_t* rowid_buf = nullptr;  // per-run scratch below: grown, never freed per run
    int64_t idcap = 0;
    int32_t* rowid_alt = nullptr;  // the row-id map after an odd number of row compactions
    int64_t idcap2 = 0;
    uint32_t* alive_c = nullptr;   // row bitmaps of repacked tiles
    int64_t accap = 0;
    int* n_compact = nullptr;
    int* probe_flag = nullptr;  // layer-1 walk chosen by quad_probe_kernel
    uint32_t* prune_map = nullptr;  // prune pass: one bit per (tile, output)
    int64_t pmcap = 0;
    unsigned char* pp_codes = nullptr;  // prune pass: bound codes per tile
    int64_t pccap = 0;
    unsigned* pp_tmax = nullptr;
    int64_t ptcap = 0;
    int32_t* tile_count = nullptr;
    int64_t* live_rows = nullptr;
    unsigned long long* stamps = nullptr;
    uint32_t* heap = nullptr;
    unsigned* work = nullptr;
    int64_t lcap = 0;  // layers + 1 the per-layer scratch holds
    int64_t hcap = 0;  // heap counters
    unsigned* bar = nullptr;
    int32_t* n_sel = nullptr;
    int64_t ccap = 0;
    void* cub_tmp = nullptr;
    size_t cub_cap = 0;
    void* pinned = nullptr;  // two staging buffers of pinned_cap bytes
    size_t pinned_cap = 0;
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    int layer_timing = 0;
    int compact_pct = 10;  // live-row compaction threshold (% of live tiles freed)
    int prune = 1;         // output pruning by line bounds
    // weight-ingest scratch (CSR -> ELL on the device), grown on demand
    void* ing_pinned = nullptr;
    size_t ing_pinned_cap = 0;
    void* ing_dev = nullptr;
    size_t ing_dev_cap = 0;
};

struct sdnn_batch {
    sdnn_net* net = nullptr;
    int64_t n_rows = 0, nnz = 0, n_cols = 0;
    int col_bytes = 4;        // 2: uint16 columns, 4: int32 columns
    int64_t h2d_bytes = 0;    // bytes copied host -> device by the upload
    int64_t* off = nullptr;
    void* cols = nullptr;
    void* vals = nullptr;     // null: every stored value is 1.0
    bool finite = true;       // every stored value is finite (as T)
};

struct sdnn_result {
    int64_t n_rows = 0, n_cols = 0;
    int64_t n_layers = 0;
    std::vector<int64_t> cats;  // 1-based ascending
    std::vector<int64_t> live;  // [n_layers + 1]
    double dev_ms = 0, wall_ms = 0;
    int64_t launches = 0;
    std::vector<double> layer_ms;  // per layer, when layer timing is on
    double stage_ms[3] = {0, 0, 0};  // densify, first (bit-line) layer launch, persistent layer launch
    int64_t h2d_bytes = 0;  // host -> device bytes of the call's uploads (end-to-end calls)
    int64_t segments = 0;   // row segments of a streamed call
    int64_t compactions = 0;  // live-row compactions in the run
    int64_t pruned = 0;       // (tile, output) columns pruned by their line bounds
    bool have_y = false;
    std::vector<int64_t> off, cols;
    std::vector<double> vals;
    // Y kept on the device (single-wave runs): canonical CSR, copied straight
    // into the caller's buffers by sdnn_result_y_csr
    int device = -1;
    int64_t* d_off = nullptr;
    int64_t* d_cols = nullptr;
    double* d_vals = nullptr;
    int64_t d_nnz = 0;
    ~sdnn_result() {
        if (d_off || d_cols || d_vals) {
            cudaSetDevice(device);
            cudaFree(d_off);
            cudaFree(d_cols);
            cudaFree(d_vals);
        }
    }
};

// One handle over several GPUs: a network replica per device (devices may
// repeat), the batch split into contiguous row blocks, one host thread per
// device (engine._infer_data_parallel, engine.py:237-251, one GPU per worker).
struct sdnn_group {
    std::vector<sdnn_net*> nets;
};

namespace {

int set_device(const sdnn_net* net) {
    CK(cudaSetDevice(net->device));
    return SDNN_OK;
}


// Upload one layer given output-major host arrays [n_out][width] with
// deg[j] real slots in column j (nullable: all width slots real); pads to a
// multiple of 32 slots with index -1.
int upload_layer(sdnn_net* net, int64_t n_out, int width, const int32_t* idx_om, const double* val_om,
                 double value_if_null, double bias, const int64_t* deg) {
    DevLayer L;
    L.width = width;
    L.wp = (width + 31) / 32 * 32;
    L.bias = bias;
    const size_t slots = (size_t)L.wp * (size_t)n_out;
    std::vector<int32_t> idx(std::max<size_t>(slots, 1), -1);
    std::vector<unsigned char> val(std::max<size_t>(slots, 1) * net->elem, 0);
    parallel_for(n_out, [&](int64_t j0, int64_t j1) {
        for (int64_t j = j0; j < j1; ++j) {
            const int d = deg ? (int)deg[j] : width;
            for (int s = 0; s < d; ++s) {
                const size_t src = (size_t)j * width + s, dst = (size_t)j * L.wp + s;
                idx[dst] = idx_om[src];
                const double v = val_om ? val_om[src] : value_if_null;
                if (net->dtype == SDNN_F64)
                    reinterpret_cast<double*>(val.data())[dst] = v;
                else
                    reinterpret_cast<float*>(val.data())[dst] = (float)v;
            }
        }
    });
    CK(cudaMalloc(&L.idx, std::max<size_t>(slots, 1) * sizeof(int32_t)));
    CK(cudaMalloc(&L.val, std::max<size_t>(slots, 1) * net->elem));
    CK(cudaMemcpy(L.idx, idx.data(), slots * sizeof(int32_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(L.val, val.data(), slots * net->elem, cudaMemcpyHostToDevice));
    L.bytes = (int64_t)slots * (4 + net->elem);
    net->layers.push_back(L);
    return SDNN_OK;
}

// Mirror the layer table on the device (LayerDesc<T>[]).
template <typename T>
int sync_descs(sdnn_net* net) {
    const int64_t L = (int64_t)net->layers.size();
    if (net->descs_n == L && net->descs) return SDNN_OK;
    std::vector<LayerDesc<T>> d(std::max<int64_t>(L, 1));
    for (int64_t i = 0; i < L; ++i) {
        d[i].idx = net->layers[i].idx;
        d[i].val = reinterpret_cast<const T*>(net->layers[i].val);
        d[i].wp = net->layers[i].wp;
        d[i].bias = (T)net->layers[i].bias;
    }
    if (net->descs) CK(cudaFree(net->descs));
    CK(cudaMalloc(&net->descs, d.size() * sizeof(LayerDesc<T>)));
    CK(cudaMemcpy(net->descs, d.data(), d.size() * sizeof(LayerDesc<T>), cudaMemcpyHostToDevice));
    net->descs_n = L;
    return SDNN_OK;
}

template <typename P>
int grow(P*& p, int64_t& cap, int64_t need, size_t elem) {
    if (need <= cap && p) return SDNN_OK;
    if (p) CK(cudaFree(p));
    p = nullptr;
    CK(cudaMalloc(&p, std::max<int64_t>(need, 1) * elem));
    cap = need;
    return SDNN_OK;
}

int ensure_tiles(sdnn_net* net, int64_t tiles, int64_t ld) {
    if (tiles > net->tcap || !net->slab[0] || ld * std::max<int64_t>(tiles, 1) > net->tcap_lines) {
        for (int b = 0; b < 2; ++b) {
            if (net->slab[b]) CK(cudaFree(net->slab[b]));
            if (net->meta[b]) CK(cudaFree(net->meta[b]));
            net->slab[b] = nullptr;
            net->meta[b] = nullptr;
        }
        const int64_t lines = std::max<int64_t>(tiles, 1) * ld;
        for (int b = 0; b < 2; ++b) {
            CK(cudaMalloc(&net->slab[b], lines * kLineBytes));
            CK(cudaMalloc(&net->meta[b], lines * sizeof(uint2)));
        }
        net->tcap = tiles;
        net->tcap_lines = lines;
    }
    return SDNN_OK;
}

// Rows per wave so the two tile slabs fit next to everything else.
int64_t wave_rows(sdnn_net* net, int64_t n_rows, int64_t ld, int tr) {
    int64_t forced = env_int("SDNN_WAVE_ROWS", 0);
    if (forced > 0) return std::min(forced, std::max<int64_t>(n_rows, 1));
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const int64_t per_tile = 2 * ld * (kLineBytes + 8);
    int64_t held = net->tcap_lines * (kLineBytes + 8) * 2;
    int64_t avail = (int64_t)free_b + held - (int64_t)(2ull << 30);
    // the layer kernels keep the wave's live-tile list and row prefix in
    // dynamic shared memory ((2 * tiles + 1) * 4 bytes beside ~6 KB static):
    // more tiles than fit there become more waves, not a capacity error
    const int64_t smem_tiles = 24000;
    int64_t w = std::min(std::max<int64_t>(1, avail / per_tile), smem_tiles) * tr;
    return std::min(w, std::max<int64_t>(n_rows, 1));
}

struct LivePred {
    const int64_t* off;
    __device__ bool operator()(int r) const { return off[r + 1] > off[r]; }
};

// Assemble the full B-row CSR from per-wave pieces (rows listed in any order).
struct Piece {
    std::vector<int32_t> rows;
    std::vector<int64_t> nnz;
    std::vector<int32_t> cols;
    std::vector<double> vals;
};

void assemble(sdnn_result* res, std::vector<Piece>& pieces) {
    const int64_t B = res->n_rows;
    std::vector<int64_t> cnt(B + 1, 0);
    std::vector<std::pair<int32_t, int64_t>> src(B, {-1, 0});
    for (size_t w = 0; w < pieces.size(); ++w) {
        int64_t at = 0;
        for (size_t i = 0; i < pieces[w].rows.size(); ++i) {
            const int32_t r = pieces[w].rows[i];
            if (r >= 0) {
                cnt[r + 1] = pieces[w].nnz[i];
                src[r] = {(int32_t)w, at};
            }
            at += pieces[w].nnz[i];
        }
    }
    res->off.assign(B + 1, 0);
    for (int64_t r = 0; r < B; ++r) res->off[r + 1] = res->off[r] + cnt[r + 1];
    const int64_t total = res->off[B];
    res->cols.resize(total);
    res->vals.resize(total);
    parallel_for(B, [&](int64_t a, int64_t b) {
        for (int64_t r = a; r < b; ++r) {
            if (src[r].first < 0) continue;
            const Piece& p = pieces[src[r].first];
            const int64_t at = src[r].second, dst = res->off[r], m = cnt[r + 1];
            for (int64_t q = 0; q < m; ++q) {
                res->cols[dst + q] = p.cols[at + q];
                res->vals[dst + q] = p.vals[at + q];
            }
        }
    });
    res->have_y = true;
}

// Final Y of the tiles that are still live -> host CSR pieces.
template <typename T>
int extract(sdnn_net* net, const T* slab, const uint2* meta, int ld, int n_cols, int64_t n_tiles,
            const std::vector<uint32_t>& alive, const std::vector<int32_t>& rowid, Piece& p) {
    constexpr int TR = tile_rows<T>(), AW = alive_words<T>(), RPL = rows_per_lane<T>();
    p.rows.assign(rowid.begin(), rowid.end());
    p.nnz.assign(rowid.size(), 0);
    if (n_tiles == 0) return SDNN_OK;
    int32_t* counts = nullptr;
    int64_t* pos = nullptr;
    int32_t* cols = nullptr;
    T* vals = nullptr;
    const int64_t lanes = n_tiles * TR;
    CK(cudaMalloc(&counts, lanes * 4));
    const int grid = (int)std::min<int64_t>((n_tiles + 7) / 8, (int64_t)net->sm_count * 16);
    extract_kernel<T><<<grid, 256, 0, net->stream>>>(slab, meta, ld, n_cols, (int)n_tiles, nullptr, counts,
                                                     nullptr, nullptr);
    CK(cudaGetLastError());
    std::vector<int32_t> cnt(lanes);
    CK(cudaMemcpyAsync(cnt.data(), counts, lanes * 4, cudaMemcpyDeviceToHost, net->stream));
    CK(cudaStreamSynchronize(net->stream));
    std::vector<int64_t> at(lanes);
    int64_t total = 0;
    for (int64_t i = 0; i < lanes; ++i) {
        const int64_t t = i / TR;
        const int r = (int)(i % TR);
        // a row counts only if it is live at the end; dead tiles hold stale data
        const bool live = (alive[t * AW + r / 32] >> (r % 32)) & 1u;
        const int64_t c = (live && rowid[i] >= 0) ? cnt[i] : 0;
        at[i] = total;
        p.nnz[i] = c;
        total += c;
    }
    CK(cudaMalloc(&pos, lanes * 8));
    CK(cudaMemcpyAsync(pos, at.data(), lanes * 8, cudaMemcpyHostToDevice, net->stream));
    CK(cudaMalloc(&cols, std::max<int64_t>(total, 1) * 4));
    CK(cudaMalloc(&vals, std::max<int64_t>(total, 1) * sizeof(T)));
    // write pass over runs of consecutive live tiles only
    std::vector<int32_t> live_ids;
    for (int64_t t = 0; t < n_tiles; ++t)
        if (alive[t * AW + AW - 1]) live_ids.push_back((int32_t)t);
    for (size_t i = 0; i < live_ids.size();) {
        size_t j = i;
        while (j + 1 < live_ids.size() && live_ids[j + 1] == live_ids[j] + 1) ++j;
        const int64_t t0 = live_ids[i], nt = live_ids[j] - t0 + 1;
        const int g = (int)std::min<int64_t>((nt + 7) / 8, (int64_t)net->sm_count * 16);
        extract_kernel<T><<<g, 256, 0, net->stream>>>(slab + (size_t)t0 * ld * TR, meta + (size_t)t0 * ld, ld, n_cols,
                                                      (int)nt, pos + t0 * TR, nullptr, cols, vals);
        CK(cudaGetLastError());
        i = j + 1;
    }
    std::vector<int32_t> hc(total);
    std::vector<T> hv(total);
    CK(cudaMemcpyAsync(hc.data(), cols, total * 4, cudaMemcpyDeviceToHost, net->stream));
    CK(cudaMemcpyAsync(hv.data(), vals, total * sizeof(T), cudaMemcpyDeviceToHost, net->stream));
    CK(cudaStreamSynchronize(net->stream));
    // rows that are not live keep nnz 0 and are excluded from the write pass,
    // but a live row's count may include stale dead-row slots: none exist,
    // because extraction only reads rows flagged live
    p.cols.assign(hc.begin(), hc.end());
    p.vals.assign(hv.begin(), hv.end());
    cudaFree(counts);
    cudaFree(pos);
    cudaFree(cols);
    cudaFree(vals);
    return SDNN_OK;
}

// Live rows per layer: popcount of the per-lane words (not the tile flag).
__global__ void live_rows_kernel(const uint32_t* __restrict__ alive, int n_tiles, int aw, int64_t* __restrict__ live) {
    __shared__ int s[32];
    const uint32_t* a = alive + (size_t)blockIdx.x * n_tiles * aw;
    int c = 0;
    for (int i = threadIdx.x; i < n_tiles * aw; i += blockDim.x)
        if (i % aw != aw - 1) c += __popc(a[i]);
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t v = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += s[w];
        live[blockIdx.x] = v;
    }
}

// Final Y of a single-wave run, materialised on the device in the
// reference's layout (engine._wrap, engine.py:158-160: row-ordered canonical
// CSR, int64 columns, float64 values); sdnn_result_y_csr then copies it
// straight into the caller's buffers.  Returns 1 (nothing allocated) when
// the device cannot hold it, so the caller falls back to host assembly.
template <typename T>
int extract_device(sdnn_net* net, const T* slab, const uint2* meta, int ld, int n_cols, int64_t n_tiles,
                   const uint32_t* alive_last, int64_t B, sdnn_result* res) {
    constexpr int TR = tile_rows<T>();
    const int64_t lanes = n_tiles * TR;
    cudaStream_t st = net->stream;
    int32_t* counts = nullptr;
    int64_t* rowcnt = nullptr;
    auto give_up = [&]() {
        cudaGetLastError();  // clear the allocation failure
        if (counts) cudaFree(counts);
        if (rowcnt) cudaFree(rowcnt);
        cudaFree(res->d_off);
        cudaFree(res->d_cols);
        cudaFree(res->d_vals);
        res->d_off = res->d_cols = nullptr;
        res->d_vals = nullptr;
        return 1;
    };
    res->device = net->device;
    if (cudaMalloc(&res->d_off, (B + 1) * 8) != cudaSuccess) return give_up();
    if (cudaMalloc(&rowcnt, (B + 1) * 8) != cudaSuccess) return give_up();
    if (lanes && cudaMalloc(&counts, lanes * 4) != cudaSuccess) return give_up();
    CK(cudaMemsetAsync(rowcnt, 0, (B + 1) * 8, st));
    if (lanes) {
        const int grid = (int)std::min<int64_t>((n_tiles + 7) / 8, (int64_t)net->sm_count * 16);
        extract_kernel<T><<<grid, 256, 0, st>>>(slab, meta, ld, n_cols, (int)n_tiles, nullptr, counts, nullptr,
                                                nullptr);
        CK(cudaGetLastError());
        row_counts_kernel<T><<<(unsigned)std::min<int64_t>((lanes + 255) / 256, 4096), 256, 0, st>>>(
            counts, net->rowid, alive_last, lanes, rowcnt);
        CK(cudaGetLastError());
    }
    size_t tmp_bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, rowcnt, res->d_off, (int)(B + 1), st));
    if (tmp_bytes > net->cub_cap) {
        if (net->cub_tmp) CK(cudaFree(net->cub_tmp));
        CK(cudaMalloc(&net->cub_tmp, tmp_bytes));
        net->cub_cap = tmp_bytes;
    }
    CK(cub::DeviceScan::ExclusiveSum(net->cub_tmp, tmp_bytes, rowcnt, res->d_off, (int)(B + 1), st));
    int64_t nnz = 0;
    CK(cudaMemcpyAsync(&nnz, res->d_off + B, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (cudaMalloc(&res->d_cols, std::max<int64_t>(nnz, 1) * 8) != cudaSuccess) return give_up();
    if (cudaMalloc(&res->d_vals, std::max<int64_t>(nnz, 1) * 8) != cudaSuccess) return give_up();
    if (nnz) {
        const int grid = (int)std::min<int64_t>((n_tiles + 7) / 8, (int64_t)net->sm_count * 16);
        extract_rows_kernel<T><<<grid, 256, 0, st>>>(slab, meta, ld, n_cols, (int)n_tiles, alive_last, net->rowid,
                                                     res->d_off, res->d_cols, res->d_vals);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(st));
    cudaFree(counts);
    cudaFree(rowcnt);
    res->d_nnz = nnz;
    res->have_y = true;
    return SDNN_OK;
}

// Large device -> pageable host copy: chunks go through two pinned staging
// buffers (DMA at full link speed) while host threads copy the previous
// chunk out in parallel (which also spreads the first-touch page faults of
// a freshly allocated destination over all cores).
int d2h_large(void* dst, const void* src, size_t bytes) {
    constexpr size_t kChunk = 64ull << 20;
    if (bytes <= kChunk) {
        CK(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
        return SDNN_OK;
    }
    char* stage = nullptr;
    CK(cudaMallocHost(&stage, 2 * kChunk));
    cudaStream_t st = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int rc = SDNN_OK;
    auto check = [&](cudaError_t e) {
        if (e != cudaSuccess && rc == SDNN_OK)
            rc = fail(SDNN_ERR_CAPACITY, "Y copy failed: %s", cudaGetErrorString(e));
        return e == cudaSuccess;
    };
    if (check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) && check(cudaEventCreate(&ev[0])) &&
        check(cudaEventCreate(&ev[1]))) {
        const size_t n = (bytes + kChunk - 1) / kChunk;
        for (size_t i = 0; i <= n && rc == SDNN_OK; ++i) {
            if (i < n) {  // chunk i -> buffer i & 1
                const size_t len = std::min(kChunk, bytes - i * kChunk);
                check(cudaMemcpyAsync(stage + (i & 1) * kChunk, static_cast<const char*>(src) + i * kChunk, len,
                                      cudaMemcpyDeviceToHost, st));
                check(cudaEventRecord(ev[i & 1], st));
            }
            if (i > 0) {  // chunk i-1 out of its buffer, in parallel
                const size_t j = i - 1, len = std::min(kChunk, bytes - j * kChunk);
                if (!check(cudaEventSynchronize(ev[j & 1]))) break;
                const char* from = stage + (j & 1) * kChunk;
                char* to = static_cast<char*>(dst) + j * kChunk;
                const int64_t parts = 64;
#pragma omp parallel for schedule(static)
                for (int64_t q = 0; q < parts; ++q) {
                    const size_t a = len * q / parts, b = len * (q + 1) / parts;
                    memcpy(to + a, from + a, b - a);
                }
            }
        }
    }
    if (st) cudaStreamSynchronize(st);
    for (auto e : ev)
        if (e) cudaEventDestroy(e);
    if (st) cudaStreamDestroy(st);
    cudaFreeHost(stage);
    return rc;
}

// Device-held Y -> the result's host vectors (for merging streamed parts).
int y_to_host(sdnn_result* r) {
    if (!r->d_off) return SDNN_OK;
    CK(cudaSetDevice(r->device));
    r->off.resize(r->n_rows + 1);
    r->cols.resize(r->d_nnz);
    r->vals.resize(r->d_nnz);
    if (int rc = d2h_large(r->off.data(), r->d_off, (r->n_rows + 1) * 8)) return rc;
    if (r->d_nnz) {
        if (int rc = d2h_large(r->cols.data(), r->d_cols, r->d_nnz * 8)) return rc;
        if (int rc = d2h_large(r->vals.data(), r->d_vals, r->d_nnz * 8)) return rc;
    }
    cudaFree(r->d_off);
    cudaFree(r->d_cols);
    cudaFree(r->d_vals);
    r->d_off = r->d_cols = nullptr;
    r->d_vals = nullptr;
    return SDNN_OK;
}

// One wave of rows [r0, r1) through layers [first, first + nl).
template <typename T>
int run_wave(sdnn_net* net, const sdnn_batch* batch, double ymax, int64_t first, int64_t nl, int epilogue,
             int64_t r0, int64_t r1, int64_t n_in, int64_t n_out, int want_y, sdnn_result* res,
             std::vector<int32_t>& final_rows, std::vector<Piece>& pieces, float& dev_ms) {
    constexpr int TR = tile_rows<T>(), RPL = rows_per_lane<T>(), AW = alive_words<T>();
    const int64_t ld = std::max(n_in, n_out);
    const int64_t rows = r1 - r0;
    // ascending list of the wave's rows that hold an entry
    if (int rc = grow(net->rowlist, net->rcap, std::max<int64_t>(rows, TR), 4)) return rc;
    if (int rc = grow(net->n_sel, net->ccap, std::max<int64_t>(nl + 2, 2), 8)) return rc;
    size_t tmp_bytes = 0;
    thrust::counting_iterator<int> it((int)r0);
    LivePred pred{batch->off};
    cub::DeviceSelect::If(nullptr, tmp_bytes, it, net->rowlist, net->n_sel, (int)rows, pred, net->stream);
    if (tmp_bytes > net->cub_cap) {
        if (net->cub_tmp) CK(cudaFree(net->cub_tmp));
        CK(cudaMalloc(&net->cub_tmp, tmp_bytes));
        net->cub_cap = tmp_bytes;
    }
    // the run's device time starts here: the live-row select, the host round
    // trip for its count and the scratch clears are part of the timed pass
    CK(cudaEventRecord(net->ev0, net->stream));
    CK(cub::DeviceSelect::If(net->cub_tmp, tmp_bytes, it, net->rowlist, net->n_sel, (int)rows, pred, net->stream));
    int32_t n_live = 0;
    CK(cudaMemcpyAsync(&n_live, net->n_sel, 4, cudaMemcpyDeviceToHost, net->stream));
    CK(cudaStreamSynchronize(net->stream));
    const int64_t n_tiles = (n_live + TR - 1) / TR;
    if (int rc = ensure_tiles(net, n_tiles, ld)) return rc;
    if (int rc = grow(net->rowid_buf, net->idcap, std::max<int64_t>(n_tiles * TR, 1), 4)) return rc;
    if (int rc = grow(net->rowid_alt, net->idcap2, std::max<int64_t>(n_tiles * TR, 1), 4)) return rc;
    net->rowid = net->rowid_buf;
    CK(cudaMemsetAsync(net->rowid, 0xff, std::max<int64_t>(n_tiles * TR, 1) * 4, net->stream));
    if (n_live) CK(cudaMemcpyAsync(net->rowid, net->rowlist, n_live * 4, cudaMemcpyDeviceToDevice, net->stream));
    const int64_t tiles1 = std::max<int64_t>(n_tiles, 1);
    if (int rc = grow(net->alive, net->acap, (nl + 1) * tiles1 * AW, 4)) return rc;
    // per-layer scratch (no cudaMalloc/cudaFree per run: both synchronise
    // and made back-to-back runs stall for hundreds of ms)
    if (nl + 1 > net->lcap) {
        int64_t c1 = 0, c2 = 0, c3 = 0, c4 = 0;
        if (int rc = grow(net->tile_count, c1, nl + 1, 4)) return rc;
        if (int rc = grow(net->live_rows, c2, nl + 1, 8)) return rc;
        if (int rc = grow(net->stamps, c3, nl + 1, 8)) return rc;
        if (int rc = grow(net->work, c4, 5 * (nl + 1), 4)) return rc;  // layers, compactions, pruned columns, prune pass x2
        net->lcap = nl + 1;
    }
    int32_t* tile_count = net->tile_count;
    int64_t* live = net->live_rows;
    unsigned long long* stamps = net->stamps;
    if (!net->bar) CK(cudaMalloc(&net->bar, 8));
    CK(cudaMemsetAsync(net->alive, 0, (nl + 1) * tiles1 * AW * 4, net->stream));
    CK(cudaMemsetAsync(tile_count, 0, (nl + 1) * 4, net->stream));
    CK(cudaMemsetAsync(stamps, 0, (nl + 1) * 8, net->stream));
    CK(cudaMemsetAsync(net->bar, 0, 8, net->stream));
    if (!net->zero) {
        CK(cudaMalloc(&net->zero, 64));
        CK(cudaMemset(net->zero, 0, 64));
    }
    if (int rc = grow(net->heap, net->hcap, (nl + 1) * tiles1, 4)) return rc;
    uint32_t* heap = net->heap;
    CK(cudaMemsetAsync(heap, 0, (nl + 1) * tiles1 * 4, net->stream));
    unsigned* work = net->work;
    CK(cudaMemsetAsync(work, 0, 5 * (nl + 1) * 4, net->stream));
    if (int rc = grow(net->alive_c, net->accap, tiles1 * AW, 4)) return rc;
    if (!net->n_compact) CK(cudaMalloc(&net->n_compact, 4));
    CK(cudaMemsetAsync(net->n_compact, 0, 4, net->stream));

    NetArgs<T> a{};
    a.n_in = (int)n_in;
    a.n_out = (int)n_out;
    a.ld = (int)ld;
    a.L = (int)nl;
    a.layers = reinterpret_cast<const LayerDesc<T>*>(net->descs) + first;
    a.ymax = (T)ymax;
    a.epilogue = epilogue;
    a.n_tiles = (int)n_tiles;
    for (int b = 0; b < 2; ++b) {
        a.slab[b] = reinterpret_cast<T*>(net->slab[b]);
        a.meta[b] = net->meta[b];
    }
    a.heap = heap;
    a.zero = reinterpret_cast<const T*>(net->zero);
    a.alive = net->alive;
    a.tile_count = tile_count;
    a.bar = net->bar;
    a.work = work;
    a.stamps = net->layer_timing ? stamps : nullptr;
    a.rowid[0] = net->rowid_buf;
    a.rowid[1] = net->rowid_alt;
    a.alive_c = net->alive_c;
    a.n_compact = net->n_compact;
    // live-row compaction: repack once that % of the live tiles would be freed
    a.compact_pct = env_int("SDNN_COMPACT", net->compact_pct);
    // ... and only when it frees at least this many tiles: a repack costs a
    // pass over the live rows and a grid barrier (C1 as specified: 4 rows
    // left in 4 tiles, repacking them cost more than it saved)
    a.compact_min = std::max(1, env_int("SDNN_COMPACT_MIN", 16));
    // output pruning by line bounds (sdnn_net_set_pruning; SDNN_PRUNE=0 turns it off)
    a.prune = epilogue ? env_int("SDNN_PRUNE", net->prune) : 0;  // raw Z (engine.spmm) keeps every entry
    a.pruned = work + 2 * (nl + 1);
    a.pp_work = work + 3 * (nl + 1);
    a.jb = env_int("SDNN_JB", net->jb);
    // dense inputs (>= 60 % of sectors kept): 64-output items -- measured on
    // the K2 companion's dense layers, 36.7 -> 29.9 ms at JB 256 -> 64; C4's
    // 34 %-dense layer 2 is fastest at 256 (17.7 vs 18.3 ms at 64)
    a.jb_dense = env_int("SDNN_JB_DENSE", 64);
    a.dense_pct = env_int("SDNN_DENSE_PCT", 60);
    const int kc = std::min(1024, env_int("SDNN_DENSIFY_KC", 96));  // input neurons per staging chunk
    const size_t dsmem = (size_t)kc * kLineBytes;
    const void* dfn = (const void*)densify_kernel<T>;
    CK(cudaFuncSetAttribute(dfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem));
    // Dead-sector handling in the gather: without zero-fill a dead lane keeps
    // its previous (finite) registers and adds them with weight 0, which is
    // exact only when every value the kernel can read is finite.
    const bool zfill = !batch->finite || !std::isfinite((T)ymax) || env_int("SDNN_ZFILL", 0) != 0;
#ifndef SDNN_NET_GB
#define SDNN_NET_GB 4
#endif
    const void* fn = zfill ? (const void*)net_kernel<T, SDNN_NET_GB, true>
                           : (const void*)net_kernel<T, SDNN_NET_GB, false>;
    size_t smem = (size_t)(2 * tiles1 + 1) * 4;  // live-tile list + row prefix
    const size_t smem_list = smem;
    {
        // prune pass: n_in bytes of bound codes behind the tile list, when that
        // keeps the kernel's CTAs per SM (SDNN_PRUNE_PASS=0: never)
        const size_t pp_off = (smem + 15) / 16 * 16, with = pp_off + (size_t)((ld + 15) / 16 * 16);
        int occ0 = 0, occ1 = 0;
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::min<size_t>(with, 200 << 10)));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, fn, kThreads, smem));
        if (with <= (200u << 10)) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, fn, kThreads, with));
        if (a.prune && env_int("SDNN_PRUNE_PASS", 1) != 0 && occ1 >= 1 && occ1 == occ0) {
            if (int rc = grow(net->prune_map, net->pmcap, tiles1 * ((ld + 31) / 32), 4)) return rc;
            a.pp_ldc = (int)((ld + 15) / 16 * 16);
            if (int rc = grow(net->pp_codes, net->pccap, tiles1 * a.pp_ldc, 1)) return rc;
            if (int rc = grow(net->pp_tmax, net->ptcap, tiles1, 4)) return rc;
            a.pp_codes = net->pp_codes;
            a.pp_tmax = net->pp_tmax;
            a.prune_pass = env_int("SDNN_PRUNE_PASS", 1) == 2 ? 2 : 1;
            a.pp_off = (int)pp_off;
            a.prune_map = net->prune_map;
            smem = with;
        }
    }
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, smem));
    if (occ < 1) return fail(SDNN_ERR_CAPACITY, "layer kernel does not fit an SM (smem %zu)", smem);
    occ = std::min(occ, std::max(1, env_int("SDNN_OCC", occ)));
    const int grid = net->sm_count * occ;
    void* args[] = {(void*)&a};
    bool quad = false;  // layer 1 over quad (float) / oct (double) bit-lines
    if (n_tiles) {
        const bool bin = batch->vals == nullptr && env_int("SDNN_BIN", 1) != 0;
        quad = bin && env_int("SDNN_QUAD", 1) != 0;
        constexpr int TPQ = quad_tiles<T>();
        // lines densify does not touch stay {mask 0}: zero the meta first
        // (quad mode: one liveness word per (tile group, line))
        const int64_t meta_rows = quad ? (n_tiles + TPQ - 1) / TPQ : n_tiles;
        CK(cudaMemsetAsync(a.meta[0], 0, (size_t)meta_rows * ld * sizeof(uint2), net->stream));
        // each tile's neurons are split into spans handled by separate blocks
        const int spans = std::max(1, env_int("SDNN_DENSIFY_SPANS", 16));
        a.bin_in = bin ? 1 : 0;
        if (bin) {  // binary Y0: bit-line tiles
            if (quad)  // group lines of dead neurons / missing tiles must read as zero
                CK(cudaMemsetAsync(a.slab[0], 0, (size_t)((n_tiles + TPQ - 1) / TPQ) * ld * kQuadLine,
                                   net->stream));
            // densify_quad_kernel pays one row search per (tile, span): it wins once rows are
            // at least ~6 % dense (C5 p = 0.35: 1.36 -> 1.15 ms, p = 0.7: 2.3 -> 1.8 ms; p = 0.1,
            // 3.9 % dense: 0.68 -> 0.79 ms, so sparser batches keep the chunked kernel);
            // SDNN_DENSIFY_QUAD=0 never, 2 always
            const int dq = env_int("SDNN_DENSIFY_QUAD", 1);
            const bool dense_rows = batch->nnz * 16 >= std::max<int64_t>(batch->n_rows, 1) * n_in;
            if (quad && (dq == 2 || (dq == 1 && dense_rows))) {
                // a span of the tile's bit-lines in shared memory: float 1,024 lines (32 KB, four
                // blocks per SM), double 2,048 lines (SDNN_QSPAN overrides; sweep in DESIGN.md)
                const int qdef = sizeof(T) == 4 ? 1024 : 2048;
                const int qspan = (int)std::min<int64_t>(std::max(32, env_int("SDNN_QSPAN", qdef) / 32 * 32),
                                                         (n_in + 31) / 32 * 32);
                const int64_t qblocks = n_tiles * ((n_in + qspan - 1) / qspan);
                const size_t qsm = (size_t)qspan * (TR / 32) * 4;
                CK(cudaFuncSetAttribute((const void*)densify_quad_kernel<T>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsm));
                densify_quad_kernel<T><<<(int)std::min<int64_t>(qblocks, (int64_t)net->sm_count * 32), kDensifyThreads,
                                         qsm, net->stream>>>(batch->off, batch->cols, batch->col_bytes, net->rowid,
                                                             (int)n_in, (int)ld, (int)n_tiles, qspan, a.slab[0],
                                                             a.meta[0], net->alive, tile_count);
            } else {
            const int kcb = 1024;
            const int span = (int)(((n_in + spans - 1) / spans + kcb - 1) / kcb * kcb);
            const int64_t blocks = n_tiles * ((n_in + span - 1) / span);
            const int dgrid = (int)std::min<int64_t>(blocks, (int64_t)net->sm_count * 32);
            const size_t bsmem = (size_t)kcb * (TR / 32) * 4;
            CK(cudaFuncSetAttribute((const void*)densify_bin_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)bsmem));
            densify_bin_kernel<T><<<dgrid, kDensifyThreads, bsmem, net->stream>>>(
                batch->off, batch->cols, batch->col_bytes, net->rowid, (int)n_in, (int)ld, (int)n_tiles, kcb, span,
                a.slab[0], a.meta[0], heap, net->alive, tile_count, quad ? 1 : 0);
            }
        } else {
            const int span = (int)(((n_in + spans - 1) / spans + kc - 1) / kc * kc);
            const int64_t blocks = n_tiles * ((n_in + span - 1) / span);
            const int dgrid = (int)std::min<int64_t>(blocks, (int64_t)net->sm_count * 32);
            densify_kernel<T><<<dgrid, kDensifyThreads, dsmem, net->stream>>>(
                batch->off, batch->cols, batch->col_bytes, reinterpret_cast<const T*>(batch->vals), net->rowid,
                (int)n_in, (int)ld, (int)n_tiles, kc, span, a.slab[0], a.meta[0], heap, net->alive, tile_count);
        }
        CK(cudaGetLastError());
        res->launches += 1;
    }
    CK(cudaEventRecord(net->ev_d, net->stream));
    if (a.bin_in && quad) {  // layer 1 over quad / oct bit-lines: its own launch
        // dense walk, or -- when a device-side probe of sampled columns says few
        // rows can reach -bias -- the row-prefilter walk (SDNN_PREFILTER=0: never);
        // both variants are launched, the one the probe's flag does not name returns
        const bool pre = a.prune && env_int("SDNN_PREFILTER", 1) != 0;
        const void* qfn = (const void*)bin_quad_kernel<T, false>;
        int qocc = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&qocc, qfn, kThreads, 0));
        int* flag = nullptr;
        if (pre) {
            if (!net->probe_flag) CK(cudaMalloc(&net->probe_flag, 4));
            flag = net->probe_flag;
            quad_probe_kernel<T><<<1, kThreads, 0, net->stream>>>(a, flag, env_int("SDNN_PREFILTER", 1) == 2);
            const void* pfn = (const void*)bin_quad_kernel<T, true>;
            const size_t qsmem = (size_t)kWarps * quad_warp_smem<T>();
            CK(cudaFuncSetAttribute(pfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsmem));
            int pocc = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pocc, pfn, kThreads, qsmem));
            bin_quad_kernel<T, true><<<net->sm_count * std::max(pocc, 1), kThreads, qsmem, net->stream>>>(a, flag);
            res->launches += 2;
        }
        bin_quad_kernel<T, false><<<net->sm_count * std::max(qocc, 1), kThreads, 0, net->stream>>>(a, flag);
        CK(cudaGetLastError());
        res->launches += 1;
        a.first_l = 1;
    } else if (a.bin_in) {  // layer 1 over bit-line tiles: its own launch
        const void* bfn = (const void*)bin_layer_kernel<T>;
        CK(cudaFuncSetAttribute(bfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_list));
        int bocc = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bocc, bfn, kThreads, smem_list));
        bin_layer_kernel<T><<<net->sm_count * std::max(bocc, 1), kThreads, smem_list, net->stream>>>(a);
        CK(cudaGetLastError());
        res->launches += 1;
        a.first_l = 1;
    }
    CK(cudaEventRecord(net->ev_b, net->stream));
    if (a.first_l < a.L) {
        CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), args, smem, net->stream));
        res->launches += 1;
    }
    CK(cudaEventRecord(net->ev1, net->stream));
    live_rows_kernel<<<(unsigned)(nl + 1), 256, 0, net->stream>>>(net->alive, (int)tiles1, AW, live);
    CK(cudaGetLastError());
    res->launches += 1;
    std::vector<int64_t> lr(nl + 1);
    std::vector<unsigned long long> st(nl + 1);
    std::vector<uint32_t> alive_last(tiles1 * AW);
    std::vector<int32_t> rowid(n_tiles * TR);
    int n_compact = 0;
    std::vector<unsigned> pruned(nl + 1);
    CK(cudaMemcpyAsync(pruned.data(), a.pruned, (nl + 1) * 4, cudaMemcpyDeviceToHost, net->stream));
    CK(cudaMemcpyAsync(&n_compact, net->n_compact, 4, cudaMemcpyDeviceToHost, net->stream));
    CK(cudaMemcpyAsync(lr.data(), live, (nl + 1) * 8, cudaMemcpyDeviceToHost, net->stream));
    CK(cudaMemcpyAsync(st.data(), stamps, (nl + 1) * 8, cudaMemcpyDeviceToHost, net->stream));
    CK(cudaMemcpyAsync(alive_last.data(), net->alive + nl * tiles1 * AW, tiles1 * AW * 4, cudaMemcpyDeviceToHost,
                       net->stream));
    CK(cudaStreamSynchronize(net->stream));
    // an odd number of compactions leaves the row-id map in the other buffer
    // and the final slab in the other parity
    if (n_compact & 1) net->rowid = net->rowid_alt;
    res->compactions += n_compact;
    for (unsigned c : pruned) res->pruned += c;
    if (n_tiles) CK(cudaMemcpy(rowid.data(), net->rowid, n_tiles * TR * 4, cudaMemcpyDeviceToHost));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, net->ev0, net->ev1));
    dev_ms += ms;
    {
        float m0 = 0, m1 = 0, m2 = 0;
        CK(cudaEventElapsedTime(&m0, net->ev0, net->ev_d));
        CK(cudaEventElapsedTime(&m1, net->ev_d, net->ev_b));
        CK(cudaEventElapsedTime(&m2, net->ev_b, net->ev1));
        res->stage_ms[0] += m0;
        res->stage_ms[1] += m1;
        res->stage_ms[2] += m2;
    }
    for (int64_t l = 0; l <= nl; ++l) res->live[l] += lr[l];
    if (net->layer_timing)
        for (int64_t l = 0; l < nl; ++l)
            if (st[l + 1] && st[l]) res->layer_ms[l] += (double)(st[l + 1] - st[l]) * 1e-6;
    for (int64_t t = 0; t < n_tiles; ++t)
        for (int r = 0; r < TR; ++r)
            if ((alive_last[t * AW + r / 32] >> (r % 32)) & 1u) final_rows.push_back(rowid[t * TR + r]);
    if (want_y && r0 == 0 && r1 == batch->n_rows && env_int("SDNN_HOST_Y", 0) == 0) {
        // the whole batch in one wave: Y goes straight into a device CSR
        const int last = (int)((nl + n_compact) & 1);
        res->n_rows = batch->n_rows;
        int rc = extract_device<T>(net, reinterpret_cast<const T*>(net->slab[last]), net->meta[last], (int)ld,
                                   (int)n_out, n_tiles, net->alive + nl * tiles1 * AW, batch->n_rows, res);
        if (rc == SDNN_OK) return SDNN_OK;
        if (rc != 1) return rc;  // a CUDA failure; 1 = no room, assemble on the host instead
    }
    if (want_y) {
        Piece p;
        const int last = (int)((nl + n_compact) & 1);  // layer nl-1 wrote buffer (nl + flips) & 1
        if (int rc = extract<T>(net, reinterpret_cast<const T*>(net->slab[last]), net->meta[last], (int)ld,
                                (int)n_out, n_tiles, alive_last, rowid, p))
            return rc;
        pieces.push_back(std::move(p));
    }

    return SDNN_OK;
}

template <typename T>
int run_impl(sdnn_net* net, const sdnn_batch* batch, double ymax, int64_t first, int64_t nl, int want_y,
             int epilogue, int64_t n_in, int64_t n_out, sdnn_result* res) {
    const int64_t B = batch->n_rows;
    const int64_t ld = std::max(n_in, n_out);
    if (int rc = sync_descs<T>(net)) return rc;
    const int64_t wave = wave_rows(net, B, ld, tile_rows<T>());
    res->n_rows = B;
    res->n_cols = n_out;
    res->n_layers = nl;
    res->live.assign(nl + 1, 0);
    if (net->layer_timing) res->layer_ms.assign(nl, 0.0);
    std::vector<Piece> pieces;
    std::vector<int32_t> final_rows;
    float dev_ms = 0;
    for (int64_t r0 = 0; r0 < std::max<int64_t>(B, 1); r0 += wave) {
        const int64_t r1 = std::min(B, r0 + wave);
        if (int rc = run_wave<T>(net, batch, ymax, first, nl, epilogue, r0, r1, n_in, n_out, want_y, res,
                                 final_rows, pieces, dev_ms))
            return rc;
        if (B == 0) break;
    }
    std::sort(final_rows.begin(), final_rows.end());
    res->cats.resize(final_rows.size());
    for (size_t i = 0; i < final_rows.size(); ++i) res->cats[i] = (int64_t)final_rows[i] + 1;
    res->dev_ms = dev_ms;
    if (want_y && !res->d_off) assemble(res, pieces);
    return SDNN_OK;
}

// Host CSR (int64/float64) -> device CSR (int64 offsets, int32 cols, T vals).
// Host CSR (int64 columns, float64 values: the reference's FeatureBatch) ->
// device CSR (int64 offsets, uint16 columns when n_cols <= 65536 else
// int32, T values -- or no values at all when every value is 1.0, the
// binary images of the challenge).  Converted by OpenMP threads chunk by
// chunk into two pinned staging buffers while the previous chunk's copy is
// in flight; device buffers come from the stream-ordered pool.
template <typename T>
int upload_csr(sdnn_net* net, int64_t n_rows, const int64_t* off, const int64_t* cols,
               const double* vals, int64_t n_cols, sdnn_batch* b, bool raw = false,
               cudaStream_t stream = nullptr) {
    if (!stream) stream = net->stream;
    const int64_t nnz = n_rows > 0 ? off[n_rows] : 0;
    if (n_rows > 0 && off[0] != 0) return fail(SDNN_ERR_PARAMETER, "row_offsets[0] must be 0");
    for (int64_t i = 0; i < n_rows; ++i)
        if (off[i + 1] < off[i]) return fail(SDNN_ERR_PARAMETER, "row_offsets non-monotone at %lld", (long long)i);
    b->n_rows = n_rows;
    b->nnz = nnz;
    b->n_cols = n_cols;
    b->col_bytes = (n_cols <= 65536 && !raw) ? 2 : 4;
    b->h2d_bytes = (n_rows + 1) * 8;
    const int64_t chunk = std::max<int64_t>(1, env_int("SDNN_UPLOAD_CHUNK", 16 << 20));  // entries
    const size_t stage_bytes = (size_t)std::min<int64_t>(chunk, std::max<int64_t>(nnz, 1)) * sizeof(T);
    if (stage_bytes > net->pinned_cap) {
        if (net->pinned) CK(cudaFreeHost(net->pinned));
        net->pinned = nullptr;
        CK(cudaMallocHost(&net->pinned, 2 * stage_bytes));
        net->pinned_cap = stage_bytes;
        for (auto& e : net->stage_ev)
            if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    char* stage[2] = {reinterpret_cast<char*>(net->pinned), reinterpret_cast<char*>(net->pinned) + net->pinned_cap};
    CK(cudaMallocAsync(reinterpret_cast<void**>(&b->off), (n_rows + 1) * sizeof(int64_t), stream));
    CK(cudaMallocAsync(&b->cols, std::max<int64_t>(nnz, 1) * b->col_bytes, stream));
    CK(cudaMemcpyAsync(b->off, off, (n_rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream));
    int bad = 0, binary = 1;
    // pass 1: columns (and the binary check on values)
    int buf = 0;
    for (int64_t c0 = 0; c0 < nnz; c0 += chunk, buf ^= 1) {
        const int64_t c1 = std::min(nnz, c0 + chunk);
        CK(cudaEventSynchronize(net->stage_ev[buf]));  // the copy that last used this buffer
        char* dst = stage[buf];
        const int cb = b->col_bytes;
        int chunk_bad = 0, chunk_bin = 1;
        // branch-free bodies (one loop per column width) so the compiler
        // vectorises them; this pass is bound by host memory bandwidth
        const int64_t* cc = cols + c0;
        const double* vv = vals + c0;
        const int64_t m = c1 - c0;
        const uint64_t ncu = (uint64_t)n_cols;
        if (cb == 2 && (reinterpret_cast<uintptr_t>(dst) & 31) == 0 && env_int("SDNN_NARROW_AVX2", 1)) {
            sdnn_host_narrow16(cc, vv, reinterpret_cast<uint16_t*>(dst), m, n_cols, &chunk_bad, &chunk_bin);
        } else if (cb == 2) {
            uint16_t* d16 = reinterpret_cast<uint16_t*>(dst);
#pragma omp parallel for simd reduction(| : chunk_bad) reduction(& : chunk_bin) schedule(static)
            for (int64_t p = 0; p < m; ++p) {
                chunk_bad |= (int)((uint64_t)cc[p] >= ncu);
                chunk_bin &= (int)(vv[p] == 1.0);
                d16[p] = (uint16_t)cc[p];
            }
        } else {
            int32_t* d32 = reinterpret_cast<int32_t*>(dst);
#pragma omp parallel for simd reduction(| : chunk_bad) reduction(& : chunk_bin) schedule(static)
            for (int64_t p = 0; p < m; ++p) {
                chunk_bad |= (int)((uint64_t)cc[p] >= ncu);
                chunk_bin &= (int)(vv[p] == 1.0);
                d32[p] = (int32_t)cc[p];
            }
        }
        bad |= chunk_bad;
        binary &= chunk_bin;
        CK(cudaMemcpyAsync(reinterpret_cast<char*>(b->cols) + c0 * cb, dst, (c1 - c0) * cb, cudaMemcpyHostToDevice,
                           stream));
        CK(cudaEventRecord(net->stage_ev[buf], stream));
    }
    if (bad) {
        CK(cudaStreamSynchronize(stream));
        return fail(SDNN_ERR_PARAMETER, "column index outside [0, %lld)", (long long)n_cols);
    }
    b->h2d_bytes += nnz * b->col_bytes;
    b->vals = nullptr;
    if (raw || env_int("SDNN_FORCE_VALUES", 0)) binary = 0;
    if (!binary) {  // pass 2: values
        CK(cudaMallocAsync(&b->vals, std::max<int64_t>(nnz, 1) * sizeof(T), stream));
        for (int64_t c0 = 0; c0 < nnz; c0 += chunk, buf ^= 1) {
            const int64_t c1 = std::min(nnz, c0 + chunk);
            CK(cudaEventSynchronize(net->stage_ev[buf]));
            T* dst = reinterpret_cast<T*>(stage[buf]);
            int chunk_fin = 1;
#pragma omp parallel for reduction(& : chunk_fin) schedule(static)
            for (int64_t p = c0; p < c1; ++p) {
                dst[p - c0] = (T)vals[p];
                chunk_fin &= std::isfinite(dst[p - c0]) ? 1 : 0;
            }
            b->finite = b->finite && chunk_fin;
            CK(cudaMemcpyAsync(reinterpret_cast<T*>(b->vals) + c0, dst, (c1 - c0) * sizeof(T), cudaMemcpyHostToDevice,
                               stream));
            CK(cudaEventRecord(net->stage_ev[buf], stream));
        }
        b->h2d_bytes += nnz * (int64_t)sizeof(T);
    }
    CK(cudaStreamSynchronize(stream));
    return SDNN_OK;
}

// ingest.resize_threshold_flatten (ingest.py:128-156) on the device: raw
// uint8 images in, the binary feature batch (device CSR, no values) out.
// The interpolation taps are computed here exactly as numpy computes
// _interp_matrix (ingest.py:111-125): every operation separately rounded.
int images_upload(sdnn_net* net, int64_t n, int side, const uint8_t* pixels, int t, sdnn_batch* b) {
    static const int kSides[] = {32, 64, 128, 256};  // ingest.TARGET_SIDES
    if (std::find(std::begin(kSides), std::end(kSides), t) == std::end(kSides))
        return fail(SDNN_ERR_PARAMETER, "target side %d is not one of (32, 64, 128, 256)", t);
    if (side < 1 || n < 0 || (n > 0 && !pixels)) return fail(SDNN_ERR_PARAMETER, "bad image set");
    if ((int64_t)t * t != net->n)
        return fail(SDNN_ERR_SHAPE, "images resize to %d columns but the network has %lld neurons", t * t,
                    (long long)net->n);
    const size_t smem = ((size_t)side * side + (size_t)t * side + 256) * sizeof(double) +
                        (size_t)t * (sizeof(double2) + sizeof(int2));
    if (smem > 200 * 1024) return fail(SDNN_ERR_CAPACITY, "images of side %d are too large to resample", side);
    std::vector<int2> taps(t);
    std::vector<double2> w(t);
    const volatile double ratio = (double)side / (double)t;
    for (int i = 0; i < t; ++i) {
        volatile double x = ((double)i + 0.5) * ratio;
        x = x - 0.5;
        const double x0 = std::floor(x);
        const volatile double frac = x - x0;
        const volatile double wlo = 1.0 - frac;
        const int64_t a = (int64_t)x0;
        const int lo = (int)std::min<int64_t>(std::max<int64_t>(a, 0), side - 1);
        const int hi = (int)std::min<int64_t>(std::max<int64_t>(a + 1, 0), side - 1);
        if (lo == hi) {
            volatile double one = 0.0 + wlo;
            one = one + frac;  // np.add.at into the same entry
            taps[i] = make_int2(lo, -1);
            w[i] = make_double2(one, 0.0);
        } else {
            taps[i] = make_int2(lo, hi);
            w[i] = make_double2(wlo, frac);
        }
    }
    cudaStream_t st = net->stream;
    b->n_rows = n;
    b->n_cols = (int64_t)t * t;
    b->col_bytes = b->n_cols <= 65536 ? 2 : 4;
    b->vals = nullptr;
    b->finite = true;
    const int words = t * t / 32;
    uint8_t* dpix = nullptr;
    int2* dtaps = nullptr;
    double2* dw = nullptr;
    uint32_t* bits = nullptr;
    int64_t* cnt = nullptr;
    const int64_t npix = n * side * side;
    // scratch freed on every exit path (stream-ordered)
    struct Scratch {
        cudaStream_t st;
        std::vector<void*> p;
        ~Scratch() {
            for (void* q : p) cudaFreeAsync(q, st);
        }
    } scratch{st, {}};
    auto alloc = [&](void** q, size_t bytes) {
        cudaError_t e = cudaMallocAsync(q, bytes, st);
        if (e == cudaSuccess) scratch.p.push_back(*q);
        return e;
    };
    CK(cudaMallocAsync(reinterpret_cast<void**>(&b->off), (n + 1) * sizeof(int64_t), st));
    CK(alloc(reinterpret_cast<void**>(&dpix), std::max<int64_t>(npix, 1)));
    CK(alloc(reinterpret_cast<void**>(&dtaps), t * sizeof(int2)));
    CK(alloc(reinterpret_cast<void**>(&dw), t * sizeof(double2)));
    CK(alloc(reinterpret_cast<void**>(&bits), std::max<int64_t>(n * words, 1) * 4));
    CK(alloc(reinterpret_cast<void**>(&cnt), std::max<int64_t>(n, 1) * 8));
    if (npix) {  // pageable pixels -> pinned staging (host threads) -> device, chunk by chunk
        const int64_t chunk = 16 << 20;
        const size_t stage_bytes = (size_t)std::min<int64_t>(chunk, npix);
        if (stage_bytes > net->pinned_cap) {
            if (net->pinned) CK(cudaFreeHost(net->pinned));
            net->pinned = nullptr;
            CK(cudaMallocHost(&net->pinned, 2 * stage_bytes));
            net->pinned_cap = stage_bytes;
        }
        for (auto& e : net->stage_ev)
            if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        char* stage[2] = {reinterpret_cast<char*>(net->pinned), reinterpret_cast<char*>(net->pinned) + net->pinned_cap};
        int buf = 0;
        for (int64_t c0 = 0; c0 < npix; c0 += (int64_t)net->pinned_cap, buf ^= 1) {
            const int64_t len = std::min<int64_t>((int64_t)net->pinned_cap, npix - c0);
            CK(cudaEventSynchronize(net->stage_ev[buf]));
            char* dst = stage[buf];
            const int64_t parts = 16;
#pragma omp parallel for schedule(static)
            for (int64_t q = 0; q < parts; ++q) {
                const int64_t a = len * q / parts, e = len * (q + 1) / parts;
                memcpy(dst + a, pixels + c0 + a, e - a);
            }
            CK(cudaMemcpyAsync(dpix + c0, dst, len, cudaMemcpyHostToDevice, st));
            CK(cudaEventRecord(net->stage_ev[buf], st));
        }
    }
    CK(cudaMemcpyAsync(dtaps, taps.data(), t * sizeof(int2), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dw, w.data(), t * sizeof(double2), cudaMemcpyHostToDevice, st));
    b->h2d_bytes = npix + t * (int64_t)(sizeof(int2) + sizeof(double2));
    CK(cudaMemsetAsync(b->off, 0, 8, st));
    int64_t nnz = 0;
    if (n > 0) {
        CK(cudaFuncSetAttribute((const void*)resize_bits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
        const int grid = (int)std::min<int64_t>(n, (int64_t)net->sm_count * 8);
        resize_bits_kernel<<<grid, 256, smem, st>>>(dpix, n, side, t, dtaps, dw, bits, cnt);
        CK(cudaGetLastError());
        size_t tmp_bytes = 0;
        CK(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, cnt, b->off + 1, (int)n, st));
        if (tmp_bytes > net->cub_cap) {
            if (net->cub_tmp) CK(cudaFree(net->cub_tmp));
            CK(cudaMalloc(&net->cub_tmp, tmp_bytes));
            net->cub_cap = tmp_bytes;
        }
        CK(cub::DeviceScan::InclusiveSum(net->cub_tmp, tmp_bytes, cnt, b->off + 1, (int)n, st));
        CK(cudaMemcpyAsync(&nnz, b->off + n, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    b->nnz = nnz;
    CK(cudaMallocAsync(&b->cols, std::max<int64_t>(nnz, 1) * b->col_bytes, st));
    if (nnz > 0) {
        const int grid = (int)std::min<int64_t>(n, (int64_t)net->sm_count * 8);
        if (b->col_bytes == 2)
            bits_to_cols_kernel<uint16_t><<<grid, 256, 0, st>>>(bits, n, words, b->off,
                                                                reinterpret_cast<uint16_t*>(b->cols));
        else
            bits_to_cols_kernel<int32_t><<<grid, 256, 0, st>>>(bits, n, words, b->off,
                                                               reinterpret_cast<int32_t*>(b->cols));
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(st));
    return SDNN_OK;
}

void free_batch(sdnn_batch* b) {
    if (!b) return;
    cudaStream_t st = b->net ? b->net->stream : nullptr;
    if (b->off) cudaFreeAsync(b->off, st);
    if (b->cols) cudaFreeAsync(b->cols, st);
    if (b->vals) cudaFreeAsync(b->vals, st);
    if (st) cudaStreamSynchronize(st);
    delete b;
}

// CSR by input row (reference LayerWeights) -> output-major ELL, inputs
// ascending per output (rows are visited in ascending order).
// CSR by input -> device ELL by output (weight ingest).
// Host: validate offsets, narrow columns to int32 and values to T into a
// pinned buffer (threads), one H2D.  Device: entry rows, column check and
// degrees, stable radix sort by column, degree scan, max degree, ELL fill.
// Errors as the reference raises them: bad offsets / columns -> parameter.
template <typename T>
int ingest_csr(sdnn_net* net, int64_t n_in, int64_t n_out, const int64_t* off, const int64_t* cols,
               const double* vals, double bias) {
    if (off[0] != 0) return fail(SDNN_ERR_PARAMETER, "inconsistent weight offsets");
    for (int64_t i = 0; i < n_in; ++i)
        if (off[i + 1] < off[i]) return fail(SDNN_ERR_PARAMETER, "weight offsets non-monotone");
    const int64_t nnz = off[n_in];
    if (nnz >= (1LL << 31) || n_out >= (1LL << 31))
        return fail(SDNN_ERR_CAPACITY, "layer with %lld entries exceeds int32 indexing", (long long)nnz);
    const int64_t nz = std::max<int64_t>(nnz, 1);
    const bool timing = env_int("SDNN_INGEST_TIMING", 0) != 0;
    double t_prev = now_ms();
    auto lap = [&](const char* what) {
        if (!timing) return;
        const double t = now_ms();
        fprintf(stderr, "ingest %-12s %8.2f ms\n", what, t - t_prev);
        t_prev = t;
    };
    // pinned: offsets (int64), columns (int32), values (T)
    const size_t pin_bytes = (size_t)(n_in + 1) * 8 + (size_t)nz * (4 + sizeof(T));
    if (pin_bytes > net->ing_pinned_cap) {
        if (net->ing_pinned) CK(cudaFreeHost(net->ing_pinned));
        net->ing_pinned = nullptr;
        CK(cudaMallocHost(&net->ing_pinned, pin_bytes));
        net->ing_pinned_cap = pin_bytes;
    }
    char* hp = reinterpret_cast<char*>(net->ing_pinned);
    int64_t* h_off = reinterpret_cast<int64_t*>(hp);
    int32_t* h_cols = reinterpret_cast<int32_t*>(hp + (size_t)(n_in + 1) * 8);
    T* h_vals = reinterpret_cast<T*>(hp + (size_t)(n_in + 1) * 8 + (size_t)nz * 4);
    std::memcpy(h_off, off, (size_t)(n_in + 1) * 8);
    parallel_for(nnz, [&](int64_t a, int64_t b) {
        for (int64_t p = a; p < b; ++p) {
            const int64_t c = cols[p];
            h_cols[p] = (c < 0 || c >= n_out) ? -1 : (int32_t)c;  // flagged on the device
            h_vals[p] = (T)vals[p];
        }
    });
    lap("host narrow");
    // device scratch: off, cols, keys_out, perm_in, perm_out, rowid, vals, deg, start, flags, cub temp
    size_t sort_bytes = 0, scan_bytes = 0, max_bytes = 0;
    int end_bit = 1;
    while ((1LL << end_bit) < n_out) ++end_bit;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, (int)nz, 0, end_bit, net->stream);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const int32_t*)nullptr, (int32_t*)nullptr, (int)n_out,
                                  net->stream);
    cub::DeviceReduce::Max(nullptr, max_bytes, (const int32_t*)nullptr, (int32_t*)nullptr, (int)n_out, net->stream);
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t o_off = 0, o_cols = o_off + al((size_t)(n_in + 1) * 8), o_keys = o_cols + al((size_t)nz * 4),
                 o_pin = o_keys + al((size_t)nz * 4), o_pout = o_pin + al((size_t)nz * 4),
                 o_row = o_pout + al((size_t)nz * 4), o_vals = o_row + al((size_t)nz * 4),
                 o_deg = o_vals + al((size_t)nz * sizeof(T)), o_start = o_deg + al((size_t)n_out * 4),
                 o_flag = o_start + al((size_t)n_out * 4), o_tmp = o_flag + 256,
                 total = o_tmp + al(std::max(sort_bytes, std::max(scan_bytes, max_bytes)));
    if (total > net->ing_dev_cap) {
        if (net->ing_dev) CK(cudaFree(net->ing_dev));
        net->ing_dev = nullptr;
        CK(cudaMalloc(&net->ing_dev, total));
        net->ing_dev_cap = total;
    }
    char* d = reinterpret_cast<char*>(net->ing_dev);
    int64_t* d_off = reinterpret_cast<int64_t*>(d + o_off);
    int32_t* d_cols = reinterpret_cast<int32_t*>(d + o_cols);
    int32_t* d_keys = reinterpret_cast<int32_t*>(d + o_keys);
    int32_t* d_pin = reinterpret_cast<int32_t*>(d + o_pin);
    int32_t* d_pout = reinterpret_cast<int32_t*>(d + o_pout);
    int32_t* d_row = reinterpret_cast<int32_t*>(d + o_row);
    T* d_vals = reinterpret_cast<T*>(d + o_vals);
    int32_t* d_deg = reinterpret_cast<int32_t*>(d + o_deg);
    int32_t* d_start = reinterpret_cast<int32_t*>(d + o_start);
    int* d_flag = reinterpret_cast<int*>(d + o_flag);  // [0] bad column, [1] max degree
    void* d_tmp = d + o_tmp;
    cudaStream_t st = net->stream;
    CK(cudaMemcpyAsync(d_off, h_off, (size_t)(n_in + 1) * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_cols, h_cols, (size_t)nnz * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_vals, h_vals, (size_t)nnz * sizeof(T), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(d_deg, 0, (size_t)n_out * 4, st));
    CK(cudaMemsetAsync(d_flag, 0, 8, st));
    const int grid = net->sm_count * 8;
    if (nnz) {
        csr_rowid_kernel<<<grid, 256, 0, st>>>(d_off, n_in, d_row);
        csr_degree_kernel<<<grid, 256, 0, st>>>(d_cols, nnz, n_out, d_deg, d_pin, d_flag);
        CK(cudaGetLastError());
        CK(cub::DeviceRadixSort::SortPairs(d_tmp, sort_bytes, d_cols, d_keys, d_pin, d_pout, (int)nnz, 0, end_bit,
                                           st));
    }
    CK(cub::DeviceScan::ExclusiveSum(d_tmp, scan_bytes, d_deg, d_start, (int)n_out, st));
    CK(cub::DeviceReduce::Max(d_tmp, max_bytes, d_deg, d_flag + 1, (int)n_out, st));
    int flags[2] = {0, 0};
    CK(cudaMemcpyAsync(flags, d_flag, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    lap("h2d+sort");
    if (flags[0]) return fail(SDNN_ERR_PARAMETER, "weight column out of range [0, %lld)", (long long)n_out);
    DevLayer L;
    L.width = flags[1];
    L.wp = (L.width + 31) / 32 * 32;
    L.bias = bias;
    const size_t slots = (size_t)L.wp * (size_t)n_out;
    CK(cudaMalloc(&L.idx, std::max<size_t>(slots, 1) * sizeof(int32_t)));
    CK(cudaMalloc(&L.val, std::max<size_t>(slots, 1) * sizeof(T)));
    lap("alloc");
    CK(cudaMemsetAsync(L.idx, 0xff, slots * sizeof(int32_t), st));  // padding: index -1
    CK(cudaMemsetAsync(L.val, 0, slots * sizeof(T), st));            // weight 0
    if (nnz) {
        ell_fill_kernel<T><<<grid, 256, 0, st>>>(d_keys, d_pout, d_start, d_row, d_vals, nnz, L.wp, L.idx,
                                                 reinterpret_cast<T*>(L.val));
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(st));
    lap("fill");
    L.bytes = (int64_t)slots * (4 + (int64_t)sizeof(T));
    net->layers.push_back(L);
    return SDNN_OK;
}

int make_net(int device, int dtype, int64_t n, sdnn_net** out) {
    if (dtype != SDNN_F32 && dtype != SDNN_F64) return fail(SDNN_ERR_PARAMETER, "dtype must be 0 (f32) or 1 (f64)");
    if (n < 1 || n > (1LL << 30)) return fail(SDNN_ERR_PARAMETER, "neuron count %lld out of range", (long long)n);
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) return fail(SDNN_ERR_PARAMETER, "no CUDA device %d", device);
    CK(cudaSetDevice(device));
    int coop = 0;
    CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
    if (!coop) return fail(SDNN_ERR_CAPACITY, "device %d lacks cooperative launch", device);
    sdnn_net* net = new sdnn_net;
    net->device = device;
    net->dtype = dtype;
    net->n = n;
    net->elem = dtype == SDNN_F64 ? 8 : 4;
    CK(cudaDeviceGetAttribute(&net->sm_count, cudaDevAttrMultiProcessorCount, device));
    CK(cudaStreamCreateWithFlags(&net->stream, cudaStreamNonBlocking));
    {  // keep freed upload buffers in the stream-ordered pool between calls
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    CK(cudaEventCreate(&net->ev0));
    CK(cudaEventCreate(&net->ev1));
    CK(cudaEventCreate(&net->ev_d));
    CK(cudaEventCreate(&net->ev_b));
    *out = net;
    return SDNN_OK;
}


// engine.infer end to end with the upload hidden behind the run.  Y0 is cut
// into row segments of about equal nnz; a producer thread converts and
// uploads segment s+1 (host memory bound: int64/float64 CSR in) on its own
// stream while segment s runs on the engine stream.  Rows are independent
// (engine.py:237-251 tiles them the same way), so the segments' outputs
// concatenate to exactly the one-shot result.
int auto_segments(int64_t n_rows, int64_t nnz) {
    const int64_t forced = env_int("SDNN_SEGMENTS", 0);
    if (forced > 0) return (int)std::min<int64_t>(forced, std::max<int64_t>(n_rows, 1));
    const int64_t per = 96ll << 20;  // entries per segment: ~1 GB of host CSR
    int64_t s = std::min<int64_t>(nnz / per, 6);
    s = std::min<int64_t>(s, n_rows / 4096);
    return (int)std::max<int64_t>(s, 1);
}

void merge_part(sdnn_result* res, const sdnn_result& part, int64_t r0, int want_y) {
    for (int64_t c : part.cats) res->cats.push_back(c + r0);
    for (size_t l = 0; l < part.live.size(); ++l) res->live[l] += part.live[l];
    res->dev_ms += part.dev_ms;
    res->launches += part.launches;
    res->compactions += part.compactions;
    res->pruned += part.pruned;
    for (int k = 0; k < 3; ++k) res->stage_ms[k] += part.stage_ms[k];
    for (size_t l = 0; l < part.layer_ms.size() && l < res->layer_ms.size(); ++l) res->layer_ms[l] += part.layer_ms[l];
    if (want_y) {
        const int64_t base = res->off[r0];
        for (int64_t r = 1; r < (int64_t)part.off.size(); ++r) res->off[r0 + r] = base + part.off[r];
        res->cols.insert(res->cols.end(), part.cols.begin(), part.cols.end());
        res->vals.insert(res->vals.end(), part.vals.begin(), part.vals.end());
    }
}

template <typename T>
int infer_streamed(sdnn_net* net, int64_t n_rows, const int64_t* off, const int64_t* cols, const double* vals,
                   double ymax, int want_y, int segments, sdnn_result* res) {
    const int64_t L = (int64_t)net->layers.size();
    if (L < 1) return fail(SDNN_ERR_PARAMETER, "the network has no layers");
    if (n_rows > 0 && off[0] != 0) return fail(SDNN_ERR_PARAMETER, "row_offsets[0] must be 0");
    for (int64_t i = 0; i < n_rows; ++i)
        if (off[i + 1] < off[i]) return fail(SDNN_ERR_PARAMETER, "row_offsets non-monotone at %lld", (long long)i);
    const int64_t nnz = n_rows > 0 ? off[n_rows] : 0;
    const int S = segments > 0 ? (int)std::min<int64_t>(segments, std::max<int64_t>(n_rows, 1))
                               : auto_segments(n_rows, nnz);
    if (int rc = sync_descs<T>(net)) return rc;
    struct Seg {
        int64_t r0 = 0, r1 = 0;
        std::vector<int64_t> off;
        sdnn_batch* b = nullptr;
        int rc = 0;
        std::string err;
    };
    std::vector<Seg> seg(S);
    for (int s = 0; s < S; ++s) {  // row bounds at equal shares of the entries
        auto at = [&](int k) -> int64_t {
            if (k == 0) return 0;
            if (k == S) return n_rows;
            if (nnz == 0) return n_rows * k / S;
            const int64_t want = nnz * k / S;
            return std::min<int64_t>(std::lower_bound(off, off + n_rows + 1, want) - off, n_rows);
        };
        seg[s].r0 = at(s);
        seg[s].r1 = std::max(at(s + 1), seg[s].r0);
    }
    res->n_rows = n_rows;
    res->n_cols = net->n;
    res->n_layers = L;
    res->live.assign(L + 1, 0);
    res->segments = S;
    if (net->layer_timing) res->layer_ms.assign(L, 0.0);
    if (want_y) res->off.assign(n_rows + 1, 0);
    if (!net->ustream) CK(cudaStreamCreateWithFlags(&net->ustream, cudaStreamNonBlocking));

    std::mutex mu;
    std::condition_variable cv;
    int ready = 0;  // segments whose upload finished (or failed)
    bool stop = false;
    // the caller's OpenMP budget (OMP_NUM_THREADS: bench.py splits the host
    // cores over the local ranks), one core left for the engine thread
    const int threads = std::min(omp_get_max_threads(), host_threads());
    std::thread producer([&] {
        cudaSetDevice(net->device);
        omp_set_num_threads(std::max(1, threads - 1));  // one core runs the engine stream
        for (int s = 0; s < S; ++s) {
            {
                std::lock_guard<std::mutex> g(mu);
                if (stop) break;
            }
            Seg& g = seg[s];
            const int64_t rows = g.r1 - g.r0, c0 = off[g.r0];
            g.off.resize(rows + 1);
            for (int64_t i = 0; i <= rows; ++i) g.off[i] = off[g.r0 + i] - c0;
            g.b = new sdnn_batch;
            g.b->net = net;
            g.rc = upload_csr<T>(net, rows, g.off.data(), cols ? cols + c0 : cols, vals ? vals + c0 : vals, net->n,
                                 g.b, false, net->ustream);
            if (g.rc) g.err = g_err;
            {
                std::lock_guard<std::mutex> lk(mu);
                ready = s + 1;
                if (g.rc) stop = true;
            }
            cv.notify_one();
            if (g.rc) break;
        }
        std::lock_guard<std::mutex> lk(mu);
        stop = true;
        cv.notify_one();
    });
    int rc = SDNN_OK;
    for (int s = 0; s < S && rc == SDNN_OK; ++s) {
        {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return ready > s || stop; });
            if (ready <= s) {  // the producer stopped before this segment
                rc = -1;
                break;
            }
        }
        Seg& g = seg[s];
        if (g.rc) {
            rc = g.rc;
            g_err = g.err;
            break;
        }
        sdnn_result part;
        rc = run_impl<T>(net, g.b, ymax, 0, L, want_y, 1, net->n, net->n, &part);
        if (rc == SDNN_OK && want_y && S > 1) rc = y_to_host(&part);
        if (rc == SDNN_OK && S == 1) {  // one segment: the result is the part (Y may stay on the device)
            const double keep_wall = res->wall_ms;
            std::swap(*res, part);
            res->wall_ms = keep_wall;
            res->segments = 1;
            res->h2d_bytes = g.b->h2d_bytes;
        } else if (rc == SDNN_OK) {
            merge_part(res, part, g.r0, want_y);
            res->h2d_bytes += g.b->h2d_bytes;
        }
    }
    {
        std::lock_guard<std::mutex> lk(mu);
        stop = true;
    }
    producer.join();
    for (auto& g : seg)
        if (g.b) free_batch(g.b);
    if (rc < 0) {  // a segment failed after an earlier one: report its error
        for (auto& g : seg)
            if (g.rc) {
                g_err = g.err;
                return g.rc;
            }
        return fail(SDNN_ERR_CAPACITY, "streamed upload stopped early");
    }
    if (rc == SDNN_OK && want_y && S > 1) res->have_y = true;
    return rc;
}

// Layers [first, end) of the group's first network copied to every other
// member, device to device (a peer copy over NVLink/NVSwitch between GPUs;
// untimed, like the reference's model loading).
int replicate_layers(sdnn_group* g, size_t first) {
    sdnn_net* src = g->nets[0];
    for (size_t i = 1; i < g->nets.size(); ++i) {
        sdnn_net* dst = g->nets[i];
        if (int rc = set_device(dst)) return rc;
        if (dst->device != src->device) {
            int can = 0;
            CK(cudaDeviceCanAccessPeer(&can, dst->device, src->device));
            if (can) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(src->device, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else CK(e);
            }
        }
        for (size_t l = first; l < src->layers.size(); ++l) {
            const DevLayer& S = src->layers[l];
            DevLayer L = S;
            const size_t slots = std::max<size_t>((size_t)S.wp * (size_t)src->n, 1);
            CK(cudaMalloc(&L.idx, slots * sizeof(int32_t)));
            CK(cudaMalloc(&L.val, slots * src->elem));
            CK(cudaMemcpyPeer(L.idx, dst->device, S.idx, src->device, slots * sizeof(int32_t)));
            CK(cudaMemcpyPeer(L.val, dst->device, S.val, src->device, slots * src->elem));
            dst->layers.push_back(L);
        }
    }
    return SDNN_OK;
}

}  // namespace

// ===================================================================== C ABI

extern "C" {

int sdnn_version(void) { return 1; }

const char* sdnn_last_error(void) { return g_err.c_str(); }

int sdnn_device_count(int* n) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        *n = 0;
        return fail(SDNN_ERR_CAPACITY, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    }
    *n = c;
    return SDNN_OK;
}

int sdnn_net_create(int device, int dtype, int64_t n_neurons, sdnn_net** out) {
    if (!out) return fail(SDNN_ERR_PARAMETER, "null output pointer");
    return make_net(device, dtype, n_neurons, out);
}

void sdnn_net_destroy(sdnn_net* net) {
    if (!net) return;
    cudaSetDevice(net->device);
    for (auto& L : net->layers) {
        cudaFree(L.idx);
        cudaFree(L.val);
    }
    cudaFree(net->descs);
    for (int b = 0; b < 2; ++b) {
        cudaFree(net->slab[b]);
        cudaFree(net->meta[b]);
    }
    cudaFree(net->zero);
    cudaFree(net->rowid_buf);
    cudaFree(net->rowid_alt);
    cudaFree(net->alive_c);
    cudaFree(net->n_compact);
    cudaFree(net->probe_flag);
    cudaFree(net->prune_map);
    cudaFree(net->pp_codes);
    cudaFree(net->pp_tmax);
    cudaFree(net->rowlist);
    cudaFree(net->live_rows);
    cudaFree(net->stamps);
    cudaFree(net->heap);
    cudaFree(net->work);
    cudaFree(net->alive);
    cudaFree(net->tile_count);
    cudaFree(net->bar);
    cudaFree(net->n_sel);
    cudaFree(net->cub_tmp);
    if (net->pinned) cudaFreeHost(net->pinned);
    if (net->ing_pinned) cudaFreeHost(net->ing_pinned);
    cudaFree(net->ing_dev);
    for (auto e : net->stage_ev)
        if (e) cudaEventDestroy(e);
    if (net->ev0) cudaEventDestroy(net->ev0);
    if (net->ev1) cudaEventDestroy(net->ev1);
    if (net->ev_d) cudaEventDestroy(net->ev_d);
    if (net->ev_b) cudaEventDestroy(net->ev_b);
    if (net->stream) cudaStreamDestroy(net->stream);
    if (net->ustream) cudaStreamDestroy(net->ustream);
    delete net;
}

int sdnn_net_add_layer_csr(sdnn_net* net, const int64_t* w_off, const int64_t* w_cols,
                           const double* w_vals, int64_t nnz, double bias) {
    if (!net || !w_off) return fail(SDNN_ERR_PARAMETER, "null argument");
    if (int rc = set_device(net)) return rc;
    if (w_off[net->n] != nnz) return fail(SDNN_ERR_PARAMETER, "inconsistent weight offsets");
    return net->dtype == SDNN_F64 ? ingest_csr<double>(net, net->n, net->n, w_off, w_cols, w_vals, bias)
                                  : ingest_csr<float>(net, net->n, net->n, w_off, w_cols, w_vals, bias);
}

int sdnn_net_add_layer_ell(sdnn_net* net, int32_t width, const int32_t* idx, const double* vals,
                           double bias) {
    if (!net || width < 0 || (width > 0 && !idx)) return fail(SDNN_ERR_PARAMETER, "bad ELL layer");
    if (int rc = set_device(net)) return rc;
    for (int64_t j = 0; j < net->n; ++j)
        for (int s = 0; s < width; ++s) {
            const int32_t v = idx[(size_t)j * width + s];
            if (v < 0 || v >= net->n) return fail(SDNN_ERR_PARAMETER, "ELL index out of range");
            if (s > 0 && v <= idx[(size_t)j * width + s - 1])
                return fail(SDNN_ERR_PARAMETER, "ELL column %lld not strictly ascending", (long long)j);
        }
    return upload_layer(net, net->n, width, idx, vals, 0.0, bias, nullptr);
}

int sdnn_net_add_layers_permunion(sdnn_net* net, uint64_t seed, int64_t first_layer, int64_t count,
                                  int32_t width, double value, double bias, int threads) {
    if (!net || count < 0 || width < 0 || width > net->n) return fail(SDNN_ERR_PARAMETER, "bad perm-union request");
    if (int rc = set_device(net)) return rc;
    if (threads < 1) threads = host_threads();
    const int64_t batch = std::max(1, threads);
    std::vector<int32_t> idx((size_t)batch * net->n * width);
    for (int64_t l0 = 0; l0 < count; l0 += batch) {
        const int64_t m = std::min(batch, count - l0);
        int rc = sdnn_gen_permunion_ell_layers(seed, first_layer + l0, m, (int32_t)net->n, width, threads, idx.data());
        if (rc) return fail(rc, "perm-union generation failed");
        for (int64_t l = 0; l < m; ++l)
            if (int rc2 = upload_layer(net, net->n, width, idx.data() + (size_t)l * net->n * width, nullptr, value, bias,
                                       nullptr))
                return rc2;
    }
    return SDNN_OK;
}

int sdnn_net_add_layers_uninit(sdnn_net* net, int64_t count, int32_t width, double bias) {
    if (!net || count < 0 || width < 0) return fail(SDNN_ERR_PARAMETER, "bad layer request");
    if (int rc = set_device(net)) return rc;
    for (int64_t l = 0; l < count; ++l) {
        DevLayer L;
        L.width = width;
        L.wp = (width + 31) / 32 * 32;
        L.bias = bias;
        const size_t slots = (size_t)L.wp * (size_t)net->n;
        CK(cudaMalloc(&L.idx, std::max<size_t>(slots, 1) * sizeof(int32_t)));
        CK(cudaMalloc(&L.val, std::max<size_t>(slots, 1) * net->elem));
        L.bytes = (int64_t)slots * (4 + net->elem);
        net->layers.push_back(L);
    }
    return SDNN_OK;
}

int sdnn_net_layer_buffers(const sdnn_net* net, int64_t layer, void** idx, void** val, int32_t* wp,
                           int64_t* val_bytes) {
    if (!net || !idx || !val || !wp || !val_bytes) return fail(SDNN_ERR_PARAMETER, "null argument");
    if (layer < 0 || layer >= (int64_t)net->layers.size())
        return fail(SDNN_ERR_PARAMETER, "layer %lld outside the %zu-layer network", (long long)layer,
                    net->layers.size());
    const DevLayer& L = net->layers[layer];
    *idx = L.idx;
    *val = L.val;
    *wp = L.wp;
    *val_bytes = (int64_t)L.wp * net->n * net->elem;
    return SDNN_OK;
}

int sdnn_net_n_layers(const sdnn_net* net, int64_t* n) {
    if (!net || !n) return fail(SDNN_ERR_PARAMETER, "null argument");
    *n = (int64_t)net->layers.size();
    return SDNN_OK;
}

int sdnn_net_weight_bytes(const sdnn_net* net, int64_t* bytes) {
    if (!net || !bytes) return fail(SDNN_ERR_PARAMETER, "null argument");
    int64_t s = 0;
    for (auto& L : net->layers) s += L.bytes;
    *bytes = s;
    return SDNN_OK;
}

int sdnn_batch_h2d_bytes(const sdnn_batch* b, int64_t* bytes) {
    if (!b || !bytes) return fail(SDNN_ERR_PARAMETER, "null argument");
    *bytes = b->h2d_bytes;
    return SDNN_OK;
}

int sdnn_batch_upload(sdnn_net* net, int64_t n_rows, const int64_t* y_off, const int64_t* y_cols,
                      const double* y_vals, sdnn_batch** out) {
    if (!net || !out || n_rows < 0 || (n_rows > 0 && !y_off)) return fail(SDNN_ERR_PARAMETER, "bad batch");
    if (n_rows >= (1LL << 31)) return fail(SDNN_ERR_CAPACITY, "batch of %lld rows exceeds int32 row ids", (long long)n_rows);
    if (int rc = set_device(net)) return rc;
    sdnn_batch* b = new sdnn_batch;
    b->net = net;
    static const int64_t zero_off[1] = {0};
    const int64_t* off = n_rows > 0 ? y_off : zero_off;
    int rc = net->dtype == SDNN_F64 ? upload_csr<double>(net, n_rows, off, y_cols, y_vals, net->n, b)
                                    : upload_csr<float>(net, n_rows, off, y_cols, y_vals, net->n, b);
    if (rc) {
        free_batch(b);
        return rc;
    }
    *out = b;
    return SDNN_OK;
}

int sdnn_batch_from_result(sdnn_net* net, const sdnn_result* r, sdnn_batch** out) {
    if (!net || !r || !out) return fail(SDNN_ERR_PARAMETER, "null argument");
    if (!r->have_y) return fail(SDNN_ERR_PARAMETER, "result was produced without Y (use sdnn_run_y)");
    if (r->n_cols != net->n)
        return fail(SDNN_ERR_SHAPE, "result has %lld columns but the network has %lld neurons", (long long)r->n_cols,
                    (long long)net->n);
    if (int rc = set_device(net)) return rc;
    sdnn_batch* b = new sdnn_batch;
    b->net = net;
    int rc = SDNN_OK;
    if (!r->d_off) {  // Y assembled on the host (multi-wave run): upload it
        rc = net->dtype == SDNN_F64
                 ? upload_csr<double>(net, r->n_rows, r->off.data(), r->cols.data(), r->vals.data(), net->n, b, true)
                 : upload_csr<float>(net, r->n_rows, r->off.data(), r->cols.data(), r->vals.data(), net->n, b, true);
        if (rc) {
            free_batch(b);
            return rc;
        }
        *out = b;
        return SDNN_OK;
    }
    cudaStream_t st = net->stream;
    const int64_t n = r->n_rows, nnz = r->d_nnz;
    b->n_rows = n;
    b->nnz = nnz;
    b->n_cols = net->n;
    b->col_bytes = net->n <= 65536 ? 2 : 4;
    const int elem = net->dtype == SDNN_F64 ? 8 : 4;
    const int64_t* src_off = r->d_off;
    const int64_t* src_cols = r->d_cols;
    const double* src_vals = r->d_vals;
    int64_t* tcols = nullptr;
    double* tvals = nullptr;
    int* fin = nullptr;
    auto cleanup = [&]() {
        if (tcols) cudaFreeAsync(tcols, st);
        if (tvals) cudaFreeAsync(tvals, st);
        if (fin) cudaFreeAsync(fin, st);
    };
#define CKB(call)                        \
    do {                                 \
        cudaError_t e_ = (call);         \
        if (e_ != cudaSuccess) {         \
            cleanup();                   \
            free_batch(b);               \
            return fail(SDNN_ERR_CAPACITY, "%s failed: %s", #call, cudaGetErrorString(e_)); \
        }                                \
    } while (0)
    CKB(cudaMallocAsync(reinterpret_cast<void**>(&b->off), (n + 1) * 8, st));
    CKB(cudaMallocAsync(&b->cols, std::max<int64_t>(nnz, 1) * b->col_bytes, st));
    CKB(cudaMallocAsync(&b->vals, std::max<int64_t>(nnz, 1) * elem, st));
    CKB(cudaMallocAsync(reinterpret_cast<void**>(&fin), 4, st));
    if (r->device != net->device) {  // hand-off across GPUs: peer copies (NVLink / NVSwitch)
        CKB(cudaMallocAsync(reinterpret_cast<void**>(&tcols), std::max<int64_t>(nnz, 1) * 8, st));
        CKB(cudaMallocAsync(reinterpret_cast<void**>(&tvals), std::max<int64_t>(nnz, 1) * 8, st));
        CKB(cudaMemcpyPeerAsync(b->off, net->device, src_off, r->device, (n + 1) * 8, st));
        if (nnz) {
            CKB(cudaMemcpyPeerAsync(tcols, net->device, src_cols, r->device, nnz * 8, st));
            CKB(cudaMemcpyPeerAsync(tvals, net->device, src_vals, r->device, nnz * 8, st));
        }
        src_cols = tcols;
        src_vals = tvals;
    } else {
        CKB(cudaMemcpyAsync(b->off, src_off, (n + 1) * 8, cudaMemcpyDeviceToDevice, st));
    }
    CKB(cudaMemsetAsync(fin, 0xff, 4, st));
    if (nnz) {
        const int grid = (int)std::min<int64_t>((nnz + 255) / 256, (int64_t)net->sm_count * 8);
        if (b->col_bytes == 2 && elem == 4)
            narrow_csr_kernel<uint16_t, float><<<grid, 256, 0, st>>>(src_cols, src_vals, nnz, (uint16_t*)b->cols, (float*)b->vals, fin);
        else if (b->col_bytes == 2)
            narrow_csr_kernel<uint16_t, double><<<grid, 256, 0, st>>>(src_cols, src_vals, nnz, (uint16_t*)b->cols, (double*)b->vals, fin);
        else if (elem == 4)
            narrow_csr_kernel<int32_t, float><<<grid, 256, 0, st>>>(src_cols, src_vals, nnz, (int32_t*)b->cols, (float*)b->vals, fin);
        else
            narrow_csr_kernel<int32_t, double><<<grid, 256, 0, st>>>(src_cols, src_vals, nnz, (int32_t*)b->cols, (double*)b->vals, fin);
        CKB(cudaGetLastError());
    }
    int hfin = 1;
    CKB(cudaMemcpyAsync(&hfin, fin, 4, cudaMemcpyDeviceToHost, st));
    CKB(cudaStreamSynchronize(st));
#undef CKB
    b->finite = hfin != 0;
    b->h2d_bytes = 0;
    cleanup();
    CK(cudaStreamSynchronize(st));
    *out = b;
    return SDNN_OK;
}

int sdnn_batch_from_images(sdnn_net* net, int64_t n_images, int32_t side, const uint8_t* pixels,
                           int32_t target_side, sdnn_batch** out) {
    if (!net || !out) return fail(SDNN_ERR_PARAMETER, "null argument");
    if (n_images >= (1LL << 31)) return fail(SDNN_ERR_CAPACITY, "batch of %lld rows exceeds int32 row ids", (long long)n_images);
    if (int rc = set_device(net)) return rc;
    sdnn_batch* b = new sdnn_batch;
    b->net = net;
    if (int rc = images_upload(net, n_images, side, pixels, target_side, b)) {
        free_batch(b);
        return rc;
    }
    *out = b;
    return SDNN_OK;
}

int sdnn_batch_nnz(const sdnn_batch* b, int64_t* nnz) {
    if (!b || !nnz) return fail(SDNN_ERR_PARAMETER, "null argument");
    *nnz = b->nnz;
    return SDNN_OK;
}

int sdnn_batch_csr(const sdnn_batch* b, int64_t* off, int64_t* cols, double* vals) {
    if (!b || !off) return fail(SDNN_ERR_PARAMETER, "null argument");
    if (int rc = set_device(b->net)) return rc;
    cudaStream_t st = b->net->stream;
    CK(cudaMemcpyAsync(off, b->off, (b->n_rows + 1) * 8, cudaMemcpyDeviceToHost, st));
    std::vector<char> c((size_t)std::max<int64_t>(b->nnz, 1) * b->col_bytes);
    std::vector<char> v;
    if (b->nnz) CK(cudaMemcpyAsync(c.data(), b->cols, b->nnz * b->col_bytes, cudaMemcpyDeviceToHost, st));
    const int elem = b->net->dtype == SDNN_F64 ? 8 : 4;
    if (b->vals && b->nnz) {
        v.resize((size_t)b->nnz * elem);
        CK(cudaMemcpyAsync(v.data(), b->vals, b->nnz * elem, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < b->nnz; ++i) {
        if (cols)
            cols[i] = b->col_bytes == 2 ? (int64_t)reinterpret_cast<const uint16_t*>(c.data())[i]
                                        : (int64_t)reinterpret_cast<const int32_t*>(c.data())[i];
        if (vals)
            vals[i] = !b->vals ? 1.0
                      : elem == 8 ? reinterpret_cast<const double*>(v.data())[i]
                                  : (double)reinterpret_cast<const float*>(v.data())[i];
    }
    return SDNN_OK;
}

void sdnn_batch_free(sdnn_batch* b) {
    if (b && b->net) cudaSetDevice(b->net->device);
    free_batch(b);
}

static int run_checked(sdnn_net* net, const sdnn_batch* batch, double ymax, int64_t first, int64_t nl,
                       int want_y, sdnn_result** out) {
    if (!net || !batch || !out) return fail(SDNN_ERR_PARAMETER, "null argument");
    if (!(ymax > 0)) return fail(SDNN_ERR_PARAMETER, "ymax must be positive, got %g", ymax);
    const int64_t L = (int64_t)net->layers.size();
    if (nl < 0) nl = L - first;
    if (first < 0 || nl < 1 || first + nl > L)
        return fail(SDNN_ERR_PARAMETER, "layer range [%lld, %lld) outside the %lld-layer network",
                    (long long)first, (long long)(first + nl), (long long)L);
    if (int rc = set_device(net)) return rc;
    sdnn_result* res = new sdnn_result;
    const double t0 = now_ms();
    int rc = net->dtype == SDNN_F64 ? run_impl<double>(net, batch, ymax, first, nl, want_y, 1, net->n, net->n, res)
                                    : run_impl<float>(net, batch, ymax, first, nl, want_y, 1, net->n, net->n, res);
    if (rc) {
        delete res;
        return rc;
    }
    res->wall_ms = now_ms() - t0;
    *out = res;
    return SDNN_OK;
}

int sdnn_run(sdnn_net* net, const sdnn_batch* batch, double ymax, int64_t first_layer, int64_t n_layers,
             sdnn_result** out) {
    return run_checked(net, batch, ymax, first_layer, n_layers, 0, out);
}

int sdnn_run_y(sdnn_net* net, const sdnn_batch* batch, double ymax, int64_t first_layer, int64_t n_layers,
               sdnn_result** out) {
    return run_checked(net, batch, ymax, first_layer, n_layers, 1, out);
}

int sdnn_infer_streamed(sdnn_net* net, int64_t n_rows, const int64_t* y_off, const int64_t* y_cols,
                        const double* y_vals, double ymax, int want_y, int segments, sdnn_result** out) {
    if (!net || !out || n_rows < 0 || (n_rows > 0 && !y_off)) return fail(SDNN_ERR_PARAMETER, "bad batch");
    if (n_rows >= (1LL << 31)) return fail(SDNN_ERR_CAPACITY, "batch of %lld rows exceeds int32 row ids", (long long)n_rows);
    if (!(ymax > 0)) return fail(SDNN_ERR_PARAMETER, "ymax must be positive, got %g", ymax);
    if (int rc = set_device(net)) return rc;
    static const int64_t zero_off[1] = {0};
    const int64_t* off = n_rows > 0 ? y_off : zero_off;
    const double t0 = now_ms();
    sdnn_result* res = new sdnn_result;
    int rc = net->dtype == SDNN_F64
                 ? infer_streamed<double>(net, n_rows, off, y_cols, y_vals, ymax, want_y, segments, res)
                 : infer_streamed<float>(net, n_rows, off, y_cols, y_vals, ymax, want_y, segments, res);
    if (rc) {
        delete res;
        return rc;
    }
    res->wall_ms = now_ms() - t0;
    *out = res;
    return SDNN_OK;
}

int sdnn_infer(sdnn_net* net, int64_t n_rows, const int64_t* y_off, const int64_t* y_cols,
               const double* y_vals, double ymax, sdnn_result** out) {
    return sdnn_infer_streamed(net, n_rows, y_off, y_cols, y_vals, ymax, 1, 0, out);
}

int sdnn_result_h2d_bytes(const sdnn_result* r, int64_t* bytes) {
    if (!r || !bytes) return fail(SDNN_ERR_PARAMETER, "null argument");
    *bytes = r->h2d_bytes;
    return SDNN_OK;
}

int sdnn_result_segments(const sdnn_result* r, int64_t* n) {
    if (!r || !n) return fail(SDNN_ERR_PARAMETER, "null argument");
    *n = r->segments;
    return SDNN_OK;
}

int sdnn_result_n_categories(const sdnn_result* r, int64_t* n) {
    if (!r || !n) return fail(SDNN_ERR_PARAMETER, "null argument");
    *n = (int64_t)r->cats.size();
    return SDNN_OK;
}

int sdnn_result_categories(const sdnn_result* r, int64_t* buf) {
    if (!r || (!buf && !r->cats.empty())) return fail(SDNN_ERR_PARAMETER, "null argument");
    if (!r->cats.empty()) memcpy(buf, r->cats.data(), r->cats.size() * sizeof(int64_t));
    return SDNN_OK;
}

double sdnn_result_device_ms(const sdnn_result* r) { return r ? r->dev_ms : -1.0; }
double sdnn_result_wall_ms(const sdnn_result* r) { return r ? r->wall_ms : -1.0; }

int sdnn_result_n_layers(const sdnn_result* r, int64_t* n) {
    if (!r || !n) return fail(SDNN_ERR_PARAMETER, "null argument");
    *n = r->n_layers;
    return SDNN_OK;
}

int sdnn_result_live_rows(const sdnn_result* r, int64_t* live) {
    if (!r || !live) return fail(SDNN_ERR_PARAMETER, "null argument");
    for (size_t i = 0; i < r->live.size(); ++i) live[i] = r->live[i];
    return SDNN_OK;
}

int sdnn_net_set_layer_timing(sdnn_net* net, int on) {
    if (!net) return fail(SDNN_ERR_PARAMETER, "null argument");
    net->layer_timing = on;
    return SDNN_OK;
}

int sdnn_net_set_compaction(sdnn_net* net, int pct) {
    if (!net) return fail(SDNN_ERR_PARAMETER, "null argument");
    net->compact_pct = pct;
    return SDNN_OK;
}

int sdnn_result_compactions(const sdnn_result* r, int64_t* n) {
    if (!r || !n) return fail(SDNN_ERR_PARAMETER, "null argument");
    *n = r->compactions;
    return SDNN_OK;
}

int sdnn_net_set_pruning(sdnn_net* net, int on) {
    if (!net) return fail(SDNN_ERR_PARAMETER, "null argument");
    net->prune = on ? 1 : 0;
    return SDNN_OK;
}

int sdnn_result_pruned(const sdnn_result* r, int64_t* n) {
    if (!r || !n) return fail(SDNN_ERR_PARAMETER, "null argument");
    *n = r->pruned;
    return SDNN_OK;
}

int sdnn_result_stage_ms(const sdnn_result* r, double* ms) {
    if (!r || !ms) return fail(SDNN_ERR_PARAMETER, "null argument");
    for (int i = 0; i < 3; ++i) ms[i] = r->stage_ms[i];
    return SDNN_OK;
}

int sdnn_result_layer_ms(const sdnn_result* r, double* ms) {
    if (!r || !ms) return fail(SDNN_ERR_PARAMETER, "null argument");
    if (r->layer_ms.empty()) return fail(SDNN_ERR_PARAMETER, "layer timing was off for this run");
    for (size_t i = 0; i < r->layer_ms.size(); ++i) ms[i] = r->layer_ms[i];
    return SDNN_OK;
}

int sdnn_result_launches(const sdnn_result* r, int64_t* n) {
    if (!r || !n) return fail(SDNN_ERR_PARAMETER, "null argument");
    *n = r->launches;
    return SDNN_OK;
}

int sdnn_result_y_nnz(sdnn_result* r, int64_t* nnz) {
    if (!r || !nnz) return fail(SDNN_ERR_PARAMETER, "null argument");
    if (!r->have_y) return fail(SDNN_ERR_PARAMETER, "result was produced without Y (use sdnn_run_y / sdnn_infer)");
    *nnz = r->d_off ? r->d_nnz : (r->off.empty() ? 0 : r->off.back());
    return SDNN_OK;
}

int sdnn_result_y_csr(sdnn_result* r, int64_t* off, int64_t* cols, double* vals) {
    if (!r || !off) return fail(SDNN_ERR_PARAMETER, "null argument");
    if (!r->have_y) return fail(SDNN_ERR_PARAMETER, "result was produced without Y");
    if (r->d_off) {  // device-held Y: straight into the caller's buffers
        CK(cudaSetDevice(r->device));
        if (int rc = d2h_large(off, r->d_off, (r->n_rows + 1) * 8)) return rc;
        if (r->d_nnz && cols)
            if (int rc = d2h_large(cols, r->d_cols, r->d_nnz * 8)) return rc;
        if (r->d_nnz && vals)
            if (int rc = d2h_large(vals, r->d_vals, r->d_nnz * 8)) return rc;
        return SDNN_OK;
    }
    memcpy(off, r->off.data(), r->off.size() * sizeof(int64_t));
    const size_t nnz = r->cols.size();
    for (size_t i = 0; i < nnz; ++i) cols[i] = r->cols[i];
    if (nnz) memcpy(vals, r->vals.data(), nnz * sizeof(double));
    return SDNN_OK;
}

void sdnn_result_free(sdnn_result* r) { delete r; }

int sdnn_open_devices(const int* devices, int n_devices, int dtype, int64_t n_neurons, sdnn_group** out) {
    if (!out || !devices || n_devices < 1) return fail(SDNN_ERR_PARAMETER, "bad device list");
    sdnn_group* g = new sdnn_group;
    for (int i = 0; i < n_devices; ++i) {
        sdnn_net* net = nullptr;
        if (int rc = make_net(devices[i], dtype, n_neurons, &net)) {
            sdnn_close(g);
            return rc;
        }
        g->nets.push_back(net);
    }
    *out = g;
    return SDNN_OK;
}

int sdnn_open(int n_gpus, int dtype, int64_t n_neurons, sdnn_group** out) {
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    if (n_gpus <= 0) n_gpus = count;
    if (n_gpus > count) return fail(SDNN_ERR_PARAMETER, "%d GPUs requested, %d visible", n_gpus, count);
    std::vector<int> devs(std::max(n_gpus, 1));
    for (int i = 0; i < n_gpus; ++i) devs[i] = i;
    return sdnn_open_devices(devs.data(), n_gpus, dtype, n_neurons, out);
}

void sdnn_close(sdnn_group* g) {
    if (!g) return;
    for (auto* net : g->nets) sdnn_net_destroy(net);
    delete g;
}

int sdnn_group_size(const sdnn_group* g, int* n) {
    if (!g || !n) return fail(SDNN_ERR_PARAMETER, "null argument");
    *n = (int)g->nets.size();
    return SDNN_OK;
}

sdnn_net* sdnn_group_net(sdnn_group* g, int i) {
    if (!g || i < 0 || i >= (int)g->nets.size()) return nullptr;
    return g->nets[i];
}

int sdnn_group_add_layer_csr(sdnn_group* g, const int64_t* w_off, const int64_t* w_cols, const double* w_vals,
                             int64_t nnz, double bias) {
    if (!g) return fail(SDNN_ERR_PARAMETER, "null argument");
    const size_t first = g->nets[0]->layers.size();
    if (int rc = sdnn_net_add_layer_csr(g->nets[0], w_off, w_cols, w_vals, nnz, bias)) return rc;
    return replicate_layers(g, first);
}

int sdnn_group_add_layers_permunion(sdnn_group* g, uint64_t seed, int64_t first_layer, int64_t count,
                                    int32_t width, double value, double bias, int threads) {
    if (!g) return fail(SDNN_ERR_PARAMETER, "null argument");
    const size_t first = g->nets[0]->layers.size();
    if (int rc = sdnn_net_add_layers_permunion(g->nets[0], seed, first_layer, count, width, value, bias, threads))
        return rc;
    return replicate_layers(g, first);
}

int sdnn_group_infer(sdnn_group* g, int64_t n_rows, const int64_t* y_off, const int64_t* y_cols,
                     const double* y_vals, double ymax, int want_y, sdnn_result** out) {
    if (!g || !out || n_rows < 0 || (n_rows > 0 && !y_off)) return fail(SDNN_ERR_PARAMETER, "bad batch");
    if (n_rows > 0 && y_off[0] != 0) return fail(SDNN_ERR_PARAMETER, "row_offsets[0] must be 0");
    const int G = (int)g->nets.size();
    const int64_t L = (int64_t)g->nets[0]->layers.size();
    for (auto* net : g->nets)
        if ((int64_t)net->layers.size() != L) return fail(SDNN_ERR_PARAMETER, "group members hold different layers");
    const double t0 = now_ms();
    const int64_t per = std::max<int64_t>(1, (n_rows + G - 1) / G);  // engine.py:240 tile
    struct Block {
        int64_t r0 = 0, r1 = 0;
        std::vector<int64_t> off;
        sdnn_result* res = nullptr;
        int rc = 0;
        std::string err;
    };
    std::vector<Block> blk(G);
    const int hw = host_threads();
    std::vector<std::thread> workers;
    for (int i = 0; i < G; ++i) {
        Block& b = blk[i];
        b.r0 = std::min<int64_t>(n_rows, i * per);
        b.r1 = std::min<int64_t>(n_rows, b.r0 + per);
        workers.emplace_back([&, i] {
            Block& b = blk[i];
            omp_set_num_threads(std::max(2, hw / G));  // the host cores shared by the blocks' producers
            const int64_t rows = b.r1 - b.r0, c0 = rows > 0 ? y_off[b.r0] : 0;
            b.off.resize(rows + 1);
            for (int64_t r = 0; r <= rows; ++r) b.off[r] = (rows > 0 ? y_off[b.r0 + r] : 0) - c0;
            b.rc = sdnn_infer_streamed(g->nets[i], rows, b.off.data(), y_cols ? y_cols + c0 : y_cols,
                                       y_vals ? y_vals + c0 : y_vals, ymax, want_y, 0, &b.res);
            if (b.rc == SDNN_OK && want_y) b.rc = y_to_host(b.res);
            if (b.rc) b.err = g_err;
        });
    }
    for (auto& t : workers) t.join();
    int rc = SDNN_OK;
    for (auto& b : blk)
        if (b.rc && rc == SDNN_OK) {
            rc = b.rc;
            g_err = b.err;
        }
    sdnn_result* res = nullptr;
    if (rc == SDNN_OK) {
        res = new sdnn_result;
        res->n_rows = n_rows;
        res->n_cols = g->nets[0]->n;
        res->n_layers = L;
        res->live.assign(L + 1, 0);
        if (want_y) {
            res->off.assign(n_rows + 1, 0);
            res->have_y = true;
        }
        for (auto& b : blk) {  // row order; the devices ran concurrently: device time is the slowest's
            const sdnn_result& p = *b.res;
            for (int64_t c : p.cats) res->cats.push_back(c + b.r0);
            for (size_t l = 0; l < p.live.size() && l < res->live.size(); ++l) res->live[l] += p.live[l];
            res->dev_ms = std::max(res->dev_ms, p.dev_ms);
            for (int k = 0; k < 3; ++k) res->stage_ms[k] = std::max(res->stage_ms[k], p.stage_ms[k]);
            res->launches += p.launches;
            res->compactions += p.compactions;
            res->pruned += p.pruned;
            res->h2d_bytes += p.h2d_bytes;
            res->segments += p.segments;
            if (want_y) {
                const int64_t base = res->off[b.r0];
                for (int64_t r = 1; r <= b.r1 - b.r0; ++r) res->off[b.r0 + r] = base + p.off[r];
                res->cols.insert(res->cols.end(), p.cols.begin(), p.cols.end());
                res->vals.insert(res->vals.end(), p.vals.begin(), p.vals.end());
            }
        }
        res->wall_ms = now_ms() - t0;
    }
    for (auto& b : blk) delete b.res;
    if (rc) return rc;
    *out = res;
    return SDNN_OK;
}

int sdnn_spmm(int device, int dtype, int64_t n_rows, int64_t n_inner, int64_t n_out, const int64_t* y_off,
              const int64_t* y_cols, const double* y_vals, const int64_t* w_off, const int64_t* w_cols,
              const double* w_vals, sdnn_result** out) {
    if (!out || n_rows < 0 || n_inner < 1 || n_out < 1) return fail(SDNN_ERR_PARAMETER, "bad spmm shape");
    // one rectangular layer run raw (no epilogue) through the same kernel
    sdnn_net* net = nullptr;
    if (int rc = make_net(device, dtype, std::max(n_inner, n_out), &net)) return rc;
    int rc = SDNN_OK;
    sdnn_batch* b = nullptr;
    sdnn_result* res = nullptr;
    do {
        rc = dtype == SDNN_F64 ? ingest_csr<double>(net, n_inner, n_out, w_off, w_cols, w_vals, 0.0)
                               : ingest_csr<float>(net, n_inner, n_out, w_off, w_cols, w_vals, 0.0);
        if (rc) break;
        b = new sdnn_batch;
        b->net = net;
        static const int64_t zero_off[1] = {0};
        const int64_t* yo = n_rows > 0 ? y_off : zero_off;
        rc = dtype == SDNN_F64 ? upload_csr<double>(net, n_rows, yo, y_cols, y_vals, n_inner, b)
                               : upload_csr<float>(net, n_rows, yo, y_cols, y_vals, n_inner, b);
        if (rc) break;
        res = new sdnn_result;
        rc = dtype == SDNN_F64 ? run_impl<double>(net, b, 32.0, 0, 1, 1, 0, n_inner, n_out, res)
                               : run_impl<float>(net, b, 32.0, 0, 1, 1, 0, n_inner, n_out, res);
    } while (0);
    if (b) free_batch(b);
    sdnn_net_destroy(net);
    if (rc) {
        delete res;
        return rc;
    }
    *out = res;
    return SDNN_OK;
}

int sdnn_bias_relu_clamp(int device, int dtype, int64_t n_rows, int64_t n_cols, const int64_t* off,
                         const int64_t* cols, const double* vals, double bias, double ymax, sdnn_result** out) {
    if (!out || n_rows < 0 || n_cols < 1) return fail(SDNN_ERR_PARAMETER, "bad shape");
    sdnn_net* net = nullptr;
    if (int rc = make_net(device, dtype, n_cols, &net)) return rc;
    sdnn_batch* b = new sdnn_batch;
    b->net = net;
    static const int64_t zero_off[1] = {0};
    const int64_t* yo = n_rows > 0 ? off : zero_off;
    // raw upload: int32 columns and every value, as the CSR kernels need
    int rc = dtype == SDNN_F64 ? upload_csr<double>(net, n_rows, yo, cols, vals, n_cols, b, true)
                               : upload_csr<float>(net, n_rows, yo, cols, vals, n_cols, b, true);
    sdnn_result* res = nullptr;
    if (!rc) {
        res = new sdnn_result;
        res->n_rows = n_rows;
        res->n_cols = n_cols;
        auto body = [&](auto tag) -> int {
            using T = decltype(tag);
            if (n_rows == 0) {
                res->off.assign(1, 0);
                res->have_y = true;
                return SDNN_OK;
            }
            int32_t* counts = nullptr;
            int64_t* pos = nullptr;
            int32_t* oc = nullptr;
            T* ov = nullptr;
            CK(cudaMalloc(&counts, n_rows * 4));
            const int grid = (int)std::min<int64_t>(n_rows, (int64_t)net->sm_count * 8);
            csr_brc_count_kernel<T><<<grid, 256, 0, net->stream>>>(b->off, reinterpret_cast<const T*>(b->vals),
                                                                   n_rows, (T)bias, (T)ymax, counts);
            CK(cudaGetLastError());
            std::vector<int32_t> cnt(n_rows);
            CK(cudaMemcpyAsync(cnt.data(), counts, n_rows * 4, cudaMemcpyDeviceToHost, net->stream));
            CK(cudaStreamSynchronize(net->stream));
            res->off.assign(n_rows + 1, 0);
            for (int64_t i = 0; i < n_rows; ++i) res->off[i + 1] = res->off[i] + cnt[i];
            const int64_t total = res->off[n_rows];
            CK(cudaMalloc(&pos, n_rows * 8));
            CK(cudaMemcpyAsync(pos, res->off.data(), n_rows * 8, cudaMemcpyHostToDevice, net->stream));
            CK(cudaMalloc(&oc, std::max<int64_t>(total, 1) * 4));
            CK(cudaMalloc(&ov, std::max<int64_t>(total, 1) * sizeof(T)));
            csr_brc_write_kernel<T><<<grid, 256, 0, net->stream>>>(b->off, reinterpret_cast<const int32_t*>(b->cols),
                                                                   reinterpret_cast<const T*>(b->vals),
                                                                   n_rows, (T)bias, (T)ymax, pos, oc, ov);
            CK(cudaGetLastError());
            std::vector<int32_t> hc(total);
            std::vector<T> hv(total);
            CK(cudaMemcpyAsync(hc.data(), oc, total * 4, cudaMemcpyDeviceToHost, net->stream));
            CK(cudaMemcpyAsync(hv.data(), ov, total * sizeof(T), cudaMemcpyDeviceToHost, net->stream));
            CK(cudaStreamSynchronize(net->stream));
            res->cols.assign(hc.begin(), hc.end());
            res->vals.assign(hv.begin(), hv.end());
            for (int64_t i = 0; i < n_rows; ++i)
                if (cnt[i] > 0) res->cats.push_back(i + 1);
            res->have_y = true;
            cudaFree(counts);
            cudaFree(pos);
            cudaFree(oc);
            cudaFree(ov);
            return SDNN_OK;
        };
        rc = dtype == SDNN_F64 ? body(double{}) : body(float{});
    }
    if (b) free_batch(b);
    sdnn_net_destroy(net);
    if (rc) {
        delete res;
        return rc;
    }
    *out = res;
    return SDNN_OK;
}

}  // extern "C"
