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
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sdnn.h"
#include "sdnn_kernels.cuh"

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
    int width = 0;
    int32_t* idx = nullptr;  // [width][n]
    void* val = nullptr;     // [width][n] of T
    uint16_t* bnd = nullptr; // [(n_chunks+1)][n] when chunked
    double bias = 0;
    int64_t bytes = 0;
};

}  // namespace

struct sdnn_net {
    int device = 0;
    int dtype = SDNN_F32;
    int64_t n = 0;
    int elem = 4;
    // launch geometry of the layer kernel for this (n, dtype)
    int R = 1, n_chunks = 1, chunk_len = 0, threads = 256, blocks = 0;
    size_t smem = 0;
    int sm_count = 0;
    std::vector<DevLayer> layers;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // run scratch, grown on demand
    void* ybuf[2] = {nullptr, nullptr};
    int64_t ycap = 0;  // rows per buffer
    int32_t* rows[2] = {nullptr, nullptr};
    int64_t rcap = 0;
    int32_t* counts = nullptr;
    int64_t ccap = 0;
    void* pinned = nullptr;
    size_t pinned_cap = 0;
    // optional per-layer events (profiling pass, off in timed runs)
    int layer_timing = 0;
    std::vector<cudaEvent_t> lev;
};

struct sdnn_batch {
    sdnn_net* net = nullptr;
    int64_t n_rows = 0, nnz = 0;
    int64_t* off = nullptr;
    int32_t* cols = nullptr;
    void* vals = nullptr;
};

struct sdnn_result {
    int64_t n_rows = 0, n_cols = 0;
    int64_t n_layers = 0;
    std::vector<int64_t> cats;  // 1-based ascending
    std::vector<int64_t> live;  // [n_layers + 1]
    double dev_ms = 0, wall_ms = 0;
    int64_t launches = 0;
    std::vector<double> layer_ms;  // per layer, when layer timing is on
    bool have_y = false;
    std::vector<int64_t> off, cols;
    std::vector<double> vals;
};

namespace {

int set_device(const sdnn_net* net) {
    CK(cudaSetDevice(net->device));
    return SDNN_OK;
}

template <typename T>
const void* layer_fn(int R) {
    switch (R) {
        case 1: return (const void*)layer_kernel<T, 1>;
        case 2: return (const void*)layer_kernel<T, 2>;
        case 4: return (const void*)layer_kernel<T, 4>;
        default: return (const void*)layer_kernel<T, 8>;
    }
}

const void* layer_fn_for(const sdnn_net* net) {
    return net->dtype == SDNN_F64 ? layer_fn<double>(net->R) : layer_fn<float>(net->R);
}

// Pick rows-per-group R and the input chunking for (n, dtype): rows of up
// to `budget` bytes stay whole in shared memory, R of them per CTA; longer
// rows are split into equal chunks of whole 32-element multiples.
int configure(sdnn_net* net) {
    const int64_t budget = env_int("SDNN_SMEM_BUDGET", 96 * 1024);
    const int64_t row_bytes = net->n * net->elem;
    int R = env_int("SDNN_R", 0);
    if (row_bytes <= budget) {
        net->n_chunks = 1;
        net->chunk_len = (int)net->n;
        if (R <= 0) {
            int64_t fit = budget / std::max<int64_t>(row_bytes, 1);
            R = fit >= 8 ? 8 : fit >= 4 ? 4 : fit >= 2 ? 2 : 1;
        }
    } else {
        int64_t c = (row_bytes + budget - 1) / budget;
        int64_t len = (net->n + c - 1) / c;
        len = (len + 31) / 32 * 32;
        net->chunk_len = (int)len;
        net->n_chunks = (int)((net->n + len - 1) / len);
        if (R <= 0) R = 1;
    }
    if (R != 1 && R != 2 && R != 4 && R != 8) R = 1;
    net->R = R;
    net->threads = env_int("SDNN_THREADS", 256);
    net->smem = (size_t)R * net->chunk_len * net->elem;
    const void* fn = layer_fn_for(net);
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)net->smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, net->threads, net->smem));
    if (occ < 1) return fail(SDNN_ERR_CAPACITY, "layer kernel does not fit an SM (smem %zu)", net->smem);
    net->blocks = net->sm_count * occ;
    return SDNN_OK;
}

template <typename T>
void to_T(const double* src, T* dst, int64_t n) {
    for (int64_t i = 0; i < n; ++i) dst[i] = (T)src[i];
}

// Upload one ELL-by-output layer given output-major host arrays.  deg[j]
// (nullable: every column has `width` real slots) counts column j's real
// inputs; slots past it are padding.
int upload_layer(sdnn_net* net, int width, const int32_t* idx_om, const double* val_om,
                 double value_if_null, double bias, const int64_t* deg) {
    const int64_t n = net->n;
    DevLayer L;
    L.width = width;
    L.bias = bias;
    if (width > 65535) return fail(SDNN_ERR_CAPACITY, "column degree %d exceeds 65535", width);
    const size_t slots = (size_t)width * (size_t)n;
    std::vector<int32_t> idx_sm(std::max<size_t>(slots, 1));
    std::vector<unsigned char> val_sm(std::max<size_t>(slots, 1) * net->elem);
    // transpose output-major -> slot-major
    parallel_for(n, [&](int64_t j0, int64_t j1) {
        for (int64_t j = j0; j < j1; ++j) {
            for (int s = 0; s < width; ++s) {
                const size_t om = (size_t)j * width + s, sm = (size_t)s * n + j;
                idx_sm[sm] = idx_om[om];
                const double v = val_om ? val_om[om] : value_if_null;
                if (net->dtype == SDNN_F64)
                    reinterpret_cast<double*>(val_sm.data())[sm] = v;
                else
                    reinterpret_cast<float*>(val_sm.data())[sm] = (float)v;
            }
        }
    });
    bool uniform = true;
    if (deg)
        for (int64_t j = 0; j < n && uniform; ++j) uniform = deg[j] == width;
    std::vector<uint16_t> bnd;
    if (net->n_chunks > 1 || !uniform) {
        const int C = net->n_chunks;
        bnd.assign((size_t)(C + 1) * n, 0);
        parallel_for(n, [&](int64_t j0, int64_t j1) {
            for (int64_t j = j0; j < j1; ++j) {
                const int32_t* row = idx_om + (size_t)j * width;
                const int d = deg ? (int)deg[j] : width;
                int s = 0;
                for (int c = 0; c <= C; ++c) {
                    const int64_t lim = (int64_t)c * net->chunk_len;
                    while (s < d && row[s] < lim) ++s;
                    bnd[(size_t)c * n + j] = (uint16_t)(c == C ? d : s);
                }
            }
        });
    }
    CK(cudaMalloc(&L.idx, std::max<size_t>(slots, 1) * sizeof(int32_t)));
    CK(cudaMalloc(&L.val, std::max<size_t>(slots, 1) * net->elem));
    CK(cudaMemcpy(L.idx, idx_sm.data(), slots * sizeof(int32_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(L.val, val_sm.data(), slots * net->elem, cudaMemcpyHostToDevice));
    L.bytes = (int64_t)slots * (4 + net->elem);
    if (!bnd.empty()) {
        CK(cudaMalloc(&L.bnd, bnd.size() * sizeof(uint16_t)));
        CK(cudaMemcpy(L.bnd, bnd.data(), bnd.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
        L.bytes += (int64_t)bnd.size() * 2;
    }
    net->layers.push_back(L);
    return SDNN_OK;
}

int ensure_scratch(sdnn_net* net, int64_t rows, int64_t n_layers) {
    if (rows > net->ycap) {
        for (auto& b : net->ybuf) {
            if (b) CK(cudaFree(b));
            b = nullptr;
        }
        for (auto& b : net->ybuf) CK(cudaMalloc(&b, std::max<int64_t>(rows, 1) * net->n * net->elem));
        net->ycap = rows;
    }
    if (rows > net->rcap) {
        for (auto& b : net->rows) {
            if (b) CK(cudaFree(b));
            b = nullptr;
        }
        for (auto& b : net->rows) CK(cudaMalloc(&b, std::max<int64_t>(rows, 1) * sizeof(int32_t)));
        net->rcap = rows;
    }
    if (n_layers + 1 > net->ccap) {
        if (net->counts) CK(cudaFree(net->counts));
        CK(cudaMalloc(&net->counts, (n_layers + 1) * sizeof(int32_t)));
        net->ccap = n_layers + 1;
    }
    return SDNN_OK;
}

// Rows per wave so two activation buffers fit next to everything else.
int64_t wave_rows(sdnn_net* net, int64_t n_rows) {
    int64_t forced = env_int("SDNN_WAVE_ROWS", 0);
    if (forced > 0) return std::min(forced, std::max<int64_t>(n_rows, 1));
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    // buffers we already hold can be reused
    int64_t held = net->ycap * net->n * net->elem * 2 + net->rcap * 8;
    int64_t avail = (int64_t)free_b + held - (int64_t)(1ull << 30);
    int64_t per_row = net->n * net->elem * 2 + 8;
    int64_t w = std::max<int64_t>(1, avail / per_row);
    return std::min(w, std::max<int64_t>(n_rows, 1));
}

template <typename T>
LayerArgs<T> make_args(sdnn_net* net, const DevLayer& L, double ymax) {
    LayerArgs<T> a{};
    a.n_in = (int)net->n;
    a.n_out = (int)net->n;
    a.ld = (int)net->n;
    a.width = L.width;
    a.idx = L.idx;
    a.val = reinterpret_cast<const T*>(L.val);
    a.bnd = L.bnd;
    a.n_chunks = net->n_chunks;
    a.chunk_len = net->chunk_len;
    a.bias = (T)L.bias;
    a.ymax = (T)ymax;
    a.epilogue = 1;
    return a;
}

template <typename T>
int launch_layer(sdnn_net* net, const LayerArgs<T>& a) {
    const void* fn = layer_fn<T>(net->R);
    void* args[] = {(void*)&a};
    CK(cudaLaunchKernel(fn, dim3(net->blocks), dim3(net->threads), args, net->smem, net->stream));
    return SDNN_OK;
}

// Dense rows of a live list -> host CSR pieces (ascending row id).
template <typename T>
int gather_rows(sdnn_net* net, const T* y, int64_t row_base, int n_cols, const int32_t* rows_dev,
                int64_t n_list, std::vector<int32_t>& rows_host, std::vector<int64_t>& row_nnz,
                std::vector<int32_t>& cols_h, std::vector<T>& vals_h) {
    rows_host.resize(n_list);
    row_nnz.assign(n_list, 0);
    cols_h.clear();
    vals_h.clear();
    if (n_list == 0) return SDNN_OK;
    int32_t* counts = nullptr;
    int64_t* pos = nullptr;
    int32_t* cols = nullptr;
    T* vals = nullptr;
    CK(cudaMemcpyAsync(rows_host.data(), rows_dev, n_list * 4, cudaMemcpyDeviceToHost, net->stream));
    CK(cudaMalloc(&counts, n_list * 4));
    const int grid = (int)std::min<int64_t>(n_list, (int64_t)net->sm_count * 8);
    dense_count_kernel<T><<<grid, 256, 0, net->stream>>>(y, row_base, n_cols, rows_dev, (int)n_list, counts);
    CK(cudaGetLastError());
    std::vector<int32_t> cnt(n_list);
    CK(cudaMemcpyAsync(cnt.data(), counts, n_list * 4, cudaMemcpyDeviceToHost, net->stream));
    CK(cudaStreamSynchronize(net->stream));
    std::vector<int64_t> p(n_list);
    int64_t total = 0;
    for (int64_t i = 0; i < n_list; ++i) {
        p[i] = total;
        total += cnt[i];
        row_nnz[i] = cnt[i];
    }
    CK(cudaMalloc(&pos, n_list * 8));
    CK(cudaMemcpyAsync(pos, p.data(), n_list * 8, cudaMemcpyHostToDevice, net->stream));
    CK(cudaMalloc(&cols, std::max<int64_t>(total, 1) * 4));
    CK(cudaMalloc(&vals, std::max<int64_t>(total, 1) * sizeof(T)));
    dense_write_kernel<T><<<grid, 256, 0, net->stream>>>(y, row_base, n_cols, rows_dev, (int)n_list, pos, cols, vals);
    CK(cudaGetLastError());
    cols_h.resize(total);
    vals_h.resize(total);
    CK(cudaMemcpyAsync(cols_h.data(), cols, total * 4, cudaMemcpyDeviceToHost, net->stream));
    CK(cudaMemcpyAsync(vals_h.data(), vals, total * sizeof(T), cudaMemcpyDeviceToHost, net->stream));
    CK(cudaStreamSynchronize(net->stream));
    cudaFree(counts);
    cudaFree(pos);
    cudaFree(cols);
    cudaFree(vals);
    return SDNN_OK;
}

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
    // locate each row's segment inside its piece
    std::vector<std::pair<int32_t, int64_t>> src(B, {-1, 0});
    for (size_t w = 0; w < pieces.size(); ++w) {
        int64_t at = 0;
        for (size_t i = 0; i < pieces[w].rows.size(); ++i) {
            const int32_t r = pieces[w].rows[i];
            cnt[r + 1] = pieces[w].nnz[i];
            src[r] = {(int32_t)w, at};
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

template <typename T>
int run_impl(sdnn_net* net, const sdnn_batch* batch, double ymax, int64_t first, int64_t nl,
             int want_y, sdnn_result* res) {
    const int64_t B = batch->n_rows;
    const int64_t wave = wave_rows(net, B);
    if (int rc = ensure_scratch(net, std::min(wave, std::max<int64_t>(B, 1)), nl)) return rc;
    res->n_rows = B;
    res->n_cols = net->n;
    res->n_layers = nl;
    res->live.assign(nl + 1, 0);
    std::vector<Piece> pieces;
    std::vector<int32_t> final_rows;
    float total_ms = 0;
    int64_t launches = 0;
    const bool timing = net->layer_timing != 0;
    if (timing) {
        while ((int64_t)net->lev.size() < nl + 1) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            net->lev.push_back(e);
        }
        res->layer_ms.assign(nl, 0.0);
    }
    for (int64_t r0 = 0; r0 < std::max<int64_t>(B, 1); r0 += wave) {
        const int64_t r1 = std::min(B, r0 + wave);
        CK(cudaMemsetAsync(net->counts, 0, (nl + 1) * sizeof(int32_t), net->stream));
        CK(cudaEventRecord(net->ev0, net->stream));
        if (r1 > r0) {
            const int grid = (int)std::min<int64_t>((r1 - r0 + 255) / 256, 65535LL * 16);
            init_rows_kernel<<<grid, 256, 0, net->stream>>>(batch->off, r0, r1, 0, net->rows[0], net->counts);
            CK(cudaGetLastError());
            ++launches;
        }
        for (int64_t i = 0; i < nl; ++i) {
            const DevLayer& L = net->layers[first + i];
            if (timing) CK(cudaEventRecord(net->lev[i], net->stream));
            LayerArgs<T> a = make_args<T>(net, L, ymax);
            if (i == 0) {
                a.csr_off = batch->off;
                a.csr_cols = batch->cols;
                a.csr_vals = reinterpret_cast<const T*>(batch->vals);
            } else {
                a.y_in = reinterpret_cast<const T*>(net->ybuf[(i - 1) & 1]);
            }
            a.y_out = reinterpret_cast<T*>(net->ybuf[i & 1]);
            a.row_base = r0;
            a.rows_in = net->rows[i & 1];
            a.count_in = net->counts + i;
            a.rows_out = net->rows[(i + 1) & 1];
            a.count_out = net->counts + i + 1;
            if (int rc = launch_layer<T>(net, a)) return rc;
            ++launches;
        }
        if (timing) CK(cudaEventRecord(net->lev[nl], net->stream));
        CK(cudaEventRecord(net->ev1, net->stream));
        std::vector<int32_t> cnt(nl + 1);
        CK(cudaMemcpyAsync(cnt.data(), net->counts, (nl + 1) * 4, cudaMemcpyDeviceToHost, net->stream));
        CK(cudaStreamSynchronize(net->stream));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, net->ev0, net->ev1));
        total_ms += ms;
        for (int64_t l = 0; l <= nl; ++l) res->live[l] += cnt[l];
        if (timing)
            for (int64_t l = 0; l < nl; ++l) {
                float lm = 0;
                CK(cudaEventElapsedTime(&lm, net->lev[l], net->lev[l + 1]));
                res->layer_ms[l] += lm;
            }
        const int64_t F = cnt[nl];
        const int32_t* rows_dev = net->rows[nl & 1];
        if (want_y) {
            Piece p;
            std::vector<int32_t> cols;
            std::vector<T> vals;
            if (int rc = gather_rows<T>(net, reinterpret_cast<const T*>(net->ybuf[(nl - 1) & 1]), r0,
                                        (int)net->n, rows_dev, F, p.rows, p.nnz, p.cols, vals))
                return rc;
            p.vals.assign(vals.begin(), vals.end());
            // rows whose final entries all vanished cannot be listed (the
            // live list is exact), so every listed row has nnz > 0
            for (int32_t r : p.rows) final_rows.push_back(r);
            pieces.push_back(std::move(p));
        } else {
            std::vector<int32_t> fr(F);
            if (F) CK(cudaMemcpy(fr.data(), rows_dev, F * 4, cudaMemcpyDeviceToHost));
            final_rows.insert(final_rows.end(), fr.begin(), fr.end());
        }
        if (B == 0) break;
    }
    std::sort(final_rows.begin(), final_rows.end());
    res->cats.resize(final_rows.size());
    for (size_t i = 0; i < final_rows.size(); ++i) res->cats[i] = (int64_t)final_rows[i] + 1;
    res->dev_ms = total_ms;
    res->launches = launches;
    if (want_y) assemble(res, pieces);
    return SDNN_OK;
}

// Host CSR (int64/float64) -> device CSR (int64 offsets, int32 cols, T vals).
template <typename T>
int upload_csr(sdnn_net* net, int64_t n_rows, const int64_t* off, const int64_t* cols,
               const double* vals, int64_t n_cols, sdnn_batch* b) {
    const int64_t nnz = n_rows > 0 ? off[n_rows] : 0;
    if (n_rows > 0 && off[0] != 0) return fail(SDNN_ERR_PARAMETER, "row_offsets[0] must be 0");
    for (int64_t i = 0; i < n_rows; ++i)
        if (off[i + 1] < off[i]) return fail(SDNN_ERR_PARAMETER, "row_offsets non-monotone at %lld", (long long)i);
    b->n_rows = n_rows;
    b->nnz = nnz;
    const size_t bytes = (size_t)nnz * (4 + sizeof(T));
    if (bytes > net->pinned_cap) {
        if (net->pinned) CK(cudaFreeHost(net->pinned));
        net->pinned = nullptr;
        CK(cudaMallocHost(&net->pinned, std::max<size_t>(bytes, 64)));
        net->pinned_cap = std::max<size_t>(bytes, 64);
    }
    int32_t* pc = reinterpret_cast<int32_t*>(net->pinned);
    T* pv = reinterpret_cast<T*>(reinterpret_cast<char*>(net->pinned) + (size_t)nnz * 4);
    std::vector<int> bad(1, 0);
    parallel_for(nnz, [&](int64_t a, int64_t e) {
        for (int64_t p = a; p < e; ++p) {
            const int64_t c = cols[p];
            if (c < 0 || c >= n_cols) bad[0] = 1;
            pc[p] = (int32_t)c;
            pv[p] = (T)vals[p];
        }
    });
    if (bad[0]) return fail(SDNN_ERR_PARAMETER, "column index outside [0, %lld)", (long long)n_cols);
    CK(cudaMalloc(&b->off, (n_rows + 1) * sizeof(int64_t)));
    CK(cudaMalloc(&b->cols, std::max<int64_t>(nnz, 1) * 4));
    CK(cudaMalloc(&b->vals, std::max<int64_t>(nnz, 1) * sizeof(T)));
    CK(cudaMemcpyAsync(b->off, off, (n_rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, net->stream));
    CK(cudaMemcpyAsync(b->cols, pc, nnz * 4, cudaMemcpyHostToDevice, net->stream));
    CK(cudaMemcpyAsync(b->vals, pv, nnz * sizeof(T), cudaMemcpyHostToDevice, net->stream));
    CK(cudaStreamSynchronize(net->stream));
    return SDNN_OK;
}

void free_batch(sdnn_batch* b) {
    if (!b) return;
    cudaFree(b->off);
    cudaFree(b->cols);
    cudaFree(b->vals);
    delete b;
}

// CSR by input row (reference LayerWeights) -> output-major ELL, inputs
// ascending per output (rows are visited in ascending order).
int csr_to_ell(int64_t n_in, int64_t n_out, const int64_t* off, const int64_t* cols,
               const double* vals, int64_t nnz, std::vector<int32_t>& idx,
               std::vector<double>& val, int& width, std::vector<int64_t>& degree) {
    if (off[0] != 0 || off[n_in] != nnz) return fail(SDNN_ERR_PARAMETER, "inconsistent weight offsets");
    std::vector<int64_t> deg(n_out + 1, 0);
    for (int64_t i = 0; i < n_in; ++i) {
        if (off[i + 1] < off[i]) return fail(SDNN_ERR_PARAMETER, "weight offsets non-monotone");
        for (int64_t p = off[i]; p < off[i + 1]; ++p) {
            if (cols[p] < 0 || cols[p] >= n_out)
                return fail(SDNN_ERR_PARAMETER, "weight column %lld out of range", (long long)cols[p]);
            deg[cols[p]]++;
        }
    }
    int64_t w = 0;
    for (int64_t j = 0; j < n_out; ++j) w = std::max(w, deg[j]);
    width = (int)w;
    idx.assign((size_t)n_out * w, 0);
    val.assign((size_t)n_out * w, 0.0);
    std::vector<int64_t> fill(n_out, 0);
    degree.assign(deg.begin(), deg.begin() + n_out);
    for (int64_t i = 0; i < n_in; ++i) {
        for (int64_t p = off[i]; p < off[i + 1]; ++p) {
            const int64_t j = cols[p];
            const size_t e = (size_t)j * w + fill[j]++;
            idx[e] = (int32_t)i;
            val[e] = vals[p];
        }
    }
    return SDNN_OK;
}

int make_net(int device, int dtype, int64_t n, sdnn_net** out) {
    if (dtype != SDNN_F32 && dtype != SDNN_F64) return fail(SDNN_ERR_PARAMETER, "dtype must be 0 (f32) or 1 (f64)");
    if (n < 1 || n > (1LL << 30)) return fail(SDNN_ERR_PARAMETER, "neuron count %lld out of range", (long long)n);
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) return fail(SDNN_ERR_PARAMETER, "no CUDA device %d", device);
    CK(cudaSetDevice(device));
    sdnn_net* net = new sdnn_net;
    net->device = device;
    net->dtype = dtype;
    net->n = n;
    net->elem = dtype == SDNN_F64 ? 8 : 4;
    CK(cudaDeviceGetAttribute(&net->sm_count, cudaDevAttrMultiProcessorCount, device));
    CK(cudaStreamCreateWithFlags(&net->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&net->ev0));
    CK(cudaEventCreate(&net->ev1));
    if (int rc = configure(net)) {
        sdnn_net_destroy(net);
        return rc;
    }
    *out = net;
    return SDNN_OK;
}

}  // namespace

namespace sdnn {
__global__ void init_rows_kernel(const int64_t* __restrict__ off, int64_t r0, int64_t r1, int all_rows,
                                 int32_t* __restrict__ rows, int32_t* __restrict__ count) {
    for (int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r1;
         r += (int64_t)gridDim.x * blockDim.x) {
        const bool live = all_rows || off[r + 1] > off[r];
        const unsigned b = __ballot_sync(__activemask(), live);
        // warp-aggregated append
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(__activemask()) - 1;
        int base = 0;
        if (lane == leader && b) base = atomicAdd(count, __popc(b));
        base = __shfl_sync(__activemask(), base, leader);
        if (live) rows[base + __popc(b & ((1u << lane) - 1u))] = (int32_t)r;
    }
}
}  // namespace sdnn

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
        cudaFree(L.bnd);
    }
    for (auto b : net->ybuf) cudaFree(b);
    for (auto b : net->rows) cudaFree(b);
    cudaFree(net->counts);
    if (net->pinned) cudaFreeHost(net->pinned);
    for (auto e : net->lev) cudaEventDestroy(e);
    if (net->ev0) cudaEventDestroy(net->ev0);
    if (net->ev1) cudaEventDestroy(net->ev1);
    if (net->stream) cudaStreamDestroy(net->stream);
    delete net;
}

int sdnn_net_add_layer_csr(sdnn_net* net, const int64_t* w_off, const int64_t* w_cols,
                           const double* w_vals, int64_t nnz, double bias) {
    if (!net || !w_off) return fail(SDNN_ERR_PARAMETER, "null argument");
    if (int rc = set_device(net)) return rc;
    std::vector<int32_t> idx;
    std::vector<double> val;
    std::vector<int64_t> deg;
    int width = 0;
    if (int rc = csr_to_ell(net->n, net->n, w_off, w_cols, w_vals, nnz, idx, val, width, deg)) return rc;
    return upload_layer(net, width, idx.data(), val.data(), 0.0, bias, deg.data());
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
    return upload_layer(net, width, idx, vals, 0.0, bias, nullptr);
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
            if (int rc2 = upload_layer(net, width, idx.data() + (size_t)l * net->n * width, nullptr, value, bias,
                                       nullptr))
                return rc2;
    }
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
    int rc = net->dtype == SDNN_F64 ? run_impl<double>(net, batch, ymax, first, nl, want_y, res)
                                    : run_impl<float>(net, batch, ymax, first, nl, want_y, res);
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

int sdnn_infer(sdnn_net* net, int64_t n_rows, const int64_t* y_off, const int64_t* y_cols,
               const double* y_vals, double ymax, sdnn_result** out) {
    const double t0 = now_ms();
    sdnn_batch* b = nullptr;
    if (int rc = sdnn_batch_upload(net, n_rows, y_off, y_cols, y_vals, &b)) return rc;
    int rc = run_checked(net, b, ymax, 0, -1, 1, out);
    sdnn_batch_free(b);
    if (rc == SDNN_OK) (*out)->wall_ms = now_ms() - t0;
    return rc;
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
    *nnz = r->off.empty() ? 0 : r->off.back();
    return SDNN_OK;
}

int sdnn_result_y_csr(sdnn_result* r, int64_t* off, int64_t* cols, double* vals) {
    if (!r || !off) return fail(SDNN_ERR_PARAMETER, "null argument");
    if (!r->have_y) return fail(SDNN_ERR_PARAMETER, "result was produced without Y");
    memcpy(off, r->off.data(), r->off.size() * sizeof(int64_t));
    const size_t nnz = r->cols.size();
    for (size_t i = 0; i < nnz; ++i) cols[i] = r->cols[i];
    if (nnz) memcpy(vals, r->vals.data(), nnz * sizeof(double));
    return SDNN_OK;
}

void sdnn_result_free(sdnn_result* r) { delete r; }

int sdnn_spmm(int device, int dtype, int64_t n_rows, int64_t n_inner, int64_t n_out, const int64_t* y_off,
              const int64_t* y_cols, const double* y_vals, const int64_t* w_off, const int64_t* w_cols,
              const double* w_vals, sdnn_result** out) {
    if (!out || n_rows < 0 || n_inner < 1 || n_out < 1) return fail(SDNN_ERR_PARAMETER, "bad spmm shape");
    // one rectangular layer: build a scratch net of max(n_inner, n_out)
    // neurons whose geometry covers both extents, then run it raw
    sdnn_net* net = nullptr;
    const int64_t n = std::max(n_inner, n_out);
    if (int rc = make_net(device, dtype, n, &net)) return rc;
    int rc = SDNN_OK;
    sdnn_batch* b = nullptr;
    sdnn_result* res = nullptr;
    do {
        std::vector<int32_t> idx;
        std::vector<double> val;
        std::vector<int64_t> deg;
        int width = 0;
        const int64_t nnz_w = w_off[n_inner];
        // pad the weight CSR to n x n rows (extra rows empty)
        std::vector<int64_t> off(n + 1, nnz_w);
        memcpy(off.data(), w_off, (n_inner + 1) * sizeof(int64_t));
        if ((rc = csr_to_ell(n, n, off.data(), w_cols, w_vals, nnz_w, idx, val, width, deg))) break;
        if ((rc = upload_layer(net, width, idx.data(), val.data(), 0.0, 0.0, deg.data()))) break;
        b = new sdnn_batch;
        b->net = net;
        {
            static const int64_t zero_off[1] = {0};
            const int64_t* yo = n_rows > 0 ? y_off : zero_off;
            rc = dtype == SDNN_F64 ? upload_csr<double>(net, n_rows, yo, y_cols, y_vals, n_inner, b)
                                   : upload_csr<float>(net, n_rows, yo, y_cols, y_vals, n_inner, b);
            if (rc) break;
        }
        if ((rc = ensure_scratch(net, std::max<int64_t>(n_rows, 1), 1))) break;
        res = new sdnn_result;
        res->n_rows = n_rows;
        res->n_cols = n_out;
        res->n_layers = 1;
        res->live.assign(2, 0);
        auto body = [&](auto tag) -> int {
            using T = decltype(tag);
            CK(cudaMemsetAsync(net->counts, 0, 2 * sizeof(int32_t), net->stream));
            if (n_rows > 0) {
                const int grid = (int)std::min<int64_t>((n_rows + 255) / 256, 65535LL * 16);
                init_rows_kernel<<<grid, 256, 0, net->stream>>>(b->off, 0, n_rows, 1, net->rows[0], net->counts);
                CK(cudaGetLastError());
            }
            LayerArgs<T> a = make_args<T>(net, net->layers[0], 32.0);
            a.n_in = (int)n_inner;
            a.n_out = (int)n_out;
            a.epilogue = 0;
            a.csr_off = b->off;
            a.csr_cols = b->cols;
            a.csr_vals = reinterpret_cast<const T*>(b->vals);
            a.y_out = reinterpret_cast<T*>(net->ybuf[0]);
            a.rows_in = net->rows[0];
            a.count_in = net->counts;
            a.rows_out = net->rows[1];
            a.count_out = net->counts + 1;
            if (int e = launch_layer<T>(net, a)) return e;
            Piece p;
            std::vector<int32_t> cols;
            std::vector<T> vals;
            if (int e = gather_rows<T>(net, reinterpret_cast<const T*>(net->ybuf[0]), 0, (int)n_out, net->rows[0],
                                       n_rows, p.rows, p.nnz, p.cols, vals))
                return e;
            p.vals.assign(vals.begin(), vals.end());
            for (size_t i = 0; i < p.rows.size(); ++i)
                if (p.nnz[i] > 0) res->cats.push_back((int64_t)p.rows[i] + 1);
            std::sort(res->cats.begin(), res->cats.end());
            std::vector<Piece> ps;
            ps.push_back(std::move(p));
            assemble(res, ps);
            return SDNN_OK;
        };
        rc = dtype == SDNN_F64 ? body(double{}) : body(float{});
    } while (0);
    if (b) sdnn_batch_free(b);
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
    sdnn_batch* b = nullptr;
    int rc = sdnn_batch_upload(net, n_rows, off, cols, vals, &b);
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
            csr_brc_write_kernel<T><<<grid, 256, 0, net->stream>>>(b->off, b->cols, reinterpret_cast<const T*>(b->vals),
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
    if (b) sdnn_batch_free(b);
    sdnn_net_destroy(net);
    if (rc) {
        delete res;
        return rc;
    }
    *out = res;
    return SDNN_OK;
}

}  // extern "C"
