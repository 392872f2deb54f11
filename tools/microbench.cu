// microbench.cu -- B200 gather-rate probes that decide the layer-kernel design.
//   A: shared-memory gathers, 32 random addresses per warp (bank conflicts)
//   B: shared-memory gathers, conflict-free (lane-distinct banks)
//   C: L2 gathers of whole 128-byte lines (neuron-major slab, lane = row)
//   D: L2 gathers of 4-byte words at random addresses (row-major, lane = output)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t lcg(uint32_t& s) { s = s * 1664525u + 1013904223u; return s; }

template <int MODE>
__global__ void smem_gather(int iters, int words, float* out) {
    extern __shared__ float s[];
    for (int i = threadIdx.x; i < words; i += blockDim.x) s[i] = (float)(i & 7);
    __syncthreads();
    uint32_t st = threadIdx.x * 2654435761u + blockIdx.x;
    const int lane = threadIdx.x & 31;
    float acc = 0.f;
    const uint32_t mask = words - 1;
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
        uint32_t r = lcg(st);
        uint32_t a;
        if (MODE == 0) a = (r >> 8) & mask;                       // random
        else a = ((((r >> 8) & mask) & ~31u) | lane);           // conflict-free
        acc += s[a];
    }
    if (acc == -1.f) out[0] = acc;
}

__global__ void l2_line_gather(const float* __restrict__ slab, int n_lines, int iters, float* out) {
    // slab: [n_lines][32] floats; each warp reads whole random lines
    const int lane = threadIdx.x & 31;
    uint32_t st = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    st = st * 2654435761u + 12345u;
    float acc = 0.f;
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
        uint32_t r = lcg(st);
        uint32_t line = (r >> 4) % n_lines;
        acc += __ldg(slab + (size_t)line * 32 + lane);
    }
    if (acc == -1.f) out[0] = acc;
}

__global__ void l2_word_gather(const float* __restrict__ buf, int n_words, int iters, float* out) {
    uint32_t st = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 7u;
    float acc = 0.f;
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
        uint32_t r = lcg(st);
        acc += __ldg(buf + (r >> 4) % n_words);
    }
    if (acc == -1.f) out[0] = acc;
}

// 512-byte line per warp request (16 B per lane), MLP = U lines in flight
template <int U>
__global__ void l2_line512_gather(const float4* __restrict__ slab, int n_lines, int iters, float* out) {
    const int lane = threadIdx.x & 31;
    uint32_t st = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 2654435761u + 99u;
    float acc = 0.f;
    for (int i = 0; i < iters; i += U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t r = lcg(st);
            uint32_t line = (r >> 4) % n_lines;
            v[u] = slab[(size_t)line * 32 + lane];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    if (acc == -1.f) out[0] = acc;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    printf("SMs %d, max clock %.0f MHz\n", sms, clk / 1e3);
    float* out;
    CK(cudaMalloc(&out, 4));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int words = 16384;  // 64 KB
    const int iters = 4096;
    for (int mode = 0; mode < 2; ++mode) {
        for (int threads : {256, 512, 1024}) {
            auto fn = mode == 0 ? smem_gather<0> : smem_gather<1>;
            CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, words * 4));
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, words * 4);
            int grid = sms * occ;
            fn<<<grid, threads, words * 4>>>(iters, words, out);
            cudaEventRecord(a);
            fn<<<grid, threads, words * 4>>>(iters, words, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double g = (double)grid * threads * iters / (ms * 1e-3);
            printf("smem %s threads=%d occ=%d: %.3g gathers/s = %.2f per SM per ns\n",
                   mode ? "conflict-free" : "random", threads, occ, g, g / sms / 1e9);
        }
    }
    for (int mb : {8, 32, 96, 512}) {
        size_t bytes = (size_t)mb << 20;
        float* slab;
        CK(cudaMalloc(&slab, bytes));
        cudaMemset(slab, 0, bytes);
        int n_lines = (int)(bytes / 128);
        int grid = sms * 8, threads = 256, it = 2048;
        l2_line_gather<<<grid, threads>>>(slab, n_lines, it, out);
        cudaEventRecord(a);
        l2_line_gather<<<grid, threads>>>(slab, n_lines, it, out);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double lines = (double)grid * (threads / 32) * it;
        printf("L2 line gather %d MB slab: %.2f TB/s (%.3g lines/s)\n", mb, lines * 128 / (ms * 1e-3) / 1e12,
               lines / (ms * 1e-3));
        int n_words = (int)(bytes / 4);
        l2_word_gather<<<grid, threads>>>(slab, n_words, it, out);
        cudaEventRecord(a);
        l2_word_gather<<<grid, threads>>>(slab, n_words, it, out);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        double words_s = (double)grid * threads * it / (ms * 1e-3);
        printf("L2 word gather %d MB: %.3g words/s (%.2f per SM per ns)\n", mb, words_s, words_s / sms / 1e9);
        cudaFree(slab);
    }
    for (int mb : {32, 96}) {
        size_t bytes = (size_t)mb << 20;
        float4* slab;
        CK(cudaMalloc(&slab, bytes));
        cudaMemset(slab, 0, bytes);
        int n_lines = (int)(bytes / 512);
        for (int occ : {2, 4, 8}) {
            int grid = sms * occ, threads = 256, it = 1024;
            float ms;
            l2_line512_gather<8><<<grid, threads>>>(slab, n_lines, it, out);
            cudaEventRecord(a);
            l2_line512_gather<8><<<grid, threads>>>(slab, n_lines, it, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            cudaEventElapsedTime(&ms, a, b);
            double lines = (double)grid * (threads / 32) * it;
            printf("L2 512B-line gather %d MB, %d CTA/SM, MLP 8: %.2f TB/s\n", mb, occ, lines * 512 / (ms * 1e-3) / 1e12);
            l2_line512_gather<16><<<grid, threads>>>(slab, n_lines, it, out);
            cudaEventRecord(a);
            l2_line512_gather<16><<<grid, threads>>>(slab, n_lines, it, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            cudaEventElapsedTime(&ms, a, b);
            printf("L2 512B-line gather %d MB, %d CTA/SM, MLP 16: %.2f TB/s\n", mb, occ, lines * 512 / (ms * 1e-3) / 1e12);
        }
        cudaFree(slab);
    }
    return 0;
}
