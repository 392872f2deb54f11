// microbenchmark: does SHFL use the L1 data-pipe (lsu wavefronts) like a broadcast LDS?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_shfl(unsigned* out, int iters) {
    unsigned v = threadIdx.x * 7u, acc = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            acc += __shfl_sync(0xffffffffu, v + acc, (i + u) & 31);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_lds(unsigned* out, int iters) {
    __shared__ unsigned s[8][32];
    s[threadIdx.x / 32 % 8][threadIdx.x % 32] = threadIdx.x * 7u;
    __syncthreads();
    unsigned acc = 0;
    const unsigned* w = s[threadIdx.x / 32 % 8];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            acc += w[(i + u + acc) & 31];  // broadcast-ish: same index for all lanes of a warp (acc uniform)
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    unsigned* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(a); k_shfl<<<148 * 4, 256>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("shfl: %.3f ms, %.2f warp-shfl/clk/SM @1.965GHz\n", ms, 148.0*4*8*iters*8 / (ms*1e-3) / 148 / 1.965e9);
        cudaEventRecord(a); k_lds<<<148 * 4, 256>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("lds : %.3f ms, %.2f warp-lds/clk/SM\n", ms, 148.0*4*8*iters*8 / (ms*1e-3) / 148 / 1.965e9);
    }
    return 0;
}
