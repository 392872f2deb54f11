// microbenchmark: L1 data-pipe wavefronts per broadcast shared load of 32/64/128 bits
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int W>
__global__ void k(unsigned* out, int iters) {
    __shared__ __align__(16) unsigned s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i * 3u;
    __syncthreads();
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) {
        const int idx = ((i * 4) & 1023);  // warp-uniform address
        if (W == 1) acc += s[idx];
        if (W == 2) { uint2 v = *reinterpret_cast<const uint2*>(&s[idx]); acc += v.x ^ v.y; }
        if (W == 4) { uint4 v = *reinterpret_cast<const uint4*>(&s[idx]); acc += v.x ^ v.y ^ v.z ^ v.w; }
        if (W == 5) { uint4 v = *reinterpret_cast<const uint4*>(&s[(idx + 4 * (threadIdx.x & 31)) & 1023]); acc += v.x ^ v.y ^ v.z ^ v.w; }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    unsigned* d; cudaMalloc(&d, 148 * 4 * 256 * 4);
    k<1><<<148 * 4, 256>>>(d, 4096); k<2><<<148 * 4, 256>>>(d, 4096); k<4><<<148 * 4, 256>>>(d, 4096);
    k<5><<<148 * 4, 256>>>(d, 4096);
    cudaDeviceSynchronize();
    printf("lds per kernel = %d\n", 148 * 4 * 8 * 4096);
    return 0;
}
