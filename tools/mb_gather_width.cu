// mb_gather_width.cu -- L1 data-pipe cost of a packed, predicated gather of
// one activation line, by access width.
//
// A line of 256 rows is stored sector-packed: only the pieces holding a
// nonzero are kept, in lane order.  Each lane loads its own piece if it is
// live (predicated), at base + popc(live & lanes_below) * W.
//   W = 32: lane = 8 rows (one 256-bit load per lane per line)
//   W = 16: lane = 4 rows, two 128-bit loads per line (rows 0-127, 128-255)
// Live pieces are drawn per lane with probability p (C4 layer 2: 5 % of
// values nonzero -> p = 0.34 for 8-row pieces, 0.185 for 4-row pieces).
// Read the wavefronts per load with ncu:
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_lg.sum,smsp__inst_executed_op_global_ld.sum,
//       l1tex__data_pipe_lsu_wavefronts.sum,gpu__time_duration.sum ./mb_gather_width
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_gather_width mb_gather_width.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                \
    do {                                                                     \
        cudaError_t e = (x);                                                 \
        if (e != cudaSuccess) {                                              \
            printf("%s: %s\n", #x, cudaGetErrorString(e));                   \
            return 1;                                                        \
        }                                                                    \
    } while (0)

__device__ __forceinline__ uint32_t lcg(uint32_t& s) {
    s = s * 1664525u + 1013904223u;
    return s;
}

__device__ __forceinline__ void ld32(float (&d)[8], const char* p, bool live) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %9, 0;\n\t"
                 "@q ld.global.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n\t}"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]), "+f"(d[4]), "+f"(d[5]), "+f"(d[6]), "+f"(d[7])
                 : "l"(p), "r"((unsigned)live));
}
__device__ __forceinline__ void ld16(float (&d)[4], const char* p, bool live) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t"
                 "@q ld.global.v4.f32 {%0, %1, %2, %3}, [%4];\n\t}"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "l"(p), "r"((unsigned)live));
}

// MODE 0: 256-bit pieces.  MODE 1: 128-bit pieces, two loads per line.
// MODE 2: 128-bit pieces, lane owns pieces 2l and 2l+1 (interleaved halves).
// MODE 3: 32-byte sectors packed as in MODE 0 (a sector is stored when either
//         half holds a nonzero), each half loaded by its own predicated
//         128-bit load (half-sector live masks).
template <int MODE>
__global__ void gather(const char* __restrict__ buf, int iters, uint32_t thresh, float* out) {
    const int lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    uint32_t st = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 99u;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // 64 line slots of 2 KB: L1-resident after the first pass
    for (int i = 0; i < iters; ++i) {
        const char* line = buf + (size_t)(i & 63) * 2048;
        if (MODE == 0) {
            const bool live = lcg(st) < thresh;
            const unsigned m = __ballot_sync(0xffffffffu, live);
            float d[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) d[c] = acc[c];
            ld32(d, line + __popc(m & below) * 32, live);
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] += d[c];
        } else {
            const bool l0 = lcg(st) < thresh, l1 = lcg(st) < thresh;
            const unsigned m0 = __ballot_sync(0xffffffffu, l0), m1 = __ballot_sync(0xffffffffu, l1);
            float d[4], e[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) d[c] = e[c] = acc[c];
            if (MODE == 3) {  // sector-packed, two predicated halves
                const unsigned ms = m0 | m1;
                const char* sec = line + __popc(ms & below) * 32;
                ld16(d, sec, l0);
                ld16(e, sec + 16, l1);
            } else if (MODE == 1) {  // pieces l and 32 + l
                ld16(d, line + __popc(m0 & below) * 16, l0);
                ld16(e, line + (__popc(m0) + __popc(m1 & below)) * 16, l1);
            } else {  // pieces 2l and 2l + 1 in one packed order
                // interleave: piece 2l live = l0, 2l+1 = l1; rank among pieces below
                const int r0 = __popc(m0 & below) + __popc(m1 & below);
                ld16(d, line + r0 * 16, l0);
                ld16(e, line + (r0 + (l0 ? 1 : 0)) * 16, l1);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[c] += d[c] + e[c];
        }
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c];
    if (s == -1.f) out[0] = s;
}

int main() {
    char* buf;
    float* out;
    CK(cudaMalloc(&buf, 64 * 2048 + 4096));
    CK(cudaMemset(buf, 0, 64 * 2048 + 4096));
    CK(cudaMalloc(&out, 4));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int iters = 1 << 14;
    const dim3 grid(sms * 4), block(256);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    struct P {
        const char* name;
        int mode;
        double p;
    } ps[] = {{"w32 p=0.34", 0, 0.34}, {"w16 halves p=0.185", 1, 0.185}, {"w16 interleaved p=0.185", 2, 0.185},
              {"w32 p=1.0", 0, 1.0},   {"w16 halves p=1.0", 1, 1.0},     {"w32 p=0.1", 0, 0.1},
              {"w16 halves p=0.05", 1, 0.05},  {"w16 sector-packed p=0.185", 3, 0.185},
              {"w16 sector-packed p=1.0", 3, 1.0}};
    for (auto& q : ps) {
        const uint32_t th = q.p >= 1.0 ? 0xffffffffu : (uint32_t)(q.p * 4294967296.0);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (q.mode == 0) gather<0><<<grid, block>>>(buf, iters, th, out);
            else if (q.mode == 1) gather<1><<<grid, block>>>(buf, iters, th, out);
            else if (q.mode == 3) gather<3><<<grid, block>>>(buf, iters, th, out);
            else gather<2><<<grid, block>>>(buf, iters, th, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double lines = (double)grid.x * (block.x / 32) * iters;
        printf("%-26s %8.3f ms  %.3f ns per warp-line per SM\n", q.name, ms, ms * 1e6 / (lines / sms));
    }
    return 0;
}
