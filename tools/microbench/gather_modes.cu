// Random gathers from an L2-resident table: one divergent LDG per warp (32
// lines) vs 32 broadcast LDGs (1 line each, lane j's address shuffled to the
// whole warp).  Prints gathers/s and sectors/clk/SM for each mode.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void __launch_bounds__(256, 3) k(const uint4* __restrict__ tab, uint32_t mask, int iters, uint32_t* out) {
    const int lane = threadIdx.x & 31;
    uint32_t acc = 0, st = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    for (int it = 0; it < iters; ++it) {
        uint32_t idx[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { st = hash32(st + u); idx[u] = st & mask; }
        if (MODE == 0) {
#pragma unroll
            for (int u = 0; u < 4; ++u) { uint4 v = __ldg(tab + idx[u]); acc ^= v.x ^ v.y; }
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                uint32_t mine = 0;
#pragma unroll 8
                for (int j = 0; j < 32; ++j) {
                    const uint32_t a = __shfl_sync(0xffffffffu, idx[u], j);
                    const uint4 v = __ldg(tab + a);
                    if (lane == j) mine = v.x ^ v.y;
                }
                acc ^= mine;
            }
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    const size_t n = 1 << 18;  // 256k entries x 16 B = 4 MB (L2-resident)
    uint4* tab; uint32_t* out;
    cudaMalloc(&tab, n * 16); cudaMemset(tab, 1, n * 16); cudaMalloc(&out, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 200, grid = sms * 3;
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<grid, 256>>>(tab, (uint32_t)(n - 1), iters, out);
            else k<1><<<grid, 256>>>(tab, (uint32_t)(n - 1), iters / 8, out);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double gathers = (double)grid * 256 * 4 * (mode == 0 ? iters : iters / 8);
            double gps = gathers / (ms * 1e-3);
            if (rep == 2) printf("mode %s: %.1f G gathers/s, %.2f sectors/clk/SM (at %.0f MHz)\n",
                                 mode == 0 ? "divergent LDG (32 lines)" : "32 broadcast LDGs      ",
                                 gps / 1e9, gps / ((double)sms * clk * 1e3), clk / 1e3);
        }
    }
    return 0;
}
