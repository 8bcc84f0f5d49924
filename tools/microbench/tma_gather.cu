// Random 16-byte row gathers from an L2-resident table through TMA
// tile::gather4 (4 rows per instruction, into shared memory, mbarrier
// completion) vs plain divergent LDGs.  Question: does the TMA path beat the
// ~1 line/clk/SM LSU ceiling for random rows?
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int WARPS = 4;
constexpr int NB = 2;  // buffers in flight per warp

__global__ void __launch_bounds__(WARPS * 32) k_tma(const __grid_constant__ CUtensorMap tmap, uint32_t mask,
                                                    int iters, uint32_t* out) {
    __shared__ __align__(128) uint4 buf[WARPS][NB][256];   // 32 gathers x (4 rows x 16 B, 128-byte aligned)
    __shared__ __align__(8) uint64_t bar[WARPS][NB];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0)
        for (int b = 0; b < NB; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[w][b])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncwarp();
    uint32_t st = hash32(blockIdx.x * blockDim.x + threadIdx.x), acc = 0;
    auto issue = [&](int b) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[w][b])), "r"(128 * 16));
        __syncwarp();
        int r[4];
        for (int u = 0; u < 4; ++u) { st = hash32(st + u); r[u] = (int)(st & mask); }
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
            :: "r"(smem_u32(&buf[w][b][lane * 8])), "l"(&tmap), "r"(smem_u32(&bar[w][b])),
               "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
    };
    uint32_t phase[NB] = {0, 0};
    for (int b = 0; b < NB; ++b) issue(b);
    for (int it = 0; it < iters; ++it) {
        const int b = it % NB;
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
            :: "r"(smem_u32(&bar[w][b])), "r"(phase[b]));
        phase[b] ^= 1;
        uint4 v = buf[w][b][lane * 8];
        acc ^= v.x;
        __syncwarp();
        if (it + NB < iters) issue(b);
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// mixed: the CTA's first WARPS warps run the TMA loop, the remaining LW warps divergent LDGs
template <int LW>
__global__ void __launch_bounds__((WARPS + LW) * 32) k_mix(const __grid_constant__ CUtensorMap tmap, const uint4* __restrict__ tab,
                                                           uint32_t mask, int iters, int ldg_iters, uint32_t* out) {
    __shared__ __align__(128) uint4 buf[WARPS][NB][256];
    __shared__ __align__(8) uint64_t bar[WARPS][NB];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t st = hash32(blockIdx.x * blockDim.x + threadIdx.x), acc = 0;
    if (w >= WARPS) {
        for (int it = 0; it < ldg_iters; ++it) {
            uint32_t idx[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { st = hash32(st + u); idx[u] = st & mask; }
#pragma unroll
            for (int u = 0; u < 4; ++u) { uint4 v = __ldg(tab + idx[u]); acc ^= v.x ^ v.y; }
        }
        if (acc == 0x12345678u) out[0] = acc;
        return;
    }
    if (lane == 0)
        for (int b = 0; b < NB; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[w][b])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncwarp();
    auto issue = [&](int b) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[w][b])), "r"(128 * 16));
        __syncwarp();
        int r[4];
        for (int u = 0; u < 4; ++u) { st = hash32(st + u); r[u] = (int)(st & mask); }
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
            :: "r"(smem_u32(&buf[w][b][lane * 8])), "l"(&tmap), "r"(smem_u32(&bar[w][b])),
               "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
    };
    uint32_t phase[NB] = {0, 0};
    for (int b = 0; b < NB; ++b) issue(b);
    for (int it = 0; it < iters; ++it) {
        const int b = it % NB;
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
            :: "r"(smem_u32(&bar[w][b])), "r"(phase[b]));
        phase[b] ^= 1;
        uint4 v = buf[w][b][lane * 8];
        acc ^= v.x;
        __syncwarp();
        if (it + NB < iters) issue(b);
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void __launch_bounds__(256, 3) k_ldg(const uint4* __restrict__ tab, uint32_t mask, int iters, uint32_t* out) {
    uint32_t acc = 0, st = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    for (int it = 0; it < iters; ++it) {
        uint32_t idx[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { st = hash32(st + u); idx[u] = st & mask; }
#pragma unroll
        for (int u = 0; u < 4; ++u) { uint4 v = __ldg(tab + idx[u]); acc ^= v.x ^ v.y; }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    const size_t n = 1 << 18;  // 256k rows x 16 B = 4 MB
    uint4* tab; uint32_t* out;
    cudaMalloc(&tab, n * 16); cudaMemset(tab, 1, n * 16); cudaMalloc(&out, 4);
    CUtensorMap tmap;
    cuuint64_t dims[2] = {4, n};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {4, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult rc = cuTensorMapEncodeTiled(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, tab, dims, strides, box, estr,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) { printf("tensor map encode failed %d\n", (int)rc); return 1; }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int blocks_per_sm : {4, 8, 16}) {
        const int iters = 400, grid = sms * blocks_per_sm;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_tma<<<grid, WARPS * 32>>>(tmap, (uint32_t)(n - 1), iters, out);
            cudaEventRecord(b); cudaEventSynchronize(b);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) { printf("tma kernel: %s\n", cudaGetErrorString(e)); return 1; }
            float ms; cudaEventElapsedTime(&ms, a, b);
            double rows = (double)grid * WARPS * 128 * iters;
            if (rep == 1) printf("TMA gather4, %d CTAs/SM: %.1f G rows/s = %.2f rows/clk/SM\n", blocks_per_sm,
                                 rows / (ms * 1e-3) / 1e9, rows / (ms * 1e-3) / ((double)sms * clk * 1e3));
        }
    }
    for (int rep = 0; rep < 2; ++rep) {  // mixed: 4 TMA warps + 4 LDG warps per CTA, 4 CTAs/SM
        const int iters = 400, ldg_iters = 400, grid = sms * 4;
        cudaEventRecord(a);
        k_mix<4><<<grid, (WARPS + 4) * 32>>>(tmap, tab, (uint32_t)(n - 1), iters, ldg_iters, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double rows = (double)grid * (WARPS * 128.0 * iters + 4 * 32 * 4.0 * ldg_iters);
        if (rep == 1) printf("mixed TMA + LDG: %.1f G rows/s = %.2f rows/clk/SM (ms %.3f)\n", rows / (ms * 1e-3) / 1e9,
                             rows / (ms * 1e-3) / ((double)sms * clk * 1e3), ms);
    }
    for (int rep = 0; rep < 2; ++rep) {
        const int iters = 200, grid = sms * 3;
        cudaEventRecord(a);
        k_ldg<<<grid, 256>>>(tab, (uint32_t)(n - 1), iters, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double rows = (double)grid * 256 * 4 * iters;
        if (rep == 1) printf("LDG divergent: %.1f G rows/s = %.2f rows/clk/SM\n", rows / (ms * 1e-3) / 1e9,
                             rows / (ms * 1e-3) / ((double)sms * clk * 1e3));
    }
    return 0;
}
