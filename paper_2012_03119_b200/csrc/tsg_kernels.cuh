// tsg_kernels.cuh -- the hot-path kernels (sm_100a).
//
//   K1+K2    k_encode  int8 snapshots -> lane words + aggregates   (bitpack.py:81-117, 152-167, 211-244)
//   K3+K4+K5 k_test    two-stage trigger test, report emission,
//                      activity bump, counters                      (engine.py:238-254, 437-467)
//
// Both are memory-bound integer kernels; DESIGN.md §4 gives their rooflines.
#pragma once
#include <climits>
#include <cstdint>

#include "../../include/tsg.h"
#include "tsg_device.cuh"

namespace tsg {

constexpr int MAXG = 64;

#ifndef TSG_TEST_MIN_BLOCKS
#define TSG_TEST_MIN_BLOCKS 3
#endif

// ---------------------------------------------------------------------------
// K1+K2: encoder.
//
// Block = 32 x 8 threads covers 128 variables of one chunk.  Thread (x, y)
// owns variables 4x..4x+3 and groups y, y+8, ...  For each group it streams
// the group's rows as one u32 (4 variables) per row, so every warp load is a
// coalesced 128-byte row segment.  Bytes become lane bits without per-bit
// work: exact per-byte "== TRUE" / "!= UNDEF" masks land in each byte's MSB
// (SWAR zero-byte tests), and eight rows are transposed into one byte per
// variable by shift-merging the MSB masks.  Lane words are written
// group-major (lane[g][v]), four consecutive variables per thread, so the
// stores are contiguous; aggregate bits are OR-reduced across groups in
// shared memory.

struct EncodeChunk {
    int32_t G;            // groups in the chunk
    int32_t num_vars;
    int64_t pitch;        // bytes between rows (multiple of 4)
    int64_t vstride;      // lane-table row length (num_vars + 2)
    int64_t row0[MAXG];   // first row of each group
    int32_t lanes[MAXG];  // rows (lanes) of each group
    unsigned long long* polarity;  // [2] += (var, group) pairs that can be True / can be False
};

// 0x80 in every byte of w that is != 0
__device__ __forceinline__ uint32_t nz_msb(uint32_t w) {
    uint32_t t = (w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
    return (t | w) & 0x80808080u;
}
// 0x80 in every byte of w that is == 0x01 (TRUE)
__device__ __forceinline__ uint32_t eq1_msb(uint32_t w) {
    uint32_t y = w ^ 0x01010101u;
    uint32_t t = (y & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
    return ~(t | y) & 0x80808080u;
}

template <class LW>
__device__ __forceinline__ void st_lane4(LaneEntry<LW>* p, const LW* t, const LW* s);
template <>
__device__ __forceinline__ void st_lane4<uint32_t>(LaneEntry<uint32_t>* p, const uint32_t* t, const uint32_t* s) {
    uint4* q = reinterpret_cast<uint4*>(p);
    q[0] = make_uint4(t[0], s[0], t[1], s[1]);
    q[1] = make_uint4(t[2], s[2], t[3], s[3]);
}
template <>
__device__ __forceinline__ void st_lane4<uint64_t>(LaneEntry<uint64_t>* p, const uint64_t* t, const uint64_t* s) {
    ulonglong2* q = reinterpret_cast<ulonglong2*>(p);
#pragma unroll
    for (int b = 0; b < 4; ++b) q[b] = make_ulonglong2(t[b], s[b]);
}

template <class LW, class GW>
__global__ void __launch_bounds__(256) k_encode(const int8_t* __restrict__ rows, const __grid_constant__ EncodeChunk c,
                                                LaneEntry<LW>* __restrict__ lane,
                                                AggEntry<GW>* __restrict__ agg) {
    __shared__ GW sT[128], sF[128], sU[128];
    const int x = threadIdx.x, y = threadIdx.y, t = y * 32 + x;
    if (t < 128) { sT[t] = 0; sF[t] = 0; sU[t] = 0; }
    __syncthreads();
    const int64_t vbase = (int64_t)blockIdx.x * 128;
    const int64_t v0 = vbase + 4 * x;
    const int64_t V = c.num_vars;
    for (int g = y; g < c.G; g += 8) {
        const int n = c.lanes[g];
        LW tw[4] = {0, 0, 0, 0}, sw[4] = {0, 0, 0, 0};
        if (v0 <= V) {
            const int8_t* base = rows + c.row0[g] * c.pitch + v0;
            for (int r0 = 0; r0 < n; r0 += 16) {  // 16 row loads in flight per thread
                uint32_t w[16];
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    w[k] = (r0 + k < n) ? __ldg(reinterpret_cast<const uint32_t*>(base + (int64_t)(r0 + k) * c.pitch)) : 0u;
#pragma unroll
                for (int h = 0; h < 16; h += 8) {
                    uint32_t aT = 0, aS = 0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {  // row r0+h+k ends at bit k of each byte
                        aT = ((aT >> 1) & 0x7F7F7F7Fu) | eq1_msb(w[h + k]);
                        aS = ((aS >> 1) & 0x7F7F7F7Fu) | nz_msb(w[h + k]);
                    }
                    if (r0 + h < (int)(sizeof(LW) * 8)) {
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            tw[b] |= (LW)((aT >> (8 * b)) & 0xFFu) << (r0 + h);
                            sw[b] |= (LW)((aS >> (8 * b)) & 0xFFu) << (r0 + h);
                        }
                    }
                }
            }
        }
        if (v0 == 0) { tw[0] = 0; sw[0] = 0; }  // slot 0 is never set (bitpack.py:110-111)
        LaneEntry<LW>* dst = lane + (int64_t)g * c.vstride + v0;
        if (v0 + 3 <= V + 1) {
            if (v0 + 3 == V + 1) { tw[3] = 0; sw[3] = ~LW(0); }  // sentinel: always False
            st_lane4<LW>(dst, tw, sw);
        } else {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                if (v0 + b <= V) dst[b] = LaneEntry<LW>{tw[b], sw[b]};
                else if (v0 + b == V + 1) dst[b] = LaneEntry<LW>{LW(0), ~LW(0)};
            }
        }
        const LW lm = width_mask<LW>(n);
        const GW bit = GW(1) << g;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t v = v0 + b;
            if (v >= 1 && v <= V) {  // AggregateAssignment.from_packed, bitpack.py:156-166
                if (tw[b] != 0) or_shared(&sT[4 * x + b], bit);
                if ((sw[b] & ~tw[b]) != 0) or_shared(&sF[4 * x + b], bit);
                if (n == 0 || (~sw[b] & lm) != 0) or_shared(&sU[4 * x + b], bit);
            }
        }
    }
    __syncthreads();
    if (t < 128) {
        const int64_t v = vbase + t;
        if (v <= V) agg[v] = AggEntry<GW>{sT[t], sF[t], sU[t], GW(0)};
        else if (v == V + 1) agg[v] = AggEntry<GW>{~GW(0), ~GW(0), GW(0), GW(0)};
        // polarity statistics for the store's literal placement
        unsigned nt = (v >= 1 && v <= V) ? __popcll((unsigned long long)sT[t]) : 0u;
        unsigned nf = (v >= 1 && v <= V) ? __popcll((unsigned long long)sF[t]) : 0u;
        nt = __reduce_add_sync(0xffffffffu, nt);
        nf = __reduce_add_sync(0xffffffffu, nf);
        if ((t & 31) == 0 && c.polarity) {
            atomicAdd(c.polarity, (unsigned long long)nt);
            atomicAdd(c.polarity + 1, (unsigned long long)nf);
        }
    }
}

// ---------------------------------------------------------------------------
// K1+K2 from packed rows: every snapshot row arrives as
// 2 bits per variable -- u64 word k holds variables 32k..32k+31, low half
// "== TRUE", high half "!= UNDEF" (tsg_pack_rows) -- a quarter of the int8
// bytes.  Block = 32 x 8 threads covers 128 variables (4 words per row);
// warp y takes groups y, y+8, ...  Lane r loads row r of the group (32
// contiguous bytes), and a 5-step shuffle transpose turns the 32 rows x 32
// variables bit matrix into one lane word per variable, so lane v ends up
// with is_true / is_set of variable v exactly as k_encode produces them.

// 32x32 bit transpose across the warp: afterwards bit j of lane i's word is
// bit i of lane j's word before.  Stage s exchanges s-blocks with lane^s: a
// per-lane rotate (left by s, or right by s when lane bit s is set) brings the
// partner's block into place and one LOP3 merges it under the stage mask --
// SHFL + SHF + LOP3 per stage (the wrapped-around bits fall outside the mask).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
#pragma unroll
    for (int sft = 16; sft >= 1; sft >>= 1) {
        const uint32_t m = sft == 16 ? 0x0000FFFFu : sft == 8 ? 0x00FF00FFu : sft == 4 ? 0x0F0F0F0Fu
                         : sft == 2 ? 0x33333333u : 0x55555555u;
        const bool up = lane & sft;
        const uint32_t keep = up ? ~m : m;
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, sft);
        const uint32_t yy = __funnelshift_l(y, y, up ? 32 - sft : sft);  // rotate
        x = (x & keep) | (yy & ~keep);
    }
    return x;
}

struct EncodePackedChunk {
    int32_t G;
    int32_t num_vars;
    int64_t pitch_words;  // u64 words between rows (multiple of 4)
    int64_t vstride;
    int64_t row0[MAXG];
    int32_t lanes[MAXG];
    unsigned long long* polarity;  // [2] += (var, group) pairs that can be True / can be False
    // k_encode_packed32 only: encode groups [gbeg, gend) of the chunk (the
    // others' lane entries are left alone and their aggregate bits are 0,
    // so the ranks' tables combine by all-gather + sum); `sentinel` writes
    // the always-False entry of variable num_vars + 1 (exactly one rank)
    int32_t gbeg, gend, sentinel;
};

template <class LW, class GW>
__global__ void __launch_bounds__(256) k_encode_packed(const uint64_t* __restrict__ rows,
                                                       const __grid_constant__ EncodePackedChunk c,
                                                       LaneEntry<LW>* __restrict__ lane_tab,
                                                       AggEntry<GW>* __restrict__ agg) {
    __shared__ GW sT[128], sF[128], sU[128];
    const int lane = threadIdx.x, y = threadIdx.y, t = y * 32 + lane;
    if (t < 128) { sT[t] = 0; sF[t] = 0; sU[t] = 0; }
    __syncthreads();
    const int64_t vbase = (int64_t)blockIdx.x * 128;
    const int64_t V = c.num_vars;
    const int64_t w0 = (int64_t)blockIdx.x * 4;  // first word of the block in every row
    // this lane's 32 bytes of row `half * 32 + lane` of group g (zeros past the group)
    auto load_row = [&](int g, int half, uint4& a, uint4& b) {
        const int r = half * 32 + lane;
        a = make_uint4(0, 0, 0, 0);
        b = make_uint4(0, 0, 0, 0);
        if (g < c.G && r < c.lanes[g]) {
            const uint4* src = reinterpret_cast<const uint4*>(rows + (c.row0[g] + r) * c.pitch_words + w0);
            a = __ldg(src);
            b = __ldg(src + 1);
        }
    };
    uint4 na, nb;  // <= 32 lanes: the warp's next group is loaded while this one is transposed
    if constexpr (sizeof(LW) == 4) load_row(y, 0, na, nb);
    for (int g = y; g < c.G; g += 8) {
        const int n = c.lanes[g];
        LW tw[4] = {0, 0, 0, 0}, sw[4] = {0, 0, 0, 0};
#pragma unroll
        for (int half = 0; half < (int)(sizeof(LW) / 4); ++half) {
            if (half * 32 >= n) break;
            uint4 a, b;
            if constexpr (sizeof(LW) == 4) {
                a = na;
                b = nb;
                load_row(g + 8, 0, na, nb);
            } else {
                load_row(g, half, a, b);
            }
            const uint32_t tv[4] = {a.x, a.z, b.x, b.z}, sv[4] = {a.y, a.w, b.y, b.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                tw[k] |= (LW)warp_transpose32(tv[k], lane) << (32 * half);
                sw[k] |= (LW)warp_transpose32(sv[k], lane) << (32 * half);
            }
        }
        if constexpr (sizeof(LW) == 4) {
            if (n == 0) load_row(g + 8, 0, na, nb);  // the half loop did not run
        }
        const LW lm = width_mask<LW>(n);
        const GW bit = GW(1) << g;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t v = vbase + 32 * k + lane;
            LW tk = tw[k], sk = sw[k];
            if (v == 0) { tk = 0; sk = 0; }  // slot 0 is never set (bitpack.py:110-111)
            LaneEntry<LW>* dst = lane_tab + (int64_t)g * c.vstride + v;
            if (v <= V) *dst = LaneEntry<LW>{tk, sk};
            else if (v == V + 1) *dst = LaneEntry<LW>{LW(0), ~LW(0)};  // sentinel: always False
            if (v >= 1 && v <= V) {  // AggregateAssignment.from_packed, bitpack.py:156-166
                if (tk != 0) or_shared(&sT[32 * k + lane], bit);
                if ((sk & ~tk) != 0) or_shared(&sF[32 * k + lane], bit);
                if (n == 0 || (~sk & lm) != 0) or_shared(&sU[32 * k + lane], bit);
            }
        }
    }
    __syncthreads();
    if (t < 128) {
        const int64_t v = vbase + t;
        if (v <= V) agg[v] = AggEntry<GW>{sT[t], sF[t], sU[t], GW(0)};
        else if (v == V + 1) agg[v] = AggEntry<GW>{~GW(0), ~GW(0), GW(0), GW(0)};
        // polarity statistics for the store's literal placement
        unsigned nt = (v >= 1 && v <= V) ? __popcll((unsigned long long)sT[t]) : 0u;
        unsigned nf = (v >= 1 && v <= V) ? __popcll((unsigned long long)sF[t]) : 0u;
        nt = __reduce_add_sync(0xffffffffu, nt);
        nf = __reduce_add_sync(0xffffffffu, nf);
        if ((t & 31) == 0 && c.polarity) {
            atomicAdd(c.polarity, (unsigned long long)nt);
            atomicAdd(c.polarity + 1, (unsigned long long)nf);
        }
    }
}

// Lane width <= 32 (one row per lane): every warp first queues ALL its
// groups' rows (32 bytes per row) as 16-byte cp.async copies into its own
// shared-memory stage, one commit group per group, then transposes group j
// as soon as its copies land (cp.async.wait_group) -- up to 64 KB per SM in
// flight instead of one group per warp, so the encoder streams the rows at
// HBM rate rather than waiting on each group's load.  A lane reads back only
// the row it copied, so no warp barrier is needed; the two 16-byte halves
// are swapped on every other 4-lane quad (conflict-free 128-bit reads).
constexpr int ENC_MAX_GPW = 8;  // groups per warp (G <= 64, 8 warps)

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_upto(int pending) {  // wait until <= pending groups are in flight
    switch (pending) {
        case 0: asm volatile("cp.async.wait_group 0;\n" ::: "memory"); break;
        case 1: asm volatile("cp.async.wait_group 1;\n" ::: "memory"); break;
        case 2: asm volatile("cp.async.wait_group 2;\n" ::: "memory"); break;
        case 3: asm volatile("cp.async.wait_group 3;\n" ::: "memory"); break;
        case 4: asm volatile("cp.async.wait_group 4;\n" ::: "memory"); break;
        case 5: asm volatile("cp.async.wait_group 5;\n" ::: "memory"); break;
        case 6: asm volatile("cp.async.wait_group 6;\n" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 7;\n" ::: "memory"); break;
    }
}

// Lane-dependent constants of warp_transpose32, computed once per thread.
struct Transpose32 {
    uint32_t keep[5], amt[5];
    uint32_t sel[2];  // byte stages (16, 8): one PRMT takes the partner's bytes in place
    __device__ __forceinline__ explicit Transpose32(int lane) {
        sel[0] = (lane & 16) ? 0x3276u : 0x5410u;
        sel[1] = (lane & 8) ? 0x3715u : 0x6240u;
        asm volatile("" : "+r"(sel[0]), "+r"(sel[1]));
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const int sft = 16 >> i;
            const uint32_t m = i == 0 ? 0x0000FFFFu : i == 1 ? 0x00FF00FFu : i == 2 ? 0x0F0F0F0Fu
                             : i == 3 ? 0x33333333u : 0x55555555u;
            const bool up = lane & sft;
            keep[i] = up ? ~m : m;
            amt[i] = up ? 32 - sft : sft;
            // opaque from here on: one register each, so a stage is SHFL +
            // SHF + one LOP3 select instead of the masks being refolded
            asm volatile("" : "+r"(keep[i]), "+r"(amt[i]));
        }
    }
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
#pragma unroll
        for (int i = 0; i < 2; ++i) x = __byte_perm(x, __shfl_xor_sync(0xffffffffu, x, 16 >> i), sel[i]);
#pragma unroll
        for (int i = 2; i < 5; ++i) {
            const uint32_t y = __shfl_xor_sync(0xffffffffu, x, 16 >> i);
            const uint32_t yy = __funnelshift_l(y, y, amt[i]);  // rotate the partner's block into place
            uint32_t r;
            asm("lop3.b32 %0, %1, %2, %3, 0xE2;" : "=r"(r) : "r"(x), "r"(keep[i]), "r"(yy));  // keep ? x : yy
            x = r;
        }
        return x;
    }
};

template <class GW, int GPW>
__global__ void __launch_bounds__(256) k_encode_packed32(const uint64_t* __restrict__ rows,
                                                         const __grid_constant__ EncodePackedChunk c,
                                                         LaneEntry<uint32_t>* __restrict__ lane_tab,
                                                         AggEntry<GW>* __restrict__ agg) {
    extern __shared__ uint4 stage[];  // [8 warps][GPW groups][32 rows][2 halves]
    // per-warp aggregate bits: bit j of part[plane][warp][var] = group warp + 8j
    __shared__ uint8_t part[3][8][128];
    const int lane = threadIdx.x, y = threadIdx.y, t = y * 32 + lane;
    const int64_t vbase = (int64_t)blockIdx.x * 128;
    const int64_t V = c.num_vars;
    const int64_t w0 = (int64_t)blockIdx.x * 4;  // first word of the block in every row
    const int sw = (lane >> 2) & 1;              // half swap of this lane's quad
    uint4* mine = stage + (size_t)y * GPW * 64 + lane * 2;
#pragma unroll
    for (int j = 0; j < GPW; ++j) {
        const int g = y + 8 * j;
        const bool ok = g >= c.gbeg && g < c.gend && lane < c.lanes[g];
        const uint64_t* src = ok ? rows + (c.row0[g] + lane) * c.pitch_words + w0 : rows;
        cp_async16(mine + j * 64 + sw, src, ok ? 16 : 0);  // zero-filled past the group
        cp_async16(mine + j * 64 + (sw ^ 1), src + 2, ok ? 16 : 0);
        cp_async_commit();
    }
    const Transpose32 xp(lane);
    uint32_t nT[4] = {0, 0, 0, 0}, nF[4] = {0, 0, 0, 0}, nU[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < GPW; ++j) {
        const int g = y + 8 * j;
        cp_async_wait_upto(GPW - 1 - j);
        // no branch around the shuffles (they must stay provably converged):
        // groups past G transpose zero-filled rows and store nothing
        const bool live = g >= c.gbeg && g < c.gend;
        const int n = live ? c.lanes[g] : 0;
        const uint4 a = mine[j * 64 + sw], b = mine[j * 64 + (sw ^ 1)];
        const uint32_t tv[4] = {a.x, a.z, b.x, b.z}, sv[4] = {a.y, a.w, b.y, b.w};
        const uint32_t lm = width_mask<uint32_t>(n);
        uint32_t T[4], S[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) { T[k] = tv[k]; S[k] = sv[k]; }
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // eight independent shuffle chains
            T[k] = xp(T[k]);
            S[k] = xp(S[k]);
        }
        LaneEntry<uint32_t>* dst = lane_tab + (int64_t)g * c.vstride + vbase + lane;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int v = (int)vbase + 32 * k + lane;  // num_vars < 2^30
            if (v == 0) { T[k] = 0; S[k] = 0; }  // slot 0 is never set (bitpack.py:110-111)
            const bool sentinel = v == (int)V + 1;   // always False
            if (live && v <= (int)V + 1)
                dst[32 * k] = sentinel ? LaneEntry<uint32_t>{0u, ~0u} : LaneEntry<uint32_t>{T[k], S[k]};
            // AggregateAssignment.from_packed, bitpack.py:156-166 (slot 0 / past V masked below)
            if (T[k] != 0) nT[k] |= 1u << j;
            if ((S[k] & ~T[k]) != 0) nF[k] |= 1u << j;
            if (live && (n == 0 || (~S[k] & lm) != 0)) nU[k] |= 1u << j;
        }
    }
    cp_async_wait_upto(0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        part[0][y][32 * k + lane] = (uint8_t)nT[k];
        part[1][y][32 * k + lane] = (uint8_t)nF[k];
        part[2][y][32 * k + lane] = (uint8_t)nU[k];
    }
    __syncthreads();
    if (t < 128) {
        const int64_t v = vbase + t;
        GW aT = 0, aF = 0, aU = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w)
#pragma unroll
            for (int j = 0; j < GPW; ++j) {
                const GW bit = GW(1) << (w + 8 * j);  // groups past G never set a bit
                if (part[0][w][t] >> j & 1) aT |= bit;
                if (part[1][w][t] >> j & 1) aF |= bit;
                if (part[2][w][t] >> j & 1) aU |= bit;
            }
        if (v >= 1 && v <= V) agg[v] = AggEntry<GW>{aT, aF, aU, GW(0)};
        else if (v == 0) agg[v] = AggEntry<GW>{GW(0), GW(0), GW(0), GW(0)};
        else if (v == V + 1)
            agg[v] = c.sentinel ? AggEntry<GW>{~GW(0), ~GW(0), GW(0), GW(0)} : AggEntry<GW>{GW(0), GW(0), GW(0), GW(0)};
        // polarity statistics for the store's literal placement
        unsigned nt = (v >= 1 && v <= V) ? __popcll((unsigned long long)aT) : 0u;
        unsigned nf = (v >= 1 && v <= V) ? __popcll((unsigned long long)aF) : 0u;
        nt = __reduce_add_sync(0xffffffffu, nt);
        nf = __reduce_add_sync(0xffffffffu, nf);
        if ((t & 31) == 0 && c.polarity) {
            atomicAdd(c.polarity, (unsigned long long)nt);
            atomicAdd(c.polarity + 1, (unsigned long long)nf);
        }
    }
}

// ---------------------------------------------------------------------------
// K3+K4+K5: trigger test, one launch per round.  Persistent grid; one warp
// per tile of 32 clauses of one bucket, one clause per lane.
//
// The kernel is bound by L2 sectors (every table gather touches a 32-byte
// sector: DESIGN.md §4) and by the latency of the gather chains, so:
//  * the first PF literal rows of a warp's next tile are loaded into
//    registers while the current tile is tested (software pipeline);
//  * stage 1 (aggregate filter, engine.py:238-254) gathers the aggregate
//    entries of literals 0-3 together -- literal 0 is the clause's pivot,
//    shared by the pivot-ordered tile, so that gather costs the warp a few
//    sectors -- then two at a time, and stops as soon as every group is
//    negative: the live set (all_false | one_undef) only shrinks, so a zero
//    word is final;
//  * stage 2 (lane test, bitpack.py:120-135) runs per positive group with
//    the same early exit; the clause's activity and engine id are loaded at
//    stage-2 entry.
// Rounds of more than one chunk (engine.py:403-407) run in the same launch:
// a chunk-level aggregate (the 32x32x32 hierarchy of PAPER.md:425, k_top)
// is swept first, and only the chunks it leaves positive get a stage 1.  A
// lane walks its clause's chunks in order, so the reference's "one report
// per (clause, thread)" set (engine.py:462-464) is a register: the tid of
// the last report (a thread's groups are contiguous in round order).
// Every triggering group bumps the clause's activity by inc * popcount (fp64
// round-to-nearest mul then add, no FMA: engine.py:460); the first
// triggering group of each thread emits the report, or every triggering
// group in all-pairs mode (multi_trigger's pair set, bitpack.py:282-300).
// Records collect in a per-warp shared-memory buffer and leave in coalesced
// batches, each reserved with one atomic for exactly its count: the record
// buffer has no holes and needs no compaction pass.

struct BucketDesc {
    const int32_t* lits;
    double* acts;
    const int64_t* ids;
    int32_t size;
    int32_t rank;   // creation rank of the bucket
    int64_t count;
    int64_t tile0;  // first global tile of the bucket
};

// one group of the round, in round order (engine.py:390-399)
struct GroupDesc {
    uint64_t lane_mask;
    int32_t tid;
    int32_t pad;
};

// Host report ring (north_star subsystem 4): k_test writes
// its records straight into page-locked host memory mapped into the device
// address space -- no device record buffer, no copy-out -- and CPU threads
// drain them while the kernel runs (tsg_ring_drain).  A record is two u64
// words, each tagged in its top 16 bits with its lap (position / capacity,
// mod 65535, plus one), so a drainer knows a slot holds this lap's record
// without the slots ever being cleared (an aligned 8-byte store reaches host
// memory whole); drainers publish how many positions they consumed in
// `tail`.  Warps reserve positions with one atomic per record-buffer flush
// and wait (bounded by wait_ns) while the ring is full.
struct RingDesc {
    unsigned long long* slots;                 // host-mapped [cap][2] words; null: ring off
    unsigned long long* pos;                   // device: positions reserved so far (monotone over rounds)
    const volatile unsigned long long* tail;   // host-mapped: positions the drainers consumed
    unsigned long long* fail;                  // host-mapped: set when a flush gave up waiting for room
    unsigned long long mask;                   // cap - 1 (cap a power of two, >= RECBUF)
    unsigned long long wait_ns;                // longest wait for room, per flush
    unsigned long long tail0;                  // the drainers' tail when the launch was queued (a lower
                                               // bound: flushes read the host copy only past it)
    int32_t shift;                             // log2(cap)
};

__host__ __device__ __forceinline__ unsigned long long ring_tag(unsigned long long q, int shift) {
    return (q >> shift) % 65535ull + 1ull;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <class LW, class GW>
struct TestParams {
    const BucketDesc* buckets;
    int32_t nb;
    int32_t n_tiles;                 // the host keeps tiles < 2^30
    const uint8_t* tables;           // the round's table slot: chunk c at tables + c * chunk_stride
    int64_t chunk_stride;
    int64_t lane_off;                // lane table offset inside a chunk (after its aggregate table)
    int64_t vstride;                 // lane-table row length
    const AggEntry<uint32_t>* top;   // chunk-level aggregate (n_chunks > 1; null: every chunk tested)
    int32_t n_chunks, group_width, n_groups, per_bit;  // per_bit: chunks per bit of the top table
    int32_t sentinel;                // num_vars + 1
    const GroupDesc* groups;         // [n_groups]
    double inc;
    void* out;                       // records: tsg_report, or u64 (rec8)
    unsigned long long out_cap;
    unsigned long long* ctr;         // [0] records, [1] aggregate positives, [2] lane triggers,
                                     // [3] (clause, chunk) pairs left positive by the chunk-level sweep, [5] CTAs done
    unsigned long long* pub;         // the round's first run: host-mapped [8] the last CTA publishes ctr to
    int32_t emit_only;               // replay after record-buffer overflow: no activity / counter side effects
    int32_t rec8;                    // 8-byte records engine_id << 37 | group << 32 | lane_mask
    int32_t all_pairs;               // every triggering (clause, group), not the first per thread
    RingDesc ring;                   // host report ring (16-byte records, lane width <= 32), or off
};

#ifndef TSG_PF
#define TSG_PF 8
#endif
constexpr int PF = TSG_PF;     // literal rows prefetched per tile (4..8)
static_assert(PF >= 4 && PF <= 8 && PF % 2 == 0, "PF: 4, 6 or 8 (stage 1 takes rows 4.. in pairs)");
constexpr int TEST_THREADS = 256;
#ifndef TSG_RECBUF  // 128: measured best (64: 0.277 ms, 128: 0.265 ms at C3)
#define TSG_RECBUF 128
#endif
constexpr int RECBUF = TSG_RECBUF;  // records buffered per warp
// dynamic shared memory of k_test: the warps' record buffers
// (+ 16 bytes per warp: the report ring's cached tail)
__host__ __device__ constexpr int test_rec_stride(bool rec8) { return RECBUF * (rec8 ? 8 : 16) + 16; }
__host__ __device__ constexpr int test_smem_bytes(bool rec8) { return (TEST_THREADS / 32) * test_rec_stride(rec8); }

__device__ __forceinline__ int lit_var(int32_t lit) { return lit < 0 ? -lit : lit; }

// Tiles of a warp increase monotonically, so the warp walks the bucket table
// forward: `bi` is the tile's bucket, `nt0` the first tile of bucket bi + 1.
__device__ __forceinline__ void seek_bucket(const BucketDesc* b, int nb, int tile, int& bi, int& nt0) {
    while (tile >= nt0) {
        ++bi;
        nt0 = bi + 1 < nb ? (int)b[bi + 1].tile0 : INT_MAX;
    }
}

// this lane's literal 0 in `tile` of bucket `bd` (literal j at + j * STRIDE)
__device__ __forceinline__ const int32_t* lane_lits(const BucketDesc* bd, int tile, int lane) {
    return bd->lits + (int64_t)(tile - (int)bd->tile0) * bd->size * STRIDE + lane;
}

__device__ __forceinline__ bool lane_active(const BucketDesc* bd, int tile, int lane) {
    return (int64_t)(tile - bd->tile0) * STRIDE + lane < bd->count;
}

// load the first PF literal rows of a tile (this lane's column)
__device__ __forceinline__ void load_rows(const BucketDesc* bd, int tile, int lane, int32_t sentinel,
                                          int32_t (&buf)[PF]) {
    const int32_t* lp = lane_lits(bd, tile, lane);
    const bool act = lane_active(bd, tile, lane);
    const int size = bd->size;
#pragma unroll
    for (int u = 0; u < PF; ++u) buf[u] = (act && u < size) ? ld_lit(lp + u * STRIDE) : sentinel;
}

// Polarity-adjusted (can be False, can be Undef) words of a literal
// (bitpack.py:138-182 seen through a literal, bitpack.py:263-268).
template <class W>
__device__ __forceinline__ void lit_fu(const AggEntry<W>* agg, int32_t lit, W& f, W& u) {
    const AggEntry<W> e = ld_agg(agg + lit_var(lit));
    f = lit < 0 ? e.t : e.f;
    u = e.u;
}

// Stage 1 over one aggregate table (a chunk's groups, or the chunk-level
// table): the live word (all_false | one_undef) of the clause whose first PF
// literals are `r` and whose literal j sits at lp[j * STRIDE].
template <class W, class ROWS>
__device__ __forceinline__ W sweep(const AggEntry<W>* agg, const ROWS& r, const int32_t* lp, int size,
                                   int32_t sentinel) {
    W af = ~W(0), ou = W(0);
    {  // literals 0..3 together: nearly every clause needs them (sentinel past the end)
        W f[4], u[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) lit_fu<W>(agg, r[k], f[k], u[k]);
#pragma unroll
        for (int k = 0; k < 4; ++k) step<W>(af, ou, f[k], u[k]);
    }
#pragma unroll
    for (int h = 4; h < PF; h += 2) {  // then two at a time while any group is live
        if (h >= size || (af | ou) == W(0)) break;
        W f0, u0, f1, u1;
        lit_fu<W>(agg, r[h], f0, u0);
        lit_fu<W>(agg, r[h + 1], f1, u1);
        step<W>(af, ou, f0, u0);
        step<W>(af, ou, f1, u1);
    }
    for (int j = PF; j < size && (af | ou) != W(0); j += 4) {  // the rest, four at a time
        int32_t l[4];
        W f[4], u[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) l[k] = (j + k < size) ? ld_lit_tail(lp + (j + k) * STRIDE) : sentinel;
#pragma unroll
        for (int k = 0; k < 4; ++k) lit_fu<W>(agg, l[k], f[k], u[k]);
#pragma unroll
        for (int k = 0; k < 4; ++k) step<W>(af, ou, f[k], u[k]);
    }
    return af | ou;
}

// one batch of stage-2 literals (lane words for literals h..h+3)
template <class LW, class ROWS>
__device__ __forceinline__ void lane_batch(const LaneEntry<LW>* lt, const ROWS& r, const int32_t* lp, int h, int size,
                                           LW& lf, LW& lo) {
    LaneEntry<LW> e[4];
    int32_t l[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)  // rows past the prefetched ones from memory (L1)
        l[u] = h + u < PF ? r[h + u] : (h + u < size ? ld_lit_tail(lp + (h + u) * STRIDE) : 0);
#pragma unroll
    for (int u = 0; u < 4; ++u)
        if (h + u < size) e[u] = ld_lane(lt + lit_var(l[u]));
#pragma unroll
    for (int u = 0; u < 4; ++u)
        if (h + u < size)
            step<LW>(lf, lo, l[u] < 0 ? (e[u].s & e[u].t) : (e[u].s & ~e[u].t), ~e[u].s);
}

// Stage 2 (assignment_trigger, bitpack.py:120-135) for one group's lane table.
template <class LW, class ROWS>
__device__ __forceinline__ LW lane_test(const LaneEntry<LW>* lt, const ROWS& r, const int32_t* lp, int size) {
    LW lf = ~LW(0), lo = LW(0);
    lane_batch<LW>(lt, r, lp, 0, size, lf, lo);
    if (size > 4 && (lf | lo) != LW(0)) lane_batch<LW>(lt, r, lp, 4, size, lf, lo);
    for (int j = 8; j < size && (lf | lo) != LW(0); ++j) {
        const int32_t l = ld_lit_tail(lp + j * STRIDE);
        const LaneEntry<LW> e = ld_lane(lt + lit_var(l));
        step<LW>(lf, lo, l < 0 ? (e.s & e.t) : (e.s & ~e.t), ~e.s);
    }
    return lf | lo;
}

// The warp's record buffer in shared memory: `n` records (warp-uniform),
// u64 in 8-byte rounds (rec8) else 16-byte tsg_report; flush() reserves
// exactly n slots with one atomic and writes them coalesced.  (A double-
// buffered form that issues the atomic one half-buffer early measured
// slower: profiles/r02_k_test_variants.md.)
struct RecBuf {
    uint32_t off;  // this warp's buffer: byte offset into the dynamic shared memory
    int rec8;
    // (addressed through the shared array itself, not a generic pointer,
    // so the stores are plain STS with no shared-window base recomputed)
    __device__ __forceinline__ unsigned char* buf() const {
        extern __shared__ __align__(16) unsigned char s_rec[];
        return s_rec + off;
    }
    int n = 0;
    // ring form of flush (lane width <= 32, 16-byte records in `buf`)
    __device__ __forceinline__ void flush_ring(unsigned long long* ctr, const RingDesc& r, int lane) {
        unsigned long long base = 0;
        int ok = 1;
        if (lane == 0) {
            // the drainer's progress as last read, kept after this warp's records (test_smem_bytes)
            unsigned long long& tail_seen = *reinterpret_cast<unsigned long long*>(buf() + RECBUF * 16);
            base = atomicAdd(r.pos, (unsigned long long)n);
            atomicAdd(ctr, (unsigned long long)n);
            const unsigned long long cap = r.mask + 1;
            if (base + n > tail_seen + cap) {  // wait for the drainer to free the slots
                const unsigned long long t0 = globaltimer_ns();
                for (;;) {
                    tail_seen = *r.tail;
                    if (base + n <= tail_seen + cap) break;
                    if (*(volatile unsigned long long*)r.fail || globaltimer_ns() - t0 > r.wait_ns) {
                        *(volatile unsigned long long*)r.fail = 1;  // records dropped: the round fails
                        ok = 0;
                        break;
                    }
                    __nanosleep(1000);
                }
            }
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (ok) {
            for (int i = lane; i < n; i += 32) {
                const ulonglong2 rec = reinterpret_cast<const ulonglong2*>(buf())[i];
                const unsigned long long q = base + (unsigned long long)i;
                const unsigned long long tag = ring_tag(q, r.shift) << 48;
                // id | group, lane mask: both words tagged, one 16-byte store (a warp
                // covers whole 128-byte lines; each 8-byte half lands whole)
                reinterpret_cast<ulonglong2*>(r.slots)[q & r.mask] =
                    make_ulonglong2(tag | (rec.x >> 16), tag | ((rec.x & 0xFFFFull) << 32) | (rec.y & 0xFFFFFFFFull));
            }
            // the writers' records reach the system before anything they do
            // after -- in particular before their CTA reports itself done and
            // the launch's last CTA publishes the record count
            __threadfence_system();
        }
        __syncwarp();
        n = 0;
    }
    __device__ __forceinline__ void flush(void* out, unsigned long long cap, unsigned long long* ctr,
                                          const RingDesc& ring, int lane) {
        __syncwarp();
        if (__builtin_expect(ring.slots != nullptr, 0)) {
            flush_ring(ctr, ring, lane);
            return;
        }
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(ctr, (unsigned long long)n);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int i = lane; i < n; i += 32) {
            const unsigned long long q = base + (unsigned long long)i;
            if (q < cap) {  // past the capacity only counted: the host grows the buffer and replays
                if (rec8) reinterpret_cast<uint64_t*>(out)[q] = reinterpret_cast<const uint64_t*>(buf())[i];
                else reinterpret_cast<ulonglong2*>(out)[q] = reinterpret_cast<const ulonglong2*>(buf())[i];
            }
        }
        __syncwarp();
        n = 0;
    }
    // warp-wide: lanes with `has` append `rec`
    __device__ __forceinline__ void append(bool has, ulonglong2 rec, void* out, unsigned long long cap,
                                           unsigned long long* ctr, const RingDesc& ring, int lane) {
        const unsigned b = __ballot_sync(0xffffffffu, has);
        if (has) {
            const int i = n + __popc(b & ((1u << lane) - 1u));
            if (rec8) reinterpret_cast<uint64_t*>(buf())[i] = rec.x;
            else reinterpret_cast<ulonglong2*>(buf())[i] = rec;
        }
        n += __popc(b);
        if (n > RECBUF - 32) flush(out, cap, ctr, ring, lane);
    }
};

// Chunk-level aggregate: bit b of top[v].{t,f,u} = some
// group of a chunk of slot b (chunks b*per_bit .. b*per_bit + per_bit - 1)
// has the bit in its aggregate entry.  Sound: a group that stays positive
// through stage 1 keeps its slot positive here (the recurrence is monotone
// in its inputs).  The always-False sentinel entry stays always False.
template <class GW>
__global__ void k_top(const uint8_t* __restrict__ tables, int64_t chunk_stride, int32_t n_chunks, int32_t per_bit,
                      int64_t nv2, AggEntry<uint32_t>* __restrict__ top) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; v < nv2; v += (int64_t)gridDim.x * blockDim.x) {
        uint32_t t = 0, f = 0, u = 0;
        for (int c = 0; c < n_chunks; ++c) {
            const AggEntry<GW> e = ld_agg(reinterpret_cast<const AggEntry<GW>*>(tables + c * chunk_stride) + v);
            const uint32_t bit = 1u << (c / per_bit);
            if (e.t) t |= bit;
            if (e.f) f |= bit;
            if (e.u) u |= bit;
        }
        top[v] = AggEntry<uint32_t>{t, f, u, 0u};
    }
}

// The current tile's first PF literal rows of this lane's clause (sentinel
// past the clause end and on inactive lanes), in registers, loaded one tile
// ahead.  (A per-warp shared-memory ring filled 1-3 tiles ahead with
// cp.async freed 16 registers -- 4 CTAs per SM -- but measured slower at
// every depth: profiles/r02_k_test_variants.md.)
struct RegRows {
    int32_t r[PF];
    __device__ __forceinline__ int32_t operator[](int u) const { return r[u]; }
};

template <class LW, class GW, bool MULTI>
__global__ void __launch_bounds__(TEST_THREADS, (sizeof(LW) == 8 || sizeof(GW) == 8) ? 2 : TSG_TEST_MIN_BLOCKS)
k_test(const __grid_constant__ TestParams<LW, GW> p) {
    constexpr int WARPS = TEST_THREADS / 32;
    extern __shared__ __align__(16) unsigned char s_rec[];  // [WARPS][RECBUF] records (test_smem_bytes)
    __shared__ unsigned int s_acc[3][WARPS];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = (int)(((int64_t)gridDim.x * TEST_THREADS) >> 5);
    RecBuf rb{(uint32_t)(warp * test_rec_stride(p.rec8)), p.rec8};
    if (lane == 0 && p.ring.slots) *reinterpret_cast<unsigned long long*>(rb.buf() + RECBUF * 16) = p.ring.tail0;
    unsigned int pos_acc = 0, trig_acc = 0, top_acc = 0;
    const uint32_t top_mask = MULTI ? width_mask<uint32_t>((p.n_chunks + p.per_bit - 1) / p.per_bit) : 1u;
    // single-chunk rounds (<= 64 groups): the group table in shared memory
    // (read through group(i): a direct shared-memory access in single-chunk
    // rounds -- a generic pointer would recompute the shared window's base
    // on every stage-2 iteration)
    __shared__ GroupDesc s_groups[MULTI ? 1 : MAXG];
    if constexpr (!MULTI) {
        for (int i = threadIdx.x; i < p.n_groups; i += TEST_THREADS) s_groups[i] = p.groups[i];
        __syncthreads();
    }
    auto group = [&](int i) -> const GroupDesc& {
        if constexpr (MULTI) return p.groups[i];
        else return s_groups[i];
    };

    int tile = (int)(((int64_t)blockIdx.x * TEST_THREADS + threadIdx.x) >> 5);
    int bi = 0, nt0 = 0;
    if (tile < p.n_tiles) {  // first bucket by binary search, then walk forward
        int lo = 0, hi = p.nb - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (p.buckets[mid].tile0 <= tile) lo = mid; else hi = mid - 1;
        }
        bi = lo;
        nt0 = bi + 1 < p.nb ? (int)p.buckets[bi + 1].tile0 : INT_MAX;
    }
    // one tile: test it with its rows in `cur` while the next tile's rows
    // load into `nxt` (unrolling the loop by two over alternating buffers, or
    // an L2 prefetch two tiles ahead, measured no faster:
    // profiles/r02_k_test_variants.md)
    auto tile_step = [&](const RegRows& cur, RegRows& nxt) -> bool {
            const BucketDesc* bd = p.buckets + bi;
            const int ntile = tile + nwarps;
            // software pipeline: the next tile's first rows are in flight while this one is tested
            if (ntile < p.n_tiles) {
                seek_bucket(p.buckets, p.nb, ntile, bi, nt0);
                load_rows(p.buckets + bi, ntile, lane, p.sentinel, nxt.r);
            }
            const int size = bd->size;
            const bool active = lane_active(bd, tile, lane);
            const int32_t* lp = lane_lits(bd, tile, lane);
            // stage-2 state of this lane's clause, across the chunks of the round
            bool loaded = false, touched = false;
            double act = 0.0;
            uint64_t key_hi = 0;
            int last_tid = INT_MIN;
            // stage 1 + stage 2 of chunk c for the lanes with `mine` (warp-uniform call)
            auto test_chunk = [&](const uint8_t* tab, int g0, int G, bool mine) {
                // ---- stage 1: aggregate filter (engine.py:238-254) -----------------
                GW left = GW(0);
                if (mine)
                    left = sweep<GW>(reinterpret_cast<const AggEntry<GW>*>(tab), cur, lp, size, p.sentinel) &
                           width_mask<GW>(G);
                pos_acc += __popcll((unsigned long long)left);
#ifdef TSG_ABL_NO_STAGE2  // ablation timing only (wrong results)
                left = GW(0);
#endif
                if (left != GW(0) && !loaded) {  // stage-2 entry: id and activity of the clause
                    loaded = true;
                    const int slot = (tile - (int)bd->tile0) * STRIDE + lane;
                    key_hi = (uint64_t)bd->ids[slot] << (p.rec8 ? 37 : 16);
                    if (!p.emit_only) act = bd->acts[slot];
                }
                const LaneEntry<LW>* lanes = reinterpret_cast<const LaneEntry<LW>*>(tab + p.lane_off);
                // one triggering group's effects on this lane's clause, in group
                // order: hits, the fp64 bump (engine.py:460), the first
                // triggering group of each thread (or every one) as a record
                auto settle = [&](int g, LW mask, bool& has, ulonglong2& rec) {
                    if (mask == LW(0)) return;
                    const int hits = __popcll((unsigned long long)mask);
                    trig_acc += hits;
                    if (!p.emit_only) {
                        act = __dadd_rn(act, __dmul_rn(p.inc, (double)hits));
                        touched = true;
                    }
                    const int tid = group(g0 + g).tid;
                    if (p.all_pairs || tid != last_tid) {  // first triggering group of its thread
                        last_tid = tid;
                        has = true;
                        const uint64_t grp = (uint64_t)(g0 + g);
                        rec = p.rec8 ? make_ulonglong2(key_hi | (grp << 32) | (uint32_t)mask, 0)
                                     : make_ulonglong2(key_hi | grp, (unsigned long long)mask);
                    }
                };
                // ---- stage 2: exact lane test per positive group --------------------
                // (each lane settles one group per iteration; a task-parallel
                // form -- the tile's (clause, group) pairs spread over all lanes,
                // literal rows by shuffle -- measured slower:
                // profiles/r02_k_test_variants.md)
                while (__any_sync(0xffffffffu, left != GW(0))) {
                    bool has = false;
                    ulonglong2 rec = make_ulonglong2(0, 0);
                    if (left != GW(0)) {
                        const int g = __ffsll((long long)(unsigned long long)left) - 1;
                        left &= left - GW(1);
                        // the group's lane table, addressed once (kept opaque, so the
                        // literals' loads do not each redo the 64-bit g * vstride)
                        const LaneEntry<LW>* lt = lanes + (int64_t)g * p.vstride;
                        asm volatile("" : "+l"(lt));
                        settle(g, lane_test<LW>(lt, cur, lp, size) & (LW)group(g0 + g).lane_mask, has, rec);
                    }
#ifndef TSG_ABL_NO_RECORDS  // ablation timing only (wrong results)
                    rb.append(has, rec, p.out, p.out_cap, p.ctr, p.ring, lane);
#else
                    if (has && rec.x == 1234567) trig_acc += 1;
#endif
                }
            };
            if constexpr (MULTI) {
                // chunk-level sweep first: only the chunks it leaves positive get a stage 1
                const uint32_t cw = !active ? 0u : p.top ? sweep<uint32_t>(p.top, cur, lp, size, p.sentinel) & top_mask : top_mask;
                top_acc += __popc(cw);
                uint32_t wcw = __reduce_or_sync(0xffffffffu, cw);
                while (wcw) {
                    const int b = __ffs(wcw) - 1;
                    wcw &= wcw - 1u;
                    const bool mine = (cw >> b) & 1u;
                    const int c1 = min((b + 1) * p.per_bit, p.n_chunks);
                    for (int c = b * p.per_bit; c < c1; ++c) {
                        const int g0 = c * p.group_width;
                        test_chunk(p.tables + c * p.chunk_stride, g0, min(p.group_width, p.n_groups - g0), mine);
                    }
                }
            } else {
                test_chunk(p.tables, 0, p.n_groups, active);
            }
            if (touched) bd->acts[(tile - (int)bd->tile0) * STRIDE + lane] = act;
            tile = ntile;
            return tile < p.n_tiles;
    };
    RegRows cur, nxt;
    if (tile < p.n_tiles) load_rows(p.buckets + bi, tile, lane, p.sentinel, cur.r);
    while (tile < p.n_tiles) {
        if (!tile_step(cur, nxt)) break;
        cur = nxt;
    }
    if (rb.n) rb.flush(p.out, p.out_cap, p.ctr, p.ring, lane);

    // counters: warp reduce, block reduce, one atomic per block
    pos_acc = __reduce_add_sync(0xffffffffu, pos_acc);
    trig_acc = __reduce_add_sync(0xffffffffu, trig_acc);
    top_acc = __reduce_add_sync(0xffffffffu, top_acc);
    if (lane == 0) { s_acc[0][warp] = pos_acc; s_acc[1][warp] = trig_acc; s_acc[2][warp] = top_acc; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a = 0, t = 0, c = 0;
        for (int i = 0; i < WARPS; ++i) { a += s_acc[0][i]; t += s_acc[1][i]; c += s_acc[2][i]; }
        if (!p.emit_only) {
            if (a) atomicAdd(p.ctr + 1, a);
            if (t) atomicAdd(p.ctr + 2, t);
            if (c) atomicAdd(p.ctr + 3, c);
        }
        // the launch's last CTA hands the counters to the host (the round's
        // first run) and re-zeroes them, or just re-zeroes the CTA count
        __threadfence();
        if (atomicAdd(p.ctr + 5, 1ull) == gridDim.x - 1) {
            __threadfence();
            if (p.pub) {
#pragma unroll
                for (int i = 0; i < 8; ++i) p.pub[i] = atomicExch(p.ctr + i, 0ull);
                __threadfence_system();
            } else {
                atomicExch(p.ctr + 5, 0ull);
            }
        }
    }
}

}  // namespace tsg
