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
#ifndef TSG_LANE_TAIL2  // stage-2 literals past the prefetched rows two at a time
#define TSG_LANE_TAIL2 0
#endif
#ifndef TSG_TAIL  // stage-1 gather batch after the first four literals
#define TSG_TAIL 2
#endif
#ifdef TSG_LIT_L1  // literal rows through L1 (default: streamed past L1, keeping it for the tables)
#define LD_LIT(p) __ldg(p)
#else
#define LD_LIT(p) ld_lit(p)
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
constexpr int ENC_MAX_GPW = 8;
#ifndef TSG_ENC_WAIT_ALL
#define TSG_ENC_WAIT_ALL 0
#endif
#ifndef TSG_ENC_PAIR
#define TSG_ENC_PAIR 0
#endif  // groups per warp (G <= 64, 8 warps)

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
    // Two transposes, one shuffle per stage: a lane only ever uses the half
    // of its partner's word the partner discards (the ~keep blocks), so A's
    // discarded blocks and B's, rotated into the keep blocks, share one word.
    __device__ __forceinline__ void pair(uint32_t& a, uint32_t& b) const {
#pragma unroll
        for (int i = 0; i < 2; ++i) {  // byte stages: shuffle + PRMT each
            a = __byte_perm(a, __shfl_xor_sync(0xffffffffu, a, 16 >> i), sel[i]);
            b = __byte_perm(b, __shfl_xor_sync(0xffffffffu, b, 16 >> i), sel[i]);
        }
#pragma unroll
        for (int i = 2; i < 5; ++i) {
            const uint32_t br = __funnelshift_r(b, b, amt[i]);  // B's ~keep blocks onto the keep blocks
            uint32_t p, na, nb;
            asm("lop3.b32 %0, %1, %2, %3, 0xE2;" : "=r"(p) : "r"(br), "r"(keep[i]), "r"(a));  // keep ? br : a
            const uint32_t q = __shfl_xor_sync(0xffffffffu, p, 16 >> i);
            const uint32_t qa = __funnelshift_l(q, q, amt[i]);  // partner's A blocks into place
            asm("lop3.b32 %0, %1, %2, %3, 0xE2;" : "=r"(na) : "r"(a), "r"(keep[i]), "r"(qa));  // keep ? a : qa
            asm("lop3.b32 %0, %1, %2, %3, 0xE2;" : "=r"(nb) : "r"(b), "r"(keep[i]), "r"(q));   // keep ? b : q
            a = na;
            b = nb;
        }
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
    if (TSG_ENC_WAIT_ALL) cp_async_wait_upto(0);  // all groups landed: the compiler may interleave them
    uint32_t nT[4] = {0, 0, 0, 0}, nF[4] = {0, 0, 0, 0}, nU[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < GPW; ++j) {
        const int g = y + 8 * j;
        if (!TSG_ENC_WAIT_ALL) cp_async_wait_upto(GPW - 1 - j);
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
        for (int k = 0; k < 4; ++k) {  // eight independent shuffle chains (paired in the bit stages)
            if (TSG_ENC_PAIR) xp.pair(T[k], S[k]);
            else { T[k] = xp(T[k]); S[k] = xp(S[k]); }
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
// K3+K4+K5: trigger test.  Persistent grid; one warp per tile of 32 clauses
// of one bucket, one clause per lane.
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
//    stage-2 entry, off the report path.
// Every triggering group bumps the clause's activity by inc * popcount (fp64
// round-to-nearest mul then add, no FMA: engine.py:460); the first
// triggering group of each thread emits the report (engine.py:462-464).
// Report slots come from a warp-private chunk refilled by one atomic per
// REPORT_CHUNK slots, reserved for an upper bound (the positive-group
// count); unused slots are written as padding (key = ~0) and squeezed out
// when the records are fetched.

struct BucketDesc {
    const int32_t* lits;
    double* acts;
    const int64_t* ids;
    int32_t size;
    int32_t rank;   // creation rank of the bucket
    int64_t count;
    int64_t tile0;  // first global tile of the bucket
};

template <class LW, class GW>
struct TestParams {
    const BucketDesc* buckets;
    int32_t nb;
    int32_t G;                 // groups in this chunk
    int64_t n_tiles;
    const AggEntry<GW>* agg;
    const void* codes;         // per-literal-code table (shared-memory variant), codes_bytes long
    int64_t codes_bytes;
    const LaneEntry<LW>* lane; // [G][vstride]
    int64_t vstride;
    int32_t sentinel;          // num_vars + 1
    int32_t g0;                // global index of the chunk's first group
    GW group_mask;
    double inc;
    tsg_report* out;
    unsigned long long* ctr;   // [0] slots reserved, [1] aggregate positives, [2] lane triggers, [3] reports
    int64_t out_cap;
    int64_t* carry;            // per-clause "(round, tid) reported" stamp for multi-chunk rounds
    int64_t stamp_base;        // round sequence << 32
    int32_t carry_in_tid;      // first tid of the chunk if it continues from the previous chunk, else -1
    int32_t carry_out_tid;     // last tid of the chunk if it continues into the next chunk, else -1
    int32_t emit_only;         // replay after report-buffer overflow: no activity / counter side effects
    unsigned long long* pub;   // last launch of a round: host-mapped [8] the last CTA publishes ctr to
    int32_t dyn_tiles;         // tiles from the counters `tiles` (DynTiles) instead of a static stride
    int32_t rec8;              // records as 8-byte u64 (st_record)
    unsigned long long* tiles; // [TSG_DYN_NC * DYN_STRIDE] per-launch tile counters (zero between launches)
    const int64_t* slab_tile0; // slab kernel: first tile of each slab (+ end)
    const int32_t* slab_desc0; // slab kernel: first descriptor of each slab (+ end)
    const uint64_t* sched;     // slab kernel: per CTA slab << 32 | rank << 16 | CTAs on the slab
    int32_t n_sched;
    int32_t slab_w;            // slab kernel: variables per slab
    int32_t tid[MAXG];
    LW lane_mask[MAXG];
};

constexpr int PF = 8;  // literal rows prefetched per tile
#ifndef TSG_TEST_THREADS
#define TSG_TEST_THREADS 256
#endif
constexpr int TEST_THREADS = TSG_TEST_THREADS;  // block of the L2-table variant
constexpr int TEST_THREADS_SMEM = 768;  // block of the shared-memory-table variant (one per SM)
constexpr int64_t SMEM_TABLE_MAX = 200 * 1024;
#ifndef TSG_SLAB_THREADS
#define TSG_SLAB_THREADS 768
#endif
constexpr int TEST_THREADS_SLAB = TSG_SLAB_THREADS;  // block of the slab variant (one per SM)
constexpr int64_t SLAB_SMEM_BYTES = 132 * 1024;     // one slab's words: keeps the CTA under the 164 KB carveout,
                                                    // leaving ~92 KB of L1 for in-flight gathers (measured cliff below ~60 KB)

constexpr uint64_t REPORT_PAD = ~0ull;
#ifndef REPORT_CHUNK  // report slots a warp reserves per atomic
#define REPORT_CHUNK 128ull
#endif

__device__ __forceinline__ void st_report(tsg_report* p, uint64_t key, uint64_t mask) {
    *reinterpret_cast<ulonglong2*>(p) = make_ulonglong2(key, mask);
}
// Record i of the round: 16-byte tsg_report, or -- rounds launched for
// 8-byte egress (TestParams::rec8) -- one u64 engine_id << 37 | group << 32 |
// lane_mask written straight from the kernel (half the bytes, no pack pass).
// `hi` is the engine id already shifted for the format.
__device__ __forceinline__ void st_record(tsg_report* out, int rec8, int pos, uint64_t hi, uint32_t group,
                                          uint64_t mask) {
    if (rec8) reinterpret_cast<uint64_t*>(out)[pos] = hi | ((uint64_t)group << 32) | (uint32_t)mask;
    else st_report(out + pos, hi | group, mask);
}
__device__ __forceinline__ void st_pad(tsg_report* out, int rec8, int pos) {
    if (rec8) reinterpret_cast<uint64_t*>(out)[pos] = REPORT_PAD;
    else st_report(out + pos, REPORT_PAD, 0);
}

__device__ __forceinline__ int lit_var(int32_t lit) { return lit < 0 ? -lit : lit; }

// Polarity-adjusted value subset of a literal in every group of the chunk:
// bit g of t / f / u says that some lane of group g makes the literal True /
// False / leaves it Undef (bitpack.py:138-182 seen through a literal,
// bitpack.py:263-268).
template <class GW>
struct Subset {
    GW t, f, u;
};

// Aggregates gathered from the L2-resident table AggEntry[num_vars + 2]:
// one 32-byte sector per lookup; works for any num_vars.
template <class GW>
struct GlobalTable {
    static constexpr bool kSmem = false;
    static constexpr bool kSlab = false;
    const AggEntry<GW>* agg;
    __device__ __forceinline__ Subset<GW> get(int32_t lit) const {
        const AggEntry<GW> e = ld_agg(agg + lit_var(lit));
        return lit < 0 ? Subset<GW>{e.f, e.t, e.u} : Subset<GW>{e.t, e.f, e.u};
    }
};

// Per-literal-code words {can_be_false | can_be_undef << H} in shared memory
// (code = 2 * var + negative): used when 2 * (num_vars + 2) codes fit, i.e.
// small num_vars x groups; stage 1 then needs no L2 gathers at all.
template <class GW, class EW>
struct SmemTable {
    static constexpr bool kSmem = true;
    static constexpr bool kSlab = false;
    static constexpr int H = sizeof(EW) * 4;
    const EW* code;
    __device__ __forceinline__ Subset<GW> get(int32_t lit) const {
        const int c = 2 * lit_var(lit) + (lit < 0);
        const EW a = code[c], b = code[c ^ 1];
        const EW m = (EW)((EW(1) << H) - 1);
        return Subset<GW>{(GW)(b & m), (GW)(a & m), (GW)(a >> H)};  // True for lit = False for ~lit
    }
};

// One variable slab [lo, lo + w) in shared memory (slab kernel): the
// can-be-False word of each literal code and the can-be-Undef word of each
// variable; literals outside the slab are gathered from the L2 table.
template <class GW>
struct SlabTable {
    static constexpr bool kSmem = true;
    static constexpr bool kSlab = true;
    const GW* fc;  // [2 * w]: code 2i = +(lo+i), 2i+1 = -(lo+i)
    const GW* u;   // [w]
    const AggEntry<GW>* agg;
    int32_t lo, w;
    __device__ __forceinline__ bool hot(int32_t lit) const {
        return (uint32_t)(lit_var(lit) - lo) < (uint32_t)w;
    }
    __device__ __forceinline__ void get_hot(int32_t lit, GW& f, GW& uu) const {
        const int i = lit_var(lit) - lo;
        f = fc[2 * i + (lit < 0)];
        uu = u[i];
    }
    __device__ __forceinline__ Subset<GW> get(int32_t lit) const {
        const AggEntry<GW> e = ld_agg(agg + lit_var(lit));
        return lit < 0 ? Subset<GW>{e.f, e.t, e.u} : Subset<GW>{e.t, e.f, e.u};
    }
};

template <class EW>
__global__ void k_codes(const AggEntry<uint32_t>* __restrict__ agg, int64_t nv2, EW* __restrict__ code) {
    constexpr int H = sizeof(EW) * 4;
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; v < nv2; v += (int64_t)gridDim.x * blockDim.x) {
        const AggEntry<uint32_t> e = agg[v];
        const EW m = (EW)((EW(1) << H) - 1);
        code[2 * v] = (EW)((EW)(e.f & m) | (EW)((EW)(e.u & m) << H));      // +v is False where v is False
        code[2 * v + 1] = (EW)((EW)(e.t & m) | (EW)((EW)(e.u & m) << H));  // -v is False where v is True
    }
}


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
    return (tile - bd->tile0) * STRIDE + lane < bd->count;
}

// load the first PF literal rows of a tile (this lane's column)
__device__ __forceinline__ void load_rows(const BucketDesc* bd, int tile, int lane, int32_t sentinel,
                                          int32_t (&buf)[PF]) {
    const int32_t* lp = lane_lits(bd, tile, lane);
    const bool act = lane_active(bd, tile, lane);
    const int size = bd->size;
#pragma unroll
    for (int u = 0; u < PF; ++u) buf[u] = (act && u < size) ? LD_LIT(lp + u * STRIDE) : sentinel;
}

template <class GW, class TAB, int THREADS>
constexpr size_t test_smem_bytes(int64_t codes_bytes) {
    return TAB::kSmem ? (size_t)codes_bytes : 16;
}

// The current tile's first PF literal rows of this lane's clause.
// RegRows keeps them in registers (indexed with compile-time positions);
// SmemRows keeps them in a per-warp shared-memory buffer [PF][32] so the slab
// kernel can index them with lane-dependent positions (one LDS, no select
// chains, no local memory).
struct RegRows {
    int32_t r[PF];
    __device__ __forceinline__ int32_t get(int j) const { return r[j]; }
    __device__ __forceinline__ void take(const int32_t (&nxt)[PF]) {
#pragma unroll
        for (int u = 0; u < PF; ++u) r[u] = nxt[u];
    }
};
struct SmemRows {
    int32_t* buf;  // this warp's [PF][32] buffer, offset by lane
    __device__ __forceinline__ int32_t get(int j) const { return buf[j * 32]; }
    __device__ __forceinline__ void take(const int32_t (&nxt)[PF]) {
        __syncwarp();
#pragma unroll
        for (int u = 0; u < PF; ++u) buf[u * 32] = nxt[u];
        __syncwarp();
    }
};

// one batch of stage-2 literals (lane words of group g for literals h..h+3)
template <class LW, class ROWS>
__device__ __forceinline__ void lane_batch(const LaneEntry<LW>* lt, const ROWS& rows, int h, int size, LW& lf,
                                           LW& lo) {
    LaneEntry<LW> e[4];
    int32_t l[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) l[u] = rows.get(h + u);
#pragma unroll
    for (int u = 0; u < 4; ++u)
        if (h + u < size) e[u] = ld_lane(lt + lit_var(l[u]));
#pragma unroll
    for (int u = 0; u < 4; ++u)
        if (h + u < size)
            step<LW>(lf, lo, l[u] < 0 ? (e[u].s & e[u].t) : (e[u].s & ~e[u].t), ~e[u].s);
}

// Per-warp running state of the tile loop: the warp's report-slot chunk
// [cpos, cend) and its counter accumulators.
struct WarpAcc {
    int cpos = 0, cend = 0;  // report slots (the host keeps out_cap < 2^31)
    unsigned int pos = 0, trig = 0, rep = 0;
};

#ifndef TSG_COLD0  // literals in the first cold gather batch of the slab kernel
#define TSG_COLD0 3
#endif

// Stage 1 of the slab kernel for one clause: the hot prefix (literals whose
// variable lies in the CTA's slab, stored first) is looked up in shared
// memory; the cold rest is gathered from the L2-resident table in batches
// aligned to each lane's own first cold position (TSG_COLD0 literals, then
// 2 at a time) while any group is live, so a warp needs only as many L2
// round trips as its lanes' longest chain.
template <class LW, class GW>
__device__ __forceinline__ void stage1_slab(const TestParams<LW, GW>& p, const SlabTable<GW>& tab,
                                            const SmemRows& rows, const int32_t* lp, int size, GW& af, GW& ou) {
    auto lit_at = [&](int i) -> int32_t {
        if (i >= size) return p.sentinel;
        return i < PF ? rows.get(i) : __ldg(lp + i * STRIDE);
    };
    int hp = 0;  // hot prefix length
    while (hp < size) {
        const int32_t l = lit_at(hp);
        if (!tab.hot(l)) break;
        GW f, uu;
        tab.get_hot(l, f, uu);
        step<GW>(af, ou, f, uu);
        ++hp;
    }
    int j = hp;  // next cold position of this lane
    if (j < size && (af | ou) != GW(0)) {
        int32_t l[TSG_COLD0];
#pragma unroll
        for (int k = 0; k < TSG_COLD0; ++k) l[k] = lit_at(j + k);
        Subset<GW> sb[TSG_COLD0];
#pragma unroll
        for (int k = 0; k < TSG_COLD0; ++k) sb[k] = tab.get(l[k]);
#pragma unroll
        for (int k = 0; k < TSG_COLD0; ++k) step<GW>(af, ou, sb[k].f, sb[k].u);
        j += TSG_COLD0;
        while (j < size && (af | ou) != GW(0)) {
            const int32_t l0 = lit_at(j), l1 = lit_at(j + 1);
            const Subset<GW> s0 = tab.get(l0), s1 = tab.get(l1);
            step<GW>(af, ou, s0.f, s0.u);
            step<GW>(af, ou, s1.f, s1.u);
            j += 2;
        }
    }
}

// Tile sources (warp-uniform, strictly increasing per warp; -1 = done).
// Warps take tiles one at a time from TSG_DYN_NC per-launch counters
// (counter c hands out tiles c, c + NC, c + 2 NC, ...; warp w uses counter
// w % NC), so SMs that run faster -- the two dies' L2 distances differ --
// take more tiles instead of idling at the end of a static share.  The
// atomic for the tile after next is issued when `next` returns, so its
// latency overlaps a whole tile.
#ifndef TSG_DYN_NC
#define TSG_DYN_NC 8
#endif
constexpr int DYN_STRIDE = 32;  // u64 words between counters (separate L2 lines)
struct DynTiles {
    unsigned long long* ctr;  // this warp's counter
    int c, end;
    unsigned long long ahead = 0;  // lane 0: the next k, in flight
    bool primed = false;
    __device__ __forceinline__ int next(int lane) {
        if (!primed) {
            primed = true;
            if (lane == 0) ahead = atomicAdd(ctr, 1ull);
        }
        const unsigned long long k = __shfl_sync(0xffffffffu, ahead, 0);
        const long long t = (long long)c + (long long)TSG_DYN_NC * (long long)k;
        if (t >= end) return -1;
        if (lane == 0) ahead = atomicAdd(ctr, 1ull);
        return (int)t;
    }
};

struct StrideTiles {  // tiles t, t + step, ... < end
    int t, step, end;  // tile indices (the host keeps n_tiles < 2^31)
    bool started = false;
    __device__ __forceinline__ int next(int) {
        if (started) t += step;
        started = true;
        return t < end ? t : -1;
    }
};
// The tile loop shared by every k_test variant (one clause per lane).
// `descs[0, nb)` covers every tile the source hands out (global memory, or
// the slab's share staged in shared memory).
template <class LW, class GW, class TAB, class SRC, class ROWS>
__device__ __forceinline__ void test_tiles(const TestParams<LW, GW>& p, const TAB& tab, const BucketDesc* descs,
                                           int nb, SRC& src, ROWS& cur, int lane, WarpAcc& acc) {
    int tile = src.next(lane);
    if (tile < 0) return;
    int bi = 0;
    int nt0 = 0;
    {  // first bucket by binary search, then walk forward
        int lo = 0, hi = nb - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (descs[mid].tile0 <= tile) lo = mid; else hi = mid - 1;
        }
        bi = lo;
        nt0 = bi + 1 < nb ? (int)descs[bi + 1].tile0 : INT_MAX;
    }
    int32_t nxt[PF];
    load_rows(descs + bi, tile, lane, p.sentinel, nxt);
    cur.take(nxt);

    while (tile >= 0) {
        const BucketDesc* bd = descs + bi;
        // software pipeline: the next tile's first rows are in flight while this one is tested
        const int ntile = src.next(lane);
        if (ntile >= 0) {
            seek_bucket(descs, nb, ntile, bi, nt0);
            load_rows(descs + bi, ntile, lane, p.sentinel, nxt);
        }
        const int size = bd->size;
        const bool active = lane_active(bd, tile, lane);

        // ---- stage 1: aggregate filter (engine.py:238-254) -----------------
        GW af = ~GW(0), ou = GW(0);
        if (active) {
            if constexpr (TAB::kSlab) {
                stage1_slab<LW, GW>(p, tab, cur, lane_lits(bd, tile, lane), size, af, ou);
            } else {
                {  // literals 0..3 together: nearly every clause needs them
                    Subset<GW> s[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) s[u] = tab.get(cur.get(u));
#pragma unroll
                    for (int u = 0; u < 4; ++u) step<GW>(af, ou, s[u].f, s[u].u);
                }
#pragma unroll
                for (int h = 4; h < PF; h += TSG_TAIL) {  // then batches of TSG_TAIL while any group is live
                    if (h >= size || (af | ou) == GW(0)) break;
                    Subset<GW> s[TSG_TAIL];
#pragma unroll
                    for (int u = 0; u < TSG_TAIL; ++u) s[u] = tab.get(cur.get(h + u));
#pragma unroll
                    for (int u = 0; u < TSG_TAIL; ++u) step<GW>(af, ou, s[u].f, s[u].u);
                }
                if (size > PF && (af | ou) != GW(0)) {
                    const int32_t* lp = lane_lits(bd, tile, lane);
                    for (int j = PF; j < size && (af | ou) != GW(0); j += 4) {
                        int32_t l[4];
                        Subset<GW> s[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) l[u] = (j + u < size) ? ld_lit_tail(lp + (j + u) * STRIDE) : p.sentinel;
#pragma unroll
                        for (int u = 0; u < 4; ++u) s[u] = tab.get(l[u]);
#pragma unroll
                        for (int u = 0; u < 4; ++u) step<GW>(af, ou, s[u].f, s[u].u);
                    }
                }
            }
        }
        const GW word = active ? ((af | ou) & p.group_mask) : GW(0);

        // ---- report slot reservation from the warp's chunk ------------------
        const int ub = __popcll((unsigned long long)word);
        int incl = ub;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int o = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += o;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        if (total) {
            if (acc.cpos + total > acc.cend) {  // chunk exhausted: pad its tail, take a new one
                for (int q = acc.cpos + lane; q < acc.cend; q += 32)
                    if (q < p.out_cap) st_pad(p.out, p.rec8, q);
                const unsigned long long want = total > REPORT_CHUNK ? (unsigned long long)total : REPORT_CHUNK;
                unsigned long long base = 0;
                if (lane == 31) base = atomicAdd(p.ctr, want);
                acc.cpos = (int)__shfl_sync(0xffffffffu, base, 31);
                acc.cend = acc.cpos + (int)want;
            }
            int pos = acc.cpos + incl - ub;
            const int pend = pos + ub;
            acc.cpos += total;

            // ---- stage 2: exact lane test per positive group (bitpack.py:120-135)
            if (word) {
                acc.pos += ub;
                const int slot = (tile - (int)bd->tile0) * STRIDE + lane;
                double act = 0.0;
                if (!p.emit_only) act = bd->acts[slot];
                const uint64_t key_hi = (uint64_t)bd->ids[slot] << (p.rec8 ? 37 : 16);  // issued early: off the report's path
                bool touched = false;
                int last_tid = INT_MIN;
                GW left = word;
                // the first triggering group of each thread emits the report
                // (engine.py:462); every triggering group bumps the activity
                // in group order (engine.py:460, fp64 mul then add, no FMA)
                auto settle = [&](int g, LW mask) {
                    if (!mask) return;
                    const int hits = __popcll((unsigned long long)mask);
                    acc.trig += hits;
                    if (!p.emit_only) {
                        act = __dadd_rn(act, __dmul_rn(p.inc, (double)hits));
                        touched = true;
                    }
                    const int tid = p.tid[g];
                    if (tid != last_tid) {
                        last_tid = tid;
                        bool dup = false;
                        if (tid == p.carry_in_tid)
                            dup = p.carry[bd->tile0 * STRIDE + slot] == (p.stamp_base | (uint32_t)tid);
                        if (!dup) {
                            if (pos < p.out_cap) st_record(p.out, p.rec8, pos, key_hi, (uint32_t)(p.g0 + g), (uint64_t)mask);
                            ++pos;
                            ++acc.rep;
                        }
                    }
                };
                auto lane_tail = [&](const LaneEntry<LW>* lt, LW& lf, LW& lo2) {
                    if (size > PF && (lf | lo2) != LW(0)) {
                        const int32_t* lp = lane_lits(bd, tile, lane);
#if TSG_LANE_TAIL2
                        for (int j = PF; j < size && (lf | lo2) != LW(0); j += 2) {  // two lane gathers in flight
                            const int32_t l0 = ld_lit_tail(lp + j * STRIDE);
                            const int32_t l1 = j + 1 < size ? ld_lit_tail(lp + (j + 1) * STRIDE) : p.sentinel;
                            const LaneEntry<LW> e0 = ld_lane(lt + lit_var(l0)), e1 = ld_lane(lt + lit_var(l1));
                            step<LW>(lf, lo2, l0 < 0 ? (e0.s & e0.t) : (e0.s & ~e0.t), ~e0.s);
                            step<LW>(lf, lo2, l1 < 0 ? (e1.s & e1.t) : (e1.s & ~e1.t), ~e1.s);
                        }
#else
                        for (int j = PF; j < size && (lf | lo2) != LW(0); ++j) {
                            const int32_t l = ld_lit_tail(lp + j * STRIDE);
                            const LaneEntry<LW> e = ld_lane(lt + lit_var(l));
                            step<LW>(lf, lo2, l < 0 ? (e.s & e.t) : (e.s & ~e.t), ~e.s);
                        }
#endif
                    }
                };
                while (left) {
                    const int g = __ffsll((long long)(unsigned long long)left) - 1;
                    left &= left - GW(1);
                    const LaneEntry<LW>* lt = p.lane + (int64_t)g * p.vstride;
                    LW lf = ~LW(0), lo2 = LW(0);
                    lane_batch<LW>(lt, cur, 0, size, lf, lo2);
                    if (size > 4 && (lf | lo2) != LW(0)) lane_batch<LW>(lt, cur, 4, size, lf, lo2);
                    lane_tail(lt, lf, lo2);
                    settle(g, (lf | lo2) & p.lane_mask[g]);
                }
                if (touched) bd->acts[slot] = act;
                if (p.carry_out_tid >= 0 && last_tid == p.carry_out_tid)
                    p.carry[bd->tile0 * STRIDE + slot] = p.stamp_base | (uint32_t)last_tid;
                for (; pos < pend; ++pos)  // padding for reserved-but-unused slots
                    if (pos < p.out_cap) st_pad(p.out, p.rec8, pos);
            }
        }
        if (ntile >= 0) cur.take(nxt);
        tile = ntile;
    }
}

// pad the warp's last chunk; counters: warp reduce, block reduce, one atomic per block
template <class LW, class GW, int WARPS>
__device__ __forceinline__ void finish_block(const TestParams<LW, GW>& p, WarpAcc& acc, int lane, int warp,
                                             unsigned int (&s_acc)[3][WARPS]) {
    for (int q = acc.cpos + lane; q < acc.cend; q += 32)
        if (q < p.out_cap) st_pad(p.out, p.rec8, q);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        acc.pos += __shfl_down_sync(0xffffffffu, acc.pos, d);
        acc.trig += __shfl_down_sync(0xffffffffu, acc.trig, d);
        acc.rep += __shfl_down_sync(0xffffffffu, acc.rep, d);
    }
    if (lane == 0) { s_acc[0][warp] = acc.pos; s_acc[1][warp] = acc.trig; s_acc[2][warp] = acc.rep; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a = 0, bb = 0, r = 0;
        for (int i = 0; i < WARPS; ++i) { a += s_acc[0][i]; bb += s_acc[1][i]; r += s_acc[2][i]; }
        if (r) atomicAdd(p.ctr + 3, r);
        if (!p.emit_only) {
            if (a) atomicAdd(p.ctr + 1, a);
            if (bb) atomicAdd(p.ctr + 2, bb);
        }
        // the launch's last CTA re-zeroes the tile counters and the CTA count
        // [5]; on a round's last launch it also hands the counters to the
        // host and re-zeroes them
        __threadfence();
        if (atomicAdd(p.ctr + 5, 1ull) == gridDim.x - 1) {
            __threadfence();
            if (p.tiles)
                for (int c = 0; c < TSG_DYN_NC; ++c) atomicExch(p.tiles + c * DYN_STRIDE, 0ull);
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

// Grid-stride variant: persistent warps over all tiles; the aggregate table
// is gathered from L2 (GlobalTable) or held whole in shared memory (SmemTable).
template <class LW, class GW, class TAB, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_test(const __grid_constant__ TestParams<LW, GW> p) {
    constexpr int WARPS = THREADS / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ unsigned int s_acc[3][WARPS];
    TAB tab;
    if constexpr (TAB::kSmem) {  // per-block copy of the literal-code table
        const uint4* src = reinterpret_cast<const uint4*>(p.codes);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (int64_t i = threadIdx.x; i < p.codes_bytes / 16; i += THREADS) dst[i] = __ldg(src + i);
        __syncthreads();
        tab.code = reinterpret_cast<decltype(tab.code)>(smem);
    } else {
        tab.agg = p.agg;
    }
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
    WarpAcc acc;
    RegRows rows;
    if (p.dyn_tiles) {
        const int gw = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
        const int c = gw % TSG_DYN_NC;
        DynTiles src{p.tiles + c * DYN_STRIDE, c, (int)p.n_tiles};
        test_tiles<LW, GW, TAB>(p, tab, p.buckets, p.nb, src, rows, lane, acc);
    } else {
        StrideTiles src{(int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), nwarps, (int)p.n_tiles};
        test_tiles<LW, GW, TAB>(p, tab, p.buckets, p.nb, src, rows, lane, acc);
    }
    finish_block<LW, GW, WARPS>(p, acc, lane, warp, s_acc);
}

// Slab variant: one CTA per SM.  The host schedule gives
// every CTA one slab and its rank among the n CTAs sharing that slab (n
// proportional to the slab's tiles).  The CTA stages the slab's aggregate
// words in shared memory (can-be-False word per literal code, can-be-Undef
// word per variable) plus the slab's tile descriptors, then its warps walk
// the slab's tiles interleaved with the other CTAs of the slab
// (tile = first + rank * WARPS + warp + k * n * WARPS), which mixes short-
// and long-clause tiles evenly over the CTAs.  sched[c] = slab << 32 |
// rank << 16 | n; a CTA index beyond the schedule picks up entries c + grid...
constexpr int SLAB_DESC_MAX = 80;  // descriptors staged in shared memory (else read from global)

template <class LW, class GW, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) k_test_slab(const __grid_constant__ TestParams<LW, GW> p) {
    constexpr int WARPS = THREADS / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ unsigned int s_acc[3][WARPS];
    __shared__ BucketDesc s_desc[SLAB_DESC_MAX];
    __shared__ int32_t s_rows[WARPS][PF][32];
    SlabTable<GW> tab;
    tab.fc = reinterpret_cast<GW*>(smem);
    tab.u = tab.fc + 2 * (int64_t)p.slab_w;
    tab.agg = p.agg;
    tab.w = p.slab_w;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    WarpAcc acc;
    for (int c = blockIdx.x; c < p.n_sched; c += gridDim.x) {
        const uint64_t e = p.sched[c];
        const int s = (int)(e >> 32), rank = (int)((e >> 16) & 0xFFFF), n = (int)(e & 0xFFFF);
        const int64_t lo = (int64_t)s * p.slab_w;
        const int d0 = p.slab_desc0[s], nd = p.slab_desc0[s + 1] - d0;
        __syncthreads();  // the previous entry's table and descriptors are no longer read
        GW* fc = const_cast<GW*>(tab.fc);
        GW* us = const_cast<GW*>(tab.u);
        for (int i = threadIdx.x; i < p.slab_w; i += THREADS) {
            const int64_t v = lo + i;
            AggEntry<GW> ae{~GW(0), ~GW(0), GW(0), GW(0)};
            if (v <= p.sentinel) ae = ld_agg(p.agg + v);
            fc[2 * i] = ae.f;      // +v is False where v can be False
            fc[2 * i + 1] = ae.t;  // -v is False where v can be True
            us[i] = ae.u;
        }
        const bool staged = nd <= SLAB_DESC_MAX;
        if (staged)
            for (int i = threadIdx.x; i < nd; i += THREADS) s_desc[i] = p.buckets[d0 + i];
        __syncthreads();
        tab.lo = (int32_t)lo;
        StrideTiles src{(int)p.slab_tile0[s] + rank * WARPS + warp, n * WARPS, (int)p.slab_tile0[s + 1]};
        SmemRows rows{&s_rows[warp][0][lane]};
        test_tiles<LW, GW, SlabTable<GW>>(p, tab, staged ? s_desc : p.buckets + d0, nd, src, rows, lane, acc);
    }
    finish_block<LW, GW, WARPS>(p, acc, lane, warp, s_acc);
}

}  // namespace tsg
