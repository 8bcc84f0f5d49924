// tsg_device.cuh -- device-side data layout and the trigger recurrence.
//
// HBM layout:
//   * clause store: one bucket per clause size (engine.py:122-163).  Bucket
//     literals are literal-major inside blocks of STRIDE=32 clauses: literal j
//     of slot k lives at data[(k/32)*size*32 + j*32 + k%32], so one warp
//     (one clause per lane) reads every literal row as a single 128-byte line.
//   * per-round tables, per chunk of <= group_width groups:
//       agg  [V+2]      AggEntry<GW>  {can_be_true, can_be_false, can_be_undef}
//       lane [V+2][G]   LaneEntry<LW> {is_true, is_set}   (variable-major)
//     Entry V+1 is the SENTINEL literal: always False on every lane and every
//     group (cbF=all, cbU=0; is_set=all, is_true=0).  It is the identity of
//     the recurrence and pads unrolled loads past the clause end.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tsg {

constexpr int STRIDE = 32;  // clauses per interleave block == warp width

template <class W>
struct alignas(sizeof(W) * 4) AggEntry {
    W t, f, u, pad;
};
template <class W>
struct alignas(sizeof(W) * 2) LaneEntry {
    W t, s;
};

template <class W>
__host__ __device__ __forceinline__ W width_mask(int w) {
    return w >= (int)(sizeof(W) * 8) ? ~W(0) : ((W(1) << w) - W(1));
}

// L2 eviction hints (TSG_L2_HINTS; measured slower, default off): 1 =
// evict_last on the table gathers + evict_first on the literal stream
// (k_test 0.288 vs 0.267 ms), 2 = evict_first on the stream only (0.269).
#ifndef TSG_L2_HINTS
#define TSG_L2_HINTS 0
#endif
__device__ __forceinline__ uint64_t l2_keep_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_stream_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ AggEntry<uint32_t> ld_agg(const AggEntry<uint32_t>* p) {
#if TSG_L2_HINTS == 1
    uint4 v;
    asm("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(l2_keep_policy()));
#else
    uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
#endif
    return {v.x, v.y, v.z, v.w};
}
__device__ __forceinline__ AggEntry<uint64_t> ld_agg(const AggEntry<uint64_t>* p) {
    ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(p));
    ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(p) + 1);
    return {a.x, a.y, b.x, b.y};
}
__device__ __forceinline__ LaneEntry<uint32_t> ld_lane(const LaneEntry<uint32_t>* p) {
#if TSG_L2_HINTS == 1
    uint2 v;
    asm("ld.global.nc.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(l2_keep_policy()));
#else
    uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
#endif
    return {v.x, v.y};
}
__device__ __forceinline__ LaneEntry<uint64_t> ld_lane(const LaneEntry<uint64_t>* p) {
    ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p));
    return {v.x, v.y};
}

// Streaming literal load: the clause DB is read once per round.
__device__ __forceinline__ int32_t ld_lit(const int32_t* p) {
    int32_t r;
#if TSG_L2_HINTS
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(l2_stream_policy()));
#else
    asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r) : "l"(p));
#endif
    return r;
}
// literals past the prefetched rows: through L1 (stage 2 re-reads them), first out of L2
__device__ __forceinline__ int32_t ld_lit_tail(const int32_t* p) {
#if TSG_L2_HINTS
    int32_t r;
    asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(l2_stream_policy()));
    return r;
#else
    return __ldg(p);
#endif
}

__device__ __forceinline__ void or_shared(uint32_t* p, uint32_t v) { atomicOr(p, v); }
__device__ __forceinline__ void or_shared(uint64_t* p, uint64_t v) {
    atomicOr(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

// The recurrence of bitpack.py:131-135 / 263-270, engine.py:249-254:
//   one_undef = (all_false & undef_ok) | (one_undef & is_false)
//   all_false &= is_false
// For stage 1 (aggregate) is_false = can_be_false(lit), undef_ok = can_be_undef;
// for stage 2 (lanes)     is_false = lanes where lit is False, undef_ok = ~is_set.
template <class W>
__device__ __forceinline__ void step(W& af, W& ou, W is_false, W undef_ok) {
    ou = (af & undef_ok) | (ou & is_false);
    af &= is_false;
}

}  // namespace tsg
