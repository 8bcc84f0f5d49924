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

__device__ __forceinline__ AggEntry<uint32_t> ld_agg(const AggEntry<uint32_t>* p) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    return {v.x, v.y, v.z, v.w};
}
__device__ __forceinline__ AggEntry<uint64_t> ld_agg(const AggEntry<uint64_t>* p) {
    const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(p));
    const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(p) + 1);
    return {a.x, a.y, b.x, b.y};
}
__device__ __forceinline__ LaneEntry<uint32_t> ld_lane(const LaneEntry<uint32_t>* p) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    return {v.x, v.y};
}
__device__ __forceinline__ LaneEntry<uint64_t> ld_lane(const LaneEntry<uint64_t>* p) {
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p));
    return {v.x, v.y};
}

// Streaming literal load: the clause DB is read once per round, past L1
// (which it would only evict the table lines from).
__device__ __forceinline__ int32_t ld_lit(const int32_t* p) {
    int32_t r;
    asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
// literals past the prefetched rows: through L1 (stage 2 re-reads them)
__device__ __forceinline__ int32_t ld_lit_tail(const int32_t* p) { return __ldg(p); }

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
