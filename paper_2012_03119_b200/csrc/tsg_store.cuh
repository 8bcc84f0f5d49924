// tsg_store.cuh -- clause-store maintenance kernels: append (K6), reduce key
// build (K7), order-preserving compaction (K8), activity scaling (K9), and the
// literal de-interleave used by store views.  Maintenance runs between rounds;
// none of it is on the per-round hot path.
#pragma once
#include <cstdint>

#include "tsg_device.cuh"
#include "../../include/tsg.h"

namespace tsg {

// K6: scatter n clause-major clauses (n x size) into interleaved slots
// [count0, count0+n) of a bucket (engine.py:150-163).
__global__ void k_append(const int32_t* __restrict__ src, int64_t n, int32_t size, int64_t count0,
                         int32_t* __restrict__ dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = n * size;
    for (; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = i / size;
        int32_t j = (int32_t)(i - c * size);
        int64_t slot = count0 + c;
        dst[(slot / STRIDE) * size * STRIDE + (int64_t)j * STRIDE + (slot % STRIDE)] = src[i];
    }
}

// K6 for a whole insert batch: the batch's clauses bucket-major (bucket b's
// at [first, first + k) of the batch, literals clause-major from lit0), each
// appended at slot count0 + local of its bucket with its id, origin, order
// word and initial activity; also the clause size by engine id.
struct AppendDesc {
    int32_t* lits;
    double* acts;
    int64_t* ids;
    int32_t* org;
    uint64_t* order;
    int64_t count0, first, lit0;
    int32_t size, pad;
};

__global__ void k_append_batch(const AppendDesc* __restrict__ d, int32_t nd, int64_t k_total,
                               const int32_t* __restrict__ lits_src, const int64_t* __restrict__ ids_src,
                               const int32_t* __restrict__ org_src, const uint64_t* __restrict__ order_src,
                               double act, int32_t* __restrict__ size_of_id) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; c < k_total; c += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nd - 1;  // the bucket: last descriptor with first <= c
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (d[mid].first <= c) lo = mid; else hi = mid - 1;
        }
        const AppendDesc b = d[lo];
        const int64_t local = c - b.first, slot = b.count0 + local;
        b.ids[slot] = ids_src[c];
        b.org[slot] = org_src[c];
        b.order[slot] = order_src[c];
        b.acts[slot] = act;
        if (size_of_id) size_of_id[ids_src[c]] = b.size;
        const int32_t* src = lits_src + b.lit0 + local * b.size;
        int32_t* dst = b.lits + (slot / STRIDE) * b.size * STRIDE + (slot % STRIDE);
        for (int j = 0; j < b.size; ++j) dst[(int64_t)j * STRIDE] = src[j];
    }
}

__global__ void k_fill_f64(double* p, int64_t n, double v) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

// K9: ClauseStore.scale_activities (engine.py:233-235)
__global__ void k_scale_f64(double* p, int64_t n, double f) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = __dmul_rn(p[i], f);
}

// interleaved -> clause-major in the clause's original literal order
// (lits_at / literal_columns, engine.py:165-182).  A stored clause is laid
// out [pivot][tier-2 literals][the rest], each part in original order; its
// order word says where they came from: bits 58-63 = pivot position + 1
// (0: no pivot), bits 0-57 = original positions of the tier-2 literals.
constexpr int ORDER_MASK_BITS = 58;

__host__ __device__ __forceinline__ uint64_t order_word(int32_t pivot, uint64_t tier2) {
    return ((uint64_t)(pivot + 1) << ORDER_MASK_BITS) | (tier2 & ((1ull << ORDER_MASK_BITS) - 1));
}

__global__ void k_deinterleave(const int32_t* __restrict__ src, const uint64_t* __restrict__ order, int64_t n,
                               int32_t size, int32_t* __restrict__ dst) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        const int32_t* s = src + (c / STRIDE) * size * STRIDE + (c % STRIDE);
        const uint64_t w = order[c];
        const int32_t pivot = (int32_t)(w >> ORDER_MASK_BITS) - 1;
        const uint64_t m = w & ((1ull << ORDER_MASK_BITS) - 1);
        int32_t t2 = pivot >= 0, rest = t2 + __popcll(m);
        for (int32_t j = 0; j < size; ++j) {
            int32_t k;
            if (j == pivot) k = 0;
            else if (j < ORDER_MASK_BITS && ((m >> j) & 1)) k = t2++;
            else k = rest++;
            dst[c * size + j] = s[(int64_t)k * STRIDE];
        }
    }
}

// 16-byte report records -> 12-byte egress records {key, 32-bit lane mask}
// (lane_width <= 32), three 4-byte words each
__global__ void k_pack_records12(const tsg_report* __restrict__ in, int64_t n, uint8_t* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const tsg_report r = in[i];
        uint32_t* o = reinterpret_cast<uint32_t*>(out + i * 12);
        o[0] = (uint32_t)r.key;
        o[1] = (uint32_t)(r.key >> 32);
        o[2] = (uint32_t)r.lane_mask;
    }
}

// Clause lookup by engine id (tsg_get_clauses): every stored slot binary-
// searches the sorted query ids; a hit records (bucket, slot) for its query.
__global__ void k_find_ids(const int64_t* __restrict__ ids, int64_t n, const int64_t* __restrict__ q,
                           const int64_t* __restrict__ qidx, int64_t nq, int64_t part, int64_t* __restrict__ loc) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t id = ids[c];
        int64_t lo = 0, hi = nq;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (q[mid] < id) lo = mid + 1; else hi = mid;
        }
        for (; lo < nq && q[lo] == id; ++lo) loc[qidx[lo]] = (part << 40) | c;
    }
}

// literals of the selected slots in their original order (k_deinterleave for a slot list)
__global__ void k_deinterleave_sel(const int32_t* __restrict__ src, const uint64_t* __restrict__ order,
                                   const int64_t* __restrict__ slots, int64_t n, int32_t size,
                                   int32_t* __restrict__ dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = slots[i];
        const int32_t* s = src + (c / STRIDE) * size * STRIDE + (c % STRIDE);
        const uint64_t w = order[c];
        const int32_t pivot = (int32_t)(w >> ORDER_MASK_BITS) - 1;
        const uint64_t m = w & ((1ull << ORDER_MASK_BITS) - 1);
        int32_t t2 = pivot >= 0, rest = t2 + __popcll(m);
        for (int32_t j = 0; j < size; ++j) {
            int32_t k;
            if (j == pivot) k = 0;
            else if (j < ORDER_MASK_BITS && ((m >> j) & 1)) k = t2++;
            else k = rest++;
            dst[i * size + j] = s[(int64_t)k * STRIDE];
        }
    }
}

// 8-byte egress records: engine_id << 37 | group << 32 | lane_mask (engine
// ids < 2^27, groups < 32, lane width <= 32; checked by the host).
__global__ void k_pack_records8(const tsg_report* __restrict__ in, int64_t n, uint64_t* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const tsg_report r = in[i];
        out[i] = ((r.key >> 16) << 37) | ((r.key & 0x1F) << 32) | (uint32_t)r.lane_mask;
    }
}

// K7: reduce_store's selection (engine.py:482-490) as an exact radix select
// on the 128-bit key (activity bits, engine id) -- non-negative doubles order
// like their IEEE bit patterns and ids are unique, so "the `target` smallest
// keys" is "every key <= the target-th smallest".  The store's slots are laid
// out bucket by bucket in one flat key array, each bucket padded to a
// multiple of KEEP_BLOCK slots; ineligible slots (id >= watermark,
// engine.py:486) and padding carry the key_act NO_KEY.
constexpr uint64_t NO_KEY = ~0ull;  // a NaN with the sign bit: never a stored activity
constexpr int KEEP_BLOCK = 1024;    // compaction block (one slot per thread)

__global__ void k_reduce_keys(const double* __restrict__ acts, const int64_t* __restrict__ ids, int64_t n,
                              int64_t base, int64_t watermark, uint64_t* __restrict__ key_act,
                              uint64_t* __restrict__ key_id, uint8_t* __restrict__ keep,
                              unsigned long long* n_eligible) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long mine = 0;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const bool el = ids[i] < watermark;
        key_act[base + i] = el ? (uint64_t)__double_as_longlong(acts[i]) : NO_KEY;
        key_id[base + i] = (uint64_t)ids[i];
        keep[base + i] = 1;
        mine += el;
    }
    mine = __reduce_add_sync(0xffffffffu, (unsigned)mine);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(n_eligible, mine);
}

// the key's top `bits` bits (the rest zeroed), as (hi, lo)
__device__ __forceinline__ void key_top(uint64_t a, uint64_t id, int bits, uint64_t& hi, uint64_t& lo) {
    if (bits <= 64) {
        hi = bits == 0 ? 0 : a & (~0ull << (64 - bits));
        lo = 0;
    } else {
        hi = a;
        lo = id & (~0ull << (128 - bits));
    }
}

// histogram of the next 8 key bits among eligible keys whose top `bits` bits are (ph, pl)
__global__ void k_select_hist(const uint64_t* __restrict__ key_act, const uint64_t* __restrict__ key_id, int64_t n,
                              uint64_t ph, uint64_t pl, int bits, unsigned long long* __restrict__ hist) {
    __shared__ unsigned int sh[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t a = key_act[i];
        if (a == NO_KEY) continue;
        const uint64_t id = key_id[i];
        uint64_t hi, lo;
        key_top(a, id, bits, hi, lo);
        if (hi != ph || lo != pl) continue;
        const int d = bits < 64 ? (int)((a >> (56 - bits)) & 0xFF) : (int)((id >> (120 - bits)) & 0xFF);
        atomicAdd(&sh[d], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += blockDim.x)
        if (sh[d]) atomicAdd(hist + d, (unsigned long long)sh[d]);
}

// doom every eligible key whose top `bits` bits are <= (ph, pl)
__global__ void k_select_mark(const uint64_t* __restrict__ key_act, const uint64_t* __restrict__ key_id, int64_t n,
                              uint64_t ph, uint64_t pl, int bits, uint8_t* __restrict__ keep,
                              int64_t* __restrict__ doomed_ids, unsigned long long* n_doomed) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t a = key_act[i];
        if (a == NO_KEY) continue;
        uint64_t hi, lo;
        key_top(a, key_id[i], bits, hi, lo);
        if (hi < ph || (hi == ph && lo <= pl)) {
            keep[i] = 0;
            doomed_ids[atomicAdd(n_doomed, 1ull)] = (int64_t)key_id[i];
        }
    }
}

// Order-preserving stream compaction of the flat keep array (K8's slot
// selection): kept slots per KEEP_BLOCK block, then -- with the host's
// exclusive scan of those counts in blk_off -- the flat index of every kept
// slot at its rank.
__global__ void __launch_bounds__(KEEP_BLOCK) k_keep_count(const uint8_t* __restrict__ keep, int32_t* __restrict__ cnt) {
    const int64_t i = (int64_t)blockIdx.x * KEEP_BLOCK + threadIdx.x;
    const int c = __syncthreads_count(keep[i] != 0);
    if (threadIdx.x == 0) cnt[blockIdx.x] = c;
}

__global__ void __launch_bounds__(KEEP_BLOCK) k_keep_select(const uint8_t* __restrict__ keep,
                                                            const int64_t* __restrict__ blk_off,
                                                            int64_t* __restrict__ sel) {
    __shared__ int warp_sum[KEEP_BLOCK / 32];
    const int64_t i = (int64_t)blockIdx.x * KEEP_BLOCK + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const bool k = keep[i] != 0;
    const unsigned b = __ballot_sync(0xffffffffu, k);
    if (lane == 0) warp_sum[w] = __popc(b);
    __syncthreads();
    if (w == 0) {  // exclusive scan of the warp sums
        int x = warp_sum[lane], inc = x;
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += o;
        }
        warp_sum[lane] = inc - x;
    }
    __syncthreads();
    if (k) sel[blk_off[blockIdx.x] + warp_sum[w] + __popc(b & ((1u << lane) - 1u))] = i;
}

// explicit delete: keep[base + i] = ids[i] not in sorted(del)
__global__ void k_mark_deleted(const int64_t* __restrict__ ids, int64_t n, int64_t base,
                               const int64_t* __restrict__ del, int64_t nd, uint8_t* __restrict__ keep,
                               unsigned long long* removed) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long mine = 0;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t x = ids[i];
        int64_t lo = 0, hi = nd;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (del[mid] < x) lo = mid + 1; else hi = mid;
        }
        bool gone = lo < nd && del[lo] == x;
        keep[base + i] = !gone;
        mine += gone;
    }
    for (int d = 16; d > 0; d >>= 1) mine += __shfl_down_sync(0xffffffffu, mine, d);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(removed, mine);
}

// K8: order-preserving compaction, _SizeBucket.compact (engine.py:184-200).
// sel[k] - base = old slot of new slot k (k_keep_select over the bucket's range).
__global__ void k_compact(const int64_t* __restrict__ sel, int64_t base, int64_t kept, int32_t size,
                          const int32_t* __restrict__ lits_in, const double* __restrict__ acts_in,
                          const int64_t* __restrict__ ids_in, const int32_t* __restrict__ org_in,
                          const uint64_t* __restrict__ hm_in,
                          int32_t* __restrict__ lits_out, double* __restrict__ acts_out,
                          int64_t* __restrict__ ids_out, int32_t* __restrict__ org_out,
                          uint64_t* __restrict__ hm_out) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; k < kept; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = sel[k] - base;
        acts_out[k] = acts_in[o];
        ids_out[k] = ids_in[o];
        org_out[k] = org_in[o];
        hm_out[k] = hm_in[o];
        const int32_t* s = lits_in + (o / STRIDE) * size * STRIDE + (o % STRIDE);
        int32_t* d = lits_out + (k / STRIDE) * size * STRIDE + (k % STRIDE);
        for (int j = 0; j < size; ++j) d[(int64_t)j * STRIDE] = s[(int64_t)j * STRIDE];
    }
}

// largest |literal| stored in a bucket's live slots (out-of-range check)
__global__ void k_max_var(const int32_t* __restrict__ lits, int64_t n, int32_t size, unsigned long long* out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long m = 0;
    for (; i < n * size; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = i / size;
        int32_t j = (int32_t)(i - c * size);
        int32_t l = lits[(c / STRIDE) * size * STRIDE + (int64_t)j * STRIDE + (c % STRIDE)];
        unsigned long long v = l < 0 ? (unsigned long long)(-(int64_t)l) : (unsigned long long)l;
        m = v > m ? v : m;
    }
    for (int d = 16; d > 0; d >>= 1) {
        unsigned long long o = __shfl_down_sync(0xffffffffu, m, d);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// int8 snapshot rows -> 2-bit packed rows on the device (tsg_stage_packed_mixed):
// the same words tsg_pack_rows writes on the host -- u64 word k of a row
// holds variables 32k..32k+31, low half (value == 1), high half (value != 0),
// zero past the row -- one thread per word.
__global__ void k_pack_rows(const int8_t* __restrict__ raw, int64_t raw_pitch, int64_t n_rows, int64_t nv1,
                            uint64_t* __restrict__ out, int64_t out_pitch_words, int64_t words) {
    const int64_t total = n_rows * words;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / words, k = i - r * words;
        const int8_t* src = raw + r * raw_pitch + 32 * k;
        uint32_t t = 0, st = 0;
        if (32 * k + 32 <= nv1 && (((uintptr_t)src) & 15) == 0) {
            const uint4 a = *reinterpret_cast<const uint4*>(src), b = *reinterpret_cast<const uint4*>(src + 16);
            const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t eq1 = __vcmpeq4(w[q], 0x01010101u), nz = __vcmpne4(w[q], 0u);  // 0xFF per matching byte
                t |= ((eq1 & 1u) | ((eq1 >> 7) & 2u) | ((eq1 >> 14) & 4u) | ((eq1 >> 21) & 8u)) << (4 * q);
                st |= ((nz & 1u) | ((nz >> 7) & 2u) | ((nz >> 14) & 4u) | ((nz >> 21) & 8u)) << (4 * q);
            }
        } else {
            for (int j = 0; j < 32; ++j) {
                if (32 * k + j >= nv1) break;
                const int8_t v = src[j];
                t |= (uint32_t)(v == 1) << j;
                st |= (uint32_t)(v != 0) << j;
            }
        }
        out[r * out_pitch_words + k] = (uint64_t)t | ((uint64_t)st << 32);
    }
}

}  // namespace tsg
