// tsg_sort.cuh -- ordering a round's report records the reference's way on
// the device (engine.py:403-414, 462-464): per destination thread, by
// (chunk, creation rank of the clause's size bucket, engine id, group).
//
// Each record gets a 64-bit key whose fields are packed at widths the host
// computes for the round (destination index | chunk | bucket rank | engine id
// | group in chunk), then a stable LSD radix sort over the key's significant
// bits (8 bits per pass) orders (key, record index) pairs, and the records
// are gathered into per-field output arrays, destination-major.
#pragma once
#include <cstdint>

#include "tsg_device.cuh"

namespace tsg {

constexpr int SORT_THREADS = 256;
constexpr int SORT_ITEMS = 8;                           // items per thread per block
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;    // items per block

// Key layout of one round (host-computed): key = ((((gkey[g] << rank_bits) |
// rank) << id_bits) | eid) << g_bits | g % group_width, where gkey[g] =
// destination index << chunk_bits | chunk of group g.
struct OrderKey {
    const uint64_t* gkey;       // [n_groups]
    const int32_t* size_of_id;  // clause size by engine id (this store)
    const int32_t* rank_of_size;
    int32_t n_sizes;
    int32_t rank_bits, id_bits, g_bits, group_width;
    int32_t rec8;               // records are u64 engine_id << 37 | group << 32 | mask, else tsg_report
};

__device__ __forceinline__ void rec_fields(const void* recs, int rec8, int64_t i, uint64_t& eid, uint32_t& g,
                                           uint64_t& mask) {
    if (rec8) {
        const uint64_t r = reinterpret_cast<const uint64_t*>(recs)[i];
        eid = r >> 37;
        g = (uint32_t)(r >> 32) & 31u;
        mask = (uint32_t)r;
    } else {
        const ulonglong2 r = reinterpret_cast<const ulonglong2*>(recs)[i];
        eid = r.x >> 16;
        g = (uint32_t)(r.x & 0xFFFFu);
        mask = r.y;
    }
}

// keys of records [0, n) (vals = base + i)
__global__ void k_order_keys(const void* __restrict__ recs, int64_t n, int64_t base, OrderKey k,
                             uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t eid, mask;
        uint32_t g;
        rec_fields(recs, k.rec8, i, eid, g, mask);
        const int32_t s = k.size_of_id[eid];
        const uint64_t rank = (uint64_t)(s < k.n_sizes ? k.rank_of_size[s] : 0);
        uint64_t key = (k.gkey[g] << k.rank_bits) | rank;
        key = (key << k.id_bits) | eid;
        key = (key << k.g_bits) | (uint64_t)(g % (uint32_t)k.group_width);
        keys[i] = key;
        vals[i] = (uint32_t)(base + i);
    }
}

// first sorted position of every destination: start[d] for d in [0, n_dest]
// (start[n_dest] = n), from the destination field (key >> dshift) of the
// sorted keys -- each position opens the destinations since its neighbour's
__global__ void k_dest_starts(const uint64_t* __restrict__ keys, int64_t n, int dshift, int32_t n_dest,
                              int64_t* __restrict__ start) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = i < n ? (int64_t)(dshift >= 64 ? 0 : keys[i] >> dshift) : n_dest;
        const int64_t dp = i > 0 ? (int64_t)(dshift >= 64 ? 0 : keys[i - 1] >> dshift) : -1;
        for (int64_t x = dp + 1; x <= d; ++x) start[x] = i;
    }
}

// pass `shift`: per-block 256-bin digit histogram, digit-major [256][nblk]
__global__ void __launch_bounds__(SORT_THREADS) k_sort_hist(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                                             uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t b0 = (int64_t)blockIdx.x * SORT_TILE;
#pragma unroll 4
    for (int r = 0; r < SORT_ITEMS; ++r) {
        const int64_t i = b0 + (int64_t)r * SORT_THREADS + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan of the digit-major histogram [256][nblk] in two kernels:
// block d scans row d in place and leaves its total in rowsum[d]; then every
// row gets the sum of the rows before it added
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* wsum, uint32_t& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        const uint32_t s = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0u;
        uint32_t si = s;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, si, d);
            if (lane >= d) si += o;
        }
        wsum[lane] = si - s;
        if (lane == 31) wsum[32] = si;
    }
    __syncthreads();
    const uint32_t r = wsum[w] + inc - x;
    total = wsum[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(1024) k_scan_rows(uint32_t* __restrict__ hist, int64_t nblk,
                                                     uint32_t* __restrict__ rowsum) {
    __shared__ uint32_t wsum[33];
    uint32_t* row = hist + (int64_t)blockIdx.x * nblk;
    uint32_t carry = 0;
    for (int64_t b = 0; b < nblk; b += 1024) {
        const int64_t i = b + threadIdx.x;
        const uint32_t x = i < nblk ? row[i] : 0u;
        uint32_t total;
        const uint32_t e = block_excl_scan(x, wsum, total);
        if (i < nblk) row[i] = carry + e;
        carry += total;
    }
    if (threadIdx.x == 0) rowsum[blockIdx.x] = carry;
}

__global__ void __launch_bounds__(1024) k_scan_add(uint32_t* __restrict__ hist, int64_t nblk,
                                                    const uint32_t* __restrict__ rowsum) {
    __shared__ uint32_t wsum[33];
    const uint32_t x = threadIdx.x < blockIdx.x ? rowsum[threadIdx.x] : 0u;  // rows before this one (< 256)
    uint32_t total;
    block_excl_scan(x, wsum, total);
    uint32_t* row = hist + (int64_t)blockIdx.x * nblk;
    for (int64_t i = threadIdx.x; i < nblk; i += 1024) row[i] += total;
}

// pass `shift`: stable scatter of (key, val) by digit.  Items of a block are
// taken in SORT_ITEMS rounds of one per thread (item order = round-major,
// then thread order), each ranked among equal digits with warp match +
// per-warp digit counts.  They are first placed in shared memory in digit
// order (the block's own digit histogram, scanned, gives each digit's run),
// then written out run by run, so consecutive threads write consecutive
// output slots -- coalesced, instead of one partial sector per item.
__global__ void __launch_bounds__(SORT_THREADS) k_sort_scatter(const uint64_t* __restrict__ keys,
                                                                const uint32_t* __restrict__ vals, int64_t n,
                                                                int shift, const uint32_t* __restrict__ offs,
                                                                uint64_t* __restrict__ keys_out,
                                                                uint32_t* __restrict__ vals_out) {
    constexpr int WARPS = SORT_THREADS / 32;
    __shared__ uint32_t gbase[256];      // this block's first output slot per digit
    __shared__ uint32_t lbase[256];      // the digit's run in the block's shared tile
    __shared__ uint32_t next[256];       // next free slot of the digit's run
    __shared__ uint32_t wc[WARPS][256];  // per-warp digit counts of the current round
    __shared__ uint32_t wsum[33];
    __shared__ uint64_t skey[SORT_TILE];
    __shared__ uint32_t sval[SORT_TILE];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t b0 = (int64_t)blockIdx.x * SORT_TILE;
    const int cnt = (int)(n - b0 < SORT_TILE ? n - b0 : SORT_TILE);
    next[threadIdx.x] = 0;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < SORT_ITEMS; ++r) {
        const int64_t i = b0 + (int64_t)r * SORT_THREADS + threadIdx.x;
        if (i < n) atomicAdd(&next[(keys[i] >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    uint32_t total;
    const uint32_t ex = block_excl_scan(next[threadIdx.x], wsum, total);
    lbase[threadIdx.x] = ex;
    next[threadIdx.x] = ex;
    gbase[threadIdx.x] = offs[(int64_t)threadIdx.x * gridDim.x + blockIdx.x];
    for (int r = 0; r < SORT_ITEMS; ++r) {
#pragma unroll
        for (int k = 0; k < WARPS; ++k) wc[k][threadIdx.x] = 0;
        __syncthreads();
        const int64_t i = b0 + (int64_t)r * SORT_THREADS + threadIdx.x;
        const bool ok = i < n;
        uint64_t key = 0;
        uint32_t d = 256u + lane;  // out of range items: a digit of their own (never placed)
        if (ok) {
            key = keys[i];
            d = (uint32_t)(key >> shift) & 0xFFu;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int before = __popc(peers & ((1u << lane) - 1u));
        if (ok && before == 0) wc[w][d] = __popc(peers);
        __syncthreads();
        if (ok) {
            uint32_t pos = next[d] + before;
            for (int k = 0; k < w; ++k) pos += wc[k][d];
            skey[pos] = key;
            sval[pos] = vals[i];
        }
        __syncthreads();
        uint32_t t = 0;
#pragma unroll
        for (int k = 0; k < WARPS; ++k) t += wc[k][threadIdx.x];
        next[threadIdx.x] += t;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += SORT_THREADS) {
        const uint64_t key = skey[j];
        const uint32_t d = (uint32_t)(key >> shift) & 0xFFu;
        const uint32_t pos = gbase[d] + (uint32_t)j - lbase[d];
        keys_out[pos] = key;
        vals_out[pos] = sval[j];
    }
}

// the sorted records' fields, destination-major (vals index the records of
// all stores concatenated: store s at [rec_base[s], rec_base[s+1]))
__global__ void k_order_gather(const uint32_t* __restrict__ vals, int64_t n, const void* __restrict__ recs,
                               int rec8, int eid_bytes, int mask_bytes, void* __restrict__ eids,
                               void* __restrict__ masks, int32_t* __restrict__ groups) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t eid, mask;
        uint32_t g;
        rec_fields(recs, rec8, vals[i], eid, g, mask);
        if (eid_bytes == 4) reinterpret_cast<int32_t*>(eids)[i] = (int32_t)eid;
        else reinterpret_cast<int64_t*>(eids)[i] = (int64_t)eid;
        if (mask_bytes == 4) reinterpret_cast<uint32_t*>(masks)[i] = (uint32_t)mask;
        else reinterpret_cast<uint64_t*>(masks)[i] = mask;
        if (groups) groups[i] = (int32_t)g;
    }
}

// clause sizes by engine id for newly added clauses
__global__ void k_set_sizes(const int64_t* __restrict__ ids, const int32_t* __restrict__ sizes, int64_t n,
                            int32_t* __restrict__ size_of_id) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) size_of_id[ids[i]] = sizes[i];
}

}  // namespace tsg
