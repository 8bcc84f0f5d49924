// tsg_kernels.cuh -- the hot-path kernels (sm_100a).
//
//   K1+K2  k_encode        int8 snapshots -> lane words + aggregates   (bitpack.py:81-117, 152-167, 211-244)
//   K3+K4+K5 k_test        two-stage trigger test, report emission,
//                          activity bump, counters                      (engine.py:238-254, 437-467)
//
// Both are HBM/L2-bound integer kernels; DESIGN.md §4 gives their rooflines.
#pragma once
#include <cstdint>
#include <climits>

#include "tsg_device.cuh"
#include "../../include/tsg.h"

namespace tsg {

constexpr int MAXG = 64;

// ---------------------------------------------------------------------------
// K1+K2: encoder.  Block = 32 x 8 threads covers 128 variables of one chunk.
// Thread (x, y) owns variables 4x..4x+3 of the tile and groups y, y+8, ...;
// for each group it reads the group's lane rows as one u32 (4 variables) per
// row -- every warp load is one coalesced 128-byte segment of a row -- and
// turns bytes into lane bits with SIMD byte compares.  Aggregate bits are
// OR-reduced across groups in shared memory.

struct EncodeChunk {
    int32_t G;               // groups in the chunk
    int32_t num_vars;
    int64_t pitch;           // bytes between rows (multiple of 4)
    int64_t row0[MAXG];      // first row of each group
    int32_t lanes[MAXG];     // rows (lanes) of each group
};

template <class LW, class GW>
__global__ void __launch_bounds__(256) k_encode(const int8_t* __restrict__ rows, const EncodeChunk c,
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
#pragma unroll 4
            for (int i = 0; i < n; ++i) {
                uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(base + (int64_t)i * c.pitch));
                uint32_t e1 = __vcmpeq4(w, 0x01010101u);  // byte == TRUE
                uint32_t nz = __vcmpne4(w, 0u);           // byte != UNDEF
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    tw[b] |= (LW)((e1 >> (8 * b)) & 1u) << i;
                    sw[b] |= (LW)((nz >> (8 * b)) & 1u) << i;
                }
            }
        }
        const LW lm = width_mask<LW>(n);
        const GW bit = GW(1) << g;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t v = v0 + b;
            if (v <= V) {
                LW tv = v == 0 ? LW(0) : tw[b];
                LW sv = v == 0 ? LW(0) : sw[b];
                lane[v * c.G + g] = LaneEntry<LW>{tv, sv};
                if (v != 0) {
                    // AggregateAssignment.from_packed, bitpack.py:156-166
                    if (tv != 0) or_shared(&sT[4 * x + b], bit);
                    if ((sv & ~tv) != 0) or_shared(&sF[4 * x + b], bit);
                    if (n == 0 || (~sv & lm) != 0) or_shared(&sU[4 * x + b], bit);
                }
            } else if (v == V + 1) {
                lane[v * c.G + g] = LaneEntry<LW>{LW(0), ~LW(0)};  // sentinel: always False
            }
        }
    }
    __syncthreads();
    if (t < 128) {
        const int64_t v = vbase + t;
        if (v <= V) agg[v] = AggEntry<GW>{sT[t], sF[t], sU[t], GW(0)};
        else if (v == V + 1) agg[v] = AggEntry<GW>{~GW(0), ~GW(0), GW(0), GW(0)};
    }
}

// ---------------------------------------------------------------------------
// K3+K4+K5: trigger test.  Persistent grid; one warp per tile of 32 clauses
// of one bucket, one clause per lane.
//
// Stage 1 (aggregate filter, engine.py:238-254) walks the clause's literals
// four at a time (four coalesced literal-row loads, then four L2 gathers into
// the aggregate table) and stops as soon as every group is negative: the
// live set (all_false | one_undef) only shrinks, so a zero word is final and
// the remaining literals cannot change the result.
// Stage 2 (lane test, bitpack.py:120-135) runs per positive group in
// ascending order with the same early exit.  Every triggering group bumps the
// clause's activity by inc * popcount (fp64, explicit round-to-nearest ops,
// no FMA: engine.py:460); the first triggering group of each thread emits the
// report (engine.py:462-464).  Records are allocated with one atomic per warp.

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
    const LaneEntry<LW>* lane;
    int32_t sentinel;          // num_vars + 1
    int32_t g0;                // global index of the chunk's first group
    GW group_mask;
    double inc;
    tsg_report* out;
    unsigned long long* ctr;   // [0] records, [1] aggregate positives, [2] lane triggers
    int64_t out_cap;
    int64_t* carry;            // per-clause "(round, tid) reported" stamp for multi-chunk rounds
    int64_t stamp_base;        // round sequence << 32
    int32_t carry_in_tid;      // first tid of the chunk if it continues from the previous chunk, else -1
    int32_t carry_out_tid;     // last tid of the chunk if it continues into the next chunk, else -1
    int32_t emit_only;         // replay after report-buffer overflow: no activity / counter side effects
    int32_t tid[MAXG];
    LW lane_mask[MAXG];
};

template <class LW, class GW>
__global__ void __launch_bounds__(256) k_test(const __grid_constant__ TestParams<LW, GW> p) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long pos_acc = 0, trig_acc = 0;
    LW masks[MAXG];

    for (int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; tile < p.n_tiles;
         tile += nwarps) {
        int lo = 0, hi = p.nb - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (p.buckets[mid].tile0 <= tile) lo = mid; else hi = mid - 1;
        }
        const BucketDesc* bd = p.buckets + lo;
        const int size = bd->size;
        const int64_t blk = tile - bd->tile0;
        const int64_t slot = blk * STRIDE + lane;
        const bool active = slot < bd->count;
        const int32_t* lp = bd->lits + blk * (int64_t)size * STRIDE + lane;

        // ---- stage 1: aggregate filter -------------------------------------
        GW af = ~GW(0), ou = GW(0);
        if (active) {
            for (int j = 0; j < size; j += 4) {
                int32_t l[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) l[u] = (j + u < size) ? ld_lit(lp + (j + u) * STRIDE) : p.sentinel;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int32_t lit = l[u];
                    const AggEntry<GW> e = ld_agg(p.agg + (lit < 0 ? -lit : lit));
                    step<GW>(af, ou, lit < 0 ? e.t : e.f, e.u);
                }
                if ((af | ou) == GW(0)) break;
            }
        }
        const GW word = active ? ((af | ou) & p.group_mask) : GW(0);

        // ---- stage 2: exact lane test per positive group --------------------
        int n_emit = 0;
        uint64_t emit = 0;
        if (word) {
            pos_acc += __popcll((unsigned long long)word);
            double act = 0.0;
            bool touched = false;
            int last_tid = INT_MIN;
            GW left = word;
            while (left) {
                const int g = __ffsll((long long)(unsigned long long)left) - 1;
                left &= left - GW(1);
                LW lf = ~LW(0), lo2 = LW(0);
                for (int j = 0; j < size; j += 4) {
                    int32_t l[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) l[u] = (j + u < size) ? ld_lit(lp + (j + u) * STRIDE) : p.sentinel;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int32_t lit = l[u];
                        const int64_t v = lit < 0 ? -lit : lit;
                        const LaneEntry<LW> e = ld_lane(p.lane + v * p.G + g);
                        const LW isf = lit < 0 ? (e.s & e.t) : (e.s & ~e.t);
                        step<LW>(lf, lo2, isf, ~e.s);
                    }
                    if ((lf | lo2) == LW(0)) break;
                }
                const LW mask = (lf | lo2) & p.lane_mask[g];
                if (!mask) continue;
                const int hits = __popcll((unsigned long long)mask);
                trig_acc += hits;
                if (!p.emit_only) {
                    if (!touched) { act = bd->acts[slot]; touched = true; }
                    act = __dadd_rn(act, __dmul_rn(p.inc, (double)hits));
                }
                const int tid = p.tid[g];
                if (tid != last_tid) {  // first triggering group of this thread (engine.py:462)
                    last_tid = tid;
                    bool dup = false;
                    if (tid == p.carry_in_tid)
                        dup = p.carry[bd->tile0 * STRIDE + slot] == (p.stamp_base | (uint32_t)tid);
                    if (!dup) {
                        emit |= 1ull << g;
                        masks[g] = mask;
                        ++n_emit;
                    }
                }
            }
            if (touched) bd->acts[slot] = act;
            if (p.carry_out_tid >= 0 && last_tid == p.carry_out_tid)
                p.carry[bd->tile0 * STRIDE + slot] = p.stamp_base | (uint32_t)last_tid;
        }

        // ---- K4: report emission, one atomic per warp ------------------------
        int incl = n_emit;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int o = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += o;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        if (total) {
            unsigned long long base = 0;
            if (lane == 31) base = atomicAdd(p.ctr, (unsigned long long)total);
            base = __shfl_sync(0xffffffffu, base, 31);
            int64_t pos = (int64_t)base + incl - n_emit;
            if (emit) {
                const int64_t eid = bd->ids[slot];
                while (emit) {
                    const int g = __ffsll((long long)emit) - 1;
                    emit &= emit - 1;
                    if (pos < p.out_cap) {
                        tsg_report r;
                        r.engine_id = eid;
                        r.lane_mask = (uint64_t)masks[g];
                        r.group = p.g0 + g;
                        r.bucket = bd->rank;
                        r.slot = slot;
                        p.out[pos] = r;
                    }
                    ++pos;
                }
            }
        }
    }

    if (p.emit_only) return;
    // counters: warp reduce, then block reduce, one atomic per block
    __shared__ unsigned long long s_pos[32], s_trig[32];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        pos_acc += __shfl_down_sync(0xffffffffu, pos_acc, d);
        trig_acc += __shfl_down_sync(0xffffffffu, trig_acc, d);
    }
    const int w = threadIdx.x >> 5;
    if (lane == 0) { s_pos[w] = pos_acc; s_trig[w] = trig_acc; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a = 0, b = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { a += s_pos[i]; b += s_trig[i]; }
        if (a) atomicAdd(p.ctr + 1, a);
        if (b) atomicAdd(p.ctr + 2, b);
    }
}

}  // namespace tsg
