// tsg_engine.cu -- C ABI (include/tsg.h) over the sm_100a kernels.
//
// Host runtime of the device engine: bucket bookkeeping, staging, the round
// (encode, chunk-level aggregate, one trigger launch), record buffers and
// egress, and store maintenance (radix-select reduce, order-preserving
// compaction).  Every device kernel on these paths is in tsg_kernels.cuh /
// tsg_store.cuh; no library kernels.
#include <cuda_runtime.h>
#include <immintrin.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/tsg.h"
#include "tsg_kernels.cuh"
#include "tsg_store.cuh"
#include "tsg_sort.cuh"

using namespace tsg;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                           \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            return fail(e_ == cudaErrorMemoryAllocation ? TSG_ENOMEM : TSG_ECUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                \
        }                                                                                  \
    } while (0)

#define CKR(expr)                 \
    do {                          \
        int r_ = (expr);          \
        if (r_ != TSG_OK) return r_; \
    } while (0)

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

int grid_for(int64_t n, int threads = 256, int cap = 148 * 16) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (int)b;
}

// A size bucket of the reference store (engine.py:122-163): one interleaved
// array, slots in placement order (pivot-sorted per insert batch, DESIGN.md
// §3); the reference's slot order is engine-id order (reports.py).
struct Bucket {
    int32_t size = 0, rank = 0;
    int64_t count = 0, cap = 0;  // cap: multiple of STRIDE
    int32_t* lits = nullptr;
    double* acts = nullptr;
    int64_t* ids = nullptr;
    int32_t* origins = nullptr;
    uint64_t* order = nullptr;   // where the stored literal order came from (tsg_store.cuh order_word)
};

}  // namespace

// The group description of one round (tsg_round_prepare), kept per round
// so a launched round can be collected -- and its report emission replayed --
// after the next round has been prepared and encoded.
struct RoundDesc {
    int32_t n_groups = 0, n_chunks = 0;
    std::vector<int32_t> glanes, gtid;
    std::vector<int64_t> grow0;
    int64_t chunk_stride = 0;  // bytes between chunk tables inside a table slot
    int64_t top_off = 0;       // chunk-level aggregate (n_chunks > 1)
    int32_t per_bit = 1;       // chunks per bit of the chunk-level aggregate
};

struct tsg_engine {
    int dev = 0;
    int nsm = 148;
    int32_t V = 0;
    tsg_config cfg{};
    cudaStream_t st = nullptr;
    std::vector<Bucket> buckets;
    std::unordered_map<int32_t, int> by_size;

    // staged snapshot rows
    const int8_t* rows = nullptr;  // device rows used by the encoder (owned or aliased)
    int8_t* rows_own = nullptr;
    int64_t rows_cap = 0, pitch = 0, n_rows = 0;
    // packed rows (2 bits per variable, tsg_pack_rows) when `packed`
    bool packed = false;
    const uint64_t* prows = nullptr;
    int64_t ppitch = 0;
    // two staging buffers filled on the ingress stream: the rows of round
    // i+1 copy in while round i is encoded and tested
    uint64_t* pbuf[2] = {nullptr, nullptr};
    int64_t pbuf_cap[2] = {0, 0};
    int8_t* rawbuf[2] = {nullptr, nullptr};  // tsg_stage_packed_mixed: int8 rows packed on the device
    int64_t rawbuf_cap[2] = {0, 0};
    int pk = 1;                           // buffer of the last stage
    bool pstaged = false;                 // prows is pbuf[pk], copied on the ingress stream
    cudaStream_t ingress = nullptr;
    cudaEvent_t ev_staged[2] = {nullptr, nullptr};  // copy into pbuf[b] done
    cudaEvent_t ev_read[2] = {nullptr, nullptr};    // encoder done reading pbuf[b]

    RoundDesc rd;  // as prepared
    // round tables: two slots (slot stride slot_bytes); encode writes slot
    // `tslot`; tsg_round_launch flips it, so the next round encodes while the
    // launched one still owns its tables
    int8_t* tables = nullptr;
    int64_t tables_bytes = 0, slot_bytes = 0;
    int tslot = 0;
    cudaEvent_t ev_enc[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // per table slot: encode start/end

    // Two round states alternate: a launched round keeps its
    // group description, table slot, counters and record buffer until it is
    // collected -- and the buffer until its records were copied out -- so up
    // to two rounds are in flight.
    struct RoundState {
        RoundDesc fl;
        int slot = 0;                         // table slot it tests
        double inc = 0.0;
        int64_t seq = 0;                      // launch sequence: collect order
        bool inflight = false;                // launched, not collected
        // device [8]: [0] records, [1] aggregate positives, [2] lane triggers,
        // [5] CTAs done, [6..7] polarity counts; zero between rounds (the
        // round's last CTA publishes them to h_ctr and re-zeroes them)
        unsigned long long* ctr = nullptr;
        unsigned long long* h_ctr = nullptr;  // pinned [8], written by the kernel
        bool pol_pending = false;             // an encode counted into ctr[6..7] since the last launch
        bool timed = false;                   // its encode / test are bracketed by timing events
        bool rec8 = false;                    // its records are 8-byte u64
        bool all_pairs = false;
        bool ringed = false;                  // its records went to the host report ring
        GroupDesc* d_groups = nullptr;        // the round's groups (device)
        GroupDesc* h_groups = nullptr;        // pinned staging of the same
        int64_t groups_cap = 0;
        cudaEvent_t ev_done = nullptr;        // its counters are on the host
        cudaEvent_t ev_tst[2] = {nullptr, nullptr};
        // records: exact count n_out in out (tsg_report or u64); egress
        // repacking in out12; ev_copied = the last copy-out from them is done
        tsg_report* out = nullptr;
        int64_t out_cap = 0, n_out = 0;
        uint8_t* out12 = nullptr;
        int64_t out12_cap = 0;
        cudaEvent_t ev_copied = nullptr;
    } rs[2];
    int next_rs = 0;                      // state of the next launch
    int fetch_rs = 0;                     // state the fetch calls read (the last collected)
    unsigned long long* mctr = nullptr;   // device [8]: maintenance scratch
    unsigned long long* h_mctr = nullptr; // pinned [8]
    cudaStream_t egress = nullptr;
    cudaEvent_t ev_ready = nullptr;       // records ready for copy-out
    cudaEvent_t ev_peer = nullptr;        // tsg_round_tables_copy: tables encoded / copied

    BucketDesc* d_desc = nullptr;
    int64_t desc_cap = 0;
    std::vector<BucketDesc> h_desc;
    int64_t n_tiles = 0;
    bool desc_dirty = true;               // store changed since the tile table was built

    int32_t record_bytes = 16;      // egress record format (tsg_set_record_bytes)
    bool all_pairs = false;         // tsg_set_all_pairs
    int64_t max_id = -1;            // largest engine id ever added (8-byte records need < 2^27)
    int32_t* size_of_id = nullptr;  // clause size by engine id (record ordering, tsg_fetch_ordered)
    int64_t size_of_id_cap = 0;
    bool oob = false;               // a stored literal may exceed num_vars (checked before testing)
    int64_t round_seq = 0;
    uint8_t* ord_host = nullptr;    // tsg_fetch_ordered small-round scratch: page-locked host ...
    uint8_t* ord_dev = nullptr;     // ... and device, same size
    int64_t ord_cap = 0;
    uint8_t* add_host = nullptr;    // page-locked staging block of tsg_add_clauses (streaming batches)
    int64_t add_host_cap = 0;
    cudaEvent_t ev_add = nullptr;   // its last copy
    int enc_attr = 0;               // k_encode_packed32 shared-memory attribute set, per (GPW, GW)
    // tsg_round_encode_groups: encode groups [enc_g0, enc_g1) only (enc_g1 < 0: all)
    int32_t enc_g0 = 0, enc_g1 = -1;
    bool enc_sentinel = true;
    tsg_counters_t totals{};        // cumulative figures (tsg_counters)
    int32_t timing_every = 1;       // TSG_F_TIMING: events on rounds whose sequence is a multiple (tsg_set_timing)
    int64_t grid[16] = {0};         // persistent grid per k_test variant (0: not computed)

    // a reduce selection in progress (tsg_reduce_begin .. tsg_reduce_commit):
    // the flat key arrays over the store as it was at begin
    struct Select {
        bool open = false;
        uint64_t *ka = nullptr, *ki = nullptr;
        uint8_t* keep = nullptr;
        unsigned long long* hist = nullptr;
        std::vector<int64_t> base;
        int64_t flat = 0, n_eligible = 0, store_seq = 0;
    } sel;
    int64_t store_seq = 0;          // bumped by every store change (a selection must not outlive one)

    bool pivot = true;              // pivot-first clause layout (TSG_PIVOT=0 disables)
    // chunk-level aggregate sweep before the chunks of a multi-chunk round
    // (TSG_F_CHUNK_FILTER or TSG_CHUNK_FILTER=1): measured
    // faster on synthetic per-thread windows, slower on real CDCL snapshots
    // (profiles/r02_hier_aggregate.md), so off by default
    bool chunk_filter = false;
    // literal polarity placed right after the pivot (+1 / -1 / 0 none).  Prior
    // before any round: +1 -- in the paper's measured value subsets
    // a variable can be True in a window more often
    // (.208) than False (.153), so positive literals are non-False more often
    int prefer = 1;
    bool prefer_fixed = false;      // TSG_PREFER fixes it; else set from each round's statistics

    // host report ring (tsg_ring_open): rounds launched while
    // it is open write their records into it instead of the device buffer
    struct Ring {
        unsigned long long* slots = nullptr;    // page-locked, mapped: [cap][2] tagged words
        unsigned long long* d_slots = nullptr;  // its device view
        unsigned long long* ctl = nullptr;      // page-locked, mapped: [0] consumed (tail), [1] failed
        unsigned long long* d_ctl = nullptr;
        unsigned long long* d_pos = nullptr;    // device: positions reserved by the kernels
        int64_t cap = 0, wait_ns = 0;
        int32_t shift = 0;                      // log2(cap)
        // drainers claim blocks of `blk` consecutive positions (block b =
        // positions b*blk ..), consume a block in order, and hand it back
        // when they stop early; the tail is the consumed prefix
        int64_t blk = 1;
        std::mutex mtx;                         // guards the block bookkeeping below
        int64_t next_block = 0;                 // blocks handed out so far
        std::map<int64_t, int64_t> open;        // handed-out, unfinished block -> positions consumed
        std::set<int64_t> idle;                 // open blocks no drainer holds (resumable)
        int active = 0;                         // drainers inside tsg_ring_drain (under mtx)
        std::atomic<bool> closing{false};       // tsg_ring_close waits for active == 0
        std::atomic<int64_t> expected{0};       // records of the collected rounds
    } ring;
};

namespace {

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
        // a non-sticky error left by another library in this thread (torch,
        // NCCL, gloo) must not be reported by our own launch checks
        cudaGetLastError();
    }
    ~DevGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

bool any_inflight(const tsg_engine* h) { return h->rs[0].inflight || h->rs[1].inflight; }

// Timing events stall the stream front end (≈2.5 µs each between dependent
// kernels), so they can be limited to every n-th round (tsg_set_timing).
bool timed_round(const tsg_engine* h, int64_t seq) {
    return (h->cfg.flags & TSG_F_TIMING) && h->timing_every > 0 && seq % h->timing_every == 0;
}

int dalloc(tsg_engine* h, void** p, int64_t bytes) {
    *p = nullptr;
    if (bytes <= 0) return TSG_OK;
    CK(cudaMallocAsync(p, (size_t)bytes, h->st));
    return TSG_OK;
}

void dfree(tsg_engine* h, void* p) {
    if (p) cudaFreeAsync(p, h->st);
}

template <class T>
int dgrow(tsg_engine* h, T** p, int64_t* cap, int64_t need) {
    if (need <= *cap) return TSG_OK;
    int64_t nc = std::max<int64_t>(need, *cap * 2);
    T* np = nullptr;
    CKR(dalloc(h, (void**)&np, nc * (int64_t)sizeof(T)));
    dfree(h, *p);
    *p = np;
    *cap = nc;
    return TSG_OK;
}

void bucket_free(tsg_engine* h, Bucket& b) {
    dfree(h, b.lits); dfree(h, b.acts); dfree(h, b.ids); dfree(h, b.origins); dfree(h, b.order);
    b.lits = nullptr; b.acts = nullptr; b.ids = nullptr; b.origins = nullptr; b.order = nullptr;
}

// arrays of a bucket with `cap` slots (count and bookkeeping unchanged)
int bucket_alloc(tsg_engine* h, Bucket& b, int64_t cap) {
    CKR(dalloc(h, (void**)&b.lits, cap * (int64_t)std::max(b.size, 1) * 4));
    CKR(dalloc(h, (void**)&b.acts, cap * 8));
    CKR(dalloc(h, (void**)&b.ids, cap * 8));
    CKR(dalloc(h, (void**)&b.origins, cap * 4));
    CKR(dalloc(h, (void**)&b.order, cap * 8));
    b.cap = cap;
    return TSG_OK;
}

int bucket_reserve(tsg_engine* h, Bucket& b, int64_t need) {
    if (need <= b.cap) return TSG_OK;
    // _SizeBucket._grow doubles with a floor of 4 blocks (engine.py:141-148)
    int64_t nc = std::max<int64_t>(b.cap ? b.cap : 4 * STRIDE, 4 * STRIDE);
    while (nc < need) nc *= 2;
    Bucket n = b;
    CKR(bucket_alloc(h, n, nc));
    if (b.count) {
        const int64_t used = round_up(b.count, STRIDE);
        if (b.size) CK(cudaMemcpyAsync(n.lits, b.lits, used * b.size * 4, cudaMemcpyDeviceToDevice, h->st));
        CK(cudaMemcpyAsync(n.acts, b.acts, b.count * 8, cudaMemcpyDeviceToDevice, h->st));
        CK(cudaMemcpyAsync(n.ids, b.ids, b.count * 8, cudaMemcpyDeviceToDevice, h->st));
        CK(cudaMemcpyAsync(n.origins, b.origins, b.count * 4, cudaMemcpyDeviceToDevice, h->st));
        CK(cudaMemcpyAsync(n.order, b.order, b.count * 8, cudaMemcpyDeviceToDevice, h->st));
    }
    bucket_free(h, b);
    b = n;
    return TSG_OK;
}

bool wide_lane(const tsg_engine* h) { return h->cfg.lane_width > 32; }
bool wide_group(const tsg_engine* h) { return h->cfg.group_width > 32; }
int64_t agg_entry_bytes(const tsg_engine* h) { return wide_group(h) ? 32 : 16; }
int64_t vstride(const tsg_engine* h) { return round_up((int64_t)h->V + 2, 4); }
int64_t agg_bytes(const tsg_engine* h) { return round_up((int64_t)(h->V + 2) * agg_entry_bytes(h), 256); }
int64_t lane_entry_bytes(const tsg_engine* h) { return wide_lane(h) ? 16 : 8; }
// one chunk's tables: its aggregate table, then its groups' lane tables
int64_t chunk_bytes(const tsg_engine* h) {
    return agg_bytes(h) + round_up(vstride(h) * h->cfg.group_width * lane_entry_bytes(h), 256);
}
int64_t top_bytes(const tsg_engine* h) { return round_up((int64_t)(h->V + 2) * 16, 256); }

// u64 words of one packed row: every 128-variable encoder block reads 4 words
int64_t packed_words(int32_t V) { return round_up(((int64_t)V + 2 + 31) / 32, 4); }

template <class LW, class GW>
int launch_encode(tsg_engine* h, int c) {
    const RoundDesc& rd = h->rd;
    const int32_t g0 = c * h->cfg.group_width;
    const int32_t G = std::min(h->cfg.group_width, rd.n_groups - g0);
    int8_t* tab = h->tables + h->tslot * h->slot_bytes + c * rd.chunk_stride;
    auto* agg = reinterpret_cast<AggEntry<GW>*>(tab);
    auto* lane = reinterpret_cast<LaneEntry<LW>*>(tab + agg_bytes(h));
    unsigned long long* polarity = h->rs[h->next_rs].ctr + 6;  // counted for the round this encode feeds
    const dim3 grid((unsigned)((h->V + 2 + 127) / 128)), block(32, 8);
    if (!h->packed) {
        EncodeChunk ec{};
        ec.G = G;
        ec.num_vars = h->V;
        ec.pitch = h->pitch;
        ec.vstride = vstride(h);
        for (int g = 0; g < G; ++g) {
            ec.row0[g] = rd.grow0[g0 + g];
            ec.lanes[g] = rd.glanes[g0 + g];
        }
        ec.polarity = polarity;
        k_encode<LW, GW><<<grid, block, 0, h->st>>>(h->rows, ec, lane, agg);
        CK(cudaGetLastError());
        return TSG_OK;
    }
    EncodePackedChunk pc{};
    pc.G = G;
    pc.num_vars = h->V;
    pc.pitch_words = h->ppitch;
    pc.vstride = vstride(h);
    // a group range (tsg_round_encode_groups): the rows hold only its groups
    const int64_t row_base = h->enc_g1 >= 0 ? rd.grow0[h->enc_g0] : 0;
    for (int g = 0; g < G; ++g) {
        pc.row0[g] = rd.grow0[g0 + g] - row_base;
        pc.lanes[g] = rd.glanes[g0 + g];
    }
    pc.polarity = polarity;
    pc.gbeg = h->enc_g1 >= 0 ? std::max(0, h->enc_g0 - g0) : 0;
    pc.gend = h->enc_g1 >= 0 ? std::min(G, h->enc_g1 - g0) : G;
    pc.sentinel = h->enc_sentinel ? 1 : 0;
    if constexpr (sizeof(LW) == 4) {
        const int need = (G + 7) / 8;  // groups per warp
        const int gpw = need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : 8;
        const size_t smem = (size_t)8 * gpw * 32 * 32;
        auto* fn = gpw == 1 ? k_encode_packed32<GW, 1> : gpw == 2 ? k_encode_packed32<GW, 2>
                 : gpw == 4 ? k_encode_packed32<GW, 4> : k_encode_packed32<GW, 8>;
        const int bit = 1 << (gpw + 8 * (int)(sizeof(GW) / 8));
        if (!(h->enc_attr & bit)) {  // 64 KB of row stage at 8 groups per warp
            CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            h->enc_attr |= bit;
        }
        fn<<<grid, block, smem, h->st>>>(h->prows, pc, lane, agg);
    } else {
        if (h->enc_g1 >= 0) return fail(TSG_EINVAL, "group-range encode needs lane_width <= 32");
        k_encode_packed<LW, GW><<<grid, block, 0, h->st>>>(h->prows, pc, lane, agg);
    }
    CK(cudaGetLastError());
    return TSG_OK;
}

int do_encode(tsg_engine* h) {
    const RoundDesc& rd = h->rd;
    for (int c = 0; c < rd.n_chunks; ++c) {
        int r;
        if (wide_lane(h)) r = wide_group(h) ? launch_encode<uint64_t, uint64_t>(h, c) : launch_encode<uint64_t, uint32_t>(h, c);
        else r = wide_group(h) ? launch_encode<uint32_t, uint64_t>(h, c) : launch_encode<uint32_t, uint32_t>(h, c);
        if (r) return r;
    }
    if (rd.n_chunks > 1 && h->chunk_filter) {  // chunk-level aggregate over the chunks' tables
        const uint8_t* slot = reinterpret_cast<const uint8_t*>(h->tables + h->tslot * h->slot_bytes);
        auto* top = reinterpret_cast<AggEntry<uint32_t>*>(h->tables + h->tslot * h->slot_bytes + rd.top_off);
        const int64_t nv2 = (int64_t)h->V + 2;
        if (wide_group(h)) k_top<uint64_t><<<grid_for(nv2), 256, 0, h->st>>>(slot, rd.chunk_stride, rd.n_chunks, rd.per_bit, nv2, top);
        else k_top<uint32_t><<<grid_for(nv2), 256, 0, h->st>>>(slot, rd.chunk_stride, rd.n_chunks, rd.per_bit, nv2, top);
        CK(cudaGetLastError());
    }
    return TSG_OK;
}

// Tile table of the round: buckets in creation order, tiles of 32 slots.
int build_desc(tsg_engine* h) {
    if (!h->desc_dirty) return TSG_OK;  // store unchanged since the last round
    h->h_desc.clear();
    int64_t tiles = 0;
    for (auto& b : h->buckets) {
        if (!b.count) continue;
        BucketDesc d{};
        d.lits = b.lits; d.acts = b.acts; d.ids = b.ids;
        d.size = b.size; d.rank = b.rank; d.count = b.count; d.tile0 = tiles;
        tiles += (b.count + STRIDE - 1) / STRIDE;
        h->h_desc.push_back(d);
    }
    h->n_tiles = tiles;
    CKR(dgrow(h, &h->d_desc, &h->desc_cap, std::max<int64_t>(1, (int64_t)h->h_desc.size())));
    if (!h->h_desc.empty()) {
        CK(cudaMemcpyAsync(h->d_desc, h->h_desc.data(), h->h_desc.size() * sizeof(BucketDesc),
                           cudaMemcpyHostToDevice, h->st));
        CK(cudaStreamSynchronize(h->st));  // pageable source
    }
    h->desc_dirty = false;
    return TSG_OK;
}

template <class LW, class GW>
int launch_test(tsg_engine* h, int k, int emit_only) {
    auto& R = h->rs[k];
    const RoundDesc& rd = R.fl;
    TestParams<LW, GW> p{};
    p.buckets = h->d_desc;
    p.nb = (int32_t)h->h_desc.size();
    p.n_tiles = (int32_t)h->n_tiles;
    p.tables = reinterpret_cast<const uint8_t*>(h->tables + R.slot * h->slot_bytes);
    p.chunk_stride = rd.chunk_stride;
    p.lane_off = agg_bytes(h);
    p.vstride = vstride(h);
    p.top = h->chunk_filter ? reinterpret_cast<const AggEntry<uint32_t>*>(p.tables + rd.top_off) : nullptr;
    p.n_chunks = rd.n_chunks;
    p.group_width = h->cfg.group_width;
    p.n_groups = rd.n_groups;
    p.per_bit = rd.per_bit;
    p.sentinel = h->V + 1;
    p.groups = R.d_groups;
    p.inc = R.inc;
    p.out = R.out;
    p.out_cap = (unsigned long long)R.out_cap;
    p.ctr = R.ctr;
    p.pub = emit_only ? nullptr : R.h_ctr;
    p.emit_only = emit_only;
    p.rec8 = R.rec8 ? 1 : 0;
    p.all_pairs = R.all_pairs ? 1 : 0;
    if (R.ringed) {  // records straight into the host ring (never replayed: no device buffer to overflow)
        p.out = nullptr;
        p.out_cap = 0;
        p.ring = RingDesc{h->ring.d_slots, h->ring.d_pos, h->ring.d_ctl, h->ring.d_ctl + 1,
                          (unsigned long long)(h->ring.cap - 1), (unsigned long long)h->ring.wait_ns,
                          ((volatile unsigned long long*)h->ring.ctl)[0], h->ring.shift};
    }
    const bool multi = rd.n_chunks > 1;
    auto* fn = multi ? k_test<LW, GW, true> : k_test<LW, GW, false>;
    const size_t smem = (size_t)test_smem_bytes(R.rec8);
    const int key = (int)(sizeof(LW) / 8) * 8 + (int)(sizeof(GW) / 8) * 4 + (multi ? 2 : 0) + (R.rec8 ? 1 : 0);
    if (!h->grid[key]) {  // persistent grid: as many CTAs as fit on every SM
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, TEST_THREADS, smem));
        h->grid[key] = (int64_t)std::max(1, per_sm) * h->nsm;
    }
    const int64_t want = (h->n_tiles + TEST_THREADS / 32 - 1) / (TEST_THREADS / 32);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, h->grid[key]));
    fn<<<grid, TEST_THREADS, smem, h->st>>>(p);
    CK(cudaGetLastError());
    return TSG_OK;
}

// the round of state k
int run_test(tsg_engine* h, int k, int emit_only) {
    if (wide_lane(h)) return wide_group(h) ? launch_test<uint64_t, uint64_t>(h, k, emit_only) : launch_test<uint64_t, uint32_t>(h, k, emit_only);
    return wide_group(h) ? launch_test<uint32_t, uint64_t>(h, k, emit_only) : launch_test<uint32_t, uint32_t>(h, k, emit_only);
}

int64_t store_size(const tsg_engine* h) {
    int64_t n = 0;
    for (auto& b : h->buckets) n += b.count;
    return n;
}

int validate_handle(tsg_engine* h) {
    if (!h) return fail(TSG_EINVAL, "null engine handle");
    return TSG_OK;
}

// Order-preserving compaction of every bucket by the flat keep array
// (bucket b's slots at base[b], each bucket padded to KEEP_BLOCK; padding
// keeps 0): K8 through k_keep_count / k_keep_select / k_compact.
int compact_all(tsg_engine* h, const uint8_t* keep, const std::vector<int64_t>& base, int64_t flat) {
    const int64_t nblk = flat / KEEP_BLOCK;
    h->store_seq++;
    if (!nblk) return TSG_OK;
    int32_t* cnt = nullptr;
    int64_t *off = nullptr, *sel = nullptr;
    CKR(dalloc(h, (void**)&cnt, nblk * 4));
    CKR(dalloc(h, (void**)&off, nblk * 8));
    CKR(dalloc(h, (void**)&sel, flat * 8));
    k_keep_count<<<(unsigned)nblk, KEEP_BLOCK, 0, h->st>>>(keep, cnt);
    CK(cudaGetLastError());
    std::vector<int32_t> hc(nblk);
    CK(cudaMemcpyAsync(hc.data(), cnt, nblk * 4, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    std::vector<int64_t> ho(nblk);
    int64_t acc = 0;
    for (int64_t i = 0; i < nblk; ++i) { ho[i] = acc; acc += hc[i]; }
    CK(cudaMemcpyAsync(off, ho.data(), nblk * 8, cudaMemcpyHostToDevice, h->st));
    k_keep_select<<<(unsigned)nblk, KEEP_BLOCK, 0, h->st>>>(keep, off, sel);
    CK(cudaGetLastError());
    for (size_t bi = 0; bi < h->buckets.size(); ++bi) {
        Bucket& b = h->buckets[bi];
        if (!b.count) continue;
        const int64_t blk0 = base[bi] / KEEP_BLOCK, blk1 = blk0 + (b.count + KEEP_BLOCK - 1) / KEEP_BLOCK;
        int64_t kept = 0;
        for (int64_t i = blk0; i < blk1; ++i) kept += hc[i];
        if (kept == b.count) continue;
        Bucket n = b;
        CKR(bucket_alloc(h, n, b.cap));  // keep capacity (the reference never shrinks, engine.py:184-200)
        if (kept)
            k_compact<<<grid_for(kept), 256, 0, h->st>>>(sel + ho[blk0], base[bi], kept, b.size, b.lits, b.acts,
                                                         b.ids, b.origins, b.order, n.lits, n.acts, n.ids,
                                                         n.origins, n.order);
        CK(cudaGetLastError());
        bucket_free(h, b);
        n.count = kept;
        b = n;
    }
    CK(cudaStreamSynchronize(h->st));  // ho is pageable
    dfree(h, cnt); dfree(h, off); dfree(h, sel);
    return TSG_OK;
}

// per-bucket offsets into the flat maintenance arrays (KEEP_BLOCK-aligned)
std::vector<int64_t> bucket_bases(tsg_engine* h, int64_t* flat) {
    std::vector<int64_t> base;
    int64_t acc = 0;
    for (auto& b : h->buckets) {
        base.push_back(acc);
        acc += round_up(b.count, KEEP_BLOCK);
    }
    *flat = acc;
    return base;
}

void ring_free(tsg_engine* h);      // the host report ring (end of file)
void ring_shutdown(tsg_engine* h);

void select_free(tsg_engine* h) {
    auto& S = h->sel;
    dfree(h, S.ka); dfree(h, S.ki); dfree(h, S.keep); dfree(h, S.hist);
    S = tsg_engine::Select{};
}

// Placement of one clause: the pivot -- the literal with the
// smallest variable among the first 58 -- goes first (add_clauses orders
// each batch by pivot, so a warp's first gathers share table lines), then
// the literals of the preferred polarity (those more likely to be non-False
// under the recent rounds' assignments: they end the early-exit recurrence
// sooner), then the rest.  The order word lets readback restore the
// reference's literal order.
// Host worker threads for batch-parallel loops (clause placement), created
// once: spawning threads per tsg_add_clauses call cost more than the
// placement of a streaming batch itself.  parallel_for(n, f) runs f(a, b) over
// [0, n) in contiguous ranges on up to `workers` threads plus the caller.
class HostPool {
  public:
    static HostPool& get() {
        // never destroyed: the workers end with the process (no join at exit,
        // where a forked child would join threads it does not have)
        static HostPool* p = new HostPool;
        return *p;
    }
    int workers() const { return (int)th_.size(); }
    template <class F>
    void parallel_for(int64_t n, int parts, F&& f) {
        // a forked child has none of the parent's workers: run in the caller
        if (getpid() != pid_) parts = 1;
        parts = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)parts, (int64_t)workers() + 1, n}));
        if (parts == 1) { f(0, n); return; }
        std::unique_lock<std::mutex> run(run_mtx_);  // one batch at a time
        std::function<void(int64_t, int64_t)> job = f;
        {
            std::lock_guard<std::mutex> lk(mtx_);
            job_ = &job;
            n_ = n;
            parts_ = parts;
            next_ = 1;  // part 0 is the caller's
            left_ = parts - 1;
            ++gen_;
        }
        cv_.notify_all();
        f(0, n / parts);
        std::unique_lock<std::mutex> lk(mtx_);
        done_cv_.wait(lk, [&] { return left_ == 0; });
        job_ = nullptr;
    }

  private:
    HostPool() : pid_(getpid()) {
        const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
        for (int i = 0; i < std::min(hw, 16) - 1; ++i) th_.emplace_back([this] { loop(); });
    }
    void loop() {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(mtx_);
        for (;;) {
            cv_.wait(lk, [&] { return gen_ != seen && next_ < parts_; });
            seen = gen_;
            while (next_ < parts_) {
                const int k = next_++;
                const int64_t a = n_ * k / parts_, b = n_ * (k + 1) / parts_;
                auto* job = job_;
                lk.unlock();
                (*job)(a, b);
                lk.lock();
                if (--left_ == 0) done_cv_.notify_all();
            }
        }
    }
    const pid_t pid_;
    std::vector<std::thread> th_;  // detached in effect: the pool lives until exit
    std::mutex mtx_, run_mtx_;
    std::condition_variable cv_, done_cv_;
    std::function<void(int64_t, int64_t)>* job_ = nullptr;
    int64_t n_ = 0;
    int parts_ = 0, next_ = 0, left_ = 0;
    uint64_t gen_ = 0;
};

void place_clause(const tsg_engine* h, const int32_t* lits, int32_t size, int32_t* out, uint64_t* order) {
    const int32_t lim = std::min(size, ORDER_MASK_BITS);
    int32_t jp = -1;
    uint64_t m = 0;
    if (h->pivot && lim > 0) {
        jp = 0;
        int64_t best = std::llabs((long long)lits[0]);
        for (int32_t j = 1; j < lim; ++j) {
            const int64_t a = std::llabs((long long)lits[j]);
            if (a < best) { best = a; jp = j; }
        }
        if (h->prefer != 0) {  // branch-free: the signs are random
            const bool pos = h->prefer > 0;
            for (int32_t j = 0; j < lim; ++j) m |= (uint64_t)((j != jp) & ((lits[j] > 0) == pos)) << j;
        }
    }
    // pivot, the preferred-polarity literals, the others (each group in
    // clause order) -- branch-free compaction through a small buffer -- then
    // the literals past the order word's reach, in clause order
    int32_t tmp[ORDER_MASK_BITS + 2];
    int32_t o = 0;
    if (jp >= 0) tmp[o++] = lits[jp];
    for (int32_t j = 0; j < lim; ++j) {
        tmp[o] = lits[j];
        o += (int32_t)((m >> j) & 1);
    }
    for (int32_t j = 0; j < lim; ++j) {
        tmp[o] = lits[j];
        o += (int32_t)((j != jp) & !((m >> j) & 1));
    }
    std::memcpy(out, tmp, (size_t)lim * 4);
    if (size > lim) std::memcpy(out + lim, lits + lim, (size_t)(size - lim) * 4);
    *order = order_word(jp, m);
}

}  // namespace

// ===========================================================================
extern "C" {

const char* tsg_last_error(void) { return g_err.c_str(); }
void tsg__set_error(const char* msg) { g_err = msg ? msg : ""; }
int tsg_abi_version(void) { return TSG_ABI_VERSION; }

int tsg_device_count(int32_t* n) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) { *n = 0; return fail(TSG_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e)); }
    *n = c;
    return TSG_OK;
}

int tsg_destroy(tsg_engine* h);

int tsg_create(int32_t num_vars, const tsg_config* cfg, tsg_engine** out) {
    if (!out || !cfg) return fail(TSG_EINVAL, "null argument");
    *out = nullptr;
    if (num_vars < 0 || num_vars > (1 << 30)) return fail(TSG_EINVAL, "num_vars out of range: %d", num_vars);
    if (cfg->lane_width < 1 || cfg->lane_width > 64) return fail(TSG_EINVAL, "lane_width must be in 1..64, got %d", cfg->lane_width);
    if (cfg->group_width < 1 || cfg->group_width > 64) return fail(TSG_EINVAL, "group_width must be in 1..64, got %d", cfg->group_width);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(TSG_ECUDA, "no CUDA device");
    if (cfg->device < 0 || cfg->device >= ndev) return fail(TSG_EINVAL, "device %d out of range (%d)", cfg->device, ndev);
    auto* h = new tsg_engine();
    h->dev = cfg->device;
    h->cfg = *cfg;
    h->V = num_vars;
    h->all_pairs = (cfg->flags & TSG_F_ALL_PAIRS) != 0;
    h->chunk_filter = (cfg->flags & TSG_F_CHUNK_FILTER) != 0;
    if (const char* e = getenv("TSG_PIVOT")) h->pivot = atoi(e) != 0;
    if (const char* e = getenv("TSG_CHUNK_FILTER")) h->chunk_filter = atoi(e) != 0;
    if (const char* e = getenv("TSG_PREFER")) { h->prefer = atoi(e); h->prefer_fixed = true; }
    DevGuard g(h->dev);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, h->dev) != cudaSuccess) { delete h; return fail(TSG_ECUDA, "device properties"); }
    h->nsm = prop.multiProcessorCount;
    if (cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking) != cudaSuccess) { delete h; return fail(TSG_ECUDA, "stream"); }
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, h->dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    bool ok = cudaStreamCreateWithFlags(&h->egress, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&h->ingress, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&h->ev_ready, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&h->ev_peer, cudaEventDisableTiming) == cudaSuccess;
    for (int b = 0; b < 2; ++b)
        ok = ok && cudaEventCreateWithFlags(&h->ev_staged[b], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&h->ev_read[b], cudaEventDisableTiming) == cudaSuccess;
    for (int sl = 0; sl < 2; ++sl)
        for (int k = 0; k < 2; ++k) ok = ok && cudaEventCreate(&h->ev_enc[sl][k]) == cudaSuccess;
    const int64_t cap0 = cfg->report_capacity > 0 ? cfg->report_capacity : (1 << 16);
    for (auto& R : h->rs) {
        ok = ok && cudaEventCreateWithFlags(&R.ev_done, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&R.ev_copied, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreate(&R.ev_tst[0]) == cudaSuccess && cudaEventCreate(&R.ev_tst[1]) == cudaSuccess &&
             cudaMallocHost(&R.h_ctr, 8 * sizeof(unsigned long long)) == cudaSuccess &&
             dalloc(h, (void**)&R.ctr, 8 * sizeof(unsigned long long)) == TSG_OK &&
             cudaMemsetAsync(R.ctr, 0, 8 * sizeof(unsigned long long), h->st) == cudaSuccess &&
             dalloc(h, (void**)&R.out, cap0 * (int64_t)sizeof(tsg_report)) == TSG_OK;
        R.out_cap = cap0;
    }
    ok = ok && cudaMallocHost(&h->h_mctr, 8 * sizeof(unsigned long long)) == cudaSuccess &&
         dalloc(h, (void**)&h->mctr, 8 * sizeof(unsigned long long)) == TSG_OK;
    if (!ok) {
        tsg_destroy(h);
        return fail(TSG_ECUDA, "engine resources could not be created");
    }
    *out = h;
    return TSG_OK;
}

int tsg_destroy(tsg_engine* h) {
    if (!h) return TSG_OK;
    DevGuard g(h->dev);
    if (h->st) select_free(h);
    if (h->st) ring_shutdown(h);
    if (h->st) cudaStreamSynchronize(h->st);
    if (h->ingress) cudaStreamSynchronize(h->ingress);
    if (h->egress) cudaStreamSynchronize(h->egress);
    if (h->st) {
        for (auto& b : h->buckets) bucket_free(h, b);
        dfree(h, h->rows_own); dfree(h, h->pbuf[0]); dfree(h, h->pbuf[1]); dfree(h, h->tables); dfree(h, h->d_desc);
        dfree(h, h->rawbuf[0]); dfree(h, h->rawbuf[1]);
        dfree(h, h->mctr);
        dfree(h, h->size_of_id);
        dfree(h, h->ord_dev);
        for (auto& R : h->rs) { dfree(h, R.ctr); dfree(h, R.out); dfree(h, R.out12); dfree(h, R.d_groups); }
        cudaStreamSynchronize(h->st);
    }
    if (h->h_mctr) cudaFreeHost(h->h_mctr);
    if (h->add_host) cudaFreeHost(h->add_host);
    if (h->ord_host) cudaFreeHost(h->ord_host);
    if (h->ev_add) cudaEventDestroy(h->ev_add);
    for (auto& R : h->rs) {
        if (R.h_ctr) cudaFreeHost(R.h_ctr);
        if (R.h_groups) cudaFreeHost(R.h_groups);
        for (cudaEvent_t e : {R.ev_done, R.ev_copied, R.ev_tst[0], R.ev_tst[1]}) if (e) cudaEventDestroy(e);
    }
    for (int sl = 0; sl < 2; ++sl)
        for (int k = 0; k < 2; ++k)
            if (h->ev_enc[sl][k]) cudaEventDestroy(h->ev_enc[sl][k]);
    for (int b = 0; b < 2; ++b) {
        if (h->ev_staged[b]) cudaEventDestroy(h->ev_staged[b]);
        if (h->ev_read[b]) cudaEventDestroy(h->ev_read[b]);
    }
    for (cudaEvent_t e : {h->ev_ready, h->ev_peer}) if (e) cudaEventDestroy(e);
    if (h->egress) cudaStreamDestroy(h->egress);
    if (h->ingress) cudaStreamDestroy(h->ingress);
    if (h->st) cudaStreamDestroy(h->st);
    delete h;
    return TSG_OK;
}

int tsg_add_clauses(tsg_engine* h, const int32_t* lits, const int64_t* offsets, int64_t n,
                    const int64_t* ids, const int32_t* origins, double activity) {
    CKR(validate_handle(h));
    if (any_inflight(h)) return fail(TSG_EINVAL, "the store cannot change while a launched round is not collected");
    if (n <= 0) return TSG_OK;
    if (!offsets || !ids || !origins) return fail(TSG_EINVAL, "null argument");
    // validate the whole batch before any state changes
    for (int64_t i = 0; i < n; ++i) {
        const int64_t s64 = offsets[i + 1] - offsets[i];
        if (s64 < 0 || s64 > (1 << 24)) return fail(TSG_EINVAL, "bad clause size at clause %lld", (long long)i);
    }
    if (offsets[n] > offsets[0] && !lits) return fail(TSG_EINVAL, "null literals");
    DevGuard g(h->dev);
    static const bool trace_host = getenv("TSG_TRACE_HOST") != nullptr;
    std::vector<std::pair<const char*, double>> tp;
    auto mark = [&](const char* what) {
        if (trace_host) tp.push_back({what, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count()});
    };
    mark("start");
    h->desc_dirty = true;
    h->store_seq++;
    // group clauses by size, preserving arrival order; new sizes create buckets
    // in first-seen order (dict insertion order of ClauseStore.buckets)
    std::unique_ptr<int[]> bucket_of(new int[n]);  // (uninitialised buffers below: every element is written)
    {
        // (the literal range check runs in the placement pass below)
        int64_t top = h->max_id;
        for (int64_t i = 0; i < n; ++i) top = std::max<int64_t>(top, ids[i] < 0 ? INT64_MAX : ids[i]);
        h->max_id = top;
        // size -> bucket through a small direct cache (sizes < 256), the map beyond
        int cache[256];
        std::fill(cache, cache + 256, -1);
        for (const auto& kv : h->by_size)
            if (kv.first < 256) cache[kv.first] = kv.second;
        for (int64_t i = 0; i < n; ++i) {
            const int32_t s = (int32_t)(offsets[i + 1] - offsets[i]);
            int b = s < 256 ? cache[s] : -1;
            if (b < 0) {
                auto it = h->by_size.find(s);
                if (it == h->by_size.end()) {
                    Bucket nb;
                    nb.size = s;
                    nb.rank = (int32_t)h->buckets.size();
                    b = (int)h->buckets.size();
                    h->by_size[s] = b;
                    h->buckets.push_back(nb);
                } else {
                    b = it->second;
                }
                if (s < 256) cache[s] = b;
            }
            bucket_of[i] = b;
        }
    }
    mark("buckets");
    // place every clause (pivot first), then one H2D + scatter per bucket
    std::unique_ptr<int32_t[]> placed(new int32_t[(size_t)std::max<int64_t>(offsets[n] - offsets[0], 1)]);
    std::unique_ptr<uint64_t[]> hm(new uint64_t[n]);
    {  // placement is independent per clause: split large batches over host threads
        // the literals are read once: placed, and range-checked on the way
        // (stored as-is; testing raises, numpy IndexError, engine.py:251)
        std::atomic<bool> oob{false};
        auto place_range = [&](int64_t a, int64_t b) {
            int32_t lo = 0, hi = 0;
            for (int64_t i = a; i < b; ++i) {
                const int32_t* l = lits + offsets[i];
                const int32_t sz = (int32_t)(offsets[i + 1] - offsets[i]);
                for (int32_t j = 0; j < sz; ++j) {
                    lo = std::min(lo, l[j]);
                    hi = std::max(hi, l[j]);
                }
                place_clause(h, l, sz, placed.get() + (offsets[i] - offsets[0]), &hm[i]);
            }
            if ((int64_t)hi > h->V || -(int64_t)lo > h->V) oob = true;
        };
        HostPool::get().parallel_for(n, (int)std::min<int64_t>(16, n / 1024), place_range);
        if (oob) h->oob = true;
    }
    mark("place");
    std::vector<std::vector<int64_t>> members(h->buckets.size());
    {
        std::vector<int64_t> cnt(h->buckets.size(), 0);
        for (int64_t i = 0; i < n; ++i) ++cnt[bucket_of[i]];
        for (size_t b = 0; b < cnt.size(); ++b) members[b].reserve(cnt[b]);
        for (int64_t i = 0; i < n; ++i) members[bucket_of[i]].push_back(i);
    }
    mark("members");
    if (h->pivot) {  // each bucket's new clauses in pivot-variable order (stable: ties keep arrival order)
        // only batches dense enough for a 32-clause tile to share pivot lines
        // gain from the order; a streaming batch of a few hundred clauses per
        // bucket would only pay for the sort
        std::vector<int> big;  // buckets sorted, in parallel (one per worker at a time)
        for (size_t bi = 0; bi < members.size(); ++bi)
            if (members[bi].size() >= 4096) big.push_back((int)bi);
        HostPool::get().parallel_for((int64_t)big.size(), (int)std::min<size_t>(16, big.size()), [&](int64_t a, int64_t b) {
            std::vector<uint64_t> key;
            for (int64_t q = a; q < b; ++q) {
                auto& mem = members[big[q]];
                key.resize(mem.size());
                for (size_t c = 0; c < mem.size(); ++c) {
                    const int64_t i = mem[c];
                    const uint64_t v = offsets[i + 1] > offsets[i] ? (uint64_t)std::llabs((long long)placed[offsets[i] - offsets[0]]) : 0;
                    key[c] = v << 32 | (uint64_t)c;  // (pivot variable, position in the batch's bucket list)
                }
                std::sort(key.begin(), key.end());
                std::vector<int64_t> sorted(mem.size());
                for (size_t c = 0; c < mem.size(); ++c) sorted[c] = mem[key[c] & 0xFFFFFFFFu];
                mem.swap(sorted);
            }
        });
    }
    mark("sort");
    // one host staging block for the whole batch (a pageable copy waits for
    // the stream, so there is exactly one), clauses bucket-major: literals,
    // ids, origins, order words, then the buckets' append descriptors; one
    // append kernel for every bucket (k_append_batch)
    auto al8 = [](int64_t x) { return (x + 7) / 8 * 8; };
    int64_t n_lits = 0;
    std::vector<AppendDesc> desc;
    int64_t first = 0;
    for (size_t bi = 0; bi < members.size(); ++bi) {
        const int64_t k = (int64_t)members[bi].size();
        if (!k) continue;
        Bucket& b = h->buckets[bi];
        CKR(bucket_reserve(h, b, b.count + k));
        desc.push_back(AppendDesc{b.lits, b.acts, b.ids, b.origins, b.order, b.count, first, n_lits, b.size, 0});
        first += k;
        n_lits += k * b.size;
        b.count += k;
    }
    const int64_t o_ids = al8(n_lits * 4), o_org = o_ids + n * 8, o_ord = o_org + al8(n * 4), o_desc = o_ord + n * 8;
    const int64_t total_bytes = o_desc + (int64_t)(desc.size() * sizeof(AppendDesc));
    // The staging block (not zero-filled: every field below is written;
    // alignment padding is never read).  Streaming batches (<= 64 MB) go
    // through a persistent page-locked block -- an asynchronous copy, reused
    // once the previous batch's copy is done; bulk loads through pageable
    // memory (page-locking hundreds of MB once costs more than it saves).
    std::unique_ptr<uint8_t[]> host_buf;
    uint8_t* host_p = nullptr;
    const bool pinned_stage = total_bytes <= ((int64_t)64 << 20);
    if (pinned_stage) {
        if (h->ev_add) CK(cudaEventSynchronize(h->ev_add));  // the last batch's copy has read the block
        else CK(cudaEventCreateWithFlags(&h->ev_add, cudaEventDisableTiming));
        if (total_bytes > h->add_host_cap) {
            const int64_t cap = std::max<int64_t>({total_bytes, 2 * h->add_host_cap, (int64_t)1 << 20});
            if (h->add_host) cudaFreeHost(h->add_host);
    if (h->ord_host) cudaFreeHost(h->ord_host);
            h->add_host = nullptr;
            h->add_host_cap = 0;
            CK(cudaHostAlloc((void**)&h->add_host, (size_t)cap, cudaHostAllocPortable));
            h->add_host_cap = cap;
        }
        host_p = h->add_host;
    } else {
        host_buf.reset(new uint8_t[(size_t)std::max<int64_t>(total_bytes, 8)]);
        host_p = host_buf.get();
    }
    struct { uint8_t* p; uint8_t* data() const { return p; } } host{host_p};
    {
        int32_t* hl = reinterpret_cast<int32_t*>(host.data());
        int64_t* hid = reinterpret_cast<int64_t*>(host.data() + o_ids);
        int32_t* hor = reinterpret_cast<int32_t*>(host.data() + o_org);
        uint64_t* hmk = reinterpret_cast<uint64_t*>(host.data() + o_ord);
        // every bucket's first clause / literal slot in the block, then the
        // buckets filled in parallel
        std::vector<int64_t> c0(members.size() + 1, 0), l0(members.size() + 1, 0);
        for (size_t bi = 0; bi < members.size(); ++bi) {
            c0[bi + 1] = c0[bi] + (int64_t)members[bi].size();
            l0[bi + 1] = l0[bi] + (int64_t)members[bi].size() * h->buckets[bi].size;
        }
        HostPool::get().parallel_for((int64_t)members.size(), n >= 8192 ? 16 : 1, [&](int64_t a, int64_t b) {
            for (int64_t bi = a; bi < b; ++bi) {
                const int32_t sz = h->buckets[bi].size;
                int64_t c = c0[bi], l = l0[bi];
                for (const int64_t i : members[bi]) {
                    if (sz) memcpy(hl + l, placed.get() + (offsets[i] - offsets[0]), sz * 4);
                    l += sz;
                    hid[c] = ids[i];
                    hor[c] = origins[i];
                    hmk[c] = hm[i];
                    ++c;
                }
            }
        });
        memcpy(host.data() + o_desc, desc.data(), desc.size() * sizeof(AppendDesc));
    }
    const bool sizes_by_id = h->max_id < ((int64_t)1 << 40);
    if (sizes_by_id) {  // clause size by engine id: the record ordering looks up each record's bucket
        const int64_t need = h->max_id + 1;
        if (need > h->size_of_id_cap) {
            const int64_t nc = std::max<int64_t>(need, 2 * h->size_of_id_cap);
            int32_t* np = nullptr;
            CKR(dalloc(h, (void**)&np, nc * 4));
            if (h->size_of_id) CK(cudaMemcpyAsync(np, h->size_of_id, h->size_of_id_cap * 4, cudaMemcpyDeviceToDevice, h->st));
            dfree(h, h->size_of_id);
            h->size_of_id = np;
            h->size_of_id_cap = nc;
        }
    }
    mark("block");
    uint8_t* dev = nullptr;
    CKR(dalloc(h, (void**)&dev, std::max<int64_t>(total_bytes, 8)));
    CK(cudaMemcpyAsync(dev, host.data(), total_bytes, cudaMemcpyHostToDevice, h->st));  // pageable: consumed on return
    if (pinned_stage) CK(cudaEventRecord(h->ev_add, h->st));
    mark("h2d");
    k_append_batch<<<grid_for(n), 256, 0, h->st>>>(reinterpret_cast<const AppendDesc*>(dev + o_desc), (int32_t)desc.size(), n,
                                                   reinterpret_cast<const int32_t*>(dev),
                                                   reinterpret_cast<const int64_t*>(dev + o_ids),
                                                   reinterpret_cast<const int32_t*>(dev + o_org),
                                                   reinterpret_cast<const uint64_t*>(dev + o_ord), activity,
                                                   sizes_by_id ? h->size_of_id : nullptr);
    CK(cudaGetLastError());
    dfree(h, dev);
    mark("launches");
    if (trace_host) {
        fprintf(stderr, "tsg_add_clauses n=%lld:", (long long)n);
        for (size_t i = 1; i < tp.size(); ++i) fprintf(stderr, " %s %.3f", tp[i].first, tp[i].second - tp[i - 1].second);
        fprintf(stderr, " ms\n");
    }
    h->totals.clauses_added += n;
    return TSG_OK;
}

int tsg_store_size(tsg_engine* h, int64_t* n) {
    CKR(validate_handle(h));
    *n = store_size(h);
    return TSG_OK;
}

int tsg_bucket_count(tsg_engine* h, int32_t* nb) {
    CKR(validate_handle(h));
    *nb = (int32_t)h->buckets.size();
    return TSG_OK;
}

int tsg_bucket_info(tsg_engine* h, int32_t b, int32_t* size, int64_t* count) {
    CKR(validate_handle(h));
    if (b < 0 || b >= (int32_t)h->buckets.size()) return fail(TSG_ERANGE, "bucket %d out of range", b);
    *size = h->buckets[b].size;
    *count = h->buckets[b].count;
    return TSG_OK;
}

int tsg_bucket_read(tsg_engine* h, int32_t bi, int32_t* lits, int64_t* ids, int32_t* origins, double* acts) {
    CKR(validate_handle(h));
    if (bi < 0 || bi >= (int32_t)h->buckets.size()) return fail(TSG_ERANGE, "bucket %d out of range", bi);
    DevGuard g(h->dev);
    Bucket& b = h->buckets[bi];
    const int64_t total = b.count;
    if (!total) return TSG_OK;
    // slot order (original literal order restored), then sorted by engine id
    // = the reference's slot order (reports.py)
    std::vector<int32_t> hl(lits && b.size ? total * b.size : 0);
    std::vector<int64_t> hid(total);
    std::vector<int32_t> hor(origins ? total : 0);
    std::vector<double> hac(acts ? total : 0);
    if (lits && b.size) {
        int32_t* tmp = nullptr;
        CKR(dalloc(h, (void**)&tmp, total * b.size * 4));
        k_deinterleave<<<grid_for(total), 256, 0, h->st>>>(b.lits, b.order, total, b.size, tmp);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(hl.data(), tmp, total * b.size * 4, cudaMemcpyDeviceToHost, h->st));
        dfree(h, tmp);
    }
    CK(cudaMemcpyAsync(hid.data(), b.ids, total * 8, cudaMemcpyDeviceToHost, h->st));
    if (origins) CK(cudaMemcpyAsync(hor.data(), b.origins, total * 4, cudaMemcpyDeviceToHost, h->st));
    if (acts) CK(cudaMemcpyAsync(hac.data(), b.acts, total * 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    std::vector<int64_t> ord(total);
    for (int64_t i = 0; i < total; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return hid[x] < hid[y]; });
    for (int64_t k = 0; k < total; ++k) {
        const int64_t i = ord[k];
        if (ids) ids[k] = hid[i];
        if (origins) origins[k] = hor[i];
        if (acts) acts[k] = hac[i];
        if (lits && b.size) memcpy(lits + k * b.size, hl.data() + i * b.size, b.size * 4);
    }
    return TSG_OK;
}

// Literals of stored clauses by engine id, in their original order (the
// reference's `lits_at` / Report.lits, engine.py:165-169, 409-414): a C host
// that keeps no literal copy of its own resolves report records with this.
int tsg_get_clauses(tsg_engine* h, const int64_t* ids, int64_t n, int32_t* sizes, int32_t* lits, int64_t lits_cap,
                    int64_t* n_lits) {
    CKR(validate_handle(h));
    if (n < 0 || (n > 0 && (!ids || !sizes || !n_lits))) return fail(TSG_EINVAL, "bad arguments");
    if (n_lits) *n_lits = 0;
    if (n == 0) return TSG_OK;
    DevGuard g(h->dev);
    std::vector<int64_t> qi(n);
    for (int64_t i = 0; i < n; ++i) qi[i] = i;
    std::sort(qi.begin(), qi.end(), [&](int64_t a, int64_t b) { return ids[a] < ids[b]; });
    std::vector<int64_t> q(n);
    for (int64_t i = 0; i < n; ++i) q[i] = ids[qi[i]];
    int64_t* d = nullptr;  // [q | qidx | loc]
    CKR(dalloc(h, (void**)&d, 3 * n * 8));
    CK(cudaMemcpyAsync(d, q.data(), n * 8, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(d + n, qi.data(), n * 8, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemsetAsync(d + 2 * n, 0xFF, n * 8, h->st));
    for (int64_t k = 0; k < (int64_t)h->buckets.size(); ++k) {
        const Bucket& b = h->buckets[k];
        if (b.count) k_find_ids<<<grid_for(b.count), 256, 0, h->st>>>(b.ids, b.count, d, d + n, n, k, d + 2 * n);
    }
    CK(cudaGetLastError());
    std::vector<int64_t> loc(n);
    CK(cudaMemcpyAsync(loc.data(), d + 2 * n, n * 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    dfree(h, d);
    int64_t total = 0;
    std::vector<int64_t> off(n);
    for (int64_t i = 0; i < n; ++i) {
        off[i] = total;
        if (loc[i] < 0) { sizes[i] = -1; continue; }
        sizes[i] = h->buckets[loc[i] >> 40].size;
        total += sizes[i];
    }
    *n_lits = total;
    if (!lits || total == 0) return TSG_OK;
    if (total > lits_cap) return fail(TSG_ECAPACITY, "%lld literals do not fit %lld", (long long)total, (long long)lits_cap);
    // per bucket: gather its hits' literals, then place them in request order
    std::vector<std::vector<int64_t>> hit(h->buckets.size());
    for (int64_t i = 0; i < n; ++i)
        if (loc[i] >= 0) hit[loc[i] >> 40].push_back(i);
    for (size_t k = 0; k < h->buckets.size(); ++k) {
        const Bucket& b = h->buckets[k];
        const int64_t m = (int64_t)hit[k].size();
        if (!m || b.size == 0) continue;
        std::vector<int64_t> slots(m);
        for (int64_t j = 0; j < m; ++j) slots[j] = loc[hit[k][j]] & ((int64_t(1) << 40) - 1);
        int64_t* ds = nullptr;
        int32_t* dl = nullptr;
        CKR(dalloc(h, (void**)&ds, m * 8));
        CKR(dalloc(h, (void**)&dl, m * b.size * 4));
        CK(cudaMemcpyAsync(ds, slots.data(), m * 8, cudaMemcpyHostToDevice, h->st));
        k_deinterleave_sel<<<grid_for(m), 256, 0, h->st>>>(b.lits, b.order, ds, m, b.size, dl);
        CK(cudaGetLastError());
        std::vector<int32_t> hl(m * b.size);
        CK(cudaMemcpyAsync(hl.data(), dl, m * b.size * 4, cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
        dfree(h, ds);
        dfree(h, dl);
        for (int64_t j = 0; j < m; ++j) memcpy(lits + off[hit[k][j]], hl.data() + j * b.size, b.size * 4);
    }
    return TSG_OK;
}

int tsg_set_timing(tsg_engine* h, int32_t every) {
    CKR(validate_handle(h));
    if (every < 0) return fail(TSG_EINVAL, "timing stride must be >= 0, got %d", every);
    h->timing_every = every;
    return TSG_OK;
}

int tsg_set_all_pairs(tsg_engine* h, int32_t on) {
    CKR(validate_handle(h));
    h->all_pairs = on != 0;
    return TSG_OK;
}

int tsg_counters(tsg_engine* h, tsg_counters_t* out) {
    CKR(validate_handle(h));
    if (!out) return fail(TSG_EINVAL, "null argument");
    *out = h->totals;
    return TSG_OK;
}

int tsg_scale_activities(tsg_engine* h, double factor) {
    CKR(validate_handle(h));
    if (any_inflight(h)) return fail(TSG_EINVAL, "the store cannot change while a launched round is not collected");
    DevGuard g(h->dev);
    for (auto& b : h->buckets)
        if (b.count) k_scale_f64<<<grid_for(b.count), 256, 0, h->st>>>(b.acts, b.count, factor);
    CK(cudaGetLastError());
    return TSG_OK;
}

// reduce_store (engine.py:469-505) as a radix select on the 128-bit key
// (activity bits, engine id), split so that several stores (clause shards
// on several GPUs) can select their global `target` smallest keys exactly:
// begin builds the keys of the eligible clauses (id < eligible_below,
// engine.py:486); hist counts, per value of the next 8 key bits, the
// eligible keys whose top `bits` bits equal the prefix -- the caller sums
// the shards' histograms and steers the prefix; commit removes every
// eligible key whose top `bits` bits are <= the prefix (order-preserving
// compaction, engine.py:184-200).  tsg_reduce runs the loop for one store.
int tsg_reduce_begin(tsg_engine* h, int64_t eligible_below, int64_t* n_eligible) {
    CKR(validate_handle(h));
    if (!n_eligible) return fail(TSG_EINVAL, "null argument");
    if (any_inflight(h)) return fail(TSG_EINVAL, "the store cannot change while a launched round is not collected");
    DevGuard g(h->dev);
    select_free(h);
    auto& S = h->sel;
    S.base = bucket_bases(h, &S.flat);
    *n_eligible = 0;
    if (S.flat == 0) { S.open = true; S.store_seq = h->store_seq; return TSG_OK; }
    CKR(dalloc(h, (void**)&S.ka, S.flat * 8));
    CKR(dalloc(h, (void**)&S.ki, S.flat * 8));
    CKR(dalloc(h, (void**)&S.keep, S.flat));
    CKR(dalloc(h, (void**)&S.hist, 256 * 8));
    CK(cudaMemsetAsync(S.ka, 0xFF, S.flat * 8, h->st));  // padding: NO_KEY
    CK(cudaMemsetAsync(S.keep, 0, S.flat, h->st));
    CK(cudaMemsetAsync(h->mctr + 4, 0, 8, h->st));
    for (size_t bi = 0; bi < h->buckets.size(); ++bi) {
        const Bucket& b = h->buckets[bi];
        if (b.count)
            k_reduce_keys<<<grid_for(b.count), 256, 0, h->st>>>(b.acts, b.ids, b.count, S.base[bi], eligible_below,
                                                                S.ka, S.ki, S.keep, h->mctr + 4);
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h->h_mctr + 4, h->mctr + 4, 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    S.n_eligible = (int64_t)h->h_mctr[4];
    S.open = true;
    S.store_seq = h->store_seq;
    *n_eligible = S.n_eligible;
    return TSG_OK;
}

int tsg_reduce_hist(tsg_engine* h, uint64_t prefix_hi, uint64_t prefix_lo, int32_t bits, uint64_t* hist) {
    CKR(validate_handle(h));
    auto& S = h->sel;
    if (!S.open || S.store_seq != h->store_seq) return fail(TSG_EINVAL, "no reduce selection open on this store");
    if (bits < 0 || bits > 120 || bits % 8 || !hist) return fail(TSG_EINVAL, "bad prefix length %d", bits);
    if (S.flat == 0) { memset(hist, 0, 256 * 8); return TSG_OK; }
    DevGuard g(h->dev);
    CK(cudaMemsetAsync(S.hist, 0, 256 * 8, h->st));
    k_select_hist<<<grid_for(S.flat), 256, 0, h->st>>>(S.ka, S.ki, S.flat, prefix_hi, prefix_lo, bits, S.hist);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(hist, S.hist, 256 * 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    return TSG_OK;
}

int tsg_reduce_commit(tsg_engine* h, uint64_t prefix_hi, uint64_t prefix_lo, int32_t bits, int64_t* removed,
                      int64_t* removed_ids, int64_t cap) {
    CKR(validate_handle(h));
    if (!removed) return fail(TSG_EINVAL, "null argument");
    auto& S = h->sel;
    if (!S.open || S.store_seq != h->store_seq) return fail(TSG_EINVAL, "no reduce selection open on this store");
    if (bits < 0 || bits > 128 || bits % 8) return fail(TSG_EINVAL, "bad prefix length %d", bits);
    DevGuard g(h->dev);
    *removed = 0;
    int64_t rem = 0;
    if (S.flat && bits > 0) {
        int64_t* doomed = nullptr;
        CKR(dalloc(h, (void**)&doomed, std::max<int64_t>(S.n_eligible, 1) * 8));
        CK(cudaMemsetAsync(h->mctr + 3, 0, 8, h->st));
        k_select_mark<<<grid_for(S.flat), 256, 0, h->st>>>(S.ka, S.ki, S.flat, prefix_hi, prefix_lo, bits, S.keep,
                                                           doomed, h->mctr + 3);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h->h_mctr + 3, h->mctr + 3, 8, cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
        rem = (int64_t)h->h_mctr[3];
        if (removed_ids && rem > cap) { dfree(h, doomed); return fail(TSG_ECAPACITY, "%lld removed ids exceed %lld", (long long)rem, (long long)cap); }
        if (removed_ids && rem) {  // ascending engine id
            CK(cudaMemcpyAsync(removed_ids, doomed, rem * 8, cudaMemcpyDeviceToHost, h->st));
            CK(cudaStreamSynchronize(h->st));
            std::sort(removed_ids, removed_ids + rem);
        }
        if (rem) {
            h->desc_dirty = true;
            CKR(compact_all(h, S.keep, S.base, S.flat));
        }
        dfree(h, doomed);
    }
    select_free(h);
    CK(cudaStreamSynchronize(h->st));
    *removed = rem;
    h->totals.reduces += 1;
    h->totals.clauses_removed += rem;
    return TSG_OK;
}

int tsg_reduce(tsg_engine* h, int64_t eligible_below, int64_t target, int64_t* removed, int64_t* removed_ids) {
    CKR(validate_handle(h));
    if (!removed) return fail(TSG_EINVAL, "null argument");
    *removed = 0;
    if (store_size(h) == 0 || target <= 0) {  // nothing selected; still counts as a reduce
        if (any_inflight(h)) return fail(TSG_EINVAL, "the store cannot change while a launched round is not collected");
        h->totals.reduces += 1;
        return TSG_OK;
    }
    int64_t n_el = 0;
    CKR(tsg_reduce_begin(h, eligible_below, &n_el));
    const int64_t rem = std::min(target, n_el);
    // the prefix (ph, pl) of `bits` bits: rem - k keys lie strictly below it,
    // and k of the keys with this prefix are still to be taken
    uint64_t ph = 0, pl = 0;
    int bits = 0;
    int64_t k = rem;
    uint64_t hh[256];
    while (k > 0 && bits < 128) {
        CKR(tsg_reduce_hist(h, ph, pl, bits, hh));
        int d = 0;
        for (; d < 256 && (int64_t)hh[d] < k; ++d) k -= (int64_t)hh[d];
        if (d == 256) return fail(TSG_ECUDA, "reduce select lost %lld keys", (long long)k);
        if (bits < 64) ph |= (uint64_t)d << (56 - bits);
        else pl |= (uint64_t)d << (120 - bits);
        bits += 8;
        if ((int64_t)hh[d] == k) break;  // every key with this prefix goes
    }
    CKR(tsg_reduce_commit(h, ph, pl, rem > 0 ? bits : 0, removed, removed_ids, target));
    if (*removed != rem)
        return fail(TSG_ECUDA, "reduce select removed %lld of %lld keys", (long long)*removed, (long long)rem);
    return TSG_OK;
}

int tsg_remove_clauses(tsg_engine* h, const int64_t* ids, int64_t n, int64_t* removed) {
    CKR(validate_handle(h));
    if (!removed) return fail(TSG_EINVAL, "null argument");
    if (any_inflight(h)) return fail(TSG_EINVAL, "the store cannot change while a launched round is not collected");
    DevGuard g(h->dev);
    *removed = 0;
    if (store_size(h) == 0 || n <= 0) return TSG_OK;
    h->desc_dirty = true;
    int64_t flat = 0;
    const std::vector<int64_t> base = bucket_bases(h, &flat);
    std::vector<int64_t> del(ids, ids + n);
    std::sort(del.begin(), del.end());
    int64_t* d_del = nullptr;
    uint8_t* keep = nullptr;
    CKR(dalloc(h, (void**)&d_del, n * 8));
    CKR(dalloc(h, (void**)&keep, flat));
    CK(cudaMemcpyAsync(d_del, del.data(), n * 8, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemsetAsync(keep, 0, flat, h->st));
    CK(cudaMemsetAsync(h->mctr + 4, 0, 8, h->st));
    for (size_t bi = 0; bi < h->buckets.size(); ++bi) {
        const Bucket& b = h->buckets[bi];
        if (b.count)
            k_mark_deleted<<<grid_for(b.count), 256, 0, h->st>>>(b.ids, b.count, base[bi], d_del, n, keep, h->mctr + 4);
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h->h_mctr + 4, h->mctr + 4, 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    const int64_t gone = (int64_t)h->h_mctr[4];
    if (gone) CKR(compact_all(h, keep, base, flat));
    dfree(h, d_del); dfree(h, keep);
    CK(cudaStreamSynchronize(h->st));
    *removed = gone;
    h->totals.clauses_deleted += gone;
    return TSG_OK;
}

int tsg_stage_snapshots(tsg_engine* h, const int8_t* rows, int64_t n_rows, int64_t row_pitch, int32_t on_device) {
    CKR(validate_handle(h));
    DevGuard g(h->dev);
    if (n_rows < 0) return fail(TSG_EINVAL, "n_rows < 0");
    if (n_rows > 0 && row_pitch < h->V + 1) return fail(TSG_EINVAL, "row pitch %lld < num_vars+1", (long long)row_pitch);
    h->n_rows = n_rows;
    h->packed = false;
    if (n_rows == 0) return TSG_OK;
    if (on_device && row_pitch % 4 == 0) {  // encode straight from the caller's HBM rows
        h->rows = rows;
        h->pitch = row_pitch;
        return TSG_OK;
    }
    const int64_t pitch = round_up(h->V + 1, 16);
    const int64_t need = pitch * n_rows;
    if (need > h->rows_cap) {
        dfree(h, h->rows_own);
        h->rows_own = nullptr;
        const int64_t cap = std::max(need, h->rows_cap * 2);
        CKR(dalloc(h, (void**)&h->rows_own, cap));
        CK(cudaMemsetAsync(h->rows_own, 0, cap, h->st));  // pad bytes stay zero (Undef)
        h->rows_cap = cap;
    }
    CK(cudaMemcpy2DAsync(h->rows_own, pitch, rows, row_pitch, h->V + 1, n_rows,
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDefault, h->st));
    h->rows = h->rows_own;
    h->pitch = pitch;
    return TSG_OK;
}

int tsg_packed_words(int32_t num_vars, int64_t* words) {
    if (num_vars < 0) return fail(TSG_EINVAL, "num_vars < 0");
    *words = packed_words(num_vars);
    return TSG_OK;
}

// SWAR pack of one row into 2-bit words (AVX2 when the host has it)
__attribute__((target("avx2"))) static inline uint64_t pack_word_avx2(const int8_t* r) {
    const __m256i x = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(r));
    const uint32_t t = (uint32_t)_mm256_movemask_epi8(_mm256_cmpeq_epi8(x, _mm256_set1_epi8(1)));
    const uint32_t z = (uint32_t)_mm256_movemask_epi8(_mm256_cmpeq_epi8(x, _mm256_setzero_si256()));
    return (uint64_t)t | ((uint64_t)~z << 32);
}

__attribute__((target("avx2"))) static void pack_row_avx2(const int8_t* r, int64_t nv1, uint64_t* out, int64_t words) {
    // (plain stores: the packed rows stay in the last-level cache for the
    // copy engine's read -- streaming stores measured slower in the e2e loop)
    int64_t k = 0;
    for (; 32 * k + 32 <= nv1; ++k) out[k] = pack_word_avx2(r + 32 * k);
    for (; k < words; ++k) {
        uint32_t t = 0, st = 0;
        for (int64_t i = 32 * k; i < 32 * k + 32 && i < nv1; ++i) {
            t |= (uint32_t)(r[i] == 1) << (i - 32 * k);
            st |= (uint32_t)(r[i] != 0) << (i - 32 * k);
        }
        out[k] = (uint64_t)t | ((uint64_t)st << 32);
    }
}

static void pack_row_scalar(const int8_t* r, int64_t nv1, uint64_t* out, int64_t words) {
    for (int64_t k = 0; k < words; ++k) {
        uint32_t t = 0, st = 0;
        for (int64_t i = 32 * k; i < 32 * k + 32 && i < nv1; ++i) {
            t |= (uint32_t)(r[i] == 1) << (i - 32 * k);
            st |= (uint32_t)(r[i] != 0) << (i - 32 * k);
        }
        out[k] = (uint64_t)t | ((uint64_t)st << 32);
    }
}

int tsg_pack_rows(const int8_t* rows, int64_t n_rows, int64_t row_pitch, int32_t num_vars, uint64_t* out,
                  int64_t out_pitch_words) {
    if (n_rows < 0 || num_vars < 0) return fail(TSG_EINVAL, "negative size");
    const int64_t words = packed_words(num_vars);
    if (n_rows > 0 && (!rows || !out)) return fail(TSG_EINVAL, "null argument");
    if (n_rows > 0 && row_pitch < (int64_t)num_vars + 1)
        return fail(TSG_EINVAL, "row pitch %lld < num_vars+1", (long long)row_pitch);
    if (out_pitch_words < words) return fail(TSG_EINVAL, "out pitch %lld < %lld words", (long long)out_pitch_words, (long long)words);
    static const bool avx2 = __builtin_cpu_supports("avx2");
    auto pack = [&](int64_t a, int64_t b) {
        for (int64_t r = a; r < b; ++r) {
            uint64_t* o = out + r * out_pitch_words;
            if (avx2) pack_row_avx2(rows + r * row_pitch, (int64_t)num_vars + 1, o, words);
            else pack_row_scalar(rows + r * row_pitch, (int64_t)num_vars + 1, o, words);
            for (int64_t k = words; k < out_pitch_words; ++k) o[k] = 0;
        }
    };
    // a round's worth of rows (the solver threads pack one row each at
    // submit): split over the host worker pool -- the packing is bound by
    // host memory bandwidth, which one thread cannot draw
    const int64_t bytes = n_rows * ((int64_t)num_vars + 1);
    HostPool::get().parallel_for(n_rows, bytes >= ((int64_t)4 << 20) ? 16 : 1, pack);
    return TSG_OK;
}

int tsg_stage_packed(tsg_engine* h, const uint64_t* rows, int64_t n_rows, int64_t pitch_words, int32_t on_device) {
    CKR(validate_handle(h));
    DevGuard g(h->dev);
    const int64_t words = packed_words(h->V);
    if (n_rows < 0) return fail(TSG_EINVAL, "n_rows < 0");
    if (n_rows > 0 && pitch_words < words)
        return fail(TSG_EINVAL, "packed pitch %lld < %lld words", (long long)pitch_words, (long long)words);
    h->n_rows = n_rows;
    h->packed = true;
    h->pstaged = false;
    if (n_rows == 0) return TSG_OK;
    if (on_device && pitch_words % 4 == 0 && ((uintptr_t)rows % 32) == 0) {
        h->prows = rows;
        h->ppitch = pitch_words;
        return TSG_OK;
    }
    // copy into the staging buffer the previous stage did not use, on the
    // ingress stream, once the encoder that read it last is done (ev_read,
    // recorded by tsg_round_encode) -- not behind the rounds in flight
    const int b = h->pk ^ 1;
    const int64_t need = words * n_rows;
    CK(cudaStreamWaitEvent(h->ingress, h->ev_read[b], 0));
    if (need > h->pbuf_cap[b] || on_device) {
        if (need > h->pbuf_cap[b]) {
            dfree(h, h->pbuf[b]);  // stream-ordered after its last reader (the encoder runs on st)
            h->pbuf[b] = nullptr;
            const int64_t cap = std::max(need, h->pbuf_cap[b] * 2);
            CKR(dalloc(h, (void**)&h->pbuf[b], cap * 8));
            h->pbuf_cap[b] = cap;
        }
        // the allocation, and device-side sources written on h->st, come first
        CK(cudaEventRecord(h->ev_staged[b], h->st));
        CK(cudaStreamWaitEvent(h->ingress, h->ev_staged[b], 0));
    }
    if (pitch_words == words)
        CK(cudaMemcpyAsync(h->pbuf[b], rows, need * 8, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDefault,
                           h->ingress));
    else
        CK(cudaMemcpy2DAsync(h->pbuf[b], words * 8, rows, pitch_words * 8, words * 8, n_rows,
                             on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDefault, h->ingress));
    CK(cudaEventRecord(h->ev_staged[b], h->ingress));
    h->pk = b;
    h->pstaged = true;
    h->prows = h->pbuf[b];
    h->ppitch = words;
    return TSG_OK;
}

int tsg_stage_packed_mixed(tsg_engine* h, const uint64_t* packed, int64_t n_packed, int64_t pitch_words,
                           const int8_t* raw, int64_t n_raw, int64_t raw_pitch) {
    CKR(validate_handle(h));
    DevGuard g(h->dev);
    const int64_t words = packed_words(h->V);
    if (n_packed < 0 || n_raw < 0) return fail(TSG_EINVAL, "negative row count");
    if (n_packed > 0 && (!packed || pitch_words < words))
        return fail(TSG_EINVAL, "packed rows: null or pitch %lld < %lld words", (long long)pitch_words, (long long)words);
    if (n_raw > 0 && (!raw || raw_pitch < (int64_t)h->V + 1))
        return fail(TSG_EINVAL, "int8 rows: null or pitch %lld < num_vars+1", (long long)raw_pitch);
    const int64_t n = n_packed + n_raw;
    h->n_rows = n;
    h->packed = true;
    h->pstaged = false;
    if (n == 0) return TSG_OK;
    // as tsg_stage_packed: the staging buffer the previous stage did not use,
    // on the ingress stream; the int8 rows land in a device buffer of the
    // same slot and are packed on the device behind the packed ones
    const int b = h->pk ^ 1;
    const int64_t need = words * n;
    const int64_t rpitch = round_up((int64_t)h->V + 1, 16);
    CK(cudaStreamWaitEvent(h->ingress, h->ev_read[b], 0));
    bool grown = false;
    if (need > h->pbuf_cap[b]) {
        dfree(h, h->pbuf[b]);
        h->pbuf[b] = nullptr;
        const int64_t cap = std::max(need, h->pbuf_cap[b] * 2);
        CKR(dalloc(h, (void**)&h->pbuf[b], cap * 8));
        h->pbuf_cap[b] = cap;
        grown = true;
    }
    if (rpitch * n_raw > h->rawbuf_cap[b]) {
        dfree(h, h->rawbuf[b]);
        h->rawbuf[b] = nullptr;
        const int64_t cap = std::max(rpitch * n_raw, h->rawbuf_cap[b] * 2);
        CKR(dalloc(h, (void**)&h->rawbuf[b], cap));
        h->rawbuf_cap[b] = cap;
        grown = true;
    }
    if (grown) {  // the allocations (stream-ordered on st) come first
        CK(cudaEventRecord(h->ev_staged[b], h->st));
        CK(cudaStreamWaitEvent(h->ingress, h->ev_staged[b], 0));
    }
    if (n_packed > 0) {
        if (pitch_words == words)
            CK(cudaMemcpyAsync(h->pbuf[b], packed, n_packed * words * 8, cudaMemcpyDefault, h->ingress));
        else
            CK(cudaMemcpy2DAsync(h->pbuf[b], words * 8, packed, pitch_words * 8, words * 8, n_packed,
                                 cudaMemcpyDefault, h->ingress));
    }
    if (n_raw > 0) {
        CK(cudaMemcpy2DAsync(h->rawbuf[b], rpitch, raw, raw_pitch, h->V + 1, n_raw, cudaMemcpyDefault, h->ingress));
        k_pack_rows<<<grid_for(n_raw * words), 256, 0, h->ingress>>>(h->rawbuf[b], rpitch, n_raw, (int64_t)h->V + 1,
                                                                     h->pbuf[b] + n_packed * words, words, words);
        CK(cudaGetLastError());
    }
    CK(cudaEventRecord(h->ev_staged[b], h->ingress));
    h->pk = b;
    h->pstaged = true;
    h->prows = h->pbuf[b];
    h->ppitch = words;
    return TSG_OK;
}

int tsg_round_prepare(tsg_engine* h, const int32_t* group_lanes, const int32_t* group_tid, int32_t n_groups) {
    CKR(validate_handle(h));
    DevGuard g(h->dev);
    if (n_groups < 0 || n_groups > TSG_MAX_GROUPS)
        return fail(TSG_EINVAL, "n_groups must be in 0..%d, got %d", TSG_MAX_GROUPS, n_groups);
    if (n_groups > 0 && (!group_lanes || !group_tid)) return fail(TSG_EINVAL, "null argument");
    RoundDesc rd;
    rd.n_groups = n_groups;
    rd.glanes.assign(group_lanes, group_lanes + n_groups);
    rd.gtid.assign(group_tid, group_tid + n_groups);
    rd.grow0.resize(n_groups);
    int64_t r = 0;
    std::unordered_set<int32_t> closed;  // threads whose run of groups has ended
    for (int i = 0; i < n_groups; ++i) {
        if (rd.glanes[i] < 0 || rd.glanes[i] > h->cfg.lane_width)
            return fail(TSG_ECAPACITY, "%d assignments exceed lane width %d", rd.glanes[i], h->cfg.lane_width);
        // a thread's groups are consecutive (engine.py:390-399 groups per sorted
        // tid): the kernel's one-report-per-(clause, thread) rule relies on it
        if (i > 0 && rd.gtid[i] != rd.gtid[i - 1]) {
            closed.insert(rd.gtid[i - 1]);
            if (closed.count(rd.gtid[i]))
                return fail(TSG_EINVAL, "thread %d's groups are not consecutive (group %d)", rd.gtid[i], i);
        }
        rd.grow0[i] = r;
        r += rd.glanes[i];
    }
    rd.n_chunks = (n_groups + h->cfg.group_width - 1) / h->cfg.group_width;
    rd.chunk_stride = chunk_bytes(h);
    rd.per_bit = std::max(1, (rd.n_chunks + 31) / 32);
    rd.top_off = (int64_t)rd.n_chunks * rd.chunk_stride;
    const int64_t off = rd.top_off + (rd.n_chunks > 1 ? top_bytes(h) : 0);
    // table slots never shrink and hold at least one full chunk, so rounds of
    // up to group_width groups can be prepared while another is in flight
    const int64_t slot = std::max(h->slot_bytes, round_up(std::max(off, chunk_bytes(h)), 4096));
    if (slot != h->slot_bytes) {
        // grow both slots; stream order keeps in-flight rounds valid: their
        // kernels precede the copy, and a later replay reads the moved slot
        int8_t* nt = nullptr;
        CKR(dalloc(h, (void**)&nt, 2 * slot));
        if (h->tables && any_inflight(h))
            for (int i = 0; i < 2; ++i)
                CK(cudaMemcpyAsync(nt + i * slot, h->tables + i * h->slot_bytes, h->slot_bytes,
                                   cudaMemcpyDeviceToDevice, h->st));
        dfree(h, h->tables);
        h->tables = nt;
        h->slot_bytes = slot;
    }
    h->tables_bytes = off;
    h->rd = std::move(rd);
    return TSG_OK;
}

// Launch the test of the prepared, encoded round (table slot h->tslot) in
// the next round state: group upload, kernel and its event are queued,
// nothing waits.  At most two rounds are in flight.
int round_launch(tsg_engine* h, double inc, bool flip) {
    const int k = h->next_rs;
    auto& R = h->rs[k];
    if (R.inflight) return fail(TSG_EINVAL, "two rounds are in flight: collect one first");
    for (const auto& Q : h->rs)
        if (Q.inflight && Q.slot == h->tslot)
            return fail(TSG_EINVAL, "table slot %d still belongs to an uncollected round", h->tslot);
    if (h->ring.slots) {
        if (h->ring.ctl[1])
            return fail(TSG_ECAPACITY, "the report ring dropped records of an earlier round: close and reopen it");
        if (h->max_id >= (int64_t(1) << 48))
            return fail(TSG_ECAPACITY, "report ring records carry 48-bit engine ids (largest id %lld)", (long long)h->max_id);
    }
    // this state's record buffer may still be copying out from two rounds ago
    CK(cudaStreamWaitEvent(h->st, R.ev_copied, 0));
    R.n_out = 0;
    R.fl = h->rd;
    R.slot = h->tslot;
    R.inc = inc;
    R.seq = ++h->round_seq;
    R.all_pairs = h->all_pairs;
    // 8-byte egress: the kernel writes the packed u64 records itself when
    // they fit (ids < 2^27, <= 32 groups, 32-bit lane masks)
    R.rec8 = h->record_bytes == 8 && !wide_lane(h) && h->max_id < (int64_t(1) << 27) && h->rd.n_groups <= 32;
    R.ringed = h->ring.slots != nullptr;
    if (R.ringed) R.rec8 = false;  // the kernel's buffer holds 16-byte records; the ring words are its own
    const RoundDesc& rd = R.fl;
    if (rd.n_chunks && h->oob) {  // out-of-range literal stored: numpy would raise IndexError
        CK(cudaMemsetAsync(h->mctr + 4, 0, 8, h->st));
        for (auto& b : h->buckets)
            if (b.count && b.size)
                k_max_var<<<grid_for(b.count * b.size), 256, 0, h->st>>>(b.lits, b.count, b.size, h->mctr + 4);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h->h_mctr + 4, h->mctr + 4, 8, cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
        if ((int64_t)h->h_mctr[4] > h->V)
            return fail(TSG_ERANGE, "index %lld is out of bounds for axis 0 with size %d", (long long)h->h_mctr[4], h->V + 1);
        h->oob = false;
    }
    if (rd.n_chunks) {
        CKR(build_desc(h));
        if (h->n_tiles >= (int64_t)1 << 30)  // the kernel indexes tiles and slots with 32-bit integers
            return fail(TSG_ECAPACITY, "store of %lld tiles exceeds the 32-bit tile index", (long long)h->n_tiles);
        if (rd.n_groups > R.groups_cap) {
            dfree(h, R.d_groups);
            R.d_groups = nullptr;
            if (R.h_groups) { CK(cudaStreamSynchronize(h->st)); cudaFreeHost(R.h_groups); R.h_groups = nullptr; }
            const int64_t cap = std::max<int64_t>(64, rd.n_groups);
            CKR(dalloc(h, (void**)&R.d_groups, cap * (int64_t)sizeof(GroupDesc)));
            CK(cudaMallocHost(&R.h_groups, cap * sizeof(GroupDesc)));
            R.groups_cap = cap;
        }
        // (the pinned staging is free: this state's previous round was collected)
        for (int g = 0; g < rd.n_groups; ++g)
            R.h_groups[g] = GroupDesc{width_mask<uint64_t>(rd.glanes[g]), rd.gtid[g], 0};
        CK(cudaMemcpyAsync(R.d_groups, R.h_groups, rd.n_groups * sizeof(GroupDesc), cudaMemcpyHostToDevice, h->st));
        const bool timing = timed_round(h, R.seq);
        R.timed = timing;
        if (timing) CK(cudaEventRecord(R.ev_tst[0], h->st));
        if (h->n_tiles) CKR(run_test(h, k, 0));
        if (timing) CK(cudaEventRecord(R.ev_tst[1], h->st));
        if (h->n_tiles == 0) {  // no kernel ran to publish the counters
            CK(cudaMemcpyAsync(R.h_ctr, R.ctr, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->st));
            CK(cudaMemsetAsync(R.ctr, 0, 8 * sizeof(unsigned long long), h->st));
        }
        CK(cudaEventRecord(R.ev_done, h->st));
    }
    R.inflight = true;
    R.pol_pending = false;
    h->next_rs ^= 1;
    if (flip) h->tslot ^= 1;
    return TSG_OK;
}

// Collect the oldest launched round: wait for its counters; grow its record
// buffer and replay emission if it overflowed (its table slot is its own, so
// the replay is exact even with the next round in flight); fill its figures.
// The fetch calls then read its records.
int round_collect(tsg_engine* h, tsg_round_result* out) {
    int k = -1;
    for (int j = 0; j < 2; ++j)
        if (h->rs[j].inflight && (k < 0 || h->rs[j].seq < h->rs[k].seq)) k = j;
    if (k < 0) return fail(TSG_EINVAL, "no launched round to collect");
    auto& R = h->rs[k];
    R.inflight = false;
    h->fetch_rs = k;
    const RoundDesc& rd = R.fl;
    tsg_round_result res{};
    res.n_chunks = rd.n_chunks;
    if (rd.n_chunks) {
        CK(cudaEventSynchronize(R.ev_done));
        // literal placement for the next inserts: the polarity that is
        // non-False more often under this round's assignments goes right
        // after the pivot (ends the early-exit recurrence sooner)
        if (!h->prefer_fixed && R.h_ctr[6] + R.h_ctr[7] > 0)
            h->prefer = R.h_ctr[7] < R.h_ctr[6] ? 1 : (R.h_ctr[7] > R.h_ctr[6] ? -1 : 0);
        const int64_t n_rec = (int64_t)R.h_ctr[0];
        const int64_t positives = (int64_t)R.h_ctr[1];
        res.lane_triggers = (int64_t)R.h_ctr[2];
        // overflow: grow and replay emission only (no activity / counter side
        // effects); the record count is exact, so one replay suffices
        if (R.ringed) {
            h->ring.expected += n_rec;
            if (h->ring.ctl[1])
                return fail(TSG_ECAPACITY, "report ring full for longer than %lld us: records of round %lld were dropped "
                            "(drain the ring while rounds run, or open a larger one)",
                            (long long)(h->ring.wait_ns / 1000), (long long)R.seq);
        } else if (n_rec > R.out_cap) {
            dfree(h, R.out);
            R.out = nullptr;
            R.out_cap = n_rec + n_rec / 4 + 1024;
            CKR(dalloc(h, (void**)&R.out, R.out_cap * (int64_t)sizeof(tsg_report)));
            CK(cudaMemsetAsync(R.ctr, 0, 4 * sizeof(unsigned long long), h->st));
            CKR(run_test(h, k, 1));
            unsigned long long rc[4];
            CK(cudaMemcpyAsync(rc, R.ctr, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->st));
            CK(cudaMemsetAsync(R.ctr, 0, 4 * sizeof(unsigned long long), h->st));
            CK(cudaStreamSynchronize(h->st));
            if ((int64_t)rc[0] != n_rec)
                return fail(TSG_ECUDA, "report replay mismatch: %lld records, %lld in the first run",
                            (long long)rc[0], (long long)n_rec);
            res.reruns = 1;
        }
        R.n_out = R.ringed ? 0 : n_rec;
        const int64_t n = store_size(h);
        int64_t lanes_total = 0;
        for (int g = 0; g < rd.n_groups; ++g) lanes_total += rd.glanes[g];
        res.clauses_tested = n * rd.n_chunks;
        // (clause, chunk) pairs past the chunk-level sweep (every pair when it does not run)
        res.chunk_positives = rd.n_chunks > 1 && h->chunk_filter ? (int64_t)R.h_ctr[3] : res.clauses_tested;
        res.aggregate_tests = n * rd.n_groups;
        res.lane_tests = n * lanes_total;
        res.aggregate_tests_negative = res.aggregate_tests - positives;
        res.reports = n_rec;
        res.encode_ms = res.test_ms = -1.0;  // not sampled
        if (R.timed) {
            float ms = 0;
            if (cudaEventElapsedTime(&ms, h->ev_enc[R.slot][0], h->ev_enc[R.slot][1]) == cudaSuccess) res.encode_ms = ms;
            else cudaGetLastError();
            if (cudaEventElapsedTime(&ms, R.ev_tst[0], R.ev_tst[1]) == cudaSuccess) res.test_ms = ms;
            else cudaGetLastError();
        }
    }
    auto& T = h->totals;
    T.rounds += 1;
    T.reports += res.reports;
    T.clauses_tested += res.clauses_tested;
    T.aggregate_tests += res.aggregate_tests;
    T.aggregate_tests_negative += res.aggregate_tests_negative;
    T.lane_tests += res.lane_tests;
    T.lane_triggers += res.lane_triggers;
    T.reruns += res.reruns;
    if (out) *out = res;
    return TSG_OK;
}

int tsg_round_encode(tsg_engine* h) {
    CKR(validate_handle(h));
    DevGuard g(h->dev);
    const int64_t need_rows = h->rd.n_groups ? h->rd.grow0.back() + h->rd.glanes.back() : 0;
    if (need_rows > h->n_rows) return fail(TSG_EINVAL, "groups need %lld rows, %lld staged", (long long)need_rows, (long long)h->n_rows);
    if (!h->rd.n_chunks) return TSG_OK;
    for (const auto& Q : h->rs)
        if (Q.inflight && Q.slot == h->tslot)
            return fail(TSG_EINVAL, "table slot %d still belongs to an uncollected round", h->tslot);
    if (h->packed && h->pstaged) CK(cudaStreamWaitEvent(h->st, h->ev_staged[h->pk], 0));  // rows copied in
    const bool timing = timed_round(h, h->round_seq + 1);  // the round this encode feeds
    if (timing) CK(cudaEventRecord(h->ev_enc[h->tslot][0], h->st));
    auto& Rn = h->rs[h->next_rs];
    if (Rn.pol_pending)  // re-encoded without a launch: count this encode only
        CK(cudaMemsetAsync(Rn.ctr + 6, 0, 2 * sizeof(unsigned long long), h->st));
    Rn.pol_pending = true;
    const int rc = do_encode(h);
    if (h->packed && h->pstaged) CK(cudaEventRecord(h->ev_read[h->pk], h->st));
    if (timing) CK(cudaEventRecord(h->ev_enc[h->tslot][1], h->st));
    return rc;
}

// One rank's share of a round's encode when the snapshot ingress is split
// across GPUs: the staged packed rows hold exactly groups
// [g_begin, g_end); their lane entries are written, the other groups' are
// left for the all-gather, and the aggregate words carry only these groups'
// bits, so a sum all-reduce over the ranks ORs them (the bits are disjoint).
// `sentinel`: this rank writes the always-False entry (exactly one rank).
int tsg_round_encode_groups(tsg_engine* h, int32_t g_begin, int32_t g_end, int32_t sentinel) {
    CKR(validate_handle(h));
    const RoundDesc& rd = h->rd;
    if (rd.n_chunks != 1 || wide_lane(h) || !h->packed)
        return fail(TSG_EINVAL, "group-range encode needs one chunk, lane_width <= 32 and packed rows");
    if (g_begin < 0 || g_end > rd.n_groups || g_begin >= g_end)
        return fail(TSG_EINVAL, "group range [%d, %d) outside 0..%d", g_begin, g_end, rd.n_groups);
    const int64_t need = rd.grow0[g_end - 1] + rd.glanes[g_end - 1] - rd.grow0[g_begin];
    if (need > h->n_rows) return fail(TSG_EINVAL, "groups need %lld rows, %lld staged", (long long)need, (long long)h->n_rows);
    h->enc_g0 = g_begin;
    h->enc_g1 = g_end;
    h->enc_sentinel = sentinel != 0;
    const int64_t keep_rows = h->n_rows;
    h->n_rows = std::max<int64_t>(h->n_rows, rd.n_groups ? rd.grow0.back() + rd.glanes.back() : 0);  // row check of the full round
    const int rc = tsg_round_encode(h);
    h->n_rows = keep_rows;
    h->enc_g0 = 0;
    h->enc_g1 = -1;
    h->enc_sentinel = true;
    return rc;
}

// Byte layout of the prepared round's tables (first chunk): the aggregate
// table at agg_off (agg_bytes), then group g's lane entries at lane_off +
// g * group_bytes -- the regions tsg_round_encode_groups ranks combine.
int tsg_round_layout(tsg_engine* h, int64_t* agg_off, int64_t* agg_len, int64_t* lane_off, int64_t* group_bytes) {
    CKR(validate_handle(h));
    if (h->rd.n_chunks < 1) return fail(TSG_EINVAL, "no prepared round");
    *agg_off = 0;
    *agg_len = (int64_t)(h->V + 2) * agg_entry_bytes(h);
    *lane_off = agg_bytes(h);
    *group_bytes = vstride(h) * lane_entry_bytes(h);
    return TSG_OK;
}

int tsg_round_tables(tsg_engine* h, void** device_ptr, int64_t* bytes) {
    CKR(validate_handle(h));
    *device_ptr = h->tables + h->tslot * h->slot_bytes;
    *bytes = h->tables_bytes;
    return TSG_OK;
}

// In-process table broadcast (one engine per GPU in one process, DESIGN.md
// §6): copy the encoded tables of `src`'s prepared round into `dst`'s table
// slot over NVLink (peer copy), ordered after src's encode on dst's stream;
// src's next use of its slot waits for the copy.  Both must have prepared
// the same round.
int tsg_round_tables_copy(tsg_engine* dst, tsg_engine* src) {
    CKR(validate_handle(dst));
    CKR(validate_handle(src));
    if (dst->tables_bytes != src->tables_bytes || dst->V != src->V || dst->rd.n_groups != src->rd.n_groups)
        return fail(TSG_EINVAL, "the engines have not prepared the same round");
    for (const auto& Q : dst->rs)
        if (Q.inflight && Q.slot == dst->tslot)
            return fail(TSG_EINVAL, "table slot %d still belongs to an uncollected round", dst->tslot);
    if (dst->tables_bytes == 0) return TSG_OK;
    {
        DevGuard g(src->dev);
        CK(cudaEventRecord(src->ev_peer, src->st));
    }
    DevGuard g(dst->dev);
    if (dst->dev != src->dev) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, dst->dev, src->dev);
        if (can) {
            cudaError_t e = cudaDeviceEnablePeerAccess(src->dev, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return fail(TSG_ECUDA, "peer access: %s", cudaGetErrorString(e));
            cudaGetLastError();
        }
    }
    CK(cudaStreamWaitEvent(dst->st, src->ev_peer, 0));
    CK(cudaMemcpyPeerAsync(dst->tables + dst->tslot * dst->slot_bytes, dst->dev,
                           src->tables + src->tslot * src->slot_bytes, src->dev, dst->tables_bytes, dst->st));
    CK(cudaEventRecord(dst->ev_peer, dst->st));
    {
        DevGuard g2(src->dev);
        CK(cudaStreamWaitEvent(src->st, dst->ev_peer, 0));
    }
    auto& Rn = dst->rs[dst->next_rs];  // no encode counted polarity for dst's next round
    if (Rn.pol_pending) CK(cudaMemsetAsync(Rn.ctr + 6, 0, 2 * sizeof(unsigned long long), dst->st));
    Rn.pol_pending = false;
    return TSG_OK;
}

int tsg_round_test(tsg_engine* h, double activity_inc, tsg_round_result* out) {
    CKR(validate_handle(h));
    DevGuard g(h->dev);
    CKR(round_launch(h, activity_inc, false));
    return round_collect(h, out);
}

int tsg_round_launch(tsg_engine* h, double activity_inc) {
    CKR(validate_handle(h));
    DevGuard g(h->dev);
    return round_launch(h, activity_inc, true);
}

int tsg_round_collect(tsg_engine* h, tsg_round_result* out) {
    CKR(validate_handle(h));
    DevGuard g(h->dev);
    return round_collect(h, out);
}

int tsg_round(tsg_engine* h, const int32_t* group_lanes, const int32_t* group_tid, int32_t n_groups,
              double activity_inc, tsg_round_result* out) {
    CKR(tsg_round_prepare(h, group_lanes, group_tid, n_groups));
    CKR(tsg_round_encode(h));
    return tsg_round_test(h, activity_inc, out);
}

namespace {
// the source and size of the last collected round's first k records in the
// egress format (repacked on the compute stream when it differs)
int egress_view(tsg_engine* h, int64_t k, const void** src, int64_t* bytes) {
    auto& R = h->rs[h->fetch_rs];
    if (R.rec8) {  // written as 8-byte records by the kernel
        if (h->record_bytes != 8)
            return fail(TSG_EINVAL, "the round was launched with 8-byte records; fetch it before changing the format");
        *src = R.out;
        *bytes = k * 8;
        return TSG_OK;
    }
    if (h->record_bytes == 16 || k <= 0) {
        *src = R.out;
        *bytes = k * (int64_t)sizeof(tsg_report);
        return TSG_OK;
    }
    if (h->record_bytes == 8) {
        if (h->max_id >= (int64_t(1) << 27) || R.fl.n_groups > 32)
            return fail(TSG_ECAPACITY, "8-byte records need engine ids < 2^27 and <= 32 groups (largest id %lld, "
                        "%d groups): use 12-byte records", (long long)h->max_id, R.fl.n_groups);
        CKR(dgrow(h, &R.out12, &R.out12_cap, k * 8));
        k_pack_records8<<<grid_for(k), 256, 0, h->st>>>(R.out, k, reinterpret_cast<uint64_t*>(R.out12));
        CK(cudaGetLastError());
        *src = R.out12;
        *bytes = k * 8;
        return TSG_OK;
    }
    CKR(dgrow(h, &R.out12, &R.out12_cap, k * 12));
    k_pack_records12<<<grid_for(k), 256, 0, h->st>>>(R.out, k, R.out12);
    CK(cudaGetLastError());
    *src = R.out12;
    *bytes = k * 12;
    return TSG_OK;
}
}  // namespace

namespace {
int not_ringed(const tsg_engine* h) {
    if (h->rs[h->fetch_rs].ringed)
        return fail(TSG_EINVAL, "the round's records went to the host report ring: read them with tsg_ring_drain");
    return TSG_OK;
}
}  // namespace

int tsg_fetch_reports(tsg_engine* h, tsg_report* out, int64_t cap, int64_t* n) {
    CKR(validate_handle(h));
    CKR(not_ringed(h));
    DevGuard g(h->dev);
    const int64_t k = std::min(cap, h->rs[h->fetch_rs].n_out);
    if (k > 0) {
        const void* src = nullptr;
        int64_t bytes = 0;
        CKR(egress_view(h, k, &src, &bytes));
        CK(cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
    }
    *n = std::max<int64_t>(k, 0);
    return TSG_OK;
}

int tsg_set_record_bytes(tsg_engine* h, int32_t bytes) {
    CKR(validate_handle(h));
    if (bytes != 16 && bytes != 12 && bytes != 8)
        return fail(TSG_EINVAL, "record bytes must be 16, 12 or 8, got %d", bytes);
    if (bytes != 16 && h->cfg.lane_width > 32)
        return fail(TSG_EINVAL, "%d-byte records carry a 32-bit lane mask: lane_width %d > 32", bytes, h->cfg.lane_width);
    h->record_bytes = bytes;
    return TSG_OK;
}

int tsg_fetch_reports_async(tsg_engine* h, tsg_report* out, int64_t cap, int64_t* n) {
    CKR(validate_handle(h));
    CKR(not_ringed(h));
    DevGuard g(h->dev);
    auto& R = h->rs[h->fetch_rs];
    const int64_t k = std::min(cap, R.n_out);
    *n = std::max<int64_t>(k, 0);
    if (k <= 0) return TSG_OK;
    const void* src = nullptr;
    int64_t bytes = 0;
    CKR(egress_view(h, k, &src, &bytes));
    CK(cudaEventRecord(h->ev_ready, h->st));
    CK(cudaStreamWaitEvent(h->egress, h->ev_ready, 0));
    CK(cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToHost, h->egress));
    CK(cudaEventRecord(R.ev_copied, h->egress));
    return TSG_OK;
}

int tsg_fetch_wait(tsg_engine* h) {
    CKR(validate_handle(h));
    DevGuard g(h->dev);
    CK(cudaStreamSynchronize(h->egress));
    return TSG_OK;
}

int tsg_reports_device(tsg_engine* h, void** device_ptr, int64_t* n) {
    CKR(validate_handle(h));
    CKR(not_ringed(h));
    auto& R = h->rs[h->fetch_rs];
    if (R.rec8) return fail(TSG_EINVAL, "the round's records are 8-byte u64 (tsg_set_record_bytes(8)), not tsg_report");
    *device_ptr = R.out;
    *n = R.n_out;
    return TSG_OK;
}

int tsg_sync(tsg_engine* h) {
    CKR(validate_handle(h));
    DevGuard g(h->dev);
    CK(cudaStreamSynchronize(h->st));
    return TSG_OK;
}

int tsg_stream(tsg_engine* h, void** stream) {
    CKR(validate_handle(h));
    *stream = (void*)h->st;
    return TSG_OK;
}

// Pinned host memory for ingress rows / egress records (page-locked, so the
// copies run at link rate and asynchronously).
int tsg_host_alloc(int64_t bytes, void** p) {
    if (!p || bytes < 0) return fail(TSG_EINVAL, "bad arguments");
    *p = nullptr;
    if (bytes == 0) return TSG_OK;
    CK(cudaMallocHost(p, (size_t)bytes));
    return TSG_OK;
}

int tsg_host_free(void* p) {
    if (p) CK(cudaFreeHost(p));
    return TSG_OK;
}

// Device memory on the engine's device, and a host-to-device copy on the
// engine's ingress stream -- the snapshot queues of the Engine: a solver
// thread packs its snapshot into page-locked memory and queues its copy into
// the thread's device queue region at submit time, so a round's rows are on
// the device before the round starts.  tsg_ingress_copy is the one entry
// point that other host threads may call concurrently with the engine's
// worker (it touches only the ingress stream).
int tsg_device_alloc(tsg_engine* h, int64_t bytes, void** p) {
    CKR(validate_handle(h));
    if (!p || bytes < 0) return fail(TSG_EINVAL, "bad arguments");
    *p = nullptr;
    if (!bytes) return TSG_OK;
    DevGuard g(h->dev);
    CK(cudaMalloc(p, (size_t)bytes));
    return TSG_OK;
}

int tsg_device_free(tsg_engine* h, void* p) {
    CKR(validate_handle(h));
    if (!p) return TSG_OK;
    DevGuard g(h->dev);
    CK(cudaStreamSynchronize(h->ingress));  // no queued copy still targets it
    CK(cudaFree(p));
    return TSG_OK;
}

int tsg_ingress_copy(tsg_engine* h, void* dst, const void* src, int64_t bytes) {
    CKR(validate_handle(h));
    if (bytes < 0 || (bytes && (!dst || !src))) return fail(TSG_EINVAL, "bad arguments");
    if (!bytes) return TSG_OK;
    DevGuard g(h->dev);
    CK(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, h->ingress));
    return TSG_OK;
}

// The next round's packed rows from several segments in host or device
// memory (segment i: rows[i] rows at segs[i], pitch_words apart),
// concatenated in order -- the per-thread snapshot queues of the Engine,
// grouped by tid, without a host copy.  Same staging buffers and ingress
// stream as tsg_stage_packed (so copies queued by tsg_ingress_copy land
// first).
int tsg_stage_packed_segments(tsg_engine* h, const uint64_t* const* segs, const int64_t* rows, int32_t n_segs,
                              int64_t pitch_words) {
    CKR(validate_handle(h));
    if (n_segs < 0 || (n_segs > 0 && (!segs || !rows))) return fail(TSG_EINVAL, "bad arguments");
    DevGuard g(h->dev);
    const int64_t words = packed_words(h->V);
    if (pitch_words < words) return fail(TSG_EINVAL, "packed pitch %lld < %lld words", (long long)pitch_words, (long long)words);
    int64_t n_rows = 0;
    for (int32_t i = 0; i < n_segs; ++i) {
        if (rows[i] < 0) return fail(TSG_EINVAL, "segment %d: negative row count", i);
        n_rows += rows[i];
    }
    h->n_rows = n_rows;
    h->packed = true;
    h->pstaged = false;
    if (n_rows == 0) return TSG_OK;
    const int b = h->pk ^ 1;
    const int64_t need = words * n_rows;
    CK(cudaStreamWaitEvent(h->ingress, h->ev_read[b], 0));
    if (need > h->pbuf_cap[b]) {
        dfree(h, h->pbuf[b]);
        h->pbuf[b] = nullptr;
        const int64_t cap = std::max(need, h->pbuf_cap[b] * 2);
        CKR(dalloc(h, (void**)&h->pbuf[b], cap * 8));
        h->pbuf_cap[b] = cap;
        CK(cudaEventRecord(h->ev_staged[b], h->st));
        CK(cudaStreamWaitEvent(h->ingress, h->ev_staged[b], 0));
    }
    int64_t r = 0;
    for (int32_t i = 0; i < n_segs; ++i) {
        if (!rows[i]) continue;
        if (pitch_words == words)
            CK(cudaMemcpyAsync(h->pbuf[b] + r * words, segs[i], rows[i] * words * 8, cudaMemcpyDefault, h->ingress));
        else
            CK(cudaMemcpy2DAsync(h->pbuf[b] + r * words, words * 8, segs[i], pitch_words * 8, words * 8, rows[i],
                                 cudaMemcpyDefault, h->ingress));
        r += rows[i];
    }
    CK(cudaEventRecord(h->ev_staged[b], h->ingress));
    h->pk = b;
    h->pstaged = true;
    h->prows = h->pbuf[b];
    h->ppitch = words;
    return TSG_OK;
}

namespace {
int bits_for(int64_t max_value) {  // bits to hold 0..max_value
    int b = 0;
    while (b < 63 && (max_value >> b) > 0) ++b;
    return b;
}
}  // namespace

// The last collected round's records of one or more engines (clause shards
// of one round: same groups) in the reference's delivery order: destination
// thread (ascending tid) major, then chunk, creation rank of the clause's
// size bucket (rank_of_size[size], the caller's global bucket order), engine
// id, group (engine.py:403-414, 462-464).  Keys are built on each engine's
// device, the shards' records gathered to hs[0]'s device, sorted there
// (stable LSD radix sort, tsg_sort.cuh) and written into the host arrays:
// eids (eid_bytes 4 or 8), masks (mask_bytes 4 or 8), and per destination
// the record count (dest_counts[d], d = index of the thread's run of groups).
constexpr int64_t SMALL_ORDER_MAX = 16384;  // records ordered on the host below this (tsg_fetch_ordered)

int tsg_fetch_ordered(tsg_engine* const* hs, int32_t n_h, const int32_t* rank_of_size, int32_t n_sizes,
                      void* eids, int32_t eid_bytes, void* masks, int32_t mask_bytes, int32_t* groups,
                      int64_t* dest_counts, int64_t cap, int64_t* n) {
    if (!hs || n_h < 1 || !n || !dest_counts || !rank_of_size || n_sizes < 1) return fail(TSG_EINVAL, "bad arguments");
    if ((eid_bytes != 4 && eid_bytes != 8) || (mask_bytes != 4 && mask_bytes != 8))
        return fail(TSG_EINVAL, "eid_bytes / mask_bytes must be 4 or 8");
    tsg_engine* h0 = hs[0];
    CKR(validate_handle(h0));
    const RoundDesc& rd = h0->rs[h0->fetch_rs].fl;
    const bool rec8 = h0->rs[h0->fetch_rs].rec8;
    int64_t total = 0, max_id = 0;
    for (int32_t s = 0; s < n_h; ++s) {
        CKR(validate_handle(hs[s]));
        CKR(not_ringed(hs[s]));
        const auto& R = hs[s]->rs[hs[s]->fetch_rs];
        if (R.fl.n_groups != rd.n_groups || R.fl.gtid != rd.gtid || R.rec8 != rec8 ||
            hs[s]->cfg.group_width != h0->cfg.group_width)
            return fail(TSG_EINVAL, "engine %d's last round differs from engine 0's", s);
        if (!hs[s]->size_of_id && R.n_out) return fail(TSG_EINVAL, "engine %d has no clause size table", s);
        total += R.n_out;
        max_id = std::max(max_id, hs[s]->max_id);
    }
    // destinations: runs of equal tids in round order
    std::vector<int32_t> dest_of(rd.n_groups);
    int32_t n_dest = 0;
    for (int g = 0; g < rd.n_groups; ++g) {
        if (g > 0 && rd.gtid[g] != rd.gtid[g - 1]) ++n_dest;
        dest_of[g] = n_dest;
    }
    n_dest = rd.n_groups ? n_dest + 1 : 0;
    for (int32_t d = 0; d < n_dest; ++d) dest_counts[d] = 0;
    *n = total;
    if (total == 0) return TSG_OK;
    if (total > cap) return fail(TSG_ECAPACITY, "%lld records exceed %lld", (long long)total, (long long)cap);
    if (total >= ((int64_t)1 << 32)) return fail(TSG_ECAPACITY, "%lld records exceed the 32-bit sort index", (long long)total);
    if (eid_bytes == 4 && max_id >= ((int64_t)1 << 31)) return fail(TSG_ECAPACITY, "engine ids do not fit 4 bytes");
    if (mask_bytes == 4 && h0->cfg.lane_width > 32) return fail(TSG_ECAPACITY, "lane masks do not fit 4 bytes");
    const int gw = h0->cfg.group_width;
    const int dest_bits = bits_for(n_dest - 1), chunk_bits = bits_for(rd.n_chunks - 1);
    const int rank_bits = bits_for(n_sizes - 1), id_bits = bits_for(max_id), g_bits = bits_for(gw - 1);
    const int low_bits = chunk_bits + rank_bits + id_bits + g_bits;  // the destination field sits above
    const int key_bits = dest_bits + low_bits;
    if (key_bits > 64) return fail(TSG_ECAPACITY, "record order key needs %d bits", key_bits);
    std::vector<uint64_t> gkey(rd.n_groups);
    for (int g = 0; g < rd.n_groups; ++g) gkey[g] = ((uint64_t)dest_of[g] << chunk_bits) | (uint64_t)(g / gw);
    const int64_t rec_bytes = rec8 ? 8 : 16;
    if (n_h == 1 && total <= SMALL_ORDER_MAX) {
        // a small round: the keys from the device (one launch), then keys and
        // records copied out together and sorted on the host -- the radix
        // pipeline's ~20 launches cost more than the sort itself here
        DevGuard g1(h0->dev);
        const auto& R = h0->rs[h0->fetch_rs];
        // persistent scratch (page-locked host, device): group keys and size
        // ranks up, keys and records down, all asynchronous, one sync
        const int64_t o_rank = round_up((int64_t)rd.n_groups * 8, 16), o_keys = o_rank + round_up((int64_t)n_sizes * 4, 16);
        const int64_t o_recs = o_keys + round_up(total * 8, 16), o_vals = o_recs + round_up(total * rec_bytes, 16);
        const int64_t need = o_vals + round_up(total * 4, 16);
        if (need > h0->ord_cap) {
            CK(cudaStreamSynchronize(h0->st));
            if (h0->ord_host) cudaFreeHost(h0->ord_host);
            h0->ord_host = nullptr;
            dfree(h0, h0->ord_dev);
            h0->ord_dev = nullptr;
            h0->ord_cap = 0;
            const int64_t cap = std::max<int64_t>(need * 2, (int64_t)1 << 20);
            CK(cudaHostAlloc((void**)&h0->ord_host, (size_t)cap, cudaHostAllocPortable));
            CKR(dalloc(h0, (void**)&h0->ord_dev, cap));
            h0->ord_cap = cap;
        }
        uint8_t* hb = h0->ord_host;
        uint8_t* db = h0->ord_dev;
        memcpy(hb, gkey.data(), (size_t)rd.n_groups * 8);
        memcpy(hb + o_rank, rank_of_size, (size_t)n_sizes * 4);
        CK(cudaMemcpyAsync(db, hb, o_keys, cudaMemcpyHostToDevice, h0->st));
        OrderKey ok{reinterpret_cast<const uint64_t*>(db), h0->size_of_id, reinterpret_cast<const int32_t*>(db + o_rank),
                    n_sizes, rank_bits, id_bits, g_bits, gw, rec8 ? 1 : 0};
        k_order_keys<<<grid_for(total), 256, 0, h0->st>>>(R.out, total, 0, ok, reinterpret_cast<uint64_t*>(db + o_keys),
                                                         reinterpret_cast<uint32_t*>(db + o_vals));
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(hb + o_keys, db + o_keys, total * 8, cudaMemcpyDeviceToHost, h0->st));
        CK(cudaMemcpyAsync(hb + o_recs, R.out, total * rec_bytes, cudaMemcpyDeviceToHost, h0->st));
        CK(cudaStreamSynchronize(h0->st));
        const uint64_t* keys = reinterpret_cast<const uint64_t*>(hb + o_keys);
        const uint8_t* recs = hb + o_recs;
        std::vector<uint32_t> idx((size_t)total);
        for (uint32_t i = 0; i < (uint32_t)total; ++i) idx[i] = i;
        std::sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) { return keys[a] < keys[b]; });
        for (int64_t j = 0; j < total; ++j) {
            const uint32_t i = idx[j];
            uint64_t eid, mask;
            int32_t grp;
            if (rec8) {
                uint64_t x;
                memcpy(&x, recs + (size_t)i * 8, 8);
                eid = x >> 37; grp = (int32_t)((x >> 32) & 31u); mask = x & 0xFFFFFFFFull;
            } else {
                tsg_report r;
                memcpy(&r, recs + (size_t)i * 16, 16);
                eid = r.key >> 16; grp = (int32_t)(r.key & 0xFFFFu); mask = r.lane_mask;
            }
            if (eid_bytes == 4) static_cast<int32_t*>(eids)[j] = (int32_t)eid;
            else static_cast<int64_t*>(eids)[j] = (int64_t)eid;
            if (mask_bytes == 4) static_cast<uint32_t*>(masks)[j] = (uint32_t)mask;
            else static_cast<uint64_t*>(masks)[j] = mask;
            if (groups) groups[j] = grp;
            ++dest_counts[(int64_t)(keys[i] >> low_bits)];
        }
        return TSG_OK;
    }
    // device 0: concatenated records (several shards), keys / vals double buffers
    DevGuard g0(h0->dev);
    uint8_t* recs = nullptr;
    uint64_t *k0 = nullptr, *k1 = nullptr;
    uint32_t *v0 = nullptr, *v1 = nullptr, *hist = nullptr, *rowsum = nullptr;
    int64_t* starts = nullptr;
    uint8_t* out = nullptr;
    const int64_t nblk = (total + SORT_TILE - 1) / SORT_TILE;
    if (n_h > 1) CKR(dalloc(h0, (void**)&recs, total * rec_bytes));
    CKR(dalloc(h0, (void**)&k0, total * 8));
    CKR(dalloc(h0, (void**)&k1, total * 8));
    CKR(dalloc(h0, (void**)&v0, total * 4));
    CKR(dalloc(h0, (void**)&v1, total * 4));
    CKR(dalloc(h0, (void**)&hist, 256 * nblk * 4 + 256 * 4));
    rowsum = hist + 256 * nblk;
    CKR(dalloc(h0, (void**)&starts, (int64_t)(n_dest + 1) * 8));
    const int64_t eid_sec = round_up(total * eid_bytes, 256), mask_sec = round_up(total * mask_bytes, 256);
    CKR(dalloc(h0, (void**)&out, eid_sec + mask_sec + (groups ? total * 4 : 0)));
    CK(cudaEventRecord(h0->ev_peer, h0->st));  // device 0's buffers exist before any shard copies into them
    // per shard: keys on its device, then (if not device 0's own) its keys,
    // vals and records copied to device 0
    int64_t base = 0;
    for (int32_t s = 0; s < n_h; ++s) {
        tsg_engine* h = hs[s];
        const auto& R = h->rs[h->fetch_rs];
        if (!R.n_out) continue;
        DevGuard gs(h->dev);
        uint64_t* dg = nullptr;
        int32_t* dr = nullptr;
        uint64_t* kk = k0 + base;
        uint32_t* vv = v0 + base;
        if (s > 0) {
            CK(cudaStreamWaitEvent(h->st, h0->ev_peer, 0));
            CKR(dalloc(h, (void**)&kk, R.n_out * 8));
            CKR(dalloc(h, (void**)&vv, R.n_out * 4));
        }
        CKR(dalloc(h, (void**)&dg, (int64_t)rd.n_groups * 8));
        CKR(dalloc(h, (void**)&dr, (int64_t)n_sizes * 4));
        CK(cudaMemcpyAsync(dg, gkey.data(), rd.n_groups * 8, cudaMemcpyHostToDevice, h->st));
        CK(cudaMemcpyAsync(dr, rank_of_size, n_sizes * 4, cudaMemcpyHostToDevice, h->st));
        OrderKey ok{dg, h->size_of_id, dr, n_sizes, rank_bits, id_bits, g_bits, gw, rec8 ? 1 : 0};
        k_order_keys<<<grid_for(R.n_out), 256, 0, h->st>>>(R.out, R.n_out, base, ok, kk, vv);
        CK(cudaGetLastError());
        if (s > 0) {
            CK(cudaMemcpyPeerAsync(k0 + base, h0->dev, kk, h->dev, R.n_out * 8, h->st));
            CK(cudaMemcpyPeerAsync(v0 + base, h0->dev, vv, h->dev, R.n_out * 4, h->st));
            CK(cudaMemcpyPeerAsync(recs + base * rec_bytes, h0->dev, R.out, h->dev, R.n_out * rec_bytes, h->st));
            CK(cudaEventRecord(h->ev_peer, h->st));
            dfree(h, kk); dfree(h, vv);
            DevGuard gz(h0->dev);
            CK(cudaStreamWaitEvent(h0->st, h->ev_peer, 0));  // device 0 sorts after the copies
        } else if (n_h > 1) {
            CK(cudaMemcpyAsync(recs, R.out, R.n_out * rec_bytes, cudaMemcpyDeviceToDevice, h->st));
        }
        dfree(h, dg); dfree(h, dr);  // (stream-ordered after the kernel)
        base += R.n_out;
    }
    // (pageable sources: the gkey / rank_of_size copies consumed them on return)
    const void* src = n_h > 1 ? (const void*)recs : (const void*)h0->rs[h0->fetch_rs].out;
    // LSD passes over the key's significant bits
    uint64_t *ka = k0, *kb = k1;
    uint32_t *va = v0, *vb = v1;
    for (int shift = 0; shift < key_bits; shift += 8) {
        k_sort_hist<<<(unsigned)nblk, SORT_THREADS, 0, h0->st>>>(ka, total, shift, hist);
        k_scan_rows<<<256, 1024, 0, h0->st>>>(hist, nblk, rowsum);
        k_scan_add<<<256, 1024, 0, h0->st>>>(hist, nblk, rowsum);
        k_sort_scatter<<<(unsigned)nblk, SORT_THREADS, 0, h0->st>>>(ka, va, total, shift, hist, kb, vb);
        CK(cudaGetLastError());
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    k_dest_starts<<<grid_for(total + 1), 256, 0, h0->st>>>(ka, total, low_bits, n_dest, starts);
    uint8_t* oe = out;
    uint8_t* om = out + eid_sec;  // sections 256-byte aligned for the 8-byte fields
    int32_t* og = groups ? reinterpret_cast<int32_t*>(om + mask_sec) : nullptr;
    k_order_gather<<<grid_for(total), 256, 0, h0->st>>>(va, total, src, rec8 ? 1 : 0, eid_bytes, mask_bytes, oe, om,
                                                        og);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(eids, oe, total * eid_bytes, cudaMemcpyDeviceToHost, h0->st));
    CK(cudaMemcpyAsync(masks, om, total * mask_bytes, cudaMemcpyDeviceToHost, h0->st));
    if (groups) CK(cudaMemcpyAsync(groups, og, total * 4, cudaMemcpyDeviceToHost, h0->st));
    std::vector<int64_t> st(n_dest + 1);
    CK(cudaMemcpyAsync(st.data(), starts, (n_dest + 1) * 8, cudaMemcpyDeviceToHost, h0->st));
    CK(cudaStreamSynchronize(h0->st));
    for (int32_t d = 0; d < n_dest; ++d) dest_counts[d] = st[d + 1] - st[d];
    dfree(h0, recs); dfree(h0, k0); dfree(h0, k1); dfree(h0, v0); dfree(h0, v1); dfree(h0, hist);
    dfree(h0, starts); dfree(h0, out);
    return TSG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Host report ring (north_star subsystem 4)

namespace {
void ring_free(tsg_engine* h) {
    auto& r = h->ring;
    if (!r.slots) return;
    cudaStreamSynchronize(h->st);
    dfree(h, r.d_pos);
    cudaStreamSynchronize(h->st);
    cudaFreeHost(r.slots);
    cudaFreeHost(r.ctl);
    r.slots = r.d_slots = r.ctl = r.d_ctl = r.d_pos = nullptr;
    r.cap = 0;
    r.next_block = 0;
    r.open.clear();
    r.idle.clear();
    r.expected = 0;
}
}  // namespace

int tsg_ring_open(tsg_engine* h, int64_t capacity, int64_t wait_us) {
    CKR(validate_handle(h));
    if (any_inflight(h)) return fail(TSG_EINVAL, "a launched round is not collected");
    if (h->ring.slots) return fail(TSG_EINVAL, "a report ring is already open");
    if (wide_lane(h))
        return fail(TSG_EINVAL, "report ring records carry 32-bit lane masks: lane_width %d > 32", h->cfg.lane_width);
    if (capacity < RECBUF || capacity > (int64_t(1) << 36))
        return fail(TSG_EINVAL, "ring capacity must be in %d..2^36 records, got %lld", RECBUF, (long long)capacity);
    if (wait_us <= 0) return fail(TSG_EINVAL, "wait_us must be positive");
    int64_t cap = 1;
    while (cap < capacity) cap <<= 1;
    DevGuard g(h->dev);
    auto& r = h->ring;
    void *slots = nullptr, *ctl = nullptr, *dv = nullptr;
    CK(cudaHostAlloc(&slots, (size_t)cap * 16, cudaHostAllocMapped | cudaHostAllocPortable));
    if (cudaHostAlloc(&ctl, 64, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        cudaFreeHost(slots);
        return fail(TSG_ENOMEM, "report ring control block");
    }
    std::memset(slots, 0, (size_t)cap * 16);
    std::memset(ctl, 0, 64);
    r.slots = static_cast<unsigned long long*>(slots);
    r.ctl = static_cast<unsigned long long*>(ctl);
    CK(cudaHostGetDevicePointer(&dv, slots, 0));
    r.d_slots = static_cast<unsigned long long*>(dv);
    CK(cudaHostGetDevicePointer(&dv, ctl, 0));
    r.d_ctl = static_cast<unsigned long long*>(dv);
    CKR(dalloc(h, (void**)&r.d_pos, 8));
    CK(cudaMemsetAsync(r.d_pos, 0, 8, h->st));
    CK(cudaStreamSynchronize(h->st));
    r.cap = cap;
    r.shift = 0;
    while ((int64_t(1) << r.shift) < cap) ++r.shift;
    r.blk = std::max<int64_t>(1, std::min<int64_t>(4096, cap / 8));  // >= 8 blocks per lap
    r.wait_ns = wait_us * 1000;
    r.next_block = 0;
    r.open.clear();
    r.idle.clear();
    r.expected = 0;
    return TSG_OK;
}

namespace {
// close the ring once no drainer is inside tsg_ring_drain: new drain calls
// fail at once, the ones inside return (their waits end on `closing`)
void ring_shutdown(tsg_engine* h) {
    auto& r = h->ring;
    {
        std::lock_guard<std::mutex> lk(r.mtx);
        if (!r.slots) return;
        r.closing = true;
    }
    for (;;) {
        {
            std::lock_guard<std::mutex> lk(r.mtx);
            if (r.active == 0) {
                ring_free(h);
                r.closing = false;
                return;
            }
        }
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}
}  // namespace

int tsg_ring_close(tsg_engine* h) {
    CKR(validate_handle(h));
    if (any_inflight(h)) return fail(TSG_EINVAL, "a launched round is not collected");
    DevGuard g(h->dev);
    ring_shutdown(h);
    return TSG_OK;
}

namespace {
// the consumed prefix: every block below the lowest open one is finished
int64_t ring_tail(const tsg_engine::Ring& r) {
    if (r.open.empty()) return r.next_block * r.blk;
    return r.open.begin()->first * r.blk + r.open.begin()->second;
}
}  // namespace

int tsg_ring_drain(tsg_engine* h, tsg_report* out, int64_t cap, int64_t* n, int64_t timeout_us, int64_t* first_pos) {
    if (!h || !n || (cap > 0 && !out)) return fail(TSG_EINVAL, "bad arguments");
    *n = 0;
    if (first_pos) *first_pos = -1;
    auto& r = h->ring;
    {
        std::lock_guard<std::mutex> lk(r.mtx);
        if (!r.slots || r.closing) return fail(TSG_EINVAL, "no report ring is open");
        ++r.active;
    }
    struct Leave {  // the drainer count drops on every exit path
        tsg_engine::Ring& r;
        ~Leave() { std::lock_guard<std::mutex> lk(r.mtx); --r.active; }
    } leave{r};
    const volatile unsigned long long* S = r.slots;
    volatile unsigned long long* ctl = r.ctl;
    const uint64_t mask = (uint64_t)r.cap - 1;
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    auto last = t0;  // when the last record was taken
    // with records in hand, wait this long for the next one before returning
    // (records land out of order while the kernel runs)
    const double linger_us = std::min<double>((double)timeout_us, 20.0);
    int64_t k = 0;
    while (k < cap) {
        // take the lowest idle block, or the next new one
        int64_t b, p;
        {
            std::lock_guard<std::mutex> lk(r.mtx);
            if (!r.idle.empty()) {
                b = *r.idle.begin();
                r.idle.erase(r.idle.begin());
                p = r.open[b];
            } else {
                b = r.next_block++;
                p = r.open[b] = 0;
            }
        }
        // consume it in order while its records have landed (one call hands
        // out one contiguous run of positions: drainers on several threads
        // can put their batches back in ring order)
        if (first_pos) *first_pos = b * r.blk + p;
        bool stalled = false;
        while (p < r.blk && k < cap) {
            const uint64_t q = (uint64_t)(b * r.blk + p);
            const volatile unsigned long long* s = S + 2 * (q & mask);
            const unsigned long long tag = ring_tag(q, r.shift);
            const unsigned long long w0 = s[0], w1 = s[1];
            if ((w0 >> 48) != tag || (w1 >> 48) != tag) {  // not landed (yet)
                const auto now = clk::now();
                if (ctl[1] || r.closing || (k > 0 && std::chrono::duration<double, std::micro>(now - last).count() >= linger_us) ||
                    std::chrono::duration<double, std::micro>(now - t0).count() >= timeout_us) {
                    stalled = true;
                    break;
                }
                _mm_pause();
                continue;
            }
            if ((k & 255) == 0) last = clk::now();
            if (p + 16 < r.blk) _mm_prefetch((const char*)(S + 2 * ((q + 16) & mask)), _MM_HINT_T0);
            out[k].key = ((w0 & ((1ull << 48) - 1)) << 16) | ((w1 >> 32) & 0xFFFFull);
            out[k].lane_mask = w1 & 0xFFFFFFFFull;
            ++p;
            ++k;
        }
        {
            std::lock_guard<std::mutex> lk(r.mtx);
            if (p == r.blk) {
                r.open.erase(b);
            } else {
                r.open[b] = p;
                r.idle.insert(b);
            }
            ctl[0] = (unsigned long long)ring_tail(r);  // the slots below are free for the kernel
        }
        if (stalled || k > 0) break;  // one run per call
    }
    *n = k;
    return TSG_OK;
}

int tsg_ring_status(tsg_engine* h, int64_t* expected, int64_t* consumed, int32_t* failed) {
    if (!h) return fail(TSG_EINVAL, "null engine handle");
    auto& r = h->ring;
    std::lock_guard<std::mutex> lk(r.mtx);
    if (!r.slots) return fail(TSG_EINVAL, "no report ring is open");
    if (expected) *expected = r.expected.load();
    if (consumed) *consumed = (int64_t)((volatile unsigned long long*)r.ctl)[0];
    if (failed) *failed = ((volatile unsigned long long*)r.ctl)[1] ? 1 : 0;
    return TSG_OK;
}
