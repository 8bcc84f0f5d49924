// tsg_engine.cu -- C ABI (include/tsg.h) over the sm_100a kernels.
//
// Host runtime of the device engine: bucket bookkeeping, staging, chunking,
// kernel launches on one CUDA stream per handle, report-buffer management,
// store maintenance with CUB sort/select for the rare reduce path.
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "../../include/tsg.h"
#include "tsg_kernels.cuh"
#include "tsg_store.cuh"

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

// One physical interleaved array: the clauses of one size bucket whose hot
// slab is `slab`.  Slot order inside a part is append order,
// i.e. engine-id order; a logical bucket is the id-ordered merge of its parts.
struct Part {
    int32_t slab = 0;
    int64_t count = 0, cap = 0;  // cap: multiple of STRIDE
    int32_t* lits = nullptr;     // placement order (see `order`)
    double* acts = nullptr;
    int64_t* ids = nullptr;
    int32_t* origins = nullptr;
    uint64_t* order = nullptr;   // where the stored literal order came from (tsg_store.cuh order_word)
};

// A size bucket of the reference store (engine.py:122-163), split into one
// part per variable slab.
struct Bucket {
    int32_t size = 0, rank = 0;
    std::vector<Part> parts;
    int64_t count() const {
        int64_t n = 0;
        for (auto& p : parts) n += p.count;
        return n;
    }
};

}  // namespace

// The group description of one round (tsg_round_prepare), kept per round
// so a launched round can be collected -- and its report emission replayed --
// after the next round has been prepared and encoded.
struct RoundDesc {
    int32_t n_groups = 0, n_chunks = 0;
    std::vector<int32_t> glanes, gtid;
    std::vector<int64_t> grow0;
    std::vector<int64_t> chunk_off;  // byte offset of each chunk's tables within a table slot
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
    int pk = 1;                           // buffer of the last stage
    bool pstaged = false;                 // prows is pbuf[pk], copied on the ingress stream
    cudaStream_t ingress = nullptr;
    // encoder stream (TSG_ASYNC_ENCODE=1, opt-in): round i+1's encode runs
    // beside round i's trigger test, filling the SMs its CTAs leave at the
    // end; the compute stream waits for ev_encoded before the next test.
    // Measured 0.298 vs 0.293 ms per C3 step (the encode can only start as
    // k_test's CTAs retire, and the next test then waits for all of it).
    cudaStream_t enc_st = nullptr;
    cudaStream_t est = nullptr;           // stream the encoder kernels go to (enc_st or st)
    bool async_encode = false;
    bool enc_wait_main = true;            // the encoder's inputs were last written on st (tables, int8 rows)
    cudaEvent_t ev_main = nullptr, ev_encoded = nullptr;
    cudaEvent_t ev_staged[2] = {nullptr, nullptr};  // copy into pbuf[b] done
    cudaEvent_t ev_read[2] = {nullptr, nullptr};    // encoder done reading pbuf[b]

    // round description as prepared
    RoundDesc rd;
    // round tables: two slots of tables_bytes each (slot stride slot_bytes);
    // encode writes slot `tslot`; tsg_round_launch flips it, so the next
    // round encodes while the launched one still owns its tables
    int8_t* tables = nullptr;
    int64_t tables_cap = 0, tables_bytes = 0, slot_bytes = 0;
    int tslot = 0;
    cudaEvent_t ev_enc[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // per table slot: encode start/end

    // Two round states alternate: a launched round keeps its
    // group description, table slot, counters, carry stamps and record
    // buffers until it is collected, so up to two rounds are in flight and
    // the next round is queued before the previous one is collected.
    struct RoundState {
        RoundDesc fl;
        int slot = 0;                         // table slot it tests
        double inc = 0.0;
        int64_t seq = 0;                      // launch sequence: carry stamps, collect order
        int32_t run = 0;                      // 0: the round's test; 1, 2, ...: emission replays
        bool inflight = false;                // launched, not collected
        // device [8]: [0..3] round counters, [5] CTAs done, [6..7] polarity
        // counts; zero between rounds (the round's last CTA publishes them
        // to h_ctr and re-zeroes them, so no memset or copy is queued)
        unsigned long long* ctr = nullptr;
        unsigned long long* h_ctr = nullptr;  // pinned [8], written by the kernel
        bool pol_pending = false;             // an encode counted into ctr[6..7] since the last launch
        bool timed = false;                   // its encode / test are bracketed by timing events
        bool rec8 = false;                    // its records are 8-byte u64 (tsg_set_record_bytes(8) and they fit)
        unsigned long long* tiles = nullptr;  // device DynTiles counters, zero between launches
        cudaEvent_t ev_done = nullptr;        // its counters are on the host
        cudaEvent_t ev_tst[2] = {nullptr, nullptr};
        int64_t* carry = nullptr;             // per-clause (round, tid) stamps of multi-chunk rounds
        int64_t carry_cap = 0;
    } rs[2];
    int next_rs = 0;                      // state of the next launch
    int fetch_rs = 0;                     // state the fetch calls read (the last collected)
    int report_rs = 0;                    // state whose record buffers are in the fields below
    unsigned long long* mctr = nullptr;   // device [8]: maintenance scratch (reduce, remove, range check)
    unsigned long long* h_mctr = nullptr; // pinned [8]

    BucketDesc* d_desc = nullptr;
    int64_t desc_cap = 0;
    std::vector<BucketDesc> h_desc;
    int64_t n_tiles = 0;

    tsg_report* out = nullptr;
    int64_t out_cap = 0, n_out = 0, n_alloc = 0;
    tsg_report* out2 = nullptr;             // compaction target for fetch
    int64_t out2_cap = 0;
    bool compacted = true;
    // record buffers: the fields above belong to round state `report_rs`,
    // `alt` to the other one (use_reports swaps them); a state's buffers are
    // rewritten only after their copy-out event (tsg_fetch_reports_async).
    struct Slot {
        tsg_report *out = nullptr, *out2 = nullptr;
        int64_t out_cap = 0, out2_cap = 0;
        uint8_t* out12 = nullptr;
        int64_t out12_cap = 0;
        cudaEvent_t ev = nullptr;   // copy-out of these records done
        int64_t n_out = 0, n_alloc = 0;
        bool compacted = true;
    } alt;
    cudaEvent_t ev_cur = nullptr;   // copy-out of the current buffers done
    cudaStream_t egress = nullptr;
    cudaEvent_t ev_ready = nullptr; // compacted records ready for copy-out
    int32_t record_bytes = 16;      // egress record format (tsg_set_record_bytes)
    int64_t max_id = -1;            // largest engine id ever added (8-byte records need < 2^27)
    uint8_t* out12 = nullptr;       // 12-byte egress records of the current slot
    int64_t out12_cap = 0;
    bool oob = false;  // a stored literal may exceed num_vars (checked before testing)
    int64_t round_seq = 0;
    int enc_attr = 0;             // k_encode_packed32 shared-memory attribute set, per GW
    // tsg_round_encode_groups: encode groups [enc_g0, enc_g1) only (enc_g1 < 0: all)
    int32_t enc_g0 = 0, enc_g1 = -1;
    bool enc_sentinel = true;
    tsg_counters_t totals{};      // cumulative figures (tsg_counters)
    int32_t timing_every = 1;     // TSG_F_TIMING: events on rounds whose sequence is a multiple (tsg_set_timing)
    int64_t grid[32] = {0};       // persistent grid per k_test variant
    int64_t grid_smem[32];        // shared-memory size the grid was computed for (-1: none)
    // shared-memory code table when it fits: measured slower than the L2
    // table on B200 even at C1 / C2 (0.026 / 0.047 vs 0.022 / 0.043 ms per
    // round), so opt-in (TSG_SMEM_TABLE=1)
    bool smem_table = false;
    // dynamic tile counters in k_test balance the SMs (±5 % active cycles
    // with the static stride) but measured no faster: opt-in, TSG_DYN_TILES=1
    bool dyn_tiles = false;
    uint8_t* codes = nullptr;     // literal-code table of the current chunk
    int64_t codes_cap = 0;

    // variable slabs: [s * slab_w, (s + 1) * slab_w) for s < n_slabs, covering 0..V+1
    int32_t n_slabs = 1, slab_w = 0;
    bool slab_test = true;               // slab kernel when n_slabs > 1 (TSG_SLABS=0 disables)
    std::vector<int64_t> slab_load;      // clauses per slab (placement tie-break)
    std::vector<int64_t> h_slab_tile0;   // first tile of each slab (+ end)
    std::vector<int32_t> h_slab_desc0;   // first descriptor of each slab (+ end)
    int64_t* d_slab_tile0 = nullptr;     // [n_slabs + 1] tile0, then [n_slabs + 1] desc0 (int32), then schedule
    int64_t slab_tile0_cap = 0;
    std::vector<uint64_t> h_sched;
    bool desc_dirty = true;             // store changed since the tile table was built
    bool pivot = true;                  // pivot-first clause layout (TSG_PIVOT=0 disables)
    // literal polarity placed right after the pivot (+1 / -1 / 0 none).  Prior
    // before any round: +1 -- in the paper's measured value subsets
    // a variable can be True in a window more often
    // (.208) than False (.153), so positive literals are non-False more often
    int prefer = 1;
    bool prefer_fixed = false;          // TSG_PREFER fixes it; else set from each round's statistics
    bool l2_persist = false;            // persisting L2 window over the round tables (TSG_L2_PERSIST=1; measured slower)
    const void* persist_base = nullptr;
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
int dgrow(tsg_engine* h, T** p, int64_t* cap, int64_t need, bool keep = false, int64_t keep_elems = 0) {
    if (need <= *cap) return TSG_OK;
    int64_t nc = std::max<int64_t>(need, *cap * 2);
    T* np = nullptr;
    CKR(dalloc(h, (void**)&np, nc * (int64_t)sizeof(T)));
    if (keep && *p && keep_elems)
        CK(cudaMemcpyAsync(np, *p, keep_elems * sizeof(T), cudaMemcpyDeviceToDevice, h->st));
    dfree(h, *p);
    *p = np;
    *cap = nc;
    return TSG_OK;
}

void part_free(tsg_engine* h, Part& p) {
    dfree(h, p.lits); dfree(h, p.acts); dfree(h, p.ids); dfree(h, p.origins); dfree(h, p.order);
    p.lits = nullptr; p.acts = nullptr; p.ids = nullptr; p.origins = nullptr; p.order = nullptr;
}

int part_alloc(tsg_engine* h, Part& p, int32_t size, int64_t cap) {
    CKR(dalloc(h, (void**)&p.lits, cap * (int64_t)std::max(size, 1) * 4));
    CKR(dalloc(h, (void**)&p.acts, cap * 8));
    CKR(dalloc(h, (void**)&p.ids, cap * 8));
    CKR(dalloc(h, (void**)&p.origins, cap * 4));
    CKR(dalloc(h, (void**)&p.order, cap * 8));
    p.cap = cap;
    return TSG_OK;
}

int part_reserve(tsg_engine* h, Part& b, int32_t size, int64_t need) {
    if (need <= b.cap) return TSG_OK;
    // _SizeBucket._grow doubles with a floor of 4 blocks (engine.py:141-148)
    int64_t nc = std::max<int64_t>(b.cap ? b.cap : 4 * STRIDE, 4 * STRIDE);
    while (nc < need) nc *= 2;
    Part n;
    n.slab = b.slab;
    n.count = b.count;
    CKR(part_alloc(h, n, size, nc));
    if (b.count) {
        int64_t used = round_up(b.count, STRIDE);
        if (size) CK(cudaMemcpyAsync(n.lits, b.lits, used * size * 4, cudaMemcpyDeviceToDevice, h->st));
        CK(cudaMemcpyAsync(n.acts, b.acts, b.count * 8, cudaMemcpyDeviceToDevice, h->st));
        CK(cudaMemcpyAsync(n.ids, b.ids, b.count * 8, cudaMemcpyDeviceToDevice, h->st));
        CK(cudaMemcpyAsync(n.origins, b.origins, b.count * 4, cudaMemcpyDeviceToDevice, h->st));
        CK(cudaMemcpyAsync(n.order, b.order, b.count * 8, cudaMemcpyDeviceToDevice, h->st));
    }
    part_free(h, b);
    b = n;
    return TSG_OK;
}

// every physical part, bucket-major then slab (the order of reduce/remove keep flags)
template <class F>
void for_parts(tsg_engine* h, F&& f) {
    for (auto& b : h->buckets)
        for (auto& p : b.parts) f(b, p);
}

bool wide_lane(const tsg_engine* h) { return h->cfg.lane_width > 32; }
bool wide_group(const tsg_engine* h) { return h->cfg.group_width > 32; }
int64_t agg_entry_bytes(const tsg_engine* h) { return wide_group(h) ? 32 : 16; }
int64_t vstride(const tsg_engine* h) { return round_up((int64_t)h->V + 2, 4); }
int64_t agg_bytes(const tsg_engine* h) { return round_up((int64_t)(h->V + 2) * agg_entry_bytes(h), 256); }
int64_t lane_entry_bytes(const tsg_engine* h) { return wide_lane(h) ? 16 : 8; }

template <class LW, class GW>
int launch_encode(tsg_engine* h, int c) {
    EncodeChunk ec{};
    const RoundDesc& rd = h->rd;
    int32_t g0 = c * h->cfg.group_width;
    ec.G = std::min(h->cfg.group_width, rd.n_groups - g0);
    ec.num_vars = h->V;
    ec.pitch = h->pitch;
    ec.vstride = vstride(h);
    for (int g = 0; g < ec.G; ++g) {
        ec.row0[g] = rd.grow0[g0 + g];
        ec.lanes[g] = rd.glanes[g0 + g];
    }
    ec.polarity = h->rs[h->next_rs].ctr + 6;  // counted for the round this encode feeds
    int8_t* tab = h->tables + h->tslot * h->slot_bytes;
    auto* agg = reinterpret_cast<AggEntry<GW>*>(tab + rd.chunk_off[c]);
    auto* lane = reinterpret_cast<LaneEntry<LW>*>(tab + rd.chunk_off[c] + agg_bytes(h));
    dim3 grid((unsigned)((h->V + 2 + 127) / 128)), block(32, 8);
    if (h->packed) {
        EncodePackedChunk pc{};
        pc.G = ec.G;
        pc.num_vars = h->V;
        pc.pitch_words = h->ppitch;
        pc.vstride = ec.vstride;
        // a group range (tsg_round_encode_groups): rows hold only its groups
        const int64_t row_base = h->enc_g1 >= 0 ? rd.grow0[h->enc_g0] : 0;
        for (int g = 0; g < ec.G; ++g) { pc.row0[g] = ec.row0[g] - row_base; pc.lanes[g] = ec.lanes[g]; }
        pc.polarity = ec.polarity;
        pc.gbeg = h->enc_g1 >= 0 ? std::max(0, h->enc_g0 - g0) : 0;
        pc.gend = h->enc_g1 >= 0 ? std::min(ec.G, h->enc_g1 - g0) : ec.G;
        pc.sentinel = h->enc_sentinel ? 1 : 0;
        static const bool enc_stage = !getenv("TSG_ENC_STAGE") || atoi(getenv("TSG_ENC_STAGE")) != 0;
        if (h->enc_g1 >= 0 && !(sizeof(LW) == 4 && enc_stage))
            return fail(TSG_EINVAL, "group-range encode needs the staged encoder (k_encode_packed32)");
        if (sizeof(LW) == 4 && enc_stage) {
            const int need = (ec.G + 7) / 8;  // groups per warp
            const int gpw = need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : 8;
            const size_t smem = (size_t)8 * gpw * 32 * 32;
            auto* lt = reinterpret_cast<LaneEntry<uint32_t>*>(lane);
            auto* fn = gpw == 1 ? k_encode_packed32<GW, 1> : gpw == 2 ? k_encode_packed32<GW, 2>
                     : gpw == 4 ? k_encode_packed32<GW, 4> : k_encode_packed32<GW, 8>;
            const int bit = 1 << (gpw + 8 * (int)(sizeof(GW) / 8));
            if (!(h->enc_attr & bit)) {  // 64 KB of row stage at 8 groups per warp
                CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                h->enc_attr |= bit;
            }
            fn<<<grid, block, smem, h->est>>>(h->prows, pc, lt, agg);
        } else {
            k_encode_packed<LW, GW><<<grid, block, 0, h->est>>>(h->prows, pc, lane, agg);
        }
    } else {
        k_encode<LW, GW><<<grid, block, 0, h->est>>>(h->rows, ec, lane, agg);
    }
    CK(cudaGetLastError());
    return TSG_OK;
}

// u64 words of one packed row: every 128-variable encoder block reads 4 words
int64_t packed_words(int32_t V) { return round_up(((int64_t)V + 2 + 31) / 32, 4); }

int do_encode(tsg_engine* h) {
    for (int c = 0; c < h->rd.n_chunks; ++c) {
        int r;
        if (wide_lane(h)) r = wide_group(h) ? launch_encode<uint64_t, uint64_t>(h, c) : launch_encode<uint64_t, uint32_t>(h, c);
        else r = wide_group(h) ? launch_encode<uint32_t, uint64_t>(h, c) : launch_encode<uint32_t, uint32_t>(h, c);
        if (r) return r;
    }
    return TSG_OK;
}

template <class LW, class GW, class TAB, int THREADS, int MINB>
int launch_kernel(tsg_engine* h, const TestParams<LW, GW>& p, int64_t codes_bytes, int variant) {
    auto* fn = k_test<LW, GW, TAB, THREADS, MINB>;
    const size_t smem = test_smem_bytes<GW, TAB, THREADS>(codes_bytes);
    const int key = (int)(sizeof(LW) / 8) * 8 + (int)(sizeof(GW) / 8) * 4 + variant;
    if (h->grid_smem[key] != (int64_t)smem) {  // occupancy per kernel variant and smem size
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, THREADS, smem));
        h->grid[key] = std::max(1, per_sm) * h->nsm;
        h->grid_smem[key] = (int64_t)smem;
    }
    int64_t want = (h->n_tiles + THREADS / 32 - 1) / (THREADS / 32);
    int grid = (int)std::min<int64_t>(want, h->grid[key]);
    fn<<<grid, THREADS, smem, h->st>>>(p);
    CK(cudaGetLastError());
    return TSG_OK;
}

template <class LW, class GW>
int launch_slab(tsg_engine* h, const TestParams<LW, GW>& p) {
    auto* fn = k_test_slab<LW, GW, TEST_THREADS_SLAB>;
    const size_t smem = (size_t)3 * h->slab_w * sizeof(GW);
    const int key = 16 + (int)(sizeof(LW) / 8) * 2 + (int)(sizeof(GW) / 8);
    if (h->grid_smem[key] != (int64_t)smem) {
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, TEST_THREADS_SLAB, smem));
        if (per_sm < 1) return fail(TSG_ECUDA, "slab kernel does not fit an SM (%zu B shared)", smem);
        h->grid[key] = (int64_t)per_sm * h->nsm;
        h->grid_smem[key] = (int64_t)smem;
    }
    if (h->h_sched.empty()) return TSG_OK;
    int grid = (int)std::min<int64_t>(h->grid[key], (int64_t)h->h_sched.size());
    fn<<<grid, TEST_THREADS_SLAB, smem, h->st>>>(p);
    CK(cudaGetLastError());
    return TSG_OK;
}

template <class LW, class GW>
int launch_test(tsg_engine* h, int k, int c, double inc, int emit_only) {
    const auto& R = h->rs[k];
    const RoundDesc& rd = R.fl;
    const int slot = R.slot;
    TestParams<LW, GW> p{};
    int32_t g0 = c * h->cfg.group_width;
    int32_t G = std::min(h->cfg.group_width, rd.n_groups - g0);
    const int8_t* tab = h->tables + slot * h->slot_bytes;
    p.buckets = h->d_desc;
    p.nb = (int32_t)h->h_desc.size();
    p.G = G;
    p.n_tiles = h->n_tiles;
    p.agg = reinterpret_cast<const AggEntry<GW>*>(tab + rd.chunk_off[c]);
    p.lane = reinterpret_cast<const LaneEntry<LW>*>(tab + rd.chunk_off[c] + agg_bytes(h));
    p.vstride = vstride(h);
    p.sentinel = h->V + 1;
    p.g0 = g0;
    p.group_mask = width_mask<GW>(G);
    p.inc = inc;
    p.out = h->out;
    p.ctr = R.ctr;
    p.out_cap = h->out_cap;
    p.carry = R.carry;
    // carry stamps are unique per (round, run): a replay must not see the
    // stamps its own round's first run left behind
    p.stamp_base = (((R.seq << 6) | (R.run & 63)) & 0x7fffffff) << 32;
    p.carry_in_tid = (c > 0 && rd.gtid[g0] == rd.gtid[g0 - 1]) ? rd.gtid[g0] : -1;
    p.carry_out_tid = (g0 + G < rd.n_groups && rd.gtid[g0 + G - 1] == rd.gtid[g0 + G]) ? rd.gtid[g0 + G - 1] : -1;
    p.emit_only = emit_only;
    p.pub = (!emit_only && c == rd.n_chunks - 1) ? R.h_ctr : nullptr;
    p.dyn_tiles = h->dyn_tiles ? 1 : 0;
    p.rec8 = R.rec8 ? 1 : 0;
    p.tiles = R.tiles;
    p.slab_tile0 = h->d_slab_tile0;
    p.slab_desc0 = reinterpret_cast<const int32_t*>(h->d_slab_tile0 + (h->n_slabs + 1));
    p.sched = reinterpret_cast<const uint64_t*>(h->d_slab_tile0 + 2 * (h->n_slabs + 1));
    p.n_sched = (int32_t)h->h_sched.size();
    p.slab_w = h->slab_w;
    for (int g = 0; g < G; ++g) {
        p.tid[g] = rd.gtid[g0 + g];
        p.lane_mask[g] = width_mask<LW>(rd.glanes[g0 + g]);
    }
    if (h->n_tiles == 0) return TSG_OK;
    // shared-memory literal-code table when 2 * (V + 2) codes fit (G <= 32)
    const int ew = G <= 8 ? 2 : (G <= 16 ? 4 : 8);
    const int64_t codes_bytes = round_up(2 * ((int64_t)h->V + 2) * ew, 16);
    if constexpr (sizeof(GW) == 4) {
        if (h->smem_table && codes_bytes <= SMEM_TABLE_MAX) {
            CKR(dgrow(h, &h->codes, &h->codes_cap, codes_bytes));
            p.codes = h->codes;
            p.codes_bytes = codes_bytes;
            const auto* agg = reinterpret_cast<const AggEntry<uint32_t>*>(p.agg);
            if (ew == 2) {
                k_codes<uint16_t><<<grid_for(h->V + 2), 256, 0, h->st>>>(agg, h->V + 2, (uint16_t*)h->codes);
                return launch_kernel<LW, GW, SmemTable<GW, uint16_t>, TEST_THREADS_SMEM, 1>(h, p, codes_bytes, 1);
            }
            if (ew == 4) {
                k_codes<uint32_t><<<grid_for(h->V + 2), 256, 0, h->st>>>(agg, h->V + 2, (uint32_t*)h->codes);
                return launch_kernel<LW, GW, SmemTable<GW, uint32_t>, TEST_THREADS_SMEM, 1>(h, p, codes_bytes, 2);
            }
            k_codes<uint64_t><<<grid_for(h->V + 2), 256, 0, h->st>>>(agg, h->V + 2, (uint64_t*)h->codes);
            return launch_kernel<LW, GW, SmemTable<GW, uint64_t>, TEST_THREADS_SMEM, 1>(h, p, codes_bytes, 3);
        }
    }
    if (h->slab_test && h->n_slabs > 1) return launch_slab<LW, GW>(h, p);
    return launch_kernel<LW, GW, GlobalTable<GW>, TEST_THREADS, TSG_TEST_MIN_BLOCKS>(h, p, 0, 0);
}

// the round of state k (its record buffers must be the active ones)
int run_tests(tsg_engine* h, int k, double inc, int emit_only) {
    for (int c = 0; c < h->rs[k].fl.n_chunks; ++c) {
        int r;
        if (wide_lane(h)) r = wide_group(h) ? launch_test<uint64_t, uint64_t>(h, k, c, inc, emit_only) : launch_test<uint64_t, uint32_t>(h, k, c, inc, emit_only);
        else r = wide_group(h) ? launch_test<uint32_t, uint64_t>(h, k, c, inc, emit_only) : launch_test<uint32_t, uint32_t>(h, k, c, inc, emit_only);
        if (r) return r;
    }
    return TSG_OK;
}

int64_t store_size(const tsg_engine* h) {
    int64_t n = 0;
    for (auto& b : h->buckets) n += b.count();
    return n;
}

// Tile table of the round: parts ordered slab-major (then bucket creation
// order), so every slab's tiles are contiguous and a CTA of the slab kernel
// loads each slab's table once.  Report order does not depend on it (the
// host orders records by engine id, reports.py).
int build_desc(tsg_engine* h) {
    if (!h->desc_dirty) return TSG_OK;  // store unchanged since the last round
    h->h_desc.clear();
    h->h_slab_tile0.assign(h->n_slabs + 1, 0);
    h->h_slab_desc0.assign(h->n_slabs + 1, 0);
    int64_t tiles = 0;
    for (int32_t s = 0; s < h->n_slabs; ++s) {
        h->h_slab_tile0[s] = tiles;
        h->h_slab_desc0[s] = (int32_t)h->h_desc.size();
        for (auto& b : h->buckets) {
            const Part& p = b.parts[s];
            if (!p.count) continue;
            BucketDesc d{};
            d.lits = p.lits; d.acts = p.acts; d.ids = p.ids;
            d.size = b.size; d.rank = b.rank; d.count = p.count; d.tile0 = tiles;
            tiles += (p.count + STRIDE - 1) / STRIDE;
            h->h_desc.push_back(d);
        }
    }
    h->h_slab_tile0[h->n_slabs] = tiles;
    h->h_slab_desc0[h->n_slabs] = (int32_t)h->h_desc.size();
    h->n_tiles = tiles;
    CKR(dgrow(h, &h->d_desc, &h->desc_cap, std::max<int64_t>(1, (int64_t)h->h_desc.size())));
    if (!h->h_desc.empty())
        CK(cudaMemcpyAsync(h->d_desc, h->h_desc.data(), h->h_desc.size() * sizeof(BucketDesc),
                           cudaMemcpyHostToDevice, h->st));
    // slab schedule for a grid of one CTA per SM: each slab gets CTAs in
    // proportion to its tiles (largest remainder, at least one if it has any)
    h->h_sched.clear();
    {
        const int64_t grid = h->nsm;
        std::vector<int64_t> n(h->n_slabs, 0);
        std::vector<std::pair<double, int>> rem;
        int64_t used = 0, nonempty = 0;
        for (int32_t s = 0; s < h->n_slabs; ++s) {
            const int64_t t = h->h_slab_tile0[s + 1] - h->h_slab_tile0[s];
            if (!t) continue;
            ++nonempty;
            const double share = tiles ? (double)grid * t / tiles : 0.0;
            n[s] = std::max<int64_t>(1, (int64_t)share);
            n[s] = std::min<int64_t>(n[s], std::max<int64_t>(1, (t + 7) / 8));  // >= 8 tiles per CTA
            used += n[s];
            rem.push_back({share - (double)n[s], s});
        }
        std::sort(rem.begin(), rem.end(), [](auto& x, auto& y) { return x.first > y.first || (x.first == y.first && x.second < y.second); });
        for (auto& r : rem) {
            if (used >= grid) break;
            const int64_t t = h->h_slab_tile0[r.second + 1] - h->h_slab_tile0[r.second];
            if (r.first > 0 && n[r.second] < std::max<int64_t>(1, (t + 7) / 8)) { n[r.second]++; used++; }
        }
        (void)nonempty;
        for (int32_t s = 0; s < h->n_slabs; ++s)
            for (int64_t k = 0; k < n[s]; ++k)
                h->h_sched.push_back((uint64_t)s << 32 | (uint64_t)k << 16 | (uint64_t)n[s]);
    }
    const int64_t words = 2 * (int64_t)(h->n_slabs + 1) + (int64_t)h->h_sched.size() + 1;
    CKR(dgrow(h, &h->d_slab_tile0, &h->slab_tile0_cap, words));
    CK(cudaMemcpyAsync(h->d_slab_tile0, h->h_slab_tile0.data(), h->h_slab_tile0.size() * 8,
                       cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(h->d_slab_tile0 + (h->n_slabs + 1), h->h_slab_desc0.data(), h->h_slab_desc0.size() * 4,
                       cudaMemcpyHostToDevice, h->st));
    if (!h->h_sched.empty())
        CK(cudaMemcpyAsync(h->d_slab_tile0 + 2 * (h->n_slabs + 1), h->h_sched.data(), h->h_sched.size() * 8,
                           cudaMemcpyHostToDevice, h->st));
    // (pageable sources: the copies above have consumed the host vectors on return)
    h->desc_dirty = false;
    return TSG_OK;
}

int validate_handle(tsg_engine* h) {
    if (!h) return fail(TSG_EINVAL, "null engine handle");
    return TSG_OK;
}

// compact every part by keep flags laid out in for_parts order
int compact_all(tsg_engine* h, const uint8_t* keep, const std::vector<int64_t>& base) {
    int64_t* sel = nullptr;
    int64_t* nsel = nullptr;
    int64_t maxc = 0;
    for_parts(h, [&](Bucket&, Part& p) { maxc = std::max(maxc, p.count); });
    if (!maxc) return TSG_OK;
    CKR(dalloc(h, (void**)&sel, maxc * 8));
    CKR(dalloc(h, (void**)&nsel, 8));
    size_t tmp_bytes = 0;
    thrust::counting_iterator<int64_t> cnt(0);
    cub::DeviceSelect::Flagged(nullptr, tmp_bytes, cnt, keep, sel, nsel, maxc, h->st);
    void* tmp = nullptr;
    CKR(dalloc(h, &tmp, (int64_t)tmp_bytes + 16));
    size_t pi = 0;
    for (auto& b : h->buckets) {
        for (auto& p : b.parts) {
            const int64_t pb = base[pi++];
            if (!p.count) continue;
            CK(cub::DeviceSelect::Flagged(tmp, tmp_bytes, cnt, keep + pb, sel, nsel, p.count, h->st));
            int64_t kept = 0;
            CK(cudaMemcpyAsync(&kept, nsel, 8, cudaMemcpyDeviceToHost, h->st));
            CK(cudaStreamSynchronize(h->st));
            if (kept == p.count) continue;
            Part np;
            np.slab = p.slab;
            // keep capacity (the reference never shrinks, engine.py:184-200)
            CKR(part_alloc(h, np, b.size, p.cap));
            if (kept) {
                k_compact<<<grid_for(kept), 256, 0, h->st>>>(sel, kept, b.size, p.lits, p.acts, p.ids, p.origins,
                                                             p.order, np.lits, np.acts, np.ids, np.origins,
                                                             np.order);
                CK(cudaGetLastError());
            }
            part_free(h, p);
            np.count = kept;
            p = np;
        }
    }
    dfree(h, tmp); dfree(h, sel); dfree(h, nsel);
    return TSG_OK;
}

// per-part offsets into one flat keep-flag array (for_parts order)
std::vector<int64_t> part_bases(tsg_engine* h, int64_t* total) {
    std::vector<int64_t> base;
    int64_t acc = 0;
    for_parts(h, [&](Bucket&, Part& p) { base.push_back(acc); acc += p.count; });
    *total = acc;
    return base;
}

int32_t slab_of(const tsg_engine* h, int32_t lit) {
    int64_t v = lit < 0 ? -(int64_t)lit : lit;
    return (int32_t)std::min<int64_t>(v / h->slab_w, h->n_slabs - 1);
}

// Placement of one clause.  Unpartitioned store: the pivot
// -- the literal with the smallest variable among the first 58 -- goes first
// (add_clauses orders each batch by pivot, so a warp's first gathers share
// table lines), then the literals of the preferred polarity (those more
// likely to be non-False under the recent rounds' assignments: they end the
// early-exit recurrence sooner), then the rest.  Slab-partitioned store: the
// literals of the chosen slab (the one holding most of them) go first.  The
// order word lets readback restore the reference's literal order.
int32_t place_clause(tsg_engine* h, const int32_t* lits, int32_t size, std::vector<int32_t>& cnt,
                     int32_t* out, uint64_t* order) {
    const int32_t lim = std::min(size, ORDER_MASK_BITS);
    int32_t slab = 0, jp = -1;
    uint64_t m = 0;
    if (h->n_slabs > 1 && size > 0) {
        for (int32_t j = 0; j < lim; ++j) cnt[slab_of(h, lits[j])]++;
        int32_t best = -1;
        for (int32_t j = 0; j < lim; ++j) {
            int32_t s = slab_of(h, lits[j]);
            if (best < 0 || cnt[s] > cnt[best] || (cnt[s] == cnt[best] && h->slab_load[s] < h->slab_load[best]))
                best = s;
        }
        for (int32_t j = 0; j < lim; ++j) cnt[slab_of(h, lits[j])] = 0;
        slab = best;
        for (int32_t j = 0; j < lim; ++j)
            if (slab_of(h, lits[j]) == slab) m |= 1ull << j;
    } else if (h->pivot && lim > 0) {
        jp = 0;
        for (int32_t j = 1; j < lim; ++j)
            if (std::llabs((long long)lits[j]) < std::llabs((long long)lits[jp])) jp = j;
        if (h->prefer != 0)
            for (int32_t j = 0; j < lim; ++j)
                if (j != jp && (lits[j] > 0) == (h->prefer > 0)) m |= 1ull << j;
    }
    int32_t o = 0;
    if (jp >= 0) out[o++] = lits[jp];
    for (int32_t j = 0; j < lim; ++j)
        if ((m >> j) & 1) out[o++] = lits[j];
    for (int32_t j = 0; j < size; ++j)
        if (j != jp && (j >= lim || !((m >> j) & 1))) out[o++] = lits[j];
    *order = order_word(jp, m);
    h->slab_load[slab]++;
    return slab;
}

struct ValidReport {
    __host__ __device__ bool operator()(const tsg_report& r) const { return r.key != REPORT_PAD; }
};
struct ValidRecord8 {
    __host__ __device__ bool operator()(const uint64_t& r) const { return r != REPORT_PAD; }
};

// squeeze the padding slots out of the round's records (order-preserving)
int compact_reports(tsg_engine* h) {
    if (h->compacted) return TSG_OK;
    // the compacted buffer becomes the round state's record buffer: it must
    // not shrink below the current capacity, or the next round overflows
    CKR(dgrow(h, &h->out2, &h->out2_cap, std::max<int64_t>(h->out_cap, 1)));
    int64_t* nsel = nullptr;
    CKR(dalloc(h, (void**)&nsel, 8));
    size_t tb = 0;
    const bool rec8 = h->rs[h->report_rs].rec8;
    auto* o8 = reinterpret_cast<uint64_t*>(h->out);
    auto* t8 = reinterpret_cast<uint64_t*>(h->out2);
    if (rec8) cub::DeviceSelect::If(nullptr, tb, o8, t8, nsel, h->n_alloc, ValidRecord8(), h->st);
    else cub::DeviceSelect::If(nullptr, tb, h->out, h->out2, nsel, h->n_alloc, ValidReport(), h->st);
    void* tmp = nullptr;
    CKR(dalloc(h, &tmp, (int64_t)tb + 16));
    if (rec8) CK(cub::DeviceSelect::If(tmp, tb, o8, t8, nsel, h->n_alloc, ValidRecord8(), h->st));
    else CK(cub::DeviceSelect::If(tmp, tb, h->out, h->out2, nsel, h->n_alloc, ValidReport(), h->st));
    dfree(h, tmp);
    dfree(h, nsel);
    std::swap(h->out, h->out2);
    std::swap(h->out_cap, h->out2_cap);
    h->n_alloc = h->n_out;
    h->compacted = true;
    return TSG_OK;
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
    for (auto& x : h->grid_smem) x = -1;
    h->dev = cfg->device;
    h->cfg = *cfg;
    h->V = num_vars;
    if (const char* e = getenv("TSG_SMEM_TABLE")) h->smem_table = atoi(e) != 0;
    if (const char* e = getenv("TSG_DYN_TILES")) h->dyn_tiles = atoi(e) != 0;
    if (const char* e = getenv("TSG_ASYNC_ENCODE")) h->async_encode = atoi(e) != 0;
    if (const char* e = getenv("TSG_L2_PERSIST")) h->l2_persist = atoi(e) != 0;
    if (const char* e = getenv("TSG_PIVOT")) h->pivot = atoi(e) != 0;
    if (const char* e = getenv("TSG_PREFER")) { h->prefer = atoi(e); h->prefer_fixed = true; }
    // Variable slabs, opt-in: TSG_SLABS=1 partitions the store
    // into as many slabs as one CTA's shared memory needs for the aggregate
    // words, TSG_SLABS=n>1 into at least n.  Default: one slab (unpartitioned
    // store, global-table kernel), the faster layout measured on B200.
    {
        const int64_t per_var = 3 * (h->cfg.group_width > 32 ? 8 : 4);
        const int64_t nv2 = (int64_t)num_vars + 2;
        int64_t slab_bytes = SLAB_SMEM_BYTES;
        if (const char* e = getenv("TSG_SLAB_BYTES")) slab_bytes = std::min<int64_t>(SLAB_SMEM_BYTES, atol(e));
        const int64_t max_w = std::max<int64_t>(32, (slab_bytes / per_var) / 32 * 32);
        int64_t ns = 1;
        if (const char* e = getenv("TSG_SLABS")) {
            const int req = atoi(e);
            if (req >= 1) ns = std::max<int64_t>((nv2 + max_w - 1) / max_w, req);
        }
        if (ns <= 1) h->slab_test = false;
        int64_t w = round_up((nv2 + ns - 1) / ns, 32);
        h->n_slabs = (int32_t)((nv2 + w - 1) / w);
        h->slab_w = (int32_t)w;
        h->slab_load.assign(h->n_slabs, 0);
    }
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
    cudaStreamCreateWithFlags(&h->egress, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&h->ingress, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&h->enc_st, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&h->ev_main, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&h->ev_encoded, cudaEventDisableTiming);
    h->est = h->st;
    for (int b = 0; b < 2; ++b) {
        cudaEventCreateWithFlags(&h->ev_staged[b], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&h->ev_read[b], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&h->ev_cur, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&h->alt.ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&h->ev_ready, cudaEventDisableTiming);
    for (int sl = 0; sl < 2; ++sl)
        for (int k = 0; k < 2; ++k) cudaEventCreate(&h->ev_enc[sl][k]);
    for (auto& R : h->rs) {
        cudaEventCreateWithFlags(&R.ev_done, cudaEventDisableTiming);
        for (auto& e : R.ev_tst) cudaEventCreate(&e);
        if (cudaMallocHost(&R.h_ctr, 8 * sizeof(unsigned long long)) != cudaSuccess) { delete h; return fail(TSG_ECUDA, "pinned alloc"); }
        if (dalloc(h, (void**)&R.ctr, 8 * sizeof(unsigned long long))) { delete h; return TSG_ENOMEM; }
        if (cudaMemsetAsync(R.ctr, 0, 8 * sizeof(unsigned long long), h->st) != cudaSuccess) { delete h; return fail(TSG_ECUDA, "memset"); }
        const int64_t tb = (int64_t)TSG_DYN_NC * DYN_STRIDE * sizeof(unsigned long long);
        if (dalloc(h, (void**)&R.tiles, tb)) { delete h; return TSG_ENOMEM; }
        if (cudaMemsetAsync(R.tiles, 0, tb, h->st) != cudaSuccess) { delete h; return fail(TSG_ECUDA, "memset"); }
    }
    if (cudaMallocHost(&h->h_mctr, 8 * sizeof(unsigned long long)) != cudaSuccess) { delete h; return fail(TSG_ECUDA, "pinned alloc"); }
    if (dalloc(h, (void**)&h->mctr, 8 * sizeof(unsigned long long))) { delete h; return TSG_ENOMEM; }
    h->out_cap = cfg->report_capacity > 0 ? std::min<int64_t>(cfg->report_capacity, INT32_MAX / 2) : (1 << 16);
    if (dalloc(h, (void**)&h->out, h->out_cap * (int64_t)sizeof(tsg_report))) { delete h; return TSG_ENOMEM; }
    *out = h;
    return TSG_OK;
}

int tsg_destroy(tsg_engine* h) {
    if (!h) return TSG_OK;
    DevGuard g(h->dev);
    if (h->enc_st) cudaStreamSynchronize(h->enc_st);
    cudaStreamSynchronize(h->st);
    for_parts(h, [&](Bucket&, Part& p) { part_free(h, p); });
    dfree(h, h->d_slab_tile0);
    if (h->ingress) cudaStreamSynchronize(h->ingress);
    dfree(h, h->rows_own); dfree(h, h->pbuf[0]); dfree(h, h->pbuf[1]); dfree(h, h->tables); dfree(h, h->d_desc); dfree(h, h->out);
    dfree(h, h->mctr); dfree(h, h->out2); dfree(h, h->codes);
    for (auto& R : h->rs) { dfree(h, R.ctr); dfree(h, R.carry); dfree(h, R.tiles); }
    if (h->egress) cudaStreamSynchronize(h->egress);
    dfree(h, h->alt.out); dfree(h, h->alt.out2); dfree(h, h->alt.out12); dfree(h, h->out12);
    cudaStreamSynchronize(h->st);
    if (h->h_mctr) cudaFreeHost(h->h_mctr);
    for (cudaEvent_t e : {h->ev_cur, h->alt.ev, h->ev_ready}) if (e) cudaEventDestroy(e);
    for (auto& R : h->rs) {
        if (R.h_ctr) cudaFreeHost(R.h_ctr);
        if (R.ev_done) cudaEventDestroy(R.ev_done);
        for (auto& e : R.ev_tst) if (e) cudaEventDestroy(e);
    }
    for (int sl = 0; sl < 2; ++sl)
        for (int k = 0; k < 2; ++k)
            if (h->ev_enc[sl][k]) cudaEventDestroy(h->ev_enc[sl][k]);
    if (h->egress) cudaStreamDestroy(h->egress);
    for (int b = 0; b < 2; ++b) {
        if (h->ev_staged[b]) cudaEventDestroy(h->ev_staged[b]);
        if (h->ev_read[b]) cudaEventDestroy(h->ev_read[b]);
    }
    if (h->ingress) cudaStreamDestroy(h->ingress);
    if (h->enc_st) cudaStreamDestroy(h->enc_st);
    for (cudaEvent_t e : {h->ev_main, h->ev_encoded}) if (e) cudaEventDestroy(e);
    cudaStreamDestroy(h->st);
    delete h;
    return TSG_OK;
}

int tsg_add_clauses(tsg_engine* h, const int32_t* lits, const int64_t* offsets, int64_t n,
                    const int64_t* ids, const int32_t* origins, double activity) {
    CKR(validate_handle(h));
    if (any_inflight(h)) return fail(TSG_EINVAL, "the store cannot change while a launched round is not collected");
    h->desc_dirty = true;
    if (n <= 0) return TSG_OK;
    if (!offsets || !ids || !origins) return fail(TSG_EINVAL, "null argument");
    DevGuard g(h->dev);
    // group clauses by size, preserving arrival order; new sizes create buckets
    // in first-seen order (dict insertion order of ClauseStore.buckets)
    std::vector<int> bucket_of(n);
    for (int64_t i = 0; i < n; ++i) {
        int64_t s64 = offsets[i + 1] - offsets[i];
        if (s64 < 0 || s64 > (1 << 24)) return fail(TSG_EINVAL, "bad clause size");
        int32_t s = (int32_t)s64;
        for (int64_t j = offsets[i]; j < offsets[i + 1]; ++j) {
            int64_t v = lits[j] < 0 ? -(int64_t)lits[j] : lits[j];
            if (v > h->V) h->oob = true;  // stored as-is; testing raises (numpy IndexError, engine.py:251)
        }
        if (ids[i] < 0 || ids[i] > h->max_id) h->max_id = std::max<int64_t>(h->max_id, ids[i] < 0 ? INT64_MAX : ids[i]);
        auto it = h->by_size.find(s);
        int bi;
        if (it == h->by_size.end()) {
            bi = (int)h->buckets.size();
            Bucket b;
            b.size = s;
            b.rank = bi;
            b.parts.resize(h->n_slabs);
            for (int32_t q = 0; q < h->n_slabs; ++q) b.parts[q].slab = q;
            h->buckets.push_back(b);
            h->by_size[s] = bi;
        } else {
            bi = it->second;
        }
        bucket_of[i] = bi;
    }
    // place every clause in a slab part (hot literals first), then one H2D +
    // scatter per (bucket, slab) part
    const int32_t P = h->n_slabs;
    std::vector<int32_t> cnt(P, 0);
    std::vector<int32_t> placed((size_t)std::max<int64_t>(offsets[n] - offsets[0], 1));
    std::vector<uint64_t> hm(n);
    std::vector<int32_t> slab_of_clause(n);
    std::vector<std::vector<int64_t>> members(h->buckets.size() * P);
    for (int64_t i = 0; i < n; ++i) {
        const int32_t s = (int32_t)(offsets[i + 1] - offsets[i]);
        slab_of_clause[i] = place_clause(h, lits + offsets[i], s, cnt, placed.data() + (offsets[i] - offsets[0]),
                                         &hm[i]);
        members[(size_t)bucket_of[i] * P + slab_of_clause[i]].push_back(i);
    }
    if (h->pivot && P == 1) {  // each part's new clauses in pivot-variable order (stable)
        for (auto& mem : members)
            std::stable_sort(mem.begin(), mem.end(), [&](int64_t x, int64_t y) {
                const int64_t sx = offsets[x + 1] - offsets[x], sy = offsets[y + 1] - offsets[y];
                const int64_t vx = sx ? std::llabs((long long)placed[offsets[x] - offsets[0]]) : 0;
                const int64_t vy = sy ? std::llabs((long long)placed[offsets[y] - offsets[0]]) : 0;
                return vx < vy;
            });
    }
    for (size_t mi = 0; mi < members.size(); ++mi) {
        auto& mem = members[mi];
        if (mem.empty()) continue;
        Bucket& b = h->buckets[mi / P];
        Part& p = b.parts[mi % P];
        int64_t k = (int64_t)mem.size();
        CKR(part_reserve(h, p, b.size, p.count + k));
        std::vector<int32_t> hl((size_t)(k * b.size));
        std::vector<int64_t> hid(k);
        std::vector<int32_t> hor(k);
        std::vector<uint64_t> hmk(k);
        for (int64_t c = 0; c < k; ++c) {
            int64_t i = mem[c];
            if (b.size) memcpy(&hl[c * b.size], placed.data() + (offsets[i] - offsets[0]), b.size * 4);
            hid[c] = ids[i];
            hor[c] = origins[i];
            hmk[c] = hm[i];
        }
        if (b.size) {
            int32_t* tmp = nullptr;
            CKR(dalloc(h, (void**)&tmp, k * b.size * 4));
            CK(cudaMemcpyAsync(tmp, hl.data(), k * b.size * 4, cudaMemcpyHostToDevice, h->st));
            k_append<<<grid_for(k * b.size), 256, 0, h->st>>>(tmp, k, b.size, p.count, p.lits);
            CK(cudaGetLastError());
            dfree(h, tmp);
        }
        CK(cudaMemcpyAsync(p.ids + p.count, hid.data(), k * 8, cudaMemcpyHostToDevice, h->st));
        CK(cudaMemcpyAsync(p.origins + p.count, hor.data(), k * 4, cudaMemcpyHostToDevice, h->st));
        CK(cudaMemcpyAsync(p.order + p.count, hmk.data(), k * 8, cudaMemcpyHostToDevice, h->st));
        k_fill_f64<<<grid_for(k), 256, 0, h->st>>>(p.acts + p.count, k, activity);
        CK(cudaGetLastError());
        p.count += k;
        CK(cudaStreamSynchronize(h->st));  // host vectors go out of scope
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
    *count = h->buckets[b].count();
    return TSG_OK;
}

int tsg_bucket_read(tsg_engine* h, int32_t bi, int32_t* lits, int64_t* ids, int32_t* origins, double* acts) {
    CKR(validate_handle(h));
    if (bi < 0 || bi >= (int32_t)h->buckets.size()) return fail(TSG_ERANGE, "bucket %d out of range", bi);
    DevGuard g(h->dev);
    Bucket& b = h->buckets[bi];
    const int64_t total = b.count();
    if (!total) return TSG_OK;
    // every part in its own slot order (original literal order restored), then
    // merged by engine id = the reference's slot order (reports.py)
    std::vector<int32_t> hl(lits && b.size ? total * b.size : 0);
    std::vector<int64_t> hid(total);
    std::vector<int32_t> hor(origins ? total : 0);
    std::vector<double> hac(acts ? total : 0);
    int64_t off = 0;
    for (auto& p : b.parts) {
        if (!p.count) continue;
        if (lits && b.size) {
            int32_t* tmp = nullptr;
            CKR(dalloc(h, (void**)&tmp, p.count * b.size * 4));
            k_deinterleave<<<grid_for(p.count), 256, 0, h->st>>>(p.lits, p.order, p.count, b.size, tmp);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(hl.data() + off * b.size, tmp, p.count * b.size * 4, cudaMemcpyDeviceToHost, h->st));
            dfree(h, tmp);
        }
        CK(cudaMemcpyAsync(hid.data() + off, p.ids, p.count * 8, cudaMemcpyDeviceToHost, h->st));
        if (origins) CK(cudaMemcpyAsync(hor.data() + off, p.origins, p.count * 4, cudaMemcpyDeviceToHost, h->st));
        if (acts) CK(cudaMemcpyAsync(hac.data() + off, p.acts, p.count * 8, cudaMemcpyDeviceToHost, h->st));
        off += p.count;
    }
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
    // parts in a flat list: part index -> (bucket, part)
    std::vector<std::pair<int, int>> parts;
    for (int bi = 0; bi < (int)h->buckets.size(); ++bi)
        for (int pi = 0; pi < (int)h->buckets[bi].parts.size(); ++pi)
            if (h->buckets[bi].parts[pi].count) parts.push_back({bi, pi});
    int64_t* d = nullptr;  // [q | qidx | loc]
    CKR(dalloc(h, (void**)&d, 3 * n * 8));
    CK(cudaMemcpyAsync(d, q.data(), n * 8, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(d + n, qi.data(), n * 8, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemsetAsync(d + 2 * n, 0xFF, n * 8, h->st));
    for (int64_t k = 0; k < (int64_t)parts.size(); ++k) {
        const Part& p = h->buckets[parts[k].first].parts[parts[k].second];
        k_find_ids<<<grid_for(p.count), 256, 0, h->st>>>(p.ids, p.count, d, d + n, n, k, d + 2 * n);
    }
    CK(cudaGetLastError());
    std::vector<int64_t> loc(n);
    CK(cudaMemcpyAsync(loc.data(), d + 2 * n, n * 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    dfree(h, d);
    int64_t total = 0;
    std::vector<int64_t> off(n);
    for (int64_t i = 0; i < n; ++i) {
        if (loc[i] < 0) { sizes[i] = -1; off[i] = total; continue; }
        sizes[i] = h->buckets[parts[loc[i] >> 40].first].size;
        off[i] = total;
        total += sizes[i];
    }
    *n_lits = total;
    if (!lits || total == 0) return TSG_OK;
    if (total > lits_cap) return fail(TSG_ECAPACITY, "%lld literals do not fit %lld", (long long)total, (long long)lits_cap);
    // per part: gather its hits' literals, then place them in request order
    std::vector<std::vector<int64_t>> hit(parts.size());
    for (int64_t i = 0; i < n; ++i)
        if (loc[i] >= 0) hit[loc[i] >> 40].push_back(i);
    for (size_t k = 0; k < parts.size(); ++k) {
        if (hit[k].empty()) continue;
        const Bucket& b = h->buckets[parts[k].first];
        const Part& p = b.parts[parts[k].second];
        const int64_t m = (int64_t)hit[k].size();
        if (b.size == 0) continue;
        std::vector<int64_t> slots(m);
        for (int64_t j = 0; j < m; ++j) slots[j] = loc[hit[k][j]] & ((int64_t(1) << 40) - 1);
        int64_t* ds = nullptr;
        int32_t* dl = nullptr;
        CKR(dalloc(h, (void**)&ds, m * 8));
        CKR(dalloc(h, (void**)&dl, m * b.size * 4));
        CK(cudaMemcpyAsync(ds, slots.data(), m * 8, cudaMemcpyHostToDevice, h->st));
        k_deinterleave_sel<<<grid_for(m), 256, 0, h->st>>>(p.lits, p.order, ds, m, b.size, dl);
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
    for_parts(h, [&](Bucket&, Part& p) {
        if (p.count) k_scale_f64<<<grid_for(p.count), 256, 0, h->st>>>(p.acts, p.count, factor);
    });
    CK(cudaGetLastError());
    return TSG_OK;
}

int tsg_reduce(tsg_engine* h, int64_t eligible_below, int64_t target, int64_t* removed, int64_t* removed_ids) {
    CKR(validate_handle(h));
    if (any_inflight(h)) return fail(TSG_EINVAL, "the store cannot change while a launched round is not collected");
    h->desc_dirty = true;
    DevGuard g(h->dev);
    *removed = 0;
    int64_t total = 0;
    std::vector<int64_t> base = part_bases(h, &total);
    if (total == 0 || target <= 0) return TSG_OK;
    uint64_t *ka = nullptr, *ki = nullptr, *ka2 = nullptr, *ki2 = nullptr;
    int64_t *ix = nullptr, *ix2 = nullptr, *doomed_ids = nullptr;
    uint8_t* keep = nullptr;
    CKR(dalloc(h, (void**)&ka, total * 8)); CKR(dalloc(h, (void**)&ki, total * 8));
    CKR(dalloc(h, (void**)&ka2, total * 8)); CKR(dalloc(h, (void**)&ki2, total * 8));
    CKR(dalloc(h, (void**)&ix, total * 8)); CKR(dalloc(h, (void**)&ix2, total * 8));
    CKR(dalloc(h, (void**)&keep, total));
    CK(cudaMemsetAsync(h->mctr + 4, 0, 8, h->st));
    {
        size_t pi = 0;
        for_parts(h, [&](Bucket&, Part& p) {
            const int64_t pb = base[pi++];
            if (p.count)
                k_reduce_keys<<<grid_for(p.count), 256, 0, h->st>>>(p.acts, p.ids, p.count, pb, eligible_below,
                                                                    ka, ki, ix, h->mctr + 4);
        });
    }
    CK(cudaGetLastError());
    // stable LSD: sort by id, then stably by activity bits => (activity, id) order (engine.py:488)
    size_t tb = 0, tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, ki, ki2, ix, ix2, total, 0, 64, h->st);
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, ka, ka2, ix, ix2, total, 0, 64, h->st);
    void* tmp = nullptr;
    CKR(dalloc(h, &tmp, (int64_t)std::max(tb, tb2) + 16));
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, ki, ki2, ix, ix2, total, 0, 64, h->st));
    k_gather_u64<<<grid_for(total), 256, 0, h->st>>>(ka, ix2, total, ka2);  // act keys in id order
    CK(cudaGetLastError());
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, ka2, ka, ix2, ix, total, 0, 64, h->st));
    unsigned long long n_el = 0;
    CK(cudaMemcpyAsync(&n_el, h->mctr + 4, 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    int64_t rem = std::min<int64_t>(target, (int64_t)n_el);
    if (rem > 0) {
        CK(cudaMemsetAsync(keep, 1, total, h->st));
        CKR(dalloc(h, (void**)&doomed_ids, rem * 8));
        k_mark_doomed<<<grid_for(rem), 256, 0, h->st>>>(ix, rem, keep, ki, doomed_ids);
        CK(cudaGetLastError());
        if (removed_ids) CK(cudaMemcpyAsync(removed_ids, doomed_ids, rem * 8, cudaMemcpyDeviceToHost, h->st));
        CKR(compact_all(h, keep, base));
    }
    dfree(h, tmp); dfree(h, ka); dfree(h, ki); dfree(h, ka2); dfree(h, ki2); dfree(h, ix); dfree(h, ix2);
    dfree(h, keep); dfree(h, doomed_ids);
    CK(cudaStreamSynchronize(h->st));
    *removed = rem;
    h->totals.reduces += 1;
    h->totals.clauses_removed += rem;
    return TSG_OK;
}

int tsg_remove_clauses(tsg_engine* h, const int64_t* ids, int64_t n, int64_t* removed) {
    CKR(validate_handle(h));
    if (any_inflight(h)) return fail(TSG_EINVAL, "the store cannot change while a launched round is not collected");
    h->desc_dirty = true;
    DevGuard g(h->dev);
    *removed = 0;
    int64_t total = 0;
    std::vector<int64_t> base = part_bases(h, &total);
    if (total == 0 || n <= 0) return TSG_OK;
    std::vector<int64_t> del(ids, ids + n);
    std::sort(del.begin(), del.end());
    int64_t* d_del = nullptr;
    uint8_t* keep = nullptr;
    CKR(dalloc(h, (void**)&d_del, n * 8));
    CKR(dalloc(h, (void**)&keep, total));
    CK(cudaMemcpyAsync(d_del, del.data(), n * 8, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemsetAsync(h->mctr + 4, 0, 8, h->st));
    {
        size_t pi = 0;
        for_parts(h, [&](Bucket&, Part& p) {
            const int64_t pb = base[pi++];
            if (p.count)
                k_mark_deleted<<<grid_for(p.count), 256, 0, h->st>>>(p.ids, p.count, pb, d_del, n, keep, h->mctr + 4);
        });
    }
    CK(cudaGetLastError());
    unsigned long long gone = 0;
    CK(cudaMemcpyAsync(&gone, h->mctr + 4, 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (gone) CKR(compact_all(h, keep, base));
    dfree(h, d_del); dfree(h, keep);
    CK(cudaStreamSynchronize(h->st));
    *removed = (int64_t)gone;
    h->totals.clauses_deleted += (int64_t)gone;
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
    int64_t pitch = round_up(h->V + 1, 16);
    int64_t need = pitch * n_rows;
    CK(cudaStreamWaitEvent(h->st, h->ev_encoded, 0));  // the last encode on the encoder stream read rows_own
    h->enc_wait_main = true;                             // the next encode reads what st copies in
    if (need > h->rows_cap) {
        dfree(h, h->rows_own);
        h->rows_own = nullptr;
        int64_t cap = std::max(need, h->rows_cap * 2);
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
__attribute__((target("avx2"))) static void pack_row_avx2(const int8_t* r, int64_t nv1, uint64_t* out, int64_t words) {
    const __m256i one = _mm256_set1_epi8(1), zero = _mm256_setzero_si256();
    int64_t k = 0;
    for (; 32 * k + 32 <= nv1; ++k) {
        const __m256i x = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(r + 32 * k));
        const uint32_t t = (uint32_t)_mm256_movemask_epi8(_mm256_cmpeq_epi8(x, one));
        const uint32_t z = (uint32_t)_mm256_movemask_epi8(_mm256_cmpeq_epi8(x, zero));
        out[k] = (uint64_t)t | ((uint64_t)~z << 32);
    }
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
    for (int64_t r = 0; r < n_rows; ++r) {
        uint64_t* o = out + r * out_pitch_words;
        if (avx2) pack_row_avx2(rows + r * row_pitch, (int64_t)num_vars + 1, o, words);
        else pack_row_scalar(rows + r * row_pitch, (int64_t)num_vars + 1, o, words);
        for (int64_t k = words; k < out_pitch_words; ++k) o[k] = 0;
    }
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
            CK(cudaStreamWaitEvent(h->st, h->ev_read[b], 0));  // its last reader may be on the encoder stream
            dfree(h, h->pbuf[b]);  // stream-ordered after its last reader
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

void persist_tables(tsg_engine* h);

int tsg_round_prepare(tsg_engine* h, const int32_t* group_lanes, const int32_t* group_tid, int32_t n_groups) {
    CKR(validate_handle(h));
    DevGuard g(h->dev);
    if (n_groups < 0 || n_groups > TSG_MAX_GROUPS)
        return fail(TSG_EINVAL, "n_groups must be in 0..%d, got %d", TSG_MAX_GROUPS, n_groups);
    RoundDesc rd;
    rd.n_groups = n_groups;
    rd.glanes.assign(group_lanes, group_lanes + n_groups);
    rd.gtid.assign(group_tid, group_tid + n_groups);
    rd.grow0.resize(n_groups);
    int64_t r = 0;
    for (int i = 0; i < n_groups; ++i) {
        if (rd.glanes[i] < 0 || rd.glanes[i] > h->cfg.lane_width)
            return fail(TSG_ECAPACITY, "%d assignments exceed lane width %d", rd.glanes[i], h->cfg.lane_width);
        rd.grow0[i] = r;
        r += rd.glanes[i];
    }
    rd.n_chunks = (n_groups + h->cfg.group_width - 1) / h->cfg.group_width;
    rd.chunk_off.resize(rd.n_chunks);
    int64_t off = 0;
    for (int c = 0; c < rd.n_chunks; ++c) {
        int G = std::min(h->cfg.group_width, n_groups - c * h->cfg.group_width);
        rd.chunk_off[c] = off;
        off += agg_bytes(h);
        off += round_up(vstride(h) * G * lane_entry_bytes(h), 256);
    }
    // table slots never shrink and hold at least one full chunk, so rounds of
    // up to group_width groups can be prepared while another is in flight
    const int64_t one_chunk = agg_bytes(h) + round_up(vstride(h) * h->cfg.group_width * lane_entry_bytes(h), 256);
    const int64_t slot = std::max(h->slot_bytes, round_up(std::max(off, one_chunk), 4096));
    if (slot != h->slot_bytes) {
        // grow both slots; stream order keeps in-flight rounds valid: their
        // kernels precede the copy, and a later replay reads the moved slot
        int8_t* nt = nullptr;
        CK(cudaStreamWaitEvent(h->st, h->ev_encoded, 0));  // an encode may still write the old slots
        h->enc_wait_main = true;                             // the next encode writes the new buffer
        CKR(dalloc(h, (void**)&nt, 2 * slot));
        if (h->tables && any_inflight(h))
            for (int i = 0; i < 2; ++i)
                CK(cudaMemcpyAsync(nt + i * slot, h->tables + i * h->slot_bytes, h->slot_bytes,
                                   cudaMemcpyDeviceToDevice, h->st));
        dfree(h, h->tables);
        h->tables = nt;
        h->tables_cap = 2 * slot;
        h->slot_bytes = slot;
        h->persist_base = nullptr;
    }
    h->tables_bytes = off;
    h->rd = std::move(rd);
    persist_tables(h);
    return TSG_OK;
}

// Persisting L2 window over both table slots, so the 640 MB clause stream
// and the report records cannot evict the tables.  Set once per table
// allocation: changing the device-wide persisting limit stalls the device,
// so it must stay off the per-round path.  Best effort: another context may
// hold the device-wide persisting carve-out.
void persist_tables(tsg_engine* h) {
    const void* base = h->tables;
    if (!h->l2_persist || h->tables_bytes <= 0 || h->persist_base == base) return;
    h->persist_base = base;
    int max_persist = 0, max_window = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, h->dev);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, h->dev);
    const size_t win = (size_t)std::min<int64_t>(h->slot_bytes + h->tables_bytes, max_window);
    if (max_persist <= 0 || win == 0 ||
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(win, (size_t)max_persist)) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    cudaStreamAttrValue attr{};
    attr.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    attr.accessPolicyWindow.num_bytes = win;
    attr.accessPolicyWindow.hitRatio = std::min(1.0f, (float)max_persist / (float)win);
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute(h->st, cudaStreamAttributeAccessPolicyWindow, &attr) != cudaSuccess)
        cudaGetLastError();
}

// Make round state k's record buffers the active ones (the fields of
// tsg_engine); the other state's buffers wait in `alt`.
void use_reports(tsg_engine* h, int k) {
    if (h->report_rs == k) return;
    std::swap(h->out, h->alt.out); std::swap(h->out2, h->alt.out2);
    std::swap(h->out_cap, h->alt.out_cap); std::swap(h->out2_cap, h->alt.out2_cap);
    std::swap(h->out12, h->alt.out12); std::swap(h->out12_cap, h->alt.out12_cap);
    std::swap(h->ev_cur, h->alt.ev);
    std::swap(h->n_out, h->alt.n_out); std::swap(h->n_alloc, h->alt.n_alloc);
    std::swap(h->compacted, h->alt.compacted);
    h->report_rs = k;
}

// Launch the test of the prepared, encoded round (table slot h->tslot) in
// the next round state: kernels, counter copy-out and its event are queued,
// nothing waits.  At most two rounds are in flight.
int round_launch(tsg_engine* h, double inc, bool flip) {
    const int k = h->next_rs;
    auto& R = h->rs[k];
    if (R.inflight) return fail(TSG_EINVAL, "two rounds are in flight: collect one first");
    for (const auto& Q : h->rs)
        if (Q.inflight && Q.slot == h->tslot)
            return fail(TSG_EINVAL, "table slot %d still belongs to an uncollected round", h->tslot);
    use_reports(h, k);
    if (!h->out) {
        h->out_cap = std::max<int64_t>(h->alt.out_cap, 1 << 16);
        CKR(dalloc(h, (void**)&h->out, h->out_cap * (int64_t)sizeof(tsg_report)));
    }
    // this state's buffers may still be copying out from two rounds ago
    // (no-op if never recorded)
    CK(cudaStreamWaitEvent(h->st, h->ev_cur, 0));
    h->n_out = 0;
    h->n_alloc = 0;
    h->compacted = true;
    R.fl = h->rd;
    R.slot = h->tslot;
    R.inc = inc;
    R.seq = ++h->round_seq;
    R.run = 0;
    // 8-byte egress: the kernel writes the packed u64 records itself when
    // they fit (ids < 2^27, <= 32 groups, 32-bit lane masks)
    R.rec8 = h->record_bytes == 8 && !wide_lane(h) && h->max_id < (int64_t(1) << 27) && h->rd.n_groups <= 32;
    if (R.fl.n_chunks && h->oob) {  // out-of-range literal stored: numpy would raise IndexError
        CK(cudaMemsetAsync(h->mctr + 4, 0, 8, h->st));
        for_parts(h, [&](Bucket& b, Part& p) {
            if (p.count && b.size)
                k_max_var<<<grid_for(p.count * b.size), 256, 0, h->st>>>(p.lits, p.count, b.size, h->mctr + 4);
        });
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h->h_mctr + 4, h->mctr + 4, 8, cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
        if ((int64_t)h->h_mctr[4] > h->V)
            return fail(TSG_ERANGE, "index %lld is out of bounds for axis 0 with size %d", (long long)h->h_mctr[4], h->V + 1);
        h->oob = false;
    }
    if (R.fl.n_chunks) {
        CKR(build_desc(h));
        if (h->n_tiles >= (int64_t)INT32_MAX / 2)  // the kernels index tiles with 32-bit integers
            return fail(TSG_ECAPACITY, "store of %lld tiles exceeds the 32-bit tile index", (long long)h->n_tiles);
        if (R.fl.n_chunks > 1) {
            // carry stamps are matched by value ((round, run) << 32 | tid): the
            // buffer is cleared every multi-chunk round, so neither a recycled
            // allocation (another engine's stamps) nor a round 2^25 launches ago
            // can fake a "(engine id, tid) already reported"
            CKR(dgrow(h, &R.carry, &R.carry_cap, std::max<int64_t>(1, h->n_tiles * STRIDE)));
            CK(cudaMemsetAsync(R.carry, 0, (size_t)std::max<int64_t>(1, h->n_tiles * STRIDE) * sizeof(int64_t), h->st));
        }
        const bool timing = timed_round(h, R.seq);
        R.timed = timing;
        if (timing) CK(cudaEventRecord(R.ev_tst[0], h->st));
        CKR(run_tests(h, k, inc, 0));
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
// buffer and replay emission if it overflowed (its table slot and carry
// stamps are its own, so the replay is exact even with the next round in
// flight); fill its figures.  The fetch calls then read its records.
int round_collect(tsg_engine* h, tsg_round_result* out) {
    int k = -1;
    for (int j = 0; j < 2; ++j)
        if (h->rs[j].inflight && (k < 0 || h->rs[j].seq < h->rs[k].seq)) k = j;
    if (k < 0) return fail(TSG_EINVAL, "no launched round to collect");
    auto& R = h->rs[k];
    R.inflight = false;
    use_reports(h, k);
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
        int64_t n_slots = (int64_t)R.h_ctr[0];
        int64_t positives = (int64_t)R.h_ctr[1];
        res.lane_triggers = (int64_t)R.h_ctr[2];
        int64_t n_rec = (int64_t)R.h_ctr[3];
        // overflow: grow, replay emission only (no activity / counter side
        // effects).  Slot reservation depends on which warp tests which tile,
        // so a replay may need a different count.
        while (n_slots > h->out_cap) {
            dfree(h, h->out);
            h->out = nullptr;
            h->out_cap = n_slots + n_slots / 4 + 1024 + (int64_t)h->nsm * 64 * (int64_t)REPORT_CHUNK;
            if (h->out_cap >= (int64_t)INT32_MAX)  // report slots are 32-bit in the kernels
                return fail(TSG_ECAPACITY, "%lld report slots exceed the 32-bit record index", (long long)n_slots);
            CKR(dalloc(h, (void**)&h->out, h->out_cap * (int64_t)sizeof(tsg_report)));
            CK(cudaMemsetAsync(R.ctr, 0, 4 * sizeof(unsigned long long), h->st));
            R.run++;
            CKR(run_tests(h, k, R.inc, 1));
            CK(cudaMemcpyAsync(R.h_ctr, R.ctr, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->st));
            CK(cudaStreamSynchronize(h->st));
            if ((int64_t)R.h_ctr[3] != n_rec)
                return fail(TSG_ECUDA, "report replay mismatch: %lld records, %lld in the first run (replay %d, %d chunks)",
                            (long long)R.h_ctr[3], (long long)n_rec, R.run, rd.n_chunks);
            n_slots = (int64_t)R.h_ctr[0];
            res.reruns++;
        }
        if (res.reruns) CK(cudaMemsetAsync(R.ctr, 0, 4 * sizeof(unsigned long long), h->st));
        h->n_out = n_rec;
        h->n_alloc = n_slots;
        h->compacted = n_slots == n_rec;
        int64_t n = store_size(h);
        int64_t lanes_total = 0;
        for (int c = 0; c < rd.n_chunks; ++c) {
            int32_t g0 = c * h->cfg.group_width;
            int G = std::min(h->cfg.group_width, rd.n_groups - g0);
            int64_t lanes = 0;
            for (int gg = 0; gg < G; ++gg) lanes += rd.glanes[g0 + gg];
            res.aggregate_tests += n * G;
            lanes_total += lanes;
        }
        res.clauses_tested = n * rd.n_chunks;
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
    int64_t need_rows = h->rd.n_groups ? h->rd.grow0.back() + h->rd.glanes.back() : 0;
    if (need_rows > h->n_rows) return fail(TSG_EINVAL, "groups need %lld rows, %lld staged", (long long)need_rows, (long long)h->n_rows);
    if (!h->rd.n_chunks) return TSG_OK;
    for (const auto& Q : h->rs)
        if (Q.inflight && Q.slot == h->tslot)
            return fail(TSG_EINVAL, "table slot %d still belongs to an uncollected round", h->tslot);
    // The encoder's inputs: rows (ingress stream, or st for int8 / device
    // copies), the table slot (free once its round was collected -- the host
    // waited for it), the state's polarity counters (zeroed by that round).
    h->est = h->async_encode ? h->enc_st : h->st;
    if (h->est != h->st && h->enc_wait_main) {
        CK(cudaEventRecord(h->ev_main, h->st));
        CK(cudaStreamWaitEvent(h->est, h->ev_main, 0));
        h->enc_wait_main = false;
    }
    if (h->packed && h->pstaged) CK(cudaStreamWaitEvent(h->est, h->ev_staged[h->pk], 0));  // rows copied in
    const bool timing = timed_round(h, h->round_seq + 1);  // the round this encode feeds
    if (timing) CK(cudaEventRecord(h->ev_enc[h->tslot][0], h->est));
    auto& Rn = h->rs[h->next_rs];
    if (Rn.pol_pending)  // re-encoded without a launch: count this encode only
        CK(cudaMemsetAsync(Rn.ctr + 6, 0, 2 * sizeof(unsigned long long), h->est));
    Rn.pol_pending = true;
    const int rc = do_encode(h);
    if (h->packed && h->pstaged) CK(cudaEventRecord(h->ev_read[h->pk], h->est));
    if (timing) CK(cudaEventRecord(h->ev_enc[h->tslot][1], h->est));
    if (h->est != h->st) {  // everything after this on st (test, broadcast) sees the tables
        CK(cudaEventRecord(h->ev_encoded, h->est));
        CK(cudaStreamWaitEvent(h->st, h->ev_encoded, 0));
    }
    h->est = h->st;
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

// Byte layout of the prepared round's tables (one chunk): the aggregate
// table at agg_off (agg_bytes), then group g's lane entries at lane_off +
// g * group_bytes -- the regions tsg_round_encode_groups ranks combine.
int tsg_round_layout(tsg_engine* h, int64_t* agg_off, int64_t* agg_len, int64_t* lane_off, int64_t* group_bytes) {
    CKR(validate_handle(h));
    if (h->rd.n_chunks < 1) return fail(TSG_EINVAL, "no prepared round");
    *agg_off = h->rd.chunk_off[0];
    *agg_len = (int64_t)(h->V + 2) * agg_entry_bytes(h);
    *lane_off = h->rd.chunk_off[0] + agg_bytes(h);
    *group_bytes = vstride(h) * lane_entry_bytes(h);
    return TSG_OK;
}

int tsg_round_tables(tsg_engine* h, void** device_ptr, int64_t* bytes) {
    CKR(validate_handle(h));
    *device_ptr = h->tables + h->tslot * h->slot_bytes;
    *bytes = h->tables_bytes;
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

// the source and size of the round's first k records in the egress format
int egress_view(tsg_engine* h, int64_t k, const void** src, int64_t* bytes) {
    if (h->rs[h->fetch_rs].rec8) {  // written as 8-byte records by the kernel
        if (h->record_bytes != 8)
            return fail(TSG_EINVAL, "the round was launched with 8-byte records; fetch it before changing the format");
        *src = h->out;
        *bytes = k * 8;
        return TSG_OK;
    }
    if (h->record_bytes == 16 || k <= 0) {
        *src = h->out;
        *bytes = k * (int64_t)sizeof(tsg_report);
        return TSG_OK;
    }
    if (h->record_bytes == 8) {
        if (h->max_id >= (int64_t(1) << 27) || h->rs[h->fetch_rs].fl.n_groups > 32)
            return fail(TSG_ECAPACITY, "8-byte records need engine ids < 2^27 and <= 32 groups (largest id %lld, "
                        "%d groups): use 12-byte records", (long long)h->max_id, h->rs[h->fetch_rs].fl.n_groups);
        CKR(dgrow(h, &h->out12, &h->out12_cap, k * 8));
        k_pack_records8<<<grid_for(k), 256, 0, h->st>>>(h->out, k, reinterpret_cast<uint64_t*>(h->out12));
        CK(cudaGetLastError());
        *src = h->out12;
        *bytes = k * 8;
        return TSG_OK;
    }
    CKR(dgrow(h, &h->out12, &h->out12_cap, k * 12));
    k_pack_records12<<<grid_for(k), 256, 0, h->st>>>(h->out, k, h->out12);
    CK(cudaGetLastError());
    *src = h->out12;
    *bytes = k * 12;
    return TSG_OK;
}

int tsg_fetch_reports(tsg_engine* h, tsg_report* out, int64_t cap, int64_t* n) {
    CKR(validate_handle(h));
    DevGuard g(h->dev);
    use_reports(h, h->fetch_rs);
    CKR(compact_reports(h));
    int64_t k = std::min(cap, h->n_out);
    if (k > 0) {
        const void* src = nullptr;
        int64_t bytes = 0;
        CKR(egress_view(h, k, &src, &bytes));
        CK(cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
    }
    *n = k;
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
    DevGuard g(h->dev);
    use_reports(h, h->fetch_rs);
    CKR(compact_reports(h));
    const int64_t k = std::min(cap, h->n_out);
    *n = k;
    if (k <= 0) return TSG_OK;
    const void* src = nullptr;
    int64_t bytes = 0;
    CKR(egress_view(h, k, &src, &bytes));
    CK(cudaEventRecord(h->ev_ready, h->st));
    CK(cudaStreamWaitEvent(h->egress, h->ev_ready, 0));
    CK(cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToHost, h->egress));
    CK(cudaEventRecord(h->ev_cur, h->egress));
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
    DevGuard g(h->dev);
    use_reports(h, h->fetch_rs);
    if (h->rs[h->fetch_rs].rec8)
        return fail(TSG_EINVAL, "the round's records are 8-byte u64 (tsg_set_record_bytes(8)), not tsg_report");
    CKR(compact_reports(h));
    *device_ptr = h->out;
    *n = h->n_out;
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

}  // extern "C"
