/*
 * tsg.h -- C ABI of the B200-native GpuShareSat clause-usefulness filter.
 *
 * This is the drop-in boundary for the hot path of the reference engine
 * (/root/reference/pkg/src/triggersat/engine.py, class Engine): the clause
 * store, the assignment encoder, the two-stage trigger test and report
 * emission.  The Python mirror of the reference API
 * (paper_2012_03119_b200/engine.py, bitpack.py) binds exactly these entry
 * points with ctypes; INTEGRATION.md shows the binding a reference maintainer
 * would add.  Plain pointers and sizes only: no torch types cross the ABI.
 *
 * Threading: one handle belongs to one engine-worker thread (the reference
 * runs run_round / reduce_store only on its worker, engine.py:257-264).  All
 * calls on a handle are serialised on the handle's CUDA stream.  Calls that
 * return host data synchronise that stream before returning.
 *
 * Errors: every entry point returns TSG_OK or a TSG_E* code; tsg_last_error()
 * gives the thread's last message.  The Python layer maps TSG_EINVAL to
 * ValueError, TSG_ECAPACITY to CapacityError, TSG_ERANGE to IndexError and
 * the rest to RuntimeError, matching bitpack.py:30-36,92-103 / engine.py:64-74.
 * There is no CPU fallback: without a CUDA device every compute call fails
 * with TSG_ECUDA.
 */
#ifndef TSG_H
#define TSG_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSG_ABI_VERSION 2

#define TSG_OK 0
#define TSG_EINVAL 1    /* ValueError    (bad width / length / config)   */
#define TSG_ECAPACITY 2 /* CapacityError (bitpack.py:28-29)              */
#define TSG_ERANGE 3    /* IndexError                                    */
#define TSG_ECUDA 4     /* CUDA runtime failure or no device             */
#define TSG_ENOMEM 5    /* device allocation failed                      */

typedef struct tsg_engine tsg_engine;

/* EngineConfig knobs that reach the device (engine.py:44-74).  The queue,
 * decay and reduce knobs stay in the host layer, as in the reference. */
typedef struct tsg_config {
    int32_t lane_width;      /* 1..64, EngineConfig.lane_width (engine.py:56)   */
    int32_t group_width;     /* 1..64, EngineConfig.group_width (engine.py:57)  */
    int32_t device;          /* CUDA device ordinal                              */
    int32_t flags;           /* TSG_F_* below                                    */
    int64_t report_capacity; /* initial device report buffer (records); 0=auto  */
} tsg_config;

#define TSG_F_TIMING 1    /* record CUDA events around encode/test (fills *_ms)      */
#define TSG_F_ALL_PAIRS 2 /* every triggering (clause, group), see tsg_set_all_pairs  */
#define TSG_F_CHUNK_FILTER 4 /* multi-chunk rounds sweep a chunk-level aggregate first
                                (PAPER.md:425's 32x32x32 hierarchy; env TSG_CHUNK_FILTER=0/1
                                overrides); off by default: profiles/r02_hier_aggregate.md */

/* Per-round figures, the quantities engine.py:437-467 adds to its counters. */
typedef struct tsg_round_result {
    int64_t reports;                  /* records emitted (after (eid, tid) dedup unless all-pairs) */
    int64_t clauses_tested;           /* engine.py:445 (once per chunk)           */
    int64_t aggregate_tests;          /* engine.py:446                            */
    int64_t aggregate_tests_negative; /* engine.py:465-467                        */
    int64_t lane_tests;               /* engine.py:447                            */
    int64_t lane_triggers;            /* engine.py:461                            */
    int32_t n_chunks;                 /* ceil(n_groups / group_width)             */
    int32_t reruns;                   /* record-buffer overflow replays (0 or 1)  */
    double encode_ms;                 /* device time, TSG_F_TIMING (-1: not sampled, tsg_set_timing) */
    double test_ms;                   /* device time of the trigger kernels       */
    int64_t chunk_positives;          /* (clause, chunk) pairs the chunk-level aggregate sweep
                                          left for stage 1; = clauses_tested when
                                         the round has one chunk                   */
} tsg_round_result;

/* Cumulative figures of an engine (tsg_counters): the reference's counter
 * dict (engine.py:284-299) as far as the device sees it -- snapshot and
 * drop counts stay with the host side that owns the queues. */
typedef struct tsg_counters_t {
    int64_t rounds;                   /* rounds collected                         */
    int64_t reports;                  /* records emitted                          */
    int64_t clauses_tested;
    int64_t aggregate_tests;
    int64_t aggregate_tests_negative;
    int64_t lane_tests;
    int64_t lane_triggers;
    int64_t reruns;                   /* report-buffer overflow replays           */
    int64_t clauses_added;
    int64_t clauses_removed;          /* by tsg_reduce (engine.py:469-505)        */
    int64_t clauses_deleted;          /* by tsg_remove_clauses                    */
    int64_t reduces;
} tsg_counters_t;

/* One report record, 16 bytes (engine.py:90-102 Report minus the literals,
 * which the host keeps): key = engine_id << 16 | group, where `group` is the
 * global group index in round order (engine.py:390-399) and the destination
 * thread is that group's tid.  Engine ids must fit in 48 bits and a round
 * holds at most 65535 groups.
 *
 * Order: inside a size bucket, slot order equals engine-id order (clauses
 * are appended in id order and compaction preserves order, engine.py:150-163,
 * 184-200), so sorting records by (group / group_width, creation rank of the
 * clause's size bucket, engine_id, group) reproduces the reference's emission
 * order (engine.py:403-464). */
typedef struct tsg_report {
    uint64_t key;
    uint64_t lane_mask;
} tsg_report;
#define TSG_REPORT_ENGINE_ID(r) ((int64_t)((r).key >> 16))
#define TSG_REPORT_GROUP(r) ((int32_t)((r).key & 0xFFFFu))
#define TSG_MAX_GROUPS 65535

const char* tsg_last_error(void);
int tsg_abi_version(void);
int tsg_device_count(int32_t* n);

/* Engine(num_vars, thread_count, EngineConfig) -- engine.py:266-301 */
int tsg_create(int32_t num_vars, const tsg_config* cfg, tsg_engine** out);
int tsg_destroy(tsg_engine* h);

/* ---- clause store (engine.py:122-235) -------------------------------------
 * _integrate_exports / ClauseStore.insert (engine.py:348-358, 213-219):
 * append n clauses in order.  Clause i has literals lits[offsets[i] ..
 * offsets[i+1]), engine id ids[i], origin origins[i]; all start at
 * `activity`.  Buckets are created in first-seen size order.  Engine ids
 * must increase with insertion order (the reference assigns them that way,
 * engine.py:305-317): the store orders clauses by id wherever the
 * reference's slot order is visible (reports, bucket reads), because the
 * device layout inside a bucket is pivot-ordered. */
int tsg_add_clauses(tsg_engine* h, const int32_t* lits, const int64_t* offsets,
                    int64_t n, const int64_t* ids, const int32_t* origins,
                    double activity);
int tsg_store_size(tsg_engine* h, int64_t* n);               /* len(store)        */
int tsg_bucket_count(tsg_engine* h, int32_t* nb);            /* buckets (created) */
int tsg_bucket_info(tsg_engine* h, int32_t b, int32_t* size, int64_t* count);
/* copy bucket b back: lits clause-major (count*size), ids, origins,
 * activities; any pointer may be NULL (engine.py:165-169, 221-231) */
int tsg_bucket_read(tsg_engine* h, int32_t b, int32_t* lits, int64_t* ids,
                    int32_t* origins, double* acts);
/* ClauseStore.scale_activities (engine.py:233-235) */
/* Literals of stored clauses by engine id, original literal order
 * (engine.py:165-169 lits_at; Report.lits, engine.py:409-414), so a host
 * that keeps no literal copy can resolve report records.  sizes[i] = size
 * of clause ids[i] or -1 if it is not stored; the found clauses' literals
 * are concatenated in request order into lits (*n_lits of them; with
 * lits == NULL only sizes and *n_lits are filled; TSG_ECAPACITY if they do
 * not fit lits_cap). */
int tsg_get_clauses(tsg_engine* h, const int64_t* ids, int64_t n, int32_t* sizes, int32_t* lits,
                    int64_t lits_cap, int64_t* n_lits);
int tsg_counters(tsg_engine* h, tsg_counters_t* out);
/* All-pairs mode (or TSG_F_ALL_PAIRS at create): rounds launched while it is
 * on emit one record for EVERY triggering (clause, group) -- the pair set of
 * multi_trigger (bitpack.py:282-300) -- instead of the reference's first
 * triggering group per (clause, thread) (engine.py:462-464).  Activities and
 * counters are unaffected; `reports` counts the records. */
int tsg_set_all_pairs(tsg_engine* h, int32_t on);
/* With TSG_F_TIMING: bracket only rounds whose launch sequence number is a
 * multiple of `every` with timing events (0 = none; default 1 = all) --
 * each event stalls the stream front end for a few microseconds.  Unsampled
 * rounds report encode_ms = test_ms = -1. */
int tsg_set_timing(tsg_engine* h, int32_t every);
int tsg_scale_activities(tsg_engine* h, double factor);
/* reduce_store selection + compaction (engine.py:476-500): remove the
 * `target` smallest (activity, engine_id) among clauses with id <
 * eligible_below (device radix select on the 128-bit key); order-preserving
 * compaction per bucket.  removed_ids (may be NULL, else room for `target`)
 * receives the removed ids in ascending order. */
int tsg_reduce(tsg_engine* h, int64_t eligible_below, int64_t target,
               int64_t* removed, int64_t* removed_ids);
/* The same selection split for clause shards (one store per GPU): begin
 * builds the keys of the clauses with id < eligible_below and returns how
 * many there are; hist fills hist[256] with the number of those keys whose
 * top `bits` bits (a multiple of 8, < 128) equal the prefix (prefix_hi =
 * key bits 127..64 = the activity's IEEE bits, prefix_lo = bits 63..0 = the
 * engine id, both left-aligned, the rest zero), per value of the next 8
 * bits; the caller sums the shards' histograms and extends the prefix
 * until it pins the global target-th smallest key; commit removes every
 * eligible key whose top `bits` bits are <= the prefix (bits = 0: none)
 * and ends the selection (removed_ids: room for cap ids, ascending; may be
 * NULL).  The store must not change between begin and commit. */
int tsg_reduce_begin(tsg_engine* h, int64_t eligible_below, int64_t* n_eligible);
int tsg_reduce_hist(tsg_engine* h, uint64_t prefix_hi, uint64_t prefix_lo, int32_t bits, uint64_t* hist);
int tsg_reduce_commit(tsg_engine* h, uint64_t prefix_hi, uint64_t prefix_lo, int32_t bits, int64_t* removed,
                      int64_t* removed_ids, int64_t cap);
/* explicit delete (streaming config C4): remove the listed ids if present,
 * order-preserving (the compact(keep) of engine.py:184-200). */
int tsg_remove_clauses(tsg_engine* h, const int64_t* ids, int64_t n, int64_t* removed);

/* ---- one exchange round (engine.py:369-467) ---------------------------------
 * 1. tsg_stage_snapshots: the round's snapshots, already grouped in round
 *    order (tids ascending, lane_width per group, engine.py:390-399), as rows of
 *    num_vars+1 int8 values ({1,-1,0}; anything non-zero and not 1 reads as
 *    False, like bitpack.py:108-109).  `row_pitch` is the byte distance between
 *    rows at `rows`; on_device=1 means `rows` is a device pointer.
 * 2. tsg_round: encode (K1/K2) and test (K3+K4+K5) every chunk of
 *    group_width groups against every bucket in ONE trigger launch (each
 *    clause's literal rows are read once for all chunks; with
 *    TSG_F_CHUNK_FILTER a chunk-level aggregate is swept first);
 *    bumps activities by activity_inc * hits (engine.py:460, fp64, no FMA).
 *    A thread's groups must be consecutive (TSG_EINVAL otherwise).
 * 3. tsg_fetch_reports: copy the round's report records out (exactly
 *    `reports` records, unordered: the host orders them, reports.py).
 * The split form (prepare / encode / tables / test) exists for multi-GPU:
 * rank 0 encodes, the packed tables are broadcast over NVLink, every rank
 * tests its own clause shard. */
int tsg_stage_snapshots(tsg_engine* h, const int8_t* rows, int64_t n_rows,
                        int64_t row_pitch, int32_t on_device);
int tsg_round(tsg_engine* h, const int32_t* group_lanes, const int32_t* group_tid,
              int32_t n_groups, double activity_inc, tsg_round_result* out);
/* Packed snapshot rows (snapshot ingress): 2 bits per
 * variable, a quarter of the int8 bytes.  u64 word k of a row covers
 * variables 32k..32k+31: bit i of the low half = (value == 1), bit i of the
 * high half = (value != 0) -- the same is_true / is_set the encoder derives
 * from int8 rows (bitpack.py:104-111).  A row has tsg_packed_words(num_vars)
 * words.  tsg_pack_rows is host code (no device, thread-safe: solver threads
 * pack their own snapshots); tsg_stage_packed replaces tsg_stage_snapshots
 * for the next round (on_device=1: `rows` is device memory, 32-byte aligned,
 * pitch a multiple of 4 words, used in place).  Host rows are copied on the
 * library's ingress stream into one of two staging buffers, so the next
 * round's rows go in while the current round is tested: the call returns
 * before a copy from pinned memory has finished, and pinned rows must stay
 * unchanged until the round encoded from them is collected (pageable rows
 * are consumed before the call returns). */
int tsg_packed_words(int32_t num_vars, int64_t* words);
int tsg_pack_rows(const int8_t* rows, int64_t n_rows, int64_t row_pitch, int32_t num_vars,
                  uint64_t* out, int64_t out_pitch_words);
int tsg_stage_packed(tsg_engine* h, const uint64_t* rows, int64_t n_rows,
                     int64_t pitch_words, int32_t on_device);
/* Stage a round whose rows arrive partly packed and partly as int8: rows
 * 0..n_packed-1 from `packed` (tsg_pack_rows words), rows n_packed.. from
 * `raw` (int8, num_vars+1 values each), copied in on the ingress stream and
 * packed on the device behind the packed ones -- host packing and the link
 * share a round's ingress (the host packs part of the rows while the rest
 * crosses as int8).  Host sources must stay unchanged until the round is
 * collected (as tsg_stage_packed's pinned rows). */
int tsg_stage_packed_mixed(tsg_engine* h, const uint64_t* packed, int64_t n_packed, int64_t pitch_words,
                           const int8_t* raw, int64_t n_raw, int64_t raw_pitch);
int tsg_round_prepare(tsg_engine* h, const int32_t* group_lanes,
                      const int32_t* group_tid, int32_t n_groups);
int tsg_round_encode(tsg_engine* h);
int tsg_round_tables(tsg_engine* h, void** device_ptr, int64_t* bytes);
/* One process driving several GPUs (one engine per device, each holding a
 * clause shard): copy the encoded tables of src's prepared round into dst's
 * table slot over NVLink (peer copy, ordered after src's encode; src's next
 * encode waits for it).  Both engines must have prepared the same round;
 * dst then launches without encoding. */
int tsg_round_tables_copy(tsg_engine* dst, tsg_engine* src);
/* Split snapshot ingress across GPUs: each rank stages the
 * packed rows of groups [g_begin, g_end) only and encodes them; lane entries
 * of the other groups are left for an all-gather, aggregate words carry only
 * these groups' bits (disjoint across ranks, so a sum all-reduce ORs them);
 * exactly one rank passes sentinel = 1.  One chunk, lane_width <= 32.
 * tsg_round_layout gives the byte offsets inside tsg_round_tables' region:
 * aggregate table [agg_off, agg_off + agg_len), group g's lane entries at
 * lane_off + g * group_bytes. */
int tsg_round_encode_groups(tsg_engine* h, int32_t g_begin, int32_t g_end, int32_t sentinel);
int tsg_round_layout(tsg_engine* h, int64_t* agg_off, int64_t* agg_len, int64_t* lane_off,
                     int64_t* group_bytes);
int tsg_round_test(tsg_engine* h, double activity_inc, tsg_round_result* out);
/* Asynchronous test (device rounds back to back): tsg_round_launch queues
 * the test of the prepared, encoded round and returns; the next round may
 * then be staged, prepared, encoded (into the other of two table slots) and
 * launched before tsg_round_collect waits for the OLDEST launched round's
 * figures -- so the GPU always has the next round queued.  Up to two rounds
 * in flight, each with its own table slot, counters and record buffers; a
 * round must be collected before its table slot is encoded again, and the
 * store must not change while any round is in flight (TSG_EINVAL).  The
 * fetch calls read the records of the last collected round. */
int tsg_round_launch(tsg_engine* h, double activity_inc);
int tsg_round_collect(tsg_engine* h, tsg_round_result* out);
int tsg_fetch_reports(tsg_engine* h, tsg_report* out, int64_t cap, int64_t* n);
/* Pipelined egress: compact the round's records and start their copy into
 * `out` (pinned host memory) on the handle's egress stream, returning the
 * record count at once.  The next round writes the other of two record
 * buffers, so its ingress and test overlap this copy (PCIe is full duplex);
 * a round never overwrites a buffer whose copy-out is still running.  `out`
 * must stay untouched until tsg_fetch_wait returns. */
int tsg_fetch_reports_async(tsg_engine* h, tsg_report* out, int64_t cap, int64_t* n);
int tsg_fetch_wait(tsg_engine* h);
/* Egress record format of tsg_fetch_reports / tsg_fetch_reports_async: 16
 * (tsg_report, default) or 12 bytes -- {uint64 key, uint32 lane_mask},
 * packed, for lane_width <= 32 -- a quarter fewer bytes over PCIe -- or 8
 * bytes, one uint64 engine_id << 37 | group << 32 | lane_mask, half the
 * bytes, when every engine id ever added is < 2^27 and the round has <= 32
 * groups (a fetch that does not fit fails with TSG_ECAPACITY). */
int tsg_set_record_bytes(tsg_engine* h, int32_t bytes);
/* The last collected round's records of n_h engines (one engine, or clause
 * shards that ran the same round) in the reference's delivery order
 * (engine.py:403-414, 462-464): destination thread major (ascending tid),
 * then chunk, creation rank of the clause's size bucket (rank_of_size[size]
 * = the caller's global bucket creation order), engine id, group.  Ordered
 * on hs[0]'s device (keys per shard, stable LSD radix sort); writes engine
 * ids (eid_bytes 4 or 8 per id), lane masks (mask_bytes 4 or 8) and, if
 * `groups` is not NULL, the int32 group of each record into the host arrays
 * and, per destination d (the d-th run of equal tids in the
 * round's groups), its record count into dest_counts[d].  *n = records;
 * TSG_ECAPACITY if they exceed cap or a field does not fit. */
int tsg_fetch_ordered(tsg_engine* const* hs, int32_t n_h, const int32_t* rank_of_size, int32_t n_sizes,
                      void* eids, int32_t eid_bytes, void* masks, int32_t mask_bytes, int32_t* groups,
                      int64_t* dest_counts, int64_t cap, int64_t* n);
/* The next round's packed rows from n_segs segments in host or device memory
 * (segment i: rows[i] rows at segs[i], pitch_words apart), concatenated in
 * order -- e.g. the per-thread snapshot queues -- staged like
 * tsg_stage_packed on the ingress stream, after every copy queued there by
 * tsg_ingress_copy (the segments must stay unchanged until the round encoded
 * from them is collected). */
int tsg_stage_packed_segments(tsg_engine* h, const uint64_t* const* segs, const int64_t* rows, int32_t n_segs,
                              int64_t pitch_words);
/* Device memory on the engine's device, and an asynchronous copy on the
 * engine's ingress stream (host -> device for queued snapshot rows).
 * tsg_ingress_copy may be called from any host thread concurrently with the
 * engine worker; the source must stay unchanged until the next round that
 * stages from the destination is collected. */
int tsg_device_alloc(tsg_engine* h, int64_t bytes, void** p);
int tsg_device_free(tsg_engine* h, void* p);
int tsg_ingress_copy(tsg_engine* h, void* dst, const void* src, int64_t bytes);
/* Page-locked host memory (cudaMallocHost) for ingress rows and records. */
int tsg_host_alloc(int64_t bytes, void** p);
int tsg_host_free(void* p);
/* device pointer + count of the round's records (for device-side consumers) */
int tsg_reports_device(tsg_engine* h, void** device_ptr, int64_t* n);
int tsg_sync(tsg_engine* h);
/* the handle's CUDA stream (cudaStream_t), for interop */
int tsg_stream(tsg_engine* h, void** stream);

/* ---- host report ring (north_star subsystem 4) ---------------
 * Replaces the copy-out of engine.py:462-464's report emission: while a ring
 * is open, every launched round's trigger kernel writes its records through
 * warp-aggregated reservations straight into page-locked host memory mapped
 * into the device, and CPU threads drain them while the kernel still runs --
 * no device record buffer, no D2H copy, no fetch call.  Records arrive in
 * reservation order (not the reference's delivery order); the (eid, tid)
 * dedup and counters are the round's as usual.  A full ring stalls the
 * reserving warps until the drainer frees slots, for at most wait_us per
 * flush; past that the round's remaining records are dropped and its collect
 * fails with TSG_ECAPACITY (the ring stays failed until reopened).
 * lane_width <= 32, engine ids < 2^48.  The fetch calls fail for ringed
 * rounds. */
/* open a ring of >= capacity records (rounded up to a power of two, >= 128);
 * no round may be in flight */
int tsg_ring_open(tsg_engine* h, int64_t capacity, int64_t wait_us);
int tsg_ring_close(tsg_engine* h);
/* Copy up to cap landed records of one contiguous run of ring positions,
 * in order, into out (key = engine_id << 16 | group, lane_mask) and free
 * their slots; *first_pos (may be NULL) = the ring position of out[0] --
 * records are numbered by position from the ring's opening, rounds in launch
 * order, so drainers on several threads can reassemble them.  Returns when
 * cap records were copied, when the run ends, when at least one was and the
 * next has not landed for min(timeout_us, 20) microseconds, or after
 * timeout_us with none.  Thread-safe against the round calls on other
 * threads; several drainers consume disjoint runs concurrently. */
int tsg_ring_drain(tsg_engine* h, tsg_report* out, int64_t cap, int64_t* n, int64_t timeout_us,
                   int64_t* first_pos);
/* records of the rounds collected so far, records drained, whether records
 * were dropped */
int tsg_ring_status(tsg_engine* h, int64_t* expected, int64_t* consumed, int32_t* failed);

/* ---- standalone bit-parallel kernels (bitpack.py) ----------------------------
 * Same device code as the engine path, exposed for the library-level API.
 * All arrays are host arrays of uint64 words indexed by variable (slot 0
 * unused), exactly the reference's numpy layout (bitpack.py:96-97). */
/* pack_assignments (bitpack.py:81-117): n rows of num_vars+1 int8 */
int tsg_pack(int32_t device, const int8_t* rows, int64_t n, int64_t row_pitch,
             int32_t num_vars, int32_t lane_width, uint64_t* is_true, uint64_t* is_set);
/* build_aggregate_batch (bitpack.py:211-244) from n_groups packed batches laid
 * out [n_groups][num_vars+1] */
int tsg_aggregate(int32_t device, const uint64_t* is_true, const uint64_t* is_set,
                  const int32_t* lane_counts, int32_t n_groups, int32_t num_vars,
                  int32_t group_width, uint64_t* cbt, uint64_t* cbf, uint64_t* cbu);
/* assignment_trigger (bitpack.py:120-135) for n clauses at once */
int tsg_lane_trigger(int32_t device, const uint64_t* is_true, const uint64_t* is_set,
                     int32_t num_vars, int32_t lane_width, uint64_t lane_mask,
                     const int32_t* lits, const int64_t* offsets, int64_t n,
                     uint64_t* masks);
/* aggregate_trigger (bitpack.py:247-271) for n clauses at once */
int tsg_aggregate_trigger(int32_t device, const uint64_t* cbt, const uint64_t* cbf,
                          const uint64_t* cbu, int32_t num_vars, int32_t group_width,
                          int32_t group_count, const int32_t* lits,
                          const int64_t* offsets, int64_t n, uint64_t* words);

#ifdef __cplusplus
}
#endif
#endif
