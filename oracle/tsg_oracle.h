/*
 * tsg_oracle.h -- CPU restatement of the triggersat clause-usefulness filter.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA product
 * (paper_2012_03119_b200/csrc).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it.  Nothing in the
 * product path links or calls it.
 *
 * Each function names the reference file:line it restates
 * (/root/reference/pkg/src/triggersat/...).  The restatement is pinned against
 * golden vectors produced by running the reference itself
 * (tests/golden/make_golden.py -> tests/golden/ fixtures).
 *
 * Words are uint64 regardless of the configured width, exactly as the
 * reference keeps numpy uint64 words (bitpack.py:96-97).
 */
#ifndef TSG_ORACLE_H
#define TSG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* bitpack.py:81-117 pack_assignments.  values: n rows of pitch bytes, slot v of
 * row i at values[i*pitch+v], v in 0..num_vars.  Returns 0, or -1 on a width error. */
int ora_pack(const int8_t* values, int64_t n, int64_t pitch, int32_t num_vars,
             int32_t lane_width, uint64_t* is_true, uint64_t* is_set,
             uint64_t* lane_mask);

/* bitpack.py:152-167 + 211-244: aggregate G packed groups into can_be_* words.
 * is_true/is_set: G arrays of num_vars+1 words, group g at offset g*(num_vars+1). */
int ora_aggregate(const uint64_t* is_true, const uint64_t* is_set,
                  const int32_t* lane_counts, int32_t n_groups, int32_t num_vars,
                  int32_t group_width, uint64_t* cbt, uint64_t* cbf, uint64_t* cbu);

/* bitpack.py:120-135 assignment_trigger. */
uint64_t ora_assignment_trigger(const uint64_t* is_true, const uint64_t* is_set,
                                int32_t lane_width, uint64_t lane_mask,
                                const int32_t* lits, int32_t n_lits);

/* bitpack.py:247-271 aggregate_trigger. */
uint64_t ora_aggregate_trigger(const uint64_t* cbt, const uint64_t* cbf,
                               const uint64_t* cbu, int32_t group_width,
                               int32_t group_count, const int32_t* lits,
                               int32_t n_lits);

/* ---- engine-level restatement (engine.py:122-235, 369-505) ------------- */

typedef struct ora_store ora_store;

typedef struct ora_report {
    int64_t engine_id;
    uint64_t lane_mask;
    int32_t group;      /* global group index in round order (engine.py:390-399) */
    int32_t bucket;     /* bucket creation rank (dict insertion order) */
    int64_t slot;
} ora_report;

typedef struct ora_counters {
    int64_t clauses_tested;           /* engine.py:445, once per chunk */
    int64_t aggregate_tests;          /* engine.py:446 */
    int64_t aggregate_tests_negative; /* engine.py:465-467 */
    int64_t lane_tests;               /* engine.py:447 */
    int64_t lane_triggers;            /* engine.py:461 */
    int64_t reports;                  /* engine.py:462-464 */
} ora_counters;

ora_store* ora_store_new(void);
void ora_store_free(ora_store* s);
/* ClauseStore.insert / _SizeBucket.insert, engine.py:150-163, 213-219 */
void ora_store_insert(ora_store* s, const int32_t* lits, int32_t size,
                      int64_t engine_id, int32_t origin, double activity);
/* bulk form: clause i = lits[offsets[i]..offsets[i+1]) */
void ora_store_insert_many(ora_store* s, const int32_t* lits, const int64_t* offsets,
                           int64_t n, const int64_t* ids, const int32_t* origins,
                           double activity);
int64_t ora_store_size(const ora_store* s);
int32_t ora_store_nbuckets(const ora_store* s);
/* bucket b in creation order: size and count */
void ora_store_bucket_info(const ora_store* s, int32_t b, int32_t* size, int64_t* count);
/* copy bucket b: lits clause-major (count*size), ids, origins, activities; any may be NULL */
void ora_store_bucket_read(const ora_store* s, int32_t b, int32_t* lits,
                           int64_t* ids, int32_t* origins, double* acts);
/* ClauseStore.scale_activities, engine.py:233-235 */
void ora_store_scale(ora_store* s, double factor);
/* reduce_store selection+compaction, engine.py:482-500: remove the `target`
 * smallest (activity, engine_id) among ids < eligible_below.  Returns removed
 * count; removed ids written in removal (sorted) order if out != NULL. */
int64_t ora_store_reduce(ora_store* s, int64_t eligible_below, int64_t target,
                         int64_t* removed_ids);
/* explicit delete by id, order-preserving (the compact(keep) of engine.py:184-200) */
int64_t ora_store_remove(ora_store* s, const int64_t* ids, int64_t n);

/* One round's test phase, engine.py:386-467: snapshots already grouped in
 * round order (rows of `pitch` bytes), group g has group_lanes[g] rows and
 * belongs to thread group_tid[g].  Chunks of group_width groups are tested
 * against every bucket in creation order; reports are emitted in the
 * reference's order (chunk, bucket, slot, group) with (engine_id, tid) dedup
 * across the whole round.  Activities are bumped in place.  nthreads>1 splits
 * every bucket's slots across pthreads (results identical).
 * *out is malloc'd; free with ora_free. */
int ora_test_round(ora_store* s, int32_t num_vars, const int8_t* snaps,
                   int64_t pitch, const int32_t* group_lanes,
                   const int32_t* group_tid, int32_t n_groups,
                   int32_t lane_width, int32_t group_width, double activity_inc,
                   int32_t nthreads, ora_report** out, int64_t* n_out,
                   ora_counters* counters);
void ora_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
