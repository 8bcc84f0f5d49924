/*
 * tsg_oracle.c -- CPU restatement of the triggersat filter (TEST INFRASTRUCTURE).
 *
 * See tsg_oracle.h.  Straight-line restatement of the reference algorithm:
 * no early exits, no filters, literals stored clause-major per size bucket.
 * Compile with -ffp-contract=off: activity bumps must round exactly like the
 * reference's `act += inc * hits` (engine.py:460).
 */
#include "tsg_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define WORD_BITS 64

static uint64_t width_mask(int32_t w) { return w >= 64 ? ~0ULL : ((1ULL << w) - 1ULL); }

/* bitpack.py:81-117 */
int ora_pack(const int8_t* values, int64_t n, int64_t pitch, int32_t num_vars,
             int32_t lane_width, uint64_t* is_true, uint64_t* is_set,
             uint64_t* lane_mask) {
    if (lane_width < 1 || lane_width > WORD_BITS) return -1; /* _check_width, :34-36 */
    if (n > lane_width) return -2;                           /* CapacityError, :92-95 */
    memset(is_true, 0, sizeof(uint64_t) * (size_t)(num_vars + 1));
    memset(is_set, 0, sizeof(uint64_t) * (size_t)(num_vars + 1));
    for (int64_t i = 0; i < n; ++i) {
        const int8_t* row = values + i * pitch;
        uint64_t bit = 1ULL << i;
        for (int32_t v = 0; v <= num_vars; ++v) {
            if (row[v] == 1) is_true[v] |= bit;  /* vals == TRUE  (:108) */
            if (row[v] != 0) is_set[v] |= bit;   /* vals != UNDEF (:109) */
        }
    }
    is_true[0] = 0;  /* :110-111 */
    is_set[0] = 0;
    if (lane_mask) *lane_mask = width_mask((int32_t)n);
    return 0;
}

/* AggregateAssignment.from_packed (bitpack.py:152-167) folded into
 * build_aggregate_batch (bitpack.py:211-244). */
/* variables [v_lo, v_hi) of the aggregate (the threads of ora_test_round
 * split the variables; the result does not depend on the split) */
static void aggregate_range(const uint64_t* is_true, const uint64_t* is_set, const int32_t* lane_counts,
                            int32_t n_groups, size_t nv, size_t v_lo, size_t v_hi,
                            uint64_t* cbt, uint64_t* cbf, uint64_t* cbu) {
    memset(cbt + v_lo, 0, sizeof(uint64_t) * (v_hi - v_lo));
    memset(cbf + v_lo, 0, sizeof(uint64_t) * (v_hi - v_lo));
    memset(cbu + v_lo, 0, sizeof(uint64_t) * (v_hi - v_lo));
    if (v_lo < 1) v_lo = 1; /* slot 0 stays False, :166 */
    for (int32_t g = 0; g < n_groups; ++g) {
        const uint64_t* t = is_true + (size_t)g * nv;
        const uint64_t* s = is_set + (size_t)g * nv;
        uint64_t bit = 1ULL << g;
        if (lane_counts[g] == 0) { /* empty group reads as all-Undef, :156-161 */
            for (size_t v = v_lo; v < v_hi; ++v) cbu[v] |= bit;
            continue;
        }
        uint64_t mask = width_mask(lane_counts[g]);
        for (size_t v = v_lo; v < v_hi; ++v) {
            if (t[v] != 0) cbt[v] |= bit;
            if ((s[v] & ~t[v]) != 0) cbf[v] |= bit;
            if ((~s[v] & mask) != 0) cbu[v] |= bit;
        }
    }
}

int ora_aggregate(const uint64_t* is_true, const uint64_t* is_set,
                  const int32_t* lane_counts, int32_t n_groups, int32_t num_vars,
                  int32_t group_width, uint64_t* cbt, uint64_t* cbf, uint64_t* cbu) {
    if (group_width < 1 || group_width > WORD_BITS) return -1;
    if (n_groups > group_width) return -2;
    size_t nv = (size_t)num_vars + 1;
    aggregate_range(is_true, is_set, lane_counts, n_groups, nv, 0, nv, cbt, cbf, cbu);
    return 0;
}

/* ora_test_round's table build, split over threads: thread w packs groups
 * w, w + nw, ... and then aggregates its share of the variables. */
typedef struct build_job {
    pthread_t th;
    int32_t w, nw, phase;
    const int8_t* snaps;
    const int64_t* row0;
    const int32_t* group_lanes;
    int64_t pitch;
    int32_t g0, ng, num_vars, lane_width;
    uint64_t *pt, *ps, *lm, *cb;
} build_job;

static void* run_build(void* arg) {
    build_job* j = (build_job*)arg;
    size_t nv = (size_t)j->num_vars + 1;
    if (j->phase == 0) {
        for (int32_t i = j->w; i < j->ng; i += j->nw)
            ora_pack(j->snaps + j->row0[j->g0 + i] * j->pitch, j->group_lanes[j->g0 + i], j->pitch, j->num_vars,
                     j->lane_width, j->pt + (size_t)i * nv, j->ps + (size_t)i * nv, &j->lm[i]);
    } else {
        size_t lo = nv * (size_t)j->w / (size_t)j->nw, hi = nv * (size_t)(j->w + 1) / (size_t)j->nw;
        aggregate_range(j->pt, j->ps, j->group_lanes + j->g0, j->ng, nv, lo, hi, j->cb, j->cb + nv, j->cb + 2 * nv);
    }
    return NULL;
}

/* bitpack.py:120-135 (literal_words :58-67) */
uint64_t ora_assignment_trigger(const uint64_t* is_true, const uint64_t* is_set,
                                int32_t lane_width, uint64_t lane_mask,
                                const int32_t* lits, int32_t n_lits) {
    uint64_t all_false = width_mask(lane_width);
    uint64_t one_undef = 0;
    for (int32_t j = 0; j < n_lits; ++j) {
        int32_t lit = lits[j];
        int32_t v = lit > 0 ? lit : -lit;
        uint64_t t = is_true[v], s = is_set[v];
        uint64_t is_false = lit > 0 ? (s & ~t) : (s & t);
        one_undef = (all_false & ~s) | (one_undef & is_false);
        all_false &= is_false;
    }
    return (all_false | one_undef) & lane_mask;
}

/* bitpack.py:247-271 */
uint64_t ora_aggregate_trigger(const uint64_t* cbt, const uint64_t* cbf,
                               const uint64_t* cbu, int32_t group_width,
                               int32_t group_count, const int32_t* lits,
                               int32_t n_lits) {
    if (group_count == 0) return 0;
    uint64_t all_false = width_mask(group_width);
    uint64_t one_undef = 0;
    for (int32_t j = 0; j < n_lits; ++j) {
        int32_t lit = lits[j];
        uint64_t f, u;
        if (lit > 0) { f = cbf[lit]; u = cbu[lit]; }
        else { f = cbt[-lit]; u = cbu[-lit]; }
        one_undef = (all_false & u) | (one_undef & f);
        all_false &= f;
    }
    return (all_false | one_undef) & width_mask(group_count);
}

/* ---------------------------------------------------------------------- */
/* store: one bucket per clause size, in creation order (engine.py:203-219) */

typedef struct bucket {
    int32_t size;
    int64_t count, cap;
    int32_t* lits; /* clause-major: slot k at lits[k*size] */
    int64_t* ids;
    int32_t* origins;
    double* acts;
} bucket;

struct ora_store {
    int32_t nb, capb;
    bucket* b;
};

ora_store* ora_store_new(void) { return (ora_store*)calloc(1, sizeof(ora_store)); }

void ora_store_free(ora_store* s) {
    if (!s) return;
    for (int32_t i = 0; i < s->nb; ++i) {
        free(s->b[i].lits); free(s->b[i].ids); free(s->b[i].origins); free(s->b[i].acts);
    }
    free(s->b);
    free(s);
}

void ora_free(void* p) { free(p); }

static bucket* find_or_make(ora_store* s, int32_t size) {
    for (int32_t i = 0; i < s->nb; ++i)
        if (s->b[i].size == size) return &s->b[i];
    if (s->nb == s->capb) {
        s->capb = s->capb ? 2 * s->capb : 16;
        s->b = (bucket*)realloc(s->b, sizeof(bucket) * (size_t)s->capb);
    }
    bucket* b = &s->b[s->nb++];
    memset(b, 0, sizeof(*b));
    b->size = size;
    return b;
}

void ora_store_insert(ora_store* s, const int32_t* lits, int32_t size,
                      int64_t engine_id, int32_t origin, double activity) {
    bucket* b = find_or_make(s, size);
    if (b->count == b->cap) {
        b->cap = b->cap ? 2 * b->cap : 128;
        b->lits = (int32_t*)realloc(b->lits, sizeof(int32_t) * (size_t)(b->cap * (size ? size : 1)));
        b->ids = (int64_t*)realloc(b->ids, sizeof(int64_t) * (size_t)b->cap);
        b->origins = (int32_t*)realloc(b->origins, sizeof(int32_t) * (size_t)b->cap);
        b->acts = (double*)realloc(b->acts, sizeof(double) * (size_t)b->cap);
    }
    if (size) memcpy(b->lits + b->count * size, lits, sizeof(int32_t) * (size_t)size);
    b->ids[b->count] = engine_id;
    b->origins[b->count] = origin;
    b->acts[b->count] = activity;
    b->count++;
}

void ora_store_insert_many(ora_store* s, const int32_t* lits, const int64_t* offsets,
                           int64_t n, const int64_t* ids, const int32_t* origins,
                           double activity) {
    for (int64_t i = 0; i < n; ++i)
        ora_store_insert(s, lits + offsets[i], (int32_t)(offsets[i + 1] - offsets[i]), ids[i],
                         origins ? origins[i] : 0, activity);
}

int64_t ora_store_size(const ora_store* s) {
    int64_t n = 0;
    for (int32_t i = 0; i < s->nb; ++i) n += s->b[i].count;
    return n;
}

int32_t ora_store_nbuckets(const ora_store* s) { return s->nb; }

void ora_store_bucket_info(const ora_store* s, int32_t b, int32_t* size, int64_t* count) {
    *size = s->b[b].size;
    *count = s->b[b].count;
}

void ora_store_bucket_read(const ora_store* s, int32_t bi, int32_t* lits,
                           int64_t* ids, int32_t* origins, double* acts) {
    const bucket* b = &s->b[bi];
    if (lits && b->size) memcpy(lits, b->lits, sizeof(int32_t) * (size_t)(b->count * b->size));
    if (ids) memcpy(ids, b->ids, sizeof(int64_t) * (size_t)b->count);
    if (origins) memcpy(origins, b->origins, sizeof(int32_t) * (size_t)b->count);
    if (acts) memcpy(acts, b->acts, sizeof(double) * (size_t)b->count);
}

void ora_store_scale(ora_store* s, double factor) {
    for (int32_t i = 0; i < s->nb; ++i)
        for (int64_t k = 0; k < s->b[i].count; ++k) s->b[i].acts[k] *= factor;
}

/* _SizeBucket.compact, engine.py:184-200: order-preserving */
static void compact(bucket* b, const unsigned char* keep) {
    int64_t w = 0;
    for (int64_t k = 0; k < b->count; ++k) {
        if (!keep[k]) continue;
        if (w != k) {
            if (b->size) memmove(b->lits + w * b->size, b->lits + k * b->size, sizeof(int32_t) * (size_t)b->size);
            b->ids[w] = b->ids[k];
            b->origins[w] = b->origins[k];
            b->acts[w] = b->acts[k];
        }
        ++w;
    }
    b->count = w;
}

typedef struct cand { double act; int64_t id; int32_t b; int64_t slot; } cand;

static int cand_cmp(const void* x, const void* y) {
    const cand* a = (const cand*)x;
    const cand* c = (const cand*)y;
    /* candidates.sort() on (act, id, size, slot), engine.py:488; ids are unique */
    if (a->act < c->act) return -1;
    if (a->act > c->act) return 1;
    return (a->id > c->id) - (a->id < c->id);
}

int64_t ora_store_reduce(ora_store* s, int64_t eligible_below, int64_t target,
                         int64_t* removed_ids) {
    int64_t total = ora_store_size(s);
    cand* cs = (cand*)malloc(sizeof(cand) * (size_t)(total ? total : 1));
    int64_t nc = 0;
    for (int32_t i = 0; i < s->nb; ++i) /* eligible = ids < watermark, :486 */
        for (int64_t k = 0; k < s->b[i].count; ++k)
            if (s->b[i].ids[k] < eligible_below)
                cs[nc++] = (cand){s->b[i].acts[k], s->b[i].ids[k], i, k};
    qsort(cs, (size_t)nc, sizeof(cand), cand_cmp);
    int64_t removed = target < nc ? target : nc; /* doomed = candidates[:target] */
    if (removed < 0) removed = 0;
    unsigned char** keep = (unsigned char**)calloc((size_t)(s->nb ? s->nb : 1), sizeof(unsigned char*));
    for (int64_t r = 0; r < removed; ++r) {
        int32_t bi = cs[r].b;
        if (!keep[bi]) {
            keep[bi] = (unsigned char*)malloc((size_t)(s->b[bi].count ? s->b[bi].count : 1));
            memset(keep[bi], 1, (size_t)s->b[bi].count);
        }
        keep[bi][cs[r].slot] = 0;
        if (removed_ids) removed_ids[r] = cs[r].id;
    }
    for (int32_t i = 0; i < s->nb; ++i)
        if (keep[i]) { compact(&s->b[i], keep[i]); free(keep[i]); }
    free(keep);
    free(cs);
    return removed;
}

static int i64cmp(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    return (a > b) - (a < b);
}

int64_t ora_store_remove(ora_store* s, const int64_t* ids, int64_t n) {
    int64_t* sorted = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    memcpy(sorted, ids, sizeof(int64_t) * (size_t)n);
    qsort(sorted, (size_t)n, sizeof(int64_t), i64cmp);
    int64_t removed = 0;
    for (int32_t i = 0; i < s->nb; ++i) {
        bucket* b = &s->b[i];
        unsigned char* keep = (unsigned char*)malloc((size_t)(b->count ? b->count : 1));
        int64_t gone = 0;
        for (int64_t k = 0; k < b->count; ++k) {
            keep[k] = bsearch(&b->ids[k], sorted, (size_t)n, sizeof(int64_t), i64cmp) == NULL;
            gone += !keep[k];
        }
        if (gone) compact(b, keep);
        removed += gone;
        free(keep);
    }
    free(sorted);
    return removed;
}

/* ---------------------------------------------------------------------- */
/* round test phase: engine.py:386-467 */

typedef struct pairset { /* open addressing set of (engine_id, tid), the `reported` set (:401) */
    int64_t* eid;
    int32_t* tid;
    unsigned char* used;
    size_t cap, n;
} pairset;

static size_t ph(int64_t e, int32_t t, size_t cap) {
    uint64_t x = (uint64_t)e * 0x9E3779B97F4A7C15ULL ^ ((uint64_t)(uint32_t)t * 0xC2B2AE3D27D4EB4FULL);
    x ^= x >> 29;
    return (size_t)(x & (cap - 1));
}

static int pairset_add(pairset* p, int64_t e, int32_t t); /* 1 if newly added */

static void pairset_grow(pairset* p) {
    pairset q = {0};
    q.cap = p->cap ? p->cap * 2 : 1024;
    q.eid = (int64_t*)malloc(sizeof(int64_t) * q.cap);
    q.tid = (int32_t*)malloc(sizeof(int32_t) * q.cap);
    q.used = (unsigned char*)calloc(q.cap, 1);
    for (size_t i = 0; i < p->cap; ++i)
        if (p->used[i]) pairset_add(&q, p->eid[i], p->tid[i]);
    free(p->eid); free(p->tid); free(p->used);
    *p = q;
}

static int pairset_add(pairset* p, int64_t e, int32_t t) {
    if (2 * (p->n + 1) > p->cap) pairset_grow(p);
    size_t i = ph(e, t, p->cap);
    while (p->used[i]) {
        if (p->eid[i] == e && p->tid[i] == t) return 0;
        i = (i + 1) & (p->cap - 1);
    }
    p->used[i] = 1; p->eid[i] = e; p->tid[i] = t; p->n++;
    return 1;
}

typedef struct chunk_ctx {
    ora_store* s;
    int32_t num_vars, lane_width, group_width, g0, ng;
    const uint64_t *pt, *ps, *lm; /* per-group packed words + lane masks */
    const uint64_t *cbt, *cbf, *cbu;
    const int32_t* group_tid;
    double inc;
} chunk_ctx;

typedef struct worker {
    const chunk_ctx* c;
    int32_t w, nw;
    pairset* reported;
    ora_report* rep;
    int64_t nrep, caprep;
    int64_t positives, lane_triggers;
    pthread_t th;
} worker;

static void emit(worker* w, int64_t eid, uint64_t mask, int32_t group, int32_t b, int64_t slot) {
    if (w->nrep == w->caprep) {
        w->caprep = w->caprep ? 2 * w->caprep : 1024;
        w->rep = (ora_report*)realloc(w->rep, sizeof(ora_report) * (size_t)w->caprep);
    }
    w->rep[w->nrep++] = (ora_report){eid, mask, group, b, slot};
}

static void* run_worker(void* arg) {
    worker* w = (worker*)arg;
    const chunk_ctx* c = w->c;
    size_t nv = (size_t)c->num_vars + 1;
    for (int32_t bi = 0; bi < c->s->nb; ++bi) { /* dict insertion order, :449 */
        bucket* b = &c->s->b[bi];
        int64_t lo = b->count * w->w / w->nw, hi = b->count * (w->w + 1) / w->nw;
        for (int64_t k = lo; k < hi; ++k) {
            const int32_t* lits = b->lits + k * b->size;
            uint64_t word = ora_aggregate_trigger(c->cbt, c->cbf, c->cbu, c->group_width,
                                                  c->ng, lits, b->size);
            w->positives += __builtin_popcountll(word);
            for (int32_t i = 0; i < c->ng; ++i) { /* iter_set_bits ascending, :457 */
                if (!((word >> i) & 1)) continue;
                uint64_t mask = ora_assignment_trigger(c->pt + (size_t)i * nv, c->ps + (size_t)i * nv,
                                                       c->lane_width, c->lm[i], lits, b->size);
                if (!mask) continue;
                int32_t hits = __builtin_popcountll(mask);
                b->acts[k] += c->inc * (double)hits; /* :460 */
                w->lane_triggers += hits;
                int32_t tid = c->group_tid[c->g0 + i];
                if (pairset_add(w->reported, b->ids[k], tid))
                    emit(w, b->ids[k], mask, c->g0 + i, bi, k);
            }
        }
    }
    return NULL;
}

typedef struct ordkey { ora_report r; int32_t chunk; } ordkey;

static int32_t g_group_width_for_sort;

static int rep_cmp(const void* x, const void* y) {
    const ora_report* a = (const ora_report*)x;
    const ora_report* b = (const ora_report*)y;
    int32_t ca = a->group / g_group_width_for_sort, cb = b->group / g_group_width_for_sort;
    if (ca != cb) return ca < cb ? -1 : 1;
    if (a->bucket != b->bucket) return a->bucket < b->bucket ? -1 : 1;
    if (a->slot != b->slot) return a->slot < b->slot ? -1 : 1;
    return (a->group > b->group) - (a->group < b->group);
}

int ora_test_round(ora_store* s, int32_t num_vars, const int8_t* snaps,
                   int64_t pitch, const int32_t* group_lanes,
                   const int32_t* group_tid, int32_t n_groups,
                   int32_t lane_width, int32_t group_width, double activity_inc,
                   int32_t nthreads, ora_report** out, int64_t* n_out,
                   ora_counters* counters) {
    memset(counters, 0, sizeof(*counters));
    *out = NULL;
    *n_out = 0;
    if (lane_width < 1 || lane_width > 64 || group_width < 1 || group_width > 64) return -1;
    if (nthreads < 1) nthreads = 1;
    size_t nv = (size_t)num_vars + 1;
    int64_t* row0 = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_groups + 1));
    row0[0] = 0;
    for (int32_t g = 0; g < n_groups; ++g) {
        if (group_lanes[g] > lane_width) { free(row0); return -2; }
        row0[g + 1] = row0[g] + group_lanes[g];
    }
    worker* ws = (worker*)calloc((size_t)nthreads, sizeof(worker));
    pairset* sets = (pairset*)calloc((size_t)nthreads, sizeof(pairset));
    uint64_t* pt = (uint64_t*)malloc(sizeof(uint64_t) * nv * (size_t)group_width);
    uint64_t* ps = (uint64_t*)malloc(sizeof(uint64_t) * nv * (size_t)group_width);
    uint64_t* cb = (uint64_t*)malloc(sizeof(uint64_t) * nv * 3);
    uint64_t lm[64];
    int64_t store_count = ora_store_size(s);
    for (int32_t g0 = 0; g0 < n_groups; g0 += group_width) { /* :403-407 */
        int32_t ng = n_groups - g0 < group_width ? n_groups - g0 : group_width;
        int32_t lanes_total = 0;
        for (int32_t i = 0; i < ng; ++i) lanes_total += group_lanes[g0 + i];
        /* pack the chunk's groups, then aggregate (bitpack.py:81-117, 152-167, 211-244) */
        for (int32_t phase = 0; phase < 2; ++phase) {
            build_job* jobs = (build_job*)calloc((size_t)nthreads, sizeof(build_job));
            for (int32_t t = 0; t < nthreads; ++t) {
                build_job jb = {0, t, nthreads, phase, snaps, row0, group_lanes, pitch, g0, ng, num_vars,
                                lane_width, pt, ps, lm, cb};
                jobs[t] = jb;
                if (nthreads > 1) pthread_create(&jobs[t].th, NULL, run_build, &jobs[t]);
                else run_build(&jobs[t]);
            }
            if (nthreads > 1)
                for (int32_t t = 0; t < nthreads; ++t) pthread_join(jobs[t].th, NULL);
            free(jobs);
        }
        chunk_ctx c = {s, num_vars, lane_width, group_width, g0, ng, pt, ps, lm,
                       cb, cb + nv, cb + 2 * nv, group_tid, activity_inc};
        int64_t positives = 0;
        for (int32_t t = 0; t < nthreads; ++t) {
            ws[t].c = &c; ws[t].w = t; ws[t].nw = nthreads; ws[t].reported = &sets[t];
            ws[t].positives = 0;
            if (nthreads > 1) pthread_create(&ws[t].th, NULL, run_worker, &ws[t]);
            else run_worker(&ws[t]);
        }
        for (int32_t t = 0; t < nthreads; ++t) {
            if (nthreads > 1) pthread_join(ws[t].th, NULL);
            positives += ws[t].positives;
        }
        counters->clauses_tested += store_count;              /* :445 */
        counters->aggregate_tests += store_count * ng;        /* :446 */
        counters->lane_tests += store_count * lanes_total;    /* :447 */
        counters->aggregate_tests_negative += store_count * ng - positives; /* :465 */
    }
    int64_t total = 0;
    for (int32_t t = 0; t < nthreads; ++t) {
        total += ws[t].nrep;
        counters->lane_triggers += ws[t].lane_triggers;
    }
    ora_report* all = (ora_report*)malloc(sizeof(ora_report) * (size_t)(total ? total : 1));
    int64_t o = 0;
    for (int32_t t = 0; t < nthreads; ++t) {
        if (ws[t].nrep) memcpy(all + o, ws[t].rep, sizeof(ora_report) * (size_t)ws[t].nrep);
        o += ws[t].nrep;
        free(ws[t].rep);
        free(sets[t].eid); free(sets[t].tid); free(sets[t].used);
    }
    g_group_width_for_sort = group_width;
    if (nthreads > 1) qsort(all, (size_t)total, sizeof(ora_report), rep_cmp);
    counters->reports = total;
    *out = all;
    *n_out = total;
    free(ws); free(sets); free(pt); free(ps); free(cb); free(row0);
    return 0;
}
