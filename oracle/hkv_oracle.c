/*
 * hkv_oracle.c — CPU restatement of the reference `cachekv.CacheTable` engine.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernels in paper_2603_17168_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * path never links or calls it.
 *
 * Parity pinned: tests/test_oracle_reference.py runs this oracle against the
 * reference package itself (differential, all modes x policies x ops), and
 * tests/test_oracle_golden.py against the committed fixtures in tests/golden/
 * that tests/golden/make_golden.py generated from the reference.
 *
 * Semantics (every function cites the reference file:line it restates; paths
 * are relative to /root/reference/pkg/src/cachekv/):
 *   The reference's vectorised engine (workers=1) equals applying each batch
 *   op one at a time in ascending batch index.  This
 *   oracle is written in exactly that serial form.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define SLOTS 128
#define EMPTY_KEY 0xFFFFFFFFFFFFFFFFull
#define LOCKED_KEY 0xFFFFFFFFFFFFFFFEull
#define MAX_SCORE 0xFFFFFFFFFFFFFFFFull
#define LOW32 0xFFFFFFFFull

enum { POL_LRU = 0, POL_LFU = 1, POL_EPOCH_LRU = 2, POL_EPOCH_LFU = 3, POL_CUSTOM = 4 };
enum { O_INSERTED = 0, O_UPDATED = 1, O_REJECTED = 2, O_EVICTED = 3, O_FOUND = 4,
       O_NOTFOUND = 5, O_ERASED = 6 };
enum { OP_UPSERT = 0, OP_FIND_OR_INSERT = 1 };
/* TxnCounters field order (metrics.py:14-20) */
enum { C_LOADS = 0, C_COMPARES = 1, C_SCANS = 2, C_RETRIES = 3, C_VFAST = 4, C_VOVER = 5 };

typedef struct {
    int64_t capacity, dim, buckets, budget;
    int32_t dual, policy, digest_filter, admit_ties_unified;
    uint64_t *keys;     /* [buckets][128] */
    uint8_t *digests;   /* [buckets][128] */
    uint64_t *scores;   /* [buckets][128] */
    int64_t *occ;       /* [buckets] */
    float *values;      /* [capacity][dim], fast rows then overflow rows */
    int64_t size;
    uint64_t clock;
    uint64_t epoch;
    int32_t fel_set;
    double fel;          /* first_eviction_lambda */
    int64_t ctr[6];
} ot_table;

/* hashing.py:21-29 (fmix64), :52-57 (second hash), :60-66 (digest bits 32..39) */
static inline uint64_t fmix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xFF51AFD7ED558CCDull;
    x ^= x >> 33;
    x *= 0xC4CEB9FE1A85EC53ull;
    x ^= x >> 33;
    return x;
}
static inline uint64_t second_hash(uint64_t h1) { return fmix64(h1 ^ 0x9E3779B97F4A7C15ull); }
static inline uint8_t digest_of(uint64_t h) { return (uint8_t)((h >> 32) & 0xFF); }

uint64_t ot_fmix64(uint64_t x) { return fmix64(x); }

ot_table *ot_create(int64_t capacity, int64_t dim, int32_t dual, int32_t policy, int64_t budget,
                    int32_t digest_filter, int32_t admit_ties_unified) {
    /* table.py:139-160, store.py:41-63 */
    ot_table *t = (ot_table *)calloc(1, sizeof(ot_table));
    if (!t) return NULL;
    t->capacity = capacity;
    t->dim = dim;
    t->buckets = capacity / SLOTS;
    t->budget = budget;
    t->dual = dual;
    t->policy = policy;
    t->digest_filter = digest_filter;
    t->admit_ties_unified = admit_ties_unified;
    t->keys = (uint64_t *)malloc(sizeof(uint64_t) * capacity);
    t->digests = (uint8_t *)calloc(capacity, 1);
    t->scores = (uint64_t *)calloc(capacity, sizeof(uint64_t));
    t->occ = (int64_t *)calloc(t->buckets, sizeof(int64_t));
    t->values = (float *)calloc((size_t)capacity * dim, sizeof(float));
    if (!t->keys || !t->digests || !t->scores || !t->occ || !t->values) return NULL;
    memset(t->keys, 0xFF, sizeof(uint64_t) * capacity);
    return t;
}

void ot_destroy(ot_table *t) {
    if (!t) return;
    free(t->keys); free(t->digests); free(t->scores); free(t->occ); free(t->values);
    free(t);
}

ot_table *ot_clone(const ot_table *s) {
    ot_table *t = ot_create(s->capacity, s->dim, s->dual, s->policy, s->budget, s->digest_filter,
                            s->admit_ties_unified);
    if (!t) return NULL;
    memcpy(t->keys, s->keys, sizeof(uint64_t) * s->capacity);
    memcpy(t->digests, s->digests, s->capacity);
    memcpy(t->scores, s->scores, sizeof(uint64_t) * s->capacity);
    memcpy(t->occ, s->occ, sizeof(int64_t) * s->buckets);
    memcpy(t->values, s->values, sizeof(float) * s->capacity * s->dim);
    t->size = s->size; t->clock = s->clock; t->epoch = s->epoch;
    t->fel_set = s->fel_set; t->fel = s->fel;
    memcpy(t->ctr, s->ctr, sizeof(t->ctr));
    return t;
}

static inline void count_row(ot_table *t, int64_t row, int64_t *ctr) {
    /* store.py:133-136 via table.py:217-220 */
    if (row >= t->budget * SLOTS) ctr[C_VOVER]++; else ctr[C_VFAST]++;
}

/* table.py:633-647 (_scalar_probe) == table.py:224-272 (_probe_rows) per query:
 * candidates are digest-equal slots whose key is not EMPTY, compared in slot
 * order; compares stop at the match. */
static int probe(ot_table *t, int64_t b, uint64_t key, uint8_t d, int64_t *ctr) {
    ctr[C_LOADS]++;
    const uint8_t *dl = t->digests + b * SLOTS;
    const uint64_t *kr = t->keys + b * SLOTS;
    for (int s = 0; s < SLOTS; s++) {
        if (t->digest_filter && dl[s] != d) continue;
        if (kr[s] == EMPTY_KEY) continue;
        ctr[C_COMPARES]++;
        if (kr[s] == key) return s;
    }
    return -1;
}

/* table.py:284-300 (_vec_lookup): probe b1, then b2 for b1-misses (dual). */
static int64_t lookup_row(ot_table *t, uint64_t key, int64_t *ctr) {
    uint64_t h = fmix64(key);
    uint8_t d = digest_of(h);
    int64_t mask = t->buckets - 1;
    int64_t b = (int64_t)(h & (uint64_t)mask);
    int s = probe(t, b, key, d, ctr);
    if (s < 0 && t->dual) {
        b = (int64_t)(second_hash(h) & (uint64_t)mask);
        s = probe(t, b, key, d, ctr);
    }
    return s < 0 ? -1 : b * SLOTS + s;
}

/* table.py:304-323 (find) + store.py:115-123 (gather_rows).  Misses leave
 * out rows untouched. */
void ot_find(ot_table *t, const uint64_t *keys, int64_t n, float *out, uint8_t *found) {
    int64_t ctr[6] = {0};
    for (int64_t i = 0; i < n; i++) {
        int64_t row = lookup_row(t, keys[i], ctr);
        found[i] = row >= 0;
        if (row >= 0) {
            if (out) memcpy(out + i * t->dim, t->values + row * t->dim, sizeof(float) * t->dim);
            count_row(t, row, ctr);
        }
    }
    for (int c = 0; c < 6; c++) t->ctr[c] += ctr[c];
}

/* Multi-threaded find for the CPU baseline leg (pure reads; counters merged).
 * pthreads, contiguous ranges, like the reference's reader split
 * (table.py:353-372). */
typedef struct {
    ot_table *t;
    const uint64_t *keys;
    float *out;
    uint8_t *found;
    int64_t lo, hi;
    int64_t ctr[6];
} find_job;

static void *find_worker(void *arg) {
    find_job *j = (find_job *)arg;
    ot_table *t = j->t;
    int64_t ctr[6] = {0}; /* thread-local: no false sharing between jobs */
    for (int64_t i = j->lo; i < j->hi; i++) {
        int64_t row = lookup_row(t, j->keys[i], ctr);
        j->found[i] = row >= 0;
        if (row >= 0) {
            if (j->out) memcpy(j->out + i * t->dim, t->values + row * t->dim, sizeof(float) * t->dim);
            count_row(t, row, ctr);
        }
    }
    memcpy(j->ctr, ctr, sizeof(ctr));
    return NULL;
}

void ot_find_mt(ot_table *t, const uint64_t *keys, int64_t n, float *out, uint8_t *found,
                int32_t threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    find_job jobs[256];
    pthread_t tids[256];
    for (int w = 0; w < threads; w++) {
        memset(&jobs[w], 0, sizeof(find_job));
        jobs[w].t = t; jobs[w].keys = keys; jobs[w].out = out; jobs[w].found = found;
        jobs[w].lo = n * w / threads;
        jobs[w].hi = n * (w + 1) / threads;
        pthread_create(&tids[w], NULL, find_worker, &jobs[w]);
    }
    for (int w = 0; w < threads; w++) {
        pthread_join(tids[w], NULL);
        for (int c = 0; c < 6; c++) t->ctr[c] += jobs[w].ctr[c];
    }
}

/* table.py:344-351 (contains) */
void ot_contains(ot_table *t, const uint64_t *keys, int64_t n, uint8_t *found) {
    int64_t ctr[6] = {0};
    for (int64_t i = 0; i < n; i++) found[i] = lookup_row(t, keys[i], ctr) >= 0;
    for (int c = 0; c < 6; c++) t->ctr[c] += ctr[c];
}

/* table.py:325-342 (find_ptr): tier = row >= budget*128, offset in the tier arena */
void ot_find_ptr(ot_table *t, const uint64_t *keys, int64_t n, uint8_t *found, uint8_t *tier,
                 int64_t *offset) {
    int64_t ctr[6] = {0};
    int64_t base = t->budget * SLOTS;
    for (int64_t i = 0; i < n; i++) {
        int64_t row = lookup_row(t, keys[i], ctr);
        found[i] = row >= 0;
        tier[i] = 0;
        offset[i] = -1;
        if (row >= 0) {
            tier[i] = row >= base;
            offset[i] = row < base ? row * t->dim : (row - base) * t->dim;
        }
    }
    for (int c = 0; c < 6; c++) t->ctr[c] += ctr[c];
}

/* scoring.py:56-76 (score_on_insert) */
static inline uint64_t insert_score(int policy, uint64_t epoch, uint64_t tick, uint64_t custom) {
    switch (policy) {
    case POL_LRU: return tick;
    case POL_LFU: return 1;
    case POL_EPOCH_LRU: return (epoch << 32) | (tick & LOW32);
    case POL_EPOCH_LFU: return (epoch << 32) | 1;
    default: return custom;
    }
}

/* scoring.py:79-102 (score_on_hit) */
static inline uint64_t hit_score(int policy, uint64_t old, uint64_t epoch, uint64_t tick,
                                 int has_custom, uint64_t custom) {
    switch (policy) {
    case POL_LRU: return tick;
    case POL_LFU: return old == MAX_SCORE ? old : old + 1;
    case POL_EPOCH_LRU: return (epoch << 32) | (tick & LOW32);
    case POL_EPOCH_LFU: {
        if ((old >> 32) == epoch) {
            uint64_t low = old & LOW32;
            if (low < LOW32) low++;
            return (epoch << 32) | low;
        }
        return (epoch << 32) | 1;
    }
    default: return has_custom ? custom : old;
    }
}

static inline int lowest_empty(const ot_table *t, int64_t b) {
    /* table.py:1171 argmax(keys == EMPTY) */
    const uint64_t *kr = t->keys + b * SLOTS;
    for (int s = 0; s < SLOTS; s++)
        if (kr[s] == EMPTY_KEY) return s;
    return -1;
}

static inline int argmin_score(const ot_table *t, int64_t b, uint64_t *minv) {
    /* table.py:1080 np.argmin (first index on ties) */
    const uint64_t *sr = t->scores + b * SLOTS;
    int m = 0;
    uint64_t v = sr[0];
    for (int s = 1; s < SLOTS; s++)
        if (sr[s] < v) { v = sr[s]; m = s; }
    *minv = v;
    return m;
}

static inline void publish(ot_table *t, int64_t b, int s, uint64_t key, uint8_t d, uint64_t score,
                           const float *val, int64_t *ctr) {
    /* table.py:1157-1162 / 1172-1178 */
    int64_t row = b * SLOTS + s;
    t->keys[row] = key;
    t->digests[row] = d;
    t->scores[row] = score;
    memcpy(t->values + row * t->dim, val, sizeof(float) * t->dim);
    count_row(t, row, ctr);
}

/*
 * table.py:515-551 (insert_or_assign / insert_and_evict / find_or_insert)
 *   -> _mutate 934-943 -> _vec_mutate 964-1004 -> _round_upsert 1025-1119,
 *      _finish_admission 1121-1163, _bulk_insert_free 1165-1181,
 * restated serially (App. A.8).  `values` is values_inout for find_or_insert.
 * ticks: NULL -> clock+i+1 and clock += n (table.py:192-196, 937); otherwise
 * the caller supplies per-op ticks and clock_advance (sharded global order).
 * Evicted tuples are written in batch order (table.py:994-1003).
 */
int64_t ot_upsert(ot_table *t, int32_t op, const uint64_t *keys, float *values,
                  const uint64_t *scores, int64_t n, uint8_t *outcomes, uint64_t *ek, float *ev,
                  uint64_t *es, const uint64_t *ticks, uint64_t clock_advance) {
    int64_t ctr[6] = {0};
    uint64_t clock0 = t->clock;
    t->clock += ticks ? clock_advance : (uint64_t)n;
    int64_t size_before = t->size;
    int64_t mask = t->buckets - 1;
    int64_t n_ev = 0, first_ev = -1, inserted_before_first = 0;
    uint64_t epoch = t->epoch;
    int custom = t->policy == POL_CUSTOM;
    for (int64_t i = 0; i < n; i++) {
        uint64_t key = keys[i];
        uint64_t tick = ticks ? ticks[i] : clock0 + (uint64_t)i + 1;
        uint64_t sc = scores ? scores[i] : 0;
        float *val = values + i * t->dim;
        uint64_t h = fmix64(key);
        uint8_t d = digest_of(h);
        int64_t b1 = (int64_t)(h & (uint64_t)mask);
        int64_t b2 = t->dual ? (int64_t)(second_hash(h) & (uint64_t)mask) : -1;
        int64_t hb = b1;
        int s = probe(t, b1, key, d, ctr);
        if (s < 0 && t->dual) { hb = b2; s = probe(t, b2, key, d, ctr); }
        if (s >= 0) {
            /* hit: table.py:1045-1062 */
            int64_t row = hb * SLOTS + s;
            t->scores[row] = hit_score(t->policy, t->scores[row], epoch, tick, custom && scores, sc);
            if (op == OP_FIND_OR_INSERT) {
                memcpy(val, t->values + row * t->dim, sizeof(float) * t->dim);
                outcomes[i] = O_FOUND;
            } else {
                memcpy(t->values + row * t->dim, val, sizeof(float) * t->dim);
                outcomes[i] = O_UPDATED;
            }
            count_row(t, row, ctr);
            continue;
        }
        uint64_t s_in = insert_score(t->policy, epoch, tick, sc);
        int64_t tb;
        int m;
        uint64_t minv;
        int admit;
        if (!t->dual) {
            if (t->occ[b1] < SLOTS) {
                int f = lowest_empty(t, b1);
                publish(t, b1, f, key, d, s_in, val, ctr);
                t->occ[b1]++; t->size++;
                outcomes[i] = O_INSERTED;
                if (first_ev < 0) inserted_before_first++;
                continue;
            }
            m = argmin_score(t, b1, &minv);
            ctr[C_SCANS]++;
            tb = b1;
            admit = s_in >= minv; /* table.py:1083 ties admitted */
        } else {
            int64_t o1 = t->occ[b1], o2 = t->occ[b2];
            if (o1 < SLOTS || o2 < SLOTS) {
                /* D1, table.py:1089-1095 */
                tb = o1 <= o2 ? b1 : b2;
                int f = lowest_empty(t, tb);
                publish(t, tb, f, key, d, s_in, val, ctr);
                t->occ[tb]++; t->size++;
                outcomes[i] = O_INSERTED;
                if (first_ev < 0) inserted_before_first++;
                continue;
            }
            /* D2, table.py:1096-1119 */
            uint64_t min1, min2;
            int m1 = argmin_score(t, b1, &min1);
            int m2 = argmin_score(t, b2, &min2);
            ctr[C_SCANS] += 2;
            int use2 = min2 < min1;
            tb = use2 ? b2 : b1;
            m = use2 ? m2 : m1;
            minv = min1 < min2 ? min1 : min2;
            admit = t->admit_ties_unified ? s_in >= minv : s_in > minv;
        }
        if (!admit) { outcomes[i] = O_REJECTED; continue; }
        /* _finish_admission, table.py:1138-1163 */
        int64_t row = tb * SLOTS + m;
        if (ek) {
            ek[n_ev] = t->keys[row];
            es[n_ev] = minv;
            memcpy(ev + n_ev * t->dim, t->values + row * t->dim, sizeof(float) * t->dim);
            count_row(t, row, ctr);
        }
        n_ev++;
        if (first_ev < 0) first_ev = i;
        publish(t, tb, m, key, d, s_in, val, ctr);
        outcomes[i] = O_EVICTED;
    }
    /* table.py:986-991 */
    if (!t->fel_set && first_ev >= 0) {
        t->fel_set = 1;
        t->fel = (double)(size_before + inserted_before_first) / (double)t->capacity;
    }
    for (int c = 0; c < 6; c++) t->ctr[c] += ctr[c];
    return n_ev;
}

/* table.py:438-442, 451-506 (assign / assign_scores, vectorised path
 * restated serially: last duplicate wins; refresh ticks are taken per found
 * key in found order, table.py:481-483). values and scores may be NULL;
 * refresh != 0 requests the policy refresh. */
void ot_assign(ot_table *t, const uint64_t *keys, const float *values, const uint64_t *scores,
               int32_t refresh, int64_t n, uint8_t *outcomes, const uint64_t *ticks,
               uint64_t clock_advance) {
    int64_t ctr[6] = {0};
    int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    int64_t nfound = 0;
    for (int64_t i = 0; i < n; i++) {
        rows[i] = lookup_row(t, keys[i], ctr);
        outcomes[i] = rows[i] >= 0 ? O_UPDATED : O_NOTFOUND;
        if (rows[i] >= 0) nfound++;
    }
    uint64_t clock0 = t->clock;
    if (refresh && !scores) t->clock += ticks ? clock_advance : (uint64_t)nfound;
    int64_t rank = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t row = rows[i];
        if (row < 0) continue;
        if (values) {
            memcpy(t->values + row * t->dim, values + i * t->dim, sizeof(float) * t->dim);
            count_row(t, row, ctr);
        }
        if (scores) {
            t->scores[row] = scores[i];
        } else if (refresh) {
            uint64_t tick = ticks ? ticks[i] : clock0 + (uint64_t)rank + 1;
            t->scores[row] = hit_score(t->policy, t->scores[row], t->epoch, tick, 0, 0);
        }
        rank++;
    }
    free(rows);
    for (int c = 0; c < 6; c++) t->ctr[c] += ctr[c];
}

/* table.py:553-558 -> _round_erase 1006-1023: key=EMPTY, digest/score/value
 * stay stale; no ticks. */
void ot_erase(ot_table *t, const uint64_t *keys, int64_t n, uint8_t *outcomes) {
    int64_t ctr[6] = {0};
    for (int64_t i = 0; i < n; i++) {
        int64_t row = lookup_row(t, keys[i], ctr);
        if (row < 0) { outcomes[i] = O_NOTFOUND; continue; }
        t->keys[row] = EMPTY_KEY;
        t->occ[row / SLOTS]--;
        t->size--;
        outcomes[i] = O_ERASED;
    }
    for (int c = 0; c < 6; c++) t->ctr[c] += ctr[c];
}

/* table.py:374-434 (export_batch_if) with the service predicate
 * `scores >= min_score` (service.py:263-268) when has_min.  Returns the count;
 * *next_cursor = -1 encodes None. */
int64_t ot_export(ot_table *t, int64_t cursor, int64_t max_count, int32_t has_min,
                  uint64_t min_score, uint64_t *out_k, float *out_v, uint64_t *out_s,
                  int64_t *next_cursor) {
    int64_t ctr[6] = {0};
    int64_t taken = 0;
    *next_cursor = -1;
    for (int64_t r = cursor; r < t->capacity; r++) {
        uint64_t k = t->keys[r];
        if (k >= LOCKED_KEY) continue;
        if (has_min && t->scores[r] < min_score) continue;
        out_k[taken] = k;
        out_s[taken] = t->scores[r];
        memcpy(out_v + taken * t->dim, t->values + r * t->dim, sizeof(float) * t->dim);
        count_row(t, r, ctr);
        taken++;
        if (taken >= max_count) {
            *next_cursor = r + 1 < t->capacity ? r + 1 : -1;
            break;
        }
    }
    for (int c = 0; c < 6; c++) t->ctr[c] += ctr[c];
    return taken;
}

/* Accessors for ctypes. */
/* ---- scalar single-key API (table.py:562-620) ----------------------------
 * ot_lookup_one: lookup (bucket < 0: h1 then h2 in dual mode, table.py:621-631)
 * or find_in_bucket (table.py:570-582).  res = {kind, bucket, slot}.
 * ot_upsert_one: upsert_single (dual = 0: bucket h1 only, 584-599 ->
 * _scalar_upsert_bucket 695-735, locked=False) or upsert_dual (dual = 1,
 * 601-620 -> _scalar_upsert_dual 859-924).  Ticks only where the scalar
 * engine takes them (_scalar_hit 760-762, _score_for_insert 662-672).
 * Returns 0, or 1 (kCustomized without a score) / 2 (a score without
 * kCustomized) before any mutation.  res = {kind, bucket, slot}, ev = {key, score}. */
void ot_lookup_one(ot_table *t, int64_t bucket, uint64_t key, int64_t *res) {
    uint64_t h = fmix64(key);
    uint8_t d = digest_of(h);
    int64_t mask = t->buckets - 1;
    int64_t b = bucket >= 0 ? bucket : (int64_t)(h & (uint64_t)mask);
    int s = probe(t, b, key, d, t->ctr);
    if (s < 0 && bucket < 0 && t->dual) {
        b = (int64_t)(second_hash(h) & (uint64_t)mask);
        s = probe(t, b, key, d, t->ctr);
    }
    res[0] = s >= 0 ? O_FOUND : O_NOTFOUND;
    res[1] = s >= 0 ? b : -1;
    res[2] = s;
}

static void evict_publish(ot_table *t, int64_t b, int m, uint64_t minv, uint64_t key, uint8_t d, uint64_t s_in,
                          const float *val, int64_t *res, uint64_t *ev, int64_t *ctr) {
    /* _scalar_evict 834-857: first eviction recorded at the decision's size */
    if (!t->fel_set) { t->fel_set = 1; t->fel = (double)t->size / (double)t->capacity; }
    ev[0] = t->keys[b * SLOTS + m];
    ev[1] = minv;
    publish(t, b, m, key, d, s_in, val, ctr);
    res[0] = O_EVICTED; res[1] = b; res[2] = m;
}

static int32_t upsert_one(ot_table *t, int32_t dual, uint64_t key, const float *val, int32_t has_score,
                          uint64_t score, int64_t *res, uint64_t *ev, int64_t *ctr) {
    uint64_t h = fmix64(key);
    uint8_t d = digest_of(h);
    int64_t mask = t->buckets - 1;
    int64_t b1 = (int64_t)(h & (uint64_t)mask), b2 = (int64_t)(second_hash(h) & (uint64_t)mask);
    int64_t b = b1;
    int s = probe(t, b1, key, d, ctr);
    if (s < 0 && dual) { b = b2; s = probe(t, b2, key, d, ctr); }
    int custom = t->policy == POL_CUSTOM;
    ev[0] = ev[1] = 0;
    res[1] = -1; res[2] = -1;
    if (s >= 0) {  /* _scalar_hit 749-772 */
        int64_t row = b * SLOTS + s;
        if (custom) {
            if (has_score) t->scores[row] = score;
        } else {
            uint64_t tick = ++t->clock;
            t->scores[row] = hit_score(t->policy, t->scores[row], t->epoch, tick, 0, 0);
        }
        memcpy(t->values + row * t->dim, val, sizeof(float) * t->dim);
        count_row(t, row, ctr);
        res[0] = O_UPDATED; res[1] = b; res[2] = s;
        return 0;
    }
    if (custom && !has_score) return 1;
    if (!custom && has_score) return 2;
    uint64_t s_in = custom ? score : insert_score(t->policy, t->epoch, ++t->clock, 0);
    if (dual) {
        if (t->occ[b1] < SLOTS || t->occ[b2] < SLOTS) {  /* D1 */
            int64_t tb = t->occ[b1] <= t->occ[b2] ? b1 : b2;
            int f = lowest_empty(t, tb);
            publish(t, tb, f, key, d, s_in, val, ctr);
            t->occ[tb]++; t->size++;
            res[0] = O_INSERTED; res[1] = tb; res[2] = f;
            return 0;
        }
        uint64_t n1, n2;
        int m1 = argmin_score(t, b1, &n1), m2 = argmin_score(t, b2, &n2);
        ctr[C_SCANS] += 2;
        uint64_t both = n1 < n2 ? n1 : n2;
        int admit = t->admit_ties_unified ? s_in >= both : s_in > both;
        if (!admit) { res[0] = O_REJECTED; return 0; }
        if (n2 < n1) evict_publish(t, b2, m2, n2, key, d, s_in, val, res, ev, ctr);
        else evict_publish(t, b1, m1, n1, key, d, s_in, val, res, ev, ctr);
        return 0;
    }
    if (t->occ[b1] < SLOTS) {  /* _scalar_claim_free 678-693 */
        int f = lowest_empty(t, b1);
        publish(t, b1, f, key, d, s_in, val, ctr);
        t->occ[b1]++; t->size++;
        res[0] = O_INSERTED; res[1] = b1; res[2] = f;
        return 0;
    }
    uint64_t mn;
    int m = argmin_score(t, b1, &mn);
    ctr[C_SCANS]++;
    if (s_in < mn) { res[0] = O_REJECTED; return 0; }
    evict_publish(t, b1, m, mn, key, d, s_in, val, res, ev, ctr);
    return 0;
}

/* a usage error leaves the table counters untouched: the reference merges a
 * call's local counters only when it returns (table.py:588-598) */
int32_t ot_upsert_one(ot_table *t, int32_t dual, uint64_t key, const float *val, int32_t has_score,
                      uint64_t score, int64_t *res, uint64_t *ev) {
    int64_t ctr[6] = {0};
    int32_t rc = upsert_one(t, dual, key, val, has_score, score, res, ev, ctr);
    if (rc == 0)
        for (int k = 0; k < 6; k++) t->ctr[k] += ctr[k];
    return rc;
}

uint64_t *ot_keys(ot_table *t) { return t->keys; }
uint8_t *ot_digests(ot_table *t) { return t->digests; }
uint64_t *ot_scores(ot_table *t) { return t->scores; }
int64_t *ot_occ(ot_table *t) { return t->occ; }
float *ot_values(ot_table *t) { return t->values; }
int64_t *ot_counters(ot_table *t) { return t->ctr; }
int64_t ot_size(ot_table *t) { return t->size; }
void ot_set_size(ot_table *t, int64_t s) { t->size = s; }
uint64_t ot_clock(ot_table *t) { return t->clock; }
void ot_set_clock(ot_table *t, uint64_t c) { t->clock = c; }
uint64_t ot_epoch(ot_table *t) { return t->epoch; }
void ot_set_epoch(ot_table *t, uint64_t e) { t->epoch = e; }
int32_t ot_fel(ot_table *t, double *out) { *out = t->fel; return t->fel_set; }
void ot_set_fel(ot_table *t, int32_t set, double v) { t->fel_set = set; t->fel = v; }

/* Metadata snapshot / restore for the CPU baseline (keeps lambda fixed
 * between timed batches; values are payload and not restored). */
typedef struct {
    uint64_t *keys, *scores;
    uint8_t *digests;
    int64_t *occ;
    int64_t size;
    uint64_t clock;
} ot_snap;

ot_snap *ot_snapshot(const ot_table *t) {
    ot_snap *s = (ot_snap *)calloc(1, sizeof(ot_snap));
    if (!s) return NULL;
    s->keys = (uint64_t *)malloc(sizeof(uint64_t) * t->capacity);
    s->scores = (uint64_t *)malloc(sizeof(uint64_t) * t->capacity);
    s->digests = (uint8_t *)malloc(t->capacity);
    s->occ = (int64_t *)malloc(sizeof(int64_t) * t->buckets);
    if (!s->keys || !s->scores || !s->digests || !s->occ) return NULL;
    memcpy(s->keys, t->keys, sizeof(uint64_t) * t->capacity);
    memcpy(s->scores, t->scores, sizeof(uint64_t) * t->capacity);
    memcpy(s->digests, t->digests, t->capacity);
    memcpy(s->occ, t->occ, sizeof(int64_t) * t->buckets);
    s->size = t->size;
    s->clock = t->clock;
    return s;
}

void ot_restore(ot_table *t, const ot_snap *s) {
    memcpy(t->keys, s->keys, sizeof(uint64_t) * t->capacity);
    memcpy(t->scores, s->scores, sizeof(uint64_t) * t->capacity);
    memcpy(t->digests, s->digests, t->capacity);
    memcpy(t->occ, s->occ, sizeof(int64_t) * t->buckets);
    t->size = s->size;
    t->clock = s->clock;
}

void ot_snap_free(ot_snap *s) {
    if (!s) return;
    free(s->keys); free(s->scores); free(s->digests); free(s->occ); free(s);
}
