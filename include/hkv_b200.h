/*
 * hkv_b200.h — C-ABI of the B200-native cache-semantic hash table.
 *
 * This is the drop-in boundary for the reference's hot path,
 * `cachekv.CacheTable` (/root/reference/pkg/src/cachekv/table.py:138-1305).
 * The reference has no FFI (pure Python on numpy); each entry point below
 * replaces one reference method, cited per function.  The Python mirror of
 * the reference class (paper_2603_17168_b200/table.py) binds these symbols
 * with ctypes; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Every array argument is a device-accessible pointer (HBM, or mapped
 *    pinned host memory), C-contiguous, owned by the caller.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    asynchronous unless documented as synchronising.
 *  - Return value: HKV_OK or an hkv_status; hkv_last_error() gives the text.
 *    Usage errors are detected on the host before any launch (shapes,
 *    policy/score mismatch, cursor range).  Reserved-sentinel keys are
 *    detected on the device: the offending batch performs no mutation and the
 *    table's device error latch is set (read it with hkv_device_error).
 *  - Keys are uint64 (EMPTY = ~0, LOCKED = ~0-1 reserved), values float32
 *    rows of value_dim, scores uint64.
 */
#ifndef HKV_B200_H
#define HKV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hkv_table hkv_table;
typedef void *hkv_stream; /* cudaStream_t */

enum hkv_status {
    HKV_OK = 0,
    HKV_EINVAL = 1,  /* usage error -> ValueError in the Python mirror */
    HKV_ECUDA = 2,   /* CUDA runtime error */
    HKV_ENOMEM = 3,  /* device / pinned host allocation failed */
    HKV_EBUSY = 4,   /* hkv_gate_acquire(mode 0): the role would have to wait */
    HKV_GATE_NESTED = 5, /* hkv_gate_acquire(mode 2): success, nested in a covering hold */
};

enum hkv_mode { HKV_MODE_SINGLE = 0, HKV_MODE_DUAL = 1 };            /* table.py:63-65 */
enum hkv_policy {                                                     /* scoring.py:27-32 */
    HKV_LRU = 0, HKV_LFU = 1, HKV_EPOCH_LRU = 2, HKV_EPOCH_LFU = 3, HKV_CUSTOMIZED = 4
};
enum hkv_outcome {                                                    /* table.py:68-75 */
    HKV_INSERTED = 0, HKV_UPDATED = 1, HKV_REJECTED = 2, HKV_EVICTED = 3,
    HKV_FOUND = 4, HKV_NOTFOUND = 5, HKV_ERASED = 6
};
enum hkv_upsert_op { HKV_OP_INSERT_OR_ASSIGN = 0, HKV_OP_FIND_OR_INSERT = 1 };
enum hkv_device_error_bits {
    HKV_DERR_SENTINEL_KEY = 1, /* a key >= LOCKED: the batch performed no mutation */
    HKV_DERR_ROLE = 2          /* a mutation kernel ran while the device mirror named a reader group */
};

/* TableConfig (table.py:94-131).  Validation errors mirror table.py:108-127. */
typedef struct {
    int64_t capacity;          /* positive multiple of 128, power-of-two bucket count */
    int64_t value_dim;         /* >= 1 */
    int32_t mode;              /* hkv_mode */
    int32_t score_policy;      /* hkv_policy */
    int64_t fast_tier_budget;  /* buckets whose values live in HBM; -1 = all (store.py:40-63) */
    int32_t digest_filter;     /* 1 = digest-accelerated probe; 0 = ablation (compare all slots) */
    int32_t admit_ties_unified;/* dual mode: admit score == min (table.py:1112-1115) */
    int32_t overflow_in_hbm;   /* 0 = overflow arena in mapped pinned host memory (tiering), 1 = HBM */
    int32_t device;            /* CUDA device ordinal */
    int32_t workers;           /* 1: serial batch-order upserts (bit-exact with the reference's
                                  workers=1 engine); > 1: concurrent LOCKED-sentinel slot-CAS
                                  upserts, the reference's threaded engine (table.py:1185-1241):
                                  serializable, policy invariants hold, order under contention
                                  unspecified */
} hkv_config;

/* TxnCounters (metrics.py:14-20), in this order. */
enum { HKV_CTR_DIGEST_LINE_LOADS = 0, HKV_CTR_FULL_KEY_COMPARES, HKV_CTR_SCORE_SCANS,
       HKV_CTR_SLOT_LOCK_RETRIES, HKV_CTR_VALUE_COPIES_FAST, HKV_CTR_VALUE_COPIES_OVERFLOW,
       HKV_NUM_COUNTERS };

const char *hkv_last_error(void);
const char *hkv_version(void);

/* CacheTable.__init__ (table.py:139-160) + TieredValueStore (store.py:41-79). */
int hkv_create(const hkv_config *cfg, hkv_table **out);
int hkv_destroy(hkv_table *t);
/* Switch the upsert engine of a live table (hkv_config.workers semantics):
 * 1 = serial batch order, > 1 = concurrent slot CAS.  Takes the inserter role. */
int hkv_set_workers(hkv_table *t, int32_t workers);

/* ---- triple-group role gate (gate.py:60-157) ----
 * Readers run with readers, updaters with updaters, an inserter alone;
 * phase-fair FIFO admission.  Every table owns one gate and EVERY entry point
 * below takes its role (find/contains/find_ptr/export/size/... reader,
 * assign updater, upsert/erase/import/restore inserter) for the duration of
 * its launches.  Device layer: each release records an event on its stream;
 * the first entrant of a new group makes its stream wait on them and
 * publishes (group, role) to a device mirror word with a one-thread kernel,
 * so incompatible groups never overlap on the device even on different
 * streams, and mutation kernels check the mirror (HKV_DERR_ROLE).
 * A thread may hold a role across several calls (hkv_gate_acquire ...
 * hkv_gate_release): entry points called by that thread with the same role,
 * or under a held inserter role, nest in the hold (their streams are still
 * fenced); an entry point whose role is incompatible with the thread's hold
 * returns HKV_EINVAL instead of deadlocking.
 * Standalone gates (hkv_gate_create) have the host layer only. */
typedef struct hkv_gate hkv_gate;
enum hkv_role { HKV_ROLE_READER = 0, HKV_ROLE_UPDATER = 1, HKV_ROLE_INSERTER = 2 };
enum hkv_gate_event { HKV_GATE_ACQUIRE = 0, HKV_GATE_RELEASE = 1 };
/* event hook (gate.py:61,70-73): called under the gate lock with the event
 * sequence number, the event, the role and the active count after it */
typedef void (*hkv_gate_hook)(void *user, int64_t seq, int32_t event, int32_t role, int32_t active_count);
int hkv_gate_create(hkv_gate **out);
int hkv_gate_destroy(hkv_gate *g);
int hkv_table_gate(hkv_table *t, hkv_gate **out); /* owned by the table */
int hkv_gate_set_hook(hkv_gate *g, hkv_gate_hook fn, void *user);
/* mode 1: acquire (gate.py:90-104), blocks; mode 0: try_acquire (HKV_EBUSY
 * instead of waiting, gate.py:106-116); mode 2: the scoped acquisition every
 * entry point makes (returns HKV_GATE_NESTED when it nested in the thread's
 * hold; pass nested = 1 to the matching release).
 * has_stream = 0: no device fencing for this acquisition. */
int hkv_gate_acquire(hkv_gate *g, int32_t role, int32_t mode, int32_t has_stream, hkv_stream stream);
/* HKV_EINVAL when no matching acquisition is active (gate.py:128-130). */
int hkv_gate_release(hkv_gate *g, int32_t role, int32_t nested, int32_t has_stream, hkv_stream stream);
/* active role (-1 = idle), active count, groups admitted so far */
int hkv_gate_state(hkv_gate *g, int32_t *role, int32_t *count, int64_t *groups);

/* find (table.py:304-323): found[i] in {0,1}; out rows of misses untouched
 * (zero_misses = 0, the reference contract for a caller-provided `out`) or
 * written with zeros (zero_misses = 1: same result as the reference's freshly
 * zeroed `out`, without a separate memset pass); out may be NULL (contains,
 * table.py:344-351). */
int hkv_find(hkv_table *t, const uint64_t *keys, int64_t n, float *out, uint8_t *found,
             int32_t zero_misses, hkv_stream stream);
int hkv_contains(hkv_table *t, const uint64_t *keys, int64_t n, uint8_t *found, hkv_stream stream);
/* find_ptr (table.py:325-342): tier 0 fast / 1 overflow, element offset in the
 * tier arena, -1 for misses. */
int hkv_find_ptr(hkv_table *t, const uint64_t *keys, int64_t n, uint8_t *found, uint8_t *tier,
                 int64_t *offset, hkv_stream stream);

/* insert_or_assign / insert_and_evict / find_or_insert (table.py:515-551,
 * 934-1181).  Serial batch-order semantics.
 *   op            hkv_upsert_op
 *   values        (n, dim) input; in/out for FIND_OR_INSERT (values_inout)
 *   scores        (n,) iff policy == HKV_CUSTOMIZED, else NULL
 *   evicted_*     NULL, or (n)-row buffers: insert_and_evict outputs ordered by
 *                 the evicting op's batch index; *n_evicted_dev (device int64)
 *                 receives the count
 *   ticks         NULL -> tick[i] = clock + i + 1 and clock += n (table.py:192-196);
 *                 else per-op ticks and clock += clock_advance (sharded tables). */
int hkv_upsert(hkv_table *t, int32_t op, const uint64_t *keys, float *values,
               const uint64_t *scores, int64_t n, uint8_t *outcomes, uint64_t *evicted_keys,
               float *evicted_values, uint64_t *evicted_scores, int64_t *n_evicted_dev,
               const uint64_t *ticks, uint64_t clock_advance, hkv_stream stream);

/* Host-buffer entry points: the same operations on HOST arrays (the
 * reference's numpy-in / numpy-out contract, table.py:304-323 and 515-551).
 * Pinned (page-locked) buffers get full PCIe bandwidth; pageable ones work
 * but stage through the driver.  The call is SYNCHRONOUS: it returns once
 * every output is in host memory.  Internally the batch is pipelined:
 *   hkv_find_host    probes chunk c+1 while chunk c's rows stream back (D2H);
 *   hkv_upsert_host  copies the value rows H2D on a second stream while the
 *                    metadata pass (which needs only the keys) runs; the value
 *                    scatter waits for that copy.
 * op: HKV_OP_INSERT_OR_ASSIGN, or HKV_OP_FIND_OR_INSERT (values in/out: the
 * rows of found keys are copied back).  ticks as in hkv_upsert (host array
 * or NULL). */
int hkv_find_host(hkv_table *t, const uint64_t *keys, int64_t n, float *out, uint8_t *found,
                  int32_t zero_misses, hkv_stream stream);
int hkv_upsert_host(hkv_table *t, int32_t op, const uint64_t *keys, float *values,
                    const uint64_t *scores, int64_t n, uint8_t *outcomes, const uint64_t *ticks,
                    uint64_t clock_advance, hkv_stream stream);

/* Sharded find over NVLink peer memory (no reference
 * counterpart: the reference leaves sharding to the application).  A
 * hash-sharded table of `world` (power of two) equal shards, contiguous
 * bucket ranges: global bucket = fmix64(key) & (world * buckets - 1), owner =
 * global bucket / buckets.  hkv_find_peer probes the owner shard's digest
 * line and keys and copies its value row in place — no routing, no
 * all-to-all — with results identical to the routed find.  Shards must keep
 * every value row in HBM (fast_tier_budget == buckets), single mode, digest
 * filter on.  Structural counters are not updated by peer finds.
 *   hkv_ipc_handles   3 cudaIpcMemHandle_t (keys, digests, values) of a shard
 *   hkv_set_peers     world x 3 handles gathered from every rank (own slot ignored)
 *   hkv_set_peers_local  shards of the same process (other devices need P2P) */
int hkv_ipc_handles(hkv_table *t, void *out, int64_t out_bytes);
int hkv_set_peers(hkv_table *t, int32_t world, int32_t rank, const void *handles);
int hkv_set_peers_local(hkv_table *t, int32_t world, hkv_table *const *shards);
int hkv_find_peer(hkv_table *t, const uint64_t *keys, int64_t n, float *out, uint8_t *found,
                  int32_t zero_misses, hkv_stream stream);

/* assign (table.py:438-442) when values != NULL; assign_scores (444-449) with
 * explicit scores (kCustomized) or refresh != 0.  Last duplicate wins.
 * Refresh ticks: NULL -> clock + (found keys before i) + 1 and clock += found
 * (table.py:481-483); else ticks[i] for found keys and clock += clock_advance. */
int hkv_assign(hkv_table *t, const uint64_t *keys, const float *values, const uint64_t *scores,
               int32_t refresh, int64_t n, uint8_t *outcomes, const uint64_t *ticks,
               uint64_t clock_advance, hkv_stream stream);

/* ---- single-key API (table.py:562-620; LookupResult / UpsertResult 78-91) ----
 * One key per call, synchronous, host arguments.  Reader role for the
 * lookups, inserter role for the upserts.
 *   hkv_lookup          probe h1, then h2 in dual mode (table.py:562-568, 621-631)
 *   hkv_find_in_bucket  probe one bucket; a miss is definitive for it (570-582)
 *   hkv_upsert_single   update / insert / reject / evict in bucket h1 only,
 *                       also on a dual-mode table (584-599, 695-735)
 *   hkv_upsert_dual     dual-mode two-bucket upsert (601-620, 859-924);
 *                       HKV_EINVAL on a single-mode table
 * has_score / score: the optional explicit score (kCustomized).  As in the
 * scalar engine, a score given to a non-kCustomized table is an error only
 * when the key is absent (table.py:662-672).  Ticks: one per non-custom hit
 * or insert decision.  result->kind is an hkv_outcome; bucket / slot are -1
 * for misses and rejections; evicted_key / evicted_score are valid for
 * HKV_EVICTED. */
typedef struct {
    int32_t kind;
    int32_t slot;
    int64_t bucket;
    uint64_t evicted_key;
    uint64_t evicted_score;
} hkv_one_result;
int hkv_lookup(hkv_table *t, uint64_t key, hkv_one_result *result, hkv_stream stream);
int hkv_find_in_bucket(hkv_table *t, int64_t bucket, uint64_t key, hkv_one_result *result, hkv_stream stream);
int hkv_upsert_single(hkv_table *t, uint64_t key, const float *value, int32_t has_score, uint64_t score,
                      hkv_one_result *result, hkv_stream stream);
int hkv_upsert_dual(hkv_table *t, uint64_t key, const float *value, int32_t has_score, uint64_t score,
                    hkv_one_result *result, hkv_stream stream);

/* erase (table.py:553-558, 1006-1023). */
int hkv_erase(hkv_table *t, const uint64_t *keys, int64_t n, uint8_t *outcomes, hkv_stream stream);

/* export_batch_if (table.py:374-434).  Scans rows [cursor, capacity) in
 * (bucket, slot) order keeping user keys with score >= min_score (when
 * has_min_score; service.py:263-268) and, when row_mask != NULL, with
 * row_mask[r - cursor] != 0 for rows r < cursor + mask_rows.  Writes up to
 * max_count entries.  SYNCHRONISING: *count and *next_cursor (-1 = None) are
 * host values. */
int hkv_export(hkv_table *t, int64_t cursor, int64_t max_count, int32_t has_min_score,
               uint64_t min_score, const uint8_t *row_mask, int64_t mask_rows, uint64_t *out_keys,
               float *out_values, uint64_t *out_scores, int64_t *count, int64_t *next_cursor,
               hkv_stream stream);

/* size / load_factor (table.py:198-204).  SYNCHRONISING. */
int hkv_size(hkv_table *t, int64_t *size, hkv_stream stream);
/* set_epoch (table.py:206; scoring.py:45-50). */
int hkv_set_epoch(hkv_table *t, uint64_t epoch);
int hkv_get_epoch(hkv_table *t, uint64_t *epoch);
/* Logical clock, first_eviction_lambda (table.py:156, 986-991), TxnCounters.
 * SYNCHRONISING. */
int hkv_clock(hkv_table *t, uint64_t *clock, hkv_stream stream);
int hkv_first_eviction_lambda(hkv_table *t, int32_t *is_set, double *value, hkv_stream stream);
int hkv_counters(hkv_table *t, int64_t *out /* HKV_NUM_COUNTERS */, hkv_stream stream);
int hkv_reset_counters(hkv_table *t, hkv_stream stream);
/* Device error latch (bitmask of hkv_device_error_bits); clears it.  SYNCHRONISING. */
int hkv_device_error(hkv_table *t, int32_t *bits, hkv_stream stream);

/* Raw state transfer (test / checkpoint support; the reference has no import
 * API).  Host pointers; layout is the reference's arrays
 * (table.py:143-146, store.py:56-61): keys/scores (B,128) u64, digests (B,128)
 * u8, values (capacity, dim) f32 in row order.  occupancy is derived from keys.
 * SYNCHRONISING. */
int hkv_import_state(hkv_table *t, const uint64_t *keys, const uint8_t *digests,
                     const uint64_t *scores, const float *values, uint64_t clock,
                     int32_t fel_set, double fel);
int hkv_export_state(hkv_table *t, uint64_t *keys, uint8_t *digests, uint64_t *scores,
                     float *values, int64_t *occupancy);

/* Keys and scores of global rows [row0, row0 + nrows) (row = bucket * 128 +
 * slot) into host or device buffers (either may be NULL).  SYNCHRONISING.
 * Serves export_batch_if with a Python predicate (table.py:402-409): the
 * predicate sees one chunk of rows at a time. */
int hkv_read_rows(hkv_table *t, int64_t row0, int64_t nrows, uint64_t *keys, uint64_t *scores,
                  hkv_stream stream);

/* Value rows [row0, row0 + nrows) (global rows; either tier) into host or
 * device memory.  SYNCHRONISING.  Reads a LookupResult's value handle
 * (store.py:96-100). */
int hkv_read_value_rows(hkv_table *t, int64_t row0, int64_t nrows, float *out, hkv_stream stream);

/* Metadata snapshot held in HBM (keys, digests, scores, occupancy bits, size,
 * clock): the bench restores it between timed repeats so the load factor
 * stays fixed.  Values are not part of the snapshot. */
int hkv_snapshot(hkv_table *t, hkv_stream stream);
int hkv_restore(hkv_table *t, hkv_stream stream);

/* Device-side consistency scan (table.py:1284-1299).  SYNCHRONISING.
 * *ok = 1 when occupancy bits, size counter and digests agree with the keys. */
int hkv_check_consistency(hkv_table *t, int32_t *ok, hkv_stream stream);

/* Sharding helper (multi-GPU routing): for each key compute the
 * destination rank of its global bucket (h & (global_buckets-1)) >> log2(local
 * buckets), and a stable counting-sort permutation grouping keys by
 * destination.  perm[j] = source index of the j-th routed key; counts[r] =
 * keys for rank r (device int64[world]). */
int hkv_route(const uint64_t *keys, int64_t n, int64_t global_buckets, int32_t world,
              int32_t *perm, int64_t *counts, hkv_stream stream);

/* Routed exchange helpers of the sharded table (device pointers, async on
 * `stream`; 0 ok, 1 bad arguments, 2 CUDA error):
 *   hkv_route_gather  for routed position j (source op i = perm[j]):
 *                     meta[j] = {key, tick_base + i + 1[, score]} (3 words
 *                     when scores != NULL) and out_values row j = values row i
 *   hkv_scatter_rows  dst[perm[j]] = src[j] for rows of row_bytes (1, or a
 *                     multiple of 4): results back into batch order */
int hkv_route_gather(const int32_t *perm, int64_t n, const uint64_t *keys, const uint64_t *scores,
                     const float *values, int64_t dim, uint64_t tick_base, uint64_t *meta, float *out_values,
                     hkv_stream stream);
int hkv_scatter_rows(const int32_t *perm, int64_t n, const void *src, void *dst, int64_t row_bytes,
                     hkv_stream stream);

/* Launch-count instrumentation: number of kernels this library has launched. */
int64_t hkv_launch_count(void);

/* Live kernel timing for roofline reporting: while enabled, the dominant
 * kernel of each op (probe / apply / assign-apply) is bracketed by CUDA
 * events on its launch stream.  hkv_kernel_times() synchronises, returns the
 * accumulated milliseconds and launch count of the kernel named `name`
 * ("find", "find_gather", "apply", "values_write", "dual_flow", "assign_apply")
 * and resets it.  enable = 2 also brackets the mutation pipeline's stages
 * ("prep", "sort", "segments", "finalize"; more events, so not for bench). */
int hkv_set_kernel_timing(int32_t enable);
int hkv_kernel_times(const char *name, double *ms, int64_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* HKV_B200_H */
