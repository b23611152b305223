// hkv_kernels.h — host-side launchers for the table kernels (internal).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "hkv_common.cuh"

namespace hkv {

constexpr int kRecU64 = 4, kRecU32 = 8;  // stride of the per-op read record (32 B)

// Per-batch device scalars (zeroed by the launcher before each batch).
struct Scalars {
  int err;                       // sentinel key seen in this batch
  union {  // the collector's k_alloc reserves both with one packed 64-bit atomic per block
    struct {
      unsigned nseg;             // single-op bucket segments
      unsigned nmulti;           // multi-op bucket segments
    };
    unsigned long long seg_pack;
  };
  unsigned first_ev;             // lowest batch index with an Evicted outcome
  unsigned npend[2];             // dual-mode pending list sizes (per round parity)
  unsigned has_runs;             // single mode: some op is followed by the same key in its bucket segment
  unsigned nlong;                // single mode: segments of >= kLongSeg ops (k_meta_long)
  long long size_before;         // table size when the batch started
  unsigned long long nfound;     // assign: found ops (clock advance for refresh)
  long long n_sel;               // DeviceSelect count
  unsigned long long fel_cnt;    // k_finalize: inserts before the first eviction (summed over blocks)
  unsigned fel_done;             // k_finalize: blocks finished
  // collector (hkv_collect.cu): k_alloc hands out both with one packed
  // 64-bit atomic per block
  union {
    struct {
      unsigned nsegd;            // segment descriptors (touched buckets)
      unsigned npos;             // sorted positions handed out
    };
    unsigned long long alloc_pack;
  };
  unsigned nbig;                 // segments of more than 16 ops (both groupings; skew hint)
};

// Per-stream scratch, grown on demand.
struct Workspace {
  int64_t cap_n = 0;
  int64_t cap_ev = 0;  // rows of evicted-value scratch
  int64_t cap_ek = 0;  // entries of evicted key/score scratch
  int dim = 0;
  uint32_t* bkt = nullptr;
  uint32_t* idx = nullptr;
  uint32_t* sbkt = nullptr;
  uint32_t* sidx = nullptr;
  uint32_t* seg = nullptr;
  uint32_t* aux = nullptr;   // assign: rows / evicted list
  uint32_t* aux2 = nullptr;  // assign: found ranks
  uint64_t* skey = nullptr;  // single mode: bucket-segment records (3 u64 per item)
  uint64_t* lrec = nullptr;  // single mode: records of long segments (3 u64 each)
  uint32_t* agg = nullptr;   // assign: per-row aggregation hash (row key | last op + 1 | count)
  int64_t agg_cap = 0;
  uint64_t* skeys = nullptr; // single mode: keys in sorted (bucket, batch index) order
  uint32_t* vrow = nullptr;  // single mode: destination row of final value writers
  // Per-op value-read record, 32 B (one sector per op that reads a row):
  // {victim key, victim score, row, provenance}.  ek / es / rrow / rsrc are
  // strided views into it: ek[kRecU64 * i], rrow[kRecU32 * i], ...
  uint64_t* rrec = nullptr;
  uint32_t* rrow = nullptr;  // single mode: row of a value read
  int32_t* rsrc = nullptr;   // single mode: provenance of a value read (-1 = pre-batch row)
  int* lwtab = nullptr;      // single mode: per-thread last-writer tables of the metadata pass
  uint32_t* b2 = nullptr;    // dual: second bucket
  uint32_t* pend = nullptr;  // dual: second pending list
  uint64_t* ek = nullptr;  // victim key of op i at ek[kRecU64 * i] (view of rrec)
  uint64_t* es = nullptr;  // victim score at es[kRecU64 * i] (view of rrec)
  float* ev = nullptr;
  // dual mode: 2n (bucket, op) pairs and per-op ranks (hkv_dual.cu)
  int64_t dcap = 0;
  uint32_t* dpk = nullptr;
  uint32_t* dpv = nullptr;
  uint32_t* dsk = nullptr;
  uint32_t* dsv = nullptr;
  uint32_t* drank = nullptr;
  int64_t dbk = 0;             // dual: per-bucket counters / offsets of the rank prep (buckets + 1)
  uint32_t* dcnt = nullptr;
  uint32_t* doff = nullptr;
  void* dcub = nullptr;
  size_t dcub_bytes = 0;
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  int64_t cub_for_n = -1;
  Scalars* sc = nullptr;
  uint32_t* col = nullptr;   // collector: per-bucket op counters / range cursors (zero between calls)
  uint32_t* segd = nullptr;  // collector: segment descriptors (4 u32 per touched bucket)
  volatile unsigned* skew_host = nullptr;  // mapped pinned word: segments of > 16 ops in the last batch
  unsigned* skew_dev = nullptr;            //   (written by k_finalize; read by the next call's path choice)
  int64_t col_buckets = 0;
};

struct OpArgs {
  const uint64_t* keys;
  float* values;
  const uint64_t* scores;
  const uint64_t* ticks;
  uint8_t* outcomes;
  uint64_t* ek;  // per-op evicted (key, score) scratch (collect): ek[kRecU64 * i], es[kRecU64 * i]
  uint64_t* es;
  float* ev;
  int op;        // 0 insert_or_assign, 1 find_or_insert, 2 erase
  int collect;
  uint64_t epoch;
  Scalars* sc;
};

enum { kOpUpsert = 0, kOpFindOrInsert = 1, kOpErase = 2 };

// mode 0: find (misses untouched), 3: find (misses zero-filled), 1: contains, 2: find_ptr.
// rows: n-entry scratch for modes 0/3.
// One shard of a hash-sharded table as seen by another rank (peer memory:
// CUDA IPC over NVLink, or a table of the same process).
struct PeerView {
  const uint64_t* ks;   // (key, score) pairs
  const uint8_t* digests;
  const float* values;  // fast tier: every row of the shard (peer find needs fast_tier_budget == buckets)
};
// find over the whole sharded table by reading the owner shard's bucket
// directly (no routing, no all-to-all): global bucket = h & gmask, owner =
// global bucket >> llog2b.
void launch_find_peer(const PeerView* views, uint64_t gmask, int llog2b, int dim, const uint64_t* keys, int64_t n,
                      float* out, uint8_t* found, int zero_misses, int* err, cudaStream_t s, int num_sms);

void launch_find(const TableDev& t, const uint64_t* keys, int64_t n, float* out, uint8_t* found,
                 uint8_t* tier, int64_t* offset, int mode, uint32_t* rows, cudaStream_t s, int num_sms);

// Returns cudaSuccess or the first error.
cudaError_t run_mutation(const TableDev& t, OpArgs a, int64_t n, int log2_buckets, Workspace& ws,
                         unsigned long long dual_tag, unsigned long long* lead, int64_t* n_evicted,
                         uint64_t* ek_out, float* ev_out, uint64_t* es_out, uint64_t clock_advance,
                         cudaStream_t s, int num_sms, cudaEvent_t values_ready = nullptr);

cudaError_t run_assign(const TableDev& t, const uint64_t* keys, const float* values,
                       const uint64_t* scores, int refresh, uint64_t epoch, int64_t n, uint8_t* outcomes,
                       const uint64_t* ticks, uint64_t clock_advance, int log2_buckets, Workspace& ws,
                       cudaStream_t s, int num_sms);

cudaError_t run_export(const TableDev& t, int64_t cursor, int64_t max_count, int has_min, uint64_t min_score,
                       const uint8_t* mask, int64_t mask_rows, uint64_t* ok, float* ov, uint64_t* os,
                       int64_t* count, int64_t* next, Workspace& ws, cudaStream_t s, int num_sms);

cudaError_t run_bits_from_keys(const TableDev& t, int64_t buckets, cudaStream_t s);
cudaError_t run_consistency(const TableDev& t, int64_t buckets, int* ok_dev, cudaStream_t s);
cudaError_t run_route(const uint64_t* keys, int64_t n, int64_t global_buckets, int world, int32_t* perm,
                      int64_t* counts, Workspace& ws, cudaStream_t s);

// Live timing of dominant kernels (hkv_set_kernel_timing).
void ktimer_begin(const char* name, cudaStream_t s, int level = 1);
void ktimer_end(const char* name, cudaStream_t s, int level = 1);

// sort-free grouping of sparse single-mode batches (hkv_collect.cu)
bool collect_eligible(int64_t n, int log2_buckets, unsigned last_big_segments);
cudaError_t run_collect(const TableDev& t, OpArgs a, int64_t n, int log2_buckets, Workspace& ws, cudaStream_t s,
                        int num_sms, uint8_t fcode);

cudaError_t ws_reserve(Workspace& ws, int64_t n, int dim, int ev_mode, bool dual);
cudaError_t ws_reserve_dual(Workspace& ws, int64_t n, int log2_buckets);
void ws_free_dual(Workspace& ws);
cudaError_t run_dual(const TableDev& t, OpArgs a, int64_t n, int log2_buckets, Workspace& ws,
                     unsigned long long* turn, unsigned long long tag, int vec, cudaStream_t s, int num_sms);
void ws_free(Workspace& ws);
// concurrent upserts (workers > 1): LOCKED-sentinel slot CAS + bucket locks
// deterministic dual mode in warp-synchronous rounds over run_dual's ranks / turns (hkv_cas.cu)
cudaError_t run_dual_rounds(const TableDev& t, OpArgs a, int64_t n, const uint32_t* rank, unsigned long long* turn,
                            unsigned long long tag, int vec, cudaStream_t s, int num_sms);
cudaError_t run_cas(const TableDev& t, OpArgs a, int64_t n, unsigned* locks, int vec, cudaStream_t s,
                    int num_sms);

}  // namespace hkv
