// hkv_api.cu — the C-ABI (include/hkv_b200.h): table construction, memory
// placement (HBM / mapped pinned host tier), per-stream workspaces and the
// entry points that replace cachekv.CacheTable's methods.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hkv_b200.h"
#include "hkv_gate.h"
#include "hkv_kernels.h"
#include "hkv_single.h"

namespace {
thread_local std::string g_err;
}

namespace hkv {
unsigned long long g_launches = 0;
void set_error(const char* msg) { g_err = msg; }

namespace {
struct KTimer {
  std::mutex mu;
  bool enabled = false;
  int level = 0;  // 1: the per-kernel regions bench.py reads; 2: also pipeline stages (tools/stage_times.py)
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
  };
  std::map<cudaStream_t, std::vector<Pending>> open;  // begun, awaiting end
  std::vector<Pending> done;
  // Events are created up front (hkv_set_kernel_timing) and recycled: creating
  // an event inside a timed region can block the host while the GPU drains its
  // queue, which shows up as idle time inside the caller's own event pairs.
  std::vector<cudaEvent_t> pool;
  cudaEvent_t take() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
};
KTimer& ktimer() {
  static KTimer k;
  return k;
}
}  // namespace

void ktimer_begin(const char* name, cudaStream_t s, int level) {
  KTimer& k = ktimer();
  std::lock_guard<std::mutex> g(k.mu);
  if (!k.enabled || level > k.level) return;
  KTimer::Pending p;
  p.name = name;
  p.a = k.take();
  p.b = k.take();
  cudaEventRecord(p.a, s);
  k.open[s].push_back(p);
}

void ktimer_end(const char* name, cudaStream_t s, int level) {
  KTimer& k = ktimer();
  std::lock_guard<std::mutex> g(k.mu);
  if (!k.enabled || level > k.level) return;
  auto& v = k.open[s];
  if (v.empty()) return;
  KTimer::Pending p = v.back();
  v.pop_back();
  cudaEventRecord(p.b, s);
  k.done.push_back(p);
}
}  // namespace hkv

using namespace hkv;

namespace {

struct TableScalars {
  unsigned long long size;
  unsigned long long clock;
  unsigned long long counters[6];
  unsigned long long round;
  int err;
  int fel_set;
  double fel;
  int check[4];  // consistency scratch: ok, pad, total(u64)
};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int gate_fail(int rc) {
  if (rc != HKV_EINVAL) g_err = "role gate: CUDA fencing failed";
  return rc;
}

int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return HKV_ECUDA;
}

}  // namespace

// Device staging for the host-buffer entry points (hkv_find_host /
// hkv_upsert_host): a copy stream, a ring of chunk slots and their events.
constexpr int kRing = 3;
struct HostStage {
  std::mutex mu;  // the staging buffers serve one host-buffer call at a time (readers may run concurrently)
  cudaStream_t copy = nullptr;
  cudaEvent_t ready[kRing] = {}, done[kRing] = {}, start = nullptr, vals = nullptr;
  uint64_t* keys = nullptr;  // find: kRing chunk slots; upsert: the batch
  size_t keys_cap = 0;
  float* rows = nullptr;
  size_t rows_cap = 0;
  uint8_t* bytes = nullptr;  // found / outcomes
  size_t bytes_cap = 0;
  uint64_t* aux = nullptr;   // scores, ticks
  size_t aux_cap = 0;
  cudaError_t init() {
    if (copy) return cudaSuccess;
    cudaError_t e = cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking);
    for (int k = 0; k < kRing && !e; k++) {
      if ((e = cudaEventCreateWithFlags(&ready[k], cudaEventDisableTiming))) break;
      e = cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming);
    }
    if (!e) e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
    if (!e) e = cudaEventCreateWithFlags(&vals, cudaEventDisableTiming);
    return e;
  }
  void release() {
    if (copy) cudaStreamSynchronize(copy);
    for (void* p : {(void*)keys, (void*)rows, (void*)bytes, (void*)aux})
      if (p) cudaFree(p);
    for (int k = 0; k < kRing; k++) {
      if (ready[k]) cudaEventDestroy(ready[k]);
      if (done[k]) cudaEventDestroy(done[k]);
    }
    if (start) cudaEventDestroy(start);
    if (vals) cudaEventDestroy(vals);
    if (copy) cudaStreamDestroy(copy);
  }
};

template <class T>
cudaError_t grow_dev(T*& p, size_t& cap, size_t need) {
  if (need <= cap) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  cudaError_t e = cudaMalloc(&p, need * sizeof(T));
  if (!e) cap = need;
  return e;
}

struct hkv_table {
  hkv_config cfg;
  int64_t buckets = 0;
  int log2b = 0;
  int num_sms = 148;
  uint64_t fast_rows = 0;
  uint64_t epoch = 0;
  unsigned long long dual_epoch = 0;  // dual-mode turn-counter tag (hkv_dual.cu)
  TableDev dev{};
  uint64_t* ks = nullptr;       // [capacity] x {key, score} (hkv_common.cuh)
  uint8_t* digests = nullptr;
  uint32_t* bits = nullptr;
  uint64_t* smin = nullptr;     // [B][8] per-16-slot-group score minima (eviction summary)
  uint32_t* svalid = nullptr;   // [B] bit g: smin[b][g] is exact
  float* vfast = nullptr;
  float* vover = nullptr;       // device pointer of the overflow arena
  float* vover_host = nullptr;  // pinned host allocation (mapped), if used
  TableScalars* sc = nullptr;
  unsigned* role_word = nullptr;  // device mirror of the gate's group (never snapshotted)
  unsigned* locks = nullptr;      // CAS engine bucket locks (workers > 1)
  OneResult* one = nullptr;       // single-key API: result + value row staging (lazy)
  float* one_val = nullptr;
  hkv_gate* gate = nullptr;
  unsigned long long* lead = nullptr;
  // metadata snapshot
  uint64_t* snap_ks = nullptr;
  uint8_t* snap_digests = nullptr;
  uint32_t* snap_bits = nullptr;
  uint64_t* snap_smin = nullptr;
  uint32_t* snap_svalid = nullptr;
  TableScalars* snap_sc = nullptr;
  // peer views of the other shards (hkv_set_peers*): device array + what was opened
  PeerView* peers_dev = nullptr;
  int peer_world = 0;
  int peer_llog2b = 0;
  std::vector<void*> ipc_opened;
  std::mutex mu;
  std::map<cudaStream_t, Workspace> ws;
  std::map<cudaStream_t, std::mutex> wsmu;
  std::map<cudaStream_t, HostStage> hs;

  // A stream's scratch serves one call at a time: the lease holds its lock
  // from the (re)allocation through the launches that use it, so concurrent
  // callers on one stream (overlapping reader groups) never see a buffer
  // freed by another caller's growth.
  struct WsLease {
    std::unique_lock<std::mutex> lk;
    Workspace& w;
    operator Workspace&() { return w; }
  };
  WsLease workspace(cudaStream_t s) {
    std::mutex* m;
    Workspace* w;
    {
      std::lock_guard<std::mutex> g(mu);
      m = &wsmu[s];
      w = &ws[s];
    }
    return WsLease{std::unique_lock<std::mutex>(*m), *w};
  }
  HostStage& stage(cudaStream_t s) {
    std::lock_guard<std::mutex> g(mu);
    return hs[s];
  }
};

namespace {

std::mutex g_route_mu;
std::map<cudaStream_t, Workspace> g_route_ws;

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

void free_table(hkv_table* t) {
  if (!t) return;
  DeviceGuard g(t->cfg.device);
  if (t->gate) gate_delete(t->gate);
  if (t->one) cudaFree(t->one);
  if (t->locks) cudaFree(t->locks);
  if (t->one_val) cudaFree(t->one_val);
  void* dptrs[] = {t->ks, t->digests, t->bits, t->smin, t->svalid, t->vfast, t->sc, t->role_word, t->lead,
                   t->snap_ks, t->snap_digests, t->snap_bits, t->snap_smin, t->snap_svalid,
                   t->snap_sc};
  for (void* p : dptrs)
    if (p) cudaFree(p);
  if (t->vover_host) cudaFreeHost(t->vover_host);
  else if (t->vover) cudaFree(t->vover);
  for (auto& kv : t->ws) ws_free(kv.second);
  for (auto& kv : t->hs) kv.second.release();
  for (void* p : t->ipc_opened) cudaIpcCloseMemHandle(p);
  if (t->peers_dev) cudaFree(t->peers_dev);
  delete t;
}

}  // namespace

extern "C" {

const char* hkv_last_error(void) { return g_err.c_str(); }
const char* hkv_version(void) { return "hkv_b200 0.1 sm_100a"; }
int64_t hkv_launch_count(void) { return (int64_t)g_launches; }

int hkv_set_kernel_timing(int32_t enable) {
  KTimer& k = ktimer();
  std::lock_guard<std::mutex> g(k.mu);
  k.enabled = enable != 0;
  k.level = enable;
  while (k.enabled && k.pool.size() < 8192) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) break;
    k.pool.push_back(e);
  }
  return HKV_OK;
}

int hkv_kernel_times(const char* name, double* ms, int64_t* launches) {
  if (!name || !ms || !launches) return fail(HKV_EINVAL, "null argument");
  KTimer& k = ktimer();
  std::lock_guard<std::mutex> g(k.mu);
  double tot = 0.0;
  int64_t cnt = 0;
  std::vector<KTimer::Pending> keep;
  for (auto& p : k.done) {
    if (p.name != name) {
      keep.push_back(p);
      continue;
    }
    cudaError_t e = cudaEventSynchronize(p.b);
    if (e) return cuda_fail(e, "kernel timing");
    float f = 0.f;
    cudaEventElapsedTime(&f, p.a, p.b);
    tot += f;
    cnt++;
    k.pool.push_back(p.a);
    k.pool.push_back(p.b);
  }
  k.done.swap(keep);
  *ms = tot;
  *launches = cnt;
  return HKV_OK;
}

int hkv_create(const hkv_config* cfg, hkv_table** out) {
  if (!cfg || !out) return fail(HKV_EINVAL, "null argument");
  *out = nullptr;
  const hkv_config c = *cfg;
  // table.py:108-127 (same messages)
  if (c.capacity <= 0 || c.capacity % kSlots != 0) return fail(HKV_EINVAL, "capacity must be a positive multiple of 128");
  const int64_t bc = c.capacity / kSlots;
  if (bc & (bc - 1)) return fail(HKV_EINVAL, "bucket count must be a power of two");
  if (c.value_dim < 1) return fail(HKV_EINVAL, "value_dim must be >= 1");
  if (c.capacity > (1ll << 31)) return fail(HKV_EINVAL, "capacity above 2^31 slots per device is not supported");
  const int64_t budget = c.fast_tier_budget < 0 ? bc : c.fast_tier_budget;
  if (budget > bc) return fail(HKV_EINVAL, "fast_tier_budget out of range");
  if (c.mode != HKV_MODE_SINGLE && c.mode != HKV_MODE_DUAL) return fail(HKV_EINVAL, "unknown mode");
  if (c.score_policy < HKV_LRU || c.score_policy > HKV_CUSTOMIZED) return fail(HKV_EINVAL, "unknown policy");
  if (c.value_dim > (1 << 20)) return fail(HKV_EINVAL, "value_dim too large");
  if (c.workers < 1) return fail(HKV_EINVAL, "workers must be >= 1");

  DeviceGuard g(c.device);
  hkv_table* t = new hkv_table();
  t->cfg = c;
  t->cfg.fast_tier_budget = budget;
  t->buckets = bc;
  while ((1ll << t->log2b) < bc) t->log2b++;
  cudaDeviceGetAttribute(&t->num_sms, cudaDevAttrMultiProcessorCount, c.device);
  t->fast_rows = (uint64_t)budget * kSlots;
  const uint64_t cap = (uint64_t)c.capacity;
  const uint64_t dim = (uint64_t)c.value_dim;
  const uint64_t over_rows = cap - t->fast_rows;
  cudaError_t e;
  if ((e = cudaMalloc((void**)&t->ks, cap * 16)) || (e = cudaMalloc((void**)&t->digests, cap)) ||
      (e = cudaMalloc((void**)&t->bits, (size_t)bc * 16)) ||
      (e = cudaMalloc((void**)&t->smin, (size_t)bc * 64)) || (e = cudaMalloc((void**)&t->svalid, (size_t)bc * 4)) ||
      (e = cudaMalloc((void**)&t->sc, sizeof(TableScalars))) || (e = cudaMalloc((void**)&t->role_word, 4))) {
    free_table(t);
    return fail(HKV_ENOMEM, std::string("device allocation failed: ") + cudaGetErrorString(e));
  }
  if (t->fast_rows && (e = cudaMalloc((void**)&t->vfast, t->fast_rows * dim * 4))) {
    free_table(t);
    return fail(HKV_ENOMEM, std::string("HBM value arena allocation failed: ") + cudaGetErrorString(e));
  }
  if (over_rows) {
    if (c.overflow_in_hbm) {
      e = cudaMalloc((void**)&t->vover, over_rows * dim * 4);
    } else {
      // tiered KV separation: overflow values in mapped pinned host memory
      e = cudaHostAlloc((void**)&t->vover_host, over_rows * dim * 4, cudaHostAllocMapped | cudaHostAllocPortable);
      if (!e) e = cudaHostGetDevicePointer((void**)&t->vover, t->vover_host, 0);
    }
    if (e) {
      free_table(t);
      return fail(HKV_ENOMEM, std::string("overflow arena allocation failed: ") + cudaGetErrorString(e));
    }
  }
  if (c.workers > 1 && ((e = cudaMalloc((void**)&t->locks, (size_t)bc * 4)) ||
                         (e = cudaMemset(t->locks, 0, (size_t)bc * 4)))) {
    free_table(t);
    return fail(HKV_ENOMEM, "bucket lock allocation failed");
  }
  if (c.mode == HKV_MODE_DUAL && (e = cudaMalloc((void**)&t->lead, (size_t)bc * 8))) {
    free_table(t);
    return fail(HKV_ENOMEM, "lead array allocation failed");
  }
  // initial state, table.py:143-149 / store.py:36-37
  // keys EMPTY, scores 0: the two halves of every 16-B pair
  if ((e = cudaMemset2D(t->ks, 16, 0xFF, 8, cap)) || (e = cudaMemset2D(t->ks + 1, 16, 0, 8, cap)) ||
      (e = cudaMemset(t->digests, 0, cap)) || (e = cudaMemset(t->bits, 0, (size_t)bc * 16)) ||
      (e = cudaMemset(t->smin, 0, (size_t)bc * 64)) || (e = cudaMemset(t->svalid, 0, (size_t)bc * 4)) ||
      (e = cudaMemset(t->sc, 0, sizeof(TableScalars))) || (e = cudaMemset(t->role_word, 0, 4)) ||
      (t->vfast && (e = cudaMemset(t->vfast, 0, t->fast_rows * dim * 4))) ||
      (t->vover && (e = cudaMemset(t->vover, 0, over_rows * dim * 4))) ||
      (t->lead && (e = cudaMemset(t->lead, 0, (size_t)bc * 8)))) {
    free_table(t);
    return cuda_fail(e, "hkv_create init");
  }
  if ((e = cudaDeviceSynchronize())) {
    free_table(t);
    return cuda_fail(e, "hkv_create sync");
  }
  TableDev& d = t->dev;
  d.ks = t->ks;
  d.digests = t->digests;
  d.bits = t->bits;
  d.smin = t->smin;
  d.svalid = t->svalid;
  d.vfast = t->vfast;
  d.vover = t->vover;
  d.fast_rows = t->fast_rows;
  d.mask = (uint64_t)(bc - 1);
  d.capacity = cap;
  d.dim = (int)c.value_dim;
  d.dual = c.mode == HKV_MODE_DUAL;
  d.policy = c.score_policy;
  d.digest_filter = c.digest_filter;
  d.admit_unified = c.admit_ties_unified;
  d.size = &t->sc->size;
  d.clock = &t->sc->clock;
  d.counters = t->sc->counters;
  d.err = &t->sc->err;
  d.fel_set = &t->sc->fel_set;
  d.fel = &t->sc->fel;
  d.role_word = t->role_word;
  d.cas = c.workers > 1;
  d.locks = t->locks;
  t->gate = gate_new_device(c.device, t->role_word);
  *out = t;
  return HKV_OK;
}

int hkv_set_workers(hkv_table* t, int32_t workers) {
  if (!t) return fail(HKV_EINVAL, "null table");
  if (workers < 1) return fail(HKV_EINVAL, "workers must be >= 1");
  DeviceGuard _g(t->cfg.device);
  // an engine switch is a structural event: no batch of either engine may be in flight
  GateScope _gs(t->gate, HKV_ROLE_INSERTER, (cudaStream_t)0);
  if (_gs.rc) return gate_fail(_gs.rc);
  cudaError_t e = cudaSuccess;
  if (workers > 1 && !t->locks) {
    if ((e = cudaMalloc((void**)&t->locks, (size_t)t->buckets * 4)) ||
        (e = cudaMemset(t->locks, 0, (size_t)t->buckets * 4)) || (e = cudaDeviceSynchronize()))
      return fail(HKV_ENOMEM, "bucket lock allocation failed");
  }
  t->cfg.workers = workers;
  t->dev.cas = workers > 1;
  t->dev.locks = t->locks;
  return HKV_OK;
}

int hkv_table_gate(hkv_table* t, hkv_gate** out) {
  if (!t || !out) return fail(HKV_EINVAL, "null argument");
  *out = t->gate;
  return HKV_OK;
}

int hkv_destroy(hkv_table* t) {
  if (!t) return HKV_OK;
  {
    DeviceGuard g(t->cfg.device);
    cudaDeviceSynchronize();
  }
  free_table(t);
  return HKV_OK;
}

// mutation batches index ops with uint32 and hand (int)n to CUB: cap them
#define CHECK_MUT_N() \
  if (n > 0x7FFFFFFFll) return fail(HKV_EINVAL, "batch too large (at most 2^31-1 keys per mutation call)")

#define CHECK_T()                                   \
  if (!t) return fail(HKV_EINVAL, "null table");    \
  if (n < 0) return fail(HKV_EINVAL, "negative batch size"); \
  DeviceGuard _g(t->cfg.device)

int hkv_find(hkv_table* t, const uint64_t* keys, int64_t n, float* out, uint8_t* found, int32_t zero_misses,
             hkv_stream stream) {
  CHECK_T();
  if (n && (!keys || !found)) return fail(HKV_EINVAL, "null keys/found");
  GateScope _gs(t->gate, HKV_ROLE_READER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  uint32_t* rows = nullptr;
  auto lease = t->workspace((cudaStream_t)stream);
  if (out && n > 0) {
    Workspace& ws = lease.w;
    cudaError_t e0 = ws_reserve(ws, n, (int)t->cfg.value_dim, 0, false);
    if (e0) return cuda_fail(e0, "hkv_find workspace");
    rows = ws.vrow;
  }
  launch_find(t->dev, keys, n, out, found, nullptr, nullptr, out ? (zero_misses ? 3 : 0) : 1, rows,
              (cudaStream_t)stream, t->num_sms);
  cudaError_t e = cudaGetLastError();
  return e ? cuda_fail(e, "hkv_find") : HKV_OK;
}

int hkv_contains(hkv_table* t, const uint64_t* keys, int64_t n, uint8_t* found, hkv_stream stream) {
  CHECK_T();
  if (n && (!keys || !found)) return fail(HKV_EINVAL, "null keys/found");
  GateScope _gs(t->gate, HKV_ROLE_READER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  launch_find(t->dev, keys, n, nullptr, found, nullptr, nullptr, 1, nullptr, (cudaStream_t)stream, t->num_sms);
  cudaError_t e = cudaGetLastError();
  return e ? cuda_fail(e, "hkv_contains") : HKV_OK;
}

int hkv_find_ptr(hkv_table* t, const uint64_t* keys, int64_t n, uint8_t* found, uint8_t* tier, int64_t* offset,
                 hkv_stream stream) {
  CHECK_T();
  if (n && (!keys || !found || !tier || !offset)) return fail(HKV_EINVAL, "null argument");
  GateScope _gs(t->gate, HKV_ROLE_READER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  launch_find(t->dev, keys, n, nullptr, found, tier, offset, 2, nullptr, (cudaStream_t)stream, t->num_sms);
  cudaError_t e = cudaGetLastError();
  return e ? cuda_fail(e, "hkv_find_ptr") : HKV_OK;
}

int hkv_upsert(hkv_table* t, int32_t op, const uint64_t* keys, float* values, const uint64_t* scores, int64_t n,
               uint8_t* outcomes, uint64_t* evicted_keys, float* evicted_values, uint64_t* evicted_scores,
               int64_t* n_evicted_dev, const uint64_t* ticks, uint64_t clock_advance, hkv_stream stream) {
  CHECK_T();
  if (op != HKV_OP_INSERT_OR_ASSIGN && op != HKV_OP_FIND_OR_INSERT) return fail(HKV_EINVAL, "unknown upsert op");
  // table.py:178-188
  const bool custom = t->cfg.score_policy == HKV_CUSTOMIZED;
  if (custom && !scores) return fail(HKV_EINVAL, "kCustomized requires explicit scores");
  if (!custom && scores) return fail(HKV_EINVAL, "explicit scores require the kCustomized policy");
  if (n && (!keys || !values || !outcomes)) return fail(HKV_EINVAL, "null keys/values/outcomes");
  const bool collect = evicted_keys || evicted_values || evicted_scores;
  if (collect && (!evicted_keys || !evicted_values || !evicted_scores || !n_evicted_dev))
    return fail(HKV_EINVAL, "insert_and_evict needs all evicted outputs");
  if (collect && op != HKV_OP_INSERT_OR_ASSIGN) return fail(HKV_EINVAL, "evicted outputs need insert_or_assign");
  CHECK_MUT_N();
  GateScope _gs(t->gate, HKV_ROLE_INSERTER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  cudaStream_t s = (cudaStream_t)stream;
  OpArgs a{};
  a.keys = keys;
  a.values = values;
  a.scores = scores;
  a.ticks = ticks;
  a.outcomes = outcomes;
  a.op = op == HKV_OP_FIND_OR_INSERT ? kOpFindOrInsert : kOpUpsert;
  a.collect = collect;
  a.epoch = t->epoch;
  cudaError_t e = run_mutation(t->dev, a, n, t->log2b, t->workspace(s), (++t->dual_epoch) << 32, t->lead, n_evicted_dev,
                               evicted_keys, evicted_values, evicted_scores, ticks ? clock_advance : (uint64_t)n,
                               s, t->num_sms);
  return e ? cuda_fail(e, "hkv_upsert") : HKV_OK;
}

// Host-buffer find: chunks of keys go H2D, are probed into a ring slot, and
// the slot's found bytes and rows come back D2H on the copy stream while the
// next chunk is probed.  A caller `out` with zero_misses == 0 keeps its miss
// rows: the chunk's rows go H2D first (the PCIe link is full duplex, so this
// rides beside the previous chunk's D2H).
int hkv_find_host(hkv_table* t, const uint64_t* keys, int64_t n, float* out, uint8_t* found, int32_t zero_misses,
                  hkv_stream stream) {
  CHECK_T();
  if (n && (!keys || !found)) return fail(HKV_EINVAL, "null keys/found");
  if (n == 0) return HKV_OK;
  GateScope _gs(t->gate, HKV_ROLE_READER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  cudaStream_t s = (cudaStream_t)stream;
  HostStage& h = t->stage(s);
  std::lock_guard<std::mutex> hold(h.mu);
  cudaError_t e = h.init();
  if (e) return cuda_fail(e, "hkv_find_host init");
  const int64_t dim = t->cfg.value_dim;
  int64_t chunk = out ? ((int64_t)16 << 20) / (dim * 4) : n;  // ~16 MB of rows per slot
  if (chunk < 4096) chunk = 4096;
  if (chunk > n) chunk = n;
  if ((e = grow_dev(h.keys, h.keys_cap, (size_t)(kRing * chunk)))) return cuda_fail(e, "hkv_find_host staging");
  if ((e = grow_dev(h.bytes, h.bytes_cap, (size_t)(kRing * chunk)))) return cuda_fail(e, "hkv_find_host staging");
  if (out && (e = grow_dev(h.rows, h.rows_cap, (size_t)(kRing * chunk * dim))))
    return cuda_fail(e, "hkv_find_host staging");
  auto lease = t->workspace(s);
  Workspace& ws = lease.w;
  if (out && (e = ws_reserve(ws, chunk, (int)dim, 0, false))) return cuda_fail(e, "hkv_find_host workspace");
  if ((e = cudaEventRecord(h.start, s)) || (e = cudaStreamWaitEvent(h.copy, h.start, 0)))
    return cuda_fail(e, "hkv_find_host");
  const int64_t nchunks = (n + chunk - 1) / chunk;
  for (int64_t c = 0; c < nchunks; c++) {
    const int slot = (int)(c % kRing);
    const int64_t off = c * chunk, cnt = (n - off < chunk) ? n - off : chunk;
    uint64_t* dk = h.keys + (size_t)slot * chunk;
    uint8_t* df = h.bytes + (size_t)slot * chunk;
    float* dr = out ? h.rows + (size_t)slot * chunk * dim : nullptr;
    if (c >= kRing && (e = cudaStreamWaitEvent(s, h.done[slot], 0))) break;
    if ((e = cudaMemcpyAsync(dk, keys + off, cnt * 8, cudaMemcpyHostToDevice, s))) break;
    if (out && !zero_misses &&
        (e = cudaMemcpyAsync(dr, out + off * dim, cnt * dim * 4, cudaMemcpyHostToDevice, s)))
      break;
    launch_find(t->dev, dk, cnt, dr, df, nullptr, nullptr, out ? (zero_misses ? 3 : 0) : 1, out ? ws.vrow : nullptr,
                s, t->num_sms);
    if ((e = cudaGetLastError())) break;
    if ((e = cudaEventRecord(h.ready[slot], s)) || (e = cudaStreamWaitEvent(h.copy, h.ready[slot], 0))) break;
    if ((e = cudaMemcpyAsync(found + off, df, cnt, cudaMemcpyDeviceToHost, h.copy))) break;
    if (out && (e = cudaMemcpyAsync(out + off * dim, dr, cnt * dim * 4, cudaMemcpyDeviceToHost, h.copy))) break;
    if ((e = cudaEventRecord(h.done[slot], h.copy))) break;
  }
  cudaError_t e2 = cudaEventRecord(h.vals, h.copy);
  if (!e2) e2 = cudaStreamWaitEvent(s, h.vals, 0);
  if (!e2) e2 = cudaStreamSynchronize(s);
  if (e || e2) return cuda_fail(e ? e : e2, "hkv_find_host");
  return HKV_OK;
}

// Host-buffer upsert: keys (and scores / ticks) go H2D on the caller's stream
// and the metadata pass starts at once; the value rows go H2D on the copy
// stream in parallel, and run_mutation holds the value phase until they land.
int hkv_upsert_host(hkv_table* t, int32_t op, const uint64_t* keys, float* values, const uint64_t* scores, int64_t n,
                    uint8_t* outcomes, const uint64_t* ticks, uint64_t clock_advance, hkv_stream stream) {
  CHECK_T();
  if (op != HKV_OP_INSERT_OR_ASSIGN && op != HKV_OP_FIND_OR_INSERT) return fail(HKV_EINVAL, "unknown upsert op");
  const bool custom = t->cfg.score_policy == HKV_CUSTOMIZED;
  if (custom && !scores) return fail(HKV_EINVAL, "kCustomized requires explicit scores");
  if (!custom && scores) return fail(HKV_EINVAL, "explicit scores require the kCustomized policy");
  if (n && (!keys || !values || !outcomes)) return fail(HKV_EINVAL, "null keys/values/outcomes");
  CHECK_MUT_N();
  GateScope _gs(t->gate, HKV_ROLE_INSERTER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  cudaStream_t s = (cudaStream_t)stream;
  HostStage& h = t->stage(s);
  std::lock_guard<std::mutex> hold(h.mu);
  cudaError_t e = h.init();
  if (e) return cuda_fail(e, "hkv_upsert_host init");
  const int64_t dim = t->cfg.value_dim;
  const size_t nn = n > 0 ? (size_t)n : 1;
  if ((e = grow_dev(h.keys, h.keys_cap, nn)) || (e = grow_dev(h.bytes, h.bytes_cap, nn)) ||
      (e = grow_dev(h.rows, h.rows_cap, nn * dim)) || (e = grow_dev(h.aux, h.aux_cap, 2 * nn)))
    return cuda_fail(e, "hkv_upsert_host staging");
  uint64_t* dscores = scores ? h.aux : nullptr;
  uint64_t* dticks = ticks ? h.aux + nn : nullptr;
  if (n > 0) {
    if ((e = cudaEventRecord(h.start, s)) || (e = cudaStreamWaitEvent(h.copy, h.start, 0)) ||
        (e = cudaMemcpyAsync(h.keys, keys, n * 8, cudaMemcpyHostToDevice, s)) ||
        (scores && (e = cudaMemcpyAsync(dscores, scores, n * 8, cudaMemcpyHostToDevice, s))) ||
        (ticks && (e = cudaMemcpyAsync(dticks, ticks, n * 8, cudaMemcpyHostToDevice, s))) ||
        (e = cudaMemcpyAsync(h.rows, values, n * dim * 4, cudaMemcpyHostToDevice, h.copy)) ||
        (e = cudaEventRecord(h.vals, h.copy)))
      return cuda_fail(e, "hkv_upsert_host copy-in");
  }
  OpArgs a{};
  a.keys = h.keys;
  a.values = h.rows;
  a.scores = dscores;
  a.ticks = dticks;
  a.outcomes = h.bytes;
  a.op = op == HKV_OP_FIND_OR_INSERT ? kOpFindOrInsert : kOpUpsert;
  a.collect = 0;
  a.epoch = t->epoch;
  e = run_mutation(t->dev, a, n, t->log2b, t->workspace(s), (++t->dual_epoch) << 32, t->lead, nullptr, nullptr,
                   nullptr, nullptr, ticks ? clock_advance : (uint64_t)n, s, t->num_sms, n > 0 ? h.vals : nullptr);
  if (e) return cuda_fail(e, "hkv_upsert_host");
  if (n > 0) {
    if ((e = cudaMemcpyAsync(outcomes, h.bytes, n, cudaMemcpyDeviceToHost, s))) return cuda_fail(e, "hkv_upsert_host");
    if (op == HKV_OP_FIND_OR_INSERT &&
        (e = cudaMemcpyAsync(values, h.rows, n * dim * 4, cudaMemcpyDeviceToHost, s)))
      return cuda_fail(e, "hkv_upsert_host");
  }
  if ((e = cudaStreamSynchronize(s))) return cuda_fail(e, "hkv_upsert_host");
  return HKV_OK;
}

// ---- sharded find over peer memory ----------------------------------------
static int peer_ready(hkv_table* t) {
  if (t->cfg.mode != HKV_MODE_SINGLE) return fail(HKV_EINVAL, "peer find needs single mode");
  if (!t->cfg.digest_filter) return fail(HKV_EINVAL, "peer find needs digest_filter");
  if (t->fast_rows != (uint64_t)t->cfg.capacity)
    return fail(HKV_EINVAL, "peer find needs every value row in HBM (fast_tier_budget == buckets)");
  return HKV_OK;
}

static int install_peers(hkv_table* t, int world, const std::vector<PeerView>& v) {
  if (t->peers_dev) cudaFree(t->peers_dev);
  t->peers_dev = nullptr;
  cudaError_t e = cudaMalloc((void**)&t->peers_dev, sizeof(PeerView) * (size_t)world);
  if (!e) e = cudaMemcpy(t->peers_dev, v.data(), sizeof(PeerView) * (size_t)world, cudaMemcpyHostToDevice);
  if (e) return cuda_fail(e, "hkv_set_peers");
  t->peer_world = world;
  t->peer_llog2b = t->log2b;
  return HKV_OK;
}

int hkv_ipc_handles(hkv_table* t, void* out, int64_t out_bytes) {
  if (!t || !out) return fail(HKV_EINVAL, "null argument");
  if (out_bytes < 3 * (int64_t)sizeof(cudaIpcMemHandle_t)) return fail(HKV_EINVAL, "handle buffer too small");
  if (int rc = peer_ready(t)) return rc;
  DeviceGuard _g(t->cfg.device);
  cudaIpcMemHandle_t* h = reinterpret_cast<cudaIpcMemHandle_t*>(out);
  cudaError_t e;
  if ((e = cudaIpcGetMemHandle(&h[0], t->ks)) || (e = cudaIpcGetMemHandle(&h[1], t->digests)) ||
      (e = cudaIpcGetMemHandle(&h[2], t->vfast)))
    return cuda_fail(e, "hkv_ipc_handles");
  return HKV_OK;
}

int hkv_set_peers(hkv_table* t, int32_t world, int32_t rank, const void* handles) {
  if (!t || !handles || world < 1 || rank < 0 || rank >= world || (world & (world - 1)))
    return fail(HKV_EINVAL, "bad peer arguments (world must be a power of two)");
  if (int rc = peer_ready(t)) return rc;
  DeviceGuard _g(t->cfg.device);
  const cudaIpcMemHandle_t* h = reinterpret_cast<const cudaIpcMemHandle_t*>(handles);
  std::vector<PeerView> v((size_t)world);
  for (int r = 0; r < world; r++) {
    if (r == rank) {
      v[r] = PeerView{t->ks, t->digests, t->vfast};
      continue;
    }
    void* p[3];
    for (int k = 0; k < 3; k++) {
      cudaError_t e = cudaIpcOpenMemHandle(&p[k], h[3 * r + k], cudaIpcMemLazyEnablePeerAccess);
      if (e) return cuda_fail(e, "hkv_set_peers: cudaIpcOpenMemHandle");
      t->ipc_opened.push_back(p[k]);
    }
    v[r] = PeerView{(const uint64_t*)p[0], (const uint8_t*)p[1], (const float*)p[2]};
  }
  return install_peers(t, world, v);
}

int hkv_set_peers_local(hkv_table* t, int32_t world, hkv_table* const* shards) {
  if (!t || !shards || world < 1 || (world & (world - 1))) return fail(HKV_EINVAL, "bad peer arguments");
  if (int rc = peer_ready(t)) return rc;
  DeviceGuard _g(t->cfg.device);
  std::vector<PeerView> v((size_t)world);
  for (int r = 0; r < world; r++) {
    hkv_table* o = shards[r];
    if (!o || o->cfg.capacity != t->cfg.capacity || o->cfg.value_dim != t->cfg.value_dim)
      return fail(HKV_EINVAL, "shards must share capacity and value_dim");
    if (int rc = peer_ready(o)) return rc;
    if (o->cfg.device != t->cfg.device) {
      cudaError_t e = cudaDeviceEnablePeerAccess(o->cfg.device, 0);
      if (e && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "hkv_set_peers_local: peer access");
      cudaGetLastError();
    }
    v[r] = PeerView{o->ks, o->digests, o->vfast};
  }
  return install_peers(t, world, v);
}

int hkv_find_peer(hkv_table* t, const uint64_t* keys, int64_t n, float* out, uint8_t* found, int32_t zero_misses,
                  hkv_stream stream) {
  CHECK_T();
  if (!t->peers_dev) return fail(HKV_EINVAL, "no peers set (hkv_set_peers)");
  if (n && (!keys || !found || !out)) return fail(HKV_EINVAL, "null keys/out/found");
  GateScope _gs(t->gate, HKV_ROLE_READER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  const uint64_t gmask = ((uint64_t)t->buckets * (uint64_t)t->peer_world) - 1;
  launch_find_peer(t->peers_dev, gmask, t->peer_llog2b, (int)t->cfg.value_dim, keys, n, out, found, zero_misses,
                   t->dev.err, (cudaStream_t)stream, t->num_sms);
  cudaError_t e = cudaGetLastError();
  return e ? cuda_fail(e, "hkv_find_peer") : HKV_OK;
}

// ---- single-key API -------------------------------------------------------
static int one_ready(hkv_table* t) {
  cudaError_t e = cudaSuccess;
  if (!t->one && !(e = cudaMalloc((void**)&t->one, sizeof(OneResult)))) e = cudaMemset(t->one, 0, sizeof(OneResult));
  if (!e && !t->one_val) e = cudaMalloc((void**)&t->one_val, (size_t)t->cfg.value_dim * 4);
  return e ? cuda_fail(e, "single-key staging") : HKV_OK;
}

static int one_finish(hkv_table* t, hkv_one_result* result, cudaStream_t s, const char* where) {
  OneResult h;
  cudaError_t e = cudaMemcpyAsync(&h, t->one, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (e) return cuda_fail(e, where);
  if (h.status == 1) return fail(HKV_EINVAL, "kCustomized requires an explicit score");
  if (h.status == 2) return fail(HKV_EINVAL, "explicit scores require the kCustomized policy");
  result->kind = h.kind;
  result->slot = h.slot;
  result->bucket = h.bucket;
  result->evicted_key = h.evicted_key;
  result->evicted_score = h.evicted_score;
  return HKV_OK;
}

static int lookup_one(hkv_table* t, int64_t bucket, uint64_t key, hkv_one_result* result, hkv_stream stream) {
  if (!t || !result) return fail(HKV_EINVAL, "null argument");
  DeviceGuard _g(t->cfg.device);
  if (bucket >= t->buckets) return fail(HKV_EINVAL, "bucket index out of range");
  cudaStream_t s = (cudaStream_t)stream;
  GateScope _gs(t->gate, HKV_ROLE_READER, s);
  if (_gs.rc) return gate_fail(_gs.rc);
  if (int rc = one_ready(t)) return rc;
  launch_lookup_one(t->dev, key, bucket, t->one, s);
  return one_finish(t, result, s, "hkv_lookup");
}

int hkv_lookup(hkv_table* t, uint64_t key, hkv_one_result* result, hkv_stream stream) {
  return lookup_one(t, -1, key, result, stream);
}

int hkv_find_in_bucket(hkv_table* t, int64_t bucket, uint64_t key, hkv_one_result* result, hkv_stream stream) {
  if (bucket < 0) return fail(HKV_EINVAL, "bucket index out of range");
  return lookup_one(t, bucket, key, result, stream);
}

static int upsert_one(hkv_table* t, int dual, uint64_t key, const float* value, int32_t has_score, uint64_t score,
                      hkv_one_result* result, hkv_stream stream) {
  if (!t || !value || !result) return fail(HKV_EINVAL, "null argument");
  if (dual && t->cfg.mode != HKV_MODE_DUAL) return fail(HKV_EINVAL, "upsert_dual requires dual mode");
  if (key >= 0xFFFFFFFFFFFFFFFEull) return fail(HKV_EINVAL, "keys must not equal a reserved sentinel value");
  DeviceGuard _g(t->cfg.device);
  cudaStream_t s = (cudaStream_t)stream;
  GateScope _gs(t->gate, HKV_ROLE_INSERTER, s);
  if (_gs.rc) return gate_fail(_gs.rc);
  if (int rc = one_ready(t)) return rc;
  cudaError_t e = cudaMemcpyAsync(t->one_val, value, (size_t)t->cfg.value_dim * 4, cudaMemcpyDefault, s);
  if (e) return cuda_fail(e, "single-key value");
  launch_upsert_one(t->dev, key, t->one_val, dual, has_score != 0, score, t->epoch, t->one, s);
  return one_finish(t, result, s, dual ? "hkv_upsert_dual" : "hkv_upsert_single");
}

int hkv_upsert_single(hkv_table* t, uint64_t key, const float* value, int32_t has_score, uint64_t score,
                      hkv_one_result* result, hkv_stream stream) {
  return upsert_one(t, 0, key, value, has_score, score, result, stream);
}

int hkv_upsert_dual(hkv_table* t, uint64_t key, const float* value, int32_t has_score, uint64_t score,
                    hkv_one_result* result, hkv_stream stream) {
  return upsert_one(t, 1, key, value, has_score, score, result, stream);
}

int hkv_erase(hkv_table* t, const uint64_t* keys, int64_t n, uint8_t* outcomes, hkv_stream stream) {
  CHECK_T();
  if (n && (!keys || !outcomes)) return fail(HKV_EINVAL, "null keys/outcomes");
  CHECK_MUT_N();
  GateScope _gs(t->gate, HKV_ROLE_INSERTER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  cudaStream_t s = (cudaStream_t)stream;
  OpArgs a{};
  a.keys = keys;
  a.outcomes = outcomes;
  a.op = kOpErase;
  a.epoch = t->epoch;
  a.values = nullptr;
  cudaError_t e = run_mutation(t->dev, a, n, t->log2b, t->workspace(s), (++t->dual_epoch) << 32, t->lead, nullptr, nullptr,
                               nullptr, nullptr, 0, s, t->num_sms);
  return e ? cuda_fail(e, "hkv_erase") : HKV_OK;
}

int hkv_assign(hkv_table* t, const uint64_t* keys, const float* values, const uint64_t* scores, int32_t refresh,
               int64_t n, uint8_t* outcomes, const uint64_t* ticks, uint64_t clock_advance, hkv_stream stream) {
  CHECK_T();
  const bool custom = t->cfg.score_policy == HKV_CUSTOMIZED;
  if (!values) {
    // assign_scores (table.py:444-449 -> _coerce_scores 178-188)
    if (!scores && custom) return fail(HKV_EINVAL, "kCustomized requires explicit scores");
    if (scores && !custom) return fail(HKV_EINVAL, "explicit scores require the kCustomized policy");
    if (!scores) refresh = 1;
  } else {
    refresh = 0;
  }
  if (n && (!keys || !outcomes)) return fail(HKV_EINVAL, "null keys/outcomes");
  CHECK_MUT_N();
  GateScope _gs(t->gate, HKV_ROLE_UPDATER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = run_assign(t->dev, keys, values, scores, refresh, t->epoch, n, outcomes, ticks, clock_advance,
                             t->log2b, t->workspace(s), s, t->num_sms);
  return e ? cuda_fail(e, "hkv_assign") : HKV_OK;
}

int hkv_export(hkv_table* t, int64_t cursor, int64_t max_count, int32_t has_min_score, uint64_t min_score,
               const uint8_t* row_mask, int64_t mask_rows, uint64_t* out_keys, float* out_values,
               uint64_t* out_scores, int64_t* count, int64_t* next_cursor, hkv_stream stream) {
  if (!t) return fail(HKV_EINVAL, "null table");
  DeviceGuard _g(t->cfg.device);
  // table.py:386-391
  if (cursor < 0 || cursor >= t->cfg.capacity) return fail(HKV_EINVAL, "cursor out of range");
  if (max_count < 1) return fail(HKV_EINVAL, "max_count must be >= 1");
  if (!count || !next_cursor || !out_keys || !out_values || !out_scores) return fail(HKV_EINVAL, "null output");
  if (row_mask && (mask_rows < 0 || cursor + mask_rows > t->cfg.capacity)) return fail(HKV_EINVAL, "mask range");
  GateScope _gs(t->gate, HKV_ROLE_READER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = run_export(t->dev, cursor, max_count, has_min_score, min_score, row_mask, mask_rows, out_keys,
                             out_values, out_scores, count, next_cursor, t->workspace(s), s, t->num_sms);
  return e ? cuda_fail(e, "hkv_export") : HKV_OK;
}

static int read_scalars(hkv_table* t, TableScalars* h, hkv_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(h, t->sc, sizeof(TableScalars), cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  return e ? cuda_fail(e, "read scalars") : HKV_OK;
}

int hkv_size(hkv_table* t, int64_t* size, hkv_stream stream) {
  if (!t || !size) return fail(HKV_EINVAL, "null argument");
  DeviceGuard _g(t->cfg.device);
  GateScope _gs(t->gate, HKV_ROLE_READER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  TableScalars h;
  int rc = read_scalars(t, &h, stream);
  if (rc) return rc;
  *size = (int64_t)h.size;
  return HKV_OK;
}

int hkv_set_epoch(hkv_table* t, uint64_t epoch) {
  if (!t) return fail(HKV_EINVAL, "null table");
  // scoring.py:45-50
  if (epoch < t->epoch) return fail(HKV_EINVAL, "epoch may not decrease");
  if (epoch > 0xFFFFFFFFull) return fail(HKV_EINVAL, "epoch must fit in 32 bits");
  t->epoch = epoch;
  return HKV_OK;
}

int hkv_get_epoch(hkv_table* t, uint64_t* epoch) {
  if (!t || !epoch) return fail(HKV_EINVAL, "null argument");
  *epoch = t->epoch;
  return HKV_OK;
}

int hkv_clock(hkv_table* t, uint64_t* clock, hkv_stream stream) {
  if (!t || !clock) return fail(HKV_EINVAL, "null argument");
  DeviceGuard _g(t->cfg.device);
  TableScalars h;
  int rc = read_scalars(t, &h, stream);
  if (rc) return rc;
  *clock = h.clock;
  return HKV_OK;
}

int hkv_first_eviction_lambda(hkv_table* t, int32_t* is_set, double* value, hkv_stream stream) {
  if (!t || !is_set || !value) return fail(HKV_EINVAL, "null argument");
  DeviceGuard _g(t->cfg.device);
  TableScalars h;
  int rc = read_scalars(t, &h, stream);
  if (rc) return rc;
  *is_set = h.fel_set;
  *value = h.fel;
  return HKV_OK;
}

int hkv_counters(hkv_table* t, int64_t* out, hkv_stream stream) {
  if (!t || !out) return fail(HKV_EINVAL, "null argument");
  DeviceGuard _g(t->cfg.device);
  TableScalars h;
  int rc = read_scalars(t, &h, stream);
  if (rc) return rc;
  for (int k = 0; k < HKV_NUM_COUNTERS; k++) out[k] = (int64_t)h.counters[k];
  return HKV_OK;
}

int hkv_reset_counters(hkv_table* t, hkv_stream stream) {
  if (!t) return fail(HKV_EINVAL, "null table");
  DeviceGuard _g(t->cfg.device);
  cudaError_t e = cudaMemsetAsync(t->sc->counters, 0, sizeof(t->sc->counters), (cudaStream_t)stream);
  return e ? cuda_fail(e, "reset counters") : HKV_OK;
}

int hkv_device_error(hkv_table* t, int32_t* bits, hkv_stream stream) {
  if (!t || !bits) return fail(HKV_EINVAL, "null argument");
  DeviceGuard _g(t->cfg.device);
  cudaStream_t s = (cudaStream_t)stream;
  int v = 0;
  cudaError_t e = cudaMemcpyAsync(&v, &t->sc->err, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaMemsetAsync(&t->sc->err, 0, sizeof(int), s);
  if (!e) e = cudaStreamSynchronize(s);
  if (e) return cuda_fail(e, "device error");
  *bits = v;
  return HKV_OK;
}

int hkv_import_state(hkv_table* t, const uint64_t* keys, const uint8_t* digests, const uint64_t* scores,
                     const float* values, uint64_t clock, int32_t fel_set, double fel) {
  if (!t || !keys || !digests || !scores || !values) return fail(HKV_EINVAL, "null argument");
  DeviceGuard _g(t->cfg.device);
  GateScope _gs(t->gate, HKV_ROLE_INSERTER, (cudaStream_t)0);
  if (_gs.rc) return gate_fail(_gs.rc);
  const uint64_t cap = (uint64_t)t->cfg.capacity, dim = (uint64_t)t->cfg.value_dim;
  cudaError_t e;
  if ((e = cudaMemcpy2D(t->ks, 16, keys, 8, 8, cap, cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(t->digests, digests, cap, cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy2D(t->ks + 1, 16, scores, 8, 8, cap, cudaMemcpyHostToDevice)))
    return cuda_fail(e, "import metadata");
  if (t->fast_rows && (e = cudaMemcpy(t->vfast, values, t->fast_rows * dim * 4, cudaMemcpyHostToDevice)))
    return cuda_fail(e, "import values");
  if (cap > t->fast_rows &&
      (e = cudaMemcpy(t->vover, values + t->fast_rows * dim, (cap - t->fast_rows) * dim * 4, cudaMemcpyDefault)))
    return cuda_fail(e, "import overflow values");
  if ((e = run_bits_from_keys(t->dev, t->buckets, 0))) return cuda_fail(e, "import bits");
  if ((e = cudaMemset(t->svalid, 0, (size_t)t->buckets * 4))) return cuda_fail(e, "import summary");
  TableScalars h;
  if ((e = cudaMemcpy(&h, t->sc, sizeof(h), cudaMemcpyDeviceToHost))) return cuda_fail(e, "import scalars");
  h.clock = clock;
  h.fel_set = fel_set;
  h.fel = fel;
  if ((e = cudaMemcpy(t->sc, &h, sizeof(h), cudaMemcpyHostToDevice))) return cuda_fail(e, "import scalars");
  e = cudaDeviceSynchronize();
  return e ? cuda_fail(e, "import sync") : HKV_OK;
}

int hkv_export_state(hkv_table* t, uint64_t* keys, uint8_t* digests, uint64_t* scores, float* values,
                     int64_t* occupancy) {
  if (!t) return fail(HKV_EINVAL, "null table");
  DeviceGuard _g(t->cfg.device);
  GateScope _gs(t->gate, HKV_ROLE_READER, (cudaStream_t)0);
  if (_gs.rc) return gate_fail(_gs.rc);
  const uint64_t cap = (uint64_t)t->cfg.capacity, dim = (uint64_t)t->cfg.value_dim;
  cudaError_t e = cudaDeviceSynchronize();
  if (e) return cuda_fail(e, "export sync");
  if (keys && (e = cudaMemcpy2D(keys, 8, t->ks, 16, 8, cap, cudaMemcpyDeviceToHost))) return cuda_fail(e, "export keys");
  if (digests && (e = cudaMemcpy(digests, t->digests, cap, cudaMemcpyDeviceToHost))) return cuda_fail(e, "export");
  if (scores && (e = cudaMemcpy2D(scores, 8, t->ks + 1, 16, 8, cap, cudaMemcpyDeviceToHost))) return cuda_fail(e, "export");
  if (values) {
    if (t->fast_rows && (e = cudaMemcpy(values, t->vfast, t->fast_rows * dim * 4, cudaMemcpyDeviceToHost)))
      return cuda_fail(e, "export values");
    if (cap > t->fast_rows &&
        (e = cudaMemcpy(values + t->fast_rows * dim, t->vover, (cap - t->fast_rows) * dim * 4, cudaMemcpyDefault)))
      return cuda_fail(e, "export overflow values");
  }
  if (occupancy) {
    uint32_t* hb = (uint32_t*)malloc((size_t)t->buckets * 16);
    if (!hb) return fail(HKV_ENOMEM, "host alloc");
    if ((e = cudaMemcpy(hb, t->bits, (size_t)t->buckets * 16, cudaMemcpyDeviceToHost))) {
      free(hb);
      return cuda_fail(e, "export bits");
    }
    for (int64_t b = 0; b < t->buckets; b++)
      occupancy[b] = __builtin_popcount(hb[4 * b]) + __builtin_popcount(hb[4 * b + 1]) +
                     __builtin_popcount(hb[4 * b + 2]) + __builtin_popcount(hb[4 * b + 3]);
    free(hb);
  }
  return HKV_OK;
}

int hkv_read_rows(hkv_table* t, int64_t row0, int64_t nrows, uint64_t* keys, uint64_t* scores, hkv_stream stream) {
  if (!t) return fail(HKV_EINVAL, "null table");
  if (row0 < 0 || nrows < 0 || row0 + nrows > t->cfg.capacity) return fail(HKV_EINVAL, "row range out of bounds");
  DeviceGuard _g(t->cfg.device);
  GateScope _gs(t->gate, HKV_ROLE_READER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  if (keys && nrows) e = cudaMemcpy2DAsync(keys, 8, t->ks + 2 * row0, 16, 8, (size_t)nrows, cudaMemcpyDefault, s);
  if (!e && scores && nrows)
    e = cudaMemcpy2DAsync(scores, 8, t->ks + 2 * row0 + 1, 16, 8, (size_t)nrows, cudaMemcpyDefault, s);
  if (!e) e = cudaStreamSynchronize(s);
  return e ? cuda_fail(e, "hkv_read_rows") : HKV_OK;
}

int hkv_read_value_rows(hkv_table* t, int64_t row0, int64_t nrows, float* out, hkv_stream stream) {
  if (!t || (nrows && !out)) return fail(HKV_EINVAL, "null argument");
  if (row0 < 0 || nrows < 0 || row0 + nrows > t->cfg.capacity) return fail(HKV_EINVAL, "row range out of bounds");
  DeviceGuard _g(t->cfg.device);
  cudaStream_t s = (cudaStream_t)stream;
  GateScope _gs(t->gate, HKV_ROLE_READER, s);
  if (_gs.rc) return gate_fail(_gs.rc);
  const uint64_t dim = (uint64_t)t->cfg.value_dim;
  cudaError_t e = cudaSuccess;
  for (int64_t r = row0; r < row0 + nrows && !e;) {  // a range may straddle the tier boundary
    const bool fast = (uint64_t)r < t->fast_rows;
    const int64_t end = fast ? std::min<int64_t>(row0 + nrows, (int64_t)t->fast_rows) : row0 + nrows;
    const float* src = fast ? t->vfast + (uint64_t)r * dim : t->vover + ((uint64_t)r - t->fast_rows) * dim;
    e = cudaMemcpyAsync(out + (uint64_t)(r - row0) * dim, src, (size_t)(end - r) * dim * 4, cudaMemcpyDefault, s);
    r = end;
  }
  if (!e) e = cudaStreamSynchronize(s);
  return e ? cuda_fail(e, "hkv_read_value_rows") : HKV_OK;
}

int hkv_snapshot(hkv_table* t, hkv_stream stream) {
  if (!t) return fail(HKV_EINVAL, "null table");
  DeviceGuard _g(t->cfg.device);
  GateScope _gs(t->gate, HKV_ROLE_READER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  const uint64_t cap = (uint64_t)t->cfg.capacity;
  cudaError_t e;
  if (!t->snap_ks) {
    if ((e = cudaMalloc((void**)&t->snap_ks, cap * 16)) || (e = cudaMalloc((void**)&t->snap_digests, cap)) ||
        (e = cudaMalloc((void**)&t->snap_bits, (size_t)t->buckets * 16)) ||
        (e = cudaMalloc((void**)&t->snap_smin, (size_t)t->buckets * 64)) ||
        (e = cudaMalloc((void**)&t->snap_svalid, (size_t)t->buckets * 4)) ||
        (e = cudaMalloc((void**)&t->snap_sc, sizeof(TableScalars))))
      return fail(HKV_ENOMEM, std::string("snapshot allocation failed: ") + cudaGetErrorString(e));
  }
  cudaStream_t s = (cudaStream_t)stream;
  if ((e = cudaMemcpyAsync(t->snap_ks, t->ks, cap * 16, cudaMemcpyDeviceToDevice, s)) ||
      (e = cudaMemcpyAsync(t->snap_digests, t->digests, cap, cudaMemcpyDeviceToDevice, s)) ||
      (e = cudaMemcpyAsync(t->snap_bits, t->bits, (size_t)t->buckets * 16, cudaMemcpyDeviceToDevice, s)) ||
      (e = cudaMemcpyAsync(t->snap_smin, t->smin, (size_t)t->buckets * 64, cudaMemcpyDeviceToDevice, s)) ||
      (e = cudaMemcpyAsync(t->snap_svalid, t->svalid, (size_t)t->buckets * 4, cudaMemcpyDeviceToDevice, s)) ||
      (e = cudaMemcpyAsync(t->snap_sc, t->sc, sizeof(TableScalars), cudaMemcpyDeviceToDevice, s)))
    return cuda_fail(e, "snapshot");
  return HKV_OK;
}

int hkv_restore(hkv_table* t, hkv_stream stream) {
  if (!t) return fail(HKV_EINVAL, "null table");
  if (!t->snap_ks) return fail(HKV_EINVAL, "no snapshot taken");
  DeviceGuard _g(t->cfg.device);
  GateScope _gs(t->gate, HKV_ROLE_INSERTER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  const uint64_t cap = (uint64_t)t->cfg.capacity;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if ((e = cudaMemcpyAsync(t->ks, t->snap_ks, cap * 16, cudaMemcpyDeviceToDevice, s)) ||
      (e = cudaMemcpyAsync(t->digests, t->snap_digests, cap, cudaMemcpyDeviceToDevice, s)) ||
      (e = cudaMemcpyAsync(t->bits, t->snap_bits, (size_t)t->buckets * 16, cudaMemcpyDeviceToDevice, s)) ||
      (e = cudaMemcpyAsync(t->smin, t->snap_smin, (size_t)t->buckets * 64, cudaMemcpyDeviceToDevice, s)) ||
      (e = cudaMemcpyAsync(t->svalid, t->snap_svalid, (size_t)t->buckets * 4, cudaMemcpyDeviceToDevice, s)) ||
      (e = cudaMemcpyAsync(t->sc, t->snap_sc, sizeof(TableScalars), cudaMemcpyDeviceToDevice, s)))
    return cuda_fail(e, "restore");
  return HKV_OK;
}

int hkv_check_consistency(hkv_table* t, int32_t* ok, hkv_stream stream) {
  if (!t || !ok) return fail(HKV_EINVAL, "null argument");
  DeviceGuard _g(t->cfg.device);
  GateScope _gs(t->gate, HKV_ROLE_READER, (cudaStream_t)stream);
  if (_gs.rc) return gate_fail(_gs.rc);
  cudaStream_t s = (cudaStream_t)stream;
  int init[4] = {1, 0, 0, 0};
  cudaError_t e = cudaMemcpyAsync(t->sc->check, init, sizeof(init), cudaMemcpyHostToDevice, s);
  if (!e) e = run_consistency(t->dev, t->buckets, t->sc->check, s);
  TableScalars h;
  if (!e) e = cudaMemcpyAsync(&h, t->sc, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (e) return cuda_fail(e, "consistency");
  unsigned long long total;
  memcpy(&total, &h.check[2], sizeof(total));
  *ok = h.check[0] == 1 && total == h.size;
  return HKV_OK;
}

int hkv_route(const uint64_t* keys, int64_t n, int64_t global_buckets, int32_t world, int32_t* perm,
              int64_t* counts, hkv_stream stream) {
  if (n < 0 || world < 1 || world > 64 || global_buckets < world || (global_buckets & (global_buckets - 1)) ||
      (world & (world - 1)))
    return fail(HKV_EINVAL, "bad route arguments (world and bucket count must be powers of two, world <= 64)");
  cudaStream_t s = (cudaStream_t)stream;
  std::lock_guard<std::mutex> g(g_route_mu);
  cudaError_t e = run_route(keys, n, global_buckets, world, perm, counts, g_route_ws[s], s);
  return e ? cuda_fail(e, "hkv_route") : HKV_OK;
}

}  // extern "C"
