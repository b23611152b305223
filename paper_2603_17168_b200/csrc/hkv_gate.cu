// hkv_gate.cu — the triple-group role gate, native: reader groups run with
// readers, updater groups with updaters, an inserter alone (PAPER.md:843-856
// Table 4), phase-fair FIFO admission (the reference's RoleGate contract,
// gate.py:60-141), and the paper's CPU–GPU dual-layer lock
// (PAPER.md:875-887, 1002-1007):
//
//  host layer    three std::atomic role counters + the admission state under
//                one mutex / condition variable;
//  device layer  GPU work is asynchronous, so releasing a host role when its
//                kernels are merely queued would let an incompatible group's
//                kernels overlap it on another stream.  Every release records
//                an event on the releasing stream; the first entrant of a new
//                group makes its stream wait on all of them, then launches a
//                one-thread propagation kernel that publishes
//                (group id, role) into a device mirror word and records the
//                group's fence event — the paper's store–launch–fence
//                handshake.  Later entrants of the same group wait on that one
//                fence, so same-role groups on different streams still
//                overlap on the device.  Mutation kernels read the mirror and
//                refuse to run (device error latch bit HKV_DERR_ROLE) if a
//                reader group owns the table.
//
// Re-entrancy: every hkv_* entry point takes its role through GateScope.  A
// thread that already holds the table's gate (an explicit hkv_gate_acquire
// around several calls, as the Python mirror does per public method) with
// the same role — or with the exclusive inserter role — passes straight
// through; its stream is still fenced.  A nested incompatible role is a usage
// error (it would deadlock).
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/hkv_b200.h"
#include "hkv_gate.h"

namespace hkv {

__global__ void k_gate_publish(unsigned* word, unsigned value) { *word = value; }

}  // namespace hkv

struct hkv_gate {
  std::recursive_mutex mu;  // the event hook may call back into the gate
  std::condition_variable_any cv;
  int active_role = -1;
  int active_count = 0;
  std::deque<std::pair<long long, int>> queue;  // FIFO of (ticket, role)
  long long next_ticket = 0;
  long long event_seq = 0;
  long long groups = 0;
  std::atomic<int> role_count[3] = {{0}, {0}, {0}};  // host layer
  hkv_gate_hook hook = nullptr;
  void* hook_user = nullptr;
  // holds per thread (re-entrancy): role and depth
  struct Hold {
    std::thread::id tid;
    int role;
    int depth;
  };
  std::vector<Hold> holds;
  // device layer (tables only)
  int device = -1;
  unsigned* dev_word = nullptr;
  int group_role = -1;
  cudaEvent_t fence = nullptr;
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> group_events;  // latest release event per stream
  std::vector<cudaEvent_t> pool;
  bool device_layer() const { return dev_word != nullptr; }

  cudaEvent_t take_event() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    return e;
  }

  void emit(int event, int role) {
    event_seq++;
    if (hook) hook(hook_user, event_seq, event, role, active_count);
  }

  bool compatible(int role) const {
    if (active_role < 0) return true;
    return active_role == role && role != HKV_ROLE_INSERTER;
  }
  // admitted at once only when compatible and nobody arrived earlier
  bool may_enter(long long ticket, int role) const {
    if (!compatible(role)) return false;
    for (auto& q : queue)
      if (q.first < ticket) return false;
    return true;
  }
  // a waiter enters with the maximal same-role prefix of the queue
  bool head_admissible(long long ticket, int role) const {
    if (!compatible(role)) return false;
    for (auto& q : queue) {
      if (q.first >= ticket) break;
      if (q.second != role || role == HKV_ROLE_INSERTER) return false;
    }
    return true;
  }

  // device-side entry of a stream into the current group
  cudaError_t fence_stream(cudaStream_t s) {
    if (!device_layer() || !fence) return cudaSuccess;
    return cudaStreamWaitEvent(s, fence, 0);
  }

  cudaError_t enter(int role, cudaStream_t s, bool has_stream) {
    const bool new_group = active_count == 0 && (group_role < 0 || group_role != role || role == HKV_ROLE_INSERTER);
    cudaError_t e = cudaSuccess;
    if (new_group) {
      groups++;
      group_role = role;
      if (device_layer()) {
        int prev = -1;
        cudaGetDevice(&prev);
        if (prev != device) cudaSetDevice(device);
        // the entrant's stream waits for everything the previous group queued
        for (auto& ge : group_events) {
          if (!e) e = cudaStreamWaitEvent(s, ge.second, 0);
          pool.push_back(ge.second);
        }
        group_events.clear();
        if (fence) {
          if (!e) e = cudaStreamWaitEvent(s, fence, 0);
          pool.push_back(fence);
          fence = nullptr;
        }
        if (!e) {
          hkv::k_gate_publish<<<1, 1, 0, s>>>(dev_word, ((unsigned)groups << 2) | (unsigned)(role + 1));
          e = cudaGetLastError();
        }
        cudaEvent_t f = take_event();
        if (!e && f) e = cudaEventRecord(f, s);
        fence = f;
        if (prev >= 0 && prev != device) cudaSetDevice(prev);
      }
    } else if (device_layer() && has_stream) {
      int prev = -1;
      cudaGetDevice(&prev);
      if (prev != device) cudaSetDevice(device);
      e = fence_stream(s);
      if (prev >= 0 && prev != device) cudaSetDevice(prev);
    }
    active_role = role;
    active_count++;
    role_count[role].fetch_add(1);
    return e;
  }

  cudaError_t record_release(cudaStream_t s) {
    if (!device_layer()) return cudaSuccess;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != device) cudaSetDevice(device);
    cudaEvent_t ev = take_event();
    cudaError_t e = ev ? cudaEventRecord(ev, s) : cudaErrorMemoryAllocation;
    if (!e) {
      bool placed = false;
      for (auto& ge : group_events)
        if (ge.first == s) {
          pool.push_back(ge.second);  // superseded by stream order
          ge.second = ev;
          placed = true;
        }
      if (!placed) group_events.emplace_back(s, ev);
    }
    if (prev >= 0 && prev != device) cudaSetDevice(prev);
    return e;
  }

  Hold* my_hold() {
    const auto me = std::this_thread::get_id();
    for (auto& h : holds)
      if (h.tid == me) return &h;
    return nullptr;
  }

  ~hkv_gate() {
    for (auto& ge : group_events) cudaEventDestroy(ge.second);
    for (auto e : pool) cudaEventDestroy(e);
    if (fence) cudaEventDestroy(fence);
  }
};

namespace hkv {

hkv_gate* gate_new_device(int device, unsigned* dev_word) {
  hkv_gate* g = new hkv_gate();
  g->device = device;
  g->dev_word = dev_word;
  return g;
}

void gate_delete(hkv_gate* g) { delete g; }

// Acquisition.  mode 0 = try (HKV_EBUSY instead of waiting), 1 = blocking:
// the reference's RoleGate semantics exactly, every acquisition counted.
// mode 2 = an entry point's scope: when the calling thread already holds a
// covering role (the same role, or the exclusive inserter role) through an
// explicit acquisition, the scope nests (*nested = true: no admission, no
// event, the stream is still fenced); an incompatible held role would
// deadlock and is refused (HKV_EINVAL); otherwise a blocking acquisition.
int gate_acquire(hkv_gate* g, int role, int mode, cudaStream_t s, bool has_stream, bool* nested) {
  std::unique_lock<std::recursive_mutex> lk(g->mu);
  *nested = false;
  if (mode == 2) {
    if (auto* h = g->my_hold()) {
      if (h->role != role && h->role != HKV_ROLE_INSERTER) {
        set_error("role gate: this thread holds an incompatible role on the table (the call would deadlock)");
        return HKV_EINVAL;
      }
      *nested = true;
      cudaError_t e = has_stream ? g->fence_stream(s) : cudaSuccess;
      return e ? HKV_ECUDA : HKV_OK;
    }
  }
  const long long ticket = g->next_ticket;
  if (!g->may_enter(ticket, role)) {
    if (mode == 0) return HKV_EBUSY;
    g->next_ticket++;
    g->queue.emplace_back(ticket, role);
    g->cv.wait(lk, [&] { return g->head_admissible(ticket, role); });
    for (auto it = g->queue.begin(); it != g->queue.end(); ++it)
      if (it->first == ticket) {
        g->queue.erase(it);
        break;
      }
  } else {
    g->next_ticket++;
  }
  cudaError_t e = g->enter(role, s, has_stream);
  g->holds.push_back({std::this_thread::get_id(), role, 1});
  g->emit(HKV_GATE_ACQUIRE, role);
  return e ? HKV_ECUDA : HKV_OK;
}

int gate_release(hkv_gate* g, int role, bool nested, cudaStream_t s, bool has_stream) {
  std::unique_lock<std::recursive_mutex> lk(g->mu);
  if (nested) return (has_stream && g->record_release(s)) ? HKV_ECUDA : HKV_OK;
  if (g->active_count <= 0 || g->active_role != role) {
    set_error("role gate: release does not match an active acquisition");
    return HKV_EINVAL;
  }
  {
    // drop the hold: the calling thread's, else (a guard released by another
    // thread than its acquirer) the oldest of this role
    auto me = std::this_thread::get_id();
    auto pick = g->holds.end();
    for (auto it = g->holds.begin(); it != g->holds.end(); ++it)
      if (it->role == role && (it->tid == me || pick == g->holds.end())) {
        pick = it;
        if (it->tid == me) break;
      }
    if (pick != g->holds.end()) g->holds.erase(pick);
  }
  cudaError_t e = has_stream ? g->record_release(s) : cudaSuccess;
  g->active_count--;
  g->role_count[role].fetch_sub(1);
  g->emit(HKV_GATE_RELEASE, role);
  if (g->active_count == 0) g->active_role = -1;
  g->cv.notify_all();
  return e ? HKV_ECUDA : HKV_OK;
}

}  // namespace hkv

using namespace hkv;

extern "C" {

int hkv_gate_create(hkv_gate** out) {
  if (!out) return HKV_EINVAL;
  *out = new hkv_gate();
  return HKV_OK;
}

int hkv_gate_destroy(hkv_gate* g) {
  delete g;
  return HKV_OK;
}

int hkv_gate_set_hook(hkv_gate* g, hkv_gate_hook fn, void* user) {
  if (!g) return HKV_EINVAL;
  std::unique_lock<std::recursive_mutex> lk(g->mu);
  g->hook = fn;
  g->hook_user = user;
  return HKV_OK;
}

int hkv_gate_acquire(hkv_gate* g, int32_t role, int32_t mode, int32_t has_stream, hkv_stream stream) {
  if (!g || role < HKV_ROLE_READER || role > HKV_ROLE_INSERTER || mode < 0 || mode > 2) {
    set_error("role gate: bad role or mode");
    return HKV_EINVAL;
  }
  bool nested = false;
  int rc = gate_acquire(g, role, mode, (cudaStream_t)stream, has_stream != 0, &nested);
  return (rc == HKV_OK && nested) ? HKV_GATE_NESTED : rc;
}

int hkv_gate_release(hkv_gate* g, int32_t role, int32_t nested, int32_t has_stream, hkv_stream stream) {
  if (!g || role < HKV_ROLE_READER || role > HKV_ROLE_INSERTER) {
    set_error("role gate: bad role");
    return HKV_EINVAL;
  }
  return gate_release(g, role, nested != 0, (cudaStream_t)stream, has_stream != 0);
}

int hkv_gate_state(hkv_gate* g, int32_t* role, int32_t* count, int64_t* groups) {
  if (!g) return HKV_EINVAL;
  std::unique_lock<std::recursive_mutex> lk(g->mu);
  if (role) *role = g->active_role;
  if (count) *count = g->active_count;
  if (groups) *groups = g->groups;
  return HKV_OK;
}

}  // extern "C"
