// hkv_gate.h — internal interface of the native role gate (hkv_gate.cu).
#pragma once
#include <cuda_runtime.h>

#include "../../include/hkv_b200.h"

namespace hkv {

hkv_gate* gate_new_device(int device, unsigned* dev_word);
void gate_delete(hkv_gate* g);
int gate_acquire(hkv_gate* g, int role, int mode, cudaStream_t s, bool has_stream, bool* nested);
int gate_release(hkv_gate* g, int role, bool nested, cudaStream_t s, bool has_stream);
void set_error(const char* msg);  // hkv_last_error() text (hkv_api.cu)

// RAII role for one entry point: acquired (nested when the calling thread
// already holds a covering role) before the launches, released with a stream
// event after them.
struct GateScope {
  hkv_gate* g;
  int role;
  cudaStream_t s;
  bool nested = false;
  int rc;
  GateScope(hkv_gate* g_, int role_, cudaStream_t s_) : g(g_), role(role_), s(s_) {
    rc = g ? gate_acquire(g, role, 2, s, true, &nested) : 0;
  }
  ~GateScope() {
    if (g && rc == 0) gate_release(g, role, nested, s, true);
  }
};

}  // namespace hkv
