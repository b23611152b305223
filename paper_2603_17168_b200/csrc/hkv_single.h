// hkv_single.h — single-key API kernels (hkv_single.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hkv_common.cuh"

namespace hkv {

struct OneResult {
  int kind;    // Outcome (kFound / kNotFound for lookups)
  int status;  // 0 ok; 1 kCustomized without a score; 2 a score without kCustomized
  int64_t bucket;
  int slot;
  int pad;
  uint64_t evicted_key;
  uint64_t evicted_score;
};

// bucket < 0: lookup (h1, then h2 in dual mode); else find_in_bucket
void launch_lookup_one(const TableDev& t, uint64_t key, int64_t bucket, OneResult* r, cudaStream_t s);
void launch_upsert_one(const TableDev& t, uint64_t key, const float* v, int dual, int has_score, uint64_t score,
                       uint64_t epoch, OneResult* r, cudaStream_t s);

}  // namespace hkv
