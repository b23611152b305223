// hkv_probe.cuh — probe helpers shared by the kernels.
//
// probe_line_thread: one thread reads a key's whole 128-B digest line and
// checks candidate keys in slot order (find, contains, find_ptr, assign).
// 8-lane tiles (kG): lane r holds slots [16r, 16r+16) — one 16-B slice of the
// digest line and one 16-bit slice of the occupancy bitmap — for the kernels
// that work a bucket with a tile (dual-mode ops, value copies, the occupancy
// rebuild); a lane only reads or writes its own slots' metadata.
#pragma once
#include "hkv_common.cuh"

namespace hkv {

constexpr int kG = 8;                 // lanes per bucket tile
constexpr int kSPL = kSlots / kG;     // slots per lane (16)

// Lowest (score, slot) over the bucket — np.argmin semantics (first index on
// ties), table.py:1080.  Each lane scans its 16 scores (128 contiguous bytes).
__device__ __forceinline__ void bucket_min(const TableDev& t, const Tile8& tile,
                                           uint64_t b, uint64_t& minv, int& mslot) {
  const int r = tile.thread_rank();
  const ulonglong2* sp = reinterpret_cast<const ulonglong2*>(kptr(t, b * kSlots + r * kSPL));
  ulonglong2 s[kSPL / 2];
#pragma unroll
  for (int k = 0; k < kSPL / 2; k++) s[k] = make_ulonglong2(sp[2 * k].y, sp[2 * k + 1].y);
  uint64_t v = s[0].x;
  int m = r * kSPL;
#pragma unroll
  for (int k = 0; k < kSPL / 2; k++) {
    if (k > 0 && s[k].x < v) { v = s[k].x; m = r * kSPL + 2 * k; }
    if (s[k].y < v) { v = s[k].y; m = r * kSPL + 2 * k + 1; }
  }
#pragma unroll
  for (int o = kG / 2; o > 0; o >>= 1) {
    const uint64_t ov = tile.shfl_xor(v, o);
    const int om = tile.shfl_xor(m, o);
    if (ov < v || (ov == v && om < m)) { v = ov; m = om; }
  }
  minv = v;
  mslot = m;
}

__device__ __forceinline__ uint32_t load_occ(const TableDev& t, uint64_t b, int r) {
  return reinterpret_cast<const uint16_t*>(t.bits + b * 4)[r];
}
__device__ __forceinline__ void store_occ(const TableDev& t, uint64_t b, int r, uint32_t v) {
  reinterpret_cast<uint16_t*>(t.bits + b * 4)[r] = (uint16_t)v;
}

// Any score write at `slot` of bucket b outside the summary-maintaining
// single-mode pass: the group's minimum is no longer known exactly.
__device__ __forceinline__ void summ_invalidate(const TableDev& t, uint64_t b, int slot) {
  atomicAnd(t.svalid + b, ~(1u << (slot >> 4)));
}

// bucket_min through the eviction summary (the caller owns bucket b): lane r
// of the tile owns group r (its kSPL = 16 slots).  A lane whose group minimum
// is exact reads it from smin (the 64-B summary line); the others rescan their
// 16 (key, score) pairs and make it exact.  The winning group (lowest minimum,
// lowest group on ties) then finds its first slot holding the minimum, so the
// answer is np.argmin's first index, as bucket_min.  In the winning lane,
// `rest` = the group's minimum over its other 15 slots, for the caller to keep
// the summary exact after replacing the victim's score.
__device__ __forceinline__ void bucket_min_summ(const TableDev& t, const Tile8& tile, uint64_t b, uint64_t& minv,
                                                int& mslot, uint64_t& rest) {
  const int r = tile.thread_rank();
  const uint32_t sv = t.svalid[b];
  const bool exact = (sv >> r) & 1u;
  const ulonglong2* gp = reinterpret_cast<const ulonglong2*>(kptr(t, b * kSlots + r * kSPL));
  uint64_t gm;
  if (exact) {
    gm = t.smin[b * 8 + r];
  } else {
    gm = kMaxScore;
#pragma unroll
    for (int k = 0; k < kSPL; k++) {
      const uint64_t x = gp[k].y;
      gm = x < gm ? x : gm;
    }
    t.smin[b * 8 + r] = gm;
  }
  const unsigned fixed = tile.ballot(!exact);
  if (fixed && r == 0) atomicOr(t.svalid + b, fixed);
  uint64_t v = gm;
  int g = r;
#pragma unroll
  for (int o = kG / 2; o > 0; o >>= 1) {
    const uint64_t ov = tile.shfl_xor(v, o);
    const int og = tile.shfl_xor(g, o);
    if (ov < v || (ov == v && og < g)) { v = ov; g = og; }
  }
  int slot = 0;
  rest = kMaxScore;
  if (r == g) {
    int first = -1;
#pragma unroll
    for (int k = 0; k < kSPL; k++) {
      const uint64_t x = gp[k].y;
      if (first < 0 && x == v) first = k;
      else rest = x < rest ? x : rest;
    }
    slot = r * kSPL + first;
  }
  minv = v;
  mslot = tile.shfl(slot, g);
}

// Thread-per-key probe (the default): one thread reads its key's whole
// 128-B digest line (8 x 16 B, all in flight together), matches the 128
// digests with __vcmpeq4, then checks candidate keys in slot order.  No
// cross-lane collectives: ~2.5x fewer warp instructions per key than the
// 8-lane tile, and 32 keys per warp in flight instead of 16.
__device__ __forceinline__ int probe_line_thread(const TableDev& t, uint64_t b, uint64_t key, uint32_t d,
                                                 unsigned& ncmp) {
  const uint64_t rowbase = b * kSlots;
  uint32_t c[4];
  if (t.digest_filter) {
    const uint4* dp = reinterpret_cast<const uint4*>(t.digests + rowbase);
    uint4 w[8];
#pragma unroll
    for (int k = 0; k < 8; k++) w[k] = ld_stream(dp + k);
    const uint32_t dd = d * 0x01010101u;
    uint32_t any = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) any |= any16(w[k], dd);
    if ((any & 0x80808080u) == 0) return -1;  // no digest match: a miss without touching keys
#pragma unroll
    for (int q = 0; q < 4; q++) c[q] = match16(w[2 * q], d) | (match16(w[2 * q + 1], d) << 16);
  } else {
#pragma unroll
    for (int q = 0; q < 4; q++) c[q] = ~0u;
  }
  int hit = -1;
#pragma unroll
  for (int q = 0; q < 4; q++) {
    uint32_t m = hit < 0 ? c[q] : 0u;
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const uint64_t k = __ldg(kptr(t, rowbase + 32 * q + j));
      if (k == kEmptyKey) continue;  // candidates exclude EMPTY slots (table.py:243-247)
      ncmp++;
      if (k == key) {
        hit = 32 * q + j;
        m = 0;
      }
    }
  }
  return hit;
}

template <int G>
__device__ __forceinline__ int tile_sum(const Tile8& tile, int v) {
  return (int)tile.sum((unsigned)v);  // REDUX over the tile's 8 lanes
}

}  // namespace hkv
