// ctable.cuh — per-problem table of distinct sample colours in shared memory
// (keys | pixel counts, 2^14 slots, linear probing), built by k_colour_table
// (snmf.cu) from the compacted samples.  Every SNMF quantity is a function of
// the colour, so the fit passes visit each colour once with its weight.
// (A variant that compacted straight from the image into the table, one CTA
// per item, measured slower — 11.9 ms vs 4.3 + 5.5 ms for 4096 items: one
// CTA per item serialises the raster walk on block barriers.)
#pragma once
#include <cstdint>

namespace spcn {

constexpr int kTabBits = 14;
constexpr int kTabSlots = 1 << kTabBits;
constexpr uint32_t kTabEmpty = 0xffffffffu;
constexpr uint32_t kNoColour = 0xffffffffu;   // a lane without a sample

// One colour per lane (kNoColour: none).  Sets *full when a probe sequence
// fails; the load test (more than 3/4 of the slots taken — the distinct
// colours, a set property) is made once after all inserts (ct_overfull), so
// no shared counter is contended per new key.  The caller lists the samples
// one by one when either fires.
__device__ __forceinline__ void ct_insert(uint32_t* key, uint32_t* cnt, int* full, uint32_t rgb) {
  if (rgb == kNoColour) return;
  uint32_t slot = (rgb * 2654435761u) >> (32 - kTabBits);
  for (int probe = 0; probe < 64; ++probe, slot = (slot + 1) & (kTabSlots - 1)) {
    uint32_t k = key[slot];
    if (k == kTabEmpty) k = atomicCAS(&key[slot], kTabEmpty, rgb);
    if (k == kTabEmpty || k == rgb) {
      atomicAdd(&cnt[slot], 1u);
      return;
    }
  }
  *full = 1;
}

// After the inserts (and a barrier): sets *full if more than 3/4 of the
// slots are taken.  NT threads; *used must be 0 on entry; ends with a barrier.
template <int NT>
__device__ __forceinline__ void ct_overfull(const uint32_t* key, int* used, int* full) {
  int occ = 0;
  for (int i = threadIdx.x; i < kTabSlots; i += NT) occ += key[i] != kTabEmpty;
  occ = __reduce_add_sync(0xffffffffu, occ);
  if ((threadIdx.x & 31) == 0) atomicAdd(used, occ);
  __syncthreads();
  if (threadIdx.x == 0 && *used > (3 * kTabSlots) / 4) *full = 1;
  __syncthreads();
}

// Write the table as (rgb, count) entries at ukey/ucnt[o0 ..], *ucount_p = #.
// With linear probing the SET of occupied slots, hence every cluster (maximal
// run of occupied slots) and its key set, does not depend on insertion order
// — only the order inside a cluster does.  Entries are written as if each
// cluster were sorted by colour in place and the table compacted in slot
// order, which makes the entry order, and every later floating-point
// summation order, deterministic.  Done in parallel without moving the table:
// every occupied slot's key finds its cluster and its rank r among the
// cluster's keys; its sorted slot is (cluster start + r), and that slot's
// position in slot order (pos16, from one block scan) is where the entry goes
// — O(L) work per key instead of a serial O(L^2) insertion sort per cluster.  pos16: SLOTS
// uint16 of shared scratch.  Requires at least one empty slot (the caller
// rejects tables above 3/4 load).  Ends with a barrier.
template <int NT>
__device__ void ct_finish_par(const uint32_t* key, const uint32_t* cnt, uint32_t* scan,
                              uint16_t* pos16, uint32_t* __restrict__ ukey,
                              uint32_t* __restrict__ ucnt, int64_t o0, int32_t* ucount_p) {
  constexpr int kMask = kTabSlots - 1;
  const int tid = threadIdx.x;
  constexpr int kPer = kTabSlots / NT;
  uint32_t occ = 0;
  for (int j = 0; j < kPer; ++j) occ += key[tid * kPer + j] != kTabEmpty;
  scan[tid] = occ;
  __syncthreads();
  for (int off = 1; off < NT; off <<= 1) {
    const uint32_t y = tid >= off ? scan[tid - off] : 0u;
    __syncthreads();
    scan[tid] += y;
    __syncthreads();
  }
  uint32_t pos = scan[tid] - occ;
  for (int j = 0; j < kPer; ++j) {
    const int sl = tid * kPer + j;
    if (key[sl] != kTabEmpty) pos16[sl] = static_cast<uint16_t>(pos++);
  }
  if (tid == NT - 1) *ucount_p = (int32_t)scan[NT - 1];
  __syncthreads();
  for (int s = tid; s < kTabSlots; s += NT) {
    const uint32_t k = key[s];
    if (k == kTabEmpty) continue;
    int b = s;                                    // cluster start (walk back)
    while (key[(b - 1) & kMask] != kTabEmpty) --b;
    int r = 0;                                    // rank among the cluster's keys
    for (int t = b;; ++t) {
      const uint32_t kt = key[t & kMask];
      if (kt == kTabEmpty) break;
      r += kt < k;
    }
    const int dst = pos16[(b + r) & kMask];
    ukey[o0 + dst] = k;
    ucnt[o0 + dst] = cnt[s];
  }
  __syncthreads();
}

}  // namespace spcn
