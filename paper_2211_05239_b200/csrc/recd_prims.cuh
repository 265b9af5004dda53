// Device-wide primitives used by the backward, jagged select and slicing:
// a segmented stable LSD radix sort of (uint32 key, uint32 value) pairs and a
// segmented exclusive scan of int64.  Segments have host-known capacities
// (the launch geometry) and device-resident actual counts, so no host sync is
// needed between the producer kernel and the sort.
#pragma once

#include "recd_common.cuh"

namespace recd {

struct SegDesc {
  int64_t base;          // element offset of the segment in the key/value arrays
  int64_t cap;           // capacity (host-known)
  const int64_t* count;  // device: actual element count (<= cap)
};

// Stable sort of each segment by the low `bits` bits of the key.  Sorts
// keys/vals in place (ping-pong through alt buffers; the result is copied
// back only if an odd number of passes ran: *in_alt tells where it is).
// hist scratch: sort_hist_words(...) uint32 words.
int64_t sort_hist_words(const SegDesc* segs, int S);
// gate (device, nullable): the sort's kernels do nothing unless *gate != 0.
// hist_ready: the keys' producer already added every pass's digit counts of
// segment s into hist[(s * 4 + pass) * 256 + digit] (after sort_hist_clear),
// so the sort skips its own histogram read of the keys.
int seg_sort_pairs(const SegDesc* segs, int S, int bits, uint32_t* keys, uint32_t* vals,
                   uint32_t* keys_alt, uint32_t* vals_alt, uint32_t* hist, bool* in_alt,
                   cudaStream_t stream, const int32_t* gate = nullptr, bool hist_ready = false);
int sort_hist_clear(int S, uint32_t* hist, cudaStream_t stream);
constexpr int SORT_HIST_PASSES = 4;  // hist row stride: passes per segment

struct ScanDesc {
  const int64_t* in;
  int64_t* out;          // may alias in
  int64_t cap;           // host-known capacity
  const int64_t* count;  // device count, or nullptr (= cap)
  int64_t* total;        // device: segment total, nullable
};
int64_t scan_part_words(const ScanDesc* segs, int S);

// ---- one-tile stable sort in shared memory (a CTA of LS_NT threads, up to
// LS_TILE pairs; element e = warp * (LS_TILE / 8) + r * 32 + lane is item r
// of its thread, so input order is (warp, round, lane) and every pass is
// stable: warp match_any ranking + per-warp digit counters, 8-bit digits)
constexpr int LS_NT = 256, LS_ITEMS = 16, LS_TILE = LS_NT * LS_ITEMS, LS_WARPS = LS_NT / 32;
struct LocalSortSmem {
  uint32_t wcnt[LS_WARPS][256];
  uint32_t tdb[256];
  uint32_t keys[LS_TILE];
  uint32_t vals[LS_TILE];
  int64_t scan[32];
};
__device__ __forceinline__ int ls_elem(int r) {
  return (int)(threadIdx.x >> 5) * (LS_TILE / LS_WARPS) + r * 32 + (int)(threadIdx.x & 31);
}
// sorts the tn pairs in key/val (registers, item r = element ls_elem(r)) by
// the low `bits` bits of the key; the result is left in sm.keys / sm.vals
__device__ __forceinline__ void local_sort_tile(uint32_t (&key)[LS_ITEMS], uint32_t (&val)[LS_ITEMS],
                                                int tn, int bits, LocalSortSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = lanemask_lt();
  const int npass = (bits + 7) / 8;
  if (npass == 0) {
#pragma unroll
    for (int r = 0; r < LS_ITEMS; ++r)
      if (ls_elem(r) < tn) sm.keys[ls_elem(r)] = key[r], sm.vals[ls_elem(r)] = val[r];
    __syncthreads();
  }
  for (int pass = 0; pass < npass; ++pass) {
    const int shift = 8 * pass;
    const uint32_t mask = (1u << min(8, bits - shift)) - 1u;
    for (int d = lane; d < 256; d += 32) sm.wcnt[warp][d] = 0;
    __syncwarp();
    uint32_t rank[LS_ITEMS];
#pragma unroll
    for (int r = 0; r < LS_ITEMS; ++r) {
      const bool valid = ls_elem(r) < tn;
      const uint32_t d = valid ? ((key[r] >> shift) & mask) : 0x100u;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      uint32_t before = 0;
      if (valid) before = sm.wcnt[warp][d];
      __syncwarp();
      if (valid && lane == __ffs(peers) - 1) sm.wcnt[warp][d] = before + __popc(peers);
      __syncwarp();
      rank[r] = before + __popc(peers & lt);
    }
    __syncthreads();
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < LS_WARPS; ++w) {
      const uint32_t c = sm.wcnt[w][tid];
      sm.wcnt[w][tid] = cnt;
      cnt += c;
    }
    int64_t tot;
    sm.tdb[tid] = (uint32_t)block_exclusive_scan<LS_NT>(cnt, sm.scan, &tot);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < LS_ITEMS; ++r) {
      if (ls_elem(r) < tn) {
        const uint32_t d = (key[r] >> shift) & mask;
        const uint32_t lp = sm.tdb[d] + sm.wcnt[warp][d] + rank[r];
        sm.keys[lp] = key[r];
        sm.vals[lp] = val[r];
      }
    }
    __syncthreads();
    if (pass + 1 < npass) {
#pragma unroll
      for (int r = 0; r < LS_ITEMS; ++r) {
        const int e = ls_elem(r);
        key[r] = e < tn ? sm.keys[e] : 0u;
        val[r] = e < tn ? sm.vals[e] : 0u;
      }
      __syncthreads();
    }
  }
}
int seg_exclusive_scan(const ScanDesc* segs, int S, int64_t* part, cudaStream_t stream);

}  // namespace recd
