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
int seg_exclusive_scan(const ScanDesc* segs, int S, int64_t* part, cudaStream_t stream);

}  // namespace recd
