// Batched segment copy: one launch moves many (src, dst, bytes) segments.
// Used to pack / unpack the per-(peer, feature) blocks of the row-sharded
// exchange so that each exchange is a single NCCL all-to-all.
#include <algorithm>
#include <vector>

#include "recd_common.cuh"

namespace recd {

struct CopySeg {
  const char* src;
  char* dst;
  int64_t bytes;
  int64_t chunk0;  // first 16 KB chunk of this segment in the launch
};

constexpr int64_t CP_CHUNK = 16384;

__global__ void __launch_bounds__(256) k_batched_copy(const CopySeg* __restrict__ segs, int nseg,
                                                      int64_t total_chunks) {
  for (int64_t c = blockIdx.x; c < total_chunks; c += gridDim.x) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (segs[mid].chunk0 <= c) lo = mid; else hi = mid - 1;
    }
    const CopySeg s = segs[lo];
    const int64_t off = (c - s.chunk0) * CP_CHUNK;
    const int64_t n = min(CP_CHUNK, s.bytes - off);
    const char* src = s.src + off;
    char* dst = s.dst + off;
    const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) | n) & 15) == 0;
    if (vec) {
      const int4* s4 = reinterpret_cast<const int4*>(src);
      int4* d4 = reinterpret_cast<int4*>(dst);
      for (int64_t i = threadIdx.x; i < n / 16; i += blockDim.x) d4[i] = __ldg(s4 + i);
    } else {
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    }
  }
}

}  // namespace recd

using namespace recd;

// descs: device buffer of at least recd_batched_copy_desc_bytes(n) bytes (the
// segment table is staged there with one async H2D copy from `host_staging`,
// a host buffer of the same size that must stay valid until the copy ran --
// pinned memory lets the call stay asynchronous).
extern "C" size_t recd_batched_copy_desc_bytes(int32_t num_segments) {
  return (size_t)std::max(num_segments, 1) * sizeof(CopySeg);
}

extern "C" int recd_batched_copy(int32_t num_segments, const void* const* src, void* const* dst,
                                 const int64_t* bytes, void* host_staging, void* descs,
                                 recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (num_segments < 0 || (num_segments > 0 && (!src || !dst || !bytes || !host_staging || !descs)))
    return RECD_ERR_ARG;
  CopySeg* h = reinterpret_cast<CopySeg*>(host_staging);
  int n = 0;
  int64_t chunks = 0;
  for (int i = 0; i < num_segments; ++i) {
    if (bytes[i] <= 0) continue;
    h[n].src = reinterpret_cast<const char*>(src[i]);
    h[n].dst = reinterpret_cast<char*>(dst[i]);
    h[n].bytes = bytes[i];
    h[n].chunk0 = chunks;
    chunks += ceil_div(bytes[i], CP_CHUNK);
    ++n;
  }
  if (n == 0) return RECD_OK;
  RECD_CUDA_CHECK(cudaMemcpyAsync(descs, h, sizeof(CopySeg) * n, cudaMemcpyHostToDevice, stream));
  const unsigned grid = (unsigned)std::min<int64_t>(chunks, (int64_t)num_sms() * 8);
  k_batched_copy<<<grid, 256, 0, stream>>>(reinterpret_cast<const CopySeg*>(descs), n, chunks);
  note_launch();
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}
