// Canonical wire format of KJTs / IKJTs (tensors._serialize, serialize_kjt,
// serialize_ikjt: /root/reference/pkg/src/sessiondedup/tensors.py:463-505),
// written on the GPU into one device byte buffer -- the reader -> trainer
// transport and the byte accounting of the all-to-all (trainer_sim.py:281-305).
// Little-endian:
//   u32 key count; per key: u32 byte length + UTF-8 bytes   (host-known prefix)
//   u64 batch size B; u8 inverse flag; [B x i64 inverse]
//   per key: u64 offsets count + i64 offsets   (count = rows, device-side for IKJTs)
//   per key: u64 values count + i64 values     (count on the device)
// k_wire_layout (1 thread) places the sections from the device counts and
// writes the count prefixes; k_wire_copy moves the arrays: every output
// 8-byte word fully inside a section is assembled from two aligned source
// words with a funnel shift (sections land at arbitrary byte offsets), the
// partial words at section edges are written byte by byte.
#include <algorithm>
#include <cstring>

#include "recd_common.cuh"

namespace recd {

constexpr int WIRE_MAX_PREFIX = 2048;
constexpr int WIRE_MAX_SEC = 2 * RECD_MAX_FEAT + 1;

struct WireParams {
  int K;
  int has_inverse;
  int prefix_len;
  int64_t B;
  unsigned char prefix[WIRE_MAX_PREFIX];  // key count, names, B, flag
  const int64_t* src[WIRE_MAX_SEC];       // inverse?, offsets[K], values[K]
  const int64_t* count[WIRE_MAX_SEC];     // device element counts (nullptr: use cap)
  int64_t cap[WIRE_MAX_SEC];
  unsigned char* out;
  int64_t out_cap;
  int64_t* total;        // device: bytes written (or -1 if out_cap too small)
  int64_t* sec_off;      // device scratch [WIRE_MAX_SEC] byte offset of each section's data
  int64_t* sec_len;      // device scratch [WIRE_MAX_SEC] elements
};

__global__ void k_wire_layout(const __grid_constant__ WireParams p) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t pos = 0;
  const int nsec = p.has_inverse + 2 * p.K;
  // total size first, to refuse an undersized buffer before writing
  int64_t total = p.prefix_len;
  for (int s = 0; s < nsec; ++s) {
    const int64_t n = p.count[s] ? min(*p.count[s], p.cap[s]) : p.cap[s];
    p.sec_len[s] = n;
    total += (s < p.has_inverse ? 0 : 8) + 8 * n;
  }
  if (total > p.out_cap) {
    *p.total = -1;
    for (int s = 0; s < nsec; ++s) p.sec_len[s] = 0;
    return;
  }
  for (int i = 0; i < p.prefix_len; ++i) p.out[pos++] = p.prefix[i];
  for (int s = 0; s < nsec; ++s) {
    if (s >= p.has_inverse) {  // u64 count prefix
      const uint64_t n = (uint64_t)p.sec_len[s];
      for (int b = 0; b < 8; ++b) p.out[pos++] = (unsigned char)(n >> (8 * b));
    }
    p.sec_off[s] = pos;
    pos += 8 * p.sec_len[s];
  }
  *p.total = pos;
}

// grid-stride over (section, output word) pairs: block y = section
__global__ void __launch_bounds__(256) k_wire_copy(const __grid_constant__ WireParams p) {
  const int s = blockIdx.y;
  const int64_t n = p.sec_len[s];
  if (n == 0) return;
  const int64_t d0 = p.sec_off[s], d1 = d0 + 8 * n;  // destination byte range
  const unsigned sh = (unsigned)(d0 & 7);             // byte shift of the section
  const uint64_t* src = reinterpret_cast<const uint64_t*>(p.src[s]);
  unsigned char* out = p.out;
  const int64_t w0 = (d0 + 7) >> 3, w1 = d1 >> 3;     // full output words [w0, w1)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = w0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < w1; w += stride) {
    // output bytes [8w, 8w + 8) = source bytes [8w - d0, 8w - d0 + 8)
    const int64_t sb = 8 * w - d0;
    const int64_t si = sb >> 3;  // sb = 8 si + (8 - sh) % 8
    uint64_t v;
    if (sh == 0) {
      v = src[si];
    } else {
      // sb = 8 * si + (8 - sh): low part from src[si] >> 8(8-sh), high from src[si+1]
      const uint64_t lo = src[si], hi = (si + 1 < n) ? src[si + 1] : 0ull;
      v = (lo >> (8 * (8 - sh))) | (hi << (8 * sh));
    }
    reinterpret_cast<uint64_t*>(out)[w] = v;
  }
  // edge bytes outside full words: [d0, 8 w0) and [8 w1, d1)
  if (blockIdx.x == 0 && threadIdx.x < 16) {
    const int t = threadIdx.x;
    const int64_t b = t < 8 ? d0 + t : 8 * w1 + (t - 8);
    const bool ok = t < 8 ? b < min(8 * w0, d1) : (b < d1 && b >= max(8 * w1, 8 * w0));
    if (ok) {
      const int64_t sb = b - d0;
      const unsigned char* sbytes = reinterpret_cast<const unsigned char*>(src);
      out[b] = sbytes[sb];
    }
  }
}

}  // namespace recd

using namespace recd;

extern "C" int64_t recd_wire_bound(int32_t num_keys, const char* const* key_names, int64_t batch_size,
                                   int32_t has_inverse, const int64_t* offsets_caps,
                                   const int64_t* values_caps) {
  if (num_keys < 0 || num_keys > RECD_MAX_FEAT || batch_size < 0) return -1;
  int64_t n = 4 + 8 + 1 + (has_inverse ? 8 * batch_size : 0);
  for (int k = 0; k < num_keys; ++k)
    n += 4 + (int64_t)strlen(key_names[k]) + 16 + 8 * (offsets_caps[k] + values_caps[k]);
  return n;
}

extern "C" int recd_wire_serialize(int32_t num_keys, const char* const* key_names, int64_t batch_size,
                                   const int64_t* inverse, const int64_t* const* offsets,
                                   const int64_t* const* values, const int64_t* const* offsets_counts,
                                   const int64_t* const* values_counts, const int64_t* offsets_caps,
                                   const int64_t* values_caps, void* out, int64_t out_cap,
                                   int64_t* total_out, void* scratch, size_t scratch_bytes,
                                   recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (num_keys < 0 || num_keys > RECD_MAX_FEAT || batch_size < 0 || !out || !total_out ||
      scratch_bytes < 2 * sizeof(int64_t) * WIRE_MAX_SEC)
    return RECD_ERR_ARG;
  WireParams p;
  memset(&p, 0, sizeof(p));
  p.K = num_keys;
  p.has_inverse = inverse ? 1 : 0;
  p.B = batch_size;
  // host-known prefix
  int pl = 0;
  auto put = [&](const void* d, int n) -> bool {
    if (pl + n > WIRE_MAX_PREFIX) return false;
    memcpy(p.prefix + pl, d, n);
    pl += n;
    return true;
  };
  const uint32_t kc = (uint32_t)num_keys;
  if (!put(&kc, 4)) return RECD_ERR_UNSUPPORTED;
  for (int k = 0; k < num_keys; ++k) {
    const uint32_t len = (uint32_t)strlen(key_names[k]);
    if (!put(&len, 4) || !put(key_names[k], (int)len)) return RECD_ERR_UNSUPPORTED;
  }
  const uint64_t b = (uint64_t)batch_size;
  const unsigned char flag = inverse ? 1 : 0;
  if (!put(&b, 8) || !put(&flag, 1)) return RECD_ERR_UNSUPPORTED;
  p.prefix_len = pl;
  int s = 0;
  if (inverse) {
    p.src[s] = inverse;
    p.count[s] = nullptr;
    p.cap[s++] = batch_size;
  }
  for (int k = 0; k < num_keys; ++k, ++s) {
    p.src[s] = offsets[k];
    p.count[s] = offsets_counts ? offsets_counts[k] : nullptr;
    p.cap[s] = offsets_caps[k];
    if (!p.src[s] && p.cap[s] > 0) return RECD_ERR_ARG;
  }
  for (int k = 0; k < num_keys; ++k, ++s) {
    p.src[s] = values[k];
    p.count[s] = values_counts ? values_counts[k] : nullptr;
    p.cap[s] = values_caps[k];
    if (!p.src[s] && p.cap[s] > 0) return RECD_ERR_ARG;
  }
  p.out = reinterpret_cast<unsigned char*>(out);
  p.out_cap = out_cap;
  p.total = total_out;
  p.sec_off = reinterpret_cast<int64_t*>(scratch);
  p.sec_len = p.sec_off + WIRE_MAX_SEC;
  if ((reinterpret_cast<uintptr_t>(out) & 7) != 0) return RECD_ERR_ARG;
  k_wire_layout<<<1, 32, 0, stream>>>(p);
  if (s > 0) {
    int64_t maxcap = 0;
    for (int i = 0; i < s; ++i) maxcap = std::max(maxcap, p.cap[i]);
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(maxcap, 256),
                                                                        (int64_t)num_sms() * 4));
    k_wire_copy<<<dim3(gx, (unsigned)s), 256, 0, stream>>>(p);
  }
  note_launch(2);
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}
