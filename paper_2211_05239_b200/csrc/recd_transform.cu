// Element-wise ID transforms of the reader (reader.py:54-83), applied to the
// deduplicated values of an IKJT (reader.process, reader.py:178-217: IKJT
// features are transformed on their unique values only and stay IKJTs, which
// commutes with the expansion).  One launch for every (feature, transform).
//   identity : x
//   mod_hash : splitmix64(x) mod param   (uint64 arithmetic, int64 result)
//   clamp    : min(max(x, 0), param)
#include <algorithm>

#include "recd_common.cuh"

namespace recd {

struct XformParams {
  int F;
  const int64_t* in[RECD_MAX_FEAT];
  int64_t* out[RECD_MAX_FEAT];
  const int64_t* count[RECD_MAX_FEAT];  // device element count, or null (use n)
  int64_t n[RECD_MAX_FEAT];             // host capacity
  int op[RECD_MAX_FEAT];
  uint64_t param[RECD_MAX_FEAT];
  int64_t blk0[RECD_MAX_FEAT + 1];
};

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

constexpr int XF_NT = 256, XF_IT = 8;

__global__ void __launch_bounds__(XF_NT) k_transform(const __grid_constant__ XformParams p) {
  const int f = block_feature(p.blk0, p.F, (int64_t)blockIdx.x);
  const int64_t n = p.count[f] ? min(*p.count[f], p.n[f]) : p.n[f];
  const int64_t base = ((int64_t)blockIdx.x - p.blk0[f]) * (XF_NT * XF_IT);
  const int op = p.op[f];
  const uint64_t prm = p.param[f];
#pragma unroll
  for (int k = 0; k < XF_IT; ++k) {
    const int64_t j = base + k * XF_NT + threadIdx.x;
    if (j >= n) break;
    const int64_t x = p.in[f][j];
    int64_t y = x;
    if (op == RECD_XF_MOD_HASH) y = (int64_t)(splitmix64((uint64_t)x) % prm);
    else if (op == RECD_XF_CLAMP) y = x < 0 ? 0 : (x > (int64_t)prm ? (int64_t)prm : x);
    p.out[f][j] = y;
  }
}

}  // namespace recd

using namespace recd;

extern "C" int recd_transform(int32_t num_features, const int64_t* const* values_in,
                              int64_t* const* values_out, const int64_t* num_values,
                              const int64_t* const* device_counts, const int32_t* ops,
                              const int64_t* params, recd_stream_t stream) {
  if (num_features <= 0 || !values_in || !values_out || !num_values || !ops || !params)
    return RECD_ERR_ARG;
  for (int f0 = 0; f0 < num_features; f0 += RECD_MAX_FEAT) {
    XformParams p;
    memset(&p, 0, sizeof(p));
    p.F = std::min(RECD_MAX_FEAT, num_features - f0);
    int64_t blk = 0;
    for (int f = 0; f < p.F; ++f) {
      const int g = f0 + f;
      if (ops[g] < RECD_XF_IDENTITY || ops[g] > RECD_XF_CLAMP) return RECD_ERR_ARG;
      if (ops[g] != RECD_XF_IDENTITY && params[g] < 1) return RECD_ERR_ARG;
      if (num_values[g] < 0 || (num_values[g] > 0 && (!values_in[g] || !values_out[g]))) return RECD_ERR_ARG;
      p.in[f] = values_in[g];
      p.out[f] = values_out[g];
      p.count[f] = device_counts ? device_counts[g] : nullptr;
      p.n[f] = num_values[g];
      p.op[f] = ops[g];
      p.param[f] = (uint64_t)params[g];
      p.blk0[f] = blk;
      blk += ceil_div(num_values[g], XF_NT * XF_IT);
    }
    p.blk0[p.F] = blk;
    if (blk == 0) continue;
    k_transform<<<(unsigned)blk, XF_NT, 0, (cudaStream_t)stream>>>(p);
    note_launch();
  }
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}
