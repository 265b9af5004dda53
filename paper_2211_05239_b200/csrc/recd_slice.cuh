// Row slices and the exact-order pooling reductions shared by the forward
// and backward kernels.
//
// A "worker" is LPR consecutive lanes owning one embedding row of D floats:
// lane sl of the worker holds NV float4 vectors (dims 4*(sl + LPR*v) ..) when
// D % 4 == 0, else NV scalars (dims sl + LPR*v).  D = 128 -> 32 lanes x 1
// float4 (one 512-byte row per warp, fully coalesced 128-bit loads);
// D = 64 -> 16 lanes (two rows per warp).
#pragma once

#include "recd_common.cuh"

namespace recd {

template <int LPR_, int NV_, bool F4_>
struct Slice {
  static constexpr int LPR = LPR_;
  static constexpr int NV = NV_;
  static constexpr bool F4 = F4_;
  static constexpr int N = F4 ? 4 * NV : NV;

  __device__ __forceinline__ static void zero(float (&x)[N]) {
#pragma unroll
    for (int e = 0; e < N; ++e) x[e] = 0.0f;
  }
  __device__ __forceinline__ static void load(const float* __restrict__ row, int sl, int D,
                                              float (&x)[N]) {
    if (row == nullptr) {
      zero(x);
      return;
    }
    if constexpr (F4) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int d0 = 4 * (sl + LPR * v);
        if (d0 < D) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(row + d0));
          x[4 * v] = t.x; x[4 * v + 1] = t.y; x[4 * v + 2] = t.z; x[4 * v + 3] = t.w;
        } else {
          x[4 * v] = x[4 * v + 1] = x[4 * v + 2] = x[4 * v + 3] = 0.0f;
        }
      }
    } else {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int d = sl + LPR * v;
        x[v] = d < D ? __ldg(row + d) : 0.0f;
      }
    }
  }
  // plain (coherent) load, for rows that are read-modify-written
  __device__ __forceinline__ static void load_rw(const float* row, int sl, int D, float (&x)[N]) {
    if constexpr (F4) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int d0 = 4 * (sl + LPR * v);
        if (d0 < D) {
          const float4 t = *reinterpret_cast<const float4*>(row + d0);
          x[4 * v] = t.x; x[4 * v + 1] = t.y; x[4 * v + 2] = t.z; x[4 * v + 3] = t.w;
        }
      }
    } else {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int d = sl + LPR * v;
        if (d < D) x[v] = row[d];
      }
    }
  }
  __device__ __forceinline__ static void store(float* row, int sl, int D, const float (&x)[N]) {
    if constexpr (F4) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int d0 = 4 * (sl + LPR * v);
        if (d0 < D)
          *reinterpret_cast<float4*>(row + d0) =
              make_float4(x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
      }
    } else {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int d = sl + LPR * v;
        if (d < D) row[d] = x[v];
      }
    }
  }
};

// Dispatch D -> Slice type.  Supported: D % 4 == 0 up to 1024, else D <= 256.
#define RECD_DISPATCH_SLICE(D, ...)                                                   \
  [&]() -> int {                                                                      \
    const int _d = (D);                                                               \
    if (_d <= 0) return RECD_ERR_ARG;                                                 \
    if (_d % 4 == 0) {                                                                \
      const int _v = _d / 4;                                                          \
      if (_v <= 1) { using S = ::recd::Slice<1, 1, true>; __VA_ARGS__ }               \
      else if (_v <= 2) { using S = ::recd::Slice<2, 1, true>; __VA_ARGS__ }          \
      else if (_v <= 4) { using S = ::recd::Slice<4, 1, true>; __VA_ARGS__ }          \
      else if (_v <= 8) { using S = ::recd::Slice<8, 1, true>; __VA_ARGS__ }          \
      else if (_v <= 16) { using S = ::recd::Slice<16, 1, true>; __VA_ARGS__ }        \
      else if (_v <= 32) { using S = ::recd::Slice<32, 1, true>; __VA_ARGS__ }        \
      else if (_v <= 64) { using S = ::recd::Slice<32, 2, true>; __VA_ARGS__ }        \
      else if (_v <= 128) { using S = ::recd::Slice<32, 4, true>; __VA_ARGS__ }       \
      else if (_v <= 256) { using S = ::recd::Slice<32, 8, true>; __VA_ARGS__ }       \
      else return RECD_ERR_UNSUPPORTED;                                               \
    } else {                                                                          \
      if (_d <= 1) { using S = ::recd::Slice<1, 1, false>; __VA_ARGS__ }              \
      else if (_d <= 2) { using S = ::recd::Slice<2, 1, false>; __VA_ARGS__ }         \
      else if (_d <= 4) { using S = ::recd::Slice<4, 1, false>; __VA_ARGS__ }         \
      else if (_d <= 8) { using S = ::recd::Slice<8, 1, false>; __VA_ARGS__ }         \
      else if (_d <= 16) { using S = ::recd::Slice<16, 1, false>; __VA_ARGS__ }       \
      else if (_d <= 32) { using S = ::recd::Slice<32, 1, false>; __VA_ARGS__ }       \
      else if (_d <= 64) { using S = ::recd::Slice<32, 2, false>; __VA_ARGS__ }       \
      else if (_d <= 128) { using S = ::recd::Slice<32, 4, false>; __VA_ARGS__ }      \
      else if (_d <= 256) { using S = ::recd::Slice<32, 8, false>; __VA_ARGS__ }      \
      else return RECD_ERR_UNSUPPORTED;                                               \
    }                                                                                 \
    return RECD_OK;                                                                   \
  }()

// ---------------------------------------------------------------------------
// numpy's float32 add.reduceat order for one row a[0..n):
//   out = a[0] + P(a[1..n)),  P = pairwise_sum (numpy loops_utils.h):
//     m < 8        : r = -0.0; r += x[i] sequentially
//     8 <= m <= 128: 8 accumulators over blocks of 8, combined
//                    ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the m%8 tail
//     m > 128      : P(x[:h]) + P(x[h:]), h = m/2 rounded down to a multiple of 8
// Verified bit-exact against the reference's `pool` (trainer_sim.py:336-343)
// by tests/golden/pool.npz.  Every add is a separately rounded fp32 add.
// ---------------------------------------------------------------------------
template <class S, class Row>
__device__ __forceinline__ void leaf_sum(const Row& row, int64_t a, int64_t m, int sl, int D,
                                         float (&s)[S::N]) {
  constexpr int N = S::N;
  float x[8][N];
  if (m < 8) {
#pragma unroll
    for (int t = 0; t < 7; ++t)
      if (t < m) S::load(row(a + t), sl, D, x[t]);
#pragma unroll
    for (int e = 0; e < N; ++e) s[e] = -0.0f;
#pragma unroll
    for (int t = 0; t < 7; ++t)
      if (t < m) {
#pragma unroll
        for (int e = 0; e < N; ++e) s[e] = __fadd_rn(s[e], x[t][e]);
      }
    return;
  }
  float r[8][N];
#pragma unroll
  for (int k = 0; k < 8; ++k) S::load(row(a + k), sl, D, r[k]);
  const int64_t mb = m - (m % 8);
  for (int64_t i = 8; i < mb; i += 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) S::load(row(a + i + k), sl, D, x[k]);
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int e = 0; e < N; ++e) r[k][e] = __fadd_rn(r[k][e], x[k][e]);
  }
#pragma unroll
  for (int e = 0; e < N; ++e)
    s[e] = __fadd_rn(__fadd_rn(__fadd_rn(r[0][e], r[1][e]), __fadd_rn(r[2][e], r[3][e])),
                     __fadd_rn(__fadd_rn(r[4][e], r[5][e]), __fadd_rn(r[6][e], r[7][e])));
  const int tail = (int)(m - mb);
#pragma unroll
  for (int t = 0; t < 7; ++t)
    if (t < tail) S::load(row(a + mb + t), sl, D, x[t]);
#pragma unroll
  for (int t = 0; t < 7; ++t)
    if (t < tail) {
#pragma unroll
      for (int e = 0; e < N; ++e) s[e] = __fadd_rn(s[e], x[t][e]);
    }
}

// m > 128: the pairwise recursion P(x[:h]) + P(x[h:]) run as an explicit
// post-order DFS (frames + value stack in local memory; only long rows take it).
template <class S, class Row>
__device__ __noinline__ void pairwise_big(const Row row, int64_t a, int64_t m, int sl, int D,
                                          float* out) {
  constexpr int DEPTH = 40;
  int64_t fa[DEPTH], fm[DEPTH];
  int fs[DEPTH];
  float vals[DEPTH][S::N];
  int top = 1, vtop = 0;
  fa[0] = a;
  fm[0] = m;
  fs[0] = 0;
  while (top > 0) {
    const int t = top - 1;
    if (fm[t] <= 128) {
      leaf_sum<S>(row, fa[t], fm[t], sl, D, vals[vtop]);
      ++vtop;
      --top;
      continue;
    }
    int64_t h = fm[t] / 2;
    h -= h % 8;
    if (fs[t] == 0) {
      fs[t] = 1;
      fa[top] = fa[t]; fm[top] = h; fs[top] = 0;
      ++top;
    } else if (fs[t] == 1) {
      fs[t] = 2;
      fa[top] = fa[t] + h; fm[top] = fm[t] - h; fs[top] = 0;
      ++top;
    } else {
      --vtop;
#pragma unroll
      for (int e = 0; e < S::N; ++e) vals[vtop - 1][e] = __fadd_rn(vals[vtop - 1][e], vals[vtop][e]);
      --top;
    }
  }
#pragma unroll
  for (int e = 0; e < S::N; ++e) out[e] = vals[0][e];
}

__device__ __forceinline__ float np_max(float acc, float x) {
  return (acc >= x || isnan(acc)) ? acc : x;  // numpy maximum: first operand on ties / NaN
}

// pool one jagged row a[0..n) (trainer_sim.py:324-344): empty -> 0.
template <class S, class Row>
__device__ __forceinline__ void pool_row(const Row& row, int64_t a, int64_t n, int mode, int sl,
                                         int D, float (&out)[S::N]) {
  constexpr int N = S::N;
  if (n <= 0) {
    S::zero(out);
    return;
  }
  S::load(row(a), sl, D, out);
  if (mode == RECD_POOL_MAX) {
    float x[8][N];
    for (int64_t i = 1; i < n; i += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (i + k < n) S::load(row(a + i + k), sl, D, x[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (i + k < n) {
#pragma unroll
          for (int e = 0; e < N; ++e) out[e] = np_max(out[e], x[k][e]);
        }
    }
    return;
  }
  if (n > 1) {
    float s[N];
    if (n - 1 <= 128) {
      leaf_sum<S>(row, a + 1, n - 1, sl, D, s);
    } else {
      pairwise_big<S, Row>(row, a + 1, n - 1, sl, D, s);
    }
#pragma unroll
    for (int e = 0; e < N; ++e) out[e] = __fadd_rn(out[e], s[e]);
  }
  if (mode == RECD_POOL_AVG) {
    const float fl = (float)n;
#pragma unroll
    for (int e = 0; e < N; ++e) out[e] = __fdiv_rn(out[e], fl);
  }
}

// Row accessors -----------------------------------------------------------
struct TableRows {
  const float* W;
  const int64_t* ids;
  int64_t rows;
  int D;
  int64_t* err;
  int64_t errbase;
  __device__ __forceinline__ const float* operator()(int64_t j) const {
    const int64_t id = ids[j];
    if ((uint64_t)id >= (uint64_t)rows) {
      atomicMin(reinterpret_cast<unsigned long long*>(err), (unsigned long long)(errbase + j));
      return nullptr;
    }
    return W + id * (int64_t)D;
  }
};

struct DenseRows {
  const float* A;
  int D;
  __device__ __forceinline__ const float* operator()(int64_t j) const { return A + j * (int64_t)D; }
};

// find feature f with pref[f] <= w < pref[f+1] (pref in shared memory)
__device__ __forceinline__ int find_seg(const int64_t* pref, int F, int64_t w) {
  int lo = 0, hi = F - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pref[mid] <= w) lo = mid; else hi = mid - 1;
  }
  return lo;
}

}  // namespace recd
