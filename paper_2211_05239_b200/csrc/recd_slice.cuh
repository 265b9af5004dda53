// Column-block row workers and the exact-order pooling reductions shared by
// the forward and backward kernels.
//
// A worker is one warp owning a 32*VW-float column block of an embedding row:
// lane l holds dims [off + l*VW, off + l*VW + VW).  With VW = 2 a warp moves a
// contiguous 256-byte slice per load instruction (LDG.64, fully coalesced);
// a D = 128 row is two workers, D = 64 one.  Reductions are per dimension,
// so splitting a row's dims over warps never changes the arithmetic, and the
// small per-lane state (8 accumulators x 2 floats) keeps kernels at <= 64
// registers, i.e. >= 32 resident warps per SM to hide gather latency.
#pragma once

#include "recd_common.cuh"

namespace recd {

template <int VW_, bool FULL_ = false>
struct Col {
  static constexpr int VW = VW_;
  static constexpr bool FULL = FULL_;  // D is a multiple of CB: every lane is in range
  static constexpr int CB = 32 * VW;   // floats per column block

  __device__ __forceinline__ static void zero(float (&x)[VW]) {
#pragma unroll
    for (int e = 0; e < VW; ++e) x[e] = 0.0f;
  }
  // p points at this lane's first float; ok = lane's slice lies inside the row.
  // Read-only path: tables are never written by the kernels that use it.
  __device__ __forceinline__ static void ld(const float* __restrict__ p, bool ok, float (&x)[VW]) {
    if (!FULL && !ok) {
      zero(x);
      return;
    }
    if constexpr (VW == 4) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(p));
      x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
    } else if constexpr (VW == 2) {
      const float2 t = __ldg(reinterpret_cast<const float2*>(p));
      x[0] = t.x; x[1] = t.y;
    } else {
      x[0] = __ldg(p);
    }
  }
  // coherent load, for rows that are read-modify-written
  __device__ __forceinline__ static void ld_rw(const float* p, bool ok, float (&x)[VW]) {
    if (!FULL && !ok) {
      zero(x);
      return;
    }
    if constexpr (VW == 4) {
      const float4 t = *reinterpret_cast<const float4*>(p);
      x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
    } else if constexpr (VW == 2) {
      const float2 t = *reinterpret_cast<const float2*>(p);
      x[0] = t.x; x[1] = t.y;
    } else {
      x[0] = *p;
    }
  }
  __device__ __forceinline__ static void st(float* p, bool ok, const float (&x)[VW]) {
    if (!FULL && !ok) return;
    if constexpr (VW == 4) {
      *reinterpret_cast<float4*>(p) = make_float4(x[0], x[1], x[2], x[3]);
    } else if constexpr (VW == 2) {
      *reinterpret_cast<float2*>(p) = make_float2(x[0], x[1]);
    } else {
      *p = x[0];
    }
  }
};

// (row, column block) of work item w for a D-wide row
struct ColWork {
  int64_t row;
  int lo;   // this lane's first float inside a row: block offset + lane * VW
  bool ok;  // the lane's slice lies inside the row
};
template <class C>
__device__ __forceinline__ ColWork col_work(int64_t w, int D, int lane) {
  const int ncb = (D + C::CB - 1) / C::CB;
  ColWork c;
  c.row = (ncb == 1) ? w : (ncb == 2 ? (w >> 1) : w / ncb);
  const int cb = (int)(w - c.row * ncb);
  c.lo = cb * C::CB + lane * C::VW;
  c.ok = c.lo < D;
  return c;
}
template <class C>
__host__ __device__ __forceinline__ int col_blocks(int D) {
  return (D + C::CB - 1) / C::CB;
}

// Dispatch D -> Col type: float4 lanes (one 512-byte row slice per warp load)
// when D % 4 == 0 and D >= 64, float2 lanes when D is even, else scalars.
#define RECD_DISPATCH_COL(D, ...) RECD_DISPATCH_COL_VW(D, 4, 1, __VA_ARGS__)
#define RECD_DISPATCH_COL_VW(D, MAXVW, FULLOK, ...)             \
  [&]() -> int {                                                \
    const int _d = (D);                                         \
    if (_d <= 0) return RECD_ERR_ARG;                           \
    if ((FULLOK) && (MAXVW) >= 4 && _d % 128 == 0) { using C = ::recd::Col<4, true>; __VA_ARGS__ } \
    else if ((MAXVW) >= 4 && _d % 4 == 0 && _d >= 64) { using C = ::recd::Col<4>; __VA_ARGS__ } \
    else if ((FULLOK) && _d % 64 == 0) { using C = ::recd::Col<2, true>; __VA_ARGS__ } \
    else if (_d % 2 == 0) { using C = ::recd::Col<2>; __VA_ARGS__ } \
    else { using C = ::recd::Col<1>; __VA_ARGS__ }              \
    return RECD_OK;                                             \
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
// `row(j)` returns the base pointer of value j's embedding row (nullptr = zeros).
// ---------------------------------------------------------------------------
template <class C, class Row>
__device__ __forceinline__ void ld_row(Row& row, int64_t j, bool ok, float (&x)[C::VW]) {
  row.template fetch<C>(j, ok, x);
}
// predicated variant: the row address (ID shuffle) is computed by the whole
// warp unconditionally, only the load is predicated -- no divergent region
template <class C, class Row>
__device__ __forceinline__ void ld_row_if(Row& row, int64_t j, bool pred, bool ok,
                                          float (&x)[C::VW]) {
  const float* pt = row(j);
  if (pred) C::ld(pt, ok, x);
}

template <class C, class Row>
__device__ __forceinline__ void leaf_sum(Row& row, int64_t a, int64_t m, bool ok,
                                         float (&s)[C::VW]) {
  constexpr int V = C::VW;
#define ld(j, x) ld_row<C>(row, (j), ok, x)
  float x[8][V];
  if (m < 8) {
    row.need(a, (int)m);
#pragma unroll
    for (int t = 0; t < 7; ++t) ld_row_if<C>(row, a + t, t < m, ok, x[t]);
#pragma unroll
    for (int e = 0; e < V; ++e) s[e] = -0.0f;
#pragma unroll
    for (int t = 0; t < 7; ++t)
      if (t < m) {
#pragma unroll
        for (int e = 0; e < V; ++e) s[e] = __fadd_rn(s[e], x[t][e]);
      }
    return;
  }
  float r[8][V];
  row.need(a, 8);
#pragma unroll
  for (int k = 0; k < 8; ++k) ld(a + k, r[k]);
  const int64_t mb = m - (m % 8);
  for (int64_t i = 8; i < mb; i += 8) {
    row.need(a + i, 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) ld(a + i + k, x[k]);
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int e = 0; e < V; ++e) r[k][e] = __fadd_rn(r[k][e], x[k][e]);
  }
#pragma unroll
  for (int e = 0; e < V; ++e)
    s[e] = __fadd_rn(__fadd_rn(__fadd_rn(r[0][e], r[1][e]), __fadd_rn(r[2][e], r[3][e])),
                     __fadd_rn(__fadd_rn(r[4][e], r[5][e]), __fadd_rn(r[6][e], r[7][e])));
  const int tail = (int)(m - mb);
  if (tail) row.need(a + mb, tail);
#pragma unroll
  for (int t = 0; t < 7; ++t) ld_row_if<C>(row, a + mb + t, t < tail, ok, x[t]);
#pragma unroll
  for (int t = 0; t < 7; ++t)
    if (t < tail) {
#pragma unroll
      for (int e = 0; e < V; ++e) s[e] = __fadd_rn(s[e], x[t][e]);
    }
#undef ld
}

// P over any m: the recursion P(x[:h]) + P(x[h:]) (m > 128) runs as an
// explicit post-order DFS (frames + value stack in local memory); m <= 128 is a
// single leaf.  One inlined leaf copy keeps register pressure low.
template <int V>
struct Vals {
  float v[V];
};

template <class C, class Row>
__device__ __forceinline__ Vals<C::VW> pairwise_big(Row& row, int64_t a, int64_t m, bool ok) {
  constexpr int DEPTH = 40;
  int64_t fa[DEPTH], fm[DEPTH];
  int fs[DEPTH];
  float vals[DEPTH][C::VW];
  int top = 1, vtop = 0;
  fa[0] = a;
  fm[0] = m;
  fs[0] = 0;
  while (top > 0) {
    const int t = top - 1;
    if (fm[t] <= 128) {
      leaf_sum<C>(row, fa[t], fm[t], ok, vals[vtop]);
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
      for (int e = 0; e < C::VW; ++e) vals[vtop - 1][e] = __fadd_rn(vals[vtop - 1][e], vals[vtop][e]);
      --top;
    }
  }
  Vals<C::VW> out;
#pragma unroll
  for (int e = 0; e < C::VW; ++e) out.v[e] = vals[0][e];
  return out;
}

__device__ __forceinline__ float np_max(float acc, float x) {
  return (acc >= x || isnan(acc)) ? acc : x;  // numpy maximum: first operand on ties / NaN
}

// pool one jagged row a[0..n) (trainer_sim.py:324-344): empty -> 0.
template <class C, class Row>
__device__ __forceinline__ void pool_row(Row& row, int64_t a, int64_t n, int mode, bool ok,
                                         float (&out)[C::VW]) {
  constexpr int V = C::VW;
  if (n <= 0) {
    C::zero(out);
    return;
  }
  row.need(a, 1);
  row.template fetch<C>(a, ok, out);
  if (mode == RECD_POOL_MAX) {
    float x[8][V];
    for (int64_t i = 1; i < n; i += 8) {
      row.need(a + i, (int)min((int64_t)8, n - i));
#pragma unroll
      for (int k = 0; k < 8; ++k) ld_row_if<C>(row, a + i + k, i + k < n, ok, x[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (i + k < n) {
#pragma unroll
          for (int e = 0; e < V; ++e) out[e] = np_max(out[e], x[k][e]);
        }
    }
    return;
  }
  if (n > 1) {
    // one code path for every length: a single leaf when n - 1 <= 128
    const Vals<V> s = pairwise_big<C, Row>(row, a + 1, n - 1, ok);
#pragma unroll
    for (int e = 0; e < V; ++e) out[e] = __fadd_rn(out[e], s.v[e]);
  }
  if (mode == RECD_POOL_AVG) {
    const float fl = (float)n;
#pragma unroll
    for (int e = 0; e < V; ++e) out[e] = __fdiv_rn(out[e], fl);
  }
}

// Row accessors -----------------------------------------------------------
// Table rows addressed through a warp-wide window of 32 IDs: lane l holds the
// ID at position base + l (loaded once, coalesced, range-checked lane-parallel)
// and every row gather gets its ID with one shuffle, so the gathers of a batch
// issue back to back instead of each waiting on its own ID load.  An
// out-of-range ID is recorded in `err` (the host raises the reference's
// ValueError) and reads row 0 so the gather stays branch-free.
struct TableRows {
  const float* Wl;  // table + this lane's first float
  const int64_t* ids;
  int64_t end;      // one past the last valid position
  int64_t rows;
  uint32_t D;
  int64_t* err;
  int64_t errbase;
  int lane;
  int64_t base;
  uint32_t mine;

  __device__ __forceinline__ void window(int64_t j) {
    base = j;
    const int64_t q = j + lane;
    mine = 0;
    if (q < end) {
      const int64_t id = __ldg(ids + q);
      if ((uint64_t)id < (uint64_t)rows) {
        mine = (uint32_t)id;
      } else {
        atomicMin(reinterpret_cast<unsigned long long*>(err), (unsigned long long)(errbase + q));
      }
    }
  }
  // make positions [j, j + n) (n <= 32) available
  __device__ __forceinline__ void need(int64_t j, int n) {
    if (j < base || j + n > base + 32) window(j);
  }
  __device__ __forceinline__ const float* operator()(int64_t j) const {
    const uint32_t id = __shfl_sync(0xffffffffu, mine, (int)(j - base));
    return Wl + (uint64_t)id * D;
  }
  template <class C>
  __device__ __forceinline__ void fetch(int64_t j, bool ok, float (&x)[C::VW]) {
    C::ld((*this)(j), ok, x);
  }
};

// Warp-wide window of 32 consecutive uint32 values (lane l holds base + l).
struct U32Win {
  const uint32_t* p;
  int64_t end;
  int lane;
  int64_t base;
  uint32_t mine;
  __device__ __forceinline__ void window(int64_t j) {
    base = j;
    const int64_t q = j + lane;
    mine = q < end ? __ldg(p + q) : 0u;
  }
  __device__ __forceinline__ void need(int64_t j, int n) {
    if (j < base || j + n > base + 32) window(j);
  }
  __device__ __forceinline__ uint32_t get(int64_t j) const {
    return __shfl_sync(0xffffffffu, mine, (int)(j - base));
  }
};

struct DenseRows {
  const float* Al;  // activations + this lane's first float
  int D;
  __device__ __forceinline__ void need(int64_t, int) {}
  __device__ __forceinline__ const float* operator()(int64_t j) const { return Al + j * (int64_t)D; }
  template <class C>
  __device__ __forceinline__ void fetch(int64_t j, bool ok, float (&x)[C::VW]) {
    C::ld((*this)(j), ok, x);
  }
};

// find segment f with pref[f] <= w < pref[f+1] (pref in shared memory)
__device__ __forceinline__ int find_seg(const int64_t* pref, int F, int64_t w) {
  int lo = 0, hi = F - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pref[mid] <= w) lo = mid; else hi = mid - 1;
  }
  return lo;
}

}  // namespace recd
