// Pooled embedding lookup over unique rows + inverse expansion (sm_100a).
//
// Replaces trainer_sim.embedding_lookup + pool + b[inv]
// (/root/reference/pkg/src/sessiondedup/trainer_sim.py:308-344, 539-561).
// The reference materialises weights[vals] ([N_u, D]) and reduces it with
// ufunc.reduceat; here one warp per (unique row, 64-float column block)
// gathers the table rows with coalesced 64-bit lane loads straight into
// registers and reduces them in numpy's exact summation order, so the
// [N_u, D] activations never touch HBM.
#include "recd_slice.cuh"

// Tuning knobs of the forward gather (overridable with -D at build time).
#ifndef RECD_PEER_MAXSEG
#define RECD_PEER_MAXSEG 8  // ranks a fused pooled-row scatter can address
#endif
#ifndef RECD_POOL_VW
#define RECD_POOL_VW 4
#endif
#ifndef RECD_POOL_MINB
#define RECD_POOL_MINB 2
#endif
// ring variant (sum / avg): K rows in flight per warp through shared memory
#ifndef RECD_POOL_RING
#define RECD_POOL_RING 1
#endif
#ifndef RECD_RING_CA
#define RECD_RING_CA 0
#endif
#ifndef RECD_RING_K
#define RECD_RING_K 2
#endif
#ifndef RECD_RING_MINB
#define RECD_RING_MINB 3
#endif


namespace recd {

struct PoolParams {
  int F;
  int D;
  int mode;
  int64_t B;
  const float* tables[RECD_MAX_FEAT];
  int64_t table_rows[RECD_MAX_FEAT];
  const int64_t* uvalues[RECD_MAX_FEAT];
  const int64_t* uoffsets[RECD_MAX_FEAT];
  const int64_t* inverse[RECD_MAX_FEAT];
  float* pooled[RECD_MAX_FEAT];
  float* out[RECD_MAX_FEAT];
  const int64_t* counts;  // [2 * Ftot] device, already offset by the chunk's f0
  int64_t Ftot;
  int64_t* err;
  int f0;                 // global index of feature 0 of this chunk (error packing)
  // optional scatter of the pooled rows to peers (fused owner -> source return):
  // rows [row0[f][s], row0[f][s + 1]) of feature f go to dst[f][s] (NVLink
  // memory of source s), row0 read from the device (exchange plan)
  int nseg;
  const int64_t* seg_row0[RECD_MAX_FEAT];   // device: nseg bases, ascending
  float* seg_dst[RECD_MAX_FEAT][RECD_PEER_MAXSEG];
  // optional fused expansion through the inverse CSR (recd_pool_fwd_csr): the
  // pooled row u goes straight to out[f][i] for the batch rows i of u,
  // csr_rows[f][csr_start[f][u] .. csr_start[f][u + 1]); pooled[f] may be null
  const int32_t* csr_start[RECD_MAX_FEAT];
  const uint32_t* csr_rows[RECD_MAX_FEAT];
};

// pooled row u of feature f -> its destination(s): with a CSR, the batch rows
// of u (streaming stores: written once, read by the dense model), plus the
// pooled buffer if one is given; else the pooled buffer / peer segment
template <class C>
__device__ __forceinline__ void store_pooled(const PoolParams& p, int f, int64_t u,
                                             const ColWork& cw, const float (&acc)[C::VW]);

// destination row of pooled row u of feature f (peer segment or local buffer)
__device__ __forceinline__ float* pooled_row(const PoolParams& p, int f, int64_t u) {
  if (p.nseg == 0) return p.pooled[f] + u * p.D;
  int s = 0;
  const int64_t* r0 = p.seg_row0[f];
  while (s + 1 < p.nseg && __ldg(r0 + s + 1) <= u) ++s;
  return p.seg_dst[f][s] + (u - __ldg(r0 + s)) * p.D;
}

template <class C>
__device__ __forceinline__ void store_pooled(const PoolParams& p, int f, int64_t u,
                                             const ColWork& cw, const float (&acc)[C::VW]) {
  const int32_t* cs = p.csr_start[f];
  if (cs) {
    const int32_t c0 = __ldg(cs + u), c1 = __ldg(cs + u + 1);
    const uint32_t* R = p.csr_rows[f];
    float* o = p.out[f] + cw.lo;
    const int lane = threadIdx.x & 31;
    for (int32_t j0 = c0; j0 < c1; j0 += 32) {
      const uint32_t mine = (j0 + lane < c1) ? __ldg(R + j0 + lane) : 0u;
      const int m = min(32, c1 - j0);
      for (int t = 0; t < m; ++t) {
        const uint32_t i = __shfl_sync(0xffffffffu, mine, t);
        float* dst = o + (int64_t)i * p.D;
        if constexpr (C::VW == 4) {
          if (C::FULL || cw.ok) __stcs(reinterpret_cast<float4*>(dst), make_float4(acc[0], acc[1], acc[2], acc[3]));
        } else {
          C::st(dst, cw.ok, acc);
        }
      }
    }
    if (!p.pooled[f]) return;
  }
  C::st(pooled_row(p, f, u) + cw.lo, cw.ok, acc);
}

template <class C>
__global__ void __launch_bounds__(256, RECD_POOL_MINB) k_pool_fwd(const __grid_constant__ PoolParams p) {
  RECD_PDL_PROLOGUE();
  __shared__ int64_t s_pref[RECD_MAX_FEAT + 1];
  const int ncb = col_blocks<C>(p.D);
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int f = 0; f < p.F; ++f) {
      s_pref[f] = acc;
      acc += p.counts[f] * ncb;
    }
    s_pref[p.F] = acc;
  }
  __syncthreads();
  const int64_t total = s_pref[p.F];
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total;
       w += nwarps) {
    const int f = find_seg(s_pref, p.F, w);
    const ColWork cw = col_work<C>(w - s_pref[f], p.D, lane);
    const int64_t u = cw.row;
    const int64_t U = p.counts[f], N = p.counts[p.Ftot + f];
    const int64_t* uo = p.uoffsets[f];
    const int64_t a = uo[u];
    const int64_t e = (u + 1 < U) ? uo[u + 1] : N;
    TableRows row{p.tables[f] + cw.lo, p.uvalues[f], e, p.table_rows[f], (uint32_t)p.D, p.err,
                  (int64_t)(p.f0 + f) << 40, lane, 0, 0};
    row.window(a);
    float acc[C::VW];
    pool_row<C>(row, a, e - a, p.mode, cw.ok, acc);
    store_pooled<C>(p, f, u, cw, acc);
  }
}

#ifndef RECD_EXPAND_RF
#define RECD_EXPAND_RF 8
#endif
constexpr int EXP_RF = RECD_EXPAND_RF;  // row copies in flight per lane
#ifndef RECD_EXPAND_CS
#define RECD_EXPAND_CS 1
#endif
// out[f][i] = pooled[f][inverse[f][i]]  (trainer_sim.py:558-561)
// Warp per (32-row block, column block): one coalesced load of the 32 inverse
// entries, then the rows' slices are gathered 8 at a time (8 loads in flight
// per lane) and streamed out.
template <class C>
__global__ void __launch_bounds__(256) k_expand(const __grid_constant__ PoolParams p) {
  RECD_PDL_PROLOGUE();
  __shared__ int64_t s_pref[RECD_MAX_FEAT + 1];
  const int ncb = col_blocks<C>(p.D);
  const int64_t rb = ceil_div(p.B, 32);  // 32-row blocks per feature
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int f = 0; f < p.F; ++f) {
      s_pref[f] = acc;
      const bool active = p.out[f] != nullptr && p.out[f] != p.pooled[f];
      acc += active ? rb * ncb : 0;
    }
    s_pref[p.F] = acc;
  }
  __syncthreads();
  const int64_t total = s_pref[p.F];
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total;
       w += nwarps) {
    const int f = find_seg(s_pref, p.F, w);
    const ColWork cw = col_work<C>(w - s_pref[f], p.D, lane);  // cw.row = 32-row block
    const int64_t i0 = cw.row * 32;
    const int nr = (int)min((int64_t)32, p.B - i0);
    const int64_t my = (lane < nr) ? (p.inverse[f] ? __ldg(p.inverse[f] + i0 + lane) : i0 + lane) : 0;
    const float* src = p.pooled[f] + cw.lo;
    float* dst = p.out[f] + i0 * p.D + cw.lo;
    for (int r0 = 0; r0 < nr; r0 += EXP_RF) {
      float x[EXP_RF][C::VW];
#pragma unroll
      for (int t = 0; t < EXP_RF; ++t) {
        const int64_t u = __shfl_sync(0xffffffffu, my, (r0 + t) & 31);
        if (r0 + t < nr) C::ld(src + u * p.D, cw.ok, x[t]);
      }
#pragma unroll
      for (int t = 0; t < EXP_RF; ++t)
        if (r0 + t < nr) {
          if constexpr (RECD_EXPAND_CS && C::VW == 4) {  // streaming store: keep pooled rows in L2
            if (C::FULL || cw.ok)
              __stcs(reinterpret_cast<float4*>(dst + (int64_t)(r0 + t) * p.D),
                     make_float4(x[t][0], x[t][1], x[t][2], x[t][3]));
          } else {
            C::st(dst + (int64_t)(r0 + t) * p.D, cw.ok, x[t]);
          }
        }
    }
  }
}

template <class C>
__global__ void __launch_bounds__(256) k_lookup(const float* W, int64_t rows, int D,
                                                const int64_t* ids, int64_t n, float* out,
                                                int64_t* err) {
  RECD_PDL_PROLOGUE();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t total = n * col_blocks<C>(D);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total;
       w += nwarps) {
    const ColWork cw = col_work<C>(w, D, lane);
    TableRows row{W + cw.lo, ids, n, rows, (uint32_t)D, err, 0, lane, 0, 0};
    row.window(cw.row);
    float x[C::VW];
    C::ld(row(cw.row), cw.ok, x);
    C::st(out + cw.row * D + cw.lo, cw.ok, x);
  }
}

template <class C>
__global__ void __launch_bounds__(256, 3) k_pool_dense(const float* A, int64_t nvals, int D,
                                                       const int64_t* offsets, int64_t nrows,
                                                       int mode, float* out) {
  RECD_PDL_PROLOGUE();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t total = nrows * col_blocks<C>(D);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total;
       w += nwarps) {
    const ColWork cw = col_work<C>(w, D, lane);
    DenseRows row{A + cw.lo, D};
    const int64_t r = cw.row;
    const int64_t a = offsets[r];
    const int64_t e = (r + 1 < nrows) ? offsets[r + 1] : nvals;
    float acc[C::VW];
    pool_row<C>(row, a, e - a, mode, cw.ok, acc);
    C::st(out + r * D + cw.lo, cw.ok, acc);
  }
}

// ---------------------------------------------------------------------------
// Ring variant of k_pool_fwd (sum / avg, float4 lanes).  The table rows of a
// jagged row are streamed in position order through a per-warp shared-memory
// ring of K slots with cp.async (16 bytes per lane, one 512-byte row slice per
// warp instruction): rows in flight hold no registers, so a warp keeps K rows
// in flight at ~80 registers instead of 8 at 128.  numpy's pairwise tree
// visits the values strictly left to right, so the reduction consumes the
// ring in order and stays bit-identical to pool_row / leaf_sum.
// ---------------------------------------------------------------------------
// Values 1.. of a row (value 0 is loaded directly) stream through the ring in
// batches of 8 positions.  numpy's pairwise split points h are multiples of 8,
// so relative to value 1 every leaf of the tree starts on a batch boundary and
// only the row's last batch can be partial: the reduction consumes whole
// batches (one wait + one refill per 8 rows, a handful of code sites).
template <int NB>
struct RingRows {
  float* ring;              // this lane's 16 bytes of slot 0 (slot stride 128 floats)
  const float* Wl;
  const int64_t* ids;       // IDs of positions 0.. of the streamed values
  int32_t n;                // streamed values
  int64_t rows;
  uint32_t D;
  int64_t* err;
  int64_t errpos;           // (feature << 40) | absolute position of streamed value 0
  int lane;
  bool ok;
  int32_t wb;               // IDs of positions [wb, wb + 32) in cur, the next 32 in nraw
  uint32_t cur;
  int64_t nraw;             // raw ID of position wb + 32 + lane: range-checked only when
                            // it becomes cur, so its load latency is not exposed at issue
  int32_t b;                // batches consumed

  __device__ __forceinline__ int64_t raw_id(int32_t q) const { return q < n ? __ldg(ids + q) : 0; }
  __device__ __forceinline__ uint32_t check_id(int64_t id, int32_t q) const {
    if (q >= n) return 0u;
    if ((uint64_t)id < (uint64_t)rows) return (uint32_t)id;
    atomicMin(reinterpret_cast<unsigned long long*>(err), (unsigned long long)(errpos + q));
    return 0u;
  }
  // positions [8 bi, 8 bi + 8) -> slots of batch bi % NB, one commit group
  __device__ __forceinline__ void issue(int32_t bi) {
    const int32_t p0 = bi * 8;
    if (p0 < n) {  // warp-uniform
      if (p0 >= wb + 32) {
        wb += 32;
        cur = check_id(nraw, wb + lane);
        nraw = raw_id(wb + 32 + lane);
      }
      float* dst = ring + (bi % NB) * (8 * 128);
      const int sh = p0 - wb;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t id = __shfl_sync(0xffffffffu, cur, sh + k);
        if (ok && p0 + k < n) {
#if RECD_RING_CA  // L1-allocating: the 8 warps of a CTA pool consecutive unique rows,
                  // which in session data are shifted windows of each other
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + k * 128);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa),
                       "l"(Wl + (uint64_t)id * D));
#else
          cp_async<16>(dst + k * 128, Wl + (uint64_t)id * D);
#endif
        }
      }
    }
    cp_async_commit();
  }
  __device__ __forceinline__ void start() {
    wb = 0;
    const int64_t c0 = raw_id(lane);
    nraw = raw_id(32 + lane);
    cur = check_id(c0, lane);
    b = 0;
#pragma unroll
    for (int i = 0; i < NB; ++i) issue(i);
  }
  // slots of the next batch (after its copies landed)
  __device__ __forceinline__ const float* acquire() {
    cp_async_wait<NB - 1>();
    return ring + (b % NB) * (8 * 128);
  }
  // the batch's values are consumed: reuse its slots for batch b + NB
  __device__ __forceinline__ void release() {
    issue(b + NB);
    ++b;
  }
};

__device__ __forceinline__ float4 slot4(const float* s, int k, bool ok) {
  return ok ? *reinterpret_cast<const float4*>(s + k * 128) : make_float4(0.f, 0.f, 0.f, 0.f);
}

// P(x) over the next m streamed values, m <= 128, starting on a batch boundary
// (same arithmetic as leaf_sum)
template <class RR>
__device__ __forceinline__ void leaf_ring(RR& rr, int32_t m, float (&s)[4]) {
  if (m < 8) {
#pragma unroll
    for (int e = 0; e < 4; ++e) s[e] = -0.0f;
    const float* sl = rr.acquire();
    for (int t = 0; t < m; ++t) {
      const float4 v = slot4(sl, t, rr.ok);
      s[0] = __fadd_rn(s[0], v.x);
      s[1] = __fadd_rn(s[1], v.y);
      s[2] = __fadd_rn(s[2], v.z);
      s[3] = __fadd_rn(s[3], v.w);
    }
    rr.release();
    return;
  }
  float r[8][4];
  {
    const float* sl = rr.acquire();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 v = slot4(sl, k, rr.ok);
      r[k][0] = v.x;
      r[k][1] = v.y;
      r[k][2] = v.z;
      r[k][3] = v.w;
    }
    rr.release();
  }
  const int32_t nb = m >> 3;
  for (int32_t i = 1; i < nb; ++i) {
    const float* sl = rr.acquire();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 v = slot4(sl, k, rr.ok);
      r[k][0] = __fadd_rn(r[k][0], v.x);
      r[k][1] = __fadd_rn(r[k][1], v.y);
      r[k][2] = __fadd_rn(r[k][2], v.z);
      r[k][3] = __fadd_rn(r[k][3], v.w);
    }
    rr.release();
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
    s[e] = __fadd_rn(__fadd_rn(__fadd_rn(r[0][e], r[1][e]), __fadd_rn(r[2][e], r[3][e])),
                     __fadd_rn(__fadd_rn(r[4][e], r[5][e]), __fadd_rn(r[6][e], r[7][e])));
  const int tail = m & 7;
  if (tail) {
    const float* sl = rr.acquire();
    for (int t = 0; t < tail; ++t) {
      const float4 v = slot4(sl, t, rr.ok);
      s[0] = __fadd_rn(s[0], v.x);
      s[1] = __fadd_rn(s[1], v.y);
      s[2] = __fadd_rn(s[2], v.z);
      s[3] = __fadd_rn(s[3], v.w);
    }
    rr.release();
  }
}

// P over any m (pairwise_big's post-order DFS; positions implicit, every leaf
// starts on a batch boundary because every split point is a multiple of 8)
template <class RR>
__device__ __forceinline__ void pairwise_ring(RR& rr, int32_t m, float (&out)[4]) {
  if (m <= 128) {
    leaf_ring(rr, m, out);
    return;
  }
  constexpr int DEPTH = 32;
  int32_t fm[DEPTH];
  int fs[DEPTH];
  float vals[DEPTH][4];
  int top = 1, vtop = 0;
  fm[0] = m;
  fs[0] = 0;
  while (top > 0) {
    const int t = top - 1;
    if (fm[t] <= 128) {
      float sv[4];
      leaf_ring(rr, fm[t], sv);
#pragma unroll
      for (int e = 0; e < 4; ++e) vals[vtop][e] = sv[e];
      ++vtop;
      --top;
      continue;
    }
    int32_t h = fm[t] / 2;
    h -= h % 8;
    if (fs[t] == 0) {
      fs[t] = 1;
      fm[top] = h;
      fs[top] = 0;
      ++top;
    } else if (fs[t] == 1) {
      fs[t] = 2;
      fm[top] = fm[t] - h;
      fs[top] = 0;
      ++top;
    } else {
      --vtop;
#pragma unroll
      for (int e = 0; e < 4; ++e) vals[vtop - 1][e] = __fadd_rn(vals[vtop - 1][e], vals[vtop][e]);
      --top;
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) out[e] = vals[0][e];
}

// one unique row u of feature f through this warp's own ring (value 0
// straight into registers, values 1.. through the ring; value 0's ID is
// range-checked after the ring's first IDs were loaded, so the two loads overlap)
template <class C, int K>
__device__ __forceinline__ void pool_row_ring(const PoolParams& p, int f, const ColWork& cw,
                                              float* ring, int lane) {
  const int64_t u = cw.row;
  const int64_t U = p.counts[f], N = p.counts[p.Ftot + f];
  const int64_t* uo = p.uoffsets[f];
  const int64_t a = uo[u];
  const int64_t e = (u + 1 < U) ? uo[u + 1] : N;
  const int64_t n = e - a;
  float acc[4];
  if (n <= 0) {
    C::zero(acc);
  } else {
    const int64_t id0 = __ldg(p.uvalues[f] + a);
    auto row0 = [&]() -> uint64_t {
      if ((uint64_t)id0 < (uint64_t)p.table_rows[f]) return (uint64_t)id0;
      if (lane == 0)
        atomicMin(reinterpret_cast<unsigned long long*>(p.err),
                  (unsigned long long)(((int64_t)(p.f0 + f) << 40) + a));
      return 0;
    };
    if (n > 1) {
      RingRows<K> rr;
      rr.ring = ring;
      rr.Wl = p.tables[f] + cw.lo;
      rr.ids = p.uvalues[f] + a + 1;
      rr.n = (int32_t)(n - 1);
      rr.rows = p.table_rows[f];
      rr.D = (uint32_t)p.D;
      rr.err = p.err;
      rr.errpos = ((int64_t)(p.f0 + f) << 40) + a + 1;
      rr.lane = lane;
      rr.ok = C::FULL || cw.ok;
      rr.start();
      C::ld(p.tables[f] + cw.lo + row0() * (uint32_t)p.D, cw.ok, acc);
      float sv[4];
      pairwise_ring(rr, (int32_t)(n - 1), sv);
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = __fadd_rn(acc[k], sv[k]);
    } else {
      C::ld(p.tables[f] + cw.lo + row0() * (uint32_t)p.D, cw.ok, acc);
    }
    if (p.mode == RECD_POOL_AVG) {
      const float fl = (float)n;
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = __fdiv_rn(acc[k], fl);
    }
  }
  store_pooled<C>(p, f, u, cw, acc);
}

template <class C, int K>
__global__ void __launch_bounds__(256, RECD_RING_MINB) k_pool_ring(const __grid_constant__ PoolParams p) {
  RECD_PDL_PROLOGUE();
  static_assert(C::VW == 4, "ring pool streams float4 lane slices");
  extern __shared__ __align__(128) float s_ring[];
  __shared__ int64_t s_pref[RECD_MAX_FEAT + 1];
  const int ncb = col_blocks<C>(p.D);
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int f = 0; f < p.F; ++f) {
      s_pref[f] = acc;
      acc += p.counts[f] * ncb;
    }
    s_pref[p.F] = acc;
  }
  __syncthreads();
  const int64_t total = s_pref[p.F];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  float* ring = s_ring + (int64_t)warp * K * 8 * 128 + lane * 4;
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; w < total; w += nwarps) {
    const int f = find_seg(s_pref, p.F, w);
    pool_row_ring<C, K>(p, f, col_work<C>(w - s_pref[f], p.D, lane), ring, lane);
  }
  cp_async_wait<0>();
}

// k_pool_ring for sum / avg with float4 lanes, k_pool_fwd otherwise
template <class C>
static int launch_pool_fwd(const PoolParams& p, int mode, bool share, unsigned grid,
                           cudaStream_t stream) {
  if constexpr (C::VW == 4 && RECD_POOL_RING) {
    if (mode != RECD_POOL_MAX) {
      constexpr int K = RECD_RING_K;  // batches of 8 rows in flight per warp
      constexpr int smem = 8 * K * 8 * 128 * (int)sizeof(float);
      static bool attr[64] = {};
      static int resident[64] = {};
      int dev = 0;
      RECD_CUDA_CHECK(cudaGetDevice(&dev));
      if (dev < 0 || dev >= 64 || !attr[dev]) {
        RECD_CUDA_CHECK(cudaFuncSetAttribute(k_pool_ring<C, K>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int per = 0;
        RECD_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pool_ring<C, K>, 256, smem));
        if (dev >= 0 && dev < 64) attr[dev] = true, resident[dev] = std::max(per, 1);
      }
      // Persistent grid (one wave: each CTA's ring warms up once).  With
      // RECD_POOL_SHARE one slot per SM is left to a kernel running beside
      // the lookup on another stream (TrainStep's occurrence sort).  The
      // RECD_POOL_CTAS env overrides the CTAs per SM.
      static int env_ctas = -1;
      if (env_ctas < 0) {
        const char* e = getenv("RECD_POOL_CTAS");
        env_ctas = e ? std::max(1, atoi(e)) : 0;
      }
      const int res = (dev >= 0 && dev < 64) ? resident[dev] : 1;
      const int per_sm = env_ctas ? env_ctas : std::max(1, share ? res - 1 : res);
      grid = std::min<unsigned>(grid, (unsigned)(num_sms() * per_sm));
      pdl(k_pool_ring<C, K>, grid, 256, smem, stream)(p);
      return RECD_OK;
    }
  }
  pdl(k_pool_fwd<C>, grid, 256, 0, stream)(p);
  return RECD_OK;
}

static unsigned grid_for(int64_t warps) {
  int64_t blocks = ceil_div(std::max<int64_t>(warps, 1), 8);
  const int64_t cap = (int64_t)num_sms() * 16;
  return (unsigned)std::min(blocks, cap);
}

static unsigned expand_grid(int64_t batch_size, int64_t tasks_per_32) {
  return (unsigned)std::min<int64_t>(grid_for(ceil_div(batch_size, 32) * tasks_per_32),
                                     grid_cap("RECD_EX_CTAS", 16));
}

}  // namespace recd

using namespace recd;

static int pool_fwd_impl(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                         const float* const* tables, const int64_t* table_rows,
                         const int64_t* const* uvalues, const int64_t* const* uoffsets,
                         const int64_t* counts, const int64_t* const* inverse,
                         const int32_t* const* csr_start, const uint32_t* const* csr_rows,
                         float* const* pooled_out, float* const* out, int64_t* err,
                         recd_stream_t stream_) {
  recd::PdlScope pdl_scope(batch_size * (int64_t)num_features);
  cudaStream_t stream = (cudaStream_t)stream_;
  const bool csr = csr_start != nullptr;
  const bool share = (mode & RECD_POOL_SHARE) != 0;
  mode &= ~RECD_POOL_SHARE;
  if (num_features <= 0 || batch_size < 0 || dim <= 0 || mode < 0 || mode > 2 || !counts || !err)
    return RECD_ERR_ARG;
  RECD_CUDA_CHECK(cudaMemsetAsync(err, 0x7f, sizeof(int64_t), stream));
  for (int f0 = 0; f0 < num_features; f0 += RECD_MAX_FEAT) {
    PoolParams p;
    memset(&p, 0, sizeof(p));
    p.F = std::min(RECD_MAX_FEAT, num_features - f0);
    p.D = dim;
    p.mode = mode;
    p.B = batch_size;
    p.counts = counts + f0;
    p.Ftot = num_features;
    p.err = err;
    p.f0 = f0;
    for (int f = 0; f < p.F; ++f) {
      p.tables[f] = tables[f0 + f];
      p.table_rows[f] = table_rows[f0 + f];
      p.uvalues[f] = uvalues[f0 + f];
      p.uoffsets[f] = uoffsets[f0 + f];
      p.inverse[f] = inverse ? inverse[f0 + f] : nullptr;
      p.pooled[f] = pooled_out ? pooled_out[f0 + f] : nullptr;
      p.out[f] = out ? out[f0 + f] : nullptr;
      if (csr) {
        // a feature with neither CSR array is an identity (plain KJT) feature:
        // its unique rows are the batch rows, pooled straight into out
        const bool ident = !csr_start[f0 + f] && !csr_rows[f0 + f];
        p.csr_start[f] = csr_start[f0 + f];
        p.csr_rows[f] = csr_rows[f0 + f];
        if ((!ident && (!p.csr_start[f] || !p.csr_rows[f])) || !p.out[f] ||
            (dim % 4 == 0 && (uintptr_t)p.out[f] % 16))
          return RECD_ERR_ARG;
        if (!p.pooled[f]) p.pooled[f] = p.out[f];  // (alignment check below; written only if ident)
      }
      if (!p.tables[f] || !p.uoffsets[f] || !p.pooled[f]) return RECD_ERR_ARG;
      if (dim % 2 == 0 && ((uintptr_t)p.tables[f] % 8 || (uintptr_t)p.pooled[f] % 8 ||
                           (p.out[f] && (uintptr_t)p.out[f] % 8)))
        return RECD_ERR_ARG;
    }
    bool any_expand = false;
    for (int f = 0; f < p.F; ++f) any_expand |= (p.out[f] != nullptr && p.out[f] != p.pooled[f]);
    if (csr) {
      any_expand = false;
      for (int f = 0; f < p.F; ++f)
        if ((!pooled_out || !pooled_out[f0 + f]) && p.csr_start[f]) p.pooled[f] = nullptr;
    }
    int rc = RECD_DISPATCH_COL_VW(dim, RECD_POOL_VW, 1, {
      const unsigned grid = grid_for(batch_size * p.F * col_blocks<C>(dim));
      hook_before("k_pool_fwd", stream);
      const int lrc = launch_pool_fwd<C>(p, mode, share, grid, stream);
      if (lrc != RECD_OK) return lrc;
      hook_after("k_pool_fwd", stream);
      note_launch();
      if (any_expand) {
        pdl(k_expand<C>, expand_grid(batch_size, p.F * col_blocks<C>(dim)), 256, 0, stream)(p);
        note_launch();
      }
    });
    if (rc != RECD_OK) return rc;
    RECD_LAUNCH_CHECK();
  }
  return RECD_OK;
}

extern "C" int recd_pool_fwd(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                             const float* const* tables, const int64_t* table_rows,
                             const int64_t* const* uvalues, const int64_t* const* uoffsets,
                             const int64_t* counts, const int64_t* const* inverse,
                             float* const* pooled_out, float* const* out, int64_t* err,
                             recd_stream_t stream) {
  if (!pooled_out) return RECD_ERR_ARG;
  return pool_fwd_impl(num_features, batch_size, dim, mode, tables, table_rows, uvalues, uoffsets,
                       counts, inverse, nullptr, nullptr, pooled_out, out, err, stream);
}

extern "C" int recd_pool_fwd_csr(int32_t num_features, int64_t batch_size, int32_t dim,
                                 int32_t mode, const float* const* tables,
                                 const int64_t* table_rows, const int64_t* const* uvalues,
                                 const int64_t* const* uoffsets, const int64_t* counts,
                                 const int32_t* const* csr_start, const uint32_t* const* csr_rows,
                                 float* const* pooled_out, float* const* out, int64_t* err,
                                 recd_stream_t stream) {
  if (!csr_start || !csr_rows || !out) return RECD_ERR_ARG;
  return pool_fwd_impl(num_features, batch_size, dim, mode, tables, table_rows, uvalues, uoffsets,
                       counts, nullptr, csr_start, csr_rows, pooled_out, out, err, stream);
}

// Owner-side pooling whose rows go straight to the sources' receive buffers
// over NVLink (the all-to-all of partial rows fused into the pooling kernel):
// feature f's row u lands at seg_dst[f * num_segs + s] + (u - row0[f][s]) * dim
// for the segment s with row0[f][s] <= u < row0[f][s + 1] (row0 on the device,
// num_segs <= 8).  Sum / avg, no expansion.
extern "C" int recd_pool_fwd_scatter(int32_t num_features, int64_t batch_size, int32_t dim,
                                     int32_t mode, const float* const* tables,
                                     const int64_t* table_rows, const int64_t* const* uvalues,
                                     const int64_t* const* uoffsets, const int64_t* counts,
                                     int32_t num_segs, const int64_t* const* seg_row0,
                                     float* const* seg_dst, int64_t* err, recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (num_features <= 0 || num_features > RECD_MAX_FEAT || batch_size < 0 || dim <= 0 ||
      mode < 0 || mode > 2 || !counts || !err || num_segs <= 0 || num_segs > RECD_PEER_MAXSEG ||
      !seg_row0 || !seg_dst)
    return RECD_ERR_ARG;
  RECD_CUDA_CHECK(cudaMemsetAsync(err, 0x7f, sizeof(int64_t), stream));
  PoolParams p;
  memset(&p, 0, sizeof(p));
  p.F = num_features;
  p.D = dim;
  p.mode = mode;
  p.B = batch_size;
  p.counts = counts;
  p.Ftot = num_features;
  p.err = err;
  p.nseg = num_segs;
  for (int f = 0; f < p.F; ++f) {
    p.tables[f] = tables[f];
    p.table_rows[f] = table_rows[f];
    p.uvalues[f] = uvalues[f];
    p.uoffsets[f] = uoffsets[f];
    p.seg_row0[f] = seg_row0[f];
    for (int s = 0; s < num_segs; ++s) {
      p.seg_dst[f][s] = seg_dst[(int64_t)f * num_segs + s];
      if (!p.seg_dst[f][s] || (dim % 2 == 0 && (uintptr_t)p.seg_dst[f][s] % 8)) return RECD_ERR_ARG;
    }
    if (!p.tables[f] || !p.uoffsets[f] || !p.seg_row0[f]) return RECD_ERR_ARG;
  }
  int rc = RECD_DISPATCH_COL_VW(dim, RECD_POOL_VW, 1, {
    const int lrc = launch_pool_fwd<C>(p, mode, false, grid_for(batch_size * p.F * col_blocks<C>(dim)), stream);
    if (lrc != RECD_OK) return lrc;
    note_launch();
  });
  if (rc != RECD_OK) return rc;
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

extern "C" int recd_embedding_lookup(const float* table, int64_t table_rows, int32_t dim,
                                     const int64_t* values, int64_t n, float* out, int64_t* err,
                                     recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (dim <= 0 || n < 0 || !err || (n > 0 && (!table || !values || !out))) return RECD_ERR_ARG;
  RECD_CUDA_CHECK(cudaMemsetAsync(err, 0x7f, sizeof(int64_t), stream));
  if (n == 0) return RECD_OK;
  int rc = RECD_DISPATCH_COL(dim, {
    pdl(k_lookup<C>, grid_for(n * col_blocks<C>(dim)), 256, 0, stream)(table, table_rows, dim,
                                                                      values, n, out, err);
    note_launch();
  });
  if (rc != RECD_OK) return rc;
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

extern "C" int recd_pool_dense(const float* acts, int64_t n_values, int32_t dim,
                               const int64_t* offsets, int64_t n_rows, int32_t mode, float* out,
                               recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (dim <= 0 || n_rows < 0 || mode < 0 || mode > 2) return RECD_ERR_ARG;
  if (n_rows == 0) return RECD_OK;
  int rc = RECD_DISPATCH_COL(dim, {
    pdl(k_pool_dense<C>, grid_for(n_rows * col_blocks<C>(dim)), 256, 0, stream)(
        acts, n_values, dim, offsets, n_rows, mode, out);
    note_launch();
  });
  if (rc != RECD_OK) return rc;
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

extern "C" int recd_expand(int32_t num_features, int64_t batch_size, int32_t dim,
                           const int64_t* const* inverse, const float* const* pooled,
                           float* const* out, recd_stream_t stream_) {
  recd::PdlScope pdl_scope(batch_size * (int64_t)num_features);
  cudaStream_t stream = (cudaStream_t)stream_;
  if (num_features <= 0 || batch_size < 0 || dim <= 0 || !pooled || !out) return RECD_ERR_ARG;
  for (int f0 = 0; f0 < num_features; f0 += RECD_MAX_FEAT) {
    PoolParams p;
    memset(&p, 0, sizeof(p));
    p.F = std::min(RECD_MAX_FEAT, num_features - f0);
    p.D = dim;
    p.B = batch_size;
    for (int f = 0; f < p.F; ++f) {
      p.inverse[f] = inverse ? inverse[f0 + f] : nullptr;
      p.pooled[f] = const_cast<float*>(pooled[f0 + f]);
      p.out[f] = out[f0 + f];
      if (!p.pooled[f] || !p.out[f]) return RECD_ERR_ARG;
    }
    int rc = RECD_DISPATCH_COL(dim, {
      pdl(k_expand<C>, expand_grid(batch_size, p.F * col_blocks<C>(dim)), 256, 0, stream)(p);
      note_launch();
    });
    if (rc != RECD_OK) return rc;
    RECD_LAUNCH_CHECK();
  }
  return RECD_OK;
}
