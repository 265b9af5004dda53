// Backward of the deduplicated pooled lookup + fused SGD (sm_100a).
//
// The reference has no backward (SPEC.md:13 puts training out of scope);
// the definition implemented here is the one in oracle/embedding.py:
//   grad_u[u]  = sum_{i: inv[i] = u} grad_out[i], fp32 from +0.0 in ascending i
//                (avg: divided by fp32(len_u));
//   g[v]       = sum over occurrences of ID v in ascending (feature, u, pos)
//                order of grad_u[u] -- a deterministic sorted scatter-add;
//   SGD        : W[v] -= fp32(lr * g[v]) (no FMA contraction).
// Steps (one launch per phase for every feature of the step):
//   1 inverse CSR  : stable radix sort of (inv[i], i) per group  -> rows of u
//   2 k_grad_u     : worker per unique row, ordered segment reduce
//   3 k_occ        : (ID, (feature << 24) | u) pairs of every unique value, laid out
//                    per table (features sharing a table are concatenated)
//   4 radix sort   : stable by ID within each table segment
//   5 k_scatter    : warp per (256-position chunk of the sorted pairs, column
//                    block); it lists the runs of equal IDs starting in its chunk,
//                    prefetches the table rows of 4 runs at a time, reduces each
//                    run in order and RMWs the row (or emits a sparse gradient row).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>

#include "recd_prims.cuh"
#include "recd_slice.cuh"

#ifndef RECD_BWD_VW
#define RECD_BWD_VW 4
#endif
#ifndef RECD_BWD_FULLOK
#define RECD_BWD_FULLOK 1
#endif
#ifndef RECD_SCATTER_MINB
#define RECD_SCATTER_MINB 4
#endif
// L2 policy of the scatter: 1 = table rows (read + write) evict_first, 2 = also
// unique-row gradient gathers evict_last, 0 = no hints
#ifndef RECD_SCATTER_L2
#define RECD_SCATTER_L2 2
#endif

namespace recd {

#ifndef RECD_RC_BIG
#define RECD_RC_BIG 256
#endif
constexpr int RC_BIG = RECD_RC_BIG;  // sorted positions per scatter work item
#ifndef RECD_RC_SMALL
#define RECD_RC_SMALL 32
#endif
constexpr int RC_SMALL = RECD_RC_SMALL;  // ... when the occurrence arrays are small (latency-bound; cfg1 32 vs 64: 0.130 vs 0.136 ms)
static int rc_for(int64_t occ_total) { return occ_total >= (4ll << 20) ? RC_BIG : RC_SMALL; }

struct BwdParams {
  int F;
  int D;
  int mode;
  int64_t B;
  int apply_sgd;
  float lr;
  int nis;  // inverse segments
  int nts;  // table segments
  // per feature
  const int64_t* uvalues[RECD_MAX_FEAT];
  const int64_t* uoffsets[RECD_MAX_FEAT];
  const float* grad_out[RECD_MAX_FEAT];
  int feat_is[RECD_MAX_FEAT];  // inverse segment or -1 (identity)
  int feat_ts[RECD_MAX_FEAT];  // table segment
  // per inverse segment
  const int64_t* inverse[RECD_MAX_FEAT];
  int is_feat[RECD_MAX_FEAT];  // a feature of the segment (for U)
  // per table segment
  float* table[RECD_MAX_FEAT];
  int64_t ts_base[RECD_MAX_FEAT];    // element base in the occurrence arrays
  int64_t ts_chunk0[RECD_MAX_FEAT];  // first scatter chunk
  int64_t ts_rows[RECD_MAX_FEAT];    // table rows (IDs must lie in [0, rows))
  int64_t* grad_ids[RECD_MAX_FEAT];
  float* grad_rows[RECD_MAX_FEAT];
  int64_t* grad_count[RECD_MAX_FEAT];
  int64_t total_rc_chunks;
  const int64_t* counts;  // [2*Ftot] device, offset to this call's f0
  int64_t Ftot;
  // scratch
  int64_t* feat_base;     // [F] device: offset of feature f inside its table segment
  int64_t* seg_count;     // [nts] device
  int64_t* is_count;      // [nis] device (= B)
  uint32_t* inv_keys;     // [nis][B] sorted
  uint32_t* inv_rows;     // [nis][B]
  int32_t* csr_start;     // [nis][B + 1]
  float* gout[RECD_MAX_FEAT];         // grad_u destination per feature ([U x D])
  const float* grow[RECD_MAX_FEAT];   // unique-row gradients read by the scatter
  const float* seg_grow[RECD_MAX_FEAT];  // per table segment: grow of its only feature, or null
  uint32_t* occ_keys;     // sorted occurrence IDs
  uint32_t* occ_vals;     // tag = (f << 24) | u
  int64_t* run_part;      // [total_rc_chunks] exclusive run counts (grad-output mode)
  int32_t* bad;           // set by k_occ when an ID is outside [0, rows): no table update
  // diagonal-run occurrences (RECD_BWD_RUNS): see k_rv*
  uint32_t* head_tag;     // [occ cap] tag of each run head (indexed by the sort's value)
  uint32_t* head_pos;     // [occ cap] position of the head in its unique row
  uint32_t* head_len;     // [occ cap] run length k (rows tag .. tag + k - 1)
  int64_t* rv_blk;        // [value blocks] heads per block -> exclusive head offsets
  int32_t* fix_list;      // [RV_FIX_CAP][3] IDs whose runs overlap: (segment, first, end head)
  uint32_t* fix_count;
  int seg_feat[RECD_MAX_FEAT];  // the feature of each (single-feature) table segment
  int64_t* head_count;    // [nts] run heads per table segment (the heads sort's counts)
  int64_t* head_off;      // [occ cap] run lengths in sorted order -> exclusive offsets
  int32_t* fallback;      // set when some ID's runs need per-value occurrences
  uint32_t* sc_ticket;    // k_scatter work counter (dynamic chunk order), zeroed per launch
  int sc_dyn;             // k_scatter: warps take chunks from sc_ticket (else grid-stride)
  uint32_t* exp_keys;     // expanded occurrences (the scatter's input)
  uint32_t* exp_vals;
  const int32_t* occ_gate;              // k_occ runs only if null or *occ_gate != 0
  uint32_t* occ_hist;                   // k_occ: add the sort's digit counts here (or null)
  uint64_t gu_mask;                     // k_grad_u(_flat): features to reduce (bit f)
  int64_t sc_chunk_lo, sc_chunk_hi;     // k_scatter: chunk window [lo, hi) of this launch
  int occ_bits;                         //        over this many key bits
  int64_t ex_chunk0[RECD_MAX_FEAT];     // k_rv_expand: first RV_EX_CH block of each segment
  int64_t occ_blk0[RECD_MAX_FEAT + 1];  // k_occ: first block of each feature (capacity)
  int64_t oc_ch;                         // k_occ / k_rv: unique values per block
  // optional scatter of grad_u rows to peers (fused source -> owner push): row u
  // of feature f goes to gseg_dst[f][j] + (*gseg_row0[f][j] + u) * D, j < gsegs
  int gsegs;
  float* gseg_dst[RECD_MAX_FEAT][8];
  const int64_t* gseg_row0[RECD_MAX_FEAT][8];
};

__global__ void k_bwd_setup(const __grid_constant__ BwdParams p) {
  RECD_PDL_PROLOGUE();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  *p.bad = 0;
  *p.fallback = 0;
  for (int s = 0; s < p.nts; ++s) {
    p.seg_count[s] = 0;
    p.head_count[s] = 0;
  }
  for (int f = 0; f < p.F; ++f) {
    const int s = p.feat_ts[f];
    p.feat_base[f] = p.seg_count[s];
    p.seg_count[s] += p.counts[p.Ftot + f];
  }
  for (int s = 0; s < p.nis; ++s) p.is_count[s] = p.B;
}

// keys = inverse value, vals = row: sorted by key -> CSR of each unique row
__global__ void k_inv_pairs(const __grid_constant__ BwdParams p, uint32_t* keys, uint32_t* vals) {
  RECD_PDL_PROLOGUE();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)p.nis * p.B) return;
  const int s = (int)(idx / p.B);
  const int64_t i = idx - (int64_t)s * p.B;
  keys[idx] = (uint32_t)p.inverse[s][i];
  vals[idx] = (uint32_t)i;
}

__global__ void k_csr_bounds(const __grid_constant__ BwdParams p) {
  RECD_PDL_PROLOGUE();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)p.nis * p.B) return;
  const int s = (int)(idx / p.B);
  const int64_t j = idx - (int64_t)s * p.B;
  const uint32_t* k = p.inv_keys + (int64_t)s * p.B;
  int32_t* start = p.csr_start + (int64_t)s * (p.B + 1);
  const uint32_t u = k[j];
  if (j == 0 || k[j - 1] != u) start[u] = (int32_t)j;
  if (j == p.B - 1) start[u + 1] = (int32_t)p.B;
}

// 1: features with an inverse reduce through k_grad_u_flat (position-parallel
// over the inverse CSR); k_grad_u keeps the identity (KJT) features
#ifndef RECD_GU_FLAT
#define RECD_GU_FLAT 1
#endif

template <class C>
__global__ void __launch_bounds__(256, 4) k_grad_u(const __grid_constant__ BwdParams p) {
  RECD_PDL_PROLOGUE();
  __shared__ int64_t s_pref[RECD_MAX_FEAT + 1];
  const int ncb = col_blocks<C>(p.D);
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int f = 0; f < p.F; ++f) {
      s_pref[f] = acc;
      if ((!RECD_GU_FLAT || p.feat_is[f] < 0) && ((p.gu_mask >> f) & 1ull)) acc += p.counts[f] * ncb;
    }
    s_pref[p.F] = acc;
  }
  __syncthreads();
  const int64_t total = s_pref[p.F];
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  constexpr int V = C::VW;
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total;
       w += nwarps) {
    const int f = find_seg(s_pref, p.F, w);
    const ColWork cw = col_work<C>(w - s_pref[f], p.D, lane);
    const int64_t u = cw.row;
    const float* G = p.grad_out[f] + cw.lo;
    const int is = p.feat_is[f];
    float acc[V];
    if (is < 0) {
      C::ld(G + u * p.D, cw.ok, acc);
    } else {
      const int32_t* start = p.csr_start + (int64_t)is * (p.B + 1);
      const uint32_t* rows = p.inv_rows + (int64_t)is * p.B;
      const int64_t a = start[u], e = start[u + 1];
      C::zero(acc);
      float x[8][V];
      for (int64_t j = a; j < e; j += 8) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (j + t < e) C::ld(G + (uint64_t)__ldg(rows + j + t) * (uint32_t)p.D, cw.ok, x[t]);
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (j + t < e) {
#pragma unroll
            for (int k = 0; k < V; ++k) acc[k] = __fadd_rn(acc[k], x[t][k]);
          }
      }
    }
    if (p.mode == RECD_POOL_AVG) {
      const int64_t U = p.counts[f], NV = p.counts[p.Ftot + f];
      const int64_t* uo = p.uoffsets[f];
      const int64_t len = ((u + 1 < U) ? uo[u + 1] : NV) - uo[u];
      if (len > 0) {
        const float fl = (float)len;
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = __fdiv_rn(acc[k], fl);
      }
    }
    if (p.gsegs == 0) {
      C::st(p.gout[f] + u * p.D + cw.lo, cw.ok, acc);
    } else {
      for (int j = 0; j < p.gsegs; ++j)
        C::st(p.gseg_dst[f][j] + (__ldg(p.gseg_row0[f][j]) + u) * p.D + cw.lo, cw.ok, acc);
    }
  }
}

// grad_u of the features with an inverse, position-parallel: warp per
// (feature, GU_CH consecutive positions of the inverse CSR, column block).  The
// warp reduces every unique row whose CSR run starts in its chunk (to the run's
// end), gathering grad_out rows 8 positions at a time across run boundaries, so
// no per-row dependent chain (CSR start -> row ids -> gradient rows) stalls it.
// Same order as k_grad_u (ascending batch row within each unique row).
#ifndef RECD_GU_CH
#define RECD_GU_CH 512
#endif
constexpr int GU_CH = RECD_GU_CH;  // positions per warp task (32 for small batches: more tasks;
                                   // 512 vs 256: grads 0.238 vs 0.243 ms, 64 / 128: 0.263 / 0.255)
#ifndef RECD_GU_CH_SMALL
#define RECD_GU_CH_SMALL 32
#endif
constexpr int GU_CH_SMALL = RECD_GU_CH_SMALL;
__device__ __forceinline__ int64_t run_end(const uint32_t* K, int64_t j, int64_t n, uint32_t id,
                                           int lane);
#ifndef RECD_GUF_CS
#define RECD_GUF_CS 0
#endif
#ifndef RECD_GUF_MINB
#define RECD_GUF_MINB 3
#endif
template <class C, int GU_CH>
__global__ void __launch_bounds__(256, RECD_GUF_MINB) k_grad_u_flat(const __grid_constant__ BwdParams p) {
  RECD_PDL_PROLOGUE();
  __shared__ int64_t s_pref[RECD_MAX_FEAT + 1];
  const int ncb = col_blocks<C>(p.D);
  const int64_t nch = (p.B + GU_CH - 1) / GU_CH;
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int f = 0; f < p.F; ++f) {
      s_pref[f] = acc;
      if (p.feat_is[f] >= 0 && ((p.gu_mask >> f) & 1ull)) acc += nch * ncb;
    }
    s_pref[p.F] = acc;
  }
  __syncthreads();
  const int64_t total = s_pref[p.F];
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  constexpr int V = C::VW;
  const int64_t B = p.B;
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total;
       w += nwarps) {
    const int f = find_seg(s_pref, p.F, w);
    const ColWork cw = col_work<C>(w - s_pref[f], p.D, lane);  // cw.row = chunk
    const int is = p.feat_is[f];
    const uint32_t* K = p.inv_keys + (int64_t)is * B;
    const uint32_t* R = p.inv_rows + (int64_t)is * B;
    const int64_t lo = cw.row * GU_CH, hi = min(B, lo + (int64_t)GU_CH);
    // first run start at or after lo
    int64_t j = lo;
    if (lo > 0) j = run_end(K, lo, B, __ldg(K + lo - 1), lane);
    if (j >= hi) continue;
    const float* G = p.grad_out[f] + cw.lo;
    const uint32_t D32 = (uint32_t)p.D;
    // window of 32 positions [wb, wb + 32): keys and rows, one per lane
    int64_t wb = j;
    uint32_t kw = wb + lane < B ? __ldg(K + wb + lane) : 0xffffffffu;
    uint32_t rw = wb + lane < B ? __ldg(R + wb + lane) : 0u;
    float acc[V];
    C::zero(acc);
    float x[8][V];
    bool done = false;
    for (int64_t k0 = j; !done; k0 += 8) {
      if (k0 + 9 > wb + 32) {
        wb = k0;
        kw = wb + lane < B ? __ldg(K + wb + lane) : 0xffffffffu;
        rw = wb + lane < B ? __ldg(R + wb + lane) : 0u;
      }
      const int sh = (int)(k0 - wb);
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const uint32_t row = __shfl_sync(0xffffffffu, rw, sh + t);
        if (k0 + t < B) {
          if constexpr (RECD_GUF_CS && V == 4) {  // grad_out is read once: evict first
            if (C::FULL || cw.ok) {
              const float4 q = __ldcs(reinterpret_cast<const float4*>(G + (uint64_t)row * D32));
              x[t][0] = q.x; x[t][1] = q.y; x[t][2] = q.z; x[t][3] = q.w;
            } else {
              C::zero(x[t]);
            }
          } else {
            C::ld(G + (uint64_t)row * D32, cw.ok, x[t]);
          }
        }
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const uint32_t u = __shfl_sync(0xffffffffu, kw, sh + t);
        const uint32_t un = __shfl_sync(0xffffffffu, kw, sh + t + 1);
        if (!done && k0 + t < B) {
#pragma unroll
          for (int e = 0; e < V; ++e) acc[e] = __fadd_rn(acc[e], x[t][e]);
          if (k0 + t + 1 == B || un != u) {  // run of u complete (warp-uniform)
            if (p.mode == RECD_POOL_AVG) {
              const int64_t U = p.counts[f], NV = p.counts[p.Ftot + f];
              const int64_t* uo = p.uoffsets[f];
              const int64_t len = ((u + 1 < U) ? uo[u + 1] : NV) - uo[u];
              if (len > 0) {
                const float fl = (float)len;
#pragma unroll
                for (int e = 0; e < V; ++e) acc[e] = __fdiv_rn(acc[e], fl);
              }
            }
            if (p.gsegs == 0) {
              C::st(p.gout[f] + (int64_t)u * p.D + cw.lo, cw.ok, acc);
            } else {
              for (int g = 0; g < p.gsegs; ++g)
                C::st(p.gseg_dst[f][g] + (__ldg(p.gseg_row0[f][g]) + u) * p.D + cw.lo, cw.ok, acc);
            }
            C::zero(acc);
            if (k0 + t + 1 >= hi) done = true;  // the next run belongs to the next chunk
          }
        }
      }
      if (k0 + 8 >= B) done = true;
    }
  }
}

// occurrence pairs (ID, (f << 24) | u) of every unique value, value-parallel:
// block per 4096 unique values of a feature; the block finds its first unique
// row with a 32-ary warp search, stages the unique offsets of the rows it
// spans in shared memory, and consecutive threads handle consecutive values
// (coalesced loads of the unique values, coalesced pair stores).
#ifndef RECD_OC_CH
#define RECD_OC_CH 16384
#endif
constexpr int OC_CH = RECD_OC_CH;   // values per block on big batches
#ifndef RECD_TINY_CH
#define RECD_TINY_CH 1
#endif
constexpr int OC_CH_SMALL = 4096;  // ... and on small ones (more blocks in flight)
constexpr int OC_MAXR = 512;
__global__ void __launch_bounds__(256) k_occ(const __grid_constant__ BwdParams p, uint32_t* keys,
                                             uint32_t* vals) {
  RECD_PDL_PROLOGUE();
  if (p.occ_gate && !*(volatile const int32_t*)p.occ_gate) return;  // runs fallback only
  const int f = block_feature(p.occ_blk0, p.F, (int64_t)blockIdx.x);
  const int64_t j0 = ((int64_t)blockIdx.x - p.occ_blk0[f]) * p.oc_ch;
  const int64_t U = p.counts[f], NV = p.counts[p.Ftot + f];
  if (j0 >= NV) return;
  const int64_t j1 = min(NV, j0 + p.oc_ch);
  const int tid = threadIdx.x;
  const int64_t* uo = p.uoffsets[f];
  const int64_t* src = p.uvalues[f];
  const int64_t dst = p.ts_base[p.feat_ts[f]] + p.feat_base[f];
  const uint64_t rows = (uint64_t)p.ts_rows[p.feat_ts[f]];
  __shared__ int64_t s_u0;
  __shared__ int64_t s_uo[OC_MAXR + 1];
  // digit counts of every radix pass of the occurrence sort (the sort then
  // skips reading the keys once more for its histogram)
  __shared__ uint32_t s_hist[SORT_HIST_PASSES][256];
  uint32_t* const hist = p.occ_hist;
  const int npass = hist ? (p.occ_bits + 7) / 8 : 0;
  if (hist) {
    for (int i = tid; i < SORT_HIST_PASSES * 256; i += 256) (&s_hist[0][0])[i] = 0u;
  }
  if (tid < 32) {
    const int64_t u = warp_last_le(uo, U, j0, tid);
    if (tid == 0) s_u0 = u;
  }
  __syncthreads();
  int64_t u0 = s_u0;
  while (true) {
    const int nr = (int)min((int64_t)OC_MAXR, U - u0);
    for (int t = tid; t <= nr; t += 256) {
      const int64_t u = u0 + t;
      s_uo[t] = (u < U) ? uo[u] : NV;
    }
    __syncthreads();
    const int64_t covered = s_uo[nr];
    const int64_t qa = max(j0, s_uo[0]), qb = min(j1, covered);
    // staged rows all of one length L: row of q = (q - s_uo[0]) / L, stepped
    // incrementally (no per-value search); 4 values per thread per batch
    const int64_t L0 = nr > 0 ? s_uo[1] - s_uo[0] : 0;
    bool uni = L0 > 0 && L0 < (1 << 23);
    for (int t = tid; t < nr; t += 256) uni &= (s_uo[t + 1] - s_uo[t]) == L0;
    if (__syncthreads_and(uni)) {
      const uint32_t L = (uint32_t)L0, dj = 256 / L, dr = 256 % L;
      const int64_t q_first = qa + tid;
      uint32_t rr = 0, rem = 0;
      if (q_first < qb) {
        const uint32_t rel = (uint32_t)(q_first - s_uo[0]);
        rr = rel / L;
        rem = rel - rr * L;
      }
      for (int64_t qq = q_first; qq < qb; qq += 4 * 256) {
        int64_t id[4];
        uint32_t row[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          row[k] = rr;
          rr += dj;
          rem += dr;
          if (rem >= L) {
            rem -= L;
            ++rr;
          }
          if (qq + k * 256 < qb) id[k] = __ldg(src + qq + k * 256);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t q = qq + k * 256;
          if (q < qb) {
            const bool in = (uint64_t)id[k] < rows;
            if (!in) *p.bad = 1;
            const uint32_t key = in ? (uint32_t)id[k] : 0u;
            keys[dst + q] = key;
            for (int ps = 0; ps < npass; ++ps) atomicAdd(&s_hist[ps][(key >> (8 * ps)) & 255u], 1u);
            vals[dst + q] = ((uint32_t)f << 24) | (uint32_t)(u0 + row[k]);
          }
        }
      }
      if (covered >= j1) break;
      __syncthreads();
      u0 += nr;
      continue;
    }
    int r = 0;
    for (int64_t q = qa + tid; q < qb; q += 256) {
      // row of q: short forward walk from the previous value's row (q moved
      // by one block stride), binary search only past 8 rows
      if (s_uo[min(r + 8, nr)] <= q) {
        int lo = r + 8, hi = nr - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_uo[mid] <= q) lo = mid; else hi = mid - 1;
        }
        r = lo;
      } else {
        while (s_uo[r + 1] <= q) ++r;
      }
      const int64_t id = __ldg(src + q);
      // an ID outside [0, rows) (the forward reports it, trainer_sim.py:312-320)
      // must not address the table: flag it, and the scatter skips every update
      const bool in = (uint64_t)id < rows;
      if (!in) *p.bad = 1;
      const uint32_t key = in ? (uint32_t)id : 0u;
      keys[dst + q] = key;
      for (int ps = 0; ps < npass; ++ps) atomicAdd(&s_hist[ps][(key >> (8 * ps)) & 255u], 1u);
      vals[dst + q] = ((uint32_t)f << 24) | (uint32_t)(u0 + r);
    }
    if (covered >= j1) break;
    __syncthreads();
    u0 += nr;
  }
  if (hist) {  // the block's digit counts into the sort's histogram
    __syncthreads();
    const int64_t row0 = (int64_t)p.feat_ts[f] * SORT_HIST_PASSES * 256;
    for (int i = tid; i < npass * 256; i += 256) {
      const uint32_t c = (&s_hist[0][0])[i];
      if (c) atomicAdd(&hist[row0 + i], c);
    }
  }
}

// ---------------------------------------------------------------------------
// Diagonal-run occurrences (RECD_BWD_RUNS=1).  In session data consecutive
// unique rows of a history feature are windows shifted by one: the ID at
// (u, p) is usually the ID at (u - 1, p + 1).  A diagonal of occurrences --
// one ID in rows u .. u + k - 1 at positions p, p - 1, ... -- is ONE sort
// element (ID, head index), so the occurrence sort orders the run heads
// (~N_ids) instead of every unique value (N_u, 3.3x more at cfg2):
//   k_rv<0>      heads per value block (a value heads a run unless it repeats
//                its diagonal predecessor)
//   scan         block offsets -> heads numbered in (u, p) order per segment
//   k_rv<1>      heads written in that order (ID, index; tag, position) + the
//                sort's digit histograms
//   k_rv_len     run length of every head (walk down its diagonal)
//   sort         heads by ID (stable: each ID's runs stay in (u, p) order)
//   k_rv_lens    run lengths in sorted order (+ the IDs whose runs overlap)
//   scan         -> expanded offsets
//   k_rv_expand  per-value (ID, tag) array, coalesced, for the unchanged scatter
//   k_rv_fix     the overlapping IDs' tags re-sorted in place
// Exactness: the oracle adds, per ID, grad_u[t] over its occurrences in
// non-decreasing tag order (equal tags add the same row, so their order does
// not matter).  An ID's runs come out of the sort in head order; concatenated
// they are already non-decreasing unless a run starts before the previous one
// ends (the ID occurs twice in one row): those IDs are listed and their
// expanded tags sorted (k_rv_fix; > RV_FIX_MAX values or a full list set
// `fallback`, and the gated per-value occurrences + full sort rebuild the
// batch -- slower, never different).  Only for one feature per table segment.
// ---------------------------------------------------------------------------
constexpr int RV_FIX_MAX = 4096;   // values of one overlapping ID re-sorted in shared memory
constexpr int RV_FIX_CAP = 65536;  // overlapping IDs listed per batch
constexpr int RV_EX_CH = 2048;     // expanded values per k_rv_expand block

template <int MODE>
__global__ void __launch_bounds__(256) k_rv(const __grid_constant__ BwdParams p, uint32_t* keys,
                                            uint32_t* vals) {
  RECD_PDL_PROLOGUE();
  const int f = block_feature(p.occ_blk0, p.F, (int64_t)blockIdx.x);
  const int64_t blk = blockIdx.x;
  const int64_t j0 = (blk - p.occ_blk0[f]) * p.oc_ch;
  const int64_t U = p.counts[f], NV = p.counts[p.Ftot + f];
  const int tid = threadIdx.x;
  if (j0 >= NV) {
    if (MODE == 0 && tid == 0) p.rv_blk[blk] = 0;
    return;
  }
  const int64_t j1 = min(NV, j0 + p.oc_ch);
  const int64_t* uo = p.uoffsets[f];
  const int64_t* src = p.uvalues[f];
  const int ts = p.feat_ts[f];
  const uint64_t rows = (uint64_t)p.ts_rows[ts];
  __shared__ int64_t s_u0;
  __shared__ int64_t s_uo[OC_MAXR + 2];  // s_uo[t] = start of row u0 - 1 + t
  __shared__ int64_t s_scan[32];
  __shared__ uint32_t s_hist[SORT_HIST_PASSES][256];
  uint32_t* const hist = MODE == 1 ? p.occ_hist : nullptr;
  const int npass = hist ? (p.occ_bits + 7) / 8 : 0;
  if (hist)
    for (int i = tid; i < SORT_HIST_PASSES * 256; i += 256) (&s_hist[0][0])[i] = 0u;
  const int64_t hbase = MODE == 1 ? p.ts_base[ts] + p.rv_blk[blk] : 0;
  int64_t count = 0;  // heads of the block so far (block-uniform)
  if (tid < 32) {
    const int64_t u = warp_last_le(uo, U, j0, tid);
    if (tid == 0) s_u0 = u;
  }
  __syncthreads();
  int64_t u0 = s_u0;
  while (true) {
    const int nr = (int)min((int64_t)OC_MAXR, U - u0);
    for (int t = tid; t <= nr + 1; t += 256) {
      const int64_t x = u0 - 1 + t;
      s_uo[t] = x < 0 ? 0 : (x < U ? uo[x] : NV);
    }
    __syncthreads();
    const int64_t covered = s_uo[nr + 1];
    const int64_t qa = max(j0, s_uo[1]), qb = min(j1, covered);
    int r = 0;
    for (int64_t base = qa; base < qb; base += 256) {  // block-uniform rounds
      const int64_t q = base + tid;
      bool head = false;
      int64_t v = 0, pp = 0;
      if (q < qb) {
        if (s_uo[min(r + 8, nr) + 1] <= q) {
          int lo = r + 8, hi = nr - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_uo[mid + 1] <= q) lo = mid; else hi = mid - 1;
          }
          r = lo;
        } else {
          while (s_uo[r + 2] <= q) ++r;
        }
        pp = q - s_uo[r + 1];
        v = __ldg(src + q);
        bool cont = false;
        if (u0 + r >= 1) {  // diagonal predecessor (u - 1, p + 1)
          const int64_t ps = s_uo[r];
          cont = pp + 1 < s_uo[r + 1] - ps && __ldg(src + ps + pp + 1) == v;
        }
        head = !cont;
      }
      if (MODE == 0) {
        count += __syncthreads_count(head);
      } else {
        int64_t tot;
        const int64_t rank = block_exclusive_scan<256>(head ? 1 : 0, s_scan, &tot);
        if (head) {
          const int64_t o = hbase + count + rank;
          const bool in = (uint64_t)v < rows;
          if (!in) *p.bad = 1;
          const uint32_t key = in ? (uint32_t)v : 0u;
          keys[o] = key;
          vals[o] = (uint32_t)o;
          p.head_tag[o] = ((uint32_t)f << 24) | (uint32_t)(u0 + r);
          p.head_pos[o] = (uint32_t)pp;
          for (int ps = 0; ps < npass; ++ps) atomicAdd(&s_hist[ps][(key >> (8 * ps)) & 255u], 1u);
        }
        count += tot;
      }
    }
    if (covered >= j1) break;
    __syncthreads();
    u0 += nr;
  }
  if (MODE == 0) {
    if (tid == 0) p.rv_blk[blk] = count;
  } else if (hist) {
    __syncthreads();
    const int64_t row0 = (int64_t)ts * SORT_HIST_PASSES * 256;
    for (int i = tid; i < npass * 256; i += 256) {
      const uint32_t c = (&s_hist[0][0])[i];
      if (c) atomicAdd(&hist[row0 + i], c);
    }
  }
}

// thread per head: run length = rows down the diagonal (u + k, p - k) that hold
// the head's ID (row starts from global memory: the next row's start is the
// current row's end, so one new offset + one value per step)
__global__ void __launch_bounds__(256) k_rv_len(const __grid_constant__ BwdParams p) {
  RECD_PDL_PROLOGUE();
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int s = 0; s < p.nts; ++s) {
    const int f = p.seg_feat[s];
    const int64_t n = p.head_count[s], base = p.ts_base[s];
    const int64_t U = p.counts[f], NV = p.counts[p.Ftot + f];
    const int64_t* uo = p.uoffsets[f];
    const int64_t* src = p.uvalues[f];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += nthr) {
      const int64_t o = base + j;
      const int64_t u = p.head_tag[o] & 0xffffffu;
      int64_t cp = p.head_pos[o];
      const int64_t v = __ldg(src + __ldg(uo + u) + cp);
      uint32_t len = 1;
      int64_t cu = u;
      int64_t ns = (cu + 1 < U) ? __ldg(uo + cu + 1) : NV;  // start of row cu + 1
      while (cp >= 1 && cu + 1 < U) {
        const int64_t ne = (cu + 2 < U) ? __ldg(uo + cu + 2) : NV;
        if (cp - 1 >= ne - ns || __ldg(src + ns + cp - 1) != v) break;
        ++len;
        ++cu;
        --cp;
        ns = ne;
      }
      p.head_len[o] = len;
    }
  }
}

// sorted head j of segment blockIdx.y -> its run length (scanned into expanded
// offsets next); the first head of each ID checks whether its runs overlap
// (a run starting before the previous one's last row) and lists the ID
__global__ void k_rv_lens(const __grid_constant__ BwdParams p, const uint32_t* skeys,
                          const uint32_t* svals) {
  RECD_PDL_PROLOGUE();
  const int s = blockIdx.y;
  const int64_t n = p.head_count[s], base = p.ts_base[s];
  const uint32_t* K = skeys + base;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t hid = svals[base + j];
    const uint32_t len = p.head_len[hid];
    p.head_off[base + j] = (int64_t)len;
    const uint32_t id = K[j];
    if (j > 0 && K[j - 1] == id) continue;
    if (j + 1 >= n || K[j + 1] != id) continue;  // one run: nothing to check
    uint32_t last = p.head_tag[hid] + len - 1;
    bool ovl = false;
    int64_t e = j + 1;
    for (; e < n && K[e] == id; ++e) {
      const uint32_t h2 = svals[base + e];
      const uint32_t t2 = p.head_tag[h2];
      ovl |= t2 < last;
      last = max(last, t2 + p.head_len[h2] - 1);
    }
    if (ovl) {
      const uint32_t k = atomicAdd(p.fix_count, 1u);
      if (k < (uint32_t)RV_FIX_CAP) {
        p.fix_list[3 * k] = s;
        p.fix_list[3 * k + 1] = (int32_t)j;
        p.fix_list[3 * k + 2] = (int32_t)e;
      } else {
        *p.fallback = 1;
      }
    }
  }
}

// block per RV_EX_CH expanded values of a segment: the heads covering them
// (two warp searches over the expanded offsets) staged in shared memory, then
// value e -> (ID, head tag + e - head offset), coalesced stores
__global__ void __launch_bounds__(256) k_rv_expand(const __grid_constant__ BwdParams p,
                                                   const uint32_t* skeys, const uint32_t* svals) {
  RECD_PDL_PROLOGUE();
  int s = 0;
  while (s + 1 < p.nts && p.ex_chunk0[s + 1] <= (int64_t)blockIdx.x) ++s;
  const int64_t E = p.seg_count[s], base = p.ts_base[s];
  const int64_t e0 = ((int64_t)blockIdx.x - p.ex_chunk0[s]) * RV_EX_CH;
  if (e0 >= E) return;
  const int64_t e1 = min(E, e0 + (int64_t)RV_EX_CH);
  const int64_t n = p.head_count[s];
  const int64_t* off = p.head_off + base;
  __shared__ int64_t s_j[2];
  __shared__ int32_t s_off[RV_EX_CH];
  __shared__ uint32_t s_key[RV_EX_CH], s_tag[RV_EX_CH];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp < 2) {
    const int64_t j = warp_last_le(off, n, warp == 0 ? e0 : e1 - 1, lane);
    if (lane == 0) s_j[warp] = j;
  }
  __syncthreads();
  const int64_t jlo = s_j[0];
  const int nh = (int)(s_j[1] - jlo + 1);
  for (int i = tid; i < nh; i += 256) {
    s_off[i] = (int32_t)(off[jlo + i] - e0);
    s_key[i] = skeys[base + jlo + i];
    s_tag[i] = p.head_tag[svals[base + jlo + i]];
  }
  __syncthreads();
  uint32_t* ok_ = p.exp_keys + base;
  uint32_t* ov_ = p.exp_vals + base;
  for (int64_t e = e0 + tid; e < e1; e += 256) {
    const int32_t x = (int32_t)(e - e0);
    int lo = 0, hi = nh - 1;  // last head with s_off <= x
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= x) lo = mid; else hi = mid - 1;
    }
    ok_[e] = s_key[lo];
    ov_[e] = s_tag[lo] + (uint32_t)(x - s_off[lo]);
  }
}

// block per listed ID: its expanded tags (all one key) sorted in shared memory
__global__ void __launch_bounds__(256) k_rv_fix(const __grid_constant__ BwdParams p) {
  RECD_PDL_PROLOGUE();
  __shared__ uint32_t s_t[RV_FIX_MAX];
  const uint32_t cnt = min(*p.fix_count, (uint32_t)RV_FIX_CAP);
  for (uint32_t k = blockIdx.x; k < cnt; k += gridDim.x) {
    const int s = p.fix_list[3 * k];
    const int64_t j = p.fix_list[3 * k + 1], e = p.fix_list[3 * k + 2];
    const int64_t base = p.ts_base[s];
    const int64_t lo = p.head_off[base + j];
    const int64_t hi = e < p.head_count[s] ? p.head_off[base + e] : p.seg_count[s];
    const int m = (int)(hi - lo);
    if (m > RV_FIX_MAX) {
      if (threadIdx.x == 0) *p.fallback = 1;
      continue;
    }
    int m2 = 1;
    while (m2 < m) m2 <<= 1;
    uint32_t* v = p.exp_vals + base + lo;
    for (int i = threadIdx.x; i < m2; i += blockDim.x) s_t[i] = i < m ? v[i] : 0xffffffffu;
    __syncthreads();
    for (int k2 = 2; k2 <= m2; k2 <<= 1)
      for (int jj = k2 >> 1; jj > 0; jj >>= 1) {
        for (int i = threadIdx.x; i < m2; i += blockDim.x) {
          const int x = i ^ jj;
          if (x > i) {
            const uint32_t a = s_t[i], b = s_t[x];
            if (((i & k2) == 0) == (a > b)) {
              s_t[i] = b;
              s_t[x] = a;
            }
          }
        }
        __syncthreads();
      }
    for (int i = threadIdx.x; i < m; i += blockDim.x) v[i] = s_t[i];
    __syncthreads();
  }
}

__device__ __forceinline__ int rc_seg(const BwdParams& p, int64_t chunk) {
  int lo = 0, hi = p.nts - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.ts_chunk0[mid] <= chunk) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// number of run starts per RC chunk (grad-output mode)
template <int RC>
__global__ void __launch_bounds__(RC) k_run_count(const __grid_constant__ BwdParams p) {
  RECD_PDL_PROLOGUE();
  const int64_t chunk = blockIdx.x;
  const int s = rc_seg(p, chunk);
  const int64_t n = p.seg_count[s];
  const int64_t j = (chunk - p.ts_chunk0[s]) * RC + threadIdx.x;
  const uint32_t* K = p.occ_keys + p.ts_base[s];
  const int start = (j < n) && (j == 0 || K[j] != K[j - 1]) && !*p.bad;
  const int cnt = __syncthreads_count(start);
  if (threadIdx.x == 0) p.run_part[chunk] = cnt;
}

// first position >= j whose key differs from `id` (lane-parallel search)
__device__ __forceinline__ int64_t run_end(const uint32_t* K, int64_t j, int64_t n, uint32_t id,
                                           int lane) {
  for (int64_t j0 = j; j0 < n; j0 += 32) {
    const int64_t q = j0 + lane;
    const bool diff = q >= n || __ldg(K + q) != id;
    const unsigned b = __ballot_sync(0xffffffffu, diff);
    if (b) return j0 + __ffs(b) - 1;
  }
  return n;
}

#ifndef RECD_SC_RS
#define RECD_SC_RS 6
#endif
constexpr int SC_RS = RECD_SC_RS;  // table rows prefetched ahead per warp (shared-memory ring)
#ifndef RECD_SC_PIPE
#define RECD_SC_PIPE 0
#endif
#ifndef RECD_SC_REV
#define RECD_SC_REV 0
#endif
#ifndef RECD_OCC_HIST  // k_occ counts the occurrence sort's digits (no k_os_hist pass)
#define RECD_OCC_HIST 1
#endif
#ifndef RECD_SC_BATCH
#define RECD_SC_BATCH 6
#endif
constexpr int SC_BATCH = RECD_SC_BATCH;  // unique-row gradient gathers in flight per warp

// One warp per (chunk of RC sorted positions, column block).  Runs of equal
// IDs that start in the chunk are reduced in position order (== ascending
// (feature, unique row, position) order, so bit-identical to the oracle).
// The table rows of the next SC_RS runs are prefetched with cp.async into a
// per-warp shared ring while grad_u rows (L2-resident) are gathered 8 positions
// at a time across run boundaries; at each run end the row is updated and
// stored, and its slot refilled with the row of run r + SC_RS.
template <class C, bool SINGLE, int RC>
__global__ void __launch_bounds__(256, RECD_SCATTER_MINB) k_scatter(const __grid_constant__ BwdParams p) {
  RECD_PDL_PROLOGUE();
  constexpr int V = C::VW;
  __shared__ uint16_t s_starts[8][RC + 2];
  __shared__ uint32_t s_ids[8][RC];
  __shared__ __align__(128) float s_ring[8][SC_RS][C::CB];
  __shared__ uint32_t s_win[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  const int ncb = col_blocks<C>(p.D);
  const int64_t total = (p.sc_chunk_hi - p.sc_chunk_lo) * ncb;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  if (*(volatile const int32_t*)p.bad) return;  // out-of-range ID in the batch: no update
  uint16_t* starts = s_starts[warp];
  uint32_t* rids = s_ids[warp];
  float* ring = &s_ring[warp][0][lane * V];
  const bool apply = p.apply_sgd != 0;
  constexpr bool HINT = RECD_SCATTER_L2 > 0 && V == 4;
  const uint64_t pol_stream = HINT ? l2_evict_first() : 0;
  const uint64_t pol_keep = (HINT && RECD_SCATTER_L2 >= 2) ? l2_evict_last() : 0;
  // next (chunk, column block) task: grid-stride, or the next ticket (dynamic:
  // tasks start in order however long each takes, so the warps in flight work
  // on neighbouring chunks -- one table segment's gradients stay hot in L2)
  auto next_task = [&](int64_t cur) -> int64_t {
    if (!p.sc_dyn) return cur + nwarps;
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(p.sc_ticket, 1u);
    return (int64_t)__shfl_sync(0xffffffffu, t, 0);
  };
  for (int64_t w = p.sc_dyn ? next_task(0) : (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
       w < total; w = next_task(w)) {
    const int64_t wc = ((ncb == 1) ? w : w / ncb) + p.sc_chunk_lo;
    // RECD_SC_REV: last table segment first -- k_grad_u_flat wrote the unique-row
    // gradients in feature order, so the last features' are still in L2
    const int64_t chunk = RECD_SC_REV ? p.sc_chunk_hi - 1 - (wc - p.sc_chunk_lo) : wc;
    const int lo_f = (int)(w - (wc - p.sc_chunk_lo) * ncb) * C::CB + lane * V;  // this lane's first float
    const bool ok = lo_f < p.D;
    const uint32_t D32 = (uint32_t)p.D;
    const int s = rc_seg(p, chunk);
    const int64_t n = p.seg_count[s];
    const int64_t lo = (chunk - p.ts_chunk0[s]) * RC;
    if (lo >= n) continue;
    const int64_t hi = min(n, lo + (int64_t)RC);
    const uint32_t* K = p.occ_keys + p.ts_base[s];
    const uint32_t* Vv = p.occ_vals + p.ts_base[s];
    // 1. runs starting inside [lo, hi): start offsets and IDs.  The chunk's
    //    keys are loaded up front (RC / 32 independent loads per lane, not one
    //    round trip per 32 positions); a position's predecessor key comes
    //    from the next lower lane, lane 0's from the previous group's lane 31
    int nruns = 0;
    {
      uint32_t kk[RC / 32];
#pragma unroll
      for (int g = 0; g < RC / 32; ++g) {
        const int64_t j = lo + g * 32 + lane;
        kk[g] = j < hi ? __ldg(K + j) : 0u;
      }
      uint32_t prev_last = lo > 0 ? __ldg(K + lo - 1) : 0u;
#pragma unroll
      for (int g = 0; g < RC / 32; ++g) {
        const int64_t j = lo + g * 32 + lane;
        const uint32_t up = __shfl_up_sync(0xffffffffu, kk[g], 1);
        const uint32_t pk = lane == 0 ? prev_last : up;
        prev_last = __shfl_sync(0xffffffffu, kk[g], 31);
        const bool st = j < hi && (j == 0 || pk != kk[g]);
        const unsigned b = __ballot_sync(0xffffffffu, st);
        if (st) {
          starts[nruns + __popc(b & lt)] = (uint16_t)(j - lo);
          rids[nruns + __popc(b & lt)] = kk[g];
        }
        nruns += __popc(b);
      }
    }
    __syncwarp();
    if (nruns == 0) continue;
    const int64_t pend = run_end(K, hi, n, rids[nruns - 1], lane);  // end of the last run
    float* table = p.table[s] + lo_f;
    // 2. prefetch the table rows of the first SC_RS runs
    if (apply) {
#pragma unroll
      for (int r = 0; r < SC_RS; ++r) {
        if (r < nruns && ok) {
          if constexpr (HINT)
            cp_async16_hint(ring + r * C::CB, table + (uint64_t)rids[r] * D32, pol_stream);
          else
            cp_async<V * 4>(ring + r * C::CB, table + (uint64_t)rids[r] * D32);
        }
        cp_async_commit();
      }
    }
    const int64_t run_base = apply ? 0 : p.run_part[chunk];
    // 3. flat pass over the positions of the chunk's runs, offsets from lo
    //    (32-bit); the occurrence tags of 32 positions at a time sit in shared
    //    memory (broadcast reads); SINGLE: one feature per table segment, so the
    //    gradient base is uniform
    const int32_t pe = (int32_t)(pend - lo);
    const uint32_t* __restrict__ Vl = Vv + lo;
    const float* gs = SINGLE ? p.seg_grow[s] + lo_f : nullptr;
    uint32_t* win = s_win[warp];
    int32_t wbase = starts[0];
    win[lane] = (wbase + lane < pe) ? __ldg(Vl + wbase + lane) : 0u;
    __syncwarp();
    int r = 0;
    int32_t bnd = (nruns > 1) ? (int32_t)starts[1] : pe;  // end of run r
    float acc[V];
    C::zero(acc);
#if RECD_SC_PIPE
    // software-pipelined: the gradient rows of the next SC_BATCH positions are
    // in flight while the current SC_BATCH are reduced (the gathers, not the
    // table RMW, are what the warps wait on -- ncu source view)
    float xa[SC_BATCH][V], xb[SC_BATCH][V];
    auto load_batch = [&](float (&x)[SC_BATCH][V], int32_t k) {
      if (k + SC_BATCH > wbase + 32) {
        __syncwarp();
        wbase = k;
        win[lane] = (k + lane < pe) ? __ldg(Vl + k + lane) : 0u;
        __syncwarp();
      }
#pragma unroll
      for (int t = 0; t < SC_BATCH; ++t) {
        if (k + t < pe) {
          const uint32_t vv = win[k + t - wbase];
          const float* gp = SINGLE ? gs + (uint64_t)(vv & 0xffffffu) * D32
                                   : p.grow[vv >> 24] + lo_f + (uint64_t)(vv & 0xffffffu) * D32;
          if constexpr (HINT && RECD_SCATTER_L2 >= 2) {
            if (C::FULL || ok) {
              const float4 q = ld_v4_hint(gp, pol_keep);
              x[t][0] = q.x; x[t][1] = q.y; x[t][2] = q.z; x[t][3] = q.w;
            } else {
              C::zero(x[t]);
            }
          } else {
            C::ld(gp, ok, x[t]);
          }
        }
      }
    };
    auto consume = [&](float (&x)[SC_BATCH][V], int32_t k0) {
#pragma unroll
      for (int t = 0; t < SC_BATCH; ++t) {
        if (k0 + t < pe) {
#pragma unroll
          for (int e = 0; e < V; ++e) acc[e] = __fadd_rn(acc[e], x[t][e]);
          if (k0 + t + 1 == bnd) {  // run r complete (warp-uniform)
            const uint32_t id = rids[r];
            if (apply) {
              cp_async_wait<SC_RS - 1>();
              float* slot = ring + (r % SC_RS) * C::CB;
              float wv[V];
#pragma unroll
              for (int e = 0; e < V; ++e) wv[e] = __fsub_rn(slot[e], __fmul_rn(p.lr, acc[e]));
              if constexpr (HINT) {
                if (C::FULL || ok)
                  st_v4_hint(table + (uint64_t)id * D32, wv[0], wv[1], wv[2], wv[3], pol_stream);
                if (r + SC_RS < nruns && ok)
                  cp_async16_hint(slot, table + (uint64_t)rids[r + SC_RS] * D32, pol_stream);
              } else {
                C::st(table + (uint64_t)id * D32, ok, wv);
                if (r + SC_RS < nruns && ok)
                  cp_async<V * 4>(slot, table + (uint64_t)rids[r + SC_RS] * D32);
              }
              cp_async_commit();
            } else {
              const int64_t ri = run_base + r;
              if (lo_f == 0) p.grad_ids[s][ri] = (int64_t)id;
              C::st(p.grad_rows[s] + ri * p.D + lo_f, ok, acc);
            }
            ++r;
            C::zero(acc);
            bnd = (r + 1 < nruns) ? (int32_t)starts[r + 1] : pe;
          }
        }
      }
    };
    int32_t kl = starts[0];
    load_batch(xa, kl);
    kl += SC_BATCH;
    for (int32_t k0 = starts[0]; k0 < pe; k0 += 2 * SC_BATCH) {
      load_batch(xb, kl);
      kl += SC_BATCH;
      consume(xa, k0);
      if (k0 + SC_BATCH >= pe) break;
      load_batch(xa, kl);
      kl += SC_BATCH;
      consume(xb, k0 + SC_BATCH);
    }
#else
    float x[SC_BATCH][V];
    for (int32_t k0 = starts[0]; k0 < pe; k0 += SC_BATCH) {
      if (k0 + SC_BATCH > wbase + 32) {
        __syncwarp();
        wbase = k0;
        win[lane] = (k0 + lane < pe) ? __ldg(Vl + k0 + lane) : 0u;
        __syncwarp();
      }
#pragma unroll
      for (int t = 0; t < SC_BATCH; ++t) {
        const uint32_t vv = win[k0 + t - wbase];
        const float* gp = SINGLE ? gs + (uint64_t)(vv & 0xffffffu) * D32
                                 : p.grow[vv >> 24] + lo_f + (uint64_t)(vv & 0xffffffu) * D32;
        if (k0 + t < pe) {
          if constexpr (HINT && RECD_SCATTER_L2 >= 2) {  // keep unique-row grads in L2
            if (C::FULL || ok) {
              const float4 q = ld_v4_hint(gp, pol_keep);
              x[t][0] = q.x; x[t][1] = q.y; x[t][2] = q.z; x[t][3] = q.w;
            } else {
              C::zero(x[t]);
            }
          } else {
            C::ld(gp, ok, x[t]);
          }
        }
      }
#pragma unroll
      for (int t = 0; t < SC_BATCH; ++t) {
        if (k0 + t < pe) {
#pragma unroll
          for (int e = 0; e < V; ++e) acc[e] = __fadd_rn(acc[e], x[t][e]);
          if (k0 + t + 1 == bnd) {  // run r complete (warp-uniform)
            const uint32_t id = rids[r];
            if (apply) {
              cp_async_wait<SC_RS - 1>();
              float* slot = ring + (r % SC_RS) * C::CB;
              float wv[V];
#pragma unroll
              for (int e = 0; e < V; ++e) wv[e] = __fsub_rn(slot[e], __fmul_rn(p.lr, acc[e]));
              if constexpr (HINT) {
                if (C::FULL || ok)
                  st_v4_hint(table + (uint64_t)id * D32, wv[0], wv[1], wv[2], wv[3], pol_stream);
                if (r + SC_RS < nruns && ok)
                  cp_async16_hint(slot, table + (uint64_t)rids[r + SC_RS] * D32, pol_stream);
              } else {
                C::st(table + (uint64_t)id * D32, ok, wv);
                if (r + SC_RS < nruns && ok)
                  cp_async<V * 4>(slot, table + (uint64_t)rids[r + SC_RS] * D32);
              }
              cp_async_commit();
            } else {
              const int64_t ri = run_base + r;
              if (lo_f == 0) p.grad_ids[s][ri] = (int64_t)id;
              C::st(p.grad_rows[s] + ri * p.D + lo_f, ok, acc);
            }
            ++r;
            C::zero(acc);
            bnd = (r + 1 < nruns) ? (int32_t)starts[r + 1] : pe;
          }
        }
      }
    }
#endif
    if (apply) cp_async_wait<0>();
    __syncwarp();
  }
}

static int64_t bits_for(int64_t n) {
  int b = 0;
  while ((1ll << b) < n) ++b;
  return b;
}

}  // namespace recd

using namespace recd;

namespace {

struct Plan {
  int F, nis, nts;
  std::vector<int> feat_is, feat_ts, is_feat;
  std::vector<const int64_t*> inverse;
  std::vector<float*> table;
  std::vector<int64_t> table_rows;  // max rows per table seg
  std::vector<int64_t> ts_base, ts_cap, ts_chunk0;
  std::vector<int64_t> caps;  // value capacity per feature
  int64_t occ_total, rc_chunks;
  int rc;  // scatter chunk (RC_BIG / RC_SMALL)
};

Plan make_plan(int F, const int64_t* const* inverse, float* const* tables, const int64_t* rows,
               const int64_t* caps) {
  Plan pl;
  pl.F = F;
  pl.caps.assign(caps, caps + F);
  pl.feat_is.assign(F, -1);
  pl.feat_ts.assign(F, -1);
  std::map<const void*, int> is_map, ts_map;
  for (int f = 0; f < F; ++f) {
    const int64_t* inv = inverse ? inverse[f] : nullptr;
    if (inv) {
      auto it = is_map.find(inv);
      if (it == is_map.end()) {
        it = is_map.emplace(inv, (int)pl.inverse.size()).first;
        pl.inverse.push_back(inv);
        pl.is_feat.push_back(f);
      }
      pl.feat_is[f] = it->second;
    }
    auto jt = ts_map.find(tables[f]);
    if (jt == ts_map.end()) {
      jt = ts_map.emplace(tables[f], (int)pl.table.size()).first;
      pl.table.push_back(tables[f]);
      pl.table_rows.push_back(rows[f]);
      pl.ts_cap.push_back(0);
    }
    pl.feat_ts[f] = jt->second;
    pl.ts_cap[jt->second] += caps[f];
    pl.table_rows[jt->second] = std::max(pl.table_rows[jt->second], rows[f]);
  }
  pl.nis = (int)pl.inverse.size();
  pl.nts = (int)pl.table.size();
  int64_t base = 0, chunk = 0;
  for (int s = 0; s < pl.nts; ++s) base += pl.ts_cap[s];
  pl.rc = rc_for(base);
  base = 0;
  for (int s = 0; s < pl.nts; ++s) {
    pl.ts_base.push_back(base);
    pl.ts_chunk0.push_back(chunk);
    base += pl.ts_cap[s];
    chunk += std::max<int64_t>(1, ceil_div(pl.ts_cap[s], pl.rc));
  }
  pl.occ_total = base;
  pl.rc_chunks = chunk;
  return pl;
}

struct BwdScratch {
  int64_t *feat_base, *seg_count, *is_count, *run_part, *scan_part;
  int32_t* bad;
  uint32_t *head_tag, *head_pos, *head_len, *fix_count;
  int64_t *rv_blk, *rv_scan_part;
  int32_t* fix_list;
  int64_t *head_count, *head_off, *runs_scan_part;
  int32_t* fallback;
  uint32_t* sc_ticket;
  uint32_t *inv_k0, *inv_v0, *inv_k1, *inv_v1, *hist, *hist_inv;
  int32_t* csr_start;
  float* grad_u;
  uint32_t *occ_k0, *occ_v0, *occ_k1, *occ_v1;
};

enum { NEED_INV = 1, NEED_GRADU = 2, NEED_OCC = 4 };

size_t carve_bwd(void* base, size_t cap, const Plan& pl, int64_t B, int D, BwdScratch* s,
                 int need = NEED_INV | NEED_GRADU | NEED_OCC) {
  Arena a(base, cap);
  s->feat_base = a.take<int64_t>(RECD_MAX_FEAT);
  s->seg_count = a.take<int64_t>(RECD_MAX_FEAT);
  s->is_count = a.take<int64_t>(RECD_MAX_FEAT);
  s->bad = a.take<int32_t>(1);
  s->run_part = a.take<int64_t>((need & NEED_OCC) ? pl.rc_chunks : 1);
  const size_t nib = (need & NEED_INV) ? (size_t)std::max(pl.nis, 1) * B : 1;
  s->inv_k0 = a.take<uint32_t>(nib);
  s->inv_v0 = a.take<uint32_t>(nib);
  s->inv_k1 = a.take<uint32_t>(nib);
  s->inv_v1 = a.take<uint32_t>(nib);
  s->csr_start = a.take<int32_t>((need & NEED_INV) ? (size_t)std::max(pl.nis, 1) * (B + 1) : 1);
  s->grad_u = a.take<float>((need & NEED_GRADU) ? (size_t)pl.F * B * D : 1);
  const size_t occ = (need & NEED_OCC) ? (size_t)pl.occ_total : 1;
  // diagonal runs: head (tag, length), head counts per segment, the heads'
  // expanded offsets (only the full backward uses runs)
  const bool rn = (need & NEED_OCC) && (need & NEED_GRADU);
  s->head_tag = a.take<uint32_t>(rn ? occ : 1);
  s->head_pos = a.take<uint32_t>(rn ? occ : 1);
  s->head_len = a.take<uint32_t>(rn ? occ : 1);
  s->head_off = a.take<int64_t>(rn ? occ : 1);
  // value blocks (k_occ's layout at its smallest chunk) and their scan partials
  int64_t nblk = 1;
  std::vector<ScanDesc> bd;
  if (rn) {
    nblk = 0;
    for (int f = 0; f < pl.F; ++f) {
      const int64_t nb = std::max<int64_t>(1, ceil_div(pl.caps[f], OC_CH_SMALL));
      bd.push_back({nullptr, nullptr, nb, nullptr, nullptr});
      nblk += nb;
    }
  }
  s->rv_blk = a.take<int64_t>(nblk);
  s->rv_scan_part = a.take<int64_t>(rn ? std::max<int64_t>(scan_part_words(bd.data(), (int)bd.size()), 1) : 1);
  s->fix_list = a.take<int32_t>(rn ? 3 * RV_FIX_CAP : 1);
  s->fix_count = a.take<uint32_t>(1);
  s->head_count = a.take<int64_t>(RECD_MAX_FEAT);
  s->fallback = a.take<int32_t>(1);
  s->sc_ticket = a.take<uint32_t>(1);
  {
    std::vector<ScanDesc> d;
    for (int t = 0; t < pl.nts; ++t) d.push_back({nullptr, nullptr, rn ? pl.ts_cap[t] : 1, nullptr, nullptr});
    s->runs_scan_part = a.take<int64_t>(std::max<int64_t>(scan_part_words(d.data(), (int)d.size()), 1));
  }
  s->occ_k0 = a.take<uint32_t>(occ);
  s->occ_v0 = a.take<uint32_t>(occ);
  s->occ_k1 = a.take<uint32_t>(occ);
  s->occ_v1 = a.take<uint32_t>(occ);
  // sort histograms: max of the inverse sort and the table sort
  std::vector<SegDesc> segs;
  // the inverse-CSR sort and the occurrence sort get separate sort state, so
  // the two stages may run concurrently (RECD_BWD_SETUP, TrainStep)
  int64_t hw_inv = 0, hw = 0;
  if (need & NEED_INV) {
    for (int i = 0; i < pl.nis; ++i) segs.push_back({(int64_t)i * B, B, nullptr});
    if (!segs.empty()) hw_inv = sort_hist_words(segs.data(), (int)segs.size());
  }
  segs.clear();
  if (need & NEED_OCC) {
    for (int t = 0; t < pl.nts; ++t) segs.push_back({pl.ts_base[t], pl.ts_cap[t], nullptr});
    hw = sort_hist_words(segs.data(), (int)segs.size());
  }
  s->hist = a.take<uint32_t>(std::max<int64_t>(hw, 256));
  s->hist_inv = a.take<uint32_t>(std::max<int64_t>(hw_inv, 256));
  // run-count scan partials (one scan segment per table)
  std::vector<ScanDesc> sd;
  for (int t = 0; t < pl.nts; ++t) {
    const int64_t nch = std::max<int64_t>(1, ceil_div(pl.ts_cap[t], pl.rc));
    sd.push_back({nullptr, nullptr, nch, nullptr, nullptr});
  }
  s->scan_part = a.take<int64_t>(std::max<int64_t>(scan_part_words(sd.data(), (int)sd.size()), 1));
  return a.used;
}

// Shared driver of the three backward entry points.
//   full    : grad_u (scratch) -> occurrences -> sort -> scatter
//   grad    : grad_u written to caller buffers only
//   scatter : occurrences -> sort -> scatter, reading caller unique-row grads
enum class BwdMode { Full, GradOnly, ScatterOnly };

// Occurrences as diagonal runs (k_rv*, one sort element per run) instead of
// one per unique value; RECD_BWD_RUNS=0/1 in the environment (read per call)
// overrides the default.
#ifndef RECD_BWD_RUNS
#define RECD_BWD_RUNS 0
#endif
static bool use_runs() {
  const char* e = getenv("RECD_BWD_RUNS");
  return e ? (atoi(e) != 0) : (RECD_BWD_RUNS != 0);
}
// stages (include/recd.h RECD_BWD_*): inverse CSR, occurrence sort, unique-row
// gradients, scatter; prepare = the first two, finish = the last two
enum { PH_INV = 1, PH_OCC = 2, PH_GRAD = 4, PH_SCAT = 8,
       PH_PREP = PH_INV | PH_OCC, PH_FINISH = PH_GRAD | PH_SCAT, PH_ALL = PH_PREP | PH_FINISH,
       PH_SETUP = RECD_BWD_SETUP, PH_SETUP_DONE = RECD_BWD_SETUP_DONE };

int run_bwd(BwdMode bm, int F, int64_t B, int dim, int mode, float* const* tables,
            const int64_t* table_rows, const int64_t* const* uvalues,
            const int64_t* const* uoffsets, const int64_t* value_caps, const int64_t* counts,
            const int64_t* const* inverse, const float* const* grad_out, float* const* gout_ext,
            const float* const* grow_ext, float lr, int apply_sgd, int64_t* const* grad_ids_out,
            float* const* grad_rows_out, int64_t* grad_counts_out, void* scratch,
            size_t scratch_bytes, cudaStream_t stream, int phase = PH_ALL,
            int gsegs = 0, float* const* gseg_dst = nullptr,
            const int64_t* const* gseg_row0 = nullptr,
            const int32_t** csr_start_out = nullptr, const uint32_t** csr_rows_out = nullptr) {
  if (F <= 0 || F > RECD_MAX_FEAT || B <= 0 || dim <= 0 || !counts) return RECD_ERR_ARG;
  if (mode != RECD_POOL_SUM && mode != RECD_POOL_AVG) return RECD_ERR_UNSUPPORTED;
  if (B >= (1ll << 24)) return RECD_ERR_UNSUPPORTED;  // occurrence tags hold u in 24 bits
  const bool do_grad = bm != BwdMode::ScatterOnly;
  const bool do_scatter = bm != BwdMode::GradOnly;
  std::vector<float*> dummy_tables(F, nullptr);
  std::vector<int64_t> dummy_rows(F, 1), dummy_caps(F, 1);
  for (int f = 0; f < F; ++f) {
    if (!uoffsets[f]) return RECD_ERR_ARG;
    if (do_grad && (phase & PH_GRAD) && !grad_out[f]) return RECD_ERR_ARG;
    if (bm == BwdMode::GradOnly && !gout_ext[f]) return RECD_ERR_ARG;
    if (bm == BwdMode::ScatterOnly && !grow_ext[f]) return RECD_ERR_ARG;
    if (do_scatter) {
      if (!tables[f]) return RECD_ERR_ARG;
      if (table_rows[f] <= 0 || table_rows[f] > (1ll << 32)) return RECD_ERR_UNSUPPORTED;
    } else {
      // grad-only: every feature its own (unused) table segment
      dummy_tables[f] = reinterpret_cast<float*>((uintptr_t)(f + 1) * 64);
    }
  }
  Plan pl = make_plan(F, do_grad ? inverse : nullptr, do_scatter ? tables : dummy_tables.data(),
                      do_scatter ? table_rows : dummy_rows.data(),
                      do_scatter ? value_caps : dummy_caps.data());
  if (pl.occ_total >= (1ll << 32)) return RECD_ERR_UNSUPPORTED;
  if (do_scatter && !apply_sgd && (!grad_ids_out || !grad_rows_out || !grad_counts_out))
    return RECD_ERR_ARG;
  const int need = (do_grad ? NEED_INV : 0) | (bm == BwdMode::Full ? NEED_GRADU : 0) |
                   (do_scatter ? NEED_OCC : 0);
  BwdScratch sc;
  if (carve_bwd(scratch, scratch_bytes, pl, B, dim, &sc, need) > scratch_bytes) return RECD_ERR_SCRATCH;

  BwdParams p;
  memset(&p, 0, sizeof(p));
  p.F = F;
  p.D = dim;
  p.mode = mode;
  p.B = B;
  p.apply_sgd = apply_sgd;
  p.lr = lr;
  p.nis = pl.nis;
  p.nts = pl.nts;
  p.counts = counts;
  p.Ftot = F;
  for (int f = 0; f < F; ++f) {
    p.uvalues[f] = uvalues ? uvalues[f] : nullptr;
    p.uoffsets[f] = uoffsets[f];
    p.grad_out[f] = (do_grad && grad_out) ? grad_out[f] : nullptr;
    p.feat_is[f] = pl.feat_is[f];
    p.feat_ts[f] = pl.feat_ts[f];
    if (bm == BwdMode::Full) {
      p.gout[f] = sc.grad_u + (int64_t)f * B * dim;
      p.grow[f] = p.gout[f];
    } else if (bm == BwdMode::GradOnly) {
      p.gout[f] = gout_ext[f];
    } else {
      p.grow[f] = grow_ext[f];
    }
  }
  for (int s = 0; s < pl.nis; ++s) {
    p.inverse[s] = pl.inverse[s];
    p.is_feat[s] = pl.is_feat[s];
  }
  int first_feat_of_ts[RECD_MAX_FEAT];
  for (int s = 0; s < pl.nts; ++s) first_feat_of_ts[s] = -1;
  for (int f = 0; f < F; ++f)
    if (first_feat_of_ts[pl.feat_ts[f]] < 0) first_feat_of_ts[pl.feat_ts[f]] = f;
  int feats_of_ts[RECD_MAX_FEAT] = {0};
  for (int f = 0; f < F; ++f) ++feats_of_ts[pl.feat_ts[f]];
  bool single = true;
  for (int s = 0; s < pl.nts; ++s) {
    p.seg_grow[s] = feats_of_ts[s] == 1 ? p.grow[first_feat_of_ts[s]] : nullptr;
    p.seg_feat[s] = first_feat_of_ts[s];
    single &= feats_of_ts[s] == 1;
    p.table[s] = pl.table[s];
    p.ts_base[s] = pl.ts_base[s];
    p.ts_chunk0[s] = pl.ts_chunk0[s];
    p.ts_rows[s] = pl.table_rows[s];
    if (do_scatter && !apply_sgd) {
      const int f = first_feat_of_ts[s];
      p.grad_ids[s] = grad_ids_out[f];
      p.grad_rows[s] = grad_rows_out[f];
      p.grad_count[s] = grad_counts_out + f;
    }
  }
  p.total_rc_chunks = pl.rc_chunks;
  if (gsegs < 0 || gsegs > 8 || (gsegs && (!gseg_dst || !gseg_row0))) return RECD_ERR_ARG;
  p.gsegs = gsegs;
  for (int f = 0; f < F && gsegs; ++f)
    for (int j = 0; j < gsegs; ++j) {
      p.gseg_dst[f][j] = gseg_dst[f * gsegs + j];
      p.gseg_row0[f][j] = gseg_row0[f * gsegs + j];
      if (!p.gseg_dst[f][j] || !p.gseg_row0[f][j]) return RECD_ERR_ARG;
    }
  p.feat_base = sc.feat_base;
  p.seg_count = sc.seg_count;
  p.is_count = sc.is_count;
  p.csr_start = sc.csr_start;
  p.run_part = sc.run_part;
  p.bad = sc.bad;
  p.head_tag = sc.head_tag;
  p.head_pos = sc.head_pos;
  p.head_len = sc.head_len;
  p.rv_blk = sc.rv_blk;
  p.fix_list = sc.fix_list;
  p.fix_count = sc.fix_count;
  p.head_off = sc.head_off;
  p.head_count = sc.head_count;
  p.fallback = sc.fallback;
  p.sc_ticket = sc.sc_ticket;
  const bool runs = bm == BwdMode::Full && do_scatter && single && use_runs();

  const bool fin = (phase & PH_FINISH) != 0;
  const bool run_grad = do_grad && (phase & PH_GRAD), run_scat = do_scatter && (phase & PH_SCAT);
  // sorted buffers: a stable LSD sort of `bits` bits ends in the alternate
  // buffers after an odd number of 8-bit passes
  auto odd_passes = [](int64_t bits) { return ((bits + 7) / 8) % 2 == 1; };
  int64_t maxrows = 1;
  for (int s = 0; s < pl.nts; ++s) maxrows = std::max(maxrows, pl.table_rows[s]);
  p.inv_keys = odd_passes(bits_for(B)) ? sc.inv_k1 : sc.inv_k0;
  p.inv_rows = odd_passes(bits_for(B)) ? sc.inv_v1 : sc.inv_v0;
  if (csr_start_out) {  // recd_pool_bwd_csr: where the inverse CSR lives, nothing launched
    for (int f = 0; f < F; ++f) {
      const int is = pl.feat_is[f];
      csr_start_out[f] = (do_grad && is >= 0) ? sc.csr_start + (int64_t)is * (B + 1) : nullptr;
      csr_rows_out[f] = (do_grad && is >= 0) ? p.inv_rows + (int64_t)is * B : nullptr;
    }
    return RECD_OK;
  }
  const bool odd = odd_passes(bits_for(maxrows));
  // the scatter's sorted occurrences: per-value sort result, or with runs the
  // expansion's output (the buffer pair the heads sort did not end in)
  p.occ_keys = (odd != runs) ? sc.occ_k1 : sc.occ_k0;
  p.occ_vals = (odd != runs) ? sc.occ_v1 : sc.occ_v0;
  p.exp_keys = p.occ_keys;
  p.exp_vals = p.occ_vals;

  // ---- prepare: everything that depends on the IKJT only (no gradient)
  if ((phase & PH_SETUP) || ((phase & PH_INV) && !(phase & PH_SETUP_DONE))) {
    pdl(k_bwd_setup, 1, 32, 0, stream)(p);
    note_launch();
  }
  {
    // 1. inverse CSR
    // (a one-CTA-per-segment kernel building the pairs, sorting them and
    // writing the run starts in one launch was slower at config 1 -- 0.119
    // vs 0.114 ms: the CSR then runs on 8 SMs on the side stream's critical
    // path; the sort alone takes the one-CTA path, k_local_sort)
    if ((phase & PH_INV) && do_grad && pl.nis > 0) {
      const int64_t n = (int64_t)pl.nis * B;
      pdl(k_inv_pairs, (unsigned)ceil_div(n, 256), 256, 0, stream)(p, sc.inv_k0, sc.inv_v0);
      note_launch();
      std::vector<SegDesc> segs;
      for (int s = 0; s < pl.nis; ++s) segs.push_back({(int64_t)s * B, B, sc.is_count + s});
      bool alt = false;
      int rc = seg_sort_pairs(segs.data(), pl.nis, (int)bits_for(B), sc.inv_k0, sc.inv_v0,
                              sc.inv_k1, sc.inv_v1, sc.hist_inv, &alt, stream);
      if (rc != RECD_OK) return rc;
      pdl(k_csr_bounds, (unsigned)ceil_div(n, 256), 256, 0, stream)(p);
      note_launch();
    }
    // 3-4. occurrences, sorted by ID per table segment
    if ((phase & PH_OCC) && do_scatter) {
      int64_t ob = 0;
      // 16K values per block on big batches, 4K on small ones, 1K on tiny
      // (config 1: ~120K values -- a latency-bound pass wants every SM busy)
      p.oc_ch = pl.occ_total >= (8ll << 20) ? OC_CH
                : (pl.occ_total >= (1ll << 20) || !RECD_TINY_CH) ? OC_CH_SMALL : OC_CH_SMALL / 4;
      for (int f = 0; f < F; ++f) {
        p.occ_blk0[f] = ob;
        ob += std::max<int64_t>(1, ceil_div(do_scatter ? value_caps[f] : 1, p.oc_ch));
      }
      p.occ_blk0[F] = ob;
      if (runs) {
        // 1. heads per value block -> block offsets -> heads in (u, p) order
        //    (+ the heads sort's digit histograms) -> run lengths
        p.oc_ch = OC_CH_SMALL;  // the block layout the scratch was sized for
        ob = 0;
        for (int f = 0; f < F; ++f) {
          p.occ_blk0[f] = ob;
          ob += std::max<int64_t>(1, ceil_div(value_caps[f], p.oc_ch));
        }
        p.occ_blk0[F] = ob;
        pdl(k_rv<0>, (unsigned)ob, 256, 0, stream)(p, nullptr, nullptr);
        std::vector<ScanDesc> bd;
        for (int f = 0; f < F; ++f)
          bd.push_back({sc.rv_blk + p.occ_blk0[f], sc.rv_blk + p.occ_blk0[f],
                        p.occ_blk0[f + 1] - p.occ_blk0[f], nullptr, sc.head_count + pl.feat_ts[f]});
        int r0 = seg_exclusive_scan(bd.data(), (int)bd.size(), sc.rv_scan_part, stream);
        if (r0 != RECD_OK) return r0;
        int rh = sort_hist_clear(pl.nts, sc.hist, stream);
        if (rh != RECD_OK) return rh;
        BwdParams q1 = p;
        q1.occ_hist = sc.hist;
        q1.occ_bits = (int)bits_for(maxrows);
        pdl(k_rv<1>, (unsigned)ob, 256, 0, stream)(q1, sc.occ_k0, sc.occ_v0);
        pdl(k_rv_len, (unsigned)num_sms() * 8, 256, 0, stream)(p);
        // 2. heads sorted by ID
        std::vector<SegDesc> hs;
        for (int s = 0; s < pl.nts; ++s) hs.push_back({pl.ts_base[s], pl.ts_cap[s], sc.head_count + s});
        bool halt = false;
        int r1 = seg_sort_pairs(hs.data(), pl.nts, (int)bits_for(maxrows), sc.occ_k0, sc.occ_v0,
                                sc.occ_k1, sc.occ_v1, sc.hist, &halt, stream, nullptr, true);
        if (r1 != RECD_OK) return r1;
        uint32_t* Hk = halt ? sc.occ_k1 : sc.occ_k0;
        uint32_t* Hv = halt ? sc.occ_v1 : sc.occ_v0;
        // 3. run lengths in sorted order (+ overlapping IDs) -> expanded offsets
        RECD_CUDA_CHECK(cudaMemsetAsync(sc.fix_count, 0, sizeof(uint32_t), stream));
        pdl(k_rv_lens, dim3((unsigned)num_sms() * 2, (unsigned)pl.nts), 256, 0, stream)(p, Hk, Hv);
        std::vector<ScanDesc> sd;
        for (int s = 0; s < pl.nts; ++s)
          sd.push_back({sc.head_off + pl.ts_base[s], sc.head_off + pl.ts_base[s], pl.ts_cap[s],
                        sc.head_count + s, nullptr});
        int r2 = seg_exclusive_scan(sd.data(), (int)sd.size(), sc.runs_scan_part, stream);
        if (r2 != RECD_OK) return r2;
        // 4. per-value occurrences in (ID, tag) order into the other buffer
        //    pair, then the overlapping IDs' tags re-sorted
        int64_t ec = 0;
        for (int s = 0; s < pl.nts; ++s) {
          p.ex_chunk0[s] = ec;
          ec += std::max<int64_t>(1, ceil_div(pl.ts_cap[s], RV_EX_CH));
        }
        pdl(k_rv_expand, (unsigned)ec, 256, 0, stream)(p, Hk, Hv);
        pdl(k_rv_fix, (unsigned)num_sms() * 2, 256, 0, stream)(p);
        note_launch(5);
        // 5. fallback (an overlapping ID with > RV_FIX_MAX values, or a full
        //    list): per-value occurrences + the full sort, gated on the flag;
        //    the sort is set up so that its result lands in the expansion's
        //    buffers
        uint32_t* Xk = odd ? Hk : p.exp_keys;
        uint32_t* Xv = odd ? Hv : p.exp_vals;
        uint32_t* Yk = odd ? p.exp_keys : Hk;
        uint32_t* Yv = odd ? p.exp_vals : Hv;
        BwdParams q = p;
        q.occ_gate = sc.fallback;
        q.oc_ch = OC_CH_SMALL;
        pdl(k_occ, (unsigned)ob, 256, 0, stream)(q, Xk, Xv);
        std::vector<SegDesc> vs;
        for (int s = 0; s < pl.nts; ++s) vs.push_back({pl.ts_base[s], pl.ts_cap[s], sc.seg_count + s});
        bool valt = false;
        int r3 = seg_sort_pairs(vs.data(), pl.nts, (int)bits_for(maxrows), Xk, Xv, Yk, Yv, sc.hist,
                                &valt, stream, sc.fallback);
        if (r3 != RECD_OK) return r3;
        note_launch(4);
      } else {
        // k_occ counts the sort's digits as it writes the keys (no histogram
        // pass over the keys in the sort)
        const bool fuse = RECD_OCC_HIST && pl.nts <= RECD_MAX_FEAT;
        if (fuse) {
          int rh = sort_hist_clear(pl.nts, sc.hist, stream);
          if (rh != RECD_OK) return rh;
        }
        BwdParams q = p;
        q.occ_hist = fuse ? sc.hist : nullptr;
        q.occ_bits = (int)bits_for(maxrows);
        pdl(k_occ, (unsigned)ob, 256, 0, stream)(q, sc.occ_k0, sc.occ_v0);
        note_launch();
        std::vector<SegDesc> segs;
        for (int s = 0; s < pl.nts; ++s) segs.push_back({pl.ts_base[s], pl.ts_cap[s], sc.seg_count + s});
        bool alt = false;
        int r2 = seg_sort_pairs(segs.data(), pl.nts, (int)bits_for(maxrows), sc.occ_k0, sc.occ_v0,
                                sc.occ_k1, sc.occ_v1, sc.hist, &alt, stream, nullptr, fuse);
        if (r2 != RECD_OK) return r2;
      }
    }
  }
  if (!fin) {
    RECD_LAUNCH_CHECK();
    return RECD_OK;
  }
  // ---- finish: gradient-dependent work
  if (run_scat && !apply_sgd)
    RECD_CUDA_CHECK(cudaMemsetAsync(grad_counts_out, 0, sizeof(int64_t) * F, stream));
  // Fused SGD: unique-row gradients and the scatter may run in groups of
  // table segments (RECD_SC_GROUP env: segments per group), so a group's
  // gradients are still in L2 when its scatter gathers them.
  int group = 0;
  if (const char* e = getenv("RECD_SC_GROUP")) group = atoi(e);
  if (!(run_grad && run_scat && apply_sgd) || group <= 0 || group >= pl.nts) group = pl.nts;
  int rc = RECD_OK;
  for (int s0 = 0; s0 < pl.nts && rc == RECD_OK; s0 += group) {
    const int s1 = std::min(pl.nts, s0 + group);
    uint64_t mask = 0;
    for (int f = 0; f < F; ++f)
      if (pl.feat_ts[f] >= s0 && pl.feat_ts[f] < s1) mask |= 1ull << f;
    if (group == pl.nts) mask = ~0ull;
    p.gu_mask = mask;
    p.sc_chunk_lo = pl.ts_chunk0[s0];
    p.sc_chunk_hi = s1 < pl.nts ? pl.ts_chunk0[s1] : pl.rc_chunks;
    rc = RECD_DISPATCH_COL_VW(dim, RECD_BWD_VW, RECD_BWD_FULLOK, {
    const int ncb = col_blocks<C>(dim);
    // 2. unique-row gradients
    if (run_grad) {
      const unsigned grid =
          (unsigned)std::min<int64_t>(ceil_div(B * F * ncb, 8), (int64_t)num_sms() * 16);
      bool any_id = !RECD_GU_FLAT, any_inv = false;
      for (int f = 0; f < F; ++f) (p.feat_is[f] < 0 ? any_id : any_inv) = true;
      if (any_id) {
        pdl(k_grad_u<C>, grid, 256, 0, stream)(p);
        note_launch();
      }
      if (RECD_GU_FLAT && any_inv) {
        const bool small = B < 32768;  // latency-bound: 32-position tasks
        const int ch = small ? GU_CH_SMALL : GU_CH;
        const unsigned gf = (unsigned)std::min<int64_t>(
            ceil_div(ceil_div(B, ch) * F * ncb, 8), (int64_t)num_sms() * 16);
        if (small)
          pdl(k_grad_u_flat<C, GU_CH_SMALL>, std::max(gf, 1u), 256, 0, stream)(p);
        else
          pdl(k_grad_u_flat<C, GU_CH>, std::max(gf, 1u), 256, 0, stream)(p);
        note_launch();
      }
    }
    // 5. sorted scatter-add (+ fused SGD)
    if (run_scat) {
      if (!apply_sgd && s0 == 0) {
        if (pl.rc == RC_BIG)
          pdl(k_run_count<RC_BIG>, (unsigned)pl.rc_chunks, RC_BIG, 0, stream)(p);
        else
          pdl(k_run_count<RC_SMALL>, (unsigned)pl.rc_chunks, RC_SMALL, 0, stream)(p);
        note_launch();
        std::vector<ScanDesc> sd;
        for (int s = 0; s < pl.nts; ++s) {
          const int64_t nch = std::max<int64_t>(1, ceil_div(pl.ts_cap[s], pl.rc));
          sd.push_back({sc.run_part + pl.ts_chunk0[s], sc.run_part + pl.ts_chunk0[s], nch,
                        nullptr, p.grad_count[s]});
        }
        int r3 = seg_exclusive_scan(sd.data(), (int)sd.size(), sc.scan_part, stream);
        if (r3 != RECD_OK) return r3;
      }
      // One task per warp (the grid covers every chunk, cap 128 CTAs per SM):
      // CTAs start in chunk order, so the warps in flight work on neighbouring
      // chunks and each CTA's slot is refilled as soon as it drains.  cfg2:
      // scatter 1.83-1.85 ms vs 1.95 with a 16-per-SM grid-stride loop (whose
      // later iterations jump far ahead in the chunk order).  RECD_SC_DYN:
      // resident grid taking tasks from a ticket counter: 1.90 ms.
      static const int sc_dyn = getenv("RECD_SC_DYN") ? atoi(getenv("RECD_SC_DYN")) : 0;
      p.sc_dyn = sc_dyn;
      if (sc_dyn) RECD_CUDA_CHECK(cudaMemsetAsync(sc.sc_ticket, 0, sizeof(uint32_t), stream));
      const unsigned g2 =
          (unsigned)std::min<int64_t>(ceil_div((p.sc_chunk_hi - p.sc_chunk_lo) * ncb, 8),
                                      grid_cap("RECD_SC_CTAS", sc_dyn ? RECD_SCATTER_MINB : 128));
      hook_before("k_scatter", stream);
      if (pl.rc == RC_BIG) {
        if (single)
          pdl(k_scatter<C, true, RC_BIG>, std::max(g2, 1u), 256, 0, stream)(p);
        else
          pdl(k_scatter<C, false, RC_BIG>, std::max(g2, 1u), 256, 0, stream)(p);
      } else {
        if (single)
          pdl(k_scatter<C, true, RC_SMALL>, std::max(g2, 1u), 256, 0, stream)(p);
        else
          pdl(k_scatter<C, false, RC_SMALL>, std::max(g2, 1u), 256, 0, stream)(p);
      }
      hook_after("k_scatter", stream);
      note_launch();
    }
  });
  }
  if (rc != RECD_OK) return rc;
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

Plan worst_plan(int F, const int64_t* caps) {
  // worst case: every feature has its own inverse and its own table
  std::vector<const int64_t*> inv(F);
  std::vector<float*> tab(F);
  std::vector<int64_t> rows(F, 1), ones(F, 1);
  for (int f = 0; f < F; ++f) {
    inv[f] = reinterpret_cast<const int64_t*>((uintptr_t)(f + 1) * 64);
    tab[f] = reinterpret_cast<float*>((uintptr_t)(f + 1) * 64);
  }
  return make_plan(F, inv.data(), tab.data(), rows.data(), caps ? caps : ones.data());
}

}  // namespace

extern "C" size_t recd_pool_bwd_scratch_bytes(int32_t num_features, int64_t batch_size,
                                              int32_t dim, const int64_t* value_caps) {
  if (num_features <= 0 || num_features > RECD_MAX_FEAT) return 0;
  Plan pl = worst_plan(num_features, value_caps);
  BwdScratch s;
  return carve_bwd(nullptr, 0, pl, batch_size, dim, &s);
}

extern "C" int recd_pool_bwd(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                             float* const* tables, const int64_t* table_rows,
                             const int64_t* const* uvalues, const int64_t* const* uoffsets,
                             const int64_t* value_caps, const int64_t* counts,
                             const int64_t* const* inverse, const float* const* grad_out,
                             float lr, int32_t apply_sgd, int64_t* const* grad_ids_out,
                             float* const* grad_rows_out, int64_t* grad_counts_out,
                             void* scratch, size_t scratch_bytes, recd_stream_t stream) {
  recd::PdlScope pdl_scope(batch_size * (int64_t)num_features);
  return run_bwd(BwdMode::Full, num_features, batch_size, dim, mode, tables, table_rows, uvalues,
                 uoffsets, value_caps, counts, inverse, grad_out, nullptr, nullptr, lr, apply_sgd,
                 grad_ids_out, grad_rows_out, grad_counts_out, scratch, scratch_bytes,
                 (cudaStream_t)stream);
}

// Split form of recd_pool_bwd: _prepare enqueues the gradient-independent
// half (inverse CSR, occurrence pairs, their sort by ID) and may run on a side
// stream as soon as the IKJT exists, overlapping the forward; _finish (same
// arguments, same scratch) enqueues the gradient reduction and the scatter.
extern "C" int recd_pool_bwd_prepare(int32_t num_features, int64_t batch_size, int32_t dim,
                                     int32_t mode, float* const* tables, const int64_t* table_rows,
                                     const int64_t* const* uvalues, const int64_t* const* uoffsets,
                                     const int64_t* value_caps, const int64_t* counts,
                                     const int64_t* const* inverse, const float* const* grad_out,
                                     float lr, int32_t apply_sgd, int64_t* const* grad_ids_out,
                                     float* const* grad_rows_out, int64_t* grad_counts_out,
                                     void* scratch, size_t scratch_bytes, recd_stream_t stream) {
  recd::PdlScope pdl_scope(batch_size * (int64_t)num_features);
  return run_bwd(BwdMode::Full, num_features, batch_size, dim, mode, tables, table_rows, uvalues,
                 uoffsets, value_caps, counts, inverse, grad_out, nullptr, nullptr, lr, apply_sgd,
                 grad_ids_out, grad_rows_out, grad_counts_out, scratch, scratch_bytes,
                 (cudaStream_t)stream, PH_PREP);
}

extern "C" int recd_pool_bwd_finish(int32_t num_features, int64_t batch_size, int32_t dim,
                                    int32_t mode, float* const* tables, const int64_t* table_rows,
                                    const int64_t* const* uvalues, const int64_t* const* uoffsets,
                                    const int64_t* value_caps, const int64_t* counts,
                                    const int64_t* const* inverse, const float* const* grad_out,
                                    float lr, int32_t apply_sgd, int64_t* const* grad_ids_out,
                                    float* const* grad_rows_out, int64_t* grad_counts_out,
                                    void* scratch, size_t scratch_bytes, recd_stream_t stream) {
  recd::PdlScope pdl_scope(batch_size * (int64_t)num_features);
  return run_bwd(BwdMode::Full, num_features, batch_size, dim, mode, tables, table_rows, uvalues,
                 uoffsets, value_caps, counts, inverse, grad_out, nullptr, nullptr, lr, apply_sgd,
                 grad_ids_out, grad_rows_out, grad_counts_out, scratch, scratch_bytes,
                 (cudaStream_t)stream, PH_FINISH);
}

extern "C" int recd_pool_bwd_csr(int32_t num_features, int64_t batch_size, int32_t dim,
                                 int32_t mode, float* const* tables, const int64_t* table_rows,
                                 const int64_t* const* uvalues, const int64_t* const* uoffsets,
                                 const int64_t* value_caps, const int64_t* counts,
                                 const int64_t* const* inverse, const float* const* grad_out,
                                 float lr, int32_t apply_sgd, int64_t* const* grad_ids_out,
                                 float* const* grad_rows_out, int64_t* grad_counts_out,
                                 void* scratch, size_t scratch_bytes,
                                 const int32_t** csr_start_out, const uint32_t** csr_rows_out) {
  if (!csr_start_out || !csr_rows_out) return RECD_ERR_ARG;
  return run_bwd(BwdMode::Full, num_features, batch_size, dim, mode, tables, table_rows, uvalues,
                 uoffsets, value_caps, counts, inverse, grad_out, nullptr, nullptr, lr, apply_sgd,
                 grad_ids_out, grad_rows_out, grad_counts_out, scratch, scratch_bytes, nullptr,
                 PH_INV, 0, nullptr, nullptr, csr_start_out, csr_rows_out);
}

extern "C" int recd_pool_bwd_stages(int32_t stages, int32_t num_features, int64_t batch_size,
                                    int32_t dim, int32_t mode, float* const* tables,
                                    const int64_t* table_rows, const int64_t* const* uvalues,
                                    const int64_t* const* uoffsets, const int64_t* value_caps,
                                    const int64_t* counts, const int64_t* const* inverse,
                                    const float* const* grad_out, float lr, int32_t apply_sgd,
                                    int64_t* const* grad_ids_out, float* const* grad_rows_out,
                                    int64_t* grad_counts_out, void* scratch, size_t scratch_bytes,
                                    recd_stream_t stream) {
  recd::PdlScope pdl_scope(batch_size * (int64_t)num_features);
  if (stages <= 0 || (stages & ~(PH_ALL | PH_SETUP | PH_SETUP_DONE))) return RECD_ERR_ARG;
  return run_bwd(BwdMode::Full, num_features, batch_size, dim, mode, tables, table_rows, uvalues,
                 uoffsets, value_caps, counts, inverse, grad_out, nullptr, nullptr, lr, apply_sgd,
                 grad_ids_out, grad_rows_out, grad_counts_out, scratch, scratch_bytes,
                 (cudaStream_t)stream, stages);
}

extern "C" size_t recd_grad_unique_scratch_bytes(int32_t num_features, int64_t batch_size) {
  if (num_features <= 0 || num_features > RECD_MAX_FEAT) return 0;
  Plan pl = worst_plan(num_features, nullptr);
  BwdScratch s;
  return carve_bwd(nullptr, 0, pl, batch_size, 1, &s, NEED_INV);
}

extern "C" int recd_grad_unique(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                                const int64_t* const* uoffsets, const int64_t* counts,
                                const int64_t* const* inverse, const float* const* grad_out,
                                float* const* grad_u_out, void* scratch, size_t scratch_bytes,
                                recd_stream_t stream) {
  return run_bwd(BwdMode::GradOnly, num_features, batch_size, dim, mode, nullptr, nullptr, nullptr,
                 uoffsets, nullptr, counts, inverse, grad_out, grad_u_out, nullptr, 0.f, 1,
                 nullptr, nullptr, nullptr, scratch, scratch_bytes, (cudaStream_t)stream);
}

// recd_grad_unique whose rows go straight to the owners' receive buffers (the
// push of unique-row gradients fused into the segment reduce): feature f's row
// u is stored at seg_dst[f * num_segs + j] + (*seg_row0[f * num_segs + j] + u) * dim
// for every j < num_segs (<= 8; seg_row0 on the device, seg_dst may be peer memory).
extern "C" int recd_grad_unique_scatter(int32_t num_features, int64_t batch_size, int32_t dim,
                                        int32_t mode, const int64_t* const* uoffsets,
                                        const int64_t* counts, const int64_t* const* inverse,
                                        const float* const* grad_out, int32_t num_segs,
                                        const int64_t* const* seg_row0, float* const* seg_dst,
                                        void* scratch, size_t scratch_bytes, recd_stream_t stream) {
  if (num_segs <= 0 || num_segs > 8 || !seg_dst || num_features <= 0 || num_features > RECD_MAX_FEAT)
    return RECD_ERR_ARG;
  std::vector<float*> first(num_features);
  for (int f = 0; f < num_features; ++f) first[f] = seg_dst[(int64_t)f * num_segs];
  return run_bwd(BwdMode::GradOnly, num_features, batch_size, dim, mode, nullptr, nullptr, nullptr,
                 uoffsets, nullptr, counts, inverse, grad_out, first.data(), nullptr, 0.f, 1,
                 nullptr, nullptr, nullptr, scratch, scratch_bytes, (cudaStream_t)stream, PH_ALL,
                 num_segs, seg_dst, seg_row0);
}

extern "C" size_t recd_sparse_sgd_scratch_bytes(int32_t num_features, const int64_t* value_caps) {
  if (num_features <= 0 || num_features > RECD_MAX_FEAT) return 0;
  Plan pl = worst_plan(num_features, value_caps);
  BwdScratch s;
  return carve_bwd(nullptr, 0, pl, 1, 1, &s, NEED_OCC);
}

extern "C" int recd_sparse_sgd(int32_t num_features, int64_t max_rows, int32_t dim,
                               float* const* tables, const int64_t* table_rows,
                               const int64_t* const* uvalues, const int64_t* const* uoffsets,
                               const int64_t* value_caps, const int64_t* counts,
                               const float* const* grad_rows, float lr, int32_t apply_sgd,
                               int64_t* const* grad_ids_out, float* const* grad_rows_out,
                               int64_t* grad_counts_out, void* scratch, size_t scratch_bytes,
                               recd_stream_t stream) {
  return run_bwd(BwdMode::ScatterOnly, num_features, max_rows, dim, RECD_POOL_SUM, tables,
                 table_rows, uvalues, uoffsets, value_caps, counts, nullptr, nullptr, nullptr,
                 grad_rows, lr, apply_sgd, grad_ids_out, grad_rows_out, grad_counts_out, scratch,
                 scratch_bytes, (cudaStream_t)stream);
}

// Split form of recd_sparse_sgd (same arguments, same scratch): _prepare
// (occurrence pairs + sort by ID) needs only the owner's ID lists and can run
// while the unique-row gradients are still being produced / pushed.
extern "C" int recd_sparse_sgd_prepare(int32_t num_features, int64_t max_rows, int32_t dim,
                               float* const* tables, const int64_t* table_rows,
                               const int64_t* const* uvalues, const int64_t* const* uoffsets,
                               const int64_t* value_caps, const int64_t* counts,
                               const float* const* grad_rows, float lr, int32_t apply_sgd,
                               int64_t* const* grad_ids_out, float* const* grad_rows_out,
                               int64_t* grad_counts_out, void* scratch, size_t scratch_bytes,
                               recd_stream_t stream) {
  return run_bwd(BwdMode::ScatterOnly, num_features, max_rows, dim, RECD_POOL_SUM, tables,
                 table_rows, uvalues, uoffsets, value_caps, counts, nullptr, nullptr, nullptr,
                 grad_rows, lr, apply_sgd, grad_ids_out, grad_rows_out, grad_counts_out, scratch,
                 scratch_bytes, (cudaStream_t)stream, PH_PREP);
}

extern "C" int recd_sparse_sgd_finish(int32_t num_features, int64_t max_rows, int32_t dim,
                               float* const* tables, const int64_t* table_rows,
                               const int64_t* const* uvalues, const int64_t* const* uoffsets,
                               const int64_t* value_caps, const int64_t* counts,
                               const float* const* grad_rows, float lr, int32_t apply_sgd,
                               int64_t* const* grad_ids_out, float* const* grad_rows_out,
                               int64_t* grad_counts_out, void* scratch, size_t scratch_bytes,
                               recd_stream_t stream) {
  return run_bwd(BwdMode::ScatterOnly, num_features, max_rows, dim, RECD_POOL_SUM, tables,
                 table_rows, uvalues, uoffsets, value_caps, counts, nullptr, nullptr, nullptr,
                 grad_rows, lr, apply_sgd, grad_ids_out, grad_rows_out, grad_counts_out, scratch,
                 scratch_bytes, (cudaStream_t)stream, PH_FINISH);
}
