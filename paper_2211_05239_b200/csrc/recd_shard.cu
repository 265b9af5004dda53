// Row-sharded embedding tables (sm_100a kernels).
//
// North_star multi-GPU path: every rank deduplicates its own
// local batch (== slice_ikjt_rows, trainer_sim.py:394-413), every table is
// split into S row shards (shard(id) = id mod S, local row = id div S) and only
// deduplicated IDs go to the shard owners; owners return partially pooled rows,
// one per (source unique row, shard), which the source sums in shard order.
//
//   recd_shard_count      per-(shard, unique row) ID counts -> exclusive offsets
//                         + per-(table, shard) totals
//   recd_shard_dispatch   unique IDs -> per-(table, shard) lists ((u, pos) order
//                         inside), optionally with row offsets; destinations
//                         may be peer memory of the owner (NVLink stores)
//   recd_shard_bucketize  count + dispatch into local shard-major lists
//   recd_shard_combine    pooled[u] = sum_{j = 0..S-1} partial[j][u] (fixed order),
//                         avg: / fp32(full row length)
//   recd_exclusive_scan   segmented exclusive scan (row counts -> offsets)
#include <algorithm>
#include <vector>

#include "recd_prims.cuh"
#include "recd_slice.cuh"

namespace recd {

constexpr int SH_MAXR = 64;      // shards per table
constexpr int SH_MAXBLK = 256;   // (table, shard) pairs per call

struct CountParams {
  int F;
  int S;
  int64_t B;  // row capacity per (feature, shard) block of rowcnt
  const int64_t* uvalues[RECD_MAX_FEAT];
  const int64_t* uoffsets[RECD_MAX_FEAT];
  const int64_t* counts;                // [2F] device
  int64_t* rowcnt[RECD_MAX_FEAT];       // [S][B] IDs per (shard, unique row)
  int64_t* rowoff1[RECD_MAX_FEAT];      // S == 1: row offsets written directly
  int64_t* totals1;                     // S == 1: [F] IDs per feature
};

// Scatter of the unique IDs into per-(table, shard) pair lists.  Pair p =
// f * S + j gets its IDs at dst_ids[p] + id_base[p] + rowoff[f][j][u] + k (local
// row id div S); with dst_ro, also the row offsets dst_ro[p][row_base[p] + u] =
// id_base[p] + rowoff[f][j][u].  dst pointers may be peer (NVLink) memory.
struct DispatchParams {
  int F;
  int S;
  int64_t B;
  const int64_t* uvalues[RECD_MAX_FEAT];
  const int64_t* uoffsets[RECD_MAX_FEAT];
  const int64_t* counts;
  const int64_t* rowoff[RECD_MAX_FEAT];  // [S][B] exclusive scan of rowcnt over u
  const int64_t* totals;                 // [F * S] (id_base fallback: prefix over shards)
  const int64_t* id_base;                // [F * S] device, or null
  const int64_t* row_base;               // [F * S] device, or null (0)
  int64_t* dst_ids[SH_MAXBLK];
  int64_t* dst_ro[SH_MAXBLK];            // null: no row offsets
};

// Owner shard and local row of an ID.  A negative ID (out of range, reported by
// the owner's lookup) goes to shard 0 as local row -1, which every owner-side
// range check rejects; `id % S` would index in front of the per-shard arrays.
__device__ __forceinline__ int shard_of(int64_t id, int S, int64_t* local) {
  if (id < 0) {
    *local = -1;
    return 0;
  }
  *local = id / S;
  return (int)(id % S);
}

__device__ __forceinline__ void feature_prefix(int64_t* s_pref, const int64_t* counts, int F) {
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int f = 0; f < F; ++f) {
      s_pref[f] = acc;
      acc += counts[f];
    }
    s_pref[F] = acc;
  }
  __syncthreads();
}

// warp per (feature, unique row): per-shard counts of its values
__global__ void __launch_bounds__(256) k_shard_count(const __grid_constant__ CountParams p) {
  __shared__ int64_t s_pref[RECD_MAX_FEAT + 1];
  __shared__ int32_t s_cnt[8][SH_MAXR];
  feature_prefix(s_pref, p.counts, p.F);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* cnt = s_cnt[warp];
  const int64_t total = s_pref[p.F];
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; w < total; w += nwarps) {
    const int f = find_seg(s_pref, p.F, w);
    const int64_t u = w - s_pref[f];
    const int64_t U = p.counts[f], N = p.counts[p.F + f];
    const int64_t* uo = p.uoffsets[f];
    const int64_t a = uo[u], e = (u + 1 < U) ? uo[u + 1] : N;
    for (int o = lane; o < p.S; o += 32) cnt[o] = 0;
    __syncwarp();
    for (int64_t j0 = a; j0 < e; j0 += 32) {
      const int64_t j = j0 + lane;
      const bool valid = j < e;
      int64_t lr;
      const int o = valid ? shard_of(__ldg(p.uvalues[f] + j), p.S, &lr) : SH_MAXR;
      const unsigned peers = __match_any_sync(0xffffffffu, o);
      if (valid && lane == __ffs(peers) - 1) cnt[o] += __popc(peers);
      __syncwarp();
    }
    for (int o = lane; o < p.S; o += 32) p.rowcnt[f][(int64_t)o * p.B + u] = cnt[o];
    __syncwarp();
  }
}

// warp per (feature, unique row): scatter local IDs to their pair lists
__global__ void __launch_bounds__(256) k_shard_scatter(const __grid_constant__ DispatchParams p) {
  __shared__ int64_t s_pref[RECD_MAX_FEAT + 1];
  __shared__ int64_t s_run[8][SH_MAXR];
  feature_prefix(s_pref, p.counts, p.F);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  int64_t* run = s_run[warp];
  const int64_t total = s_pref[p.F];
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; w < total; w += nwarps) {
    const int f = find_seg(s_pref, p.F, w);
    const int64_t u = w - s_pref[f];
    const int64_t U = p.counts[f], N = p.counts[p.F + f];
    const int64_t* uo = p.uoffsets[f];
    const int64_t a = uo[u], e = (u + 1 < U) ? uo[u + 1] : N;
    // start of (shard o, row u) inside its pair list: pair base + row offset
    for (int o = lane; o < p.S; o += 32) {
      const int pi = f * p.S + o;
      int64_t base = 0;
      if (p.id_base) {
        base = p.id_base[pi];
      } else {
        for (int q = 0; q < o; ++q) base += p.totals[(int64_t)f * p.S + q];
      }
      const int64_t off = base + p.rowoff[f][(int64_t)o * p.B + u];
      run[o] = off;
      if (p.dst_ro[pi]) p.dst_ro[pi][(p.row_base ? p.row_base[pi] : 0) + u] = off;
    }
    __syncwarp();
    for (int64_t j0 = a; j0 < e; j0 += 32) {
      const int64_t j = j0 + lane;
      const bool valid = j < e;
      const int64_t id = valid ? __ldg(p.uvalues[f] + j) : 0;
      int64_t lr = 0;
      const int o = valid ? shard_of(id, p.S, &lr) : SH_MAXR;
      const unsigned peers = __match_any_sync(0xffffffffu, o);
      int64_t pos = 0;
      if (valid) pos = run[o] + __popc(peers & lt);
      __syncwarp();
      if (valid && lane == __ffs(peers) - 1) run[o] += __popc(peers);
      __syncwarp();
      if (valid) p.dst_ids[f * p.S + o][pos] = lr;
    }
    __syncwarp();
  }
}


// S == 1 (whole tables per owner, the cfg5 placement): every ID of a feature
// goes to one pair and keeps its position, so the per-row counts are the row
// lengths, the row offsets are the unique offsets and the dispatch is a flat,
// coalesced copy -- no per-row warp work.
__global__ void __launch_bounds__(256) k_shard_count1(const __grid_constant__ CountParams p) {
  const int f = blockIdx.y;
  const int64_t U = p.counts[f], N = p.counts[p.F + f];
  const int64_t* uo = p.uoffsets[f];
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < U;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = uo[u];
    p.rowoff1[f][u] = a;
    if (p.rowcnt[f]) p.rowcnt[f][u] = ((u + 1 < U) ? uo[u + 1] : N) - a;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) p.totals1[f] = N;
}

__global__ void __launch_bounds__(256) k_shard_scatter1(const __grid_constant__ DispatchParams p) {
  const int f = blockIdx.y;
  const int64_t U = p.counts[f], N = p.counts[p.F + f];
  const int64_t base = p.id_base ? p.id_base[f] : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t* src = p.uvalues[f];
  if (p.dst_ids[f]) {
    int64_t* dst = p.dst_ids[f] + base;
    for (int64_t j = t0; j < N; j += stride) dst[j] = __ldg(src + j);
  }
  if (p.dst_ro[f]) {
    int64_t* ro = p.dst_ro[f] + (p.row_base ? p.row_base[f] : 0);
    for (int64_t u = t0; u < U; u += stride) ro[u] = base + p.rowoff[f][u];
  }
}

struct CombineParams {
  int F;
  int R;  // partial blocks per feature
  int D;
  int mode;
  const float* blk[SH_MAXBLK];      // block (f, o) = blk[f * R + o], rows indexed by u
  float* pooled[RECD_MAX_FEAT];     // [U][D]
  const int64_t* uoffsets[RECD_MAX_FEAT];
  const int64_t* counts;            // [2F] local counts
};

template <class C>
__global__ void __launch_bounds__(256) k_shard_combine(const __grid_constant__ CombineParams p) {
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
  const int lane = threadIdx.x & 31;
  const int64_t total = s_pref[p.F];
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  constexpr int V = C::VW;
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total;
       w += nwarps) {
    const int f = find_seg(s_pref, p.F, w);
    const ColWork cw = col_work<C>(w - s_pref[f], p.D, lane);
    const int64_t u = cw.row;
    float acc[V], x[V];
    C::zero(acc);
    for (int o = 0; o < p.R; ++o) {
      C::ld(p.blk[f * p.R + o] + u * p.D + cw.lo, cw.ok, x);
#pragma unroll
      for (int e = 0; e < V; ++e) acc[e] = __fadd_rn(acc[e], x[e]);
    }
    if (p.mode == RECD_POOL_AVG) {
      const int64_t U = p.counts[f], N = p.counts[p.F + f];
      const int64_t* uo = p.uoffsets[f];
      const int64_t len = ((u + 1 < U) ? uo[u + 1] : N) - uo[u];
      if (len > 0) {
        const float fl = (float)len;
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] = __fdiv_rn(acc[e], fl);
      }
    }
    C::st(p.pooled[f] + u * p.D + cw.lo, cw.ok, acc);
  }
}

}  // namespace recd

using namespace recd;

static unsigned shard_grid(int64_t batch_size, int F) {
  return (unsigned)std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(batch_size * F, 8), (int64_t)num_sms() * 8));
}

extern "C" size_t recd_shard_count_scratch_bytes(int32_t num_features, int32_t num_shards,
                                                 int64_t batch_size) {
  Arena a(nullptr, 0);
  a.take<int64_t>((size_t)std::max(num_features, 1) * num_shards * batch_size);  // rowcnt
  std::vector<ScanDesc> sd((size_t)std::max(num_features, 1) * num_shards,
                           ScanDesc{nullptr, nullptr, batch_size, nullptr, nullptr});
  a.take<int64_t>(scan_part_words(sd.data(), (int)sd.size()));
  return a.used;
}

static int check_shard_args(int F, int S, int64_t batch_size, const int64_t* const* uvalues,
                            const int64_t* const* uoffsets, const int64_t* counts) {
  if (F <= 0 || F > RECD_MAX_FEAT || S <= 0 || S > SH_MAXR || (int64_t)F * S > SH_MAXBLK ||
      batch_size <= 0 || !counts || !uvalues || !uoffsets)
    return RECD_ERR_ARG;
  for (int f = 0; f < F; ++f)
    if (!uvalues[f] || !uoffsets[f]) return RECD_ERR_ARG;
  return RECD_OK;
}

// rowcnt: caller buffers ([S][B] per feature) or null (carved from scratch)
static int shard_count(int F, int S, int64_t batch_size, const int64_t* const* uvalues,
                       const int64_t* const* uoffsets, const int64_t* counts,
                       int64_t* const* rowcnt_out, int64_t* const* rowoff_out, int64_t* totals_out,
                       void* scratch, size_t scratch_bytes, cudaStream_t stream) {
  int rc = check_shard_args(F, S, batch_size, uvalues, uoffsets, counts);
  if (rc != RECD_OK) return rc;
  if (!rowoff_out || !totals_out) return RECD_ERR_ARG;
  if (recd_shard_count_scratch_bytes(F, S, batch_size) > scratch_bytes) return RECD_ERR_SCRATCH;
  Arena a(scratch, scratch_bytes);
  int64_t* rowcnt = a.take<int64_t>((size_t)F * S * batch_size);
  CountParams p;
  memset(&p, 0, sizeof(p));
  p.F = F;
  p.S = S;
  p.B = batch_size;
  p.counts = counts;
  std::vector<ScanDesc> sd;
  for (int f = 0; f < F; ++f) {
    if (!rowoff_out[f] || (rowcnt_out && !rowcnt_out[f])) return RECD_ERR_ARG;
    p.uvalues[f] = uvalues[f];
    p.uoffsets[f] = uoffsets[f];
    p.rowcnt[f] = rowcnt_out ? rowcnt_out[f] : rowcnt + (int64_t)f * S * batch_size;
    for (int o = 0; o < S; ++o)
      sd.push_back({p.rowcnt[f] + (int64_t)o * batch_size, rowoff_out[f] + (int64_t)o * batch_size,
                    batch_size, counts + f, totals_out + (int64_t)f * S + o});
  }
  int64_t* part = a.take<int64_t>(scan_part_words(sd.data(), (int)sd.size()));
  if (S == 1) {
    for (int f = 0; f < F; ++f) {
      if (!rowcnt_out) p.rowcnt[f] = nullptr;
      p.rowoff1[f] = rowoff_out[f];
    }
    p.totals1 = totals_out;
    const unsigned gx =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(batch_size, 256), 512));
    k_shard_count1<<<dim3(gx, F), 256, 0, stream>>>(p);
    note_launch();
    RECD_LAUNCH_CHECK();
    return RECD_OK;
  }
  k_shard_count<<<shard_grid(batch_size, F), 256, 0, stream>>>(p);
  note_launch();
  rc = seg_exclusive_scan(sd.data(), (int)sd.size(), part, stream);
  if (rc != RECD_OK) return rc;
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

extern "C" int recd_shard_count(int32_t num_features, int32_t num_shards, int64_t batch_size,
                                const int64_t* const* uvalues, const int64_t* const* uoffsets,
                                const int64_t* counts, int64_t* const* rowoff_out,
                                int64_t* totals_out, void* scratch, size_t scratch_bytes,
                                recd_stream_t stream) {
  return shard_count(num_features, num_shards, batch_size, uvalues, uoffsets, counts, nullptr,
                     rowoff_out, totals_out, scratch, scratch_bytes, (cudaStream_t)stream);
}

extern "C" int recd_shard_dispatch(int32_t num_features, int32_t num_shards, int64_t batch_size,
                                   const int64_t* const* uvalues, const int64_t* const* uoffsets,
                                   const int64_t* counts, const int64_t* const* rowoff,
                                   const int64_t* totals, const int64_t* id_base,
                                   const int64_t* row_base, int64_t* const* dst_ids,
                                   int64_t* const* dst_rowoffs, recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  const int F = num_features, S = num_shards;
  int rc = check_shard_args(F, S, batch_size, uvalues, uoffsets, counts);
  if (rc != RECD_OK) return rc;
  if (!rowoff || !dst_ids || (!id_base && !totals)) return RECD_ERR_ARG;
  DispatchParams p;
  memset(&p, 0, sizeof(p));
  p.F = F;
  p.S = S;
  p.B = batch_size;
  p.counts = counts;
  p.totals = totals;
  p.id_base = id_base;
  p.row_base = row_base;
  for (int f = 0; f < F; ++f) {
    if (!rowoff[f]) return RECD_ERR_ARG;
    p.uvalues[f] = uvalues[f];
    p.uoffsets[f] = uoffsets[f];
    p.rowoff[f] = rowoff[f];
  }
  for (int i = 0; i < F * S; ++i) {
    if (!dst_ids[i] && S != 1) return RECD_ERR_ARG;  // S == 1: null = IDs already placed
    p.dst_ids[i] = dst_ids[i];
    p.dst_ro[i] = dst_rowoffs ? dst_rowoffs[i] : nullptr;
  }
  if (S == 1) {
    int64_t vmax = batch_size;
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(vmax * 8, 256),
                                                                        (int64_t)num_sms() * 4));
    k_shard_scatter1<<<dim3(gx, F), 256, 0, stream>>>(p);
  } else {
    k_shard_scatter<<<shard_grid(batch_size, F), 256, 0, stream>>>(p);
  }
  note_launch();
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

extern "C" size_t recd_shard_scratch_bytes(int32_t num_features, int32_t num_shards,
                                           int64_t batch_size) {
  Arena a(nullptr, 0);
  a.take<int64_t>((size_t)std::max(num_features, 1) * num_shards * batch_size);  // rowoff
  a.take<uint8_t>(recd_shard_count_scratch_bytes(num_features, num_shards, batch_size));
  return a.used;
}

extern "C" int recd_shard_bucketize(int32_t num_features, int32_t num_shards, int64_t batch_size,
                                    const int64_t* const* uvalues, const int64_t* const* uoffsets,
                                    const int64_t* counts, int64_t* const* ids_out,
                                    int64_t* const* rowcnt_out, int64_t* totals_out,
                                    void* scratch, size_t scratch_bytes, recd_stream_t stream_) {
  const int F = num_features, S = num_shards;
  int rc = check_shard_args(F, S, batch_size, uvalues, uoffsets, counts);
  if (rc != RECD_OK) return rc;
  if (!ids_out || !rowcnt_out || !totals_out) return RECD_ERR_ARG;
  if (recd_shard_scratch_bytes(F, S, batch_size) > scratch_bytes) return RECD_ERR_SCRATCH;
  Arena a(scratch, scratch_bytes);
  int64_t* rowoff = a.take<int64_t>((size_t)F * S * batch_size);
  const size_t cbytes = recd_shard_count_scratch_bytes(F, S, batch_size);
  void* cscr = a.take<uint8_t>(cbytes);
  std::vector<int64_t*> ro(F);
  std::vector<int64_t*> dst((size_t)F * S);
  for (int f = 0; f < F; ++f) {
    if (!ids_out[f] || !rowcnt_out[f]) return RECD_ERR_ARG;
    ro[f] = rowoff + (int64_t)f * S * batch_size;
    for (int o = 0; o < S; ++o) dst[(size_t)f * S + o] = ids_out[f];
  }
  rc = shard_count(F, S, batch_size, uvalues, uoffsets, counts, rowcnt_out, ro.data(), totals_out,
                   cscr, cbytes, (cudaStream_t)stream_);
  if (rc != RECD_OK) return rc;
  return recd_shard_dispatch(F, S, batch_size, uvalues, uoffsets, counts, ro.data(), totals_out,
                             nullptr, nullptr, dst.data(), nullptr, stream_);
}

extern "C" int recd_shard_combine(int32_t num_features, int32_t num_blocks, int64_t batch_size,
                                  int32_t dim, int32_t mode, const float* const* blocks,
                                  const int64_t* const* uoffsets, const int64_t* counts,
                                  float* const* pooled_out, recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  const int F = num_features;
  if (F <= 0 || F > RECD_MAX_FEAT || num_blocks <= 0 || (int64_t)F * num_blocks > SH_MAXBLK ||
      dim <= 0 || !counts || !blocks)
    return RECD_ERR_ARG;
  if (mode != RECD_POOL_SUM && mode != RECD_POOL_AVG) return RECD_ERR_UNSUPPORTED;
  CombineParams p;
  memset(&p, 0, sizeof(p));
  p.F = F;
  p.R = num_blocks;
  p.D = dim;
  p.mode = mode;
  p.counts = counts;
  for (int i = 0; i < F * num_blocks; ++i) {
    if (!blocks[i]) return RECD_ERR_ARG;
    p.blk[i] = blocks[i];
  }
  for (int f = 0; f < F; ++f) {
    p.pooled[f] = pooled_out[f];
    p.uoffsets[f] = uoffsets[f];
  }
  int rc = RECD_DISPATCH_COL_VW(dim, 4, 0, {
    const unsigned grid = (unsigned)std::min<int64_t>(
        ceil_div(batch_size * F * col_blocks<C>(dim), 8), (int64_t)num_sms() * 16);
    k_shard_combine<C><<<grid, 256, 0, stream>>>(p);
    note_launch();
  });
  if (rc != RECD_OK) return rc;
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

extern "C" size_t recd_exclusive_scan_scratch_bytes(int32_t num_segments, const int64_t* caps) {
  std::vector<ScanDesc> sd;
  for (int s = 0; s < num_segments; ++s) sd.push_back({nullptr, nullptr, caps[s], nullptr, nullptr});
  return (size_t)std::max<int64_t>(scan_part_words(sd.data(), num_segments), 1) * sizeof(int64_t);
}

extern "C" int recd_exclusive_scan(int32_t num_segments, const int64_t* const* in,
                                   int64_t* const* out, const int64_t* caps,
                                   const int64_t* device_counts, int64_t* totals_out,
                                   void* scratch, size_t scratch_bytes, recd_stream_t stream) {
  if (num_segments <= 0) return RECD_ERR_ARG;
  if (recd_exclusive_scan_scratch_bytes(num_segments, caps) > scratch_bytes) return RECD_ERR_SCRATCH;
  std::vector<ScanDesc> sd;
  for (int s = 0; s < num_segments; ++s)
    sd.push_back({in[s], out[s], caps[s], device_counts ? device_counts + s : nullptr,
                  totals_out ? totals_out + s : nullptr});
  return seg_exclusive_scan(sd.data(), num_segments, (int64_t*)scratch, (cudaStream_t)stream);
}
