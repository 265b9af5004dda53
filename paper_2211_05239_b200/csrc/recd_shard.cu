// Row-sharded embedding tables across R ranks (sm_100a kernels).
//
// North_star multi-GPU path: every rank deduplicates its own
// local batch (== slice_ikjt_rows, trainer_sim.py:394-413), the tables are
// row-sharded (owner(id) = id mod R, local row = id div R) and only
// deduplicated IDs go to the owners; owners return partially pooled rows, one
// per (source unique row), which the source sums in fixed owner order.
//
//   recd_shard_bucketize  unique values of every feature -> per-owner ID lists
//                         (owner-major, (u, pos) order inside) + per-(owner,
//                         unique row) counts (the jagged offsets the owner scans)
//   recd_shard_combine    pooled[u] = sum_{o = 0..R-1} partial[o][u] (fixed order),
//                         avg: / fp32(full row length)
//   recd_exclusive_scan   segmented exclusive scan (row counts -> offsets)
#include <algorithm>
#include <vector>

#include "recd_prims.cuh"
#include "recd_slice.cuh"

namespace recd {

constexpr int SH_MAXR = 64;

struct ShardParams {
  int F;
  int R;
  int64_t B;  // row capacity per (feature, owner) block of rowcnt / partial buffers
  const int64_t* uvalues[RECD_MAX_FEAT];
  const int64_t* uoffsets[RECD_MAX_FEAT];
  const int64_t* counts;  // [2F] device
  int64_t* ids_out[RECD_MAX_FEAT];      // owner-major local IDs
  int64_t* rowcnt[RECD_MAX_FEAT];       // [R][B] counts per (owner, unique row)
  const int64_t* rowoff[RECD_MAX_FEAT]; // [R][B] exclusive scan of rowcnt over u
  const int64_t* totals;                // [F][R] per-owner ID totals (scan totals)
};

// warp per (feature, unique row): per-owner counts of its values
__global__ void __launch_bounds__(256) k_shard_count(const __grid_constant__ ShardParams p) {
  __shared__ int64_t s_pref[RECD_MAX_FEAT + 1];
  __shared__ int32_t s_cnt[8][SH_MAXR];
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int f = 0; f < p.F; ++f) {
      s_pref[f] = acc;
      acc += p.counts[f];
    }
    s_pref[p.F] = acc;
  }
  __syncthreads();
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
    for (int o = lane; o < p.R; o += 32) cnt[o] = 0;
    __syncwarp();
    for (int64_t j0 = a; j0 < e; j0 += 32) {
      const int64_t j = j0 + lane;
      const bool valid = j < e;
      const int o = valid ? (int)(__ldg(p.uvalues[f] + j) % p.R) : SH_MAXR;
      const unsigned peers = __match_any_sync(0xffffffffu, o);
      if (valid && lane == __ffs(peers) - 1) cnt[o] += __popc(peers);
      __syncwarp();
    }
    for (int o = lane; o < p.R; o += 32) p.rowcnt[f][(int64_t)o * p.B + u] = cnt[o];
    __syncwarp();
  }
}

// warp per (feature, unique row): scatter local IDs to their owner segments
__global__ void __launch_bounds__(256) k_shard_scatter(const __grid_constant__ ShardParams p) {
  __shared__ int64_t s_pref[RECD_MAX_FEAT + 1];
  __shared__ int64_t s_run[8][SH_MAXR];
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int f = 0; f < p.F; ++f) {
      s_pref[f] = acc;
      acc += p.counts[f];
    }
    s_pref[p.F] = acc;
  }
  __syncthreads();
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
    // start of (owner o, row u) inside ids_out: owner base + row offset
    for (int o = lane; o < p.R; o += 32) {
      int64_t base = 0;
      for (int q = 0; q < o; ++q) base += p.totals[(int64_t)f * p.R + q];
      run[o] = base + p.rowoff[f][(int64_t)o * p.B + u];
    }
    __syncwarp();
    for (int64_t j0 = a; j0 < e; j0 += 32) {
      const int64_t j = j0 + lane;
      const bool valid = j < e;
      const int64_t id = valid ? __ldg(p.uvalues[f] + j) : 0;
      const int o = valid ? (int)(id % p.R) : SH_MAXR;
      const unsigned peers = __match_any_sync(0xffffffffu, o);
      int64_t pos = 0;
      if (valid) pos = run[o] + __popc(peers & lt);
      __syncwarp();
      if (valid && lane == __ffs(peers) - 1) run[o] += __popc(peers);
      __syncwarp();
      if (valid) p.ids_out[f][pos] = id / p.R;
    }
    __syncwarp();
  }
}

constexpr int SH_MAXBLK = 256;

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

extern "C" size_t recd_shard_scratch_bytes(int32_t num_features, int32_t num_ranks,
                                           int64_t batch_size) {
  Arena a(nullptr, 0);
  a.take<int64_t>((size_t)std::max(num_features, 1) * num_ranks * batch_size);  // rowoff
  a.take<int64_t>((size_t)std::max(num_features, 1) * num_ranks);              // totals
  std::vector<ScanDesc> sd((size_t)std::max(num_features, 1) * num_ranks,
                           ScanDesc{nullptr, nullptr, batch_size, nullptr, nullptr});
  a.take<int64_t>(scan_part_words(sd.data(), (int)sd.size()));
  return a.used;
}

extern "C" int recd_shard_bucketize(int32_t num_features, int32_t num_ranks, int64_t batch_size,
                                    const int64_t* const* uvalues, const int64_t* const* uoffsets,
                                    const int64_t* counts, int64_t* const* ids_out,
                                    int64_t* const* rowcnt_out, int64_t* totals_out,
                                    void* scratch, size_t scratch_bytes, recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  const int F = num_features, R = num_ranks;
  if (F <= 0 || F > RECD_MAX_FEAT || R <= 0 || R > SH_MAXR || batch_size <= 0 || !counts ||
      !totals_out)
    return RECD_ERR_ARG;
  if (recd_shard_scratch_bytes(F, R, batch_size) > scratch_bytes) return RECD_ERR_SCRATCH;
  Arena a(scratch, scratch_bytes);
  int64_t* rowoff = a.take<int64_t>((size_t)F * R * batch_size);
  ShardParams p;
  memset(&p, 0, sizeof(p));
  p.F = F;
  p.R = R;
  p.B = batch_size;
  p.counts = counts;
  p.totals = totals_out;
  for (int f = 0; f < F; ++f) {
    if (!uvalues[f] || !uoffsets[f] || !ids_out[f] || !rowcnt_out[f]) return RECD_ERR_ARG;
    p.uvalues[f] = uvalues[f];
    p.uoffsets[f] = uoffsets[f];
    p.ids_out[f] = ids_out[f];
    p.rowcnt[f] = rowcnt_out[f];
    p.rowoff[f] = rowoff + (int64_t)f * R * batch_size;
  }
  a.take<int64_t>((size_t)F * R);
  std::vector<ScanDesc> sd;
  for (int f = 0; f < F; ++f)
    for (int o = 0; o < R; ++o)
      sd.push_back({rowcnt_out[f] + (int64_t)o * batch_size,
                    rowoff + ((int64_t)f * R + o) * batch_size, batch_size, counts + f,
                    totals_out + (int64_t)f * R + o});
  int64_t* part = a.take<int64_t>(scan_part_words(sd.data(), (int)sd.size()));
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(batch_size * F, 8), (int64_t)num_sms() * 8);
  k_shard_count<<<grid, 256, 0, stream>>>(p);
  note_launch();
  int rc = seg_exclusive_scan(sd.data(), (int)sd.size(), part, stream);
  if (rc != RECD_OK) return rc;
  k_shard_scatter<<<grid, 256, 0, stream>>>(p);
  note_launch();
  RECD_LAUNCH_CHECK();
  return RECD_OK;
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
