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
#ifndef RECD_POOL_VW
#define RECD_POOL_VW 4
#endif
#ifndef RECD_POOL_MINB
#define RECD_POOL_MINB 2
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
};

template <class C>
__global__ void __launch_bounds__(256, RECD_POOL_MINB) k_pool_fwd(const __grid_constant__ PoolParams p) {
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
    C::st(p.pooled[f] + u * p.D + cw.lo, cw.ok, acc);
  }
}

// out[f][i] = pooled[f][inverse[f][i]]  (trainer_sim.py:558-561)
template <class C>
__global__ void __launch_bounds__(256) k_expand(const __grid_constant__ PoolParams p) {
  __shared__ int64_t s_pref[RECD_MAX_FEAT + 1];
  const int ncb = col_blocks<C>(p.D);
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int f = 0; f < p.F; ++f) {
      s_pref[f] = acc;
      const bool active = p.out[f] != nullptr && p.out[f] != p.pooled[f];
      acc += active ? p.B * ncb : 0;
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
    const int64_t i = cw.row;
    const int64_t u = p.inverse[f] ? __ldg(p.inverse[f] + i) : i;
    float x[C::VW];
    C::ld(p.pooled[f] + u * p.D + cw.lo, cw.ok, x);
    C::st(p.out[f] + i * p.D + cw.lo, cw.ok, x);
  }
}

template <class C>
__global__ void __launch_bounds__(256) k_lookup(const float* W, int64_t rows, int D,
                                                const int64_t* ids, int64_t n, float* out,
                                                int64_t* err) {
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

static unsigned grid_for(int64_t warps) {
  int64_t blocks = ceil_div(std::max<int64_t>(warps, 1), 8);
  const int64_t cap = (int64_t)num_sms() * 16;
  return (unsigned)std::min(blocks, cap);
}

}  // namespace recd

using namespace recd;

extern "C" int recd_pool_fwd(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                             const float* const* tables, const int64_t* table_rows,
                             const int64_t* const* uvalues, const int64_t* const* uoffsets,
                             const int64_t* counts, const int64_t* const* inverse,
                             float* const* pooled_out, float* const* out, int64_t* err,
                             recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
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
      p.pooled[f] = pooled_out[f0 + f];
      p.out[f] = out ? out[f0 + f] : nullptr;
      if (!p.tables[f] || !p.uoffsets[f] || !p.pooled[f]) return RECD_ERR_ARG;
      if (dim % 2 == 0 && ((uintptr_t)p.tables[f] % 8 || (uintptr_t)p.pooled[f] % 8 ||
                           (p.out[f] && (uintptr_t)p.out[f] % 8)))
        return RECD_ERR_ARG;
    }
    bool any_expand = false;
    for (int f = 0; f < p.F; ++f) any_expand |= (p.out[f] != nullptr && p.out[f] != p.pooled[f]);
    int rc = RECD_DISPATCH_COL_VW(dim, RECD_POOL_VW, 1, {
      const unsigned grid = grid_for(batch_size * p.F * col_blocks<C>(dim));
      hook_before("k_pool_fwd", stream);
      k_pool_fwd<C><<<grid, 256, 0, stream>>>(p);
      hook_after("k_pool_fwd", stream);
      note_launch();
      if (any_expand) {
        k_expand<C><<<grid, 256, 0, stream>>>(p);
        note_launch();
      }
    });
    if (rc != RECD_OK) return rc;
    RECD_LAUNCH_CHECK();
  }
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
    k_lookup<C><<<grid_for(n * col_blocks<C>(dim)), 256, 0, stream>>>(table, table_rows, dim,
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
    k_pool_dense<C><<<grid_for(n_rows * col_blocks<C>(dim)), 256, 0, stream>>>(
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
      k_expand<C><<<grid_for(batch_size * p.F * col_blocks<C>(dim)), 256, 0, stream>>>(p);
      note_launch();
    });
    if (rc != RECD_OK) return rc;
    RECD_LAUNCH_CHECK();
  }
  return RECD_OK;
}
