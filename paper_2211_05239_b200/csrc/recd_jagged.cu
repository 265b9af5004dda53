// Jagged index select and DP slice renumbering (sm_100a).
//
// recd_jagged_index_select_*  <- tensors.jagged_index_select (tensors.py:363-390)
//                                 and ikjt_to_kjt (tensors.py:393-399): output row
//                                 k = input row idx[k], no densification.
// recd_slice_renumber         <- trainer_sim.slice_ikjt_rows (trainer_sim.py:394-413):
//                                 first-occurrence renumbering of a row range
//                                 without re-hashing.
#include <algorithm>
#include <vector>

#include "recd_prims.cuh"

namespace recd {

struct JagParams {
  int F;
  int64_t nrows;
  int64_t nidx;
  const int64_t* idx;
  int64_t* lens;  // [F][nidx]
  int64_t* err;
  const int64_t* values[RECD_MAX_FEAT];
  const int64_t* offsets[RECD_MAX_FEAT];
  int64_t nvalues[RECD_MAX_FEAT];
  const int64_t* out_offsets[RECD_MAX_FEAT];
  int64_t* out_values[RECD_MAX_FEAT];
};

__global__ void __launch_bounds__(256) k_sel_len(const __grid_constant__ JagParams p) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)p.F * p.nidx) return;
  const int f = (int)(t / p.nidx);
  const int64_t k = t - (int64_t)f * p.nidx;
  const int64_t i = p.idx[k];
  const bool bad = (uint64_t)i >= (uint64_t)p.nrows;
  if (bad) {
    if (f == 0) atomicMin(reinterpret_cast<unsigned long long*>(p.err), (unsigned long long)k);
    p.lens[t] = 0;
    return;
  }
  const int64_t* off = p.offsets[f];
  const int64_t e = (i + 1 < p.nrows) ? off[i + 1] : p.nvalues[f];
  p.lens[t] = e - off[i];
}

__global__ void __launch_bounds__(256) k_sel_copy(const __grid_constant__ JagParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)p.F * p.nidx;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total;
       w += nwarps) {
    const int f = (int)(w / p.nidx);
    const int64_t k = w - (int64_t)f * p.nidx;
    const int64_t i = p.idx[k];
    const int64_t* off = p.offsets[f];
    const int64_t s = off[i];
    const int64_t e = (i + 1 < p.nrows) ? off[i + 1] : p.nvalues[f];
    const int64_t* src = p.values[f] + s;
    int64_t* dst = p.out_values[f] + p.out_offsets[f][k];
    for (int64_t j = lane; j < e - s; j += 32) dst[j] = src[j];
  }
}

// ------------------------------------------------------------ slice
struct SliceParams {
  const int64_t* inv;  // already offset by start
  int64_t n;
  int64_t U;
  unsigned long long* firstpos;  // [U]
  int64_t* ex;                   // [n] flags, then their exclusive scan
  int64_t* lut;                  // [U]
  int64_t* new_inv;
  int64_t* order;
};

__global__ void k_sl_min(SliceParams p) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < p.n) atomicMin(&p.firstpos[p.inv[k]], (unsigned long long)k);
}
__global__ void k_sl_flag(SliceParams p) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < p.n) p.ex[k] = (p.firstpos[p.inv[k]] == (unsigned long long)k) ? 1 : 0;
}
__global__ void k_sl_lut(SliceParams p) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= p.n) return;
  const int64_t u = p.inv[k];
  if (p.firstpos[u] == (unsigned long long)k) {
    p.lut[u] = p.ex[k];
    p.order[p.ex[k]] = u;
  }
}
__global__ void k_sl_inv(SliceParams p) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < p.n) p.new_inv[k] = p.lut[p.inv[k]];
}

}  // namespace recd

using namespace recd;

extern "C" size_t recd_jagged_scratch_bytes(int32_t num_features, int64_t num_indices) {
  Arena a(nullptr, 0);
  a.take<int64_t>((size_t)std::max(num_features, 1) * std::max<int64_t>(num_indices, 1));
  std::vector<ScanDesc> sd(std::max(num_features, 1), ScanDesc{nullptr, nullptr, std::max<int64_t>(num_indices, 1), nullptr, nullptr});
  a.take<int64_t>(scan_part_words(sd.data(), (int)sd.size()));
  return a.used;
}

extern "C" int recd_jagged_index_select_plan(int32_t num_features, const int64_t* const* offsets,
                                             int64_t num_rows, const int64_t* num_values,
                                             const int64_t* indices, int64_t num_indices,
                                             int64_t* const* out_offsets, int64_t* totals_out,
                                             int64_t* err, void* scratch, size_t scratch_bytes,
                                             recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (num_features <= 0 || num_features > RECD_MAX_FEAT || num_rows < 0 || num_indices < 0 || !err ||
      !totals_out)
    return RECD_ERR_ARG;
  if (recd_jagged_scratch_bytes(num_features, num_indices) > scratch_bytes) return RECD_ERR_SCRATCH;
  RECD_CUDA_CHECK(cudaMemsetAsync(err, 0x7f, sizeof(int64_t), stream));
  if (num_indices == 0) {
    RECD_CUDA_CHECK(cudaMemsetAsync(totals_out, 0, sizeof(int64_t) * num_features, stream));
    return RECD_OK;
  }
  Arena a(scratch, scratch_bytes);
  JagParams p;
  memset(&p, 0, sizeof(p));
  p.F = num_features;
  p.nrows = num_rows;
  p.nidx = num_indices;
  p.idx = indices;
  p.err = err;
  p.lens = a.take<int64_t>((size_t)num_features * num_indices);
  std::vector<ScanDesc> sd(num_features);
  for (int f = 0; f < num_features; ++f) {
    p.offsets[f] = offsets[f];
    p.nvalues[f] = num_values[f];
    sd[f] = ScanDesc{p.lens + (int64_t)f * num_indices, out_offsets[f], num_indices, nullptr,
                     totals_out + f};
  }
  int64_t* part = a.take<int64_t>(scan_part_words(sd.data(), num_features));
  const int64_t n = (int64_t)num_features * num_indices;
  k_sel_len<<<(unsigned)ceil_div(n, 256), 256, 0, stream>>>(p);
  note_launch();
  RECD_LAUNCH_CHECK();
  return seg_exclusive_scan(sd.data(), num_features, part, stream);
}

extern "C" int recd_jagged_index_select_copy(int32_t num_features, const int64_t* const* values,
                                             const int64_t* const* offsets, int64_t num_rows,
                                             const int64_t* num_values, const int64_t* indices,
                                             int64_t num_indices, const int64_t* const* out_offsets,
                                             int64_t* const* out_values, recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (num_features <= 0 || num_features > RECD_MAX_FEAT || num_indices < 0) return RECD_ERR_ARG;
  if (num_indices == 0) return RECD_OK;
  JagParams p;
  memset(&p, 0, sizeof(p));
  p.F = num_features;
  p.nrows = num_rows;
  p.nidx = num_indices;
  p.idx = indices;
  for (int f = 0; f < num_features; ++f) {
    p.values[f] = values[f];
    p.offsets[f] = offsets[f];
    p.nvalues[f] = num_values[f];
    p.out_offsets[f] = out_offsets[f];
    p.out_values[f] = out_values[f];
  }
  const int64_t warps = (int64_t)num_features * num_indices;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(warps, 8), (int64_t)num_sms() * 8);
  k_sel_copy<<<grid, 256, 0, stream>>>(p);
  note_launch();
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

extern "C" size_t recd_slice_scratch_bytes(int64_t num_unique, int64_t num_rows) {
  Arena a(nullptr, 0);
  a.take<unsigned long long>(std::max<int64_t>(num_unique, 1));
  a.take<int64_t>(std::max<int64_t>(num_rows, 1));
  a.take<int64_t>(std::max<int64_t>(num_unique, 1));
  ScanDesc sd{nullptr, nullptr, std::max<int64_t>(num_rows, 1), nullptr, nullptr};
  a.take<int64_t>(scan_part_words(&sd, 1));
  return a.used;
}

extern "C" int recd_slice_renumber(const int64_t* inverse, int64_t start, int64_t stop,
                                   int64_t num_unique, int64_t* new_inverse_out, int64_t* order_out,
                                   int64_t* count_out, void* scratch, size_t scratch_bytes,
                                   recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!inverse || start < 0 || stop <= start || num_unique <= 0 || !count_out) return RECD_ERR_ARG;
  const int64_t n = stop - start;
  if (recd_slice_scratch_bytes(num_unique, n) > scratch_bytes) return RECD_ERR_SCRATCH;
  Arena a(scratch, scratch_bytes);
  SliceParams p;
  p.inv = inverse + start;
  p.n = n;
  p.U = num_unique;
  p.firstpos = a.take<unsigned long long>(num_unique);
  p.ex = a.take<int64_t>(n);
  p.lut = a.take<int64_t>(num_unique);
  p.new_inv = new_inverse_out;
  p.order = order_out;
  ScanDesc sd{p.ex, p.ex, n, nullptr, count_out};
  int64_t* part = a.take<int64_t>(scan_part_words(&sd, 1));
  RECD_CUDA_CHECK(cudaMemsetAsync(p.firstpos, 0x7f, sizeof(unsigned long long) * num_unique, stream));
  const unsigned g = (unsigned)ceil_div(n, 256);
  k_sl_min<<<g, 256, 0, stream>>>(p);
  k_sl_flag<<<g, 256, 0, stream>>>(p);
  note_launch(2);
  int rc = seg_exclusive_scan(&sd, 1, part, stream);
  if (rc != RECD_OK) return rc;
  k_sl_lut<<<g, 256, 0, stream>>>(p);
  k_sl_inv<<<g, 256, 0, stream>>>(p);
  note_launch(2);
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}
