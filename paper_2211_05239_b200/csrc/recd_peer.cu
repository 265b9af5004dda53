// Peer-memory (NVLink / NVSwitch) transport of the row-sharded step.
//
// B200-native replacement of the NCCL exchanges of the sharded step
// (SURVEY.md §8(e)): every rank exports one device allocation, the others map
// it (CUDA IPC), and the step's kernels store straight into the owner's /
// source's buffers over NVLink:
//   recd_shard_dispatch  unique IDs + row offsets   -> owner memory
//   recd_peer_copy_rows  partial rows (owner -> source), unique-row gradients
//                        (source -> owners), sizes read on the device
//   recd_peer_exchange   all-gather of the per-pair counts + barrier + plan
// No host synchronisation is left in the step, so fwd + bwd is captured once
// into a CUDA graph and replayed.
//
// Barrier protocol: every rank keeps a monotonically increasing epoch in its
// control block; an exchange stores epoch+1 into slot [rank] of every peer's
// flag array (st.release.sys after a system fence that orders the data stores
// of the preceding kernels) and spins (ld.acquire.sys, bounded by a globaltimer
// timeout) until all R flags of its own array reach epoch+1.  A timeout sets
// the error word; every later exchange then returns at once, so a lost peer
// can never hang the stream.
#include <cstring>

#include "recd_common.cuh"

namespace recd {

constexpr int PEER_MAXR = 64;
constexpr int PEER_MAXP = 256;
constexpr int CTL_EPOCH = 64;
constexpr int CTL_ERR = 65;
constexpr int CTL_META = 128;

__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ int64_t ld_volatile(const int64_t* p) {
  return *(const volatile int64_t*)p;
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct ExchangeParams {
  int R;
  int rank;
  int P;
  int S;
  int Q;
  int64_t timeout_ns;
  int64_t* ctl;                     // own control block
  int64_t* peer_ctl[PEER_MAXR];     // every rank's control block as mapped here
  const int64_t* totals;            // [P] or null (bare barrier)
  const int64_t* counts;            // [2F] local dedup counts
  int32_t owned[PEER_MAXP];
};

__global__ void __launch_bounds__(256) k_peer_exchange(const __grid_constant__ ExchangeParams p) {
  __shared__ int s_skip, s_fail;
  int64_t* ctl = p.ctl;
  const int t = threadIdx.x;
  if (t == 0) {
    s_skip = ld_volatile(ctl + CTL_ERR) != 0;
    s_fail = 0;
  }
  __syncthreads();
  if (s_skip) return;
  const int64_t ep = ld_volatile(ctl + CTL_EPOCH) + 1;
  const int W = 2 * p.P;
  if (p.totals) {
    // all-gather of this rank's meta row into every control block
    for (int i = t; i < p.R * W; i += blockDim.x) {
      const int r = i / W, k = i - r * W;
      const int64_t v = k < p.P ? p.totals[k] : p.counts[(k - p.P) / p.S];
      p.peer_ctl[r][CTL_META + (int64_t)p.rank * W + k] = v;
    }
  }
  __threadfence_system();
  __syncthreads();
  if (t < p.R) st_release_sys(p.peer_ctl[t] + p.rank, ep);
  if (t < p.R) {
    const uint64_t t0 = global_ns();
    while (ld_acquire_sys(ctl + t) < ep) {
      if ((int64_t)(global_ns() - t0) > p.timeout_ns) {
        s_fail = 1;
        break;
      }
      __nanosleep(128);
    }
  }
  __syncthreads();
  __threadfence_system();
  if (s_fail) {
    if (t == 0) {
      ctl[CTL_ERR] = 1;
      ctl[CTL_EPOCH] = ep;
    }
    return;
  }
  if (p.totals) {
    // plan of this rank (see include/recd.h)
    const int64_t* meta = ctl + CTL_META;
    int64_t* plan = ctl + CTL_META + (int64_t)p.R * W;
    for (int q = t; q < p.P; q += blockDim.x) {
      int64_t ib = 0, rb = 0;
      for (int s = 0; s < p.rank; ++s) {
        ib += ld_volatile(meta + (int64_t)s * W + q);
        rb += ld_volatile(meta + (int64_t)s * W + p.P + q);
      }
      plan[q] = ib;
      plan[p.P + q] = rb;
    }
    int64_t* own = plan + 2 * p.P;
    int64_t* own_base = own + 2 * p.Q;
    for (int q = t; q < p.Q; q += blockDim.x) {
      const int pi = p.owned[q];
      int64_t rows = 0, ids = 0;
      for (int s = 0; s < p.R; ++s) {
        own_base[(int64_t)q * p.R + s] = rows;
        rows += ld_volatile(meta + (int64_t)s * W + p.P + pi);
        ids += ld_volatile(meta + (int64_t)s * W + pi);
      }
      own[q] = rows;
      own[p.Q + q] = ids;
    }
  }
  __syncthreads();
  if (t == 0) ctl[CTL_EPOCH] = ep;
}

// Flat 16-byte copies of contiguous row ranges; blockIdx.y = segment.
__global__ void __launch_bounds__(256) k_copy_rows(const recd_row_seg* __restrict__ segs,
                                                   const int64_t* __restrict__ ctl, int row_bytes) {
  const recd_row_seg sg = segs[blockIdx.y];
  const int64_t n = sg.count_idx >= 0 ? ctl[sg.count_idx] : 0;
  if (n <= 0) return;
  const int64_t so = sg.src_off_idx >= 0 ? ctl[sg.src_off_idx] : 0;
  const int64_t d0 = sg.dst_off_idx >= 0 ? ctl[sg.dst_off_idx] : 0;
  const int4* __restrict__ src = (const int4*)((const char*)sg.src + so * row_bytes);
  int4* __restrict__ dst = (int4*)((char*)sg.dst + d0 * row_bytes);
  const int64_t nv = n * (row_bytes >> 4);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < nv; i += 4 * stride) {
    const int4 a = __ldg(src + i), b = __ldg(src + i + stride), c = __ldg(src + i + 2 * stride),
               d = __ldg(src + i + 3 * stride);
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < nv; i += stride) dst[i] = __ldg(src + i);
}

}  // namespace recd

using namespace recd;

extern "C" int64_t recd_peer_ctl_words(int32_t num_ranks, int32_t num_pairs, int32_t num_owned) {
  return CTL_META + (int64_t)num_ranks * 2 * num_pairs + 2 * (int64_t)num_pairs +
         2 * (int64_t)num_owned + (int64_t)num_owned * num_ranks;
}

extern "C" int recd_peer_alloc(size_t bytes, void** ptr_out) {
  if (!ptr_out || bytes == 0) return RECD_ERR_ARG;
  *ptr_out = nullptr;
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return RECD_ERR_CUDA;
  if (cudaMemset(p, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(p);
    return RECD_ERR_CUDA;
  }
  *ptr_out = p;
  return RECD_OK;
}

extern "C" int recd_peer_free(void* ptr) {
  return ptr && cudaFree(ptr) == cudaSuccess ? RECD_OK : RECD_ERR_CUDA;
}

extern "C" int recd_peer_export(const void* ptr, void* handle_out) {
  static_assert(sizeof(cudaIpcMemHandle_t) == RECD_PEER_HANDLE_BYTES, "IPC handle size");
  if (!ptr || !handle_out) return RECD_ERR_ARG;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, (void*)ptr) != cudaSuccess) return RECD_ERR_CUDA;
  memcpy(handle_out, &h, sizeof(h));
  return RECD_OK;
}

extern "C" int recd_peer_import(const void* handle, void** ptr_out) {
  if (!handle || !ptr_out) return RECD_ERR_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  *ptr_out = nullptr;
  if (cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return RECD_ERR_CUDA;
  return RECD_OK;
}

extern "C" int recd_peer_close(void* ptr) {
  return ptr && cudaIpcCloseMemHandle(ptr) == cudaSuccess ? RECD_OK : RECD_ERR_CUDA;
}

extern "C" int recd_peer_exchange(int32_t num_ranks, int32_t rank, int32_t num_pairs,
                                  int32_t num_shards, int32_t num_owned, const int32_t* owned,
                                  void* const* peer_ctl, const int64_t* totals,
                                  const int64_t* counts, int64_t timeout_ns,
                                  recd_stream_t stream) {
  const int R = num_ranks, P = num_pairs, Q = num_owned;
  if (R <= 0 || R > PEER_MAXR || rank < 0 || rank >= R || P < 0 || P > PEER_MAXP || Q < 0 ||
      Q > PEER_MAXP || !peer_ctl || timeout_ns <= 0)
    return RECD_ERR_ARG;
  if (totals && (num_shards <= 0 || P <= 0 || !counts || (Q > 0 && !owned))) return RECD_ERR_ARG;
  ExchangeParams p;
  memset(&p, 0, sizeof(p));
  p.R = R;
  p.rank = rank;
  p.P = totals ? P : 0;
  p.S = num_shards;
  p.Q = totals ? Q : 0;
  p.timeout_ns = timeout_ns;
  p.ctl = (int64_t*)peer_ctl[rank];
  p.totals = totals;
  p.counts = counts;
  for (int r = 0; r < R; ++r) {
    if (!peer_ctl[r]) return RECD_ERR_ARG;
    p.peer_ctl[r] = (int64_t*)peer_ctl[r];
  }
  for (int q = 0; q < p.Q; ++q) {
    if (owned[q] < 0 || owned[q] >= P) return RECD_ERR_ARG;
    p.owned[q] = owned[q];
  }
  k_peer_exchange<<<1, 256, 0, (cudaStream_t)stream>>>(p);
  note_launch();
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

extern "C" int recd_peer_copy_rows(int32_t num_segments, const recd_row_seg* segs,
                                   const int64_t* ctl, int32_t row_bytes, int64_t max_rows,
                                   recd_stream_t stream) {
  if (num_segments < 0 || num_segments > 65535 || row_bytes <= 0 || (row_bytes & 15) ||
      max_rows < 0 || (num_segments > 0 && (!segs || !ctl)))
    return RECD_ERR_ARG;
  if (num_segments == 0 || max_rows == 0) return RECD_OK;
  const int64_t vec = max_rows * (row_bytes >> 4);
  const int64_t want = ceil_div(vec, 256 * 4);
  const int64_t cap = std::max<int64_t>(1, (int64_t)num_sms() * 8 / num_segments);
  const dim3 grid((unsigned)std::max<int64_t>(1, std::min(want, cap)), (unsigned)num_segments);
  k_copy_rows<<<grid, 256, 0, (cudaStream_t)stream>>>(segs, ctl, row_bytes);
  note_launch();
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}
