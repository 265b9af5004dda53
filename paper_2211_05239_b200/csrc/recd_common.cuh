// Shared device helpers for librecd (sm_100a).
//
// Layout conventions (mirror the reference's JaggedTensor, tensors.py:60-111):
//   a jagged feature is values int64[N] + offsets int64[R], one offset per
//   row, the last row running to N.  All counts that are only known after a
//   kernel ran (U unique rows, N_u unique values) stay in device memory; the
//   kernels that consume them read them there, so a whole training step can
//   be enqueued (and graph-captured) without a host round trip.
#pragma once

#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/recd.h"

#define RECD_MAX_FEAT 64
#define RECD_WARP 32

#define RECD_CUDA_CHECK(expr)                                   \
  do {                                                          \
    cudaError_t _e = (expr);                                    \
    if (_e != cudaSuccess) return RECD_ERR_CUDA;                \
  } while (0)

#define RECD_LAUNCH_CHECK()                                     \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return RECD_ERR_CUDA;                \
  } while (0)

namespace recd {

// Number of kernels this library enqueued (host-side counter; reported by
// bench.py as "gpu_launches").
void note_launch(int n = 1);
void hook_before(const char* name, cudaStream_t s);
void hook_after(const char* name, cudaStream_t s);

int num_sms();
// grid cap of grid-stride kernels: `per_sm` CTAs per SM, or the value of the
// environment variable `env` (tuning / A/B knob) when set
inline int64_t grid_cap(const char* env, int per_sm) {
  const char* e = getenv(env);
  return (int64_t)num_sms() * (e ? (atoi(e) > 0 ? atoi(e) : 1) : per_sm);
}

// Programmatic dependent launch (PDL).  Every kernel starts with
// RECD_PDL_PROLOGUE(): griddepcontrol.wait blocks until the preceding kernel
// of the stream has completed and its memory is visible (a no-op when the
// kernel was launched without the attribute), then launch_dependents lets the
// next kernel's CTAs be scheduled as soon as every CTA of this one started.
// So a chain of small kernels (config 1: ~25 launches per step) overlaps each
// launch with its predecessor instead of paying the launch latency in series.
// pdl(k, grid, block, smem, stream)(args...) launches with the attribute
// while a PdlScope of the calling API entry point allows it (RECD_PDL=0 never,
// 1 always, default: steps of at most RECD_PDL_MAX batch rows x features --
// on big steps early-resident CTAs would only hold SM slots a concurrent
// side-stream kernel could use).
#define RECD_PDL_PROLOGUE()                                          \
  do {                                                               \
    asm volatile("griddepcontrol.wait;" ::: "memory");               \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  \
  } while (0)

bool pdl_allowed();
struct PdlScope {
  bool prev;
  explicit PdlScope(int64_t rows_x_features);
  ~PdlScope();
};

template <typename... KArgs>
struct PdlLaunch {
  void (*k)(KArgs...);
  dim3 grid, block;
  size_t smem;
  cudaStream_t stream;
  template <typename... Args>
  void operator()(Args&&... args) const {
    if (!pdl_allowed()) {
      k<<<grid, block, smem, stream>>>(args...);
      return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k, args...) != cudaSuccess) {
      // attribute refused: launch plainly (a real launch error then shows in
      // the caller's RECD_LAUNCH_CHECK)
      (void)cudaGetLastError();
      k<<<grid, block, smem, stream>>>(args...);
    }
  }
};
template <typename... KArgs>
PdlLaunch<KArgs...> pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem = 0,
                        cudaStream_t stream = 0) {
  return PdlLaunch<KArgs...>{k, grid, block, smem, stream};
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

__host__ __device__ inline uint64_t next_pow2(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// splitmix64 finalizer.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Position-dependent element hash; a row hash is the (mod 2^64) sum of its
// element hashes plus one length term per feature, so any partition of the
// row's values over threads yields the same row hash.
__device__ __forceinline__ uint64_t elem_hash(int64_t v, int64_t pos, int f) {
  return mix64((uint64_t)v ^ ((uint64_t)pos * 0x9E3779B97F4A7C15ull) ^
               ((uint64_t)(f + 1) * 0xD1B54A32D192ED03ull));
}
__device__ __forceinline__ uint64_t len_hash(int64_t len, int f) {
  return mix64(((uint64_t)len << 7) ^ ((uint64_t)(f + 7) * 0xA0761D6478BD642Full) ^ 0x5bd1e995ull);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// cp.async (LDGSTS): asynchronous global -> shared copy of 4/8/16 bytes per
// thread; in-flight copies hold no registers, so a warp can keep many table
// rows in flight.  Completion is per thread via commit/wait groups.
#ifndef RECD_CPASYNC_CLOBBER
#define RECD_CPASYNC_CLOBBER 0
#endif
#if RECD_CPASYNC_CLOBBER
#define RECD_CLOB : "memory"
#else
#define RECD_CLOB
#endif
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  if constexpr (BYTES == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) RECD_CLOB);
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES)
                 RECD_CLOB);
  }
}
// L2 eviction-priority policies (createpolicy) and the hinted accesses that
// use them: streamed data (table rows touched once) is marked evict_first so
// it does not push out data that is re-read (unique-row gradients).
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, uint64_t pol) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "l"(pol) RECD_CLOB);
}
__device__ __forceinline__ void st_v4_hint(float* p, float a, float b, float c, float d,
                                           uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(a),
               "f"(b), "f"(c), "f"(d), "l"(pol)
               : "memory");
}
__device__ __forceinline__ float4 ld_v4_hint(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// TMA bulk copies (cp.async.bulk, no tensor map): one thread moves a
// contiguous global range (16-byte aligned, size a multiple of 16) into shared
// memory; completion is counted on an mbarrier as transaction bytes.
__device__ __forceinline__ void mbar_init1(uint64_t* m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(m))
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(m)),
      "r"(parity)
      : "memory");
}
// arrive on `m` expecting `bytes`, then (bytes > 0) copy them global -> shared
__device__ __forceinline__ void bulk_load(void* smem, const void* gmem, uint32_t bytes, uint64_t* m) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(m);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
               : "memory");
  if (bytes)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(smem)),
        "l"(gmem), "r"(bytes), "r"(mb)
        : "memory");
}

__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" :: RECD_CLOB);
}
// Waits for this thread's older copy groups.  The shared-memory reads that
// follow are ordinary loads issued after the asm volatile in program order.
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Block-wide exclusive scan of one int64 per thread; returns the exclusive
// prefix, writes the block total to *total.  `smem` needs 32 int64 slots.
template <int NT>
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* smem, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) smem[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = (lane < NT / 32) ? smem[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    smem[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  int64_t base = warp ? smem[warp - 1] : 0;
  *total = smem[NT / 32 - 1];
  __syncthreads();
  return base + x - v;
}

// Block-wide inclusive max-scan of one int64 per thread.
template <int NT>
__device__ __forceinline__ int64_t block_inclusive_max(int64_t v, int64_t* smem, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x = max(x, y);
  }
  if (lane == 31) smem[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = (lane < NT / 32) ? smem[lane] : INT64_MIN;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w = max(w, y);
    }
    smem[lane] = w;
  }
  __syncthreads();
  int64_t r = warp ? max(x, smem[warp - 1]) : x;
  *total = smem[NT / 32 - 1];
  __syncthreads();
  return r;
}

// last f in [0, F) with first[f] <= b for non-decreasing block offsets
// first[0..F) (kernel parameter arrays: block -> feature)
__device__ __forceinline__ int block_feature(const int64_t* first, int F, int64_t b) {
  int lo = 0, hi = F - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (first[mid] <= b) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Last index k in [0, n) with a[k] <= x for a non-decreasing a with a[0] <= x,
// found by the whole warp with 32-ary probing (every lane returns it).
__device__ __forceinline__ int64_t warp_last_le(const int64_t* a, int64_t n, int64_t x, int lane) {
  // last index k in [0, n) with a[k] <= x (a non-decreasing, a[0] <= x)
  int64_t lo = 0, hi = n;  // answer in [lo, hi)
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t k = lo + (int64_t)lane * step;
    const bool le = k < hi && a[k] <= x;
    const unsigned b = __ballot_sync(0xffffffffu, le);
    const int last = 31 - __clz(b);  // lane 0 always qualifies
    lo = lo + (int64_t)last * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

// Scratch arena carving helper (256-byte aligned sub-buffers).
struct Arena {
  char* base;
  size_t cap;
  size_t used;
  __host__ Arena(void* p, size_t c) : base((char*)p), cap(c), used(0) {}
  template <class T>
  __host__ T* take(size_t n) {
    size_t bytes = (n * sizeof(T) + 255) & ~size_t(255);
    T* p = (T*)(base ? base + used : nullptr);
    used += bytes;
    return p;
  }
  __host__ bool ok() const { return used <= cap; }
};

}  // namespace recd
