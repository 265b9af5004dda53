// Random 512-byte row gather probe, three transports:
//   reg   : LDG.128 per lane into registers, U rows in flight per warp
//   ldgsts: cp.async 16 B per lane into a per-warp shared ring
//   bulk  : one cp.async.bulk (TMA, 512 B) per row into a per-warp shared
//           ring, completion on an mbarrier per batch of 8 rows
// Prints GB/s of row bytes for several table footprints.  Build on the box:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_probe2 tools/gather_probe2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t h) {
  h ^= h >> 16; h *= 0x85ebca6bu; h ^= h >> 13; h *= 0xc2b2ae35u;
  return h ^ (h >> 16);
}
__device__ __forceinline__ uint64_t rowof(uint64_t w, int64_t i, uint64_t seed, uint64_t rows) {
  return mix((uint32_t)(seed ^ (w * 0x9E3779B1u + i))) & (rows - 1);
}

template <int U>
__global__ void __launch_bounds__(256) k_reg(const float4* __restrict__ t, uint64_t rows, int64_t per_warp,
                                             uint64_t seed, float* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t i = 0; i < per_warp; i += U) {
    float4 x[U];
#pragma unroll
    for (int k = 0; k < U; ++k) x[k] = __ldg(t + rowof(w, i + k, seed, rows) * 32 + lane);
#pragma unroll
    for (int k = 0; k < U; ++k) { acc.x += x[k].x; acc.y += x[k].y; acc.z += x[k].z; acc.w += x[k].w; }
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

template <int NB>  // batches of 8 rows in flight
__global__ void __launch_bounds__(256) k_ldgsts(const float4* __restrict__ t, uint64_t rows,
                                                int64_t per_warp, uint64_t seed, float* out) {
  extern __shared__ float4 ring[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t w = (uint64_t)blockIdx.x * 8 + warp;
  float4* my = ring + warp * NB * 8 * 32 + lane;
  float4 acc = make_float4(0, 0, 0, 0);
  const int64_t nb = per_warp / 8;
  auto issue = [&](int64_t b) {
    if (b < nb)
      for (int k = 0; k < 8; ++k) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(my + ((b % NB) * 8 + k) * 32);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa),
                     "l"(t + rowof(w, b * 8 + k, seed, rows) * 32 + lane));
      }
    asm volatile("cp.async.commit_group;\n");
  };
  for (int b = 0; b < NB; ++b) issue(b);
  for (int64_t b = 0; b < nb; ++b) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NB - 1) : "memory");
    for (int k = 0; k < 8; ++k) {
      const float4 v = my[((b % NB) * 8 + k) * 32];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    issue(b + NB);
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

__device__ __forceinline__ void mbar_init(uint64_t* m, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(m);
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
               "r"((uint32_t)__cvta_generic_to_shared(m)) : "memory");
}

template <int NB>
__global__ void __launch_bounds__(256) k_bulk(const float4* __restrict__ t, uint64_t rows, int64_t per_warp,
                                              uint64_t seed, float* out) {
  extern __shared__ float4 ring[];
  __shared__ __align__(8) uint64_t mbar[8][NB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t w = (uint64_t)blockIdx.x * 8 + warp;
  float4* my = ring + warp * NB * 8 * 32;
  if (lane < NB) mbar_init(&mbar[warp][lane], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  float4 acc = make_float4(0, 0, 0, 0);
  const int64_t nb = per_warp / 8;
  auto issue = [&](int64_t b) {
    if (b < nb) {
      uint64_t* m = &mbar[warp][b % NB];
      if (lane == 0) mbar_expect(m, 8 * 512);
      __syncwarp();
      if (lane < 8)
        bulk_g2s(my + ((b % NB) * 8 + lane) * 32, t + rowof(w, b * 8 + lane, seed, rows) * 32, 512, m);
    }
  };
  for (int b = 0; b < NB; ++b) issue(b);
  for (int64_t b = 0; b < nb; ++b) {
    mbar_wait(&mbar[warp][b % NB], (uint32_t)((b / NB) & 1));
    for (int k = 0; k < 8; ++k) {
      const float4 v = my[((b % NB) * 8 + k) * 32 + lane];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    __syncwarp();
    issue(b + NB);
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

// random row read-modify-write (the scatter's table update): U rows in flight
template <int U>
__global__ void __launch_bounds__(256) k_rmw(float4* __restrict__ t, uint64_t rows, int64_t per_warp,
                                             uint64_t seed, float* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  for (int64_t i = 0; i < per_warp; i += U) {
    float4 x[U];
    uint64_t r[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      r[k] = rowof(w, i + k, seed, rows);
      x[k] = t[r[k] * 32 + lane];
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      x[k].x += 1.f;
      t[r[k] * 32 + lane] = x[k];
    }
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t max_bytes = 32ull << 30;
  float4* t;
  if (cudaMalloc(&t, max_bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(t, 0, max_bytes);
  float* out;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8;
  const int64_t per_warp = 4096;
  const double bytes = (double)blocks * 8 * per_warp * 512;
  auto run_rmw = [&](const char* name, auto kern, uint64_t rows) {
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
      cudaEventRecord(e0);
      kern<<<blocks, 256>>>(t, rows, per_warp / 4, 777 + it, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it) best = ms < best ? ms : best;
    }
    printf("%8llu MB %-10s %8.0f GB/s (read+write)  %s\n", (unsigned long long)(rows * 512 >> 20), name,
           2 * bytes / 4 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  auto run = [&](const char* name, auto kern, int smem, uint64_t rows) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
      cudaEventRecord(e0);
      kern<<<blocks, 256, smem>>>(t, rows, per_warp, 12345 + it, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it) best = ms < best ? ms : best;
    }
    printf("%8llu MB %-10s %8.0f GB/s  %s\n", (unsigned long long)(rows * 512 >> 20), name, bytes / best / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (uint64_t mb : {64ull, 1024ull, 8192ull, 32768ull}) {
    const uint64_t rows = (mb << 20) / 512;
    run_rmw("rmw4", k_rmw<4>, rows);
    run_rmw("rmw8", k_rmw<8>, rows);
    run("reg8", k_reg<8>, 0, rows);
    run("reg16", k_reg<16>, 0, rows);
    run("ldgsts2", k_ldgsts<2>, 8 * 2 * 8 * 512, rows);
    run("ldgsts4", k_ldgsts<4>, 8 * 4 * 8 * 512, rows);
    run("bulk2", k_bulk<2>, 8 * 2 * 8 * 512, rows);
    run("bulk4", k_bulk<4>, 8 * 4 * 8 * 512, rows);
  }
  return 0;
}
