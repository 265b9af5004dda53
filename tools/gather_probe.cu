// Random-row gather probe: achievable bandwidth of 512-byte row gathers
// (one float4 per lane, a warp per row) as a function of the table footprint
// and of the loads in flight per warp.  Used to set the realistic roofline of
// the pool / scatter kernels.  Build + run on the GPU box:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_probe tools/gather_probe.cu
//   ./gather_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// cheap 32-bit mixer (index generation must not be the bottleneck)
__device__ __forceinline__ uint32_t mix(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  return h ^ (h >> 16);
}

// each warp: `per_warp` rows, U loads in flight, random rows in [0, rows)
template <int U>
__global__ void __launch_bounds__(256) k_gather(const float4* __restrict__ t, uint64_t rows,
                                                int64_t per_warp, uint64_t seed, float* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t i = 0; i < per_warp; i += U) {
    float4 x[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint64_t r = mix((uint32_t)(seed ^ (w * 0x9E3779B1u + i + k))) & (rows - 1);
      x[k] = __ldg(t + r * 32 + lane);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      acc.x += x[k].x; acc.y += x[k].y; acc.z += x[k].z; acc.w += x[k].w;
    }
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

// the same through a per-warp cp.async ring of K slots
template <int K>
__global__ void __launch_bounds__(256) k_gather_ring(const float4* __restrict__ t, uint64_t rows,
                                                     int64_t per_warp, uint64_t seed, float* out) {
  extern __shared__ float4 ring[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t w = (uint64_t)blockIdx.x * 8 + warp;
  float4* my = ring + warp * K * 32 + lane;
  float4 acc = make_float4(0, 0, 0, 0);
  auto issue = [&](int64_t i, int s) {
    if (i < per_warp) {
      const uint64_t r = mix((uint32_t)(seed ^ (w * 0x9E3779B1u + i))) & (rows - 1);
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(my + s * 32);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(t + r * 32 + lane));
    }
    asm volatile("cp.async.commit_group;\n");
  };
#pragma unroll
  for (int k = 0; k < K; ++k) issue(k, k);
  int s = 0;
  for (int64_t i = 0; i < per_warp; ++i) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(K - 1) : "memory");
    const float4 v = my[s * 32];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    issue(i + K, s);
    s = (s + 1 == K) ? 0 : s + 1;
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

template <class F>
static float time_it(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t max_bytes = (size_t)130 << 30;
  float4* t = nullptr;
  if (cudaMalloc(&t, max_bytes) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(t, 0, max_bytes);
  float* out;
  cudaMalloc(&out, 4);
  const size_t sizes_mb[] = {64, 256, 1024, 8192, 32768, 131072};
  const int64_t total_rows = 16 << 20;  // 8 GB of row reads per launch
  printf("footprint_MB, kernel, GB/s\n");
  for (size_t mb : sizes_mb) {
    uint64_t rows = 1;  // power of two <= footprint / 512 (mask instead of modulo)
    while (rows * 2 <= (uint64_t)mb * (1 << 20) / 512) rows *= 2;
    auto run_reg = [&](auto tag, int occ_blocks) {
      constexpr int U = decltype(tag)::value;
      const int blocks = sms * occ_blocks;
      const int64_t per_warp = total_rows / (blocks * 8);
      float ms = time_it([&] { k_gather<U><<<blocks, 256>>>(t, rows, per_warp, 7, out); });
      printf("%zu, reg_U%d_b%d, %.0f\n", mb, U, occ_blocks,
             (double)per_warp * blocks * 8 * 512 / (ms * 1e-3) / 1e9);
    };
    run_reg(std::integral_constant<int, 8>{}, 4);
    run_reg(std::integral_constant<int, 16>{}, 4);
    run_reg(std::integral_constant<int, 8>{}, 8);
    auto run_ring = [&](auto tag, int occ_blocks) {
      constexpr int K = decltype(tag)::value;
      const int smem = 8 * K * 512;
      cudaFuncSetAttribute(k_gather_ring<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int blocks = sms * occ_blocks;
      const int64_t per_warp = total_rows / (blocks * 8);
      float ms = time_it([&] { k_gather_ring<K><<<blocks, 256, smem>>>(t, rows, per_warp, 7, out); });
      printf("%zu, ring_K%d_b%d, %.0f\n", mb, K, occ_blocks,
             (double)per_warp * blocks * 8 * 512 / (ms * 1e-3) / 1e9);
    };
    run_ring(std::integral_constant<int, 16>{}, 3);
    run_ring(std::integral_constant<int, 32>{}, 2);
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
