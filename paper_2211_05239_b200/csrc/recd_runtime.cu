// Library-level bookkeeping: version, launch counter, SM count cache.
#include <atomic>

#include "recd_common.cuh"

namespace recd {

static std::atomic<int64_t> g_launches{0};

void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

}  // namespace recd

extern "C" int recd_version(void) { return 1; }

extern "C" int64_t recd_launch_count(void) { return recd::g_launches.load(); }

extern "C" const char* recd_last_error(void) {
  cudaError_t e = cudaPeekAtLastError();
  return e == cudaSuccess ? "" : cudaGetErrorString(e);
}
