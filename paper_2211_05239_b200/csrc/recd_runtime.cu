// Library-level bookkeeping: version, launch counter, SM count cache.
#include <atomic>
#include <cstdlib>
#include <string>

#include "recd_common.cuh"

namespace recd {

// Optional timing hook: CUDA events recorded right before / after the launch
// of one named kernel (bench.py times the dominant kernel live with it).
static std::string g_hook;
static cudaEvent_t g_ev0 = nullptr, g_ev1 = nullptr;
void hook_before(const char* name, cudaStream_t s) {
  if (g_ev0 && g_hook == name) cudaEventRecord(g_ev0, s);
}
void hook_after(const char* name, cudaStream_t s) {
  if (g_ev1 && g_hook == name) cudaEventRecord(g_ev1, s);
}

static std::atomic<int64_t> g_launches{0};

static thread_local bool t_pdl = false;
static int pdl_mode() {  // 0 never, 1 always, 2 small steps only
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("RECD_PDL");
    m = e ? (atoi(e) ? 1 : 0) : 2;
  }
  return m;
}
bool pdl_allowed() { return t_pdl; }
PdlScope::PdlScope(int64_t rows_x_features) : prev(t_pdl) {
  static const int64_t lim = getenv("RECD_PDL_MAX") ? atoll(getenv("RECD_PDL_MAX")) : (1 << 17);
  const int m = pdl_mode();
  t_pdl = m == 1 || (m == 2 && rows_x_features <= lim);
}
PdlScope::~PdlScope() { t_pdl = prev; }

void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    // experiment knob: L2 set-aside for evict_last / persisting lines (MB)
    if (const char* e = getenv("RECD_L2_PERSIST_MB"))
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)atoll(e) << 20);
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

extern "C" void recd_debug_kernel_events(const char* name, void* before, void* after) {
  recd::g_hook = name ? name : "";
  recd::g_ev0 = name ? (cudaEvent_t)before : nullptr;
  recd::g_ev1 = name ? (cudaEvent_t)after : nullptr;
}
