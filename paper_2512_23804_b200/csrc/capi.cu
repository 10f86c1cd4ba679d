// Library-wide state of libsgkkt_b200: error string, launch counter, SM count.
#include <mutex>

#include "sgk_common.cuh"

namespace sgk {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }
void count_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int sm_count() {
  static int cached = 0;
  static std::mutex mu;
  if (cached) return cached;
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  cached = n > 0 ? n : 148;
  return cached;
}

}  // namespace sgk

extern "C" const char* sgk_last_error(void) { return sgk::g_err.c_str(); }
extern "C" int32_t sgk_version(void) { return 1; }
extern "C" int64_t sgk_launch_count(void) { return sgk::g_launches.load(); }
