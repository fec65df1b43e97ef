// Error state, launch accounting and device queries of the C ABI
// (include/sparseconv_b200.h).
#include <atomic>

#include "common.cuh"

namespace scb {
static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};
void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace scb

extern "C" const char* scb_last_error(void) { return scb::g_last_error.c_str(); }

extern "C" int32_t scb_abi_version(void) { return 2; }

extern "C" int64_t scb_launch_count(void) { return scb::g_launches.load(); }

extern "C" int32_t scb_device_sm_count(void) {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return v;
}
