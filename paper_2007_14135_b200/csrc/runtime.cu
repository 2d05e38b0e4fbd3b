// Per-device launch configuration cache.
//
// Kernel attributes (cudaFuncAttributeMaxDynamicSharedMemorySize), occupancies and SM counts are
// properties of a (kernel, device) pair, so they are cached per device: a process that drives
// several GPUs (one plan per device) configures every kernel on every device it launches on.
// The cache is guarded by a mutex (plans may be used from several host threads, one stream each).
#include <mutex>
#include <tuple>
#include <vector>

#include "doa_internal.cuh"

namespace doa {
namespace {

struct Entry {
  const void* func;
  int dev, threads;
  size_t smem;
  int occ;
};

std::mutex g_mu;
std::vector<Entry> g_cache;        // a few dozen entries at most: linear search
std::vector<int> g_sms;            // SM count per device ordinal (0 = unknown)

}  // namespace

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

int sm_count() {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_mu);
  if ((int)g_sms.size() <= dev) g_sms.resize(dev + 1, 0);
  if (!g_sms[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = n > 0 ? n : 148;
  }
  return g_sms[dev];
}

int kernel_occupancy(const void* func, int threads, size_t smem) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_mu);
  for (const Entry& e : g_cache)
    if (e.func == func && e.dev == dev && e.threads == threads && e.smem == smem) return e.occ;
  bool attr_set = false;
  for (const Entry& e : g_cache)
    if (e.func == func && e.dev == dev && e.smem >= smem) { attr_set = true; break; }
  if (!attr_set && smem > 48 * 1024)
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, func, threads, smem);
  if (occ < 1) occ = 1;
  g_cache.push_back({func, dev, threads, smem, occ});
  return occ;
}

}  // namespace doa
