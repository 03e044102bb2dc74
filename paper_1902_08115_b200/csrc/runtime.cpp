// Per-device runtime state of the launchers, thread-safe.
//
// The reference is stateless and re-entrant (gemm.hpp:131-134:
// only a function-local configuration static).  The GPU launchers need three
// pieces of lazily initialised state, and all three live in a device's
// context, not in the process: the >48 KB dynamic shared-memory opt-in of
// each kernel (cudaFuncSetAttribute), the SM count, and the release
// threshold of the default stream-ordered memory pool.  They are cached here
// per (device, kernel) under a mutex, so one process may drive several GPUs
// from several host threads (one host thread per GPU).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <utility>

#include "launch.h"

namespace pbg {

namespace {
constexpr int kMaxDev = 64;
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, int> g_attr;  // (device, kernel) -> bytes opted in
std::atomic<int> g_sms[kMaxDev];
std::atomic<int> g_pool_done[kMaxDev];

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return dev;
}
}  // namespace

cudaError_t smem_attr(const void* fn, int bytes, bool max_carveout) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_attr_mu);
  auto key = std::make_pair(dev, fn);
  auto it = g_attr.find(key);
  if (it != g_attr.end() && it->second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  if (max_carveout) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
  }
  g_attr[key] = bytes;
  return cudaSuccess;
}

int num_sms() {
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDev) return 148;
  int v = g_sms[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
    cudaGetLastError();
    v = 148;
  }
  g_sms[dev].store(v, std::memory_order_relaxed);
  return v;
}

void mempool_keep() {
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDev || g_pool_done[dev].load(std::memory_order_acquire)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  g_pool_done[dev].store(1, std::memory_order_release);
}

}  // namespace pbg
