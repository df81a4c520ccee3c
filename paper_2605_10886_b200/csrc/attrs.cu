// attrs.cu — per-device, thread-safe kernel attribute setup (host only).
//
// cudaFuncSetAttribute (max dynamic shared memory, non-portable cluster size) is a per-device
// property of a function: a process that drives several GPUs must set it on each.  Every launcher
// calls ensure_func_attrs before its launch; the first call per (function, device) sets the
// attributes under a mutex, later calls are a lookup.
#include <map>
#include <mutex>
#include <utility>

#include "launch.h"

namespace loka {

cudaError_t ensure_func_attrs(const void* func, int smem_bytes, bool nonportable_cluster) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (function, device) -> smem bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  auto it = done.find({func, dev});
  if (it != done.end() && it->second >= smem_bytes) return cudaSuccess;
  if (nonportable_cluster) {
    e = cudaFuncSetAttribute(func, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  if (smem_bytes > 0) {
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return e;
  }
  done[{func, dev}] = smem_bytes;
  return cudaSuccess;
}

}  // namespace loka
