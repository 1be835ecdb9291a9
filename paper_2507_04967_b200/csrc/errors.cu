#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "capi_util.hpp"
#include "launch.hpp"

namespace iolmh {
namespace {
thread_local std::string g_last_error;

struct FuncAttr {
  size_t smem = 0;
  int carveout = -1;
};
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, FuncAttr> g_attr;  // (device, kernel) -> configured
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

void ensure_func_smem(const void* func, size_t bytes, int carveout) {
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_attr_mu);
  FuncAttr& a = g_attr[{dev, func}];
  if (bytes > a.smem) {
    CUDA_OK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    a.smem = bytes;
  }
  if (carveout >= 0 && carveout != a.carveout) {
    CUDA_OK(cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, carveout));
    a.carveout = carveout;
  }
}

int device_sms() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  CUDA_OK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  cache[dev] = n;
  return n;
}
}  // namespace iolmh

extern "C" const char* iolm_cuda_last_error(void) { return iolmh::g_last_error.c_str(); }
