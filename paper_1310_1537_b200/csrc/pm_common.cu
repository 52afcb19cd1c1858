// Library-level entry points and error plumbing for libpmb200.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "pm_internal.cuh"
#include "pm_math.cuh"

namespace pm {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  std::string m = std::string("CUDA error in ") + what + ": " + cudaGetErrorName(e) + " (" +
                  cudaGetErrorString(e) + ")";
  g_last_error = m;
  return e == cudaErrorMemoryAllocation ? PM_ENOMEM : PM_EDEVICE;
}

int sm_count(int device) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lk(mu);
  if (device >= (int)cache.size()) cache.resize(device + 1, 0);
  if (cache[device] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) v = 0;
    cache[device] = v;
  }
  return cache[device];
}

// Stream-ordered allocations (cudaMallocAsync) come from the device's default pool; with
// the default release threshold of 0 the pool unmaps its memory at every synchronisation,
// so each call would pay a fresh physical mapping.  Keep up to 4 GiB cached per device.
void retain_pool(int device) {
  static std::mutex mu;
  static std::vector<char> done;
  std::lock_guard<std::mutex> lk(mu);
  if (device >= (int)done.size()) done.resize(device + 1, 0);
  if (done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = uint64_t(4) << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[device] = 1;
}

cudaError_t ensure_smem_attr(const void* kernel, std::atomic<uint64_t>& mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

}  // namespace pm

extern "C" {

int pm_abi_version(void) { return PM_ABI_VERSION; }

int pm_row_terms_host(const double* t, const double* y, int64_t n, double* nll_out, double* w_out) {
  if (!t || !y || !nll_out || !w_out) return pm::fail(PM_EINVAL, "null argument");
  for (int64_t i = 0; i < n; ++i) pm::pm_row_terms(t[i], y[i], nll_out[i], w_out[i]);
  return PM_OK;
}

const char* pm_last_error(void) { return pm::g_last_error.c_str(); }

int pm_device_count(int* n) {
  if (!n) return pm::fail(PM_EINVAL, "pm_device_count: null output");
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *n = 0;
    return pm::cuda_fail(e, "cudaGetDeviceCount");
  }
  *n = c;
  return PM_OK;
}

int pm_device_info(int device, int* sm, int* cc_major, int* cc_minor, size_t* total_mem) {
  cudaDeviceProp p;
  PM_CUDA(cudaGetDeviceProperties(&p, device));
  if (sm) *sm = p.multiProcessorCount;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  if (total_mem) *total_mem = p.totalGlobalMem;
  return PM_OK;
}

}  // extern "C"
