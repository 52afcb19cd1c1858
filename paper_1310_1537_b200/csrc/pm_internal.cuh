// Internal helpers shared by the libpmb200 translation units (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>
#include <utility>

#include "../../include/pmb200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libpmb200 is written for sm_100a (B200) only"
#endif

namespace pm {

// ---------------------------------------------------------------- error plumbing
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define PM_CUDA(call)                                   \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return ::pm::cuda_fail(_e, #call); \
  } while (0)

// RAII device switch: handles own one device; every call selects it first.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int sm_count(int device);

// Kernel-dispatch overrides (A/B experiments and the layout tests): set only through the
// C ABI (pm_tune_set), never read from the environment, so the shipped library's dispatch
// is fixed unless a caller explicitly asks otherwise.  Returns `dflt` when `name` is unset.
int tune(const char* name, int dflt);

// Evict every line of the 126 MB L2 on `st` (timing of cold-cache launches): a 512 MiB
// memset, then a 256 MiB read of a second, clean buffer, so the next launch neither hits in
// L2 nor pays the write-back of dirty scrub lines.  Buffers are allocated once per device.
cudaError_t l2_scrub(int device, cudaStream_t st);
void retain_pool(int device);

}  // namespace pm

// Workspace internals shared between glm.cu (owner) and chain.cu (hidden symbols).
struct pm_ws_view {
  double* xbeta;
  const double* xt;   // [K][ld]
  const double* y;
  int64_t n, ld;
  int K;
  int device;
  int sms;
  void* stream;
};
extern "C" int pm_ws_internal_view(pm_ws_t ws, pm_ws_view* v);
extern "C" int pm_ws_internal_lock(pm_ws_t ws, int lock);

namespace pm {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device); `mask` is a
// per-kernel static bitmask of devices already configured.
cudaError_t ensure_smem_attr(const void* kernel, std::atomic<uint64_t>& mask);

// <<<grid, block, smem, stream>>> with the PDL attribute when `pdl` (see pdl_wait).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- device PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// Release a consumed shared-memory stage only after the warp's loads from it have LANDED.
// Shared loads complete asynchronously: the warp waits on a load's scoreboard only when an
// instruction reads its destination register, and neither __syncwarp nor the arrive reads
// them -- so an arrive issued right after the loads can hand the stage to the producer (whose
// next TMA copy overwrites it) while the loads are still in flight.  `dep` must be computed
// from every loaded value; storing it into the stage being released (its own first 128
// bytes: the warp is done reading them, and the producer overwrites the stage next) makes
// the warp wait for all of them, and the store cannot move past the arrive (memory clobber).
// (Measured: y values read from an overwritten stage, K=32 row-per-lane HB kernel, before
// this guard.)  No extra shared memory: the stream kernels size their ring to the limit.
// The producer refills the stage through the ASYNC proxy (TMA), so the generic-proxy
// accesses above are ordered before it with fence.proxy.async by every lane (without it a
// TMA write can land before this warp's earlier generic accesses to the stage take effect).
__device__ __forceinline__ void mbar_arrive_after(uint64_t* bar, double dep, int lane, void* stage) {
  reinterpret_cast<volatile uint32_t*>(stage)[lane] = __double2loint(dep);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  // bar == nullptr: the caller refills the stage itself (self-producing consumers) and only
  // needs the quiesce above
  if (lane == 0 && bar)
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// try_wait with a suspend-time hint: the thread sleeps in hardware until the phase
// completes (or ~the hint elapses) instead of re-polling (each poll costs issue slots).
#ifndef PM_MBAR_HINT_NS
#define PM_MBAR_HINT_NS 1000000
#endif
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(uint32_t(PM_MBAR_HINT_NS))
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// 1-D bulk async copy global -> shared (TMA engine, SASS UBLKCP), completion
// signalled as transaction bytes on `bar`.  dst/src 16-byte aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Same with an L2 eviction-priority hint (evict_first for read-once streams).
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Programmatic dependent launch (PDL): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while the previous kernel in
// its stream drains; pdl_wait() blocks until that kernel has completed and its writes are
// visible (everything before it may only touch data no earlier kernel writes), pdl_trigger()
// lets the next such kernel be scheduled as this one's CTAs exit.  No-ops without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ double shfl_d(double v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}
__device__ __forceinline__ double shfl_xor_d(double v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

// This lane's share of a cross-CTA fold: sum of p[b * stride] for b = lane, lane + 32, ... < n,
// ascending (fixed order), with the loads of up to 8 strides issued together before the adds
// (a plain strided loop waits one L2 round trip per 32 partials: ~0.3 us each on the critical
// path of every launch).  Callers finish with warp_sum.
__device__ __forceinline__ double fold_lane(const double* p, size_t stride, int n, int lane) {
  double acc = 0.0;
  for (int b0 = 0; b0 < n; b0 += 256) {
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int b = b0 + 32 * i + lane;
      v[i] = b < n ? __ldcg(p + size_t(b) * stride) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (b0 + 32 * i + lane < n) acc += v[i];
  }
  return acc;
}

// Fixed-order butterfly sum across a warp (every lane gets the same bits).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += shfl_xor_d(v, m);
  return v;
}

}  // namespace pm
