// common.h — shared helpers of the libhs implementation (host + device).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>
#include <utility>

#include "../../include/hs.h"

namespace hs {

void set_error(const std::string& msg);
const std::string& get_error();

struct Status {
  hs_status code = HS_OK;
};

#define HS_FAIL(code_, ...)                                   \
  do {                                                        \
    char buf_[512];                                           \
    snprintf(buf_, sizeof(buf_), __VA_ARGS__);                \
    ::hs::set_error(std::string(__func__) + ": " + buf_);     \
    return (code_);                                           \
  } while (0)

#define HS_CUDA(expr)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      HS_FAIL(e_ == cudaErrorMemoryAllocation ? HS_E_OOM : HS_E_CUDA, "%s -> %s (%s:%d)", \
              #expr, cudaGetErrorString(e_), __FILE__, __LINE__);                       \
    }                                                                                   \
  } while (0)

#define HS_TRY(expr)                   \
  do {                                 \
    hs_status s_ = (expr);             \
    if (s_ != HS_OK) return s_;        \
  } while (0)

using bf16 = __nv_bfloat16;

inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Number of SMs of the current device (cached per device).
int num_sms(int device);

// Kernels launched by this library since load (the bench's "gpu_launches" claim).
void count_launch(uint64_t n = 1);
uint64_t launch_total();

// Forces module loading of every kernel on the current device (no lazy-load cost at T0).
void warm_gemm_kernels();
void warm_kernels();

// Programmatic dependent launch: every kernel of the library is launched with
// programmaticStreamSerialization, calls griddepcontrol.launch_dependents at entry (so the
// next kernel's CTAs are scheduled while this one runs) and griddepcontrol.wait before its
// first access to memory written by earlier kernels (weights may be prefetched before).
// HS_PDL=0 in the environment disables it (A/B measurements).
#define PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#define PDL_LAUNCH() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")
bool pdl_enabled();

// Enqueues on st a device-side wait until the 8-byte watermark (mapped pinned memory) is >= value
// (cuStreamWaitValue64; prefetch.cc).  watermark == nullptr: no-op.
hs_status stream_wait_watermark(cudaStream_t st, const uint64_t* watermark, uint64_t value);

template <typename... KArgs, typename... Args>
inline cudaError_t launchk(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

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

}  // namespace hs
