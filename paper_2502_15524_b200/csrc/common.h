// common.h — shared helpers of the libhs implementation (host + device).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

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
