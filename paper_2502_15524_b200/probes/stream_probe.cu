// stream_probe.cu — test-only probe: how fast can 148 CTAs stream a weight matrix from HBM into
// shared memory with TMA in the decode stack's pattern (stream-K contiguous k-block ranges per
// CTA, a ring of SLOTS 16 KiB slots, no compute)?  Two layouts of the same bytes:
//   layout 0: row-major [M, K] bf16, box 64 cols x 128 rows (each box = 128 rows x 128 B
//             segments 2*K bytes apart: the image layout the library uses);
//   layout 1: tiled [M/128][K/64][128][64] bf16 (each box = one contiguous 16 KiB block).
// hs_debug_stream_probe (include/hs_probes.h) returns the achieved GB/s.
#include <vector>

#include "../../include/hs_probes.h"
#include "../csrc/gemm.h"
#include "../csrc/tc.h"

namespace hs {

template <int SLOTS>
__global__ void __launch_bounds__(64, 1) stream_probe_kernel(const __grid_constant__ CUtensorMap map, int64_t W, int nkb,
                                                             int tiled, int iters, int mma) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* btile = smem + SLOTS * 16384;  // [16][64] bf16 B operand (zeros), 2 KiB
  __shared__ uint64_t full[SLOTS], empty[SLOTS];
  __shared__ uint32_t tmem_slot;
  if (threadIdx.x == 0) {
    for (int s = 0; s < SLOTS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 512; i += 64) reinterpret_cast<uint32_t*>(btile)[i] = 0;
  if (threadIdx.x >= 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)), "r"(32u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  const int64_t beg = W * blockIdx.x / gridDim.x, end = W * (blockIdx.x + 1) / gridDim.x;
  const int64_t n = (end - beg) * iters;
  if (threadIdx.x == 0) {
    for (int64_t i = 0; i < n; ++i) {
      const int s = (int)(i % SLOTS);
      mbar_wait(&empty[s], (uint32_t)(((i / SLOTS) & 1) ^ 1));
      const int64_t x = beg + i % (end - beg);
      mbar_expect_tx(&full[s], 16384);
      if (tiled)
        tma_load_3d(&map, &full[s], smem + s * 16384, 0, 0, (int)x);
      else
        tma_load_2d(&map, &full[s], smem + s * 16384, (int)(x % nkb) * 64, (int)(x / nkb) * 128);
    }
  } else if (threadIdx.x == 32) {
    constexpr uint32_t idesc = instr_desc<16>();
    for (int64_t i = 0; i < n; ++i) {
      const int s = (int)(i % SLOTS);
      mbar_wait(&full[s], (uint32_t)((i / SLOTS) & 1));
      if (mma) {  // the decode stack's consumer: 4 x (M=128, N=16, K=16) MMAs, release by commit
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = umma_desc_sw128(smem + s * 16384), db = umma_desc_sw128(btile);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_bf16(tmem, da + 2 * kk, db + 2 * kk, idesc, (i > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&empty[s]);
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x >= 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32u));
}

}  // namespace hs

extern "C" hs_status hs_debug_stream_probe(int32_t layout, int64_t M, int64_t K, int32_t slots, int32_t iters,
                                           double* gbs) {
  using namespace hs;
  const int mma = layout >= 2;  // 2 / 3: layout 0 / 1 with the MMA consumer
  layout &= 1;
  if (M % 128 || K % 64 || !gbs || (slots != 8 && slots != 12) || iters < 1) HS_FAIL(HS_E_INVAL, "bad probe args");
  void* buf = nullptr;
  const size_t bytes = (size_t)M * K * 2;
  HS_CUDA(cudaMalloc(&buf, bytes));
  HS_CUDA(cudaMemset(buf, 0, bytes));
  const int64_t nkb = K / 64, W = (M / 128) * nkb;
  TmaMat t;
  if (layout == 0) {
    HS_TRY(make_tma(&t, buf, M, K, 128));
  } else {  // tiled: 3-D {64, 128, W} with contiguous 16 KiB blocks = make_tma3 with "layers" = blocks
    HS_TRY(make_tma3(&t, buf, W, 16384, 128, 64));
  }
  int sms = 0;
  HS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t smem = (size_t)slots * 16384 + 2048 + 1024;
  auto launch = [&]() -> hs_status {
    if (slots == 8) {
      HS_CUDA(cudaFuncSetAttribute(stream_probe_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      stream_probe_kernel<8><<<sms, 64, smem>>>(t.map, W, (int)nkb, layout, iters, mma);
    } else {
      HS_CUDA(cudaFuncSetAttribute(stream_probe_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      stream_probe_kernel<12><<<sms, 64, smem>>>(t.map, W, (int)nkb, layout, iters, mma);
    }
    HS_CUDA(cudaGetLastError());
    return HS_OK;
  };
  HS_TRY(launch());
  cudaEvent_t e0, e1;
  HS_CUDA(cudaEventCreate(&e0));
  HS_CUDA(cudaEventCreate(&e1));
  HS_CUDA(cudaEventRecord(e0));
  HS_TRY(launch());
  HS_CUDA(cudaEventRecord(e1));
  HS_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  HS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  *gbs = (double)bytes * iters / (ms / 1e3) / 1e9;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  return HS_OK;
}
