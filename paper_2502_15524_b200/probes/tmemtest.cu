// tmemtest.cu — test-only probe of the A-operand-in-TMEM path of tcgen05 (one CTA, one tile):
// the weight tile lands in shared memory by TMA (128B swizzle, as everywhere else), is copied
// to TMEM with tcgen05.cp.128x256b and multiplied with tcgen05.mma [d], [a_tmem], b_desc.  The
// same tile multiplied from shared memory (the production path) is the reference.  Exposed as
// hs_debug_tmem_a_gemm (include/hs_probes.h).  Built into libhs_probe.so, never into the product
// library libhs.so (it links against libhs.so for the TMA-descriptor helper).
#include "../../include/hs_probes.h"
#include "../csrc/gemm.h"
#include "../csrc/tc.h"

namespace hs {

__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc));
}

__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                             uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(accum));
}

// grid 1, 128 threads; nkb k-blocks; out_ss / out_ts: [16][128] fp32 (token-major)
__global__ void __launch_bounds__(128, 1)
    tmem_a_probe_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int nkb,
                        float* out_ss, float* out_ts) {
  __shared__ __align__(1024) uint8_t sa[16384];
  __shared__ __align__(1024) uint8_t sb[2048];
  __shared__ uint64_t bar_full, bar_mma;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar_full, 1);
    mbar_init(&bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(128u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;  // cols [0,16): D (SS), [16,32): D (TS), [32,64): A
  constexpr uint32_t idesc = instr_desc<16>();
  for (int kb = 0; kb < nkb; ++kb) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(&bar_full, 16384 + 2048);
      tma_load_2d(&tmA, &bar_full, sa, kb * 64, 0);
      tma_load_2d(&tmB, &bar_full, sb, kb * 64, 0);
    }
    mbar_wait(&bar_full, kb & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
      const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sb);
#pragma unroll
      for (int k = 0; k < 4; ++k) umma_bf16(tmem + 0, da + 2 * k, db + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
#pragma unroll
      for (int k = 0; k < 4; ++k) tmem_cp_128x256b(tmem + 32 + 8 * k, da + 2 * k);
#pragma unroll
      for (int k = 0; k < 4; ++k) umma_bf16_ts(tmem + 16, tmem + 32 + 8 * k, db + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
      umma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, kb & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    __syncthreads();
  }
  float v[16];
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  tmem_ld16(taddr + 0, v);
  for (int j = 0; j < 16; ++j) out_ss[j * 128 + warp * 32 + lane] = v[j];
  tmem_ld16(taddr + 16, v);
  for (int j = 0; j < 16; ++j) out_ts[j * 128 + warp * 32 + lane] = v[j];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u));
}

}  // namespace hs

extern "C" hs_status hs_debug_tmem_a_gemm(const void* A, const void* B, int32_t K, float* out_ss, float* out_ts) {
  using namespace hs;
  if (K <= 0 || K % 64) HS_FAIL(HS_E_INVAL, "K must be a positive multiple of 64");
  TmaMat ta, tb;
  HS_TRY(make_tma(&ta, A, 128, K, 128));
  HS_TRY(make_tma(&tb, B, 16, K, 16));
  tmem_a_probe_kernel<<<1, 128>>>(ta.map, tb.map, K / 64, out_ss, out_ts);
  HS_CUDA(cudaGetLastError());
  HS_CUDA(cudaDeviceSynchronize());
  return HS_OK;
}
