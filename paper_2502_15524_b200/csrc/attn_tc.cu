// attn_tc.cu — causal prefill attention on the 5th-generation tensor cores (a9, prefill half;
// the prefill computes the KV of every prompt token and attends over them).
//
// One CTA (4 warps, 128 threads) per (128-query tile, head, sequence).  Per 128-key chunk of
// the sequence's paged cache:
//   S = Q K^T          tcgen05.mma (M = 128 queries, N = 128 keys, K = head_dim) into TMEM;
//   thread t owns query row t (TMEM lane t) and reads its 128 scores with tcgen05.ld;
//   O += P V           tcgen05.mma (M = 128 queries, N = head_dim, K = 128 keys) into TMEM,
//                      P as two bf16 halves (hi + lo: fp32 probabilities to ~2^-16, the numerics
//                      contract's fp32 P, as the mma.sync kernel does).
// Two passes over the chunks: the first finds each row's exact max m and the sum
// l = Σ exp2(s - m) (rescaled when m grows), the second forms p = exp2(s - m) with the final m
// and accumulates P V in TMEM without any rescaling; o = O / l, one bf16 rounding.  Operands
// live in shared memory in the tcgen05 K-major 128B-swizzled layout: Q and K rows straight from
// the q buffer / the paged pool, V transposed on the way in (V^T [head_dim][keys]), P written
// row by row by its owner thread.  Deterministic; causal mask and ragged tails by position.
#include <cmath>
#include <cstdlib>

#include "kernels.h"
#include "tc.h"

namespace hs {

constexpr int TA_Q = 128;   // queries per CTA
constexpr int TA_KC = 128;  // keys per chunk

template <int D>
struct TaCfg {
  static constexpr int KB = D / 64;                    // 64-wide k-blocks of head_dim
  static constexpr int Q_BYTES = KB * TA_Q * 128;      // Q: KB tiles [128 q][64 d]
  static constexpr int K_BYTES = KB * TA_KC * 128;     // K: KB tiles [128 keys][64 d]
  static constexpr int V_BYTES = 2 * D * 128;          // V^T: 2 tiles [D d][64 keys]
  static constexpr int P_BYTES = 2 * TA_Q * 128;       // P half: 2 tiles [128 q][64 keys]
  static constexpr int SMEM = Q_BYTES + K_BYTES + V_BYTES + 2 * P_BYTES + 1024 + 64;
  static constexpr uint32_t TMEM_COLS = 256;           // S: 128 columns, O: D columns (at 128)
};

// 16-byte chunk c (0..7) of row r of a [rows][64] bf16 tile in the 128B-swizzled layout
__device__ __forceinline__ uint32_t sw128(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

template <int D>
__global__ void __launch_bounds__(128, 1) attn_prefill_tc_kernel(
    const bf16* __restrict__ q, const bf16* __restrict__ pool, const SeqDesc* __restrict__ seqs,
    const int* __restrict__ tables, int max_blocks, bf16* __restrict__ o, int nh, int nblocks) {
  using C = TaCfg<D>;
  PDL_LAUNCH();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + C::Q_BYTES;
  uint8_t* sV = sK + C::K_BYTES;
  uint8_t* sP = sV + C::V_BYTES;  // [hi | lo]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + 2 * C::P_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int t = threadIdx.x, warp = t >> 5;
  const SeqDesc s = seqs[blockIdx.z];
  const int head = blockIdx.y;
  const int q0 = (gridDim.x - 1 - blockIdx.x) * TA_Q;  // longest (causal) query tiles first
  if (q0 >= s.n_q) return;
  const int H = nh * D;
  if (t == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  PDL_WAIT();
  // Q rows: thread t loads query q0 + t (rows past n_q repeat the last row: never stored)
  const int qi = min(q0 + t, s.n_q - 1);
  const int pos = s.pos0 + q0 + t;  // this row's position (causal bound)
  {
    const uint4* src = reinterpret_cast<const uint4*>(q + (size_t)(s.q_start + qi) * H + head * D);
#pragma unroll
    for (int c = 0; c < D / 8; ++c)
      *reinterpret_cast<uint4*>(sQ + (c >> 3) * (TA_Q * 128) + sw128(t, c & 7)) = __ldg(src + c);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 128;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  const int* tab = tables + (size_t)s.table * max_blocks;
  const int n_keys = s.pos0 + min(q0 + TA_Q, s.n_q);  // keys any row of the tile sees
  const int n_chunks = (n_keys + TA_KC - 1) / TA_KC;
  const float sl2 = 1.4426950408889634f / sqrtf((float)D);
  constexpr uint32_t idS = instr_desc<TA_KC>();  // M = 128, N = 128 keys
  constexpr uint32_t idO = instr_desc<D>();      // M = 128, N = head_dim
  uint32_t phase = 0;

  // K rows (and V^T columns) of chunk kc: thread t takes key kc + t (zeros past the keys)
  auto load_chunk = [&](int kc, bool with_v) {
    const int j = kc + t;
    const uint4* kp = nullptr;
    if (j < n_keys) {
      int b = tab[j >> 4];
      if (b < 0 || b >= nblocks) b = 0;
      kp = reinterpret_cast<const uint4*>(pool + ((((size_t)b * 2) * nh + head) * 16 + (j & 15)) * D);
    }
#pragma unroll
    for (int c = 0; c < D / 8; ++c) {
      const uint4 kv = kp ? __ldcg(kp + c) : make_uint4(0, 0, 0, 0);
      *reinterpret_cast<uint4*>(sK + (c >> 3) * (TA_KC * 128) + sw128(t, c & 7)) = kv;
    }
    if (with_v) {  // V^T: element (d, key t) of k-block t / 64, row d, chunk (t % 64) / 8
      const uint4* vp = kp ? kp + (size_t)nh * 16 * D / 8 : nullptr;
      const int kb = t >> 6, kl = t & 63;
      uint8_t* vt = sV + kb * (D * 128);
#pragma unroll 4
      for (int c = 0; c < D / 8; ++c) {
        const uint4 vv = vp ? __ldcg(vp + c) : make_uint4(0, 0, 0, 0);
        const bf16* e = reinterpret_cast<const bf16*>(&vv);
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const int d = c * 8 + x;
          *reinterpret_cast<bf16*>(vt + sw128(d, kl >> 3) + (kl & 7) * 2) = e[x];
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
  };
  auto mma_S = [&]() {  // S = Q K^T over head_dim
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int kb = 0; kb < C::KB; ++kb) {
        const uint64_t da = umma_desc_sw128(sQ + kb * (TA_Q * 128)), db = umma_desc_sw128(sK + kb * (TA_KC * 128));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_bf16(tS, da + 2 * kk, db + 2 * kk, idS, (kb | kk) ? 1u : 0u);
      }
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  };

  // ---- pass 1: row max m and l = sum exp2(s - m)
  float m = -INFINITY, l = 0.f;
  for (int ci = 0; ci < n_chunks; ++ci) {
    const int kc = ci * TA_KC;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");  // S reads before the next MMA
    __syncthreads();  // the previous chunk's MMA has read sK
    load_chunk(kc, false);
    __syncthreads();
    mma_S();
#pragma unroll 1
    for (int c0 = 0; c0 < TA_KC; c0 += 32) {
      float v[32];
      tmem_ld32(tS + lane_base + c0, v);
      float mx = m;
#pragma unroll
      for (int x = 0; x < 32; ++x) {
        const int kp = kc + c0 + x;
        v[x] = (kp <= pos && kp < n_keys) ? v[x] * sl2 : -INFINITY;
        mx = fmaxf(mx, v[x]);
      }
      if (mx != -INFINITY) {
        l *= exp2f(m - mx);  // m = -inf: l = 0 stays 0
        m = mx;
#pragma unroll
        for (int x = 0; x < 32; ++x) l += exp2f(v[x] - m);
      }
    }
  }
  // ---- pass 2: p = exp2(s - m) (final m), O += P V (no rescaling)
  for (int ci = 0; ci < n_chunks; ++ci) {
    const int kc = ci * TA_KC;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // the previous chunk's MMAs have read sK / sV / sP
    load_chunk(kc, true);
    __syncthreads();
    mma_S();
#pragma unroll 1
    for (int c0 = 0; c0 < TA_KC; c0 += 32) {
      float v[32];
      tmem_ld32(tS + lane_base + c0, v);
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int x = 0; x < 32; x += 2) {
        const int kp = kc + c0 + x;
        const float p0 = (kp <= pos && kp < n_keys) ? exp2f(v[x] * sl2 - m) : 0.f;
        const float p1 = (kp + 1 <= pos && kp + 1 < n_keys) ? exp2f(v[x + 1] * sl2 - m) : 0.f;
        const __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
        const float2 hf = __bfloat1622float2(h);
        const __nv_bfloat162 lw = __floats2bfloat162_rn(p0 - hf.x, p1 - hf.y);
        hi[x >> 1] = *reinterpret_cast<const uint32_t*>(&h);
        lo[x >> 1] = *reinterpret_cast<const uint32_t*>(&lw);
      }
      // row t, keys c0 .. c0 + 31 = k-block c0 / 64, 16-byte chunks (c0 % 64) / 8 .. + 3
      const int kb = c0 >> 6, cb = (c0 & 63) >> 3;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const uint32_t off = kb * (TA_Q * 128) + sw128(t, cb + g);
        *reinterpret_cast<uint4*>(sP + off) = make_uint4(hi[4 * g], hi[4 * g + 1], hi[4 * g + 2], hi[4 * g + 3]);
        *reinterpret_cast<uint4*>(sP + C::P_BYTES + off) = make_uint4(lo[4 * g], lo[4 * g + 1], lo[4 * g + 2], lo[4 * g + 3]);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int half = 0; half < 2; ++half)
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {
          const uint64_t da = umma_desc_sw128(sP + half * C::P_BYTES + kb * (TA_Q * 128));
          const uint64_t db = umma_desc_sw128(sV + kb * (D * 128));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(tO, da + 2 * kk, db + 2 * kk, idO, (ci | half | kb | kk) ? 1u : 0u);
        }
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  // ---- o = O / l (one bf16 rounding); rows past n_q are not stored
  const float il = 1.f / l;
  bf16* orow = o + (size_t)(s.q_start + qi) * H + head * D;
  const bool store = q0 + t < s.n_q;
#pragma unroll 1
  for (int c0 = 0; c0 < D; c0 += 32) {
    float v[32];
    tmem_ld32(tO + lane_base + c0, v);
    if (store) {
      uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        uint4 w;
        uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const __nv_bfloat162 b = __floats2bfloat162_rn(v[8 * g + 2 * x] * il, v[8 * g + 2 * x + 1] * il);
          wp[x] = *reinterpret_cast<const uint32_t*>(&b);
        }
        dst[g] = w;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
}

// Off by default (HS_ATTN_TC=1 enables it): parity-green, but this synchronous two-pass design
// measured 78 / 374 us per 7B layer at 512 / 2048 tokens against the mma.sync kernel's 41 / 183
// (profiles/r02/attn_tc_ab.txt): every chunk serialises load -> MMA -> TMEM read -> softmax ->
// MMA, K is loaded twice and V is transposed through scalar shared-memory stores.
bool attn_tc_enabled() {
  static const bool on = [] {
    const char* e = getenv("HS_ATTN_TC");
    return e && e[0] == '1';
  }();
  return on;
}

void launch_attn_prefill_tc(const bf16* q, const bf16* pool, const SeqDesc* seqs, int n_seqs, int max_nq,
                            const int* tables, int max_blocks, bf16* o, int nh, int d, int nblocks, cudaStream_t st) {
  count_launch();
  dim3 grid((max_nq + TA_Q - 1) / TA_Q, nh, n_seqs);
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr[dev]) {
    cudaFuncSetAttribute(attn_prefill_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, TaCfg<128>::SMEM);
    cudaFuncSetAttribute(attn_prefill_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, TaCfg<64>::SMEM);
    attr[dev] = true;
  }
  if (d == 128)
    launchk(attn_prefill_tc_kernel<128>, grid, 128, TaCfg<128>::SMEM, st, q, pool, seqs, tables, max_blocks, o, nh, nblocks);
  else
    launchk(attn_prefill_tc_kernel<64>, grid, 128, TaCfg<64>::SMEM, st, q, pool, seqs, tables, max_blocks, o, nh, nblocks);
}

void warm_attn_tc() {
  cudaFuncAttributes a;
  cudaFuncSetAttribute(attn_prefill_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, TaCfg<128>::SMEM);
  cudaFuncSetAttribute(attn_prefill_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, TaCfg<64>::SMEM);
  cudaFuncGetAttributes(&a, attn_prefill_tc_kernel<128>);
  cudaFuncGetAttributes(&a, attn_prefill_tc_kernel<64>);
}

}  // namespace hs
