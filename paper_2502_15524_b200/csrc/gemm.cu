// gemm.cu — tcgen05 + TMA GEMM (sm_100a) with fused epilogues and deterministic split-K.
//
// Kernel anatomy (one output tile of 128 features x BN tokens per CTA, 128 threads):
//   warp 0 / lane 0 : TMA producer.  Per 64-wide K block it loads the weight tile
//                     [128 x 64] and the activation tile [BN x 64] (128B swizzle) into a
//                     ring of STAGES shared-memory slots, arming the slot's "full" mbarrier
//                     with the expected transaction bytes.
//   warp 1 / lane 0 : MMA issuer.  Waits "full", issues 4 x tcgen05.mma (M=128, N=BN, K=16)
//                     accumulating into TMEM, and tcgen05.commit's the slot's "empty"
//                     mbarrier so the producer can refill it; after the last K block it
//                     commits the "accumulator ready" barrier.
//   warp 2          : allocates / frees the TMEM columns.
//   all 4 warps     : epilogue.  Warp w owns TMEM lanes [32w, 32w+32) = 32 output features;
//                     tcgen05.ld 32 columns (tokens) at a time, apply the epilogue and store
//                     out[token][feature] (or fp32 split-K partials).
// The smem operand layout is the canonical K-major SWIZZLE_128B layout that TMA writes:
// 8-row x 128-byte atoms, atoms 1024 B apart (SBO = 1024), K advanced inside the atom by
// moving the descriptor start address by 32 B per UMMA_K = 16 elements.
#include "gemm.h"
#include "tc.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

namespace hs {

// R10b: the accumulator of token n scaled by the RMSNorm row scale before a bf16 / SiLU
// epilogue (rs == null: unchanged, x * 1.0f is exact)
template <int CH>
__device__ __forceinline__ void scale_rows(float* v, const float* rs, int n0, int ncol) {
  if (!rs) return;
#pragma unroll
  for (int j = 0; j < CH; ++j)
    if (j < ncol) v[j] *= __ldg(rs + n0 + j);
}

struct KParams {
  int M, N, K;
  int kb_per_split;  // K blocks (of 64) per split
  int nkb;           // total K blocks
  int epi;           // GemmEpi, or -1 = fp32 partial into workspace
  void* out;
  int ldo;
  const bf16* resid;
  int ldr;
  float* ws;
  const float* rs;
};

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = 128 * 64 * 2;
  static constexpr int B_BYTES = BN * 64 * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN >= 256 ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN>
__global__ void __launch_bounds__(128, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                KParams p) {
  using C = Cfg<BN>;
  PDL_LAUNCH();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* accf = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * BN;
  const int kb0 = blockIdx.z * p.kb_per_split;
  const int nk = min(p.kb_per_split, p.nkb - kb0);

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"((uint32_t)C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer: weights of the first stages before the grid dependency resolves
    const int pre = min(nk, C::STAGES);
    for (int i = 0; i < pre; ++i) {
      mbar_expect_tx(&full[i], C::STAGE_BYTES);
      tma_load_w(&tmA, &full[i], smem + i * C::STAGE_BYTES, (m0 / 128) * p.nkb + kb0 + i);
    }
    PDL_WAIT();
    for (int i = 0; i < pre; ++i)
      tma_load_2d(&tmB, &full[i], smem + i * C::STAGE_BYTES + C::A_BYTES, (kb0 + i) * 64, n0);
    for (int i = pre; i < nk; ++i) {
      const int s = i % C::STAGES;
      const uint32_t ph = (i / C::STAGES) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      uint8_t* sa = smem + s * C::STAGE_BYTES;
      uint8_t* sb = sa + C::A_BYTES;
      mbar_expect_tx(&full[s], C::STAGE_BYTES);
      const int kc = (kb0 + i) * 64;
      tma_load_w(&tmA, &full[s], sa, (m0 / 128) * p.nkb + kb0 + i);
      tma_load_2d(&tmB, &full[s], sb, kc, n0);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer
    constexpr uint32_t idesc = instr_desc<BN>();
    for (int i = 0; i < nk; ++i) {
      const int s = i % C::STAGES;
      const uint32_t ph = (i / C::STAGES) & 1;
      mbar_wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint8_t* sa = smem + s * C::STAGE_BYTES;
      const uint8_t* sb = sa + C::A_BYTES;
      const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sb);
#pragma unroll
      for (int k = 0; k < 4; ++k)  // 64 / UMMA_K(16); +32 B => +2 in the >>4 address field
        umma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (i | k) != 0);
      umma_commit(&empty[s]);
    }
    umma_commit(accf);
  }
  __syncwarp();
  PDL_WAIT();

  // ---- epilogue: all 4 warps
  mbar_wait(accf, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int m = m0 + warp * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  constexpr int CH = BN < 32 ? 16 : 32;
  for (int c0 = 0; c0 < BN; c0 += CH) {
    float v[32];
    if constexpr (CH == 32) tmem_ld32(trow + c0, v);
    else tmem_ld16(trow + c0, v);
    if (n0 + c0 >= p.N) break;  // warp-uniform
    const int ncol = min(CH, p.N - n0 - c0);
    if (p.epi == EPI_BF16 || p.epi == EPI_SILU_MUL) scale_rows<CH>(v, p.rs, n0 + c0, ncol);
    if (p.epi < 0) {
      float* ws = p.ws + ((size_t)blockIdx.z * p.N + n0 + c0) * p.M;
      if (m < p.M)
#pragma unroll
        for (int j = 0; j < CH; ++j)
          if (j < ncol) ws[(size_t)j * p.M + m] = v[j];
    } else if (p.epi == EPI_F32) {
      float* o = reinterpret_cast<float*>(p.out) + (size_t)(n0 + c0) * p.ldo;
      if (m < p.M)
#pragma unroll
        for (int j = 0; j < CH; ++j)
          if (j < ncol) o[(size_t)j * p.ldo + m] = v[j];
    } else if (p.epi == EPI_BF16) {
      bf16* o = reinterpret_cast<bf16*>(p.out) + (size_t)(n0 + c0) * p.ldo;
      if (m < p.M)
#pragma unroll
        for (int j = 0; j < CH; ++j)
          if (j < ncol) o[(size_t)j * p.ldo + m] = __float2bfloat16_rn(v[j]);
    } else if (p.epi == EPI_RESID) {
      bf16* o = reinterpret_cast<bf16*>(p.out) + (size_t)(n0 + c0) * p.ldo;
      const bf16* r = p.resid + (size_t)(n0 + c0) * p.ldr;
      if (m < p.M) {
        float rv[CH];  // loads first: out may alias resid for the compiler
#pragma unroll
        for (int j = 0; j < CH; ++j) rv[j] = j < ncol ? __bfloat162float(__ldg(r + (size_t)j * p.ldr + m)) : 0.f;
#pragma unroll
        for (int j = 0; j < CH; ++j)
          if (j < ncol) o[(size_t)j * p.ldo + m] = __float2bfloat16_rn(v[j] + rv[j]);
      }
    } else {  // EPI_SILU_MUL: lanes 0-15 gate rows, 16-31 the matching up rows
      bf16* o = reinterpret_cast<bf16*>(p.out) + (size_t)(n0 + c0) * p.ldo;
      const int f = (m0 + warp * 32) / 2 + lane;
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        float u = __shfl_xor_sync(0xffffffffu, v[j], 16);
        if (lane < 16 && j < ncol && m < p.M) o[(size_t)j * p.ldo + f] = __float2bfloat16_rn(silu_f(v[j]) * u);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"((uint32_t)C::TMEM_COLS));
  }
}

// Deterministic split-K reduction: sums the partials in split order, then the epilogue.
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int M, int N,
                                     int epi, void* out, int ldo, const bf16* __restrict__ resid,
                                     int ldr, const float* __restrict__ rs) {
  PDL_LAUNCH();
  PDL_WAIT();
  const int n = blockIdx.y;
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  float acc = 0.f;
  for (int s = 0; s < splits; ++s) acc += ws[((size_t)s * N + n) * M + m];
  const float rsn = (rs && (epi == EPI_BF16 || epi == EPI_SILU_MUL)) ? rs[n] : 1.0f;
  acc *= rsn;
  if (epi == EPI_F32) {
    reinterpret_cast<float*>(out)[(size_t)n * ldo + m] = acc;
  } else if (epi == EPI_BF16) {
    reinterpret_cast<bf16*>(out)[(size_t)n * ldo + m] = __float2bfloat16_rn(acc);
  } else if (epi == EPI_RESID) {
    reinterpret_cast<bf16*>(out)[(size_t)n * ldo + m] =
        __float2bfloat16_rn(acc + __bfloat162float(resid[(size_t)n * ldr + m]));
  } else {  // silu-mul: m indexes physical rows; gate rows are j < 16 in each 32-row block
    const int j = m & 31;
    if (j < 16) {
      float u = 0.f;
      for (int s = 0; s < splits; ++s) u += ws[((size_t)s * N + n) * M + m + 16];
      u *= rsn;
      reinterpret_cast<bf16*>(out)[(size_t)n * ldo + (m >> 5) * 16 + j] =
          __float2bfloat16_rn(silu_f(acc) * u);
    }
  }
}

// ------------------------------------------------------------------ stream-K (decode) -----
// Persistent weight-streaming GEMM for small N (decode, N <= 64 tokens): the flattened space
// of (tile, 64-wide K block) work is cut into G equal contiguous ranges, one per CTA
// (G = #SMs), so every SM streams the same number of weight bytes whatever M and K are (no
// wave quantisation, no idle SMs).  A CTA's range covers parts of one or more 128-row tiles;
// each part's fp32 accumulator goes to a workspace slot; the CTA that completes a tile last
// (per-tile arrival counter) sums the tile's parts in part order (deterministic) and applies
// the epilogue, fused with the row-wide ops of decode:
//   - FUSE_ROPE (QKV): bf16 rounding, RoPE of q and k, paged KV write;
//   - FUSE_NORM (O-proj, down-proj): residual add, then the CTA that completes the last tile
//     computes the RMSNorm of the whole row (grid-level arrival counter).
// Counters are reset by their last arriver, so they are zero again for the next launch.
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer, warps 2-5 epilogue
// (warp w drains TMEM lanes 32*(w%4)..); two TMEM accumulators so the MMA of part i+1
// overlaps the drain of part i.
struct SkParams {
  int M, N, nkb, tiles, G, maxp;
  float* ws;
  unsigned* ctr;  // [tiles + 1]
  int epi;
  void* out;
  int ldo;
  const bf16* resid;
  int ldr;
  int fuse;
  const bf16* norm_w;
  bf16* norm_out;
  float* rs_out;
  const float* rs;
  float eps;
  const int* pos;
  const int* slot;
  const float2* tab;
  bf16* q_out;
  bf16* pool;
  int nh, hd;  // heads, head_dim
  int nslots;
  unsigned long long* trace;  // optional per-CTA phase timestamps (globaltimer ns), 8 per CTA
};

// RMSNorm of one row with 128 threads (tid in [0,128)); fixed summation order.  Not inlined,
// so the GEMM epilogue and the standalone decode row-norm run the very same code (PP = s
// stays bitwise equal to PP = 1 across the stage boundary).
__device__ __noinline__ void row_norm128(const bf16* __restrict__ h, int M, const bf16* __restrict__ w,
                                         bf16* __restrict__ y, float* rs_out, float eps, int tid, float* red,
                                         int bar_id) {
  // 16-byte loads (8 values), all issued before use; fixed per-thread summation order
  const int n8 = M >> 3;
  const uint4* h4 = reinterpret_cast<const uint4*>(h);
  constexpr int U = 8;  // up to 8 x 1024 values per thread-iteration batch
  float ss = 0.f;
  for (int c0 = 0; c0 < n8; c0 += U * 128) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * 128 + tid;
      v[u] = c < n8 ? __ldcg(h4 + c) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(p2[k]);
        ss = fmaf(f.x, f.x, ss);
        ss = fmaf(f.y, f.y, ss);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  named_bar(bar_id, 128);
  const float tot = (red[0] + red[1]) + (red[2] + red[3]);
  const float rs_row = 1.0f / sqrtf(tot / (float)M + eps);
  if (rs_out && tid == 0) *rs_out = rs_row;
  const float rs = rs_out ? 1.0f : rs_row;  // R10b: the operand is bf16(x * w), rs scales the product
  const uint4* w4 = reinterpret_cast<const uint4*>(w);
  uint4* y4 = reinterpret_cast<uint4*>(y);
  for (int c = tid; c < n8; c += 128) {
    const uint4 hv = __ldcg(h4 + c), wv = w4[c];
    uint4 o;
    const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(&hv);
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&wv);
    __nv_bfloat162* r = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 x = __bfloat1622float2(a[k]), g = __bfloat1622float2(b[k]);
      r[k] = __floats2bfloat162_rn(x.x * rs * g.x, x.y * rs * g.y);
    }
    y4[c] = o;
  }
  named_bar(bar_id, 128);
}

template <int BN>
struct SkCfg {
  static constexpr int A_BYTES = 128 * 64 * 2;
  static constexpr int B_BYTES = BN * 64 * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // BN <= 32: 5 stages (~100 KB) so two CTAs fit an SM: the next kernel's CTA (PDL) becomes
  // resident and prefetches its weights while this one drains.  BN = 128 (small-tile-count
  // prefill chunks) uses 4 stages and no RoPE staging buffer.
  static constexpr int STAGES = BN >= 128 ? 4 : (BN >= 64 ? 6 : 5);
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int VALS_BYTES = BN <= 64 ? 128 * BN * 4 : 0;  // tile values for the RoPE pairing
  static constexpr int SMEM = STAGES * STAGE_BYTES + VALS_BYTES + 1024 + 512;
};

template <int BN>
__global__ void __launch_bounds__(192, 1)
    gemm_sk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, SkParams p) {
  using C = SkCfg<BN>;
  PDL_LAUNCH();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* vals = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + C::VALS_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  volatile int* flag = reinterpret_cast<volatile int*>(tmem_slot + 1);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long W = (long long)p.tiles * p.nkb;
  const int beg = sk_begin(blockIdx.x, W, p.G), end = sk_begin(blockIdx.x + 1, W, p.G);
  unsigned long long* tr = p.trace ? p.trace + blockIdx.x * 8 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtimer();
  const int pre = min(end - beg, C::STAGES);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the producer (this thread) requests the first weight tiles before anything else:
    // they do not depend on the previous kernel (PDL) nor on TMEM
    for (int i = 0; i < pre; ++i) {
      const int x = beg + i;
      mbar_expect_tx(&full[i], C::STAGE_BYTES);
      tma_load_w(&tmA, &full[i], smem + i * C::STAGE_BYTES, x);
    }
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer over the CTA's k-block range [beg, end)
      // (the first `pre` weight tiles were requested during setup, before the dependency)
      if (tr) tr[1] = gtimer();
      PDL_WAIT();
      if (tr) tr[2] = gtimer();
      for (int i = 0; i < pre; ++i)
        tma_load_2d(&tmB, &full[i], smem + i * C::STAGE_BYTES + C::A_BYTES, ((beg + i) % p.nkb) * 64, 0);
      for (int i = pre; beg + i < end; ++i) {
        const int x = beg + i;
        const int s = i % C::STAGES;
        mbar_wait(&empty[s], ((i / C::STAGES) & 1) ^ 1);
        uint8_t* sa = smem + s * C::STAGE_BYTES;
        mbar_expect_tx(&full[s], C::STAGE_BYTES);
        tma_load_w(&tmA, &full[s], sa, x);
        tma_load_2d(&tmB, &full[s], sa + C::A_BYTES, (x % p.nkb) * 64, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc = instr_desc<BN>();
      int i = 0, seg = 0;
      for (int cur = beg; cur < end; ++seg) {
        const int kb_lo = cur % p.nkb, kb_hi = min(p.nkb, kb_lo + (end - cur));
        const int buf = seg & 1;
        mbar_wait(&tempty[buf], ((seg >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + buf * BN;
        for (int kb = kb_lo; kb < kb_hi; ++kb, ++i) {
          const int s = i % C::STAGES;
          mbar_wait(&full[s], (i / C::STAGES) & 1);
          if (tr && i == 0) tr[3] = gtimer();
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t* sa = smem + s * C::STAGE_BYTES;
          const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + C::A_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) umma_bf16(acc, da + 2 * k, db + 2 * k, idesc, (kb > kb_lo || k > 0) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[buf]);
        cur += kb_hi - kb_lo;
      }
      if (tr) tr[4] = gtimer();
    }
  } else {
    // ---- epilogue warps 2..5 (et = 0..127 owns tile row ml = et)
    PDL_WAIT();
    const int quad = warp & 3;
    const int ml = quad * 32 + lane;
    const int et = ml;
    int seg = 0;
    for (int cur = beg; cur < end; ++seg) {
      const int t = cur / p.nkb, kb_lo = cur % p.nkb, kb_hi = min(p.nkb, kb_lo + (end - cur));
      const int buf = seg & 1;
      mbar_wait(&tfull[buf], (seg >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int first = sk_owner((long long)t * p.nkb, W, p.G);
      const int np = sk_owner((long long)(t + 1) * p.nkb - 1, W, p.G) - first + 1;
      const int part = blockIdx.x - first;
      float* tws = p.ws + (size_t)t * p.maxp * BN * 128;
      {
        float* dst = tws + (size_t)part * BN * 128 + ml;
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + buf * BN;
        constexpr int CH = BN < 32 ? 16 : 32;
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += CH) {
          float v[32];
          if constexpr (CH == 32) tmem_ld32(taddr + c0, v);
          else tmem_ld16(taddr + c0, v);
#pragma unroll
          for (int j = 0; j < CH; ++j)
            if (c0 + j < p.N) dst[(size_t)(c0 + j) * 128] = v[j];
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf])) : "memory");
      cur += kb_hi - kb_lo;
      // ---- arrival: the last CTA to finish a part of tile t applies its epilogue
      // (CTA barrier, then one gpu-scope fence + atomic by one thread: cumulative release)
      named_bar(1, 128);
      if (et == 0) {
        __threadfence();
        const unsigned old = atomicAdd(&p.ctr[t], 1u);
        const int last = old == (unsigned)(np - 1);
        if (last) p.ctr[t] = 0;
        *flag = last;
      }
      if (et == 0 && *flag) __threadfence();  // acquire side
      named_bar(1, 128);
      if (!*flag) continue;
      const int m = t * 128 + ml;
      if (p.fuse == FUSE_ROPE) {
        for (int n = 0; n < p.N; ++n) {
          float a = 0.f;
          for (int pt = 0; pt < np; ++pt) a += __ldcg(tws + (size_t)pt * BN * 128 + (size_t)n * 128 + ml);
          if (p.rs) a *= __ldg(p.rs + n);
          vals[ml * BN + n] = __bfloat162float(__float2bfloat16_rn(a));
        }
        named_bar(1, 128);
        const int H = p.nh * p.hd, half = p.hd >> 1;
        const int region = (t * 128) / H, r0 = (t * 128) % H;  // 0 q, 1 k, 2 v
        if (et < 64) {
          const int hl = et / half, i = et % half;
          const int ra = hl * p.hd + i, rb = ra + half;
          const int head = (r0 + ra) / p.hd;
          for (int n = 0; n < p.N; ++n) {
            const float a = vals[ra * BN + n], b = vals[rb * BN + n];
            const int sl = p.slot[n];
            if (sl < 0 || sl >= p.nslots) continue;  // never dereference an out-of-range slot
            const size_t blk = (size_t)(sl >> 4), off = (size_t)(sl & 15);
            if (region == 2) {
              bf16* vd = p.pool + (((blk * 2 + 1) * p.nh + head) * 16 + off) * p.hd;
              vd[i] = __float2bfloat16_rn(a);
              vd[i + half] = __float2bfloat16_rn(b);
            } else {
              const float2 cs = p.tab[(size_t)p.pos[n] * half + i];
              const bf16 x1 = __float2bfloat16_rn(a * cs.x - b * cs.y), x2 = __float2bfloat16_rn(b * cs.x + a * cs.y);
              bf16* d = region == 0 ? p.q_out + (size_t)n * H + head * p.hd
                                    : p.pool + (((blk * 2 + 0) * p.nh + head) * 16 + off) * p.hd;
              d[i] = x1;
              d[i + half] = x2;
            }
          }
        }
        named_bar(1, 128);
        continue;
      }
      for (int n = 0; n < p.N; ++n) {
        float a = 0.f;
        for (int pt = 0; pt < np; ++pt) a += __ldcg(tws + (size_t)pt * BN * 128 + (size_t)n * 128 + ml);
        if (p.rs && (p.epi == EPI_BF16 || p.epi == EPI_SILU_MUL)) a *= __ldg(p.rs + n);
        if (p.epi == EPI_F32) {
          reinterpret_cast<float*>(p.out)[(size_t)n * p.ldo + m] = a;
        } else if (p.epi == EPI_BF16) {
          reinterpret_cast<bf16*>(p.out)[(size_t)n * p.ldo + m] = __float2bfloat16_rn(a);
        } else if (p.epi == EPI_RESID) {
          reinterpret_cast<bf16*>(p.out)[(size_t)n * p.ldo + m] =
              __float2bfloat16_rn(a + __bfloat162float(p.resid[(size_t)n * p.ldr + m]));
        } else {  // silu-mul: lanes 0-15 gate rows, 16-31 their up rows
          const float u = __shfl_xor_sync(0xffffffffu, a, 16);
          if (lane < 16) reinterpret_cast<bf16*>(p.out)[(size_t)n * p.ldo + (m >> 5) * 16 + lane] = __float2bfloat16_rn(silu_f(a) * u);
        }
      }
      if (p.fuse == FUSE_NORM) {  // grid-level arrival: the last tile's CTA normalises the rows
        named_bar(1, 128);
        if (et == 0) {
          __threadfence();
          const unsigned old = atomicAdd(&p.ctr[p.tiles], 1u);
          const int last = old == (unsigned)(p.tiles - 1);
          if (last) {
            p.ctr[p.tiles] = 0;
            __threadfence();
          }
          *flag = last;
        }
        named_bar(1, 128);
        if (*flag) {
          for (int n = 0; n < p.N; ++n)
            row_norm128(reinterpret_cast<const bf16*>(p.out) + (size_t)n * p.ldo, p.M, p.norm_w,
                        p.norm_out + (size_t)n * p.ldo, p.rs_out ? p.rs_out + n : nullptr, p.eps, et, red, 1);
        }
      }
    }
  }
  if (tr && threadIdx.x == 64) tr[5] = gtimer();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[6] = gtimer();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)C::TMEM_COLS));
}

// ------------------------------------------------------------------ persistent tiled (prefill)
// Tensor-bound GEMM for many tokens.  Persistent CTAs (one per SM) walk a static tile
// schedule (tile = blockIdx.x + i * gridDim.x, consecutive tiles share the weight tile so the
// second read hits L2); warp 0 TMA producer, warp 1 MMA issuer, warps 2-5 epilogue; two TMEM
// accumulators so the epilogue of tile i overlaps the MMAs of tile i+1.
struct TpParams {
  int M, N, nkb, m_tiles, n_tiles;
  int epi;
  void* out;
  int ldo;
  const bf16* resid;
  int ldr;
  int splits = 1, kbps = 0;  // split-K (tp2 only): work item = tile * splits + split
  float* ws = nullptr;       // fp32 partials [split][N][M] when splits > 1
  const float* rs = nullptr;
};

template <int BN>
struct TpCfg {
  static constexpr int A_BYTES = 128 * 64 * 2;
  static constexpr int B_BYTES = BN * 64 * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN >= 256 ? 4 : 6;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int BN>
__global__ void __launch_bounds__(192, 1)
    gemm_tp_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TpParams p) {
  using C = TpCfg<BN>;
  PDL_LAUNCH();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = p.m_tiles * p.n_tiles;

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // weights of the first stages before the grid dependency resolves
      const int my_tiles = blockIdx.x < tiles ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
      const int pre = min(my_tiles * p.nkb, C::STAGES);
      for (int i = 0; i < pre; ++i) {
        const int t = blockIdx.x + (i / p.nkb) * gridDim.x;
        mbar_expect_tx(&full[i], C::STAGE_BYTES);
        tma_load_w(&tmA, &full[i], smem + i * C::STAGE_BYTES, (t / p.n_tiles) * p.nkb + (i % p.nkb));
      }
      PDL_WAIT();
      for (int i = 0; i < pre; ++i) {
        const int t = blockIdx.x + (i / p.nkb) * gridDim.x;
        tma_load_2d(&tmB, &full[i], smem + i * C::STAGE_BYTES + C::A_BYTES, (i % p.nkb) * 64, (t % p.n_tiles) * BN);
      }
      int i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int m0 = (t / p.n_tiles) * 128, n0 = (t % p.n_tiles) * BN;
        for (int kb = 0; kb < p.nkb; ++kb, ++i) {
          if (i < pre) continue;
          const int s = i % C::STAGES;
          mbar_wait(&empty[s], ((i / C::STAGES) & 1) ^ 1);
          uint8_t* sa = smem + s * C::STAGE_BYTES;
          mbar_expect_tx(&full[s], C::STAGE_BYTES);
          tma_load_w(&tmA, &full[s], sa, (m0 / 128) * p.nkb + kb);
          tma_load_2d(&tmB, &full[s], sa + C::A_BYTES, kb * 64, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = instr_desc<BN>();
      int i = 0, lt = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++lt) {
        const int buf = lt & 1;
        mbar_wait(&tempty[buf], ((lt >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + buf * BN;
        for (int kb = 0; kb < p.nkb; ++kb, ++i) {
          const int s = i % C::STAGES;
          mbar_wait(&full[s], (i / C::STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t* sa = smem + s * C::STAGE_BYTES;
          const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + C::A_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) umma_bf16(acc, da + 2 * k, db + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[buf]);
      }
    }
  } else {
    PDL_WAIT();
    const int quad = warp & 3;
    int lt = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++lt) {
      const int buf = lt & 1;
      const int m0 = (t / p.n_tiles) * 128, n0 = (t % p.n_tiles) * BN;
      mbar_wait(&tfull[buf], (lt >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int m = m0 + quad * 32 + lane;
      const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16) + buf * BN;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld32(trow + c0, v);
        if (n0 + c0 < p.N) {
          const int ncol = min(32, p.N - n0 - c0);
          if (p.epi == EPI_BF16 || p.epi == EPI_SILU_MUL) scale_rows<32>(v, p.rs, n0 + c0, ncol);
          if (p.epi == EPI_F32) {
            float* o = reinterpret_cast<float*>(p.out) + (size_t)(n0 + c0) * p.ldo;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < ncol) o[(size_t)j * p.ldo + m] = v[j];
          } else if (p.epi == EPI_BF16) {
            bf16* o = reinterpret_cast<bf16*>(p.out) + (size_t)(n0 + c0) * p.ldo;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < ncol) o[(size_t)j * p.ldo + m] = __float2bfloat16_rn(v[j]);
          } else if (p.epi == EPI_RESID) {
            bf16* o = reinterpret_cast<bf16*>(p.out) + (size_t)(n0 + c0) * p.ldo;
            const bf16* r = p.resid + (size_t)(n0 + c0) * p.ldr;
            // all residual loads first (out may alias resid for the compiler: interleaving the
            // loads with the stores would serialise 32 L2 round trips per chunk)
            float rv[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) rv[j] = j < ncol ? __bfloat162float(__ldg(r + (size_t)j * p.ldr + m)) : 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < ncol) o[(size_t)j * p.ldo + m] = __float2bfloat16_rn(v[j] + rv[j]);
          } else {
            bf16* o = reinterpret_cast<bf16*>(p.out) + (size_t)(n0 + c0) * p.ldo;
            const int f = (m0 + quad * 32) / 2 + (lane & 15);
            silu_mul_store32(v, lane, o + f, (size_t)p.ldo, ncol);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf])) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)C::TMEM_COLS));
}

// Decode RMSNorm with the exact arithmetic of the fused epilogue (one 128-thread CTA per row).
__global__ void __launch_bounds__(128) rownorm_kernel(const bf16* __restrict__ x, const bf16* __restrict__ w,
                                                      bf16* __restrict__ y, float* rs_out, int H, float eps) {
  PDL_LAUNCH();
  PDL_WAIT();
  __shared__ float red[4];
  row_norm128(x + (size_t)blockIdx.x * H, H, w, y + (size_t)blockIdx.x * H, rs_out ? rs_out + blockIdx.x : nullptr,
              eps, threadIdx.x, red, 1);
}

// ------------------------------------------------------------------ host side -----------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

hs_status make_tma(TmaMat* t, const void* ptr, int64_t rows, int64_t cols, int box_rows) {
  auto enc = get_encode();
  if (!enc) HS_FAIL(HS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (cols % 64 || (reinterpret_cast<uintptr_t>(ptr) & 15)) HS_FAIL(HS_E_INVAL, "bad matrix for TMA");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&t->map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) HS_FAIL(HS_E_CUDA, "cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld box=%d", (int)r,
                                 (long long)rows, (long long)cols, box_rows);
  t->ptr = ptr;
  t->rows = rows;
  t->cols = cols;
  t->box_rows = box_rows;
  return HS_OK;
}

hs_status make_tma3(TmaMat* t, const void* ptr, int64_t layers, int64_t layer_stride_bytes, int64_t rows,
                    int64_t cols) {
  auto enc = get_encode();
  if (!enc) HS_FAIL(HS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (cols % 64 || rows % 128 || (reinterpret_cast<uintptr_t>(ptr) & 15) || layer_stride_bytes % 16)
    HS_FAIL(HS_E_INVAL, "bad layered matrix for TMA");
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)layers};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)layer_stride_bytes};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&t->map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) HS_FAIL(HS_E_CUDA, "cuTensorMapEncodeTiled (3d) failed (%d)", (int)r);
  t->ptr = ptr;
  t->rows = rows;
  t->cols = cols;
  t->box_rows = 128;
  return HS_OK;
}

hs_status make_tma_w(TmaMat* t, const void* ptr, int64_t rows, int64_t cols) {
  auto enc = get_encode();
  if (!enc) HS_FAIL(HS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (cols % 64 || rows % 128 || (reinterpret_cast<uintptr_t>(ptr) & 15)) HS_FAIL(HS_E_INVAL, "bad tiled weight for TMA");
  cuuint64_t dims[3] = {64, 128, (cuuint64_t)((rows / 128) * (cols / 64))};
  cuuint64_t strides[2] = {128, 16384};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&t->map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) HS_FAIL(HS_E_CUDA, "cuTensorMapEncodeTiled (tiled weight) failed (%d)", (int)r);
  t->ptr = ptr;
  t->rows = rows;
  t->cols = cols;
  t->box_rows = 128;
  return HS_OK;
}

hs_status make_tma_w3(TmaMat* t, const void* ptr, int64_t layers, int64_t layer_stride_bytes, int64_t rows,
                      int64_t cols) {
  auto enc = get_encode();
  if (!enc) HS_FAIL(HS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (cols % 64 || rows % 128 || (reinterpret_cast<uintptr_t>(ptr) & 15) || layer_stride_bytes % 16)
    HS_FAIL(HS_E_INVAL, "bad layered tiled weight for TMA");
  cuuint64_t dims[4] = {64, 128, (cuuint64_t)((rows / 128) * (cols / 64)), (cuuint64_t)layers};
  cuuint64_t strides[3] = {128, 16384, (cuuint64_t)layer_stride_bytes};
  cuuint32_t box[4] = {64, 128, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(&t->map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) HS_FAIL(HS_E_CUDA, "cuTensorMapEncodeTiled (layered tiled weight) failed (%d)", (int)r);
  t->ptr = ptr;
  t->rows = rows;
  t->cols = cols;
  t->box_rows = 128;
  return HS_OK;
}

bool pdl_enabled() {
  static int on = [] {
    const char* e = getenv("HS_PDL");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return on != 0;
}

static const int kBN[] = {16, 32, 64, 128, 256};
static constexpr double kTp2Rate128 = 0.9, kTp2Rate256 = 1.6;  // per-SM rate vs gemm_tp_kernel<128> (measured r01)
int gemm_bn_count() { return 5; }
int gemm_bn_value(int i) { return kBN[i]; }
int gemm_bn(int N) {
  if (N <= 16) return 16;
  if (N <= 32) return 32;
  if (N <= 64) return 64;
  if (N <= 1024) return 128;
  return 256;
}

template <int BN>
static hs_status launch(const GemmArgs& a, int splits, int kbps, cudaStream_t st) {
  using C = Cfg<BN>;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_set[dev]) {
    HS_CUDA(cudaFuncSetAttribute(gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set[dev] = true;
  }
  int bi = 0;
  while (kBN[bi] != BN) ++bi;
  const TmaMat& tb = a.B[bi];
  if (tb.box_rows != BN || a.A->box_rows != 128) HS_FAIL(HS_E_INVAL, "TMA box mismatch");
  KParams p;
  p.M = a.M; p.N = a.N; p.K = a.K;
  p.nkb = a.K / 64;
  p.kb_per_split = kbps;
  p.epi = splits > 1 ? -1 : a.epi;
  p.out = a.out; p.ldo = a.ldo; p.resid = a.resid; p.ldr = a.ldr; p.ws = a.workspace; p.rs = a.rs;
  dim3 grid(cdiv(a.M, 128), cdiv(a.N, BN), splits);
  launchk(gemm_kernel<BN>, grid, 128, C::SMEM, st, a.A->map, tb.map, p);
  count_launch();
  HS_CUDA(cudaGetLastError());
  if (splits > 1) {
    dim3 g2(cdiv(a.M, 256), a.N);
    launchk(splitk_reduce_kernel, g2, 256, 0, st, (const float*)a.workspace, splits, a.M, a.N, a.epi, a.out, a.ldo, a.resid, a.ldr, a.rs);
    count_launch();
    HS_CUDA(cudaGetLastError());
  }
  return HS_OK;
}

template <int BN>
static void warm_one() {
  cudaFuncAttributes at;
  cudaFuncSetAttribute(gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM);
  cudaFuncGetAttributes(&at, gemm_kernel<BN>);
}

template <int BN>
static void warm_sk() {
  cudaFuncAttributes at;
  cudaFuncSetAttribute(gemm_sk_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, SkCfg<BN>::SMEM);
  cudaFuncGetAttributes(&at, gemm_sk_kernel<BN>);
}

template <int BN>
static void warm_tp() {
  cudaFuncAttributes at;
  cudaFuncSetAttribute(gemm_tp_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, TpCfg<BN>::SMEM);
  cudaFuncGetAttributes(&at, gemm_tp_kernel<BN>);
}

void warm_gemm_kernels() {
  warm_tp<128>();
  warm_tp<256>();
  warm_sk<16>();
  warm_sk<32>();
  warm_sk<64>();
  cudaFuncAttributes at0;
  cudaFuncGetAttributes(&at0, rownorm_kernel);
  warm_one<16>();
  warm_one<32>();
  warm_one<64>();
  warm_one<128>();
  warm_one<256>();
  cudaFuncAttributes at;
  cudaFuncGetAttributes(&at, splitk_reduce_kernel);
}

// HS_TRACE=1: the stream-K GEMM records per-CTA phase timestamps (hs_debug_gemm_trace)
static unsigned long long* g_sk_trace = nullptr;

template <int BN>
static hs_status launch_sk(const GemmArgs& a, cudaStream_t st, bool* done) {
  using C = SkCfg<BN>;
  int dev = 0;
  cudaGetDevice(&dev);
  const int G = num_sms(dev);
  const int tiles = a.M / 128, nkb = a.K / 64;
  const long long W = (long long)tiles * nkb;
  const int per = (int)(W / G);
  if (per < 2) return HS_OK;  // too little work per SM: use the tiled kernel
  const int maxp = (nkb + per - 1) / per + 1;
  const uint64_t ctr_bytes = align_up((uint64_t)(tiles + 1) * 4, 256);
  if (ctr_bytes + (uint64_t)tiles * maxp * BN * 128 * 4 > a.workspace_bytes || !a.counters) return HS_OK;
  const GemmFusion& f = a.fuse;
  if (f.kind == FUSE_ROPE && (a.epi != EPI_BF16 || (f.head_dim != 64 && f.head_dim != 128) || BN > 64)) return HS_OK;
  if (f.kind == FUSE_NORM && BN > 64) return HS_OK;
  static bool attr_set[64] = {};
  if (dev < 64 && !attr_set[dev]) {
    HS_CUDA(cudaFuncSetAttribute(gemm_sk_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set[dev] = true;
  }
  int bi = 0;
  while (kBN[bi] != BN) ++bi;
  SkParams p{};
  p.M = a.M; p.N = a.N; p.nkb = nkb; p.tiles = tiles; p.G = G; p.maxp = maxp;
  p.ws = a.workspace; p.ctr = a.counters;
  p.epi = a.epi; p.out = a.out; p.ldo = a.ldo; p.resid = a.resid; p.ldr = a.ldr; p.rs = a.rs;
  p.fuse = f.kind; p.norm_w = f.norm_w; p.norm_out = f.norm_out; p.rs_out = f.rs_out; p.eps = f.eps; p.rs = a.rs;
  p.pos = f.pos; p.slot = f.slot; p.tab = f.rope_tab; p.q_out = f.q_out; p.pool = f.pool;
  p.nh = f.n_heads; p.hd = f.head_dim; p.nslots = f.nslots;
  p.trace = g_sk_trace;
  if (p.fuse == FUSE_NORM && a.epi != EPI_RESID) p.fuse = FUSE_NONE;
  launchk(gemm_sk_kernel<BN>, G, 192, C::SMEM, st, a.A->map, a.B[bi].map, p);
  count_launch();
  HS_CUDA(cudaGetLastError());
  if (f.applied && p.fuse != FUSE_NONE) *f.applied = true;
  *done = true;
  return HS_OK;
}

template <int BN>
static hs_status launch_tp(const GemmArgs& a, cudaStream_t st) {
  using C = TpCfg<BN>;
  int dev = 0;
  cudaGetDevice(&dev);
  static bool attr_set[64] = {};
  if (dev < 64 && !attr_set[dev]) {
    HS_CUDA(cudaFuncSetAttribute(gemm_tp_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set[dev] = true;
  }
  int bi = 0;
  while (kBN[bi] != BN) ++bi;
  if (a.B[bi].box_rows != BN) HS_FAIL(HS_E_INVAL, "TMA box mismatch");
  TpParams p{};
  p.M = a.M; p.N = a.N; p.nkb = a.K / 64; p.m_tiles = a.M / 128; p.n_tiles = (int)cdiv(a.N, BN);
  p.epi = a.epi; p.out = a.out; p.ldo = a.ldo; p.resid = a.resid; p.ldr = a.ldr; p.rs = a.rs;
  const int tiles = p.m_tiles * p.n_tiles;
  const int grid = std::min(tiles, num_sms(dev));
  launchk(gemm_tp_kernel<BN>, grid, 192, C::SMEM, st, a.A->map, a.B[bi].map, p);
  count_launch();
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

// ------------------------------------------------------------------ 2-SM persistent (prefill)
// CTA pair (cluster of 2, tcgen05 cta_group::2): a 256 x 256 output tile per pair, M = 256 rows
// of weights (128 per CTA) x N = 256 tokens (128 per CTA's shared memory); the leader CTA issues
// the MMAs, both CTAs' TMA loads complete on the leader's barrier, the MMA commits multicast
// to both CTAs' "empty" / "accumulator full" barriers, and each CTA drains its own 128 TMEM lanes
// (rows) x 256 columns.  Per SM a k-block moves 32 KB for 4.2 MFLOP (2x the single-CTA 128 x 256
// tile): prefill GEMMs are bound by how fast an SM ingests operands, not by the tensor pipe.
template <int BN>
struct Tp2Cfg {
  static constexpr int A_BYTES = 128 * 64 * 2;
  static constexpr int B_BYTES = (BN / 2) * 64 * 2;  // this CTA's half of the BN-token tile
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN >= 256 ? 6 : 8;
  static constexpr int TMEM_COLS = 2 * BN;           // two BN-column accumulators
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int BN>
__global__ void __launch_bounds__(192, 1)
    gemm_tp2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TpParams p) {
  using C = Tp2Cfg<BN>;
  PDL_LAUNCH();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int tiles = p.m_tiles * p.n_tiles * p.splits;  // work items; m_tiles counts 256-row pairs
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // both CTAs' barriers initialised before any remote arrive / TMA
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // producer (both CTAs): this CTA's 128 weight rows and 128 tokens
      PDL_WAIT();
      int i = 0;
      for (int w = cid; w < tiles; w += ncl) {
        const int t = w / p.splits, sp = w % p.splits;
        const int kb0 = sp * p.kbps, kb1 = min(p.nkb, kb0 + p.kbps);
        const int m0 = (t / p.n_tiles) * 256 + (int)rank * 128, n0 = (t % p.n_tiles) * BN + (int)rank * (BN / 2);
        for (int kb = kb0; kb < kb1; ++kb, ++i) {
          const int s = i % C::STAGES;
          mbar_wait(&empty[s], ((i / C::STAGES) & 1) ^ 1);
          uint8_t* sa = smem + s * C::STAGE_BYTES;
          // bytes complete on the leader's barrier (peer bit cleared); the leader arms it for both
          const uint32_t bar = smem_u32(&full[s]) & 0xFEFFFFFFu;
          if (leader) mbar_expect_tx(&full[s], 2 * C::STAGE_BYTES);
          asm volatile(  // the weight k-block: tiled layout, block (m0 / 128) * nkb + kb
              "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(sa)),
              "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(bar), "r"(0), "r"(0), "r"((m0 / 128) * p.nkb + kb)
              : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(sa + C::A_BYTES)),
              "l"(reinterpret_cast<uint64_t>(&tmB)), "r"(bar), "r"(kb * 64), "r"(n0)
              : "memory");
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // MMA issuer (leader only): M = 256 across the pair, N = 256
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)(256 >> 4) << 24);
      int i = 0, lt = 0;
      for (int w = cid; w < tiles; w += ncl, ++lt) {
        const int sp = w % p.splits;
        const int kb0 = sp * p.kbps, kb1 = min(p.nkb, kb0 + p.kbps);
        const int buf = lt & 1;
        mbar_wait(&tempty[buf], ((lt >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + buf * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++i) {
          const int s = i % C::STAGES;
          mbar_wait(&full[s], (i / C::STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t* sa = smem + s * C::STAGE_BYTES;
          const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + C::A_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t accum = (kb > kb0 || k > 0) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, q;\n\t}" ::"r"(acc),
                "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(accum));
          }
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                       ::"r"(smem_u32(&empty[s])), "h"((uint16_t)3) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&tfull[buf])), "h"((uint16_t)3) : "memory");
      }
    }
  } else {
    PDL_WAIT();
    const int quad = warp & 3;
    int lt = 0;
    for (int w = cid; w < tiles; w += ncl, ++lt) {
      const int t = w / p.splits, sp = w % p.splits;
      const int buf = lt & 1;
      const int m0 = (t / p.n_tiles) * 256 + (int)rank * 128, n0 = (t % p.n_tiles) * BN;
      mbar_wait(&tfull[buf], (lt >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int m = m0 + quad * 32 + lane;
      const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16) + buf * BN;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld32(trow + c0, v);
        if (n0 + c0 < p.N) {
          const int ncol = min(32, p.N - n0 - c0);
          if (p.splits <= 1 && (p.epi == EPI_BF16 || p.epi == EPI_SILU_MUL)) scale_rows<32>(v, p.rs, n0 + c0, ncol);
          if (p.splits > 1) {  // fp32 partial of this split (reduced by splitk_reduce_kernel)
            float* o = p.ws + ((size_t)sp * p.N + n0 + c0) * p.M;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < ncol) o[(size_t)j * p.M + m] = v[j];
          } else if (p.epi == EPI_F32) {
            float* o = reinterpret_cast<float*>(p.out) + (size_t)(n0 + c0) * p.ldo;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < ncol) o[(size_t)j * p.ldo + m] = v[j];
          } else if (p.epi == EPI_BF16) {
            bf16* o = reinterpret_cast<bf16*>(p.out) + (size_t)(n0 + c0) * p.ldo;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < ncol) o[(size_t)j * p.ldo + m] = __float2bfloat16_rn(v[j]);
          } else if (p.epi == EPI_RESID) {
            bf16* o = reinterpret_cast<bf16*>(p.out) + (size_t)(n0 + c0) * p.ldo;
            const bf16* r = p.resid + (size_t)(n0 + c0) * p.ldr;
            float rv[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) rv[j] = j < ncol ? __bfloat162float(__ldg(r + (size_t)j * p.ldr + m)) : 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < ncol) o[(size_t)j * p.ldo + m] = __float2bfloat16_rn(v[j] + rv[j]);
          } else {
            bf16* o = reinterpret_cast<bf16*>(p.out) + (size_t)(n0 + c0) * p.ldo;
            const int f = (m0 + quad * 32) / 2 + (lane & 15);
            silu_mul_store32(v, lane, o + f, (size_t)p.ldo, ncol);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      // release the accumulator on the leader's barrier (both CTAs' 4 epilogue warps)
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf]) & 0xFEFFFFFFu)
                     : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)C::TMEM_COLS));
}

template <int BN>
static hs_status launch_tp2(const GemmArgs& a, cudaStream_t st, int splits = 1) {
  using C = Tp2Cfg<BN>;
  int dev = 0;
  cudaGetDevice(&dev);
  static bool attr_set[64] = {};
  if (dev < 64 && !attr_set[dev]) {
    HS_CUDA(cudaFuncSetAttribute(gemm_tp2_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set[dev] = true;
  }
  int bi = 0;
  while (kBN[bi] != BN / 2) ++bi;
  if (a.B[bi].box_rows != BN / 2) HS_FAIL(HS_E_INVAL, "TMA box mismatch");
  TpParams p{};
  p.M = a.M; p.N = a.N; p.nkb = a.K / 64; p.m_tiles = a.M / 256; p.n_tiles = (int)cdiv(a.N, BN);
  p.epi = a.epi; p.out = a.out; p.ldo = a.ldo; p.resid = a.resid; p.ldr = a.ldr; p.rs = a.rs;
  p.kbps = (int)cdiv(p.nkb, splits);
  p.splits = (int)cdiv(p.nkb, p.kbps);
  p.ws = a.workspace;
  if (p.splits > 1 && (!a.workspace || (uint64_t)p.splits * a.N * a.M * 4 > a.workspace_bytes))
    HS_FAIL(HS_E_INVAL, "split-K workspace too small");
  const int tiles = p.m_tiles * p.n_tiles * p.splits;
  const int pairs = std::min(tiles, num_sms(dev) / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  int na = 1;
  if (pdl_enabled()) {
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    na = 2;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  HS_CUDA(cudaLaunchKernelEx(&cfg, gemm_tp2_kernel<BN>, a.A->map, a.B[bi].map, p));
  count_launch();
  if (p.splits > 1) {
    dim3 g2(cdiv(a.M, 256), a.N);
    launchk(splitk_reduce_kernel, g2, 256, 0, st, (const float*)a.workspace, p.splits, a.M, a.N, a.epi, a.out, a.ldo,
            a.resid, a.ldr, a.rs);
    count_launch();
    HS_CUDA(cudaGetLastError());
  }
  return HS_OK;
}

void launch_rownorm_decode(const bf16* x, const bf16* w, bf16* y, float* rs_out, int T, int H, float eps,
                           cudaStream_t st) {
  launchk(rownorm_kernel, T, 128, 0, st, x, w, y, rs_out, H, eps);
  count_launch();
}

hs_status gemm(const GemmArgs& a, cudaStream_t st) {
  if (a.M % 128 || a.K % 64 || a.N <= 0) HS_FAIL(HS_E_INVAL, "gemm shape M=%d N=%d K=%d", a.M, a.N, a.K);
  if (a.fuse.applied) *a.fuse.applied = false;
  const int BN = gemm_bn(a.N);
  if (BN <= 64 && a.workspace) {  // weight-streaming decode GEMM: stream-K over all SMs
    bool done = false;
    hs_status r = BN == 16 ? launch_sk<16>(a, st, &done) : BN == 32 ? launch_sk<32>(a, st, &done) : launch_sk<64>(a, st, &done);
    if (r != HS_OK || done) return r;
  }
  if (a.N > 64) {  // tensor-bound: persistent tiles; BN minimising (waves x tile cost)
    int dev = 0;
    cudaGetDevice(&dev);
    const int G = num_sms(dev), mt = a.M / 128;
    // too few 128-token tiles to fill half the SMs (prefill chunks x small M): tiled kernel
    // with deterministic split-K below (its reduction is one fully parallel pass)
    if (!(a.workspace && 2LL * mt * cdiv(a.N, 128) <= G))
    {
      const long long c128 = cdiv((long long)mt * cdiv(a.N, 128), G) * 128;
      const long long c256 = cdiv((long long)mt * cdiv(a.N, 256), G) * 256;
      static int force = [] {
        const char* e = getenv("HS_TP_BN");
        return e ? atoi(e) : 0;
      }();
      if (force == 256) return launch_tp<256>(a, st);
      if (force == 128) return launch_tp<128>(a, st);
      static int tp2 = [] {
        const char* e = getenv("HS_TP2");
        return (e && e[0] == '0') ? 0 : 1;
      }();
      if (tp2 && a.M % 256 == 0 && force != 1) {
        // cost = waves x 128x128 tile-equivalents per SM / relative per-SM rate (measured:
        // the CTA pair halves each SM's operand bytes per flop); min over the three kernels
        const double w128 = (double)cdiv((long long)mt * cdiv(a.N, 128), G);
        const double c2_128 = (double)cdiv((long long)(a.M / 256) * cdiv(a.N, 128), G / 2) / kTp2Rate128;
        const double c2_256 = (double)cdiv((long long)(a.M / 256) * cdiv(a.N, 256), G / 2) * 2.0 / kTp2Rate256;
        if (force == 2128) return launch_tp2<128>(a, st);
        if (force == 2256) return launch_tp2<256>(a, st);
        // few pair tiles (M = 4096): split K over the pairs, fp32 partials + one reduction pass
        int best_s = 1;
        double best = c2_256;
        const long long pairs256 = (long long)(a.M / 256) * cdiv(a.N, 256);
        // only when the pairs fill less than half the clusters and K is long (down-proj): the
        // reduction's traffic (S x N x M x 4 B) outweighs the gain otherwise (measured)
        static const int split_min_kb = [] {  // A/B knob: K blocks needed before pairs split K
          const char* e = getenv("HS_TP2_SPLIT_MINKB");
          return e && atoi(e) > 0 ? atoi(e) : 128;
        }();
        for (int sk = 2; sk <= 4 && pairs256 * 2 <= G / 2 && a.K / 64 >= split_min_kb; ++sk) {
          if (!a.workspace || (uint64_t)sk * a.N * a.M * 4 > a.workspace_bytes) break;
          const double c = (double)cdiv(pairs256 * sk, G / 2) * 2.0 / kTp2Rate256 / sk + 0.1 * sk;
          if (c < best) { best = c; best_s = sk; }
        }
        if (force >= 22560 && force <= 22564) return launch_tp2<256>(a, st, force - 22560);
        if (c2_128 < w128 && c2_128 <= best) return launch_tp2<128>(a, st);
        if (best < w128) return launch_tp2<256>(a, st, best_s);
      }
      return c256 < c128 ? launch_tp<256>(a, st) : launch_tp<128>(a, st);
    }
  }
  const int tiles = (a.M / 128) * (int)cdiv(a.N, BN);
  const int nkb = a.K / 64;
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = num_sms(dev);
  // split-K (deterministic: depends on M, N, K only) when the tile grid leaves SMs idle
  int splits = 1;
  if (a.workspace && tiles < sms) {
    int best = 1;
    double best_u = (double)tiles / sms;
    for (int s = 2; s <= 16 && nkb / s >= 4; ++s) {
      const int ctas = tiles * s;
      const double waves = std::ceil((double)ctas / sms);
      const double u = (double)ctas / (waves * sms) * std::min(1.0, (double)ctas / sms);
      if (u > best_u + 1e-9 && (uint64_t)s * a.N * a.M * 4 <= a.workspace_bytes) { best = s; best_u = u; }
    }
    splits = best;
  }
  const int kbps = (int)cdiv(nkb, splits);
  splits = (int)cdiv(nkb, kbps);
  switch (BN) {
    case 16: return launch<16>(a, splits, kbps, st);
    case 32: return launch<32>(a, splits, kbps, st);
    case 64: return launch<64>(a, splits, kbps, st);
    case 128: return launch<128>(a, splits, kbps, st);
    default: return launch<256>(a, splits, kbps, st);
  }
}

}  // namespace hs

extern "C" hs_status hs_debug_gemm_trace(int32_t enable, void* host_out, int32_t n_ctas) {
  using namespace hs;
  if (enable && !g_sk_trace) {
    HS_CUDA(cudaMalloc(&g_sk_trace, 4096 * 8 * 8));
    HS_CUDA(cudaMemset(g_sk_trace, 0, 4096 * 8 * 8));
  }
  if (host_out && g_sk_trace) {
    HS_CUDA(cudaDeviceSynchronize());
    HS_CUDA(cudaMemcpy(host_out, g_sk_trace, (size_t)n_ctas * 8 * 8, cudaMemcpyDeviceToHost));
  }
  if (!enable && g_sk_trace) {
    cudaFree(g_sk_trace);
    g_sk_trace = nullptr;
  }
  return HS_OK;
}
