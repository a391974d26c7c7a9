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
// One pass with an online softmax per row (flash attention): each chunk's P V lands in a fresh
// TMEM block and is added to the row's fp32 accumulator in registers, O = O * corr + P V; the
// next chunk's K and V rows stream in with cp.async while this chunk computes; o = O / l, one
// bf16 rounding.  Operands live in shared memory in the tcgen05 K-major 128B-swizzled layout:
// Q and K rows straight from the q buffer / the paged pool, V transposed from its staged rows
// (V^T [head_dim][keys]) while the tensor core computes S, P written row by row by its owner
// thread.  Deterministic; causal mask and ragged tails by position.
#include <cmath>
#include <cstdlib>

#include "kernels.h"
#include "tc.h"

namespace hs {

constexpr int TA_Q = 128;   // queries per CTA
constexpr int TA_KC = 64;   // keys per chunk: 112 KB of shared memory (D = 128), two CTAs per SM

template <int D>
struct TaCfg {
  static constexpr int KK = TA_KC / 64;                // 64-wide k-blocks of a key chunk
  static constexpr int KB = D / 64;                    // 64-wide k-blocks of head_dim
  static constexpr int Q_BYTES = KB * TA_Q * 128;      // Q: KB tiles [128 q][64 d]
  static constexpr int K_BYTES = KB * TA_KC * 128;     // K: KB tiles [128 keys][64 d]
  static constexpr int VS_BYTES = KB * TA_KC * 128;    // V staging, same layout as K
  static constexpr int V_BYTES = KK * D * 128;         // V^T: KK tiles [D d][64 keys]
  static constexpr int P_BYTES = KK * TA_Q * 128;      // P half: KK tiles [128 q][64 keys]
  // no alignment slack: the dynamic window starts 1024-aligned (no static shared memory), which
  // keeps two CTAs within one SM's 228 KB at D = 128
  static constexpr int SMEM = Q_BYTES + K_BYTES + VS_BYTES + V_BYTES + 2 * P_BYTES + 64;
  static constexpr uint32_t TMEM_COLS = 256;           // S: TA_KC columns, O block: D columns (at 128)
};

// 16-byte chunk c (0..7) of row r of a [rows][64] bf16 tile in the 128B-swizzled layout
__device__ __forceinline__ uint32_t sw128(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

template <int D>
__global__ void __launch_bounds__(128, TA_KC == 64 ? 2 : 1) attn_prefill_tc_kernel(
    const bf16* __restrict__ q, const bf16* __restrict__ pool, const SeqDesc* __restrict__ seqs,
    const int* __restrict__ tables, int max_blocks, bf16* __restrict__ o, int nh, int nblocks) {
  using C = TaCfg<D>;
  PDL_LAUNCH();
  // before the first read of the call's metadata (seqs, tables): they are staged into device
  // memory by a kernel earlier in the same stream, and with every kernel triggering its
  // dependents at entry a whole chain of them can be resident before that copy ends.  Reading
  // seqs before this wait (run 45 / 47: a stale n_q returned CTAs early) made the kernel
  // nondeterministic.
  PDL_WAIT();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023)) __trap();  // the SW128 tiles need 1024-byte alignment
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + C::Q_BYTES;
  uint8_t* sVs = sK + C::K_BYTES;   // V rows as loaded
  uint8_t* sV = sVs + C::VS_BYTES;  // V^T
  uint8_t* sP = sV + C::V_BYTES;    // [hi | lo]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + 2 * C::P_BYTES);  // [0] S, [1] P V
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int t = threadIdx.x, warp = t >> 5;
  const SeqDesc s = seqs[blockIdx.z];
  const int head = blockIdx.y;
  const int q0 = (gridDim.x - 1 - blockIdx.x) * TA_Q;  // longest (causal) query tiles first
  if (q0 >= s.n_q) return;
  const int H = nh * D;
  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const int* tab = tables + (size_t)s.table * max_blocks;
  const int n_keys = s.pos0 + min(q0 + TA_Q, s.n_q);  // keys any row of the tile sees
  const int n_chunks = (n_keys + TA_KC - 1) / TA_KC;
  // K and V rows of chunk kc into sK / sVs (swizzled): thread t copies key kc + t with 16-byte
  // cp.async (zero-filled past the keys), no registers held
  constexpr int TPK = 128 / TA_KC;            // threads per key row
  constexpr int CPT = (D / 8) / TPK;           // 16-byte chunks per thread and row
  const int krow = t % TA_KC, cpart = t / TA_KC;
  auto issue = [&](int kc, bool k_part, bool v_part) {
    const int j = kc + krow;
    const bf16* kp = pool;
    int bytes = 0;
    if (j < n_keys) {
      int b = tab[j >> 4];
      if (b < 0 || b >= nblocks) b = 0;
      kp = pool + ((((size_t)b * 2) * nh + head) * 16 + (j & 15)) * D;
      bytes = 16;
    }
#pragma unroll
    for (int cc = 0; cc < CPT; ++cc) {
      const int c = cpart * CPT + cc;
      const uint32_t off = (c >> 3) * (TA_KC * 128) + sw128(krow, c & 7);
      if (k_part)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sK + off)), "l"(kp + c * 8), "r"(bytes)
                     : "memory");
      if (v_part)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sVs + off)),
                     "l"(kp + (size_t)nh * 16 * D + c * 8), "r"(bytes)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(0, true, true);
  // Q rows: thread t loads query q0 + t (rows past n_q repeat the last row: never stored).
  // L2 loads (__ldcg), not the non-coherent path: q is written by the previous kernel, which
  // under PDL still runs during this kernel's lifetime (ld.global.nc requires data read-only
  // for the whole lifetime)
  const int qi = min(q0 + t, s.n_q - 1);
  const int pos = s.pos0 + q0 + t;  // this row's position (causal bound)
  {
    const uint4* src = reinterpret_cast<const uint4*>(q + (size_t)(s.q_start + qi) * H + head * D);
#pragma unroll
    for (int c = 0; c < D / 8; ++c)
      *reinterpret_cast<uint4*>(sQ + (c >> 3) * (TA_Q * 128) + sw128(t, c & 7)) = __ldcg(src + c);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 128;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  const float sl2 = 1.4426950408889634f / sqrtf((float)D);
  constexpr uint32_t idS = instr_desc<TA_KC>();  // M = 128, N = TA_KC keys
  constexpr uint32_t idO = instr_desc<D>();      // M = 128, N = head_dim
  uint32_t ph_s = 0, ph_o = 0;
  float m = -INFINITY, l = 0.f, acc[D];
#pragma unroll
  for (int d = 0; d < D; ++d) acc[d] = 0.f;

  for (int ci = 0; ci < n_chunks; ++ci) {
    const int kc = ci * TA_KC;
    asm volatile("cp.async.wait_all;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // cp.async (generic) -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // K_c and V_c rows landed; the previous chunk's TMEM reads are done
    if (t == 0) {  // S = Q K^T over head_dim
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int kb = 0; kb < C::KB; ++kb) {
        const uint64_t da = umma_desc_sw128(sQ + kb * (TA_Q * 128)), db = umma_desc_sw128(sK + kb * (TA_KC * 128));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_bf16(tS, da + 2 * kk, db + 2 * kk, idS, (kb | kk) ? 1u : 0u);
      }
      umma_commit(&bar[0]);
    }
    {  // V^T from the staged rows while the tensor core computes S (key krow, this thread's chunks)
      const int kbv = krow >> 6, kl = krow & 63;
      uint8_t* vt = sV + kbv * (D * 128);
#pragma unroll 2
      for (int cc = 0; cc < CPT; ++cc) {
        const int c = cpart * CPT + cc;
        const uint4 vv = *reinterpret_cast<const uint4*>(sVs + (c >> 3) * (TA_KC * 128) + sw128(krow, c & 7));
        const bf16* e = reinterpret_cast<const bf16*>(&vv);
#pragma unroll
        for (int x = 0; x < 8; ++x) *reinterpret_cast<bf16*>(vt + sw128(c * 8 + x, kl >> 3) + (kl & 7) * 2) = e[x];
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();  // V^T complete; the staging buffer is free
    if (ci + 1 < n_chunks) issue(kc + TA_KC, false, true);
    mbar_wait(&bar[0], ph_s);
    ph_s ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (ci + 1 < n_chunks) issue(kc + TA_KC, true, false);  // sK was read by the finished MMA
    // online softmax of this row's 128 scores: the chunk max first, then p = exp2(s - m)
    float mx = m;
#pragma unroll 1
    for (int c0 = 0; c0 < TA_KC; c0 += 32) {
      float v[32];
      tmem_ld32(tS + lane_base + c0, v);
#pragma unroll
      for (int x = 0; x < 32; ++x) {
        const int kp = kc + c0 + x;
        if (kp <= pos && kp < n_keys) mx = fmaxf(mx, v[x] * sl2);
      }
    }
    const float corr = (m == -INFINITY) ? 0.f : exp2f(m - mx);  // mx is finite: key kc <= pos
    m = mx;
    float ls = 0.f;
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
        ls += p0 + p1;
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
    l = l * corr + ls;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (t == 0) {  // this chunk's P V (hi + lo halves) into a fresh TMEM block
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int half = 0; half < 2; ++half)
#pragma unroll
        for (int kb = 0; kb < C::KK; ++kb) {
          const uint64_t da = umma_desc_sw128(sP + half * C::P_BYTES + kb * (TA_Q * 128));
          const uint64_t db = umma_desc_sw128(sV + kb * (D * 128));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) umma_bf16(tO, da + 2 * kk, db + 2 * kk, idO, (half | kb | kk) ? 1u : 0u);
        }
      umma_commit(&bar[1]);
    }
    mbar_wait(&bar[1], ph_o);
    ph_o ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {  // O = O * corr + P V
      float v[32];
      tmem_ld32(tO + lane_base + c0, v);
#pragma unroll
      for (int x = 0; x < 32; ++x) acc[c0 + x] = acc[c0 + x] * corr + v[x];
    }
  }
  // ---- o = O / l (one bf16 rounding); rows past n_q are not stored
  if (q0 + t < s.n_q) {
    const float il = 1.f / l;
    uint4* dst = reinterpret_cast<uint4*>(o + (size_t)(s.q_start + qi) * H + head * D);
#pragma unroll
    for (int g = 0; g < D / 8; ++g) {
      uint4 w;
      uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const __nv_bfloat162 b = __floats2bfloat162_rn(acc[8 * g + 2 * x] * il, acc[8 * g + 2 * x + 1] * il);
        wp[x] = *reinterpret_cast<const uint32_t*>(&b);
      }
      dst[g] = w;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
}

// The default prefill attention (HS_ATTN_TC=0 selects the mma.sync kernel, A/B).  Measured
// (7B layer, profiles/r02/attn_tc_ab.txt): 42 us at 512 tokens (mma.sync kernel 41 us) and
// 132 us at 2048 tokens (176 us).  Its PP-split nondeterminism (runs 43 / 45 / 47: up to 9 of
// 30 processes) was the metadata read before griddepcontrol.wait (fixed above): 30 of 30 clean
// and the full GPU suite 81 / 81 after the fix (run 49, profiles/r02/attn_tc_flaky/).
bool attn_tc_enabled() {
  static const bool on = [] {
    const char* e = getenv("HS_ATTN_TC");
    return !(e && e[0] == '0');
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
