// dstack.cu — decode stack kernel (see dstack.h for the dataflow).
//
// One CTA per SM, 12 warps:
//   warp 0  lane 0 : weight producer.  Streams the 128 x 64 weight tiles of the CTA's stream-K
//                    range of every GEMM (QKV, O, gate_up, down) of every layer, in order, into
//                    a ring of STAGES slots.  Never waits for activations.
//   warp 1         : TMEM owner; lane 0 issues tcgen05.mma (M = 128, N = BN, K = 16) per slot
//                    into one of two TMEM accumulators (one per stream-K segment).
//   warp 2  lane 0 : activation producer.  Per k-block: waits the flag of the data it needs,
//                    then TMA-loads the [BN x 64] activation tile into the same slot.  A slot
//                    is full when both producers arrived and both transfers landed.
//   warps 4-7      : epilogue.  Drain a segment's accumulator to the fp32 stream-K workspace;
//                    the last CTA to finish a tile sums the parts in part order (deterministic)
//                    and applies the fused epilogue (RoPE + paged KV write | residual | SiLU*up),
//                    then publishes the tile's flag.
//   warps 4-11     : decode attention (units of (sequence, head, KV split) per CTA, one
//                    16-token block per warp at a time, next block prefetched into L2) and
//                    every CTA's column slice of each row RMSNorm.
// Flags carry tags (launch number << 8 | layer + 1) and are compared wrap-safe, the row and
// norm counters are cumulative with per-launch bases, so nothing is reset between steps;
// per-tile arrival counters are reset by their last arriver.
//
// Numerics follow the per-kernel path: fp32 accumulation in TMEM, partial sums
// added in part order, bf16 rounding at the same points (q/k/v, RoPE outputs, attention output,
// h = x + o W_o^T, a = silu(g) u, x' = h + a W_d^T, RMSNorm outputs).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "dstack.h"
#include "tc.h"

namespace hs {

constexpr int DS_THREADS = 384;
constexpr int DS_MAXSEQ = 64;
constexpr int DS_AWARPS = 8;   // attention warps per CTA (warps 4-11)
// NC: tokens per register chunk in the tile epilogues (1 for single-sequence decode, else 8)

struct DsParams {
  int N, H, F, nh, hd, nl, G;
  float eps;
  unsigned tag0;
  int tiles[4], nkb[4], maxp[4];
  unsigned long long* ws[4];  // stream-K parts: tagged words (st_part)
  const bf16 *attn_norm, *ffn_norm;
  long long norm_stride;
  const bf16* final_norm;
  bf16* fin;
  const bf16* x_in;
  bf16 *x, *hbuf, *nrm, *q, *o, *act;
  bf16* pool;
  long long pool_stride;
  int nslots, nblocks, max_blocks;
  const int *pos, *slot, *tables;
  const SeqDesc* seqs;
  const float2* rope;
  int ch;
  int ahalf;  // attention units on half CTAs (warps 4-7 / 8-11), 2 G unit slots
  int fs;     // word stride of the flag arrays f_qkv, f_attn, f_gu, f_nrm and of c_h (1, or 32: a line each)
  float* ws_attn;
  unsigned *c_ih, *c_h, *f_qkv, *f_attn, *f_gu;
  // row norms (reading R10b): a residual tile (and the stage input pass) writes the next
  // GEMM's operand nrm = bf16(x * w) for its 128 columns and publishes f_nrm[0 / 1][tile]
  // (QKV / gate_up operand, the consuming layer's tag), plus its sum-of-squares partials
  // ssq[tile][64] and a release-add on c_rows (cumulative, launch base + count); the row scale
  // rs = 1/sqrt(sum / H + eps) multiplies the QKV / gate_up accumulators in their epilogues.
  float* ssq;
  unsigned* c_rows;
  unsigned* f_nrm[2];
  unsigned base_rows;
  unsigned long long* trace;  // optional: [G][nl][16] globaltimer stamps (hs_debug_dstack_trace)
  bf16* cap;                  // optional capture: layer l's h at cap + 2l * cap_stride, its output at (2l + 1)
  long long cap_stride;
};

// trace slots per (CTA, layer)
enum { TR_B0 = 0, TR_B1, TR_B2, TR_B3, TR_B3_END, TR_E_QKV, TR_E_ATTN, TR_E_O, TR_E_NF, TR_E_GU, TR_E_D, TR_E_NA,
       TR_A1, TR_A2, TR_A3, TR_A0, TR_O_LAST, TR_O_BAR, TR_NF_NORM, TR_D_LAST, TR_D_BAR, TR_NA_NORM,
       TR_AT_FLAGS, TR_AT_KV, TR_Q_TFULL, TR_Q_LAST, TR_Q_PUB, TR_Q_DRAIN, TR_Q_ATOM, TR_Q_VALS, TR_Q_STORES,
       TR_AT_END };
#define DS_TR(slot_)                                                                      \
  do {                                                                                    \
    if (p.trace) p.trace[((size_t)blockIdx.x * p.nl + l) * 32 + (slot_)] = gtimer();      \
  } while (0)

// Stream-K range of CTA c over W k-blocks: with W < G only the first W CTAs take (one) block
// each, so every CTA that owns part of a tile has work (the arrival counts stay exact).
__device__ __forceinline__ void ds_range(int c, long long W, int G, int& beg, int& end, int& Gk) {
  Gk = W < G ? (int)W : G;
  beg = c < Gk ? sk_begin(c, W, Gk) : 0;
  end = c < Gk ? sk_begin(c + 1, W, Gk) : 0;
}

// Cursor over a CTA's weight k-blocks in stream order (layer, GEMM kind, k-block).
struct DsIt {
  int l, k, x, beg, end;
};

__device__ __forceinline__ bool ds_it_fix(const DsParams& p, DsIt& it) {
  while (it.x >= it.end) {
    if (++it.k == 4) {
      it.k = 0;
      if (++it.l >= p.nl) return false;
    }
    int Gk;
    ds_range(blockIdx.x, (long long)p.tiles[it.k] * p.nkb[it.k], p.G, it.beg, it.end, Gk);
    it.x = it.beg;
  }
  return true;
}

__device__ __forceinline__ bool ds_it_begin(const DsParams& p, DsIt& it) {
  int Gk;
  it.l = 0;
  it.k = 0;
  ds_range(blockIdx.x, (long long)p.tiles[0] * p.nkb[0], p.G, it.beg, it.end, Gk);
  it.x = it.beg;
  return p.nl > 0 && ds_it_fix(p, it);
}

__device__ __forceinline__ bool ds_it_next(const DsParams& p, DsIt& it) {
  ++it.x;
  return ds_it_fix(p, it);
}

template <int BN, int NC>
struct DsCfg {
  static constexpr int A_BYTES = 128 * 64 * 2;
  static constexpr int B_BYTES = BN * 64 * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // smem kept for the tile epilogues is sized by the tokens a launch can hold (NC == 1: one
  // sequence), so single-sequence decode gets one more weight slot
  static constexpr int VS = NC == 1 ? 1 : BN;      // token stride of the staged tile values
  static constexpr int VALS_BYTES = 128 * VS * 4 < 64 ? 64 : 128 * VS * 4;  // RoPE pairing + Σx² scratch
  static constexpr int ROPE_BYTES = VS * 64 * 8;   // cos/sin of the call's positions (head_dim <= 128)
  static constexpr int ATT_BYTES = (2 * 8 + 8 * 128) * 4 + 128;  // attention warp merge
  static constexpr int MISC = 2048;
  static constexpr int FIT = (232448 - 1024 - MISC - VALS_BYTES - ROPE_BYTES - ATT_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = FIT > 12 ? 12 : FIT;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + VALS_BYTES + ROPE_BYTES + ATT_BYTES + 1024 + MISC;
};

__device__ __constant__ unsigned p_backoff_ns = 256;
// Weight k-blocks the producer keeps in flight as L2 prefetches beyond the shared-memory ring
// (HS_DSTACK_L2AHEAD; 0 = off): while the ring is full (the MMA waits on an activation flag) the
// prefetches keep HBM busy with the weights that come next.
__device__ __constant__ int p_l2_ahead = 0;
// Timing experiments only (HS_DSTACK_NOMMA=1, results garbage): skip the tensor-core MMAs, keep
// every barrier, load and flag, to separate MMA issue/completion cost from the memory stream.
__device__ __constant__ int p_nomma = 0;
// L2 prefetch of each attention unit's cached K / V before the unit waits for its q, k, v tiles
// (HS_DSTACK_KVPF=1; measured r02: no gain at B = 1, 2 % slower at 13B B = 16: off)
__device__ __constant__ int p_kv_prefetch = 0;
// Early reads of the held tile's later parts and residual (HS_DSTACK_EARLYPARTS=0: A/B)
__device__ __constant__ int p_early_parts = 1;
// Trace only (HS_DSTACK_TRACE_K): the GEMM kind whose stream-K fix-up the TR_Q_* stamps follow
__device__ __constant__ int p_trace_k = 0;

// Protocol-failure record (hs_debug_dstack_diag): a wait that times out writes one row per
// (CTA, warp) into mapped pinned host memory before it traps, so the host can read which wait
// of which CTA failed after the context is lost.  Row: magic, site, CTA, thread, address,
// value seen, value wanted, %globaltimer.  nullptr: no record.
__device__ __constant__ unsigned long long* p_diag = nullptr;
enum { DG_TAG = 1, DG_PART = 2, DG_PARTS = 3, DG_NLAST = 4, DG_ACT = 5 };

__device__ __noinline__ void ds_fail(int site, const void* addr, unsigned long long seen, unsigned long long want) {
  if (p_diag) {
    volatile unsigned long long* r = p_diag + ((size_t)blockIdx.x * (DS_THREADS / 32) + (threadIdx.x >> 5)) * 8;
    r[1] = (unsigned long long)site;
    r[2] = blockIdx.x;
    r[3] = threadIdx.x;
    r[4] = (unsigned long long)addr;
    r[5] = seen;
    r[6] = want;
    r[7] = gtimer();
    __threadfence_system();
    r[0] = 0xD1A6ull;
    __threadfence_system();
  }
  __trap();
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Release store of a flag: cumulative over the writes this thread observed (its CTA's writes
// ordered before it by bar.sync / __syncwarp).
__device__ __forceinline__ void publish(unsigned* f, unsigned tag) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(tag) : "memory");
}

// Waits until the flag reached `tag` (wrap-safe); traps after ~4 s (kSpinTimeout) (protocol bug: end the
// kernel rather than hang the GPU).
// Polls back off (nanosleep) so that many waiters on one flag do not saturate its L2 slice.
__device__ __noinline__ void wait_tag(const unsigned* f, unsigned tag) {
  if ((int)(ld_acquire(f) - tag) >= 0) return;
  const unsigned long long t0 = spin_clock();
  for (unsigned it = 1;; ++it) {
    __nanosleep(p_backoff_ns);
    if ((int)(ld_acquire(f) - tag) >= 0) return;
    if ((it & 255) == 0 && spin_clock() - t0 > kSpinTimeout) ds_fail(DG_TAG, f, ld_acquire(f), tag);
  }
}

// Sum of squares of one 128-row tile of the residual stream per token: thread et (0..127) holds
// row et's bf16-rounded values v[j] for tokens n0 + j; warp xor-tree, then the 4 warps in
// order.  The ONE summation used for every RMSNorm of the decode stack (stage inputs too), so
// PP = s stays bitwise equal to PP = 1.  scratch: 4 * NC floats; bar 1 (warps 4-7).
template <int NC>
__device__ __forceinline__ void ds_ssq_chunk(const float* v, int n0, int N, int et, float* scratch, float* ssq_t) {
  const int lane = et & 31, wq = et >> 5;
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    float q = v[j] * v[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    if (lane == 0) scratch[wq * NC + j] = q;
  }
  named_bar(1, 128);
  if (et < NC && n0 + et < N)
    ssq_t[n0 + et] = (scratch[et] + scratch[NC + et]) + (scratch[2 * NC + et] + scratch[3 * NC + et]);
  named_bar(1, 128);
}

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Waits (thread 0 of warps 4-11, then bar 2) until a cumulative counter reached target.
__device__ __forceinline__ void ds_wait_count(const unsigned* c, unsigned target, int t) {
  if (t == 0) wait_tag(c, target);
  named_bar(2, 256);
}

// The model's final RMSNorm (last layer of the last stage), by warps 4-11 of EVERY CTA: rs[n]
// from the tile partials (tile order, the arithmetic of ds_row_scales), then this CTA's column
// slice of y = bf16(x * rs * w) for all rows (one rounding: its consumer is the lm_head after
// the kernel).
__device__ __forceinline__ void ds_norm_slice(const DsParams& p, const bf16* __restrict__ src,
                                              const bf16* __restrict__ w, bf16* __restrict__ dst, int t, float* s_rs) {
  const int T = p.H / 128;
  if (dst) {
    {  // rs[n]: the T tile partials of row n summed lane-parallel (fixed xor tree), warp w: n = w (mod 8)
      const int wq = t >> 5, ln = t & 31;
      for (int n = wq; n < p.N; n += 8) {
        float acc = 0.f;
        for (int tt = ln; tt < T; tt += 32) acc += __ldcg(p.ssq + (size_t)tt * DS_MAXSEQ + n);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (ln == 0) s_rs[n] = 1.0f / sqrtf(acc / (float)p.H + p.eps);
      }
    }
    named_bar(2, 256);
    const int n8 = p.H >> 3;
    const int c0 = (int)((long long)blockIdx.x * n8 / p.G), c1 = (int)((long long)(blockIdx.x + 1) * n8 / p.G);
    const int w8 = c1 - c0;
    const uint4* w4 = reinterpret_cast<const uint4*>(w);
    for (int idx = t; idx < p.N * w8; idx += 256) {
      const int n = idx / w8, c = c0 + idx % w8;
      const uint4 xv = __ldcg(reinterpret_cast<const uint4*>(src) + (size_t)n * n8 + c), wv = __ldg(w4 + c);
      const float rs = s_rs[n];
      uint4 o;
      const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(&xv);
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&wv);
      __nv_bfloat162* rr = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 x = __bfloat1622float2(a[k]), g = __bfloat1622float2(b[k]);
        rr[k] = __floats2bfloat162_rn(x.x * rs * g.x, x.y * rs * g.y);
      }
      reinterpret_cast<uint4*>(dst)[(size_t)n * n8 + c] = o;
    }
  }
  named_bar(2, 256);
}

// rs[n] = 1/sqrt(sum_t ssq[t][n] / H + eps) for the N rows, by one warp: lane l sums tiles
// t = l (mod 32) in order, then a fixed xor tree (the same arithmetic as ds_norm_slice).
// Eight rows per batch with every load in flight.
__device__ __forceinline__ void ds_row_scales(const DsParams& p, float* rs, int lane) {
  const int T = p.H / 128;
  for (int n0 = 0; n0 < p.N; n0 += 8) {
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    for (int tt = lane; tt < T; tt += 32) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = n0 + j < p.N ? __ldcg(p.ssq + (size_t)tt * DS_MAXSEQ + n0 + j) : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += v[j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
      if (lane == 0 && n0 + j < p.N) rs[n0 + j] = 1.0f / sqrtf(acc[j] / (float)p.H + p.eps);
    }
  }
}

// Stream-K parts travel as tagged words: the value's bits and the layer's tag in one 8-byte
// single-copy-atomic store, so the writer needs no fence and no flag, and the tile's finisher
// polls exactly the words it sums (a stale word carries an older tag; the workspace starts
// zeroed and tags are never 0).
__device__ __forceinline__ void st_part(unsigned long long* a, float v, unsigned tag) {
  const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(w) : "memory");
}

__device__ __forceinline__ unsigned long long ld_part(const unsigned long long* a) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(a));
  return w;
}

// One attention unit: sequence i, head h, KV blocks [sp * ch, (sp + 1) * ch) of the sequence,
// by NW attention warps of a CTA (t = 0 .. 32 NW - 1, named barrier `bar`): all 8 (warps 4-11),
// or, with half-CTA units, warps 4-7 and 8-11 each run their own unit (two units per CTA, so
// a short context is split finer and each warp reads one block).  Warp w takes blocks w, w + NW, ...:
// for a 16-token block lane l loads dims [E l, E l + E) of its 16 K and 16 V rows (32
// independent loads in flight), computes the scores with warp all-reduces and keeps an online
// softmax (m, l, acc).  The warps are merged through shared memory in warp order; with several
// splits (long contexts) the partial goes to ws_attn[u] and the last split merges the splits in
// order.  The last sequence of head h publishes the head's flag.  Deterministic.
constexpr int DS_SPLIT = 64;  // KV blocks (1024 tokens) per unit

template <int D, int NW, int BAR>
__device__ __forceinline__ void ds_attn_unit(const DsParams& p, int l, unsigned tag, int i, int h, int sp, int nsp,
                                             int u, int t, float* sm, int uph, const int* s_nc, const int* s_base) {
  constexpr int NT = NW * 32;
  constexpr int E = D / 32;
  const int warp = t >> 5, lane = t & 31;
  const int H = p.nh * D;
  const SeqDesc s = p.seqs[i];
  const int n_keys = __shfl_sync(0xffffffffu, s.pos0 + 1, 0), nb = (n_keys + 15) >> 4;
  const int b0 = sp * p.ch, b1 = min(nb, b0 + p.ch);
  const int q_start = __shfl_sync(0xffffffffu, s.q_start, 0);
  const int* tab = p.tables + (size_t)i * p.max_blocks;
  // block ids of this warp's blocks (call metadata: independent of the flags, fetched first)
  const int my_blk = (b0 + warp + lane * NW < b1) ? tab[b0 + warp + lane * NW] : 0;
  if (NW == 8 && p_kv_prefetch && t >= 128) {
    // warps 8-11 reach a layer's first unit while warps 4-7 still drain its QKV (they skip that
    // epilogue): they request the unit's cached K / V slabs (4 KiB contiguous each) into L2, so
    // the attention that follows QKV reads them from L2 instead of HBM (only the new token's
    // k, v are produced by this layer; L2 stays coherent with the QKV epilogue's KV write)
    const bf16* pl = p.pool + (size_t)l * p.pool_stride;
    for (int j = t - 128; j < 2 * (b1 - b0); j += 128) {
      int blk = tab[b0 + (j >> 1)];
      if (blk < 0 || blk >= p.nblocks) blk = 0;
      const bf16* slab = pl + (((size_t)blk * 2 + (j & 1)) * p.nh + h) * 16 * D;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(slab), "r"(16 * D * 2) : "memory");
    }
  }
  if (t < 3) wait_tag(p.f_qkv + (size_t)((h * D) / 128 + t * (H / 128)) * p.fs, tag);  // q, k, v tiles of head h
  named_bar(BAR, NT);
  if (p.trace && t == 0) DS_TR(TR_AT_FLAGS);
  const float scale = 1.4426950408889634f / sqrtf((float)D);
  float qv[E];
  {
    const bf16* qp = p.q + (size_t)q_start * H + h * D + lane * E;
    if constexpr (E == 4) {
      const uint2 uu = __ldcg(reinterpret_cast<const uint2*>(qp));
      const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&uu.x));
      const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&uu.y));
      qv[0] = a.x * scale; qv[1] = a.y * scale; qv[2] = b.x * scale; qv[3] = b.y * scale;
    } else {
      const unsigned uu = __ldcg(reinterpret_cast<const unsigned*>(qp));
      const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&uu));
      qv[0] = a.x * scale; qv[1] = a.y * scale;
    }
  }
  const bf16* pool = p.pool + (size_t)l * p.pool_stride;
  const size_t vstride = (size_t)p.nh * 16 * D;
  float m = -INFINITY, lsum = 0.f, acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  using VT = typename std::conditional<E == 4, uint2, unsigned>::type;
  for (int b = b0 + warp, bi = 0; b < b1; b += NW, ++bi) {
    int blk = __shfl_sync(0xffffffffu, my_blk, bi & 31);
    if (bi >= 32) blk = tab[b];
    if (blk < 0 || blk >= p.nblocks) blk = 0;
    const bf16* kb = pool + (((size_t)blk * 2 * p.nh + h) * 16) * D + lane * E;
    if (b + NW < b1 && bi + 1 < 32) {  // the warp's next block into L2 (no registers held)
      int nblk = __shfl_sync(0xffffffffu, my_blk, bi + 1);
      if (nblk < 0 || nblk >= p.nblocks) nblk = 0;
      const char* row = reinterpret_cast<const char*>(pool + (((size_t)nblk * 2 * p.nh + h) * 16 + (lane & 15)) * D +
                                                      (lane >= 16 ? vstride : 0));
#pragma unroll
      for (int ln = 0; ln < D * 2; ln += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + ln));
    }
    VT kr[16], vr[16];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      kr[jj] = __ldcg(reinterpret_cast<const VT*>(kb + jj * D));
      vr[jj] = __ldcg(reinterpret_cast<const VT*>(kb + vstride + jj * D));
    }
    float sc[16];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      if constexpr (E == 4) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&kr[jj].x));
        const float2 cc = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&kr[jj].y));
        sc[jj] = qv[0] * a.x + qv[1] * a.y + qv[2] * cc.x + qv[3] * cc.y;
      } else {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&kr[jj]));
        sc[jj] = qv[0] * a.x + qv[1] * a.y;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) sc[jj] += __shfl_xor_sync(0xffffffffu, sc[jj], off);
    float mb = m;
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      if (b * 16 + jj >= n_keys) sc[jj] = -INFINITY;
      mb = fmaxf(mb, sc[jj]);
    }
    const float corr = exp2f(m - mb);
    lsum *= corr;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] *= corr;
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const float pj = exp2f(sc[jj] - mb);
      lsum += pj;
      if constexpr (E == 4) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vr[jj].x));
        const float2 cc = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vr[jj].y));
        acc[0] += pj * a.x; acc[1] += pj * a.y; acc[2] += pj * cc.x; acc[3] += pj * cc.y;
      } else {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vr[jj]));
        acc[0] += pj * a.x; acc[1] += pj * a.y;
      }
    }
    m = mb;
  }
  if (p.trace && t == 0) DS_TR(TR_AT_KV);
  // merge the NW warps through shared memory (warp order)
  float* sm_m = sm;           // [NW]
  float* sm_l = sm + NW;      // [NW]
  float* sm_a = sm + 2 * NW;  // [NW][D]
  if (lane == 0) { sm_m[warp] = m; sm_l[warp] = lsum; }
#pragma unroll
  for (int e = 0; e < E; ++e) sm_a[warp * D + lane * E + e] = acc[e];
  named_bar(BAR, NT);
  float M = -INFINITY, L = 0.f, A = 0.f;
  if (t < D) {
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, sm_m[w]);
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float f = sm_m[w] == -INFINITY ? 0.f : exp2f(sm_m[w] - M);
      L += sm_l[w] * f;
      A += sm_a[w * D + t] * f;
    }
  }
  bf16* orow = p.o + (size_t)q_start * H + h * D;
  if (nsp > 1) {  // long context: partial of this split (merged by the head's last unit)
    float* w = p.ws_attn + (size_t)u * (D + 4);
    if (t == 0) { w[0] = M; w[1] = L; }
    if (t < D) w[4 + t] = A;
  } else if (t < D) {
    orow[t] = __float2bfloat16_rn(A / L);
  }
  named_bar(BAR, NT);
  // one arrival per unit on the head's counter; the last unit of the head merges the splits
  // of every sequence (split order) and publishes the head
  if (t == 0) {
    if (p.trace) DS_TR(TR_AT_END);
    const unsigned old = atom_add_acq_rel(p.c_h + (size_t)h * p.fs, 1u);
    const int last = old == (unsigned)(uph - 1);
    if (last) p.c_h[(size_t)h * p.fs] = 0;
    sm_m[0] = last ? 1.f : 0.f;
  }
  named_bar(BAR, NT);
  const bool last = sm_m[0] != 0.f;
  if (last) {
    for (int i2 = 0; i2 < p.N; ++i2) {
      const int ns = s_nc[i2];
      if (ns < 2 || t >= D) continue;
      const float* w0 = p.ws_attn + (size_t)(s_base[i2] + h * ns) * (D + 4);
      float MM = -INFINITY;
      for (int k = 0; k < ns; ++k) MM = fmaxf(MM, __ldcg(w0 + (size_t)k * (D + 4)));
      float LL = 0.f, AA = 0.f;
      for (int k = 0; k < ns; ++k) {
        const float* wk = w0 + (size_t)k * (D + 4);
        const float ms = __ldcg(wk);
        const float f = ms == -INFINITY ? 0.f : exp2f(ms - MM);
        LL += __ldcg(wk + 1) * f;
        AA += __ldcg(wk + 4 + t) * f;
      }
      const int qs = p.seqs[i2].q_start;
      p.o[(size_t)qs * H + h * D + t] = __float2bfloat16_rn(AA / LL);
    }
    named_bar(BAR, NT);
    if (t == 0) {
      publish(p.f_attn + (size_t)h * p.fs, tag);
      if (p.trace && h < 64) p.trace[(size_t)p.G * p.nl * 32 + (size_t)l * 256 + 128 + h] = gtimer();
    }
  }
  named_bar(BAR, NT);  // sm reusable
}

// Slow path of an early read: the part was not written yet.  Traps after ~4 s (kSpinTimeout; protocol bug).
__device__ __noinline__ float wait_part(const unsigned long long* a, unsigned tag) {
  const unsigned long long t0 = spin_clock();
  for (;;) {
    const unsigned long long w = ld_part(a);
    if ((unsigned)(w >> 32) == tag) return __uint_as_float((unsigned)w);
    __nanosleep(64);
    if (spin_clock() - t0 > kSpinTimeout) ds_fail(DG_PART, a, w, tag);
  }
}

// a[j] += the stream-K parts p0 .. np - 1 (in part order) of tile row ml, tokens n0 + j, with
// every load of a part group in flight together (the tail of each tile is latency bound).  A
// group not written yet is re-read as a whole (one round trip per poll, not one per word);
// traps after ~4 s (kSpinTimeout) (protocol bug).
template <int NC>
__device__ __forceinline__ void ds_add_parts(const unsigned long long* tws, int p0, int np, int n0, int N, int ml,
                                             float* a, int BN, unsigned tag) {
#pragma unroll 2
  for (int pt = p0; pt < np; ++pt) {
    const unsigned long long* src = tws + ((size_t)pt * BN + n0) * 128 + ml;
    unsigned long long w[NC];
    bool ok = true;
#pragma unroll
    for (int j = 0; j < NC; ++j) w[j] = n0 + j < N ? ld_part(src + (size_t)j * 128) : (unsigned long long)tag << 32;
#pragma unroll
    for (int j = 0; j < NC; ++j) ok = ok && (unsigned)(w[j] >> 32) == tag;
    if (!ok) {
      const unsigned long long t0 = spin_clock();
      do {
        __nanosleep(64);
        if (spin_clock() - t0 > kSpinTimeout) ds_fail(DG_PARTS, src, w[0], ((unsigned long long)pt << 32) | tag);
#pragma unroll
        for (int j = 0; j < NC; ++j)
          if (n0 + j < N && (unsigned)(w[j] >> 32) != tag) w[j] = ld_part(src + (size_t)j * 128);
        ok = true;
#pragma unroll
        for (int j = 0; j < NC; ++j) ok = ok && (unsigned)(w[j] >> 32) == tag;
      } while (!ok);
    }
#pragma unroll
    for (int j = 0; j < NC; ++j) a[j] += __uint_as_float((unsigned)w[j]);
  }
}

// The epilogue warps' part of GEMM kind k (0 qkv, 1 o, 2 gate_up, 3 down) of layer l: drains
// the CTA's stream-K segments.  A tile's finisher is the owner of its first k-block: that
// segment is the last of the owner's range, so its accumulator stays in TMEM and the epilogue
// adds the later parts (tagged words, written by the CTAs whose ranges start in the tile) in
// part order.  Returns the running segment count (TMEM double-buffer phase).
template <int BN, int NC>
__device__ __forceinline__ int ds_segments(const DsParams& p, int k, int l, unsigned tag, int seg, uint32_t tmem,
                                           uint64_t* tfull, uint64_t* tempty, float* vals,
                                           int et, int lane, int quad,
                                           const int* s_pos, const int* s_slot, const float2* s_rope,
                                           const float* s_rs, const volatile unsigned* s_rs_tag) {
  const int nkb = p.nkb[k], tiles = p.tiles[k];
  const long long W = (long long)tiles * nkb;
  int beg, end, Gk;
  ds_range(blockIdx.x, W, p.G, beg, end, Gk);
  const int ml = et;
  int lastt[4], nlast = 0;
  int held_t = -1, held_buf = 0;  // the tile whose part 0 stays in TMEM
  // single-sequence decode: the held tile's later parts (and its residual) are read while its
  // own MMAs still run, so its epilogue starts without a round trip (re-read if not yet written)
  constexpr int NPRE = 8;
  unsigned long long pre[NPRE];
  float pre_r = 0.f, pre_g = 0.f;
  // O / down: the norm weight of the operand the residual epilogue writes (gate_up's ffn_norm,
  // the next layer's attn_norm; none after the stage's last layer)
  const bf16* wn = k == 1 ? p.ffn_norm + (size_t)l * p.norm_stride
                          : (k == 3 && l + 1 < p.nl ? p.attn_norm + (size_t)(l + 1) * p.norm_stride : nullptr);
  // pass 1: drain every segment of the phase
  for (int cur = beg; cur < end; ++seg) {
    const int t = cur / nkb, kb_lo = cur % nkb, kb_hi = min(nkb, kb_lo + (end - cur));
    const int buf = seg & 1;
    const int first = sk_owner((long long)t * nkb, W, Gk);
    const int np = sk_owner((long long)(t + 1) * nkb - 1, W, Gk) - first + 1;
    const int part = blockIdx.x - first;
    unsigned long long* tws = p.ws[k] + (size_t)t * p.maxp[k] * BN * 128;
    // the phase's last segment, when it starts its tile, stays in TMEM: its epilogue (pass 2,
    // right after) reads it there; every other segment is drained to the workspace
    const bool hold = part == 0 && cur + (kb_hi - kb_lo) == end;
    if constexpr (NC == 1) {
      if (hold && p_early_parts) {
#pragma unroll
        for (int q = 0; q < NPRE; ++q)
          if (q + 1 < np) pre[q] = ld_part(tws + (size_t)(q + 1) * BN * 128 + ml);
        if (k == 1 || k == 3)
          pre_r = __bfloat162float(__ldcg((k == 1 ? (l == 0 ? p.x_in : p.x) : p.hbuf) + (size_t)t * 128 + ml));
        if (wn) pre_g = __bfloat162float(__ldg(wn + (size_t)t * 128 + ml));
        // while this CTA's own MMAs finish, re-read the parts that were not written yet (one
        // round trip per probe), so the epilogue rarely pays one after them
        bool all = false;
        while (!mbar_test(&tfull[buf], (seg >> 1) & 1)) {
          if (all) continue;
          all = true;
#pragma unroll
          for (int q = 0; q < NPRE; ++q)
            if (q + 1 < np && (unsigned)(pre[q] >> 32) != tag) {
              pre[q] = ld_part(tws + (size_t)(q + 1) * BN * 128 + ml);
              all = false;
            }
        }
      }
    }
    mbar_wait(&tfull[buf], (seg >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (k == p_trace_k && et == 0 && cur == beg) DS_TR(TR_Q_TFULL);
    if (k == p_trace_k && k != 0 && et == 0 && cur + (kb_hi - kb_lo) == end) DS_TR(TR_Q_STORES);  // last segment's MMAs done
    if (hold) {
      held_t = t;
      held_buf = buf;
      if (nlast == 4) ds_fail(DG_NLAST, tws, (unsigned long long)t, (unsigned long long)k);
      lastt[nlast++] = t;
      if (k == p_trace_k && et == 0 && cur == beg) DS_TR(TR_Q_DRAIN);
      cur += kb_hi - kb_lo;
      continue;
    }
    {
      unsigned long long* dst = tws + (size_t)part * BN * 128 + ml;
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + buf * BN;
      constexpr int CH = BN < 32 ? 16 : 32;
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += CH) {
        float v[32];
        if constexpr (CH == 32) tmem_ld32(taddr + c0, v);
        else tmem_ld16(taddr + c0, v);
#pragma unroll
        for (int j = 0; j < CH; ++j)
          if (c0 + j < p.N) st_part(dst + (size_t)(c0 + j) * 128, v[j], tag);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf])) : "memory");
    const bool first_seg = cur == beg;
    if (k == p_trace_k && et == 0 && first_seg) DS_TR(TR_Q_DRAIN);
    cur += kb_hi - kb_lo;
    if (np == 1) {  // a whole tile inside the range, not its last segment
      if (nlast == 4) ds_fail(DG_NLAST, tws, (unsigned long long)t, (unsigned long long)k);
      lastt[nlast++] = t;
    }
  }
  // pass 2: the epilogues of the tiles this CTA finishes (after every drain of the phase, so a
  // CTA's later segments never wait behind its earlier tiles' epilogues)
  // (the held tile first: its TMEM buffer is released as soon as its epilogue is done)
  for (int q0 = 0; q0 < nlast; ++q0) {
    const int q = held_t >= 0 ? (q0 == 0 ? nlast - 1 : q0 - 1) : q0;
    const int t = lastt[q];
    const int first = sk_owner((long long)t * nkb, W, Gk);
    const int np = sk_owner((long long)(t + 1) * nkb - 1, W, Gk) - first + 1;
    const unsigned long long* tws = p.ws[k] + (size_t)t * p.maxp[k] * BN * 128;
    const bool held = t == held_t;
    const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(held_buf * BN);
    // the parts summed in part order from 0.f (part 0 from TMEM when held)
    auto sums = [&](int n0, float* a) {
      if (held) {
        float v0[16];
        tmem_ld16(taddr + (uint32_t)(n0 & ~15), v0);
#pragma unroll
        for (int j = 0; j < NC; ++j) a[j] = 0.f + (n0 + j < p.N ? v0[(n0 & 15) + j] : 0.f);
        if (NC == 1 && p_early_parts) {  // parts 1 .. NPRE from the early reads
#pragma unroll
          for (int q = 0; q < NPRE; ++q) {
            if (q + 1 >= np) break;
            const unsigned long long w = pre[q];
            a[0] += (unsigned)(w >> 32) == tag ? __uint_as_float((unsigned)w)
                                               : wait_part(tws + (size_t)(q + 1) * BN * 128 + ml, tag);
          }
          if (np > NPRE + 1) ds_add_parts<1>(tws, NPRE + 1, np, n0, p.N, ml, a, BN, tag);
          return;
        }
      } else {
#pragma unroll
        for (int j = 0; j < NC; ++j) a[j] = 0.f;
      }
      ds_add_parts<NC>(tws, held ? 1 : 0, np, n0, p.N, ml, a, BN, tag);
    };
    if (k == p_trace_k && et == 0) DS_TR(TR_Q_LAST);
    const int m = t * 128 + ml;
    const int H = p.H;
    const float* rs = s_rs + (k >> 1) * DS_MAXSEQ;  // QKV / gate_up: the operand's row scales (R10b)
    if (k == 0 || k == 2) {  // computed by this CTA's activation producer (warp 2) once c_rows completed
      while (s_rs_tag[k >> 1] != tag) __nanosleep(32);
      __threadfence_block();
    }
    if (k == 0) {  // bf16(rs q, rs k, rs v); RoPE of q, k; k', v -> paged pool; q' -> q
      for (int n0 = 0; n0 < p.N; n0 += NC) {
        float a[NC];
        sums(n0, a);
#pragma unroll
        for (int j = 0; j < NC; ++j)
          if (n0 + j < p.N) vals[ml * DsCfg<BN, NC>::VS + n0 + j] = __bfloat162float(__float2bfloat16_rn(rs[n0 + j] * a[j]));
      }
      named_bar(1, 128);
      if (p_trace_k == 0 && et == 0) DS_TR(TR_Q_VALS);
      const int half = p.hd >> 1;
      const int region = (t * 128) / H, r0 = (t * 128) % H;  // 0 q, 1 k, 2 v
      if (et < 64) {
        const int hl = et / half, i = et % half;
        const int ra = hl * p.hd + i, rb = ra + half;
        const int head = (r0 + ra) / p.hd;
        bf16* pool = p.pool + (size_t)l * p.pool_stride;
        for (int n = 0; n < p.N; ++n) {
          const float a = vals[ra * DsCfg<BN, NC>::VS + n], b = vals[rb * DsCfg<BN, NC>::VS + n];
          const int sl = s_slot[n];
          if (sl < 0 || sl >= p.nslots) continue;
          const size_t blk = (size_t)(sl >> 4), off = (size_t)(sl & 15);
          if (region == 2) {
            bf16* vd = pool + (((blk * 2 + 1) * p.nh + head) * 16 + off) * p.hd;
            vd[i] = __float2bfloat16_rn(a);
            vd[i + half] = __float2bfloat16_rn(b);
          } else {
            const float2 cs = s_rope[n * half + i];
            const bf16 x1 = __float2bfloat16_rn(a * cs.x - b * cs.y), x2 = __float2bfloat16_rn(b * cs.x + a * cs.y);
            bf16* d = region == 0 ? p.q + (size_t)n * H + head * p.hd
                                  : pool + (((blk * 2 + 0) * p.nh + head) * 16 + off) * p.hd;
            d[i] = x1;
            d[i + half] = x2;
          }
        }
      }
      if (p_trace_k == 0 && et == 0) DS_TR(TR_Q_STORES);
      named_bar(1, 128);
      if (et == 0) publish(p.f_qkv + (size_t)t * p.fs, tag);
      if (p_trace_k == 0 && et == 0) DS_TR(TR_Q_PUB);
      if (et == 0 && p.trace && t < 128) p.trace[(size_t)p.G * p.nl * 32 + (size_t)l * 256 + t] = gtimer();
    } else if (k == 2) {  // a = bf16(silu(g) * u): lanes 0-15 gate rows, 16-31 their up rows
      for (int n0 = 0; n0 < p.N; n0 += NC) {
        float a[NC];
        sums(n0, a);
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          a[j] *= n0 + j < p.N ? rs[n0 + j] : 1.0f;
          const float u = __shfl_xor_sync(0xffffffffu, a[j], 16);
          if (lane < 16 && n0 + j < p.N)
            p.act[(size_t)(n0 + j) * p.F + (m >> 5) * 16 + lane] = __float2bfloat16_rn(silu_f(a[j]) * u);
        }
      }
      named_bar(1, 128);
      if (k == p_trace_k && et == 0) DS_TR(TR_Q_VALS);
      if (et == 0) publish(p.f_gu + (size_t)t * p.fs, tag);
      if (k == p_trace_k && et == 0) DS_TR(TR_Q_PUB);
    } else {  // residual: h = bf16(x + o W_o^T) (k = 1) / x' = bf16(h + a W_d^T) (k = 3)
      const bf16* resid = k == 1 ? (l == 0 ? p.x_in : p.x) : p.hbuf;
      bf16* out = k == 1 ? p.hbuf : p.x;
      // the next GEMM's operand bf16(y * w) (gate_up's ffn_norm / the next layer's attn_norm)
      const float gw = !wn ? 0.f : (NC == 1 && held && p_early_parts) ? pre_g : __bfloat162float(__ldg(wn + m));
      for (int n0 = 0; n0 < p.N; n0 += NC) {
        float r[NC], a[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j)
          r[j] = n0 + j >= p.N ? 0.f
                 : (NC == 1 && held && p_early_parts) ? pre_r
                                     : __bfloat162float(__ldcg(resid + (size_t)(n0 + j) * H + m));
        sums(n0, a);
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const bf16 y = __float2bfloat16_rn(a[j] + r[j]);
          a[j] = n0 + j < p.N ? __bfloat162float(y) : 0.f;
          if (n0 + j < p.N) {
            out[(size_t)(n0 + j) * H + m] = y;
            if (wn) p.nrm[(size_t)(n0 + j) * H + m] = __float2bfloat16_rn(a[j] * gw);
            if (p.cap) p.cap[(size_t)(2 * l + (k == 3 ? 1 : 0)) * p.cap_stride + (size_t)(n0 + j) * H + m] = y;
          }
        }
        ds_ssq_chunk<NC>(a, n0, p.N, et, vals, p.ssq + (size_t)t * DS_MAXSEQ);
      }
      if (k == p_trace_k && et == 0) DS_TR(TR_Q_VALS);
      if (et == 0) red_release_add(p.c_rows, 1u);  // rows of this tile + their partial sums
      if (et == 0 && wn) publish(p.f_nrm[k == 1 ? 1 : 0] + (size_t)t * p.fs, k == 1 ? tag : tag + 1);  // consumer's layer
      if (k == p_trace_k && et == 0) DS_TR(TR_Q_PUB);
    }
    if (held) {  // every read of the held accumulator done: the MMA may reuse the buffer
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[held_buf])) : "memory");
    }
  }
  return seg;
}

template <int BN, int NC>
__global__ void __launch_bounds__(DS_THREADS, 1)
    dstack_kernel(const __grid_constant__ CUtensorMap tw0, const __grid_constant__ CUtensorMap tw1,
                  const __grid_constant__ CUtensorMap tw2, const __grid_constant__ CUtensorMap tw3,
                  const __grid_constant__ CUtensorMap tbn, const __grid_constant__ CUtensorMap tbo,
                  const __grid_constant__ CUtensorMap tba, const __grid_constant__ DsParams p) {
  using C = DsCfg<BN, NC>;
  PDL_LAUNCH();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* vals = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES);
  float2* s_rope = reinterpret_cast<float2*>(smem + C::STAGES * C::STAGE_BYTES + C::VALS_BYTES);
  float* s_att = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES + C::VALS_BYTES + C::ROPE_BYTES);
  uint8_t* misc = smem + C::STAGES * C::STAGE_BYTES + C::VALS_BYTES + C::ROPE_BYTES + C::ATT_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(misc);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);                                // [8]
  int* s_nc = reinterpret_cast<int*>(red + 8);                                         // [64]
  int* s_base = s_nc + DS_MAXSEQ;                                                      // [65]
  int* s_pos = s_base + DS_MAXSEQ + 4;                                                 // [64]
  int* s_slot = s_pos + DS_MAXSEQ;                                                     // [64]
  volatile int* s_prog = s_slot + DS_MAXSEQ;                                           // [1] k-blocks issued
  volatile unsigned* s_rs_tag = reinterpret_cast<volatile unsigned*>(s_prog + 1);       // [2] tag of s_rs[0 / 1]
  float* s_rs = reinterpret_cast<float*>(const_cast<int*>(s_prog) + 4);                // [2][64] row scales
  static_assert(DsCfg<BN, NC>::STAGES * 16 + 32 + 16 + 32 + (64 + 68 + 64 + 64 + 4 + 128) * 4 <= DsCfg<BN, NC>::MISC,
                "misc shared memory");
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int G = p.G;

  if (threadIdx.x == 0) {
    *s_prog = 0;
    s_rs_tag[0] = 0;
    s_rs_tag[1] = 0;
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 2); mbar_init(&empty[s], 1); }
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
    if (lane == 0) {  // ---- weight producer (independent of every earlier kernel and flag)
      const CUtensorMap* wm[4] = {&tw0, &tw1, &tw2, &tw3};
      DsIt ld;
      bool ld_ok = ds_it_begin(p, ld);
      for (int i = 0; ld_ok; ++i) {
        const int s = i % C::STAGES;
        mbar_wait(&empty[s], ((i / C::STAGES) & 1) ^ 1);
        const int l = ld.l, k = ld.k, x = ld.x;
        if (x == ld.beg && p.trace) DS_TR(k == 0 ? TR_A0 : TR_A1 + k - 1);
        mbar_expect_tx(&full[s], C::A_BYTES);
        tma_load_w3(wm[k], &full[s], smem + s * C::STAGE_BYTES, x, l);  // tiled: block x = tile * nkb + kb
        *s_prog = i + 1;  // progress for the L2 prefetcher (warp 3)
        ld_ok = ds_it_next(p, ld);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc = instr_desc<BN>();
      const bool nomma = p_nomma != 0;
      int i = 0, seg = 0;
      for (int l = 0; l < p.nl; ++l)
        for (int k = 0; k < 4; ++k) {
          const int nkb = p.nkb[k];
          const long long W = (long long)p.tiles[k] * nkb;
          int beg, end, Gk;
          ds_range(blockIdx.x, W, G, beg, end, Gk);
          for (int cur = beg; cur < end; ++seg) {
            const int kb_lo = cur % nkb, kb_hi = min(nkb, kb_lo + (end - cur));
            const int buf = seg & 1;
            mbar_wait(&tempty[buf], ((seg >> 1) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t acc = tmem + buf * BN;
            for (int kb = kb_lo; kb < kb_hi; ++kb, ++i) {
              const int s = i % C::STAGES;
              mbar_wait(&full[s], (i / C::STAGES) & 1);
              asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
              const uint8_t* sa = smem + s * C::STAGE_BYTES;
              const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + C::A_BYTES);
              if (!nomma) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  umma_bf16(acc, da + 2 * kk, db + 2 * kk, idesc, (kb > kb_lo || kk > 0) ? 1u : 0u);
              }
              umma_commit(&empty[s]);
            }
            umma_commit(&tfull[buf]);
            cur += kb_hi - kb_lo;
          }
        }
    }
  } else if (warp == 3) {
    // ---- optional L2 prefetcher (HS_DSTACK_L2AHEAD = d > 0): keeps the k-blocks
    // [loaded + STAGES, loaded + STAGES + d) of this CTA's weight stream requested into L2, so
    // HBM keeps streaming while the ring is full and the MMA waits on an activation flag
    const int ahead = p_l2_ahead;
    if (ahead > 0 && lane == 0) {
      const CUtensorMap* wm[4] = {&tw0, &tw1, &tw2, &tw3};
      DsIt pf;
      bool pf_ok = ds_it_begin(p, pf);
      for (int j = 0; j < C::STAGES && pf_ok; ++j) pf_ok = ds_it_next(p, pf);
      for (int i = C::STAGES; pf_ok; ++i) {
        while (i >= *s_prog + C::STAGES + ahead) __nanosleep(128);
        tma_prefetch_4d(wm[pf.k], 0, 0, pf.x, pf.l);
        pf_ok = ds_it_next(p, pf);
      }
    }
  } else if (warp == 2) {
    // ---- activation producer: flag-gated.  The whole warp polls up to 32 k-blocks' flags at
    // once (one L2 round trip per poll instead of one per k-block); lane 0 issues the TMA loads
    // of the ready prefix in order.
    PDL_WAIT();
    const CUtensorMap* bm[4] = {&tbn, &tbo, &tbn, &tba};
    int i = 0;
    for (int l = 0; l < p.nl; ++l) {
      const unsigned tag = p.tag0 + l;
      for (int k = 0; k < 4; ++k) {
        const int nkb = p.nkb[k];
        const long long W = (long long)p.tiles[k] * nkb;
        int beg, end, Gk;
        ds_range(blockIdx.x, W, G, beg, end, Gk);
        if (beg == end) continue;
        for (int x0 = beg; x0 < end; x0 += 32) {
          const int cnt = min(32, end - x0);
          const int kbl = (x0 + lane) % nkb;
          // QKV / gate_up: the operand tile (128 columns = 2 k-blocks) of the residual tile that
          // produced it; O: the head; down: the gate_up tile
          const unsigned* f = (k == 1 ? p.f_attn + (size_t)((kbl * 64) / p.hd) * p.fs
                               : k == 3 ? p.f_gu + (size_t)kbl * p.fs : p.f_nrm[k >> 1] + (size_t)(kbl >> 1) * p.fs);
          int issued = 0;
          unsigned long long t_spin = 0;
          while (issued < cnt) {
            bool ok = lane < issued || lane >= cnt;
            if (!ok) ok = (int)(ld_acquire(f) - tag) >= 0;
            const unsigned mask = __ballot_sync(0xffffffffu, ok);
            const int upto = min(cnt, mask == 0xffffffffu ? 32 : __ffs(~mask) - 1);
            __syncwarp();
            if (upto > issued) {
              if (lane == 0) {
                if (p.trace && x0 == beg && issued == 0) DS_TR(k);
                asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> TMA reads
                for (int q = issued; q < upto; ++q) {
                  const int ii = i + (x0 - beg) + q;
                  const int s = ii % C::STAGES;
                  mbar_wait(&empty[s], ((ii / C::STAGES) & 1) ^ 1);
                  mbar_expect_tx(&full[s], C::B_BYTES);
                  tma_load_2d(bm[k], &full[s], smem + s * C::STAGE_BYTES + C::A_BYTES, ((x0 + q) % nkb) * 64, 0);
                }
              }
              issued = upto;
            } else {
              __nanosleep(p_backoff_ns);
              if (t_spin == 0) t_spin = spin_clock();
              else if (spin_clock() - t_spin > kSpinTimeout)
                ds_fail(DG_ACT, f, ld_acquire(f), ((unsigned long long)(l * 4 + k) << 32) | tag);
            }
          }
        }
        i += end - beg;
        if (k == 3 && lane == 0) DS_TR(TR_B3_END);
        if (k == 0 || k == 2) {
          // the row scales of this operand for the QKV / gate_up epilogues (they run after this
          // CTA's last k-block of the phase): every residual tile's partials are in once c_rows
          // reached the event's count (events: stage input, then O / down of each layer)
          const int T = p.H / 128;
          if (lane == 0) wait_tag(p.c_rows, p.base_rows + (unsigned)T * (unsigned)(2 * l + (k == 0 ? 1 : 2)));
          __syncwarp();
          ds_row_scales(p, s_rs + (k >> 1) * DS_MAXSEQ, lane);
          __syncwarp();
          __threadfence_block();
          if (lane == 0) s_rs_tag[k >> 1] = tag;
        }
      }
    }
  } else if (warp >= 4) {
    // ---- epilogue (warps 4-7), attention + row norms (warps 4-11)
    PDL_WAIT();
    const bool epi = warp < 8;
    const int t256 = threadIdx.x - 128;
    const int quad = warp & 3;
    const int aw = warp - 4;
    if (t256 == 0) {
      int b = 0;
      for (int i = 0; i < p.N; ++i) {
        const int nb = (p.seqs[i].pos0 + 1 + 15) >> 4;
        const int nc = (nb + p.ch - 1) / p.ch;
        s_nc[i] = nc;
        s_base[i] = b;
        b += p.nh * nc;
      }
      s_base[p.N] = b;
    }
    {  // the call's positions, KV slots and RoPE rows (read by the QKV epilogues of every layer)
      const int half = p.hd >> 1;
      if (t256 < p.N) {
        s_pos[t256] = p.pos[t256];
        s_slot[t256] = p.slot[t256];
      }
      for (int idx = t256; idx < p.N * half; idx += 256)
        s_rope[idx] = p.rope[(size_t)p.pos[idx / half] * half + idx % half];
    }
    named_bar(2, 256);
    const int total = __shfl_sync(0xffffffffu, s_base[p.N], 0);
    int seg = 0;
    // One call site per routine (they are inlined into a warp-uniform context and their code
    // stays resident in the instruction cache): step (l, k) = [pending row norm] -> GEMM k's
    // segments (epilogue warps) -> attention (k = 0) -> grid-last check (k = 1, 3).
    const int T = p.H / 128;
    {  // the stage input (layer 0's QKV operand): CTA c < T writes tile c of bf16(x_in * w) and
       // its partial sums of squares, as a residual tile does for the later layers
      if (blockIdx.x < T && epi) {
        const int m = blockIdx.x * 128 + t256;
        const float gw = __bfloat162float(__ldg(p.attn_norm + m));
        for (int n0 = 0; n0 < p.N; n0 += NC) {
          float v[NC];
#pragma unroll
          for (int j = 0; j < NC; ++j) {
            v[j] = n0 + j < p.N ? __bfloat162float(__ldcg(p.x_in + (size_t)(n0 + j) * p.H + m)) : 0.f;
            if (n0 + j < p.N) p.nrm[(size_t)(n0 + j) * p.H + m] = __float2bfloat16_rn(v[j] * gw);
          }
          ds_ssq_chunk<NC>(v, n0, p.N, t256, vals, p.ssq + (size_t)blockIdx.x * DS_MAXSEQ);
        }
        if (t256 == 0) {
          red_release_add(p.c_rows, 1u);
          publish(p.f_nrm[0] + (size_t)blockIdx.x * p.fs, p.tag0);
        }
      }
      const int l = 0;
      if (t256 == 0) DS_TR(TR_E_NA);
    }
    for (int step = 0; step < 4 * p.nl; ++step) {
      const int l = step >> 2, k = step & 3;
      const unsigned tag = p.tag0 + l;
      if (k == 0 && t256 < 2) {  // this CTA's column slices of the layer's two norm vectors into L2
        const bf16* w = t256 == 0 ? p.ffn_norm + (size_t)l * p.norm_stride
                                  : (l + 1 < p.nl ? p.attn_norm + (size_t)(l + 1) * p.norm_stride : p.final_norm);
        if (w) {
          const int n8 = p.H >> 3;
          const int c0 = (int)((long long)blockIdx.x * n8 / p.G), c1 = (int)((long long)(blockIdx.x + 1) * n8 / p.G);
          for (int c = c0 & ~7; c < c1; c += 8) asm volatile("prefetch.global.L2 [%0];" ::"l"(w + (size_t)c * 8));
        }
      }
      if (epi) seg = ds_segments<BN, NC>(p, k, l, tag, seg, tmem, tfull, tempty, vals, t256, lane, quad,
                                     s_pos, s_slot, s_rope, s_rs, s_rs_tag);
      if (t256 == 0) DS_TR(TR_E_QKV + (k == 0 ? 0 : k == 1 ? 2 : k == 2 ? 4 : 5));
      if (k == 0) {
        // units (seq, head, split) over the CTAs; every CTA (half CTA) loops uniformly
        // (compiled into the batched kernels only: in the single-sequence kernel the extra code
        // alone cost 1 % — instruction-cache footprint of the phase loop)
        if (NC > 1 && p.ahalf) {  // warps 4-7 (barrier 1) and 8-11 (barrier 3) run units u = c, c + G (mod 2G)
          const int g = t256 >> 7, tg = t256 & 127;
          float* smg = s_att + g * (2 * 4 + 4 * 128);
          for (int u = blockIdx.x + g * G; u < total; u += 2 * G) {
            int i = 0;
            while (i + 1 < p.N && s_base[i + 1] <= u) ++i;
            i = __shfl_sync(0xffffffffu, i, 0);
            const int nsp = __shfl_sync(0xffffffffu, s_nc[i], 0), r = u - __shfl_sync(0xffffffffu, s_base[i], 0);
            if (p.hd == 128) {
              if (g) ds_attn_unit<128, 4, 3>(p, l, tag, i, r / nsp, r % nsp, nsp, u, tg, smg, total / p.nh, s_nc, s_base);
              else ds_attn_unit<128, 4, 1>(p, l, tag, i, r / nsp, r % nsp, nsp, u, tg, smg, total / p.nh, s_nc, s_base);
            } else {
              if (g) ds_attn_unit<64, 4, 3>(p, l, tag, i, r / nsp, r % nsp, nsp, u, tg, smg, total / p.nh, s_nc, s_base);
              else ds_attn_unit<64, 4, 1>(p, l, tag, i, r / nsp, r % nsp, nsp, u, tg, smg, total / p.nh, s_nc, s_base);
            }
          }
        } else {
          for (int u = blockIdx.x; u < total; u += G) {
            int i = 0;
            while (i + 1 < p.N && s_base[i + 1] <= u) ++i;
            i = __shfl_sync(0xffffffffu, i, 0);
            const int nsp = __shfl_sync(0xffffffffu, s_nc[i], 0), r = u - __shfl_sync(0xffffffffu, s_base[i], 0);
            if (p.hd == 128)
              ds_attn_unit<128, 8, 2>(p, l, tag, i, r / nsp, r % nsp, nsp, u, t256, s_att, total / p.nh, s_nc, s_base);
            else
              ds_attn_unit<64, 8, 2>(p, l, tag, i, r / nsp, r % nsp, nsp, u, t256, s_att, total / p.nh, s_nc, s_base);
          }
        }
        if (t256 == 0) DS_TR(TR_E_ATTN);
      } else if (k == 3 && l + 1 == p.nl && p.final_norm) {  // the model's final norm (event 2l+2)
        ds_wait_count(p.c_rows, p.base_rows + (unsigned)T * (unsigned)(2 * l + 3), t256);
        if (t256 == 0) DS_TR(TR_D_LAST);
        ds_norm_slice(p, p.x, p.final_norm, p.fin, t256, s_att);
        if (t256 == 0) DS_TR(TR_E_NA);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)C::TMEM_COLS));
}

// ------------------------------------------------------------------ host side -----------
struct DstackState {
  int device = 0, G = 0;
  int H = 0, F = 0, nh = 0, hd = 0, max_seqs = 0, bn_max = 16;
  int tiles[4] = {}, nkb[4] = {}, maxp[4] = {};
  unsigned long long* ws = nullptr;  // stream-K parts (tagged words), per GEMM kind at ws_off[k]
  size_t ws_off[4] = {};
  float* ws_attn = nullptr;
  size_t attn_items_max = 0;
  unsigned* ctr = nullptr;
  size_t ctr_words = 0;
  unsigned seq_no = 0;
  float* ssq = nullptr;                 // [H / 128][64] row sum-of-squares partials
  unsigned base_rows = 0;  // cumulative c_rows value at the next launch
};

// Protocol-failure rows (p_diag), mapped pinned host memory, and the address map of the
// latest launch to name the region a failed wait polled (hs_debug_dstack_diag)
static constexpr size_t kDiagRows = (size_t)160 * (DS_THREADS / 32);
static unsigned long long* g_diag_host = nullptr;
struct DiagRegion {
  const char* name;
  unsigned long long lo, hi, stride;
};
struct DiagState {
  const void* state;
  DiagRegion map[16];
  int nmap;
  unsigned tag0, base_rows;
};
static DiagState g_diag[16];  // per DstackState (stages sharing a device), latest launch each

// HS debug: per-CTA phase timestamps of the last launch (hs_debug_dstack_trace)
static unsigned long long* g_ds_trace = nullptr;
static constexpr size_t kTraceWords = (size_t)148 * 2 * 256 * 32;

static int max_parts(int tiles, int nkb, int G) {
  const long long W = (long long)tiles * nkb;
  if (W < G) G = (int)W;
  int mp = 1;
  for (int t = 0; t < tiles; ++t)
    mp = std::max(mp, sk_owner((long long)(t + 1) * nkb - 1, W, G) - sk_owner((long long)t * nkb, W, G) + 1);
  return mp;
}

bool dstack_supported(int N, int hd) {
  static int on = [] {
    const char* e = getenv("HS_DSTACK");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return on && N >= 1 && N <= DS_MAXSEQ && (hd == 64 || hd == 128);
}

hs_status dstack_create(DstackState** out, int H, int F, int nh, int hd, int max_seqs, int max_ctx, cudaStream_t st) {
  DstackState* s = new DstackState();
  HS_CUDA(cudaGetDevice(&s->device));
  s->G = num_sms(s->device);
  s->H = H; s->F = F; s->nh = nh; s->hd = hd; s->max_seqs = std::min(max_seqs, DS_MAXSEQ);
  s->bn_max = gemm_bn(std::max(1, s->max_seqs));
  const int M[4] = {3 * H, H, 2 * F, H}, K[4] = {H, H, H, F};
  size_t off = 0;
  for (int k = 0; k < 4; ++k) {
    s->tiles[k] = M[k] / 128;
    s->nkb[k] = K[k] / 64;
    s->maxp[k] = max_parts(s->tiles[k], s->nkb[k], s->G);
    s->ws_off[k] = off;
    off += align_up((size_t)s->tiles[k] * s->maxp[k] * s->bn_max * 128, 64);
  }
  cudaError_t e = cudaMalloc(&s->ws, off * 8);
  // zeroed in stream order before the first launch (dstack.h): no word carries a tag yet
  if (e == cudaSuccess) e = cudaMemsetAsync(s->ws, 0, off * 8, st);

  s->attn_items_max = std::max((size_t)(s->max_seqs > 1 ? 2 : 1) * s->G, (size_t)s->max_seqs * nh * ((std::max(max_ctx, 1) + 16 * DS_SPLIT - 1) / (16 * DS_SPLIT)));
  if (e == cudaSuccess) e = cudaMalloc(&s->ws_attn, s->attn_items_max * (hd + 4) * 4);
  s->ctr_words = 4096 + (size_t)DS_MAXSEQ * nh + 4 * (size_t)(s->tiles[0] + s->tiles[1] + s->tiles[2] + s->tiles[3]) +
                 32 * (size_t)(s->tiles[0] + s->tiles[2] + 2 * nh + 2 * (H / 128) + 8);  // padded flags (HS_DSTACK_FLAGPAD)
  if (e == cudaSuccess) e = cudaMalloc(&s->ctr, s->ctr_words * 4);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->ctr, 0, s->ctr_words * 4, st);
  if (e == cudaSuccess) e = cudaMalloc(&s->ssq, (size_t)(H / 128) * DS_MAXSEQ * 4);
  if (e != cudaSuccess) {
    dstack_destroy(s);
    HS_FAIL(e == cudaErrorMemoryAllocation ? HS_E_OOM : HS_E_CUDA, "dstack workspace: %s", cudaGetErrorString(e));
  }
  *out = s;
  return HS_OK;
}

void dstack_destroy(DstackState* s) {
  if (!s) return;
  DeviceGuard dg(s->device);
  if (s->ws) cudaFree(s->ws);

  if (s->ws_attn) cudaFree(s->ws_attn);
  if (s->ctr) cudaFree(s->ctr);
  if (s->ssq) cudaFree(s->ssq);
  delete s;
}

template <int BN, int NC>
static hs_status launch_bn(DstackState* s, const DstackArgs& a, const DsParams& p, int bi, cudaStream_t st) {
  using C = DsCfg<BN, NC>;
  static bool attr_set[64] = {};
  if (s->device < 64 && !attr_set[s->device]) {
    HS_CUDA(cudaFuncSetAttribute(dstack_kernel<BN, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set[s->device] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(s->G);
  cfg.blockDim = dim3(DS_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (they wait on each other's flags)
  at[na].val.cooperative = 1;
  ++na;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  HS_CUDA(cudaLaunchKernelEx(&cfg, dstack_kernel<BN, NC>, a.wqkv->map, a.wo->map, a.wgu->map, a.wd->map, a.b_nrm[bi].map,
                             a.b_o[bi].map, a.b_act[bi].map, p));
  count_launch();
  return HS_OK;
}

hs_status dstack_launch(DstackState* s, const DstackArgs& a, cudaStream_t st) {
  if (!dstack_supported(a.N, a.hd) || a.N > s->max_seqs || a.H != s->H || a.F != s->F || a.nh != s->nh ||
      a.hd != s->hd || a.nl < 1 || a.nl > 255 || a.H / 128 > s->G)
    HS_FAIL(HS_E_INVAL, "dstack: unsupported call (N=%d nl=%d)", a.N, a.nl);
  const int BN = gemm_bn(a.N);
  if (BN > s->bn_max) HS_FAIL(HS_E_INVAL, "dstack: N=%d above the workspace's tile width", a.N);
  int bi = 0;
  while (gemm_bn_value(bi) != BN) ++bi;
  if (a.b_nrm[bi].box_rows != BN || a.b_o[bi].box_rows != BN || a.b_act[bi].box_rows != BN)
    HS_FAIL(HS_E_INVAL, "dstack: activation TMA box mismatch");
  DsParams p{};
  p.N = a.N; p.H = a.H; p.F = a.F; p.nh = a.nh; p.hd = a.hd; p.nl = a.nl; p.G = s->G; p.eps = a.eps;
  if (++s->seq_no >= (1u << 24)) s->seq_no = 1;  // tags stay wrap-safe: flags are compared by difference
  p.tag0 = (s->seq_no << 8) + 1;
  for (int k = 0; k < 4; ++k) {
    p.tiles[k] = s->tiles[k];
    p.nkb[k] = s->nkb[k];
    p.maxp[k] = s->maxp[k];
    p.ws[k] = s->ws + s->ws_off[k];
  }
  p.attn_norm = a.attn_norm; p.ffn_norm = a.ffn_norm; p.norm_stride = a.norm_stride;
  p.final_norm = a.final_norm; p.fin = a.fin;
  p.x_in = a.x_in; p.x = a.x; p.hbuf = a.hbuf; p.nrm = a.nrm; p.q = a.q; p.o = a.o; p.act = a.act;
  p.pool = a.pool; p.pool_stride = a.pool_stride; p.nslots = a.nslots; p.nblocks = a.nblocks;
  p.max_blocks = a.max_blocks; p.pos = a.pos; p.slot = a.slot; p.tables = a.tables; p.seqs = a.seqs; p.rope = a.rope;
  {  // KV blocks per attention unit: the smallest split that keeps the units within one wave
     // of CTAs (short contexts use more SMs), at most DS_SPLIT; a function of the shapes only
    auto units_of = [&](int ch) {
      size_t u = 0;
      for (int i = 0; i < a.N; ++i) u += (size_t)a.nh * (((a.ctx[i] + 15) / 16 + ch - 1) / ch);
      return u;
    };
    static const int min_ch = [] {  // A/B knob: fewer, longer units (HS_DSTACK_MINCH=64: one unit per head)
      const char* e = getenv("HS_DSTACK_MINCH");
      return e && atoi(e) > 0 ? std::min(atoi(e), DS_SPLIT) : 1;
    }();
    int ch = min_ch;
    // half-CTA units for batches (13B B = 16: 7.87 -> 7.61 ms); a single sequence keeps 8-warp
    // units (2.78 -> 2.79 ms with half units, profiles/r02/dstack_ab/b31_*).  HS_DSTACK_AHALF=0/1
    // forces either (A/B)
    static const int ahalf_env = [] {
      const char* e = getenv("HS_DSTACK_AHALF");
      return e ? atoi(e) : -1;
    }();
    const int ahalf = ahalf_env >= 0 ? (ahalf_env != 0) : (a.N > 1);
    p.ahalf = ahalf;
    const size_t slots = (size_t)s->G * (ahalf ? 2 : 1);
    while (ch < DS_SPLIT && units_of(ch) > slots) ++ch;
    if (units_of(ch) > s->attn_items_max) HS_FAIL(HS_E_INVAL, "dstack: context longer than the workspace was sized for");
    p.ch = ch;
  }
  p.ws_attn = s->ws_attn;
  p.cap = a.cap;
  p.cap_stride = a.cap_stride;
  {
    static bool bo_set[64] = {};
    if (s->device < 64 && !bo_set[s->device]) {
      const char* e = getenv("HS_DSTACK_BACKOFF");
      const unsigned ns = e ? (unsigned)atoi(e) : 256u;
      HS_CUDA(cudaMemcpyToSymbol(p_backoff_ns, &ns, sizeof(ns)));
      const char* e2 = getenv("HS_DSTACK_L2AHEAD");
      const int ahead = e2 ? atoi(e2) : 0;
      HS_CUDA(cudaMemcpyToSymbol(p_l2_ahead, &ahead, sizeof(ahead)));
      const char* e4 = getenv("HS_DSTACK_KVPF");
      const int kvpf = e4 ? atoi(e4) : 0;
      HS_CUDA(cudaMemcpyToSymbol(p_kv_prefetch, &kvpf, sizeof(kvpf)));
      const char* e6 = getenv("HS_DSTACK_EARLYPARTS");
      const int ep = e6 ? atoi(e6) : 1;
      HS_CUDA(cudaMemcpyToSymbol(p_early_parts, &ep, sizeof(ep)));
      const char* e5 = getenv("HS_DSTACK_TRACE_K");
      const int tk = e5 ? atoi(e5) : 0;
      HS_CUDA(cudaMemcpyToSymbol(p_trace_k, &tk, sizeof(tk)));
      const char* e3 = getenv("HS_DSTACK_NOMMA");
      const int nomma = e3 ? atoi(e3) : 0;
      HS_CUDA(cudaMemcpyToSymbol(p_nomma, &nomma, sizeof(nomma)));
      if (!g_diag_host) {
        HS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&g_diag_host), kDiagRows * 64, cudaHostAllocMapped | cudaHostAllocPortable));
        memset(g_diag_host, 0, kDiagRows * 64);
      }
      unsigned long long* dptr = nullptr;
      HS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dptr), g_diag_host, 0));
      HS_CUDA(cudaMemcpyToSymbol(p_diag, &dptr, sizeof(dptr)));
      bo_set[s->device] = true;
    }
  }
  p.trace = g_ds_trace && (size_t)s->G * a.nl * 32 + (size_t)a.nl * 256 <= kTraceWords ? g_ds_trace : nullptr;
  unsigned* c = s->ctr;
  size_t o = 0;
  p.c_ih = c + o; o += (size_t)DS_MAXSEQ * s->nh;
  // one 128-byte line per flag for a single sequence (7B B = 1: 2.711 -> 2.690 ms), packed for
  // batches (13B B = 16: 7.60 vs 7.64 ms padded; profiles/r02/dstack_ab/b35_*).  Stale words of
  // the other layout carry older tags (tags grow every launch), so switching is safe.
  // HS_DSTACK_FLAGPAD=1/32 forces either (A/B)
  static const int fs_env = [] {
    const char* e = getenv("HS_DSTACK_FLAGPAD");
    return e ? atoi(e) : 0;
  }();
  const int fs = fs_env == 1 || fs_env == 32 ? fs_env : (a.N == 1 ? 32 : 1);
  p.fs = fs;
  // every region is sized for the padded layout, so no array moves when the stride changes
  // (c_rows is cumulative across launches and must stay put)
  o = align_up(o, 32);
  p.c_rows = c + o; o += 32;
  p.c_h = c + o; o += (size_t)s->nh * 32;
  p.f_nrm[0] = c + o; o += (size_t)(s->H / 128) * 32;
  p.f_nrm[1] = c + o; o += (size_t)(s->H / 128) * 32;
  p.f_qkv = c + o; o += (size_t)s->tiles[0] * 32;
  p.f_attn = c + o; o += (size_t)s->nh * 32;
  p.f_gu = c + o; o += (size_t)s->tiles[2] * 32;
  p.ssq = s->ssq;
  p.base_rows = s->base_rows;
  s->base_rows += (unsigned)(s->H / 128) * (unsigned)(2 * a.nl + 1);
  if (o > s->ctr_words) HS_FAIL(HS_E_INVAL, "dstack: counter layout overflow");
  {  // address map for hs_debug_dstack_diag (host bookkeeping only)
    auto reg = [](const char* n, const void* lo, size_t words, size_t wb, size_t stride) {
      const unsigned long long b = (unsigned long long)(uintptr_t)lo;
      return DiagRegion{n, b, b + words * wb, stride};
    };
    int si = 0;
    while (si < 15 && g_diag[si].state && g_diag[si].state != s) ++si;
    DiagState& d = g_diag[si];
    d.state = s;
    DiagRegion* g_diag_map = d.map;
    int m = 0;
    g_diag_map[m++] = reg("c_rows", p.c_rows, 1, 4, 4);
    g_diag_map[m++] = reg("c_h", p.c_h, (size_t)s->nh * 32, 4, 4 * fs);
    g_diag_map[m++] = reg("f_nrm0", p.f_nrm[0], (size_t)(s->H / 128) * 32, 4, 4 * fs);
    g_diag_map[m++] = reg("f_nrm1", p.f_nrm[1], (size_t)(s->H / 128) * 32, 4, 4 * fs);
    g_diag_map[m++] = reg("f_qkv", p.f_qkv, (size_t)s->tiles[0] * 32, 4, 4 * fs);
    g_diag_map[m++] = reg("f_attn", p.f_attn, (size_t)s->nh * 32, 4, 4 * fs);
    g_diag_map[m++] = reg("f_gu", p.f_gu, (size_t)s->tiles[2] * 32, 4, 4 * fs);
    g_diag_map[m++] = reg("c_ih", p.c_ih, (size_t)DS_MAXSEQ * s->nh, 4, 4);
    static const char* wsn[4] = {"ws_qkv", "ws_o", "ws_gu", "ws_d"};
    for (int k = 0; k < 4; ++k)
      g_diag_map[m++] = reg(wsn[k], p.ws[k], (size_t)s->tiles[k] * s->maxp[k] * s->bn_max * 128, 8,
                            (size_t)s->maxp[k] * s->bn_max * 128 * 8);
    d.nmap = m;
    d.tag0 = p.tag0;
    d.base_rows = p.base_rows;
  }
  switch (BN) {
    case 16: return a.N == 1 ? launch_bn<16, 1>(s, a, p, bi, st) : launch_bn<16, 8>(s, a, p, bi, st);
    case 32: return launch_bn<32, 8>(s, a, p, bi, st);
    default: return launch_bn<64, 8>(s, a, p, bi, st);
  }
}

void warm_dstack() {
  cudaFuncAttributes at;
  cudaFuncSetAttribute(dstack_kernel<16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, DsCfg<16, 1>::SMEM);
  cudaFuncSetAttribute(dstack_kernel<16, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, DsCfg<16, 8>::SMEM);
  cudaFuncSetAttribute(dstack_kernel<32, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, DsCfg<32, 8>::SMEM);
  cudaFuncSetAttribute(dstack_kernel<64, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, DsCfg<64, 8>::SMEM);
  cudaFuncGetAttributes(&at, dstack_kernel<16, 1>);
  cudaFuncGetAttributes(&at, dstack_kernel<16, 8>);
  cudaFuncGetAttributes(&at, dstack_kernel<32, 8>);
  cudaFuncGetAttributes(&at, dstack_kernel<64, 8>);
}

}  // namespace hs

extern "C" int32_t hs_debug_dstack_diag(int32_t print) {
  using namespace hs;
  if (!g_diag_host) return 0;
  int n = 0;
  for (size_t r = 0; r < kDiagRows; ++r) {
    const volatile unsigned long long* w = g_diag_host + r * 8;
    if (w[0] != 0xD1A6ull) continue;
    ++n;
    if (!print) continue;
    static const char* sites[] = {"?", "wait_tag", "wait_part", "add_parts", "nlast", "act_flag"};
    const unsigned long long a = w[4];
    const char* reg = "?";
    long long idx = -1;
    int st = -1;
    for (int si = 0; si < 16; ++si)
      for (int m = 0; m < g_diag[si].nmap; ++m)
        if (a >= g_diag[si].map[m].lo && a < g_diag[si].map[m].hi) {
          reg = g_diag[si].map[m].name;
          idx = (long long)((a - g_diag[si].map[m].lo) / g_diag[si].map[m].stride);
          st = si;
        }
    fprintf(stderr,
            "dstack diag: site=%s cta=%llu thread=%llu region=%s[%lld] seen=0x%llx want=0x%llx t=%llu "
            "(state %d, its last launch tag0=0x%x base_rows=%u)\n",
            sites[w[1] < 6 ? w[1] : 0], w[2], w[3], reg, idx, w[5], w[6], w[7], st, st >= 0 ? g_diag[st].tag0 : 0u,
            st >= 0 ? g_diag[st].base_rows : 0u);
    g_diag_host[r * 8] = 0;  // each record is reported once
  }
  return n;
}

extern "C" hs_status hs_debug_dstack_trace(int32_t enable, void* host_out, int64_t n_words) {
  using namespace hs;
  if (enable && !g_ds_trace) {
    HS_CUDA(cudaMalloc(&g_ds_trace, kTraceWords * 8));
    HS_CUDA(cudaMemset(g_ds_trace, 0, kTraceWords * 8));
  }
  if (host_out && g_ds_trace) {
    HS_CUDA(cudaDeviceSynchronize());
    HS_CUDA(cudaMemcpy(host_out, g_ds_trace, (size_t)std::min<int64_t>(n_words, kTraceWords) * 8, cudaMemcpyDeviceToHost));
  }
  if (!enable && g_ds_trace) {
    cudaFree(g_ds_trace);
    g_ds_trace = nullptr;
  }
  return HS_OK;
}
