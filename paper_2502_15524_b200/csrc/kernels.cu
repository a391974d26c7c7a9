// kernels.cu — non-GEMM kernels of a pipeline stage (sm_100a), with warp-shuffle reductions
// and 128-bit global accesses.  See kernels.h for the contracts; DESIGN.md lists the
// roofline each is bounded by.
#include "kernels.h"

#include <cfloat>
#include <type_traits>

namespace hs {

// Data-dependent indices (token ids, KV slots, block ids) are range-checked on the device: an
// out-of-range value is never dereferenced; it sets a bit in g_bad, which the host turns into
// an error after the call (debug_bad_bits).
__device__ unsigned g_bad = 0;
__device__ __forceinline__ void flag_bad(unsigned bit) { atomicOr(&g_bad, bit); }

unsigned debug_bad_bits(bool reset) {
  unsigned v = 0;
  cudaMemcpyFromSymbol(&v, g_bad, sizeof(v));
  if (reset && v) {
    const unsigned z = 0;
    cudaMemcpyToSymbol(g_bad, &z, sizeof(z));
  }
  return v;
}

// ------------------------------------------------------------------ embedding (a5) -------
__global__ void embed_kernel(const int* __restrict__ tok, const uint4* __restrict__ E,
                             uint4* __restrict__ x, int H8, int V) {
  PDL_LAUNCH();
  PDL_WAIT();
  const int t = blockIdx.x;
  int id = tok[t];
  if (id < 0 || id >= V) {
    if (threadIdx.x == 0) flag_bad(1u);
    id = 0;
  }
  const uint4* src = E + (size_t)id * H8;
  uint4* dst = x + (size_t)t * H8;
  for (int i = threadIdx.x; i < H8; i += blockDim.x) dst[i] = __ldg(src + i);
}

void launch_embed(const int* tok, const bf16* E, bf16* x, int T, int H, int V, cudaStream_t st) {
  count_launch();
  const int H8 = H / 8;
  launchk(embed_kernel, T, H8 < 512 ? H8 : 512, 0, st, tok, reinterpret_cast<const uint4*>(E),
          reinterpret_cast<uint4*>(x), H8, V);
}

// ------------------------------------------------------------------ RMSNorm (a6) ---------
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int MAXV>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const uint4* __restrict__ x, const int* __restrict__ rows,
                                                      const uint4* __restrict__ w, uint4* __restrict__ y,
                                                      float* __restrict__ rs_out, int H8, float inv_h, float eps) {
  PDL_LAUNCH();
  PDL_WAIT();
  __shared__ float red[8];
  const int i = blockIdx.x;
  const int r = rows ? rows[i] : i;
  const uint4* xr = x + (size_t)r * H8;
  uint4 v[MAXV];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < MAXV; ++j) {
    const int c = threadIdx.x + j * 256;
    if (c < H8) {
      v[j] = xr[c];
      const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v[j]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float2 f = __bfloat1622float2(p[k]);
        ss += f.x * f.x + f.y * f.y;
      }
    }
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) tot += red[k];
  const float rs_row = 1.0f / sqrtf(tot * inv_h + eps);
  if (rs_out && threadIdx.x == 0) rs_out[i] = rs_row;
  const float rs = rs_out ? 1.0f : rs_row;  // R10b: y = bf16(x * w), the scale goes to the GEMM epilogue
#pragma unroll
  for (int j = 0; j < MAXV; ++j) {
    const int c = threadIdx.x + j * 256;
    if (c < H8) {
      uint4 wv = w[c], out;
      const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v[j]);
      const __nv_bfloat162* q = reinterpret_cast<const __nv_bfloat162*>(&wv);
      __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float2 a = __bfloat1622float2(p[k]), b = __bfloat1622float2(q[k]);
        o[k] = __floats2bfloat162_rn(a.x * rs * b.x, a.y * rs * b.y);
      }
      y[(size_t)i * H8 + c] = out;
    }
  }
}

void launch_rmsnorm(const bf16* x, const int* rows, const bf16* w, bf16* y, int T, int H,
                    float eps, cudaStream_t st, float* rs_out) {
  count_launch();
  const int H8 = H / 8;
  auto X = reinterpret_cast<const uint4*>(x);
  auto W = reinterpret_cast<const uint4*>(w);
  auto Y = reinterpret_cast<uint4*>(y);
  if (H8 <= 256) launchk(rmsnorm_kernel<1>, T, 256, 0, st, X, rows, W, Y, rs_out, H8, 1.0f / H, eps);
  else if (H8 <= 512) launchk(rmsnorm_kernel<2>, T, 256, 0, st, X, rows, W, Y, rs_out, H8, 1.0f / H, eps);
  else if (H8 <= 1024) launchk(rmsnorm_kernel<4>, T, 256, 0, st, X, rows, W, Y, rs_out, H8, 1.0f / H, eps);
  else launchk(rmsnorm_kernel<8>, T, 256, 0, st, X, rows, W, Y, rs_out, H8, 1.0f / H, eps);
}

// ------------------------------------------------------------------ RoPE + KV write (a8) -
__global__ void rope_kv_kernel(const bf16* __restrict__ qkv, const int* __restrict__ pos,
                               const int* __restrict__ slot, const float2* __restrict__ tab,
                               bf16* __restrict__ q_out, bf16* __restrict__ pool, int nh, int d, int nslots) {
  PDL_LAUNCH();
  PDL_WAIT();
  const int t = blockIdx.x;
  const int H = nh * d, hd = d / 2;
  const bf16* row = qkv + (size_t)t * 3 * H;
  const int p = pos[t];
  int s = slot[t];
  if (s < 0 || s >= nslots) {
    if (threadIdx.x == 0) flag_bad(2u);
    return;
  }
  const size_t blk = (size_t)(s >> 4), off = (size_t)(s & 15);
  const float2* cs = tab + (size_t)p * hd;
  for (int idx = threadIdx.x; idx < nh * hd; idx += blockDim.x) {
    const int h = idx / hd, i = idx % hd;
    const float2 c = cs[i];  // (cos, sin)
    const float q1 = __bfloat162float(row[h * d + i]), q2 = __bfloat162float(row[h * d + i + hd]);
    const float k1 = __bfloat162float(row[H + h * d + i]), k2 = __bfloat162float(row[H + h * d + i + hd]);
    bf16* qo = q_out + (size_t)t * H + h * d;
    qo[i] = __float2bfloat16_rn(q1 * c.x - q2 * c.y);
    qo[i + hd] = __float2bfloat16_rn(q2 * c.x + q1 * c.y);
    bf16* kd = pool + (((blk * 2 + 0) * nh + h) * 16 + off) * d;
    kd[i] = __float2bfloat16_rn(k1 * c.x - k2 * c.y);
    kd[i + hd] = __float2bfloat16_rn(k2 * c.x + k1 * c.y);
  }
  const int d8 = d / 8;
  const uint4* v = reinterpret_cast<const uint4*>(row + 2 * H);
  for (int idx = threadIdx.x; idx < nh * d8; idx += blockDim.x) {
    const int h = idx / d8, j = idx % d8;
    uint4* vd = reinterpret_cast<uint4*>(pool + (((blk * 2 + 1) * nh + h) * 16 + off) * d);
    vd[j] = v[h * d8 + j];
  }
}

void launch_rope_kv(const bf16* qkv, const int* pos, const int* slot, const float2* tab, bf16* q_out,
                    bf16* pool, int T, int nh, int d, int nslots, cudaStream_t st) {
  count_launch();
  launchk(rope_kv_kernel, T, 256, 0, st, qkv, pos, slot, tab, q_out, pool, nh, d, nslots);
}

// ------------------------------------------------------------------ attention (a9) -------
// Scores are computed in the log2 domain: s2 = (q . k) * log2(e) / sqrt(d); softmax with
// exp2 is identical to the natural-base definition.
template <int D>
struct Lanes {
  static constexpr int E = D / 32;  // elements per lane
};

template <int D>
__device__ __forceinline__ void load_lane(const bf16* p, float* out) {
  constexpr int E = D / 32;
  if constexpr (E == 4) {
    uint2 u = *reinterpret_cast<const uint2*>(p);
    float2 a = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.x));
    float2 b = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.y));
    out[0] = a.x; out[1] = a.y; out[2] = b.x; out[3] = b.y;
  } else {
    float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
    out[0] = a.x; out[1] = a.y;
  }
}

template <int D>
__device__ __forceinline__ void store_lane(bf16* p, const float* v) {
  constexpr int E = D / 32;
  if constexpr (E == 4) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p) = u;
  } else {
    *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(v[0], v[1]);
  }
}

// Prefill: flash-attention with bf16 tensor-core MMAs (m16n8k16, fp32 accumulation).
// CTA = (64-query tile, head, sequence), 4 warps x 16 query rows.  Per 64-key chunk the K and V
// rows are gathered from the paged pool into XOR-swizzled shared memory (conflict-free
// ldmatrix), S = Q K^T and O += P V run on the tensor cores, the online softmax in fp32 with
// exp2 (scores pre-scaled by log2(e)/sqrt(d)).  P is fed to the P.V MMA as a bf16 pair
// P = P_hi + P_lo (two MMAs sharing the V fragments), so the probabilities keep ~16 bits
// (the oracle's contract is fp32 probabilities; a single bf16 P would add 2^-9 relative error).
constexpr int PF_Q = 64;
constexpr int PF_KC = 64;

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void mma_bf16_16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

template <int D>
__global__ void __launch_bounds__(128) attn_prefill_kernel(
    const bf16* __restrict__ q, const bf16* __restrict__ pool, const SeqDesc* __restrict__ seqs,
    const int* __restrict__ tables, int max_blocks, bf16* __restrict__ o, int nh, int nblocks) {
  PDL_LAUNCH();
  PDL_WAIT();
  constexpr int CH = D / 8;  // 16-byte chunks per row
  constexpr int KS = D / 16; // k-steps over head_dim
  // double-buffered K / V chunks (dynamic smem): chunk t+1 streams in (cp.async) while chunk t
  // is multiplied
  extern __shared__ __align__(128) uint4 kv_smem[];
  const SeqDesc s = seqs[blockIdx.z];
  const int head = blockIdx.y;
  const int qt0 = (gridDim.x - 1 - blockIdx.x) * PF_Q;  // longest (causal) query tiles first
  if (qt0 >= s.n_q) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int H = nh * D;
  const float sl2 = 1.4426950408889634f / sqrtf((float)D);
  // Q fragments of this warp's 16 rows (rows beyond n_q read row n_q-1: results discarded)
  const int r0 = qt0 + warp * 16 + g, r1 = r0 + 8;
  const int qa = min(r0, s.n_q - 1), qb = min(r1, s.n_q - 1);
  const uint32_t* q0p = reinterpret_cast<const uint32_t*>(q + (size_t)(s.q_start + qa) * H + head * D);
  const uint32_t* q1p = reinterpret_cast<const uint32_t*>(q + (size_t)(s.q_start + qb) * H + head * D);
  uint32_t qf[KS][4];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    qf[ks][0] = q0p[ks * 8 + tig];
    qf[ks][1] = q1p[ks * 8 + tig];
    qf[ks][2] = q0p[ks * 8 + 4 + tig];
    qf[ks][3] = q1p[ks * 8 + 4 + tig];
  }
  const int pos_a = s.pos0 + r0, pos_b = s.pos0 + r1;
  float acc[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
  const int n_keys = s.pos0 + min(qt0 + PF_Q, s.n_q);
  const int* tab = tables + (size_t)s.table * max_blocks;
  const int warp_max_pos = s.pos0 + min(qt0 + warp * 16 + 15, s.n_q - 1);
  // gather K, V rows (D * 2 bytes each) of chunk kc into buffer bb, swizzled: 16-byte chunk c
  // of row r at c ^ (r & 7); rows past the keys are zero-filled (cp.async src-size 0)
  auto issue = [&](int bb, int kc) {
    uint4* Kd = kv_smem + (size_t)bb * 2 * PF_KC * CH;
    uint4* Vd = Kd + PF_KC * CH;
    const int nk = min(PF_KC, n_keys - kc);
    for (int idx = threadIdx.x; idx < PF_KC * CH; idx += 128) {
      const int r = idx / CH, c = idx % CH;
      const bf16* ks = pool;
      int bytes = 0;
      if (r < nk) {
        const int j = kc + r;
        const int b = tab[j >> 4];
        if (b >= 0 && b < nblocks) {
          ks = pool + ((((size_t)b * 2) * nh + head) * 16 + (j & 15)) * D + c * 8;
          bytes = 16;
        } else if (c == 0) {
          flag_bad(4u);
        }
      }
      const uint32_t dk = static_cast<uint32_t>(__cvta_generic_to_shared(Kd + r * CH + (c ^ (r & 7))));
      const uint32_t dv = static_cast<uint32_t>(__cvta_generic_to_shared(Vd + r * CH + (c ^ (r & 7))));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dk), "l"(ks), "r"(bytes) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dv), "l"(ks + (size_t)nh * 16 * D), "r"(bytes)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(0, 0);
  for (int kc = 0, it = 0; kc < n_keys; kc += PF_KC, ++it) {
    const int nk = min(PF_KC, n_keys - kc);
    if (kc + PF_KC < n_keys) {
      issue((it + 1) & 1, kc + PF_KC);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const uint32_t ks_base = static_cast<uint32_t>(__cvta_generic_to_shared(kv_smem + (size_t)(it & 1) * 2 * PF_KC * CH));
    const uint32_t vs_base = ks_base + PF_KC * CH * 16;
    if (kc > warp_max_pos) {  // whole chunk in this warp's causal future
      __syncthreads();
      continue;
    }
    // S = Q K^T : 16 x 64 per warp (8 n-tiles of 8 keys)
    float sc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int row = j * 8 + (lane & 7);
#pragma unroll
      for (int ks = 0; ks < KS; ks += 2) {
        const int c = 2 * ks + (lane >> 3);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(ks_base + (uint32_t)((row * CH + (c ^ (row & 7))) * 16), b0, b1, b2, b3);
        mma_bf16_16816(sc[j], qf[ks], b0, b1);
        mma_bf16_16816(sc[j], qf[ks + 1], b2, b3);
      }
    }
    // causal mask, scaling, online softmax (rows g and g+8 of the warp tile)
    float mx_a = m_a, mx_b = m_b;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k0 = kc + j * 8 + 2 * tig;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int kp = k0 + e;
        sc[j][e] = (kp <= pos_a && kp < kc + nk) ? sc[j][e] * sl2 : -INFINITY;
        sc[j][2 + e] = (kp <= pos_b && kp < kc + nk) ? sc[j][2 + e] * sl2 : -INFINITY;
        mx_a = fmaxf(mx_a, sc[j][e]);
        mx_b = fmaxf(mx_b, sc[j][2 + e]);
      }
    }
    mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 1));
    mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 2));
    mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 1));
    mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 2));
    const float ca = mx_a == -INFINITY ? 1.f : exp2f(m_a - mx_a);
    const float cb = mx_b == -INFINITY ? 1.f : exp2f(m_b - mx_b);
    m_a = mx_a;
    m_b = mx_b;
    float sa = 0.f, sb = 0.f;
    uint32_t pf[4][4], pl[4][4];  // P (hi, lo) as A fragments: k-step kk covers n-tiles 2kk, 2kk+1
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float p0 = mx_a == -INFINITY ? 0.f : exp2f(sc[j][0] - mx_a);
      const float p1 = mx_a == -INFINITY ? 0.f : exp2f(sc[j][1] - mx_a);
      const float p2 = mx_b == -INFINITY ? 0.f : exp2f(sc[j][2] - mx_b);
      const float p3 = mx_b == -INFINITY ? 0.f : exp2f(sc[j][3] - mx_b);
      sa += p0 + p1;
      sb += p2 + p3;
      const __nv_bfloat162 h01 = __floats2bfloat162_rn(p0, p1), h23 = __floats2bfloat162_rn(p2, p3);
      const float2 f01 = __bfloat1622float2(h01), f23 = __bfloat1622float2(h23);
      pf[j >> 1][(j & 1) * 2 + 0] = *reinterpret_cast<const uint32_t*>(&h01);
      pf[j >> 1][(j & 1) * 2 + 1] = *reinterpret_cast<const uint32_t*>(&h23);
      pl[j >> 1][(j & 1) * 2 + 0] = pack_bf16(p0 - f01.x, p1 - f01.y);
      pl[j >> 1][(j & 1) * 2 + 1] = pack_bf16(p2 - f23.x, p3 - f23.y);
    }
    l_a = l_a * ca + sa;
    l_b = l_b * cb + sb;
#pragma unroll
    for (int j = 0; j < D / 8; ++j) {
      acc[j][0] *= ca;
      acc[j][1] *= ca;
      acc[j][2] *= cb;
      acc[j][3] *= cb;
    }
    // O += P V : V rows are keys (k), columns head dims (n) -> transposed ldmatrix
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int vrow = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
      for (int dd = 0; dd < D / 8; dd += 2) {
        const int c = dd + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vs_base + (uint32_t)((vrow * CH + (c ^ (vrow & 7))) * 16), b0, b1, b2, b3);
        mma_bf16_16816(acc[dd], pf[kk], b0, b1);
        mma_bf16_16816(acc[dd + 1], pf[kk], b2, b3);
        mma_bf16_16816(acc[dd], pl[kk], b0, b1);
        mma_bf16_16816(acc[dd + 1], pl[kk], b2, b3);
      }
    }
    __syncthreads();  // buffer (it & 1) is refilled by the next iteration's issue
  }
  // finalize: quad-reduce the row sums, normalise, store bf16
  l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
  l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
  l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
  l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
  const float ia = 1.f / l_a, ib = 1.f / l_b;
  if (r0 < s.n_q) {
    uint32_t* oa = reinterpret_cast<uint32_t*>(o + (size_t)(s.q_start + r0) * H + head * D);
#pragma unroll
    for (int j = 0; j < D / 8; ++j) oa[j * 4 + tig] = pack_bf16(acc[j][0] * ia, acc[j][1] * ia);
  }
  if (r1 < s.n_q) {
    uint32_t* ob = reinterpret_cast<uint32_t*>(o + (size_t)(s.q_start + r1) * H + head * D);
#pragma unroll
    for (int j = 0; j < D / 8; ++j) ob[j * 4 + tig] = pack_bf16(acc[j][2] * ib, acc[j][3] * ib);
  }
}

void launch_attn_prefill(const bf16* q, const bf16* pool, const SeqDesc* seqs, int n_seqs, int max_nq,
                         const int* tables, int max_blocks, bf16* o, int nh, int d, int nblocks, cudaStream_t st) {
  if (attn_tc_enabled())
    return launch_attn_prefill_tc(q, pool, seqs, n_seqs, max_nq, tables, max_blocks, o, nh, d, nblocks, st);
  count_launch();
  dim3 grid((max_nq + PF_Q - 1) / PF_Q, nh, n_seqs);
  const size_t smem = (size_t)2 * 2 * PF_KC * d * 2;  // 2 buffers x (K, V) x 64 rows x d bf16
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr[dev]) {
    cudaFuncSetAttribute(attn_prefill_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 2 * PF_KC * 128 * 2);
    cudaFuncSetAttribute(attn_prefill_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 2 * PF_KC * 64 * 2);
    attr[dev] = true;
  }
  if (d == 128) launchk(attn_prefill_kernel<128>, grid, 128, smem, st, q, pool, seqs, tables, max_blocks, o, nh, nblocks);
  else launchk(attn_prefill_kernel<64>, grid, 128, smem, st, q, pool, seqs, tables, max_blocks, o, nh, nblocks);
}

// Decode (one query per sequence), latency-oriented: CTA = (head, seq, split), 16 warps; warp
// w owns KV blocks b0 + w, b0 + w + 16, ... of the split.  For a 16-token block lane l loads
// dims [E l, E l + E) of all 16 K rows and 16 V rows straight into registers (32 independent
// 8-byte loads in flight per lane, no shared-memory staging), computes the 16 scores with warp
// all-reduces, and keeps an online softmax (m, l, o[E]) per warp.  Warps are merged through
// shared memory in warp order; splits (long contexts only: DEC_BLOCKS_PER_SPLIT blocks each)
// are merged by the CTA that finishes a (seq, head) last, in split order.  Deterministic.
constexpr int DEC_WARPS = 16;
constexpr int DEC_BLOCKS_PER_SPLIT = 64;  // 1024 tokens per CTA

template <int D>
__global__ void __launch_bounds__(DEC_WARPS * 32) attn_decode_kernel(
    const bf16* __restrict__ q, const bf16* __restrict__ pool, const SeqDesc* __restrict__ seqs,
    const int* __restrict__ tables, int max_blocks, bf16* __restrict__ o, int nh, float* __restrict__ ws,
    int splits, unsigned* __restrict__ ctr, int nblocks) {
  PDL_LAUNCH();
  PDL_WAIT();
  constexpr int E = D / 32;  // dims per lane (4 or 2)
  __shared__ float sm_m[DEC_WARPS], sm_l[DEC_WARPS];
  __shared__ float sm_o[DEC_WARPS][D];
  __shared__ int is_last;
  const int head = blockIdx.x, si = blockIdx.y, sp = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = nh * D;
  const int* tab = tables + (size_t)si * max_blocks;  // table row == sequence index of the call
  const SeqDesc s = seqs[si];
  const int n_keys = s.pos0 + 1;
  const int nb = (n_keys + 15) >> 4;
  const int b0 = sp * DEC_BLOCKS_PER_SPLIT, b1 = min(nb, b0 + DEC_BLOCKS_PER_SPLIT);
  const float scale = 1.4426950408889634f / sqrtf((float)D);
  float qv[E];
  {
    const bf16* qp = q + (size_t)s.q_start * H + head * D + lane * E;
    if constexpr (E == 4) {
      const uint2 u = *reinterpret_cast<const uint2*>(qp);
      const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
      const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
      qv[0] = a.x * scale; qv[1] = a.y * scale; qv[2] = b.x * scale; qv[3] = b.y * scale;
    } else {
      const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(qp));
      qv[0] = a.x * scale; qv[1] = a.y * scale;
    }
  }
  float m = -INFINITY, l = 0.f, acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  const size_t vstride = (size_t)nh * 16 * D;
  for (int b = b0 + warp; b < b1; b += DEC_WARPS) {
    int blk = tab[b];
    if (blk < 0 || blk >= nblocks) {
      if (lane == 0) flag_bad(4u);
      blk = 0;
    }
    const bf16* kb = pool + ((((size_t)blk * 2) * nh + head) * 16) * D + lane * E;
    using VT = typename std::conditional<E == 4, uint2, uint32_t>::type;
    VT kr[16], vr[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      kr[j] = __ldcs(reinterpret_cast<const VT*>(kb + j * D));
      vr[j] = __ldcs(reinterpret_cast<const VT*>(kb + vstride + j * D));
    }
    float sc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float part;
      if constexpr (E == 4) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&kr[j].x));
        const float2 c = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&kr[j].y));
        part = qv[0] * a.x + qv[1] * a.y + qv[2] * c.x + qv[3] * c.y;
      } else {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&kr[j]));
        part = qv[0] * a.x + qv[1] * a.y;
      }
      sc[j] = part;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int j = 0; j < 16; ++j) sc[j] += __shfl_xor_sync(0xffffffffu, sc[j], off);
    float mb = m;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (b * 16 + j >= n_keys) sc[j] = -INFINITY;
      mb = fmaxf(mb, sc[j]);
    }
    const float corr = exp2f(m - mb);
    l *= corr;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] *= corr;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float pj = exp2f(sc[j] - mb);
      l += pj;
      if constexpr (E == 4) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vr[j].x));
        const float2 c = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vr[j].y));
        acc[0] += pj * a.x; acc[1] += pj * a.y; acc[2] += pj * c.x; acc[3] += pj * c.y;
      } else {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vr[j]));
        acc[0] += pj * a.x; acc[1] += pj * a.y;
      }
    }
    m = mb;
  }
  // merge the warps (fixed order)
  if (lane == 0) { sm_m[warp] = m; sm_l[warp] = l; }
#pragma unroll
  for (int e = 0; e < E; ++e) sm_o[warp][lane * E + e] = acc[e];
  __syncthreads();
  const int t = threadIdx.x;
  float M = -INFINITY, L = 0.f, A = 0.f;
  if (t < D) {
#pragma unroll
    for (int w = 0; w < DEC_WARPS; ++w) M = fmaxf(M, sm_m[w]);
#pragma unroll
    for (int w = 0; w < DEC_WARPS; ++w) {
      const float f = sm_m[w] == -INFINITY ? 0.f : exp2f(sm_m[w] - M);
      L += sm_l[w] * f;
      A += sm_o[w][t] * f;
    }
  }
  if (splits == 1) {
    if (t < D) o[(size_t)s.q_start * H + head * D + t] = __float2bfloat16_rn(A / L);
    return;
  }
  float* wsp = ws + (((size_t)si * nh + head) * splits + sp) * (D + 2);
  if (t < D) {
    if (t == 0) { wsp[0] = M; wsp[1] = L; }
    wsp[2 + t] = A;
  }
  __syncthreads();
  if (t == 0) {
    __threadfence();
    unsigned* c = ctr + (size_t)si * nh + head;
    const unsigned old = atomicAdd(c, 1u);
    is_last = old == (unsigned)(splits - 1);
    if (is_last) {
      *c = 0;
      __threadfence();
    }
  }
  __syncthreads();
  if (!is_last || t >= D) return;
  const float* w0 = ws + ((size_t)si * nh + head) * splits * (D + 2);
  float MM = -INFINITY;
  for (int k = 0; k < splits; ++k) MM = fmaxf(MM, __ldcg(w0 + k * (D + 2)));
  float LL = 0.f, AA = 0.f;
  for (int k = 0; k < splits; ++k) {
    const float ms = __ldcg(w0 + k * (D + 2));
    const float f = ms == -INFINITY ? 0.f : exp2f(ms - MM);
    LL += __ldcg(w0 + k * (D + 2) + 1) * f;
    AA += __ldcg(w0 + k * (D + 2) + 2 + t) * f;
  }
  o[(size_t)s.q_start * H + head * D + t] = __float2bfloat16_rn(AA / LL);
}

int attn_decode_splits(int max_ctx) {
  const int nb = (max_ctx + 15) / 16;
  return (nb + DEC_BLOCKS_PER_SPLIT - 1) / DEC_BLOCKS_PER_SPLIT;
}

void launch_attn_decode(const bf16* q, const bf16* pool, const SeqDesc* seqs, int n_seqs, int max_ctx,
                        const int* tables, int max_blocks, bf16* o, int nh, int d, float* ws, int splits,
                        unsigned* ctr, int nblocks, cudaStream_t st) {
  count_launch();
  dim3 grid(nh, n_seqs, splits);
  if (d == 128) launchk(attn_decode_kernel<128>, grid, DEC_WARPS * 32, 0, st, q, pool, seqs, tables, max_blocks, o, nh, ws, splits, ctr, nblocks);
  else launchk(attn_decode_kernel<64>, grid, DEC_WARPS * 32, 0, st, q, pool, seqs, tables, max_blocks, o, nh, ws, splits, ctr, nblocks);
}

// ------------------------------------------------------------------ argmax (a15) ---------
__global__ void __launch_bounds__(1024) argmax_kernel(const float* __restrict__ logits, int V,
                                                      int* __restrict__ out) {
  PDL_LAUNCH();
  PDL_WAIT();
  __shared__ float bv[32];
  __shared__ int bi[32];
  const float* row = logits + (size_t)blockIdx.x * V;
  float best = -INFINITY;
  int idx = 0x7fffffff;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const float x = row[v];
    if (x > best) { best = x; idx = v; }  // strided ascending scan keeps the lowest id on ties
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ob > best || (ob == best && oi < idx)) { best = ob; idx = oi; }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { bv[w] = best; bi[w] = idx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (bv[k] > best || (bv[k] == best && bi[k] < idx)) { best = bv[k]; idx = bi[k]; }
    bv[0] = best;
    bi[0] = idx;
    out[blockIdx.x] = idx == 0x7fffffff ? 0 : idx;
  }
}

void launch_argmax(const float* logits, int V, int n, int* tokens, cudaStream_t st) {
  count_launch();
  launchk(argmax_kernel, n, 1024, 0, st, logits, V, tokens);
}

// ------------------------------------------------------------------ hand-off (a13) -------
__global__ void __launch_bounds__(256) send_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                   uint64_t n16, unsigned* done_ctr, unsigned* flag,
                                                   unsigned epoch) {
  PDL_LAUNCH();
  PDL_WAIT();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = src[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(done_ctr, 1u);
    if (prev == gridDim.x - 1) {
      *done_ctr = 0;
      __threadfence_system();
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
    }
  }
}

void launch_send(const void* src, void* dst, uint64_t bytes, unsigned* done_ctr, unsigned* flag,
                 unsigned epoch, int ctas, cudaStream_t st) {
  count_launch();
  launchk(send_kernel, ctas, 256, 0, st, reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst),
          (uint64_t)(bytes / 16), done_ctr, flag, epoch);
}

__global__ void wait_kernel(const unsigned* flag, unsigned epoch, int* err) {
  PDL_LAUNCH();
  PDL_WAIT();
  // SM cycles, not %globaltimer (re-synchronised by the driver, it can step backwards; tc.h)
  const long long t0 = clock64();
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int)(v - epoch) >= 0) return;
    __nanosleep(200);
    if (clock64() - t0 > 40000000000ll) {  // ~20 s at the boost clock: the peer never signalled
      *err = 1;
      return;
    }
  }
}

void launch_wait(const unsigned* flag, unsigned epoch, int* err, cudaStream_t st) {
  count_launch();
  launchk(wait_kernel, 1, 1, 0, st, flag, epoch, err);
}

// ------------------------------------------------------------------ span copy (a17) ------
__global__ void __launch_bounds__(256) span_copy_kernel(const uint64_t* __restrict__ src,
                                                        const uint64_t* __restrict__ dst, uint64_t n16,
                                                        int parts) {
  PDL_LAUNCH();
  PDL_WAIT();
  const int span = blockIdx.x / parts, part = blockIdx.x % parts;
  const uint4* s = reinterpret_cast<const uint4*>(src[span]);
  uint4* d = reinterpret_cast<uint4*>(dst[span]);
  const uint64_t per = (n16 + parts - 1) / parts;
  const uint64_t b = per * part, e = min(n16, b + per);
  uint64_t i = b + threadIdx.x;
  for (; i + 768 < e; i += 1024) {
    uint4 x0 = s[i], x1 = s[i + 256], x2 = s[i + 512], x3 = s[i + 768];
    d[i] = x0; d[i + 256] = x1; d[i + 512] = x2; d[i + 768] = x3;
  }
  for (; i < e; i += 256) d[i] = s[i];
}

// Copy list: descriptors {src, dst, bytes} (src, dst, bytes multiples of 16, checked by the
// host-side list builder; any size: consolidation uses 1 MiB pieces by default), persistent
// grid-stride over descriptors; 4 x 16-byte loads in flight per thread before the stores.
__global__ void __launch_bounds__(256) copy_list_kernel(const CopyDesc* __restrict__ d, int n) {
  PDL_LAUNCH();
  PDL_WAIT();
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const uint4* s = reinterpret_cast<const uint4*>(d[i].src);
    uint4* o = reinterpret_cast<uint4*>(d[i].dst);
    const int n16 = (int)(d[i].bytes >> 4);
    int j = threadIdx.x;
    for (; j + 768 < n16; j += 1024) {
      uint4 a = s[j], b = s[j + 256], c = s[j + 512], e = s[j + 768];
      o[j] = a; o[j + 256] = b; o[j + 512] = c; o[j + 768] = e;
    }
    for (; j < n16; j += 256) o[j] = s[j];
  }
}

void launch_copy_list(const CopyDesc* d, int n, int ctas, cudaStream_t st) {
  if (n <= 0) return;
  count_launch();
  // plain launch (no programmatic serialisation): a one-off bulk copy has nothing to overlap,
  // and it reads peer mappings opened by another process
  copy_list_kernel<<<ctas < n ? ctas : n, 256, 0, st>>>(d, n);
}

// Small copies between mapped pinned host memory and device memory done by SMs, so they never
// queue behind the multi-GB weight stream on the copy engines (a DMA H2D of call metadata on
// the compute stream would wait for the whole load and serialise prefill after it).
__global__ void __launch_bounds__(256) small_copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                         int n16) {
  PDL_LAUNCH();
  PDL_WAIT();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) dst[i] = src[i];
  __threadfence_system();
}

void launch_small_copy(const void* src, void* dst, uint64_t bytes, cudaStream_t st) {
  const int n16 = (int)((bytes + 15) / 16);
  if (n16 <= 0) return;
  count_launch();
  const int ctas = n16 > 4096 ? 16 : 1;
  launchk(small_copy_kernel, ctas, 256, 0, st, reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), n16);
}

void launch_span_copy(const uint64_t* src, const uint64_t* dst, int n, uint64_t span_bytes, cudaStream_t st) {
  if (n <= 0) return;
  count_launch();
  const uint64_t n16 = span_bytes / 16;
  int parts = (int)((span_bytes + 65535) / 65536);
  if (parts < 1) parts = 1;
  launchk(span_copy_kernel, n * parts, 256, 0, st, src, dst, n16, parts);
}

void warm_kernels() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, embed_kernel);
  cudaFuncGetAttributes(&a, rmsnorm_kernel<1>);
  cudaFuncGetAttributes(&a, rmsnorm_kernel<2>);
  cudaFuncGetAttributes(&a, rmsnorm_kernel<4>);
  cudaFuncGetAttributes(&a, rmsnorm_kernel<8>);
  cudaFuncGetAttributes(&a, rope_kv_kernel);
  cudaFuncGetAttributes(&a, attn_prefill_kernel<64>);
  cudaFuncGetAttributes(&a, attn_prefill_kernel<128>);
  warm_attn_tc();
  cudaFuncGetAttributes(&a, attn_decode_kernel<64>);
  cudaFuncGetAttributes(&a, attn_decode_kernel<128>);
  cudaFuncGetAttributes(&a, argmax_kernel);
  cudaFuncGetAttributes(&a, send_kernel);
  cudaFuncGetAttributes(&a, wait_kernel);
  cudaFuncGetAttributes(&a, span_copy_kernel);
  cudaFuncGetAttributes(&a, copy_list_kernel);
  cudaFuncGetAttributes(&a, small_copy_kernel);
}

}  // namespace hs
