// gemm.h — tcgen05/TMA GEMM for the decoder's dense contractions (QKV, O-proj, gate_up,
// down, lm_head).  D = A . B^T with A = weights [M, K] (M = output features) and
// B = activations [N, K] (N = tokens), both K-major bf16, fp32 accumulation in TMEM.
// The result is stored "transposed" as out[n * ldo + m], i.e. row-major [tokens, features],
// with a fused epilogue.  One kernel family serves prefill (N = hundreds of tokens, tensor
// bound) and decode (N = batch, weights-streaming HBM bound, split-K across the SMs).
#pragma once
#include "common.h"

namespace hs {

// rs (optional, GemmArgs::rs): the RMSNorm row scale of reading R10b — the activations are
// bf16(x * w) and EPI_BF16 / EPI_SILU_MUL (and FUSE_ROPE) use rs[n] * acc in place of acc.
enum GemmEpi : int {
  EPI_BF16 = 0,      // out = bf16(acc)
  EPI_RESID = 1,     // out = bf16(acc + resid)            (O-proj, down: single rounding)
  EPI_SILU_MUL = 2,  // out[.., f] = bf16(silu(g) * u), gate/up rows interleaved by 16
  EPI_F32 = 3,       // out = acc (fp32)                    (lm_head logits)
};

// A 2-D TMA descriptor over a row-major bf16 matrix [rows, cols] with a (64 x box_rows) box.
struct TmaMat {
  CUtensorMap map;
  const void* ptr = nullptr;
  int64_t rows = 0, cols = 0;
  int box_rows = 0;
};

// Encodes a 128B-swizzled K-major tile map (box = 64 cols x box_rows rows).
hs_status make_tma(TmaMat* t, const void* ptr, int64_t rows, int64_t cols, int box_rows);
// Layered row-major map [layers][rows][cols] (layers layer_stride_bytes apart), box 64 x 128 x 1.
hs_status make_tma3(TmaMat* t, const void* ptr, int64_t layers, int64_t layer_stride_bytes, int64_t rows,
                    int64_t cols);
// A weight matrix [rows, cols] in the tiled weight layout (include/hs.h: 128 x 64 blocks, each
// one contiguous 16 KiB run, block b = row tile * cols/64 + k-block): 3-D map {64, 128, blocks}
// with box 64 x 128 x 1 (the same 128B-swizzled shared-memory tile as make_tma's).
hs_status make_tma_w(TmaMat* t, const void* ptr, int64_t rows, int64_t cols);
// The same matrix of every layer of a stage (layers layer_stride_bytes apart): 4-D map
// {64, 128, blocks, layers}: one descriptor streams the matrix kind of the whole stage.
hs_status make_tma_w3(TmaMat* t, const void* ptr, int64_t layers, int64_t layer_stride_bytes, int64_t rows,
                      int64_t cols);

// Decode-path fusions applied by the stream-K reduction (the whole output row of a token is
// available there):
//   FUSE_NORM : out = bf16(acc + resid) (as EPI_RESID) and norm_out = RMSNorm(out) * norm_w
//               (rs_out != null: norm_out = bf16(out * norm_w), rs_out[n] = the row scale, R10b)
//   FUSE_ROPE : (QKV GEMM, EPI_BF16) q, k, v = bf16(acc); q' / k' rotated (RoPE table), q' to
//               q_out, k' and v written into the paged KV pool at slot[n]
enum GemmFuse : int { FUSE_NONE = 0, FUSE_NORM = 1, FUSE_ROPE = 2 };
struct GemmFusion {
  int kind = FUSE_NONE;
  const bf16* norm_w = nullptr;
  bf16* norm_out = nullptr;
  float* rs_out = nullptr;
  float eps = 0.f;
  const int* pos = nullptr;
  const int* slot = nullptr;
  const float2* rope_tab = nullptr;
  bf16* q_out = nullptr;
  bf16* pool = nullptr;
  int n_heads = 0, head_dim = 0;
  int nslots = 1 << 30;     // KV slots in the pool (range check of slot[n])
  bool* applied = nullptr;  // set to true when the fusion ran (else the caller runs the op)
};

struct GemmArgs {
  const TmaMat* A;   // weights [M, K]  (box_rows must be 128)
  const TmaMat* B;   // activations [>=N, K] (box_rows must equal the chosen BN; see gemm_bn)
  int M, N, K;
  int epi;
  void* out;
  int ldo;           // elements
  const bf16* resid; // EPI_RESID: resid[n * ldr + m]
  int ldr;
  const float* rs = nullptr;  // EPI_BF16 / EPI_SILU_MUL: per-token scale of the accumulator (R10b)
  float* workspace;  // split-K / stream-K partials (may be null => no split)
  uint64_t workspace_bytes;
  unsigned* counters;  // stream-K arrival counters: >= M/128 + 1 zeroed words (null => no stream-K)
  GemmFusion fuse;
};

// Tile width (tokens) the launcher will use for N tokens; activation maps must be encoded
// with this box height.  Deterministic in N only (partition invariance).
int gemm_bn(int N);
// All box heights a buffer of up to max_tokens rows might need.
int gemm_bn_count();
int gemm_bn_value(int i);

hs_status gemm(const GemmArgs& a, cudaStream_t stream);

// RMSNorm of T rows with exactly the arithmetic of the FUSE_NORM epilogue (decode path: a
// stage's first layer normalises its input like the previous layer's fused epilogue would,
// so PP = s stays bitwise equal to PP = 1).  H <= 8192.  rs_out: as GemmFusion::rs_out.
void launch_rownorm_decode(const bf16* x, const bf16* w, bf16* y, float* rs_out, int T, int H, float eps,
                           cudaStream_t st);

}  // namespace hs
