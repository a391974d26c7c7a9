// gemm.h — tcgen05/TMA GEMM for the decoder's dense contractions (QKV, O-proj, gate_up,
// down, lm_head).  D = A . B^T with A = weights [M, K] (M = output features) and
// B = activations [N, K] (N = tokens), both K-major bf16, fp32 accumulation in TMEM.
// The result is stored "transposed" as out[n * ldo + m], i.e. row-major [tokens, features],
// with a fused epilogue.  One kernel family serves prefill (N = hundreds of tokens, tensor
// bound) and decode (N = batch, weights-streaming HBM bound, split-K across the SMs).
#pragma once
#include "common.h"

namespace hs {

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

struct GemmArgs {
  const TmaMat* A;   // weights [M, K]  (box_rows must be 128)
  const TmaMat* B;   // activations [>=N, K] (box_rows must equal the chosen BN; see gemm_bn)
  int M, N, K;
  int epi;
  void* out;
  int ldo;           // elements
  const bf16* resid; // EPI_RESID: resid[n * ldr + m]
  int ldr;
  float* workspace;  // split-K partials (may be null => no split)
  uint64_t workspace_bytes;
};

// Tile width (tokens) the launcher will use for N tokens; activation maps must be encoded
// with this box height.  Deterministic in N only (partition invariance).
int gemm_bn(int N);
// All box heights a buffer of up to max_tokens rows might need.
int gemm_bn_count();
int gemm_bn_value(int i);

hs_status gemm(const GemmArgs& a, cudaStream_t stream);

}  // namespace hs
