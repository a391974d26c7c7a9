// kapi.cu — include/hs_kernels.h: direct entry points to the kernels, for op-level parity
// tests and microbenchmarks.  Thin argument marshalling over the same launchers the group uses.
#include <mutex>
#include <vector>

#include "../../include/hs_kernels.h"
#include "common.h"
#include "gemm.h"
#include "kernels.h"

using namespace hs;

extern "C" hs_status hs_k_gemm(const void* W, int32_t M, int32_t K, const void* X, int32_t x_rows, int32_t N,
                               int32_t epi, void* out, int32_t ldo, const void* resid, int32_t ldr, void* ws,
                               uint64_t ws_bytes, void* stream) {
  if (!W || !X || !out || M <= 0 || K <= 0 || N <= 0 || x_rows < N || epi < 0 || epi > 3)
    HS_FAIL(HS_E_INVAL, "bad gemm args");
  TmaMat a;
  TmaMat b[5];
  HS_TRY(make_tma_w(&a, W, M, K));  // W in the tiled weight layout (include/hs_kernels.h)
  for (int i = 0; i < gemm_bn_count(); ++i) HS_TRY(make_tma(&b[i], X, x_rows, K, gemm_bn_value(i)));
  GemmArgs g{};
  g.A = &a; g.B = b; g.M = M; g.N = N; g.K = K; g.epi = epi; g.out = out; g.ldo = ldo;
  g.resid = reinterpret_cast<const bf16*>(resid); g.ldr = ldr;
  // the first 64 KiB of the workspace hold the stream-K arrival counters (zeroed here)
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (ws && ws_bytes > (1u << 20)) {
    HS_CUDA(cudaMemsetAsync(ws, 0, 65536, st));
    g.counters = reinterpret_cast<unsigned*>(ws);
    g.workspace = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + 65536);
    g.workspace_bytes = ws_bytes - 65536;
  } else {
    g.workspace = reinterpret_cast<float*>(ws);
    g.workspace_bytes = ws ? ws_bytes : 0;
  }
  return gemm(g, st);
}

extern "C" hs_status hs_k_rmsnorm(const void* x, const int32_t* rows, const void* w, void* y, int32_t T, int32_t H,
                                  float eps, void* stream) {
  if (!x || !w || !y || T <= 0 || H % 8) HS_FAIL(HS_E_INVAL, "bad rmsnorm args");
  launch_rmsnorm(reinterpret_cast<const bf16*>(x), rows, reinterpret_cast<const bf16*>(w),
                 reinterpret_cast<bf16*>(y), T, H, eps, reinterpret_cast<cudaStream_t>(stream));
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

extern "C" hs_status hs_k_rope_kv(const void* qkv, const int32_t* pos, const int32_t* slot, const void* tab,
                                  void* q_out, void* pool, int32_t T, int32_t nh, int32_t d, void* stream) {
  if (!qkv || !pos || !slot || !tab || !q_out || !pool || T <= 0 || (d != 64 && d != 128)) HS_FAIL(HS_E_INVAL, "bad args");
  launch_rope_kv(reinterpret_cast<const bf16*>(qkv), pos, slot, reinterpret_cast<const float2*>(tab),
                 reinterpret_cast<bf16*>(q_out), reinterpret_cast<bf16*>(pool), T, nh, d, 1 << 30,
                 reinterpret_cast<cudaStream_t>(stream));
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

extern "C" hs_status hs_k_attention(const void* q, const void* pool, const int32_t* seqs, int32_t n, int32_t max_nq,
                                    int32_t max_ctx, const int32_t* tables, int32_t max_blocks, void* o, int32_t nh,
                                    int32_t d, int32_t decode, void* ws, void* stream) {
  if (!q || !pool || !seqs || !tables || !o || n <= 0 || (d != 64 && d != 128)) HS_FAIL(HS_E_INVAL, "bad args");
  static_assert(sizeof(SeqDesc) == 16, "SeqDesc layout");
  auto st = reinterpret_cast<cudaStream_t>(stream);
  const SeqDesc* sd = reinterpret_cast<const SeqDesc*>(seqs);
  if (decode) {
    // per-device zeroed arrival counters for the split merge (self-resetting)
    static unsigned* ctr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!ctr[dev]) {
      HS_CUDA(cudaMalloc(&ctr[dev], 1 << 20));
      HS_CUDA(cudaMemsetAsync(ctr[dev], 0, 1 << 20, st));  // ordered before the launch on st
    }
    if ((size_t)n * nh * 4 > (1u << 20)) HS_FAIL(HS_E_INVAL, "too many (seq, head) pairs");
    launch_attn_decode(reinterpret_cast<const bf16*>(q), reinterpret_cast<const bf16*>(pool), sd, n, max_ctx, tables,
                       max_blocks, reinterpret_cast<bf16*>(o), nh, d, reinterpret_cast<float*>(ws),
                       attn_decode_splits(max_ctx), ctr[dev], 1 << 30, st);
  }
  else
    launch_attn_prefill(reinterpret_cast<const bf16*>(q), reinterpret_cast<const bf16*>(pool), sd, n, max_nq, tables,
                        max_blocks, reinterpret_cast<bf16*>(o), nh, d, 1 << 30, st);
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

extern "C" hs_status hs_k_argmax(const float* logits, int32_t V, int32_t n, int32_t* tokens, void* stream) {
  if (!logits || !tokens || V <= 0 || n <= 0) HS_FAIL(HS_E_INVAL, "bad args");
  launch_argmax(logits, V, n, tokens, reinterpret_cast<cudaStream_t>(stream));
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

extern "C" hs_status hs_k_embed(const int32_t* tok, const void* E, void* x, int32_t T, int32_t H, void* stream) {
  if (!tok || !E || !x || T <= 0 || H % 8) HS_FAIL(HS_E_INVAL, "bad args");
  launch_embed(tok, reinterpret_cast<const bf16*>(E), reinterpret_cast<bf16*>(x), T, H, 1 << 30,
               reinterpret_cast<cudaStream_t>(stream));
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}

extern "C" hs_status hs_k_span_copy(const uint64_t* src, const uint64_t* dst, int32_t n, uint64_t span_bytes,
                                    void* stream) {
  if (!src || !dst || n < 0 || span_bytes % 16) HS_FAIL(HS_E_INVAL, "bad args");
  launch_span_copy(src, dst, n, span_bytes, reinterpret_cast<cudaStream_t>(stream));
  HS_CUDA(cudaGetLastError());
  return HS_OK;
}
