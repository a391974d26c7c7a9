/* hs_kernels.h — test/benchmark entry points to the individual sm_100a kernels of libhs.
 * Not part of the serving path: the parity tests call them with device pointers (e.g. from
 * torch tensors) to compare each kernel against the CPU oracle op by op.  All pointers are
 * device pointers on the current device; `stream` is a cudaStream_t (0 = legacy default).
 * Calls are asynchronous; errors of the launch are returned, kernel faults surface at the
 * next synchronisation.  Layouts are those of include/hs.h and DESIGN.md "Data layout". */
#ifndef HS_KERNELS_H_
#define HS_KERNELS_H_
#include <stdint.h>
#include "hs.h"
#ifdef __cplusplus
extern "C" {
#endif

/* out = epilogue(W[M,K] . X[N,K]^T) stored as out[n*ldo + m].  W in the tiled weight layout of
 * include/hs.h ([M/128][K/64][128][64] bf16: 128 x 64 blocks, each contiguous); X row-major
 * [x_rows, K] bf16.  epi: 0 bf16, 1 bf16(acc +
 * resid[n*ldr+m]), 2 silu(gate)*up with gate/up rows interleaved by 16 (out has M/2 cols),
 * 3 fp32.  ws/ws_bytes: split-K workspace (NULL => no split-K).  X must have >= x_rows rows
 * (rows past N are read but their results discarded). */
hs_status hs_k_gemm(const void* W, int32_t M, int32_t K, const void* X, int32_t x_rows, int32_t N,
                    int32_t epi, void* out, int32_t ldo, const void* resid, int32_t ldr, void* ws,
                    uint64_t ws_bytes, void* stream);
/* y[i] = bf16(x[rows[i]] * rsqrt(mean x^2 + eps) * w), rows NULL => identity. */
hs_status hs_k_rmsnorm(const void* x, const int32_t* rows, const void* w, void* y, int32_t T,
                       int32_t H, float eps, void* stream);
/* RoPE + paged KV write; tab: float2 [max_pos][d/2] (cos, sin). */
hs_status hs_k_rope_kv(const void* qkv, const int32_t* pos, const int32_t* slot, const void* tab,
                       void* q_out, void* pool, int32_t T, int32_t n_heads, int32_t head_dim,
                       void* stream);
/* seqs: int32 [n][4] = {q_start, n_q, pos0, table_row}; tables int32 [n][max_blocks].
 * decode != 0: one query per sequence and table_row must equal the sequence's index. */
hs_status hs_k_attention(const void* q, const void* pool, const int32_t* seqs, int32_t n_seqs,
                         int32_t max_nq, int32_t max_ctx, const int32_t* tables, int32_t max_blocks,
                         void* o, int32_t n_heads, int32_t head_dim, int32_t decode, void* ws,
                         void* stream);
hs_status hs_k_argmax(const float* logits, int32_t V, int32_t n, int32_t* tokens, void* stream);
hs_status hs_k_embed(const int32_t* tok, const void* E, void* x, int32_t T, int32_t H, void* stream);
/* n spans: src[i] -> dst[i], span_bytes each (device arrays of device addresses). */
hs_status hs_k_span_copy(const uint64_t* src, const uint64_t* dst, int32_t n, uint64_t span_bytes,
                         void* stream);

/* Test-only instrumentation: enable != 0 makes the stream-K decode GEMM record per-CTA phase
 * timestamps (%globaltimer ns: start, weights requested, grid dependency resolved, first
 * stage full, last MMA issued, epilogue done, CTA end; 8 slots per CTA) of its latest launch;
 * host_out (optional) receives n_ctas * 8 uint64.  enable == 0 frees the buffer. */
hs_status hs_debug_gemm_trace(int32_t enable, void* host_out, int32_t n_ctas);

/* Test-only instrumentation of the decode-stack kernel (one launch = every layer of a stage
 * for one decode step): enable != 0 makes it record, per CTA and layer, 32 %globaltimer
 * stamps (activation loads issued per GEMM, epilogue / attention / row-norm completion,
 * weight loads issued per GEMM) of its latest launch, layout [n_sms][n_layers][32];
 * host_out (optional) receives n_words uint64.  enable == 0 frees the buffer. */
hs_status hs_debug_dstack_trace(int32_t enable, void* host_out, int64_t n_words);

/* Test-only: protocol-failure records of the decode-stack kernel.  A flag or stream-K part
 * wait that has not been satisfied after ~4 s of SM cycles (a protocol bug, not a slow step) writes one
 * row per (CTA, warp) into mapped pinned host memory and then traps (the call that launched
 * it returns HS_E_CUDA, the context is lost).  This call reads those rows on the host (no CUDA
 * call, so it works after the failure); print != 0 writes each row to stderr, naming the wait
 * site, the CTA, the flag / workspace region and index, the value seen and the value wanted,
 * and clears the rows it printed.  Returns the number of rows (0: no failure recorded). */
int32_t hs_debug_dstack_diag(int32_t print);

#ifdef __cplusplus
}
#endif
#endif
