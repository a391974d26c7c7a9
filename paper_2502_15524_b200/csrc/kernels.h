// kernels.h — the non-GEMM sm_100a kernels of the decoder stage and the group data path.
#pragma once
#include "common.h"

namespace hs {

// Per-sequence descriptor of a (prefill or decode) call, identical on every stage.
struct SeqDesc {
  int q_start;  // first row of this sequence in the packed token dimension
  int n_q;      // tokens of this sequence in the call
  int pos0;     // position of its first token (= cached tokens before the call)
  int table;    // row of the block table
};

// x[t] = E[tok[t]]  (a5)
void launch_embed(const int* tok, const bf16* E, bf16* x, int T, int H, int V, cudaStream_t st);
// Bits set by kernels that met an out-of-range index (1: token id, 2: KV slot, 4: block id).
unsigned debug_bad_bits(bool reset);

// y[i] = bf16(x[row(i)] * rsqrt(mean(x^2)+eps) * w)   (a6; rows = null => row(i) = i)
// rs_out != null (the norm feeding a GEMM, reading R10b): y[i] = bf16(x[row(i)] * w) and
// rs_out[i] = rsqrt(mean(x^2)+eps), applied by the GEMM epilogue (GemmArgs::rs)
void launch_rmsnorm(const bf16* x, const int* rows, const bf16* w, bf16* y, int T, int H,
                    float eps, cudaStream_t st, float* rs_out = nullptr);

// RoPE (rotate-half, fp32 table) on q,k of qkv [T, 3H]; writes q' [T,H] and k', v into the
// paged pool of this layer: pool[block][K|V][head][16][d]  (a8)
void launch_rope_kv(const bf16* qkv, const int* pos, const int* slot, const float2* rope_tab,
                    bf16* q_out, bf16* pool, int T, int n_heads, int head_dim, int nslots,
                    cudaStream_t st);

// Causal attention of the packed queries against the paged cache (a9).  Prefill layout:
// one CTA per (16-query tile, head, sequence).
// tcgen05 prefill attention (attn_tc.cu), the default; HS_ATTN_TC=0 selects the mma.sync kernel (A/B)
bool attn_tc_enabled();
void launch_attn_prefill_tc(const bf16* q, const bf16* pool, const SeqDesc* seqs, int n_seqs, int max_nq,
                            const int* tables, int max_blocks, bf16* o, int nh, int d, int nblocks, cudaStream_t st);
void warm_attn_tc();
void launch_attn_prefill(const bf16* q, const bf16* pool, const SeqDesc* seqs, int n_seqs,
                         int max_nq, const int* tables, int max_blocks, bf16* o, int n_heads,
                         int head_dim, int nblocks, cudaStream_t st);

// Decode attention (one query per sequence) with deterministic split-KV (64 keys per split).
// ws: n_seqs * n_heads * kv_splits * (head_dim + 2) floats; ctr: n_seqs * n_heads zeroed
// arrival counters (self-resetting).
void launch_attn_decode(const bf16* q, const bf16* pool, const SeqDesc* seqs, int n_seqs,
                        int max_ctx, const int* tables, int max_blocks, bf16* o, int n_heads,
                        int head_dim, float* ws, int kv_splits, unsigned* ctr, int nblocks,
                        cudaStream_t st);
int attn_decode_splits(int max_ctx);

// tokens[i] = argmax_v logits[i][v], ties -> lowest id (a15)
void launch_argmax(const float* logits, int V, int n, int* tokens, cudaStream_t st);

// Stage hand-off (a13): copies bytes src -> dst (dst may be a peer / IPC mapping) with 16-byte
// stores, then the last CTA to finish publishes flag = epoch with a system-scope release.
// done_ctr: a device-local counter (reset by the last CTA).
void launch_send(const void* src, void* dst, uint64_t bytes, unsigned* done_ctr,
                 unsigned* flag, unsigned epoch, int ctas, cudaStream_t st);
// Waits (one thread, acquire) until *flag >= epoch; on timeout sets *err = 1 and returns.
void launch_wait(const unsigned* flag, unsigned epoch, int* err, cudaStream_t st);

// Consolidation KV gather (a17): n spans of span_bytes each, src[i] -> dst[i] (pointers may
// be peer mappings).  Bit-exact byte copy with 16-byte accesses.
void launch_span_copy(const uint64_t* src, const uint64_t* dst, int n, uint64_t span_bytes,
                      cudaStream_t st);

// 16-byte-granular copy by SMs (src / dst may be mapped pinned host memory): call metadata
// in, tokens out, without touching the copy engines that stream the weights.
void launch_small_copy(const void* src, void* dst, uint64_t bytes, cudaStream_t st);

// Consolidation copy list (weights + KV blocks in one launch), pulled by the launching GPU.
struct CopyDesc {
  uint64_t src, dst, bytes;
};
void launch_copy_list(const CopyDesc* d, int n, int ctas, cudaStream_t st);

}  // namespace hs
