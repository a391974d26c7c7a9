// dstack.h — the decode stack: every decoder layer of a stage for one decode step (SURVEY §8
// a6-a12 with T = B tokens, a16) in ONE persistent kernel.
//
// Why: a decode step is HBM-bound (the weights are streamed once per step) but, launched as
// 5 kernels per layer, every kernel boundary drains the weight stream (launch, prologue,
// pipeline fill, stream-K fix-up tail, grid-wide norm tail: ~10 us each, 160 per 7B step).
// Here one CTA per SM walks the whole stage: its TMA producer streams the weight tiles of
// every GEMM of every layer into a deep shared-memory ring WITHOUT ever waiting for
// activations (weights do not depend on them), while the activation operand of each k-block
// is loaded by a second producer only once the flag of the data it needs is published:
//   QKV      B = RMSNorm(x)           flag norm_a      (grid-last CTA of the previous down-proj)
//   attention q, K, V of head h       flags qkv[tile]  (the last arriver of each QKV tile)
//   O-proj   B k-block = half a head  flag attn[head]  (the last (seq, chunk) of the head)
//   gate_up  B = RMSNorm(h)           flag norm_f      (grid-last CTA of the O-proj)
//   down     B k-block kb             flag gu[kb]      (gate_up tile kb = act columns of kb)
// so every dependency is a point-to-point flag and the weight stream never stops.
#pragma once
#include "gemm.h"
#include "kernels.h"

namespace hs {

struct DstackArgs {
  int N;                      // sequences (= query tokens) of the step, 1..64
  int H, F, nh, hd;           // model shape
  int nl;                     // layers of the launch (the stage's range)
  float eps;
  // weights: layered TMA maps over the stage arena + per-layer norm vectors
  const TmaMat *wqkv, *wo, *wgu, *wd;
  const bf16* attn_norm;      // layer 0 of the range; layer l at + l * norm_stride
  const bf16* ffn_norm;
  int64_t norm_stride;        // elements
  const bf16* final_norm;     // non-null on the model's last layer: RMSNorm(x) -> fin
  bf16* fin;
  // activations ([N, .] row-major bf16) and their TMA maps (index gemm_bn index)
  const bf16* x_in;           // stage input (embedding rows or the hand-off buffer)
  bf16 *x, *hbuf, *nrm, *q, *o, *act;
  const TmaMat *b_nrm, *b_o, *b_act;
  // paged KV of layer 0 of the range (layer l at + l * pool_stride elements) + call metadata
  bf16* pool;
  int64_t pool_stride;
  int nslots, nblocks, max_blocks;
  const int *pos, *slot, *tables;
  const SeqDesc* seqs;
  const float2* rope;         // RoPE table [max_seq][hd/2] (cos, sin)
  const int* ctx;             // host copy: keys of each sequence after this step (pos0 + 1)
  // test-only capture (hs_debug_capture): non-null => layer l of the range also stores its
  // h = x + o W_o^T at cap + 2l * cap_stride and its output at cap + (2l + 1) * cap_stride
  // ([N, H] bf16 rows each)
  bf16* cap = nullptr;
  int64_t cap_stride = 0;     // elements
};

// Per-stage persistent state (workspaces + flags); create once, reuse every step.
struct DstackState;
// The workspace and counters are zeroed by cudaMemsetAsync on st, the stream the first launch
// goes to (a legacy-stream cudaMemset is not ordered with the library's non-blocking streams:
// run 42 caught one landing after the first launch, which reset c_rows under the next one).
hs_status dstack_create(DstackState** out, int H, int F, int nh, int hd, int max_seqs, int max_ctx, cudaStream_t st);
void dstack_destroy(DstackState* s);
bool dstack_supported(int N, int hd);
hs_status dstack_launch(DstackState* s, const DstackArgs& a, cudaStream_t st);
void warm_dstack();

}  // namespace hs
