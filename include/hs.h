/* hs.h — C ABI of the B200-native HydraServe cold-start path (arXiv 2502.15524).
 *
 * What this library does (§1, lines 88-92; §4; §5.2;
 * §6): a decoder model's layers are range-sharded into a pipeline-parallel
 * group of s stages, one GPU per stage.  Each stage streams its contiguous slice of bf16
 * weights from pinned host memory into HBM in chunks ("pipeline the fetching and loading at
 * tensor granularity"; "obtain tensors in a streaming manner"),
 * and per-layer readiness gates the stage's prefill/decode kernels, so inference starts
 * before loading ends.  Stages hand activations to the next stage ("intermediate results
 * transmitted sequentially") over NVLink peer memory.  Pipeline
 * consolidation ("scaling down"; KV-cache migration PAPER.md:622-643)
 * migrates the weights of the other stages' layers and the paged KV blocks of live
 * sequences into one full-memory stage, which then decodes alone.
 *
 * Conventions (all entry points):
 *  - Every call returns hs_status; HS_OK == 0.  Out-parameters are written only on HS_OK.
 *    hs_last_error() returns a thread-local message describing the last failure.
 *  - Errors are returned, never raised/aborted across the ABI.  HS_E_CUDA is sticky for the
 *    group: the group may only be destroyed afterwards.
 *  - Host pointers are caller-owned.  Device memory, streams and events are library-owned.
 *  - A group is not thread-safe; the caller serialises calls on one group.
 *  - Multi-process (SPMD) mode: one process per stage GPU; every process calls every entry
 *    point with identical arguments (except per-process host buffers).  Cross-process
 *    plumbing (handle exchange, barrier) is supplied by the caller through hs_comm
 *    (e.g. torch.distributed); the data path itself uses CUDA IPC peer memory over NVLink.
 */
#ifndef HS_H_
#define HS_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t hs_status;
enum {
  HS_OK = 0,
  HS_E_INVAL = 1,       /* bad argument / unsupported shape */
  HS_E_CUDA = 2,        /* CUDA runtime/kernel failure; sticky: the group must be destroyed */
  HS_E_OOM = 3,         /* device or pinned-host allocation failed (group left usable) */
  HS_E_INFEASIBLE = 4,  /* no placement satisfies the request (Alg. 1 has no choice) */
  HS_E_STATE = 5,       /* call out of order (e.g. prefill before any load was issued) */
  HS_E_PEER = 6,        /* stage GPUs cannot reach each other over P2P */
  HS_E_TIMEOUT = 7      /* a cross-stage device wait timed out (peer never signalled) */
};

#define HS_MAX_STAGES 8
#define HS_MAX_LAYERS 128

/* Decoder shape.  The paper evaluates the Llama-2 family; this library
 * implements that architecture: pre-norm RMSNorm, multi-head attention with rotate-half
 * RoPE, SiLU-gated MLP, no biases, untied lm_head (reading R1).
 * Requirements: n_kv_heads == n_heads; head_dim in {64,128}; hidden == n_heads*head_dim;
 * hidden % 64 == 0; ffn % 64 == 0; vocab % 16 == 0; n_layers <= HS_MAX_LAYERS. */
typedef struct {
  int32_t n_layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab, max_seq;
  float rms_eps;    /* 1e-5 for Llama-2 */
  float rope_theta; /* 1e4 for Llama-2 */
} hs_model_cfg;

/* ---------------------------------------------------------------------------------------
 * Host weight image ("model file whose metadata header comes first").
 * Byte layout (all offsets from the start of the image, little endian):
 *   [0, HS_IMAGE_HEADER_BYTES)  hs_image_header (host-only metadata, never loaded)
 *   embed region                 embed [vocab, hidden] bf16, row-major
 *   layer region l (l = 0..L-1)  at layer_off[l], layer_bytes long, tensors at t_* offsets:
 *       attn_norm [hidden]; w_qkv [3*hidden, hidden] (rows: q then k then v);
 *       w_o [hidden, hidden]; ffn_norm [hidden];
 *       w_gu [2*ffn, hidden] with gate/up rows interleaved in blocks of gu_interleave:
 *            physical row p: b = p / (2*G), j = p % (2*G); j < G -> gate row b*G + j,
 *            else up row b*G + j - G  (G = gu_interleave = 16);
 *       w_d [hidden, ffn]
 *   final region                 final_norm [hidden] at t_final_norm, lm_head [vocab, hidden]
 *                                at t_lm_head
 * Every weight matrix W [out_features M, in_features K] (w_qkv, w_o, w_gu, w_d, lm_head) is
 * stored in the TILED weight layout [M/128][K/64][128][64]: the 128 x 64 block (row tile i,
 * k-block j) is one contiguous 16 KiB run at block index i * (K/64) + j, rows of 64 elements
 * (128 B) inside it (M % 128 == 0, K % 64 == 0).  That block is exactly one tensor-core operand
 * tile (TMA box 64 x 128, 128B swizzle), so weight streaming reads whole contiguous 16 KiB runs
 * (measured: 6.9-7.1 TB/s vs 5.7-5.9 TB/s for 128-byte row segments of a row-major matrix,
 * profiles/r02/stream_probe.txt).  The embedding table stays row-major [vocab, hidden] (it is
 * gathered by rows, not streamed).  Regions are HS_IMAGE_ALIGN aligned, so a stage's slice
 * [embed|layers b..e-1|final] is one contiguous byte range.
 * ------------------------------------------------------------------------------------- */
#define HS_IMAGE_MAGIC 0x31474D49534853ULL /* "SHSIMG1" */
#define HS_IMAGE_HEADER_BYTES 65536ULL
#define HS_IMAGE_ALIGN 65536ULL
#define HS_TENSOR_ALIGN 256ULL
#define HS_GU_INTERLEAVE 16

typedef struct {
  uint64_t magic;
  uint32_t version;       /* 2 (tiled weight matrices) */
  uint32_t gu_interleave; /* HS_GU_INTERLEAVE */
  hs_model_cfg cfg;
  uint64_t total_bytes;   /* whole image incl. header */
  uint64_t embed_off, embed_bytes;
  uint64_t layer_off[HS_MAX_LAYERS];
  uint64_t layer_bytes;   /* padded region size of one layer */
  uint64_t t_attn_norm, t_wqkv, t_wo, t_ffn_norm, t_wgu, t_wd; /* offsets inside a layer */
  uint64_t final_off, final_bytes;
  uint64_t t_final_norm, t_lm_head; /* offsets inside the final region */
  uint64_t param_bytes;   /* sum of tensor bytes (no padding): 2 * #params */
} hs_image_header;

/* A (slice of a) host image: data covers image bytes [data_offset, data_offset+data_bytes).
 * data should be pinned (cudaHostAlloc / cudaHostRegister); pageable memory works but the
 * copy engine then cannot stream it asynchronously.  Caller-owned; must stay valid until
 * every load issued from it has completed (hs_stage_load_stats) and every prefill issued
 * while that load was in flight has returned (a prefill reads its prompt's embedding rows
 * from a pinned, device-mapped image while the table is still streaming), or until the group
 * is destroyed. */
typedef struct {
  const hs_image_header* header;
  const void* data;
  uint64_t data_offset;
  uint64_t data_bytes;
  /* Optional 8-byte "fetched end" watermark of a region still being filled by the model
   * prefetcher (hs_prefetch_start): image offset up to which data is valid,
   * in mapped pinned memory.  NULL = the whole range is resident.  Every H2D chunk waits on the
   * device (cuStreamWaitValue64 on the copy stream) until the watermark covers it, and a prefill
   * reading embedding rows from the host image waits until the embedding region is covered. */
  const uint64_t* fetched_end;
} hs_image;

/* ---------------------------------------------------------------------------------------
 * Model prefetcher (§5.1): "the prefetcher starts to load the model
 * weights from remote storage to a shared memory region ... we use the first eight bytes to
 * store the address that represents the end of currently fetched model weights".  A library
 * thread reads bytes [file_offset, file_offset + bytes) of the model file at `path` (the host
 * image's byte layout: header first, then the regions in image order) into dst (caller-owned
 * pinned memory holding those image bytes), chunk_bytes at a time (0 = 8 MiB), and after each
 * chunk stores the image offset of the fetched end into *watermark with release semantics
 * (watermark: 8 bytes of mapped pinned memory; pass it as hs_image.fetched_end so the loader
 * streams each chunk to HBM as soon as it is fetched).  max_gbps > 0 throttles the reads to that
 * rate (emulating remote storage: Eq. 1's b).  Errors: HS_E_INVAL (cannot open the file).
 * hs_prefetch_wait joins the thread (HS_E_INVAL if the file was short / unreadable; the
 * watermark then stays at the last complete chunk); hs_prefetch_destroy stops and frees it. */
typedef struct hs_prefetch hs_prefetch;
hs_status hs_prefetch_start(const char* path, uint64_t file_offset, void* dst, uint64_t bytes,
                            uint64_t chunk_bytes, double max_gbps, uint64_t* watermark,
                            hs_prefetch** out);
hs_status hs_prefetch_wait(hs_prefetch* p, uint64_t* fetched, double* seconds);
hs_status hs_prefetch_destroy(hs_prefetch* p);

/* Computes the image layout for cfg (host only).  total_bytes etc. filled in. */
hs_status hs_image_layout(const hs_model_cfg* cfg, hs_image_header* out);

/* ---------------------------------------------------------------------------------------
 * Planning (§4.1; Eq. 1; Eq. 5).
 * ------------------------------------------------------------------------------------- */
typedef struct {
  int32_t device;     /* CUDA ordinal (as seen by the process that will own the stage) */
  double h2d_gbps;    /* p_i: host->device bandwidth of this GPU's link, GB/s (10^9 B/s) */
  int32_t link_group; /* GPUs sharing one host uplink share a group id (hs_links_*) */
  uint64_t free_bytes;/* free HBM */
  int32_t n_workers;  /* workers already running on this GPU (Alg. 1's "GPU sharing") */
} hs_gpu;

typedef struct {
  int32_t pp;                            /* s */
  int32_t device[HS_MAX_STAGES];         /* g, in stage order */
  int32_t layer_begin[HS_MAX_STAGES];    /* [b_k, e_k) */
  int32_t layer_end[HS_MAX_STAGES];
  uint64_t stage_bytes[HS_MAX_STAGES];   /* weight bytes each stage must load (image ranges) */
  uint64_t slice_begin[HS_MAX_STAGES];   /* image byte range of the stage slice */
  uint64_t slice_end[HS_MAX_STAGES];
  int32_t full_memory[HS_MAX_STAGES];    /* w flags: stage reserves whole-model memory */
  double pred_ttft_s;                    /* Eq. 5 specialised (R9) */
} hs_plan;

/* Builds a plan for pp stages (1..HS_MAX_STAGES; pp = 0 is reserved for SLO-driven choice).
 * Layers are split into contiguous ranges, floor(L/pp) each, the remainder going to the
 * earliest stages; stage 0 holds the embedding, the last stage the final norm + lm_head.
 * GPUs are chosen by the paper's selection rule (smallest 1/p_i first, PAPER.md:408-413;
 * remote fetch 1/b_i = 0 here) with full_memory_stages stages reserving the whole model
 * (Alg. 1's w).  Stage 0 is always full-memory when full_memory_stages >= 1, so it can be
 * the consolidation target.  t_prefill_s / t_hop_s are Eq. 5's t_p, t_n (may be 0).
 * Errors: HS_E_INVAL (bad cfg/pp), HS_E_INFEASIBLE (not enough GPUs or memory). */
hs_status hs_plan_stages(const hs_model_cfg* cfg, const hs_gpu* gpus, int32_t n_gpus,
                         int32_t pp, int32_t full_memory_stages, double t_prefill_s,
                         double t_hop_s, hs_plan* out);

/* SLO-driven choice of s and w (Algorithm 1) on one box: for s = 1..max_pp
 * and w = 0..s the GPUs are chosen by hs_plan_stages' selection rule, TTFT is Eq. 5 specialised
 * (R9) and TPOT is Eq. 2 (t_d, t_n); among the SLO-feasible choices the one whose
 * GPUs already host the fewest workers wins (ties: smaller s, then larger w).  If none is
 * feasible, out = (1, 1, best full-capable GPU) and HS_E_INFEASIBLE is returned (the paper's
 * "use single worker if no solution").  sharing (optional) = workers already on the chosen
 * GPUs. */
typedef struct {
  double t_prefill_s, t_decode_s, t_hop_s; /* t_p, t_d, t_n (historical measurements) */
  double slo_ttft_s, slo_tpot_s;
  int32_t max_pp;                          /* paper: 4; north star: up to 8 */
} hs_slo;
hs_status hs_plan_auto(const hs_model_cfg* cfg, const hs_gpu* gpus, int32_t n_gpus,
                       const hs_slo* slo, hs_plan* out, int32_t* sharing);

/* Contention-aware admission of simultaneous cold starts sharing a host link group
 * (§4.2, Eq. 3, Eq. 4; R17: the paper's per-server
 * network bandwidth B becomes the bandwidth of a group of GPUs behind one host uplink).
 * Units: bytes and seconds.  admit settles the group to `now` first, then accepts iff
 * S_i <= B/(N+1) (D_i - now) for every listed worker and the candidate; settle applies
 * S_i' = S_i - B/N (now - T') and drops workers with S_i' < 0. */
typedef struct hs_links hs_links;
hs_status hs_links_create(int32_t n_groups, const double* group_bytes_per_s, hs_links** out);
hs_status hs_links_admit(hs_links* l, int32_t group, double pending_bytes, double deadline_s,
                         double now_s, int32_t* accepted, int64_t* worker_id);
hs_status hs_links_settle(hs_links* l, int32_t group, double now_s);
hs_status hs_links_complete(hs_links* l, int32_t group, int64_t worker_id, double now_s);
hs_status hs_links_pending(hs_links* l, int32_t group, int32_t max_n, int32_t* n,
                           double* pending, int64_t* ids);
hs_status hs_links_destroy(hs_links* l);

/* Contention-aware placement of one cold start arriving at now_s (DESIGN.md
 * R20): Algorithm 1's selection over s = 1..max_pp on the contention-adjusted links (GPU i's
 * p'_i = min(p_i, B_g / (N_g + 1)), N_g = loads recorded on its link group g), low-memory stages
 * (w = 0), TTFT_pred(s) = max_k stage_bytes_k / min(p_k, B_g / (N_g + s_g)); admissible iff
 * TTFT_pred <= slo_ttft_s and every load already on a touched group still meets its deadline
 * under the new share (Eq. 3); the admissible candidate with the smallest prediction wins (else
 * the smallest prediction).  The chosen stages are recorded in `links` as workers (pending =
 * stage bytes, deadline = now_s + TTFT_pred); worker_ids (optional, [pp]) receive their ids
 * (hs_links_complete them when the load ends, or let Eq. 4 retire them).  gpus[i].link_group
 * indexes `links`; gpus[i].h2d_gbps = p_i (GB/s); link group bandwidths are bytes/s.
 * Errors: HS_E_INVAL, HS_E_INFEASIBLE (no GPU set holds the model). */
hs_status hs_place_cold_start(const hs_model_cfg* cfg, const hs_gpu* gpus, int32_t n_gpus, hs_links* links,
                              double now_s, double slo_ttft_s, int32_t max_pp, hs_plan* out,
                              double* pred_ttft_s, int32_t* admitted, int64_t* worker_ids);

/* Paper's predictors, exposed for the planner's tests (PAPER.md:398 Eq. 1, :417 Eq. 2,
 * :579-584 Eq. 5).  Bandwidth arrays have s entries; M in the same unit as b,p numerators. */
double hs_predict_ttft_eq1(double t_c, double M, int32_t s, int32_t w, const double* b,
                           const double* p, double t_p, double t_n);
double hs_predict_tpot_eq2(double t_d, int32_t s, int32_t w, double t_n);
double hs_predict_ttft_eq5(double t_cc, double t_cu, double t_l, double M, int32_t s,
                           int32_t w, const double* b, const double* p, double t_p,
                           double t_n);

/* ---------------------------------------------------------------------------------------
 * Groups.
 * ------------------------------------------------------------------------------------- */
typedef struct {
  int32_t block_tokens; /* 16 (only value supported) */
  int32_t num_blocks;   /* KV blocks per layer pool, identical ids on every stage */
  int32_t max_seqs;     /* max live sequences (block-table rows) */
  int32_t max_tokens;   /* max tokens in one prefill call (activation buffers) */
} hs_kv_cfg;

/* Cross-process plumbing for SPMD mode (NULL comm => every stage is driven by this process).
 * allgather: each of world ranks contributes `bytes` bytes; recv gets world*bytes in rank
 * order.  barrier: all ranks.  Both return 0 on success. */
typedef struct {
  int32_t rank;   /* == the stage index this process owns */
  int32_t world;  /* == plan->pp */
  void* ctx;
  int32_t (*allgather)(void* ctx, const void* send, uint64_t bytes, void* recv);
  int32_t (*barrier)(void* ctx);
} hs_comm;

typedef struct hs_group hs_group; /* opaque, library-owned */

/* Creates the group: per owned stage sets the device, enables peer access, allocates the
 * weight arena (slice, or whole model for full-memory stages), the per-layer KV pools
 * ([num_blocks][K|V][heads][16][head_dim] bf16 per layer), activation buffers, streams
 * (compute high priority, copy), per-layer readiness events, and warms the kernels.  All
 * before T0 (R3).  image: whole-model image (or, in SPMD mode, one covering this
 * rank's slice); stage_images: optional [pp] per-stage images (NULL => use image).
 * Errors: HS_E_INVAL, HS_E_OOM, HS_E_PEER, HS_E_CUDA. */
hs_status hs_group_create(const hs_model_cfg* cfg, const hs_plan* plan,
                          const hs_image* image, const hs_image* stage_images,
                          const hs_kv_cfg* kv, const hs_comm* comm, hs_group** out);

/* Issues the chunked H2D load of a stage's slice (critical order: layers b..e-1 in order,
 * final norm + lm_head, then the embedding table, which only decode steps wait for; with an
 * unmapped image the embedding goes first) and returns immediately; each layer's readiness
 * event is recorded after its last chunk.  chunk_bytes = 0 => 32 MiB.  Calling it again
 * re-loads (used by benchmarks).  In SPMD mode only the owned stage is issued; stage = -1
 * means "every stage this process owns".  Errors: HS_E_INVAL, HS_E_CUDA. */
hs_status hs_load_stage_async(hs_group* g, int32_t stage, uint64_t chunk_bytes);

typedef struct {
  uint64_t bytes;         /* bytes copied host->device by the last load */
  float load_ms;          /* device time from first chunk start to last chunk end */
  int32_t layers_ready;   /* layers of this stage whose readiness event has fired */
  int32_t done;           /* 1 when the whole slice is resident */
} hs_load_stats;
/* Non-blocking when wait == 0 (reports progress); wait != 0 blocks until the load ends. */
hs_status hs_stage_load_stats(hs_group* g, int32_t stage, int32_t wait, hs_load_stats* out);

/* Prefill n_seqs prompts (packed tokens, lengths seq_lens) through all stages; returns the
 * greedy first token of each sequence (ties -> lowest id).  May be called right after
 * hs_load_stage_async: readiness is enforced on the device.  out_logits ([n_seqs*vocab]
 * fp32, may be NULL) is written only by the process owning the last stage.  Sequence ids
 * are caller-chosen and must not be live.  Errors: HS_E_INVAL, HS_E_STATE (no load issued),
 * HS_E_OOM (KV blocks exhausted), HS_E_CUDA, HS_E_TIMEOUT. */
hs_status hs_prefill(hs_group* g, int32_t n_seqs, const int64_t* seq_ids,
                     const int32_t* tokens, const int32_t* seq_lens, int32_t* out_tokens,
                     float* out_logits);

/* One greedy decode step for n_seqs live sequences: in_tokens[i] is appended at position
 * ctx_i (in_tokens == NULL => the tokens produced by the previous prefill/decode call for
 * the same seq_ids, fed back on the device).  Each stage runs all its layers in one
 * persistent kernel launch (the decode stack, n_seqs <= 64; HS_DSTACK=0 or larger batches:
 * five kernels per layer), then hands off / samples.  Errors as hs_prefill; HS_E_INVAL for
 * a sequence never prefilled. */
hs_status hs_decode_step(hs_group* g, int32_t n_seqs, const int64_t* seq_ids,
                         const int32_t* in_tokens, int32_t* out_tokens, float* out_logits);

/* n_steps greedy decode steps of n_seqs live sequences with the batch split into n_micro
 * micro-batches ("virtual engines"; the per-stage t_d and t_n terms of Eq. 2,
 * PAPER.md:416-418, overlap across micro-batches): micro-batch j of step t runs on stage k while
 * stage k + 1 runs micro-batch j - 1, and the first stage starts micro-batch j of step t + 1 as
 * soon as the last stage has sampled its tokens (device feedback), so with n_micro >= pp every
 * stage streams its weights without waiting for the others.  Micro-batches are contiguous runs of
 * whole 4-sequence groups (n_micro is clamped to ceil(n_seqs / 4) and 8).  in_tokens: the first
 * step's input tokens, or NULL for device feedback from the previous call (same seq_ids order).
 * out_tokens [n_steps][n_seqs] receives every step's greedy tokens; in SPMD mode it is written
 * on the ranks owning the first and the last stage only.  Afterwards the group is in the same
 * state as after n_steps hs_decode_step calls (device feedback continues).  Each micro-batch's
 * decode stack launch sees only its own sequences, so its per-sequence results equal an
 * hs_decode_step call on the same micro-batch.  Layer-boundary capture (hs_debug_capture) does not
 * record this call.  Errors as hs_decode_step. */
hs_status hs_decode_steps(hs_group* g, int32_t n_seqs, const int64_t* seq_ids, const int32_t* in_tokens,
                          int32_t n_steps, int32_t n_micro, int32_t* out_tokens);

hs_status hs_release_seq(hs_group* g, int64_t seq_id);

typedef struct {
  uint64_t weight_bytes; /* weight bytes migrated into the target over NVLink */
  uint64_t kv_bytes;     /* KV bytes migrated into the target */
  double seconds;        /* device time of the migration (first copy start .. last end) */
  double pause_seconds;  /* host time from call entry to return (drain + migrate + rebind) */
  uint64_t weight_bytes_host; /* weight bytes that arrived by the background host load */
  uint64_t weight_bytes_background; /* weight bytes pulled from peers before the call (hs_pull_background_async) */
} hs_consolidate_stats;

/* Paper-faithful background load ("the
 * parameter manager loads the second part of model in background ... in low-priority CUDA
 * streams"): the full-memory target stage streams the weight regions it lacks from its own
 * host image over its own PCIe link, queued behind its critical load, while the group keeps
 * serving pipelined.  A later hs_consolidate waits for it and then moves only the KV blocks
 * (and any region not covered) over NVLink.  The target's image must cover the whole model.
 * Errors: HS_E_INVAL (target not full-memory / not owned / image too small), HS_E_STATE. */
hs_status hs_load_background_async(hs_group* g, int32_t target_stage, uint64_t chunk_bytes);

/* The same background step with the other stages' HBM as the source ("allowing
 * only one of them to fetch the unloaded model parts in background"): the full-memory target
 * pulls every other stage's weight slice over NVLink with copy-engine peer copies on its
 * low-priority copy stream (chunk_bytes per copy, 0 = 64 MiB) while the group keeps serving
 * pipelined; hs_consolidate then waits for it and moves only the KV blocks, so its pause is the
 * KV copy alone (stats.weight_bytes_background reports the pulled bytes).  Call it after the
 * first hs_prefill has returned (every source slice is then resident; SPMD: on every rank, only
 * the target's rank copies).  Errors: HS_E_INVAL (target not full-memory), HS_E_STATE (no call
 * yet, or a background load already issued). */
hs_status hs_pull_background_async(hs_group* g, int32_t target_stage, uint64_t chunk_bytes);

/* Scale-down consolidation: drain in-flight work, copy the
 * weight regions the target lacks and gather the used KV blocks of every live sequence
 * for the other stages' layers into the target's pools (same block ids), rebind the
 * target to all layers, release the other stages.  The target must be full_memory.
 * Afterwards the group is single-stage.  Errors: HS_E_INVAL (target not full-memory),
 * HS_E_STATE, HS_E_CUDA. */
hs_status hs_consolidate(hs_group* g, int32_t target_stage, hs_consolidate_stats* out);

/* Scale-up consolidation ("converting all cold-start
 * workers into individual serving endpoints"): every stage becomes a standalone single-stage
 * group holding the whole model.  Each stage pulls the weight slices it lacks from the other
 * stages over NVLink (an all-gather: every GPU receives (s-1)/s of the model concurrently) and
 * the KV blocks, for the layers it lacks, of the live sequences assigned to it (same block
 * ids).  seq_owner[i] is the endpoint (stage index) of the i-th live sequence in ascending
 * seq-id order (NULL: round-robin).  Every stage must be full-memory.  On success the group
 * is emptied (destroy it) and out[k] (local mode: k = 0..pp-1; SPMD: out[0] = this rank's
 * endpoint) receive the new groups; stats (optional) sums the migrated bytes.
 * Errors: HS_E_INVAL (a stage not full-memory, bad owner), HS_E_STATE, HS_E_CUDA. */
hs_status hs_scale_up(hs_group* g, const int32_t* seq_owner, int32_t n_live, hs_group** out,
                      hs_consolidate_stats* stats);

/* SPMD, collective: frees the HBM that consolidation released on the non-target ranks.  The
 * released stages' arena / KV / comm memory is exported to peers over CUDA IPC, and an exporter
 * may free it only after every importer has closed its mapping (closing multi-GB mappings costs
 * ~100 ms, so hs_consolidate defers it off the decode pause).  Each rank closes its deferred
 * mappings, meets at hs_comm.barrier, then frees its released memory.  ALWAYS collective in SPMD
 * mode: every rank must call it (also when it has nothing pending), because every rank enters the
 * barrier.  Local mode: frees the released stages' memory (consolidation defers those driver frees
 * off the pause too), no barrier.  hs_group_destroy does it too.  Errors: HS_E_INVAL (NULL),
 * HS_E_STATE (the barrier failed: the exported regions are then left allocated, never freed under
 * a peer's mapping; everything else is released). */
hs_status hs_release_peer_memory(hs_group* g);

/* Frees everything the group owns.  SPMD: collective (every rank calls it on the same group,
 * also after an HS_E_CUDA failure); the ranks close their CUDA-IPC mappings of peer memory,
 * meet at hs_comm.barrier, then free their own memory, so no exporter frees a region a peer
 * still maps.  If the barrier fails the exported regions stay allocated (leaked for the life of
 * the process) and HS_E_STATE is returned; the group is freed in every case.  After
 * hs_scale_up, destroy the emptied group (which holds the peer mappings) before the endpoints.
 * NULL is a no-op. */
hs_status hs_group_destroy(hs_group* g);
const char* hs_last_error(void);

/* Current pipeline degree (1 after consolidation) and the stage index owned by this process
 * (SPMD) or -1 (local mode). */
hs_status hs_group_info(hs_group* g, int32_t* pp, int32_t* owned_stage);

/* ---- test / benchmark helpers (not part of the serving path) ---- */
/* Reads KV of one sequence, layer, positions [pos0,pos0+n_pos) from the stage that holds
 * the layer: host_out [n_pos][2][n_heads][head_dim] bf16.  Blocking. */
hs_status hs_debug_read_kv(hs_group* g, int64_t seq_id, int32_t layer, int32_t pos0,
                           int32_t n_pos, void* host_out);
/* Layer-boundary capture (test-only; the parity tests compare every half of every decoder
 * layer on its own: a PP group computes exactly the unpartitioned layers).
 * enable != 0 allocates, per stage this process drives, a device buffer of
 * (2 n_layers + 1) x max_tokens x hidden bf16 and makes every later hs_prefill /
 * hs_decode_step store the hidden state of every token at every capture point it computes:
 * point 2l is the input of layer l (point 0 = the embedding rows, point 2L = the last layer's
 * output, the final RMSNorm's input); point 2l + 1 is layer l's h = x + Attention(RMSNorm(x)) W_o^T
 * (the residual stream between the attention and the MLP halves).  Same kernels and launch
 * configuration as without capture: the decode stack writes the extra copies from its O- and
 * down-projection epilogues; the per-kernel path copies behind each layer.  enable == 0 frees
 * the buffers.  Errors: HS_E_INVAL, HS_E_OOM. */
hs_status hs_debug_capture(hs_group* g, int32_t enable);
/* Copies capture point `point` (0..2 n_layers) of rows [row0, row0 + n_rows) of the LATEST call
 * to host_out ([n_rows][hidden] bf16).  Rows are in call order: hs_prefill's packed tokens
 * (sequence by sequence, as passed), or one row per sequence for hs_decode_step, whatever
 * micro-batch layout the call used on the device.  Blocking.  Errors: HS_E_STATE (capture
 * off), HS_E_INVAL (rows outside the latest call, or the point lives on a stage driven by
 * another process). */
hs_status hs_debug_read_hidden(hs_group* g, int32_t point, int32_t row0, int32_t n_rows, void* host_out);
/* Prefill micro-batching knobs (tests and A/B measurements; defaults are the product): a
 * prefill is cut into nchunks = max(1, min(max_chunks, shortest prompt / 16, T / min_chunk_tokens))
 * micro-batches (0 = default: max_chunks 4, min_chunk_tokens 1024).  max_chunks = 1 disables
 * micro-batching.  The choice depends on the call's shapes only, never on the number of stages.
 * Errors: HS_E_INVAL. */
hs_status hs_debug_set_prefill_chunking(hs_group* g, int32_t min_chunk_tokens, int32_t max_chunks);
/* Copies bytes [image_off, image_off+bytes) of the device weight arena of `stage` to host. */
hs_status hs_debug_read_weights(hs_group* g, int32_t stage, uint64_t image_off,
                                uint64_t bytes, void* host_out);
/* Fills a stage's weight arena with 0xFF (bf16 NaN) so a missing readiness wait shows up. */
hs_status hs_debug_poison_weights(hs_group* g, int32_t stage);
/* Number of kernels this library has launched (process-wide, since load). */
hs_status hs_debug_launch_count(hs_group* g, uint64_t* out);

/* ---- measurement (benchmarks) ---- */
/* Device-event timing of a stage for the most recent load and call: load_ms = first chunk ..
 * last chunk (copy engine); call_ms = start .. end of this stage's work in the last
 * prefill/decode call; since_load_ms = load start .. end of the last call (for the prefill
 * issued right after the load this is the device-side TTFT seen by that stage). */
typedef struct { float load_ms, call_ms, since_load_ms; } hs_stage_timing;
hs_status hs_stage_timing_get(hs_group* g, int32_t stage, hs_stage_timing* out);

/* Per-kernel-kind CUDA-event profile (off by default).  While enabled, every kernel the
 * group launches is bracketed by events on its stream; hs_profile_read synchronises and
 * returns, per kind, the launch count, summed device milliseconds and the algorithmic bytes
 * and flops of those launches. */
typedef struct { char name[32]; uint64_t count; double ms, bytes, flops; } hs_prof_entry;
hs_status hs_profile_enable(hs_group* g, int32_t on);
hs_status hs_profile_read(hs_group* g, hs_prof_entry* out, int32_t max_entries, int32_t* n,
                          int32_t reset);

/* Test-only: exercises the SPMD plumbing (allgather of rank-tagged bytes + barrier through
 * the caller's callbacks) without any device work; returns HS_OK if every rank's bytes came
 * back in rank order. */
hs_status hs_debug_comm_selftest(const hs_comm* comm);

#ifdef __cplusplus
}
#endif
#endif /* HS_H_ */
