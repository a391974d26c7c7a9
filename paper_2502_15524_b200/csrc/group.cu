// group.cu — the pipeline-parallel worker group: device arenas, chunked H2D streaming with
// per-layer readiness (a2-a4), the stage forward (a5-a15), decode (a16), consolidation (a17),
// local (one process drives every stage GPU) and SPMD (one process per stage GPU, CUDA IPC
// peer memory) modes.  See include/hs.h for the contract of every entry point.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <vector>

#include "common.h"
#include "dstack.h"
#include "gemm.h"
#include "kernels.h"

namespace hs {

static std::atomic<uint64_t> g_launches{0};
void count_launch(uint64_t n) { g_launches += n; }
uint64_t launch_total() { return g_launches.load(); }

int num_sms(int device) {
  static int cache[64] = {};
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cache[device] = v > 0 ? v : 148;
  }
  return cache[device];
}

static constexpr int kBlock = 16;
static constexpr uint64_t kDefaultChunk = 32ull << 20;
static constexpr uint64_t kWorkspace = 64ull << 20;
static constexpr int kSendCtas = 64;
static constexpr uint64_t kCounters = 1 << 16;
static constexpr int kMaxChunks = 4;       // prefill micro-batches
static constexpr int kChunkTokens = 1024;  // minimum tokens per micro-batch
static constexpr int kMaxMicro = 8;        // decode micro-batches ("virtual engines") per call

// Comm block of a stage (one allocation, shared with peers): flags + token / hidden inputs.
struct CommLayout {
  static constexpr size_t FLAG_X = 0, FLAG_TOK = 4, DONE = 8, ERR = 12;
  size_t tok_in = 256, x_in = 0, bytes = 0;
  void init(int max_seqs, int max_tokens, int H) {
    x_in = align_up(tok_in + (size_t)align_up(max_seqs * 4, 16) + 16, 256);
    bytes = x_in + (size_t)max_tokens * H * 2;
  }
};

struct LayerDev {
  const bf16 *attn_norm = nullptr, *ffn_norm = nullptr;
  TmaMat wqkv, wo, wgu, wd;
  bool maps = false;
};

struct Share {  // what a stage publishes to its peers (SPMD allgather)
  cudaIpcMemHandle_t comm, arena, kv;
  uint64_t arena_off0, arena_bytes, kv_layer_bytes;
  int32_t kv_lb, kv_le;  // layers whose pools exist in kv
  int32_t device;
};

struct Stage {
  int idx = 0, device = 0;
  bool owned = false;       // driven by this process
  bool full_memory = false;
  int lb = 0, le = 0;       // current layer range
  uint64_t slice_begin = 0, slice_end = 0;
  // memory (owned stages: allocated here; remote stages: IPC-mapped, opened lazily)
  uint8_t* arena = nullptr;
  uint64_t arena_off0 = 0, arena_bytes = 0;
  uint8_t* kv_mem = nullptr;
  int kv_lb = 0, kv_le = 0;
  uint8_t* comm = nullptr;
  bool ipc_arena_open = false, ipc_comm_open = false;
  Share share{};
  // work buffers (owned)
  float* nrm_rs = nullptr;  // row scales of s.nrm's rows (reading R10b: s.nrm = bf16(x * w))
  bf16 *xa = nullptr, *xb = nullptr, *nrm = nullptr, *qkv = nullptr, *q = nullptr, *o = nullptr,
       *act = nullptr, *fin = nullptr;
  float *logits = nullptr, *ws = nullptr, *attn_ws = nullptr;
  unsigned* ctr = nullptr;  // stream-K / attention arrival counters (zeroed; self-resetting)
  float2* rope = nullptr;
  uint8_t* d_meta = nullptr;
  uint8_t* h_meta = nullptr;  // pinned staging
  int* h_out = nullptr;       // pinned: tokens + err
  size_t meta_bytes = 0;
  int* d_tok_out = nullptr;
  cudaStream_t comp = nullptr, copy = nullptr;
  cudaEvent_t ev_embed = nullptr, ev_final = nullptr, ev_l0 = nullptr, ev_l1 = nullptr;
  cudaEvent_t ev_c0 = nullptr, ev_c1 = nullptr;  // start / end of the last call on comp
  cudaEvent_t ev_bg0 = nullptr, ev_bg = nullptr; // background (host path) load start / end
  bool bg_issued = false;   // weights the target lacks are being loaded in the background
  bool bg_from_peers = false;  // ... from the other stages' HBM over NVLink (else its host image)
  uint64_t bg_bytes = 0;
  bool called = false;
  std::vector<cudaEvent_t> ev_layer;
  bool load_issued = false;
  bool owns_streams = true;  // stages on one device share its streams (stream-ordered hand-off)
  uint64_t loaded_bytes = 0;
  std::vector<LayerDev> layers;
  TmaMat lm;
  TmaMat b_nrm[5], b_o[5], b_act[5], b_fin[5];
  const hs_image* img = nullptr;
  const bf16* host_embed = nullptr;  // device-accessible (UVA-mapped) embedding table in the host image
  // decode stack (dstack.h): workspace + layered weight maps of the current layer range
  DstackState* ds = nullptr;
  TmaMat ds_w[4];
  int ds_lb = -1, ds_le = -1;
  const void* ds_arena = nullptr;
  bf16* cap = nullptr;  // test-only capture [2 n_layers + 1][max_tokens][hidden] (hs_debug_capture)
  // consolidation copy list of a full-memory stage (a possible target), prepared before T0:
  // [0, cons_nw) the weight slices of every other stage (pieces, prebuilt at create),
  // [cons_nw, ...) the used KV blocks of the live sequences (written at the call)
  CopyDesc* cons_d = nullptr;  // device
  CopyDesc* cons_h = nullptr;  // pinned staging
  int cons_cap = 0, cons_nw = 0;
  cudaEvent_t ev_cons0 = nullptr, ev_cons1 = nullptr;

  uint8_t* wptr(uint64_t image_off) const { return arena + (image_off - arena_off0); }
  bf16* kv_pool(int l, uint64_t layer_bytes) const {
    return reinterpret_cast<bf16*>(kv_mem + (uint64_t)(l - kv_lb) * layer_bytes);
  }
  unsigned* flag_x() const { return reinterpret_cast<unsigned*>(comm + CommLayout::FLAG_X); }
  unsigned* flag_tok() const { return reinterpret_cast<unsigned*>(comm + CommLayout::FLAG_TOK); }
  unsigned* done() const { return reinterpret_cast<unsigned*>(comm + CommLayout::DONE); }
  int* err() const { return reinterpret_cast<int*>(comm + CommLayout::ERR); }
};

struct SeqState {
  std::vector<int> blocks;
  int ctx = 0;
};

struct VeBuffers {
  uint8_t* h = nullptr;  // pinned staging, R slots
  uint8_t* d = nullptr;  // device, R slots
  size_t slot_bytes = 0;
  int slots = 0;
  std::vector<cudaEvent_t> ev;
  int* h_tok = nullptr;  // pinned token log [n_steps][align(n, 4)]
  size_t tok_cap = 0;
};

}  // namespace hs

struct hs_group {
  hs_model_cfg cfg;
  hs_plan plan;
  hs_kv_cfg kv;
  hs_image_header hdr;
  bool spmd = false;
  hs_comm comm{};
  int owned_stage = -1;
  bool dead = false;
  bool comm_failed = false;  // an hs_comm callback failed: collective teardown cannot be agreed on
  std::vector<hs::Stage> st;
  std::vector<int> active;  // stage indices in pipeline order
  hs::CommLayout cl;
  uint64_t kv_layer_bytes = 0, kv_block_bytes = 0;
  int max_blocks = 0;  // per sequence
  // centralised block manager (identical on every rank)
  std::set<int> free_blocks;
  std::map<int64_t, hs::SeqState> seqs;
  std::vector<int64_t> last_ids;  // seq order of the previous call (device token feedback)
  // test-only layer-boundary capture (hs_debug_capture / hs_debug_read_hidden): buffer row of
  // each token of the latest call (call order), and the stage that stored each boundary
  int chunk_tokens = 0, max_chunks = 0;  // prefill micro-batching knobs (0 = defaults)
  std::map<int, hs::VeBuffers> ve;       // hs_decode_steps staging per owned stage
  bool capture = false;
  std::vector<int> cap_rowmap;
  std::vector<int> cap_owner;
  unsigned epoch = 0;
  // per-kernel-kind event profile (hs_profile_*)
  bool prof_on = false;
  struct ProfRec { int kind; int device; cudaEvent_t a, b; double bytes, flops; };
  std::vector<ProfRec> prof;
  std::map<int, std::vector<cudaEvent_t>> ev_free;  // per device
  struct ProfAcc { uint64_t count = 0; double ms = 0, bytes = 0, flops = 0; };
  std::map<int, ProfAcc> prof_acc;
  std::vector<void*> ipc_deferred;  // peer mappings of released stages, closed at destroy
  // SPMD: this rank's exported arena / KV / comm memory of a released stage, freed only after
  // every importer has closed its mapping (hs_release_peer_memory or destroy)
  std::vector<std::pair<int, void*>> exp_deferred;  // (device, pointer)
  // SPMD: the rest of a released stage's teardown (buffers, streams, events, comm mapping) also
  // waits for the release point, so consolidation's pause makes no driver free/unmap calls
  std::vector<hs::Stage> stage_deferred;
};

namespace hs {

static hs_status stage_of_layer(hs_group* g, int layer, int* out) {
  for (int k : g->active)
    if (layer >= g->st[k].lb && layer < g->st[k].le) { *out = k; return HS_OK; }
  HS_FAIL(HS_E_INVAL, "layer %d not held by any active stage", layer);
}

// SPMD barrier through the caller's callback; a failure is remembered (teardown then cannot
// agree with the peers and keeps exported memory alive rather than free it under a mapping).
static bool comm_barrier(hs_group* g) {
  if (!g->spmd) return true;
  if (g->comm_failed || !g->comm.barrier || g->comm.barrier(g->comm.ctx) != 0) {
    g->comm_failed = true;
    return false;
  }
  return true;
}

// ---- per-kernel-kind profile ------------------------------------------------------------
enum ProfKind { PK_EMBED, PK_RMSNORM, PK_GEMM_QKV, PK_ROPE_KV, PK_ATTN, PK_GEMM_O, PK_GEMM_GU, PK_GEMM_DOWN,
                PK_LM_HEAD, PK_ARGMAX, PK_SEND, PK_WAIT, PK_DSTACK, PK_N };
static const char* kProfNames[PK_N] = {"embed", "rmsnorm", "gemm_qkv", "rope_kv", "attention", "gemm_o",
                                       "gemm_gate_up", "gemm_down", "gemm_lm_head", "argmax", "send", "wait",
                                       "decode_stack"};

static cudaEvent_t prof_event(hs_group* g, int dev) {
  auto& v = g->ev_free[dev];
  if (!v.empty()) { cudaEvent_t e = v.back(); v.pop_back(); return e; }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {
  hs_group* g; Stage& s; int kind; double bytes, flops; cudaEvent_t a = nullptr;
  ProfScope(hs_group* g_, Stage& s_, int kind_, bool decode, double bytes_, double flops_)
      : g(g_), s(s_), kind(kind_ * 2 + (decode ? 1 : 0)), bytes(bytes_), flops(flops_) {
    if (g->prof_on) { a = prof_event(g, s.device); cudaEventRecord(a, s.comp); }
  }
  ~ProfScope() {
    if (!a) return;
    cudaEvent_t b = prof_event(g, s.device);
    cudaEventRecord(b, s.comp);
    g->prof.push_back({kind, s.device, a, b, bytes, flops});
  }
};

static hs_status prof_collect(hs_group* g) {
  for (auto& r : g->prof) {
    DeviceGuard dg(r.device);
    HS_CUDA(cudaEventSynchronize(r.b));
    float ms = 0;
    HS_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    auto& acc = g->prof_acc[r.kind];
    acc.count++; acc.ms += ms; acc.bytes += r.bytes; acc.flops += r.flops;
    g->ev_free[r.device].push_back(r.a);
    g->ev_free[r.device].push_back(r.b);
  }
  g->prof.clear();
  return HS_OK;
}

static double gemm_bytes(double M, double N, double K, double Mout, bool resid) {
  return 2.0 * (M * K + N * K + N * Mout + (resid ? N * Mout : 0.0));
}

// Free everything a stage owns (device + pinned).  keep_exported: leave the memory peers may
// map over CUDA IPC (arena, KV pools, comm block) allocated (SPMD teardown without agreement).
static void free_stage(Stage& s, bool keep_exported = false) {
  DeviceGuard dg(s.device);
  auto F = [](void* p) { if (p) cudaFree(p); };
  if (s.owned) {
    if (!keep_exported) { F(s.arena); F(s.kv_mem); F(s.comm); }
    F(s.xa); F(s.xb); F(s.nrm); F(s.nrm_rs); F(s.qkv); F(s.q); F(s.o);
    F(s.act); F(s.fin); F(s.cap); F(s.logits); F(s.ws); F(s.attn_ws); F(s.ctr); F(s.rope); F(s.d_meta); F(s.d_tok_out);
    F(s.cons_d);
    if (s.cons_h) cudaFreeHost(s.cons_h);
    for (auto e : {s.ev_cons0, s.ev_cons1}) if (e) cudaEventDestroy(e);
    if (s.h_meta) cudaFreeHost(s.h_meta);
    if (s.h_out) cudaFreeHost(s.h_out);
    if (s.ds) dstack_destroy(s.ds);
    for (auto e : s.ev_layer) if (e) cudaEventDestroy(e);
    for (auto e : {s.ev_embed, s.ev_final, s.ev_l0, s.ev_l1, s.ev_c0, s.ev_c1, s.ev_bg0, s.ev_bg}) if (e) cudaEventDestroy(e);
    if (s.owns_streams && s.comp) cudaStreamDestroy(s.comp);
    if (s.owns_streams && s.copy) cudaStreamDestroy(s.copy);
  } else {
    if (s.ipc_comm_open && s.comm) cudaIpcCloseMemHandle(s.comm);
    if (s.ipc_arena_open) {
      if (s.arena) cudaIpcCloseMemHandle(s.arena);
      if (s.kv_mem) cudaIpcCloseMemHandle(s.kv_mem);
    }
  }
  s = Stage{};
}

static hs_status make_layer_maps(hs_group* g, Stage& s, int l) {
  const hs_model_cfg& c = g->cfg;
  const hs_image_header& h = g->hdr;
  const uint64_t L0 = h.layer_off[l];
  LayerDev& d = s.layers[l];
  d.attn_norm = reinterpret_cast<const bf16*>(s.wptr(L0 + h.t_attn_norm));
  d.ffn_norm = reinterpret_cast<const bf16*>(s.wptr(L0 + h.t_ffn_norm));
  HS_TRY(make_tma_w(&d.wqkv, s.wptr(L0 + h.t_wqkv), 3 * c.hidden, c.hidden));
  HS_TRY(make_tma_w(&d.wo, s.wptr(L0 + h.t_wo), c.hidden, c.hidden));
  HS_TRY(make_tma_w(&d.wgu, s.wptr(L0 + h.t_wgu), 2 * c.ffn, c.hidden));
  HS_TRY(make_tma_w(&d.wd, s.wptr(L0 + h.t_wd), c.hidden, c.ffn));
  d.maps = true;
  return HS_OK;
}

static hs_status make_act_maps(TmaMat* m, const void* p, int64_t rows, int64_t cols) {
  for (int i = 0; i < gemm_bn_count(); ++i) HS_TRY(make_tma(&m[i], p, rows, cols, gemm_bn_value(i)));
  return HS_OK;
}

#define HS_ALLOC(ptr, bytes) HS_CUDA(cudaMalloc(reinterpret_cast<void**>(&(ptr)), (bytes)))

static hs_status setup_owned_stage(hs_group* g, int k) {
  Stage& s = g->st[k];
  const hs_model_cfg& c = g->cfg;
  const hs_image_header& h = g->hdr;
  const int T = g->kv.max_tokens, S = g->kv.max_seqs;
  const int H = c.hidden;
  DeviceGuard dg(s.device);
  HS_CUDA(cudaSetDevice(s.device));
  // arena: whole model (full-memory worker) or the stage slice (low-memory worker)
  s.arena_off0 = s.full_memory ? h.embed_off : s.slice_begin;
  s.arena_bytes = (s.full_memory ? h.total_bytes : s.slice_end) - s.arena_off0;
  HS_ALLOC(s.arena, s.arena_bytes);
  s.kv_lb = s.full_memory ? 0 : s.lb;
  s.kv_le = s.full_memory ? c.n_layers : s.le;
  HS_ALLOC(s.kv_mem, (uint64_t)(s.kv_le - s.kv_lb) * g->kv_layer_bytes);
  HS_ALLOC(s.comm, g->cl.bytes);
  HS_CUDA(cudaMemset(s.comm, 0, g->cl.bytes));
  HS_ALLOC(s.xa, (size_t)T * H * 2);
  HS_ALLOC(s.xb, (size_t)T * H * 2);
  HS_ALLOC(s.nrm, (size_t)T * H * 2);
  HS_ALLOC(s.nrm_rs, (size_t)T * 4);
  HS_ALLOC(s.qkv, (size_t)T * 3 * H * 2);
  HS_ALLOC(s.q, (size_t)T * H * 2);
  HS_ALLOC(s.o, (size_t)T * H * 2);
  HS_ALLOC(s.act, (size_t)T * c.ffn * 2);
  HS_ALLOC(s.fin, (size_t)std::max(S, 16) * H * 2);
  HS_ALLOC(s.logits, (size_t)S * c.vocab * 4);
  HS_ALLOC(s.ws, kWorkspace);
  HS_ALLOC(s.ctr, kCounters * 4);
  HS_CUDA(cudaMemset(s.ctr, 0, kCounters * 4));
  HS_ALLOC(s.attn_ws, (size_t)S * c.n_heads * attn_decode_splits(c.max_seq) * (c.head_dim + 2) * 4);
  HS_ALLOC(s.d_tok_out, (size_t)align_up(S * 4, 16) + 16);
  // RoPE table (fp32 cos/sin of angle = p * theta^(-2i/d), computed in double), DESIGN.md
  {
    const int hd = c.head_dim / 2;
    std::vector<float2> tab((size_t)c.max_seq * hd);
    for (int p = 0; p < c.max_seq; ++p)
      for (int i = 0; i < hd; ++i) {
        const double ang = (double)p * std::pow((double)c.rope_theta, -2.0 * i / c.head_dim);
        tab[(size_t)p * hd + i] = make_float2((float)std::cos(ang), (float)std::sin(ang));
      }
    HS_ALLOC(s.rope, tab.size() * sizeof(float2));
    HS_CUDA(cudaMemcpy(s.rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
  }
  s.meta_bytes = kMaxChunks * ((size_t)T * 12 + (size_t)S * (8 + sizeof(SeqDesc) + (size_t)g->max_blocks * 4) + 1024);
  HS_ALLOC(s.d_meta, s.meta_bytes);
  // mapped pinned staging: the SMs read call metadata / write tokens directly (see
  // launch_small_copy), so nothing small queues behind the weight stream on the copy engines
  HS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.h_meta), s.meta_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  HS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.h_out), align_up((size_t)S * 4 + 64, 16),
                        cudaHostAllocMapped | cudaHostAllocPortable));
  int lo = 0, hi = 0;
  HS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  s.owns_streams = true;
  for (int j = 0; j < k; ++j)
    if (g->st[j].owned && g->st[j].device == s.device) {
      s.comp = g->st[j].comp;
      s.copy = g->st[j].copy;
      s.owns_streams = false;
      break;
    }
  if (s.owns_streams) {
    HS_CUDA(cudaStreamCreateWithPriority(&s.comp, cudaStreamNonBlocking, hi));  // critical path
    HS_CUDA(cudaStreamCreateWithPriority(&s.copy, cudaStreamNonBlocking, lo));
  }
  HS_CUDA(cudaEventCreateWithFlags(&s.ev_embed, cudaEventDisableTiming));
  HS_CUDA(cudaEventCreateWithFlags(&s.ev_final, cudaEventDisableTiming));
  HS_CUDA(cudaEventCreate(&s.ev_l0));
  HS_CUDA(cudaEventCreate(&s.ev_l1));
  HS_CUDA(cudaEventCreate(&s.ev_c0));
  HS_CUDA(cudaEventCreate(&s.ev_c1));
  HS_CUDA(cudaEventCreate(&s.ev_bg0));
  HS_CUDA(cudaEventCreate(&s.ev_bg));
  s.ev_layer.assign(c.n_layers, nullptr);
  for (int l = 0; l < c.n_layers; ++l) HS_CUDA(cudaEventCreateWithFlags(&s.ev_layer[l], cudaEventDisableTiming));
  // TMA descriptors: weights of every layer the arena holds, activation operands
  s.layers.assign(c.n_layers, LayerDev{});
  const int wl0 = s.full_memory ? 0 : s.lb, wl1 = s.full_memory ? c.n_layers : s.le;
  for (int l = wl0; l < wl1; ++l) HS_TRY(make_layer_maps(g, s, l));
  if (s.full_memory || s.le == c.n_layers)
    HS_TRY(make_tma_w(&s.lm, s.wptr(h.final_off + h.t_lm_head), c.vocab, H));
  HS_TRY(make_act_maps(s.b_nrm, s.nrm, T, H));
  HS_TRY(make_act_maps(s.b_o, s.o, T, H));
  HS_TRY(make_act_maps(s.b_act, s.act, T, c.ffn));
  HS_TRY(make_act_maps(s.b_fin, s.fin, std::max(S, 16), H));
  warm_gemm_kernels();
  warm_kernels();
  warm_dstack();
  HS_CUDA(cudaDeviceSynchronize());
  return HS_OK;
}

static hs_status validate_image(hs_group* g, const hs_image* im, uint64_t b, uint64_t e) {
  if (!im || !im->data) HS_FAIL(HS_E_INVAL, "missing image for a stage");
  if (im->data_offset > b || im->data_offset + im->data_bytes < e)
    HS_FAIL(HS_E_INVAL, "image data [%llu,%llu) does not cover stage slice [%llu,%llu)",
            (unsigned long long)im->data_offset, (unsigned long long)(im->data_offset + im->data_bytes),
            (unsigned long long)b, (unsigned long long)e);
  return HS_OK;
}

// ------------------------------------------------------------------ create ---------------
static hs_status open_peer_memory(hs_group* g, Stage& s);
static hs_status add_copy(std::vector<CopyDesc>& list, uint64_t src, uint64_t dst, uint64_t bytes, uint64_t piece);

static uint64_t cons_piece() {
  static const uint64_t piece = [] {
    const char* e = getenv("HS_CONS_PIECE_KB");
    return (e && atoi(e) > 0 ? (uint64_t)atoi(e) : 1024ull) << 10;
  }();
  return piece;
}

// Prepares the consolidation of the group into full-memory stage T before T0:
// the copy list's weight part (every other stage's slice, in pieces) is built and uploaded once,
// and room for the KV part (at most every block of every layer) is reserved on the device and in
// pinned staging, so the consolidation pause does no allocation, no upload of the weight list
// and no driver call besides one small H2D of the KV descriptors.  Needs every peer arena mapped.
static hs_status prepare_consolidation(hs_group* g, Stage& T) {
  if (!T.owned || !T.full_memory || T.cons_d) return HS_OK;
  std::vector<CopyDesc> list;
  for (int k : g->active) {
    if (k == T.idx) continue;
    Stage& S = g->st[k];
    if (!S.arena) return HS_OK;  // peer arena not mapped yet (HS_CONS_LATE_OPEN): at the call
    HS_TRY(add_copy(list, reinterpret_cast<uint64_t>(S.arena + (S.slice_begin - S.arena_off0)),
                    reinterpret_cast<uint64_t>(T.wptr(S.slice_begin)), S.slice_end - S.slice_begin, cons_piece()));
  }
  DeviceGuard dg(T.device);
  T.cons_nw = (int)list.size();
  T.cons_cap = T.cons_nw + g->kv.num_blocks * g->cfg.n_layers;
  HS_CUDA(cudaMalloc(reinterpret_cast<void**>(&T.cons_d), (size_t)T.cons_cap * sizeof(CopyDesc)));
  HS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&T.cons_h), (size_t)T.cons_cap * sizeof(CopyDesc), cudaHostAllocPortable));
  if (!list.empty())
    HS_CUDA(cudaMemcpy(T.cons_d, list.data(), list.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
  HS_CUDA(cudaEventCreate(&T.ev_cons0));
  HS_CUDA(cudaEventCreate(&T.ev_cons1));
  return HS_OK;
}

static hs_status create(const hs_model_cfg* cfg, const hs_plan* plan, const hs_image* image,
                        const hs_image* stage_images, const hs_kv_cfg* kv, const hs_comm* comm,
                        hs_group** out) {
  if (!cfg || !plan || !kv || !out) HS_FAIL(HS_E_INVAL, "null argument");
  std::unique_ptr<hs_group> g(new hs_group());
  g->cfg = *cfg;
  if (hs_image_layout(cfg, &g->hdr) != HS_OK) return HS_E_INVAL;
  const hs_image* any = (image && image->header) ? image : nullptr;
  for (int k = 0; !any && stage_images && k < plan->pp && k < HS_MAX_STAGES; ++k)
    if (stage_images[k].header) any = &stage_images[k];
  if (!any || !any->header) HS_FAIL(HS_E_INVAL, "image header required");
  const hs_image_header* ih = any->header;
  if (ih->magic != HS_IMAGE_MAGIC || ih->version != g->hdr.version || ih->total_bytes != g->hdr.total_bytes ||
      ih->layer_bytes != g->hdr.layer_bytes ||
      ih->t_wgu != g->hdr.t_wgu || ih->t_lm_head != g->hdr.t_lm_head || ih->gu_interleave != HS_GU_INTERLEAVE ||
      memcmp(&ih->cfg, cfg, sizeof(hs_model_cfg)) != 0)
    HS_FAIL(HS_E_INVAL, "image header does not match the model cfg / layout");
  if (kv->block_tokens != kBlock || kv->num_blocks <= 0 || kv->max_seqs <= 0 || kv->max_tokens <= 0)
    HS_FAIL(HS_E_INVAL, "kv cfg: block_tokens must be 16 and sizes > 0");
  if (plan->pp < 1 || plan->pp > HS_MAX_STAGES) HS_FAIL(HS_E_INVAL, "bad plan");
  g->plan = *plan;
  g->kv = *kv;
  g->kv.max_seqs = std::max(kv->max_seqs, 1);
  g->max_blocks = (cfg->max_seq + kBlock - 1) / kBlock;
  g->kv_block_bytes = (uint64_t)kBlock * 2 * cfg->hidden * 2;
  g->kv_layer_bytes = g->kv_block_bytes * (uint64_t)kv->num_blocks;
  g->cl.init(g->kv.max_seqs, kv->max_tokens, cfg->hidden);
  for (int b = 0; b < kv->num_blocks; ++b) g->free_blocks.insert(b);
  const int pp = plan->pp;
  g->st.resize(pp);
  for (int k = 0; k < pp; ++k) {
    Stage& s = g->st[k];
    s.idx = k;
    s.device = plan->device[k];
    s.full_memory = plan->full_memory[k] != 0;
    s.lb = plan->layer_begin[k];
    s.le = plan->layer_end[k];
    s.slice_begin = plan->slice_begin[k];
    s.slice_end = plan->slice_end[k];
    if (s.le <= s.lb || (k > 0 && s.lb != plan->layer_end[k - 1])) HS_FAIL(HS_E_INVAL, "plan ranges not contiguous");
    g->active.push_back(k);
  }
  if (g->st[0].lb != 0 || g->st[pp - 1].le != cfg->n_layers) HS_FAIL(HS_E_INVAL, "plan does not cover all layers");
  if (comm) {
    if (comm->world != pp || comm->rank < 0 || comm->rank >= pp || !comm->allgather || !comm->barrier)
      HS_FAIL(HS_E_INVAL, "comm must have world == pp and allgather/barrier callbacks");
    g->spmd = true;
    g->comm = *comm;
    g->owned_stage = comm->rank;
  }
  for (int k = 0; k < pp; ++k) {
    Stage& s = g->st[k];
    s.owned = !g->spmd || k == g->owned_stage;
    if (!s.owned) continue;
    s.img = stage_images ? &stage_images[k] : image;
    HS_TRY(validate_image(g.get(), s.img, s.slice_begin, s.slice_end));
  }
  // peer access between every pair of stage GPUs this process drives (local mode)
  if (!g->spmd) {
    for (int a = 0; a < pp; ++a)
      for (int b = 0; b < pp; ++b) {
        const int da = g->st[a].device, db = g->st[b].device;
        if (da == db) continue;
        int ok = 0;
        HS_CUDA(cudaDeviceCanAccessPeer(&ok, da, db));
        if (!ok) HS_FAIL(HS_E_PEER, "GPU %d cannot access GPU %d", da, db);
        DeviceGuard dg(da);
        cudaSetDevice(da);
        cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) HS_CUDA(e);
        cudaGetLastError();
      }
  }
  for (int k = 0; k < pp; ++k)
    if (g->st[k].owned) {
      hs_status r = setup_owned_stage(g.get(), k);
      if (r != HS_OK) {
        for (auto& s : g->st) free_stage(s);
        return r;
      }
    }
  if (g->spmd) {  // exchange IPC handles, map every peer's comm block
    Stage& me = g->st[g->owned_stage];
    DeviceGuard dg(me.device);
    cudaSetDevice(me.device);
    Share sh{};
    HS_CUDA(cudaIpcGetMemHandle(&sh.comm, me.comm));
    HS_CUDA(cudaIpcGetMemHandle(&sh.arena, me.arena));
    HS_CUDA(cudaIpcGetMemHandle(&sh.kv, me.kv_mem));
    sh.arena_off0 = me.arena_off0;
    sh.arena_bytes = me.arena_bytes;
    sh.kv_layer_bytes = g->kv_layer_bytes;
    sh.kv_lb = me.kv_lb;
    sh.kv_le = me.kv_le;
    sh.device = me.device;
    std::vector<Share> all(pp);
    if (g->comm.allgather(g->comm.ctx, &sh, sizeof(Share), all.data()) != 0) HS_FAIL(HS_E_STATE, "allgather failed");
    for (int k = 0; k < pp; ++k) {
      if (k == g->owned_stage) continue;
      Stage& s = g->st[k];
      s.share = all[k];
      s.arena_off0 = all[k].arena_off0;
      s.arena_bytes = all[k].arena_bytes;
      s.kv_lb = all[k].kv_lb;
      s.kv_le = all[k].kv_le;
      void* p = nullptr;
      HS_CUDA(cudaIpcOpenMemHandle(&p, all[k].comm, cudaIpcMemLazyEnablePeerAccess));
      s.comm = reinterpret_cast<uint8_t*>(p);
      s.ipc_comm_open = true;
    }
    // a full-memory stage (a consolidation target) maps every peer's arena and KV pools now,
    // before T0: opening large IPC allocations costs ~100 ms that must not land in the pause
    static const bool late_open = getenv("HS_CONS_LATE_OPEN") != nullptr;  // debug: map at consolidation
    if (me.full_memory && !late_open)
      for (int k = 0; k < pp; ++k)
        if (k != g->owned_stage) HS_TRY(open_peer_memory(g.get(), g->st[k]));
    if (!comm_barrier(g.get())) HS_FAIL(HS_E_STATE, "barrier failed");
  }
  for (int k = 0; k < pp; ++k) HS_TRY(prepare_consolidation(g.get(), g->st[k]));
  *out = g.release();
  return HS_OK;
}

// ------------------------------------------------------------------ load (a3, a4) --------
static hs_status load_stage(hs_group* g, int k, uint64_t chunk) {
  Stage& s = g->st[k];
  if (!s.owned) return HS_OK;
  const hs_image_header& h = g->hdr;
  const hs_model_cfg& c = g->cfg;
  if (chunk == 0) chunk = kDefaultChunk;
  DeviceGuard dg(s.device);
  const uint8_t* src = reinterpret_cast<const uint8_t*>(s.img->data);
  auto copy_region = [&](uint64_t off, uint64_t bytes, cudaEvent_t ev) -> hs_status {
    for (uint64_t o = 0; o < bytes; o += chunk) {
      const uint64_t n = std::min(chunk, bytes - o);
      // pipelined with the prefetcher: the copy engine starts the chunk once it is fetched
      HS_TRY(stream_wait_watermark(s.copy, s.img->fetched_end, off + o + n));
      HS_CUDA(cudaMemcpyAsync(s.wptr(off + o), src + (off + o - s.img->data_offset), n, cudaMemcpyHostToDevice, s.copy));
    }
    if (ev) HS_CUDA(cudaEventRecord(ev, s.copy));
    s.loaded_bytes += bytes;
    return HS_OK;
  };
  s.loaded_bytes = 0;
  HS_CUDA(cudaEventRecord(s.ev_l0, s.copy));
  // critical order: layers b..e-1, final norm + lm_head, then the embedding table (R4).
  // The prefill reads its prompt's embedding rows straight from the pinned image (UVA-mapped),
  // so the 262 MB table (7B) is not on the TTFT path; decode steps wait for it.  Without a
  // mapped image the table goes first.
  const bool embed_here = s.lb == 0 && k == g->active.front();
  s.host_embed = nullptr;
  if (embed_here && !getenv("HS_EMBED_FIRST")) {
    void* dp = nullptr;
    const void* hp = src + (h.embed_off - s.img->data_offset);
    if (cudaHostGetDevicePointer(&dp, const_cast<void*>(hp), 0) == cudaSuccess) s.host_embed = static_cast<const bf16*>(dp);
    else cudaGetLastError();
  }
  if (embed_here && !s.host_embed) HS_TRY(copy_region(h.embed_off, h.embed_bytes, s.ev_embed));
  for (int l = s.lb; l < s.le; ++l) HS_TRY(copy_region(h.layer_off[l], h.layer_bytes, s.ev_layer[l]));
  if (s.le == c.n_layers) HS_TRY(copy_region(h.final_off, h.final_bytes, s.ev_final));
  if (embed_here && s.host_embed) HS_TRY(copy_region(h.embed_off, h.embed_bytes, s.ev_embed));
  HS_CUDA(cudaEventRecord(s.ev_l1, s.copy));
  s.load_issued = true;
  return HS_OK;
}

// Background host-path load of the regions a full-memory target lacks.
static hs_status load_background(hs_group* g, int tgt, uint64_t chunk) {
  if (tgt < 0 || tgt >= (int)g->st.size()) HS_FAIL(HS_E_INVAL, "bad stage %d", tgt);
  Stage& T = g->st[tgt];
  if (!T.owned) return HS_OK;  // SPMD: only the target's process works
  if (!T.full_memory) HS_FAIL(HS_E_INVAL, "stage %d is not a full-memory worker", tgt);
  if (!T.load_issued) HS_FAIL(HS_E_STATE, "issue the critical load of the target first");
  const hs_image_header& h = g->hdr;
  if (T.img->data_offset > h.embed_off || T.img->data_offset + T.img->data_bytes < h.total_bytes)
    HS_FAIL(HS_E_INVAL, "the target's host image must cover the whole model for a background load");
  if (chunk == 0) chunk = kDefaultChunk;
  DeviceGuard dg(T.device);
  const uint8_t* src = reinterpret_cast<const uint8_t*>(T.img->data);
  HS_CUDA(cudaEventRecord(T.ev_bg0, T.copy));
  T.bg_bytes = 0;
  for (int k : g->active) {
    if (k == tgt) continue;
    const Stage& S = g->st[k];
    for (uint64_t o = S.slice_begin; o < S.slice_end; o += chunk) {
      const uint64_t n = std::min(chunk, S.slice_end - o);
      HS_TRY(stream_wait_watermark(T.copy, T.img->fetched_end, o + n));
      HS_CUDA(cudaMemcpyAsync(T.wptr(o), src + (o - T.img->data_offset), n, cudaMemcpyHostToDevice, T.copy));
    }
    T.bg_bytes += g->plan.stage_bytes[k];
  }
  HS_CUDA(cudaEventRecord(T.ev_bg, T.copy));
  T.bg_issued = true;
  return HS_OK;
}

// Background NVLink pull of the weight regions a full-memory target lacks (the paper's "allowing
// only one of them to fetch the unloaded model parts in background", with the other
// stages' HBM as the source): copy-engine peer copies on the target's low-priority copy stream
// while the group keeps serving pipelined; a later consolidation then moves only the KV blocks.
static hs_status pull_background(hs_group* g, int tgt, uint64_t chunk) {
  if (tgt < 0 || tgt >= (int)g->st.size()) HS_FAIL(HS_E_INVAL, "bad stage %d", tgt);
  Stage& T = g->st[tgt];
  if (!T.owned) return HS_OK;  // SPMD: only the target's process works
  if (!T.full_memory) HS_FAIL(HS_E_INVAL, "stage %d is not a full-memory worker", tgt);
  if (!T.load_issued || !T.called) HS_FAIL(HS_E_STATE, "load and run one prefill first (the sources' slices must be resident)");
  if (T.bg_issued) HS_FAIL(HS_E_STATE, "a background load of the target was already issued");
  if (chunk == 0) chunk = 64ull << 20;
  DeviceGuard dg(T.device);
  HS_CUDA(cudaEventRecord(T.ev_bg0, T.copy));
  T.bg_bytes = 0;
  for (int k : g->active) {
    if (k == tgt) continue;
    Stage& S = g->st[k];
    HS_TRY(open_peer_memory(g, S));
    const uint8_t* src = S.arena + (S.slice_begin - S.arena_off0);
    uint8_t* dst = T.wptr(S.slice_begin);
    const uint64_t bytes = S.slice_end - S.slice_begin;
    for (uint64_t o = 0; o < bytes; o += chunk)
      HS_CUDA(cudaMemcpyAsync(dst + o, src + o, std::min(chunk, bytes - o), cudaMemcpyDeviceToDevice, T.copy));
    T.bg_bytes += g->plan.stage_bytes[k];
  }
  HS_CUDA(cudaEventRecord(T.ev_bg, T.copy));
  T.bg_issued = true;
  T.bg_from_peers = true;
  return HS_OK;
}

// ------------------------------------------------------------------ forward --------------
struct CallMeta {
  int T = 0, n = 0, max_nq = 0, max_ctx = 0;
  bool decode = false;
  double kv_tokens = 0, attn_pairs = 0;  // KV rows read by attention, (query, key) pairs
  size_t o_tok = 0, o_pos = 0, o_slot = 0, o_last = 0, o_seqs = 0, o_tab = 0, bytes = 0;
};

static void layout_meta(CallMeta& m, int max_blocks) {
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o = align_up(o + b, 16); return r; };
  m.o_tok = take((size_t)m.T * 4);
  m.o_pos = take((size_t)m.T * 4);
  m.o_slot = take((size_t)m.T * 4);
  m.o_last = take((size_t)m.n * 4);
  m.o_seqs = take((size_t)m.n * sizeof(SeqDesc));
  m.o_tab = take((size_t)m.n * max_blocks * 4);
  m.bytes = o;
}

// One decoder layer (a6-a12) on a stage.  `normed` says s.nrm already holds RMSNorm(x) with
// this layer's attn_norm (fused into the previous layer's down-projection epilogue in decode);
// on return it says whether s.nrm holds the next consumer's norm (next layer's attn_norm, or
// the final norm into s.fin for the model's last layer).
// HS_DEBUG_SKIP (timing experiments only; results are garbage): bit 1 attention, 2 QKV,
// 4 O-proj, 8 gate_up, 16 down, 32 norm kernels
static int debug_skip() {
  static int v = [] {
    const char* e = getenv("HS_DEBUG_SKIP");
    return e ? atoi(e) : 0;
  }();
  return v;
}

static hs_status run_layer(hs_group* g, Stage& s, int l, const bf16* x, bf16* xout, const CallMeta& m,
                           const uint8_t* meta, bool& normed, bool& fin_done) {
  const int skip = m.decode ? debug_skip() : 0;
  const hs_model_cfg& c = g->cfg;
  const int H = c.hidden, T = m.T;
  LayerDev& L = s.layers[l];
  cudaStream_t st = s.comp;
  const int* pos = reinterpret_cast<const int*>(meta + m.o_pos);
  const int* slot = reinterpret_cast<const int*>(meta + m.o_slot);
  const SeqDesc* sd = reinterpret_cast<const SeqDesc*>(meta + m.o_seqs);
  const int* tab = reinterpret_cast<const int*>(meta + m.o_tab);
  bf16* pool = s.kv_pool(l, g->kv_layer_bytes);
  bf16* hbuf = s.xb;  // h = x + o W_o^T (temporary); x lives in xout's rows (in place after layer 0)
  const bool dec = m.decode;
  const double TH2 = 2.0 * T * H, F = c.ffn;
  if (!normed && !(skip & 32)) {
    ProfScope ps(g, s, PK_RMSNORM, dec, 2 * TH2 + 2.0 * H, 0);
    if (dec && H <= 8192) launch_rownorm_decode(x, L.attn_norm, s.nrm, s.nrm_rs, T, H, c.rms_eps, st);
    else launch_rmsnorm(x, nullptr, L.attn_norm, s.nrm, T, H, c.rms_eps, st, s.nrm_rs);
  }
  bool applied = false;
  GemmArgs a{};
  a.N = T; a.K = H; a.workspace = s.ws; a.workspace_bytes = kWorkspace; a.counters = s.ctr;
  a.A = &L.wqkv; a.B = s.b_nrm; a.M = 3 * H; a.epi = EPI_BF16; a.out = s.qkv; a.ldo = 3 * H; a.rs = s.nrm_rs;
  if (dec) {  // fused bf16 rounding + RoPE + paged KV write in the stream-K reduction
    a.fuse.kind = FUSE_ROPE; a.fuse.pos = pos; a.fuse.slot = slot; a.fuse.rope_tab = s.rope; a.fuse.q_out = s.q;
    a.fuse.pool = pool; a.fuse.n_heads = c.n_heads; a.fuse.head_dim = c.head_dim; a.fuse.applied = &applied;
    a.fuse.nslots = g->kv.num_blocks * kBlock;
  }
  if (!(skip & 2)) {
    ProfScope ps(g, s, PK_GEMM_QKV, dec, gemm_bytes(3.0 * H, T, H, 3.0 * H, false), 2.0 * 3 * H * T * H);
    HS_TRY(gemm(a, st));
  } else {
    applied = true;
  }
  if (!applied) {
    ProfScope ps(g, s, PK_ROPE_KV, dec, 3 * TH2 + 3 * TH2, 0);
    launch_rope_kv(s.qkv, pos, slot, s.rope, s.q, pool, T, c.n_heads, c.head_dim, g->kv.num_blocks * kBlock, st);
  }
  if (!(skip & 1)) {
    ProfScope ps(g, s, PK_ATTN, dec, 2 * TH2 + 2.0 * 2 * H * m.kv_tokens, 4.0 * H * m.attn_pairs);
    if (m.decode)
      launch_attn_decode(s.q, pool, sd, m.n, m.max_ctx, tab, g->max_blocks, s.o, c.n_heads, c.head_dim,
                         s.attn_ws, attn_decode_splits(m.max_ctx), s.ctr + kCounters / 2, g->kv.num_blocks, st);
    else
      launch_attn_prefill(s.q, pool, sd, m.n, m.max_nq, tab, g->max_blocks, s.o, c.n_heads, c.head_dim,
                          g->kv.num_blocks, st); }
  a.fuse = GemmFusion{};
  applied = false;
  a.A = &L.wo; a.B = s.b_o; a.M = H; a.K = H; a.epi = EPI_RESID; a.out = hbuf; a.ldo = H; a.resid = x; a.ldr = H;
  a.rs = nullptr;
  if (dec) {  // fused residual + RMSNorm(ffn_norm)
    a.fuse.kind = FUSE_NORM; a.fuse.norm_w = L.ffn_norm; a.fuse.norm_out = s.nrm; a.fuse.eps = c.rms_eps;
    a.fuse.rs_out = s.nrm_rs;
    a.fuse.applied = &applied;
  }
  if (!(skip & 4)) {
    ProfScope ps(g, s, PK_GEMM_O, dec, gemm_bytes(H, T, H, H, true), 2.0 * H * T * H);
    HS_TRY(gemm(a, st));
  } else {
    applied = true;
  }
  if (!applied) {
    ProfScope ps(g, s, PK_RMSNORM, dec, 2 * TH2 + 2.0 * H, 0);
    launch_rmsnorm(hbuf, nullptr, L.ffn_norm, s.nrm, T, H, c.rms_eps, st, s.nrm_rs);
  }
  a.fuse = GemmFusion{};
  a.A = &L.wgu; a.B = s.b_nrm; a.M = 2 * c.ffn; a.K = H; a.epi = EPI_SILU_MUL; a.out = s.act; a.ldo = c.ffn;
  a.resid = nullptr; a.rs = s.nrm_rs;
  if (!(skip & 8)) {
    ProfScope ps(g, s, PK_GEMM_GU, dec, gemm_bytes(2 * F, T, H, F, false), 2.0 * 2 * F * T * H);
    HS_TRY(gemm(a, st));
  }
  a.A = &L.wd; a.B = s.b_act; a.M = H; a.K = c.ffn; a.epi = EPI_RESID; a.out = xout; a.ldo = H; a.resid = hbuf;
  a.ldr = H; a.rs = nullptr;
  applied = false;
  const bool next_here = l + 1 < s.le;
  const bool model_last = l + 1 == c.n_layers;
  if (dec && (next_here || model_last)) {  // fused residual + next consumer's RMSNorm
    a.fuse.kind = FUSE_NORM;
    a.fuse.eps = c.rms_eps;
    a.fuse.applied = &applied;
    if (next_here) {
      a.fuse.norm_w = s.layers[l + 1].attn_norm;
      a.fuse.norm_out = s.nrm;
      a.fuse.rs_out = s.nrm_rs;
    } else {  // decode: every row is a sequence's last position -> final norm into s.fin
      a.fuse.norm_w = reinterpret_cast<const bf16*>(s.wptr(g->hdr.final_off + g->hdr.t_final_norm));
      a.fuse.norm_out = s.fin;
    }
  }
  if (!(skip & 16)) {
    ProfScope ps(g, s, PK_GEMM_DOWN, dec, gemm_bytes(H, T, F, H, true), 2.0 * H * T * F);
    HS_TRY(gemm(a, st));
  } else {
    applied = next_here || model_last;
  }
  normed = applied && next_here;
  fin_done = applied && model_last;
  return HS_OK;
}

// Decode through the decode-stack kernel (dstack.h): every layer of the stage in one launch.
// Returns false in *used when the call's shape is not covered (the per-kernel path runs).
static hs_status run_dstack(hs_group* g, Stage& s, const CallMeta& m, const uint8_t* meta, const bf16* x_in,
                            bf16* x, const std::vector<int>& ctx, bool* used, bool* fin_done) {
  *used = false;
  const hs_model_cfg& c = g->cfg;
  if (!m.decode || !dstack_supported(m.n, c.head_dim) || m.n != m.T) return HS_OK;
  const int nl = s.le - s.lb;
  if (nl < 1 || nl > 255) return HS_OK;
  if (!s.ds) {
    HS_TRY(dstack_create(&s.ds, c.hidden, c.ffn, c.n_heads, c.head_dim, g->kv.max_seqs, c.max_seq, s.comp));
  }
  if (m.n > std::min(64, g->kv.max_seqs)) return HS_OK;
  const hs_image_header& h = g->hdr;
  if (s.ds_lb != s.lb || s.ds_le != s.le || s.ds_arena != s.arena) {
    const uint64_t L0 = h.layer_off[s.lb];
    HS_TRY(make_tma_w3(&s.ds_w[0], s.wptr(L0 + h.t_wqkv), nl, h.layer_bytes, 3 * c.hidden, c.hidden));
    HS_TRY(make_tma_w3(&s.ds_w[1], s.wptr(L0 + h.t_wo), nl, h.layer_bytes, c.hidden, c.hidden));
    HS_TRY(make_tma_w3(&s.ds_w[2], s.wptr(L0 + h.t_wgu), nl, h.layer_bytes, 2 * c.ffn, c.hidden));
    HS_TRY(make_tma_w3(&s.ds_w[3], s.wptr(L0 + h.t_wd), nl, h.layer_bytes, c.hidden, c.ffn));
    s.ds_lb = s.lb;
    s.ds_le = s.le;
    s.ds_arena = s.arena;
  }
  const uint64_t L0 = h.layer_off[s.lb];
  DstackArgs a{};
  a.N = m.n; a.H = c.hidden; a.F = c.ffn; a.nh = c.n_heads; a.hd = c.head_dim; a.nl = nl; a.eps = c.rms_eps;
  a.wqkv = &s.ds_w[0]; a.wo = &s.ds_w[1]; a.wgu = &s.ds_w[2]; a.wd = &s.ds_w[3];
  a.attn_norm = reinterpret_cast<const bf16*>(s.wptr(L0 + h.t_attn_norm));
  a.ffn_norm = reinterpret_cast<const bf16*>(s.wptr(L0 + h.t_ffn_norm));
  a.norm_stride = (int64_t)(h.layer_bytes / 2);
  const bool model_last = s.le == c.n_layers;
  a.final_norm = model_last ? reinterpret_cast<const bf16*>(s.wptr(h.final_off + h.t_final_norm)) : nullptr;
  a.fin = s.fin;
  a.x_in = x_in; a.x = x; a.hbuf = s.xb; a.nrm = s.nrm; a.q = s.q; a.o = s.o; a.act = s.act;
  a.b_nrm = s.b_nrm; a.b_o = s.b_o; a.b_act = s.b_act;
  a.pool = s.kv_pool(s.lb, g->kv_layer_bytes);
  a.pool_stride = (int64_t)(g->kv_layer_bytes / 2);
  a.nslots = g->kv.num_blocks * kBlock; a.nblocks = g->kv.num_blocks; a.max_blocks = g->max_blocks;
  a.pos = reinterpret_cast<const int*>(meta + m.o_pos);
  a.slot = reinterpret_cast<const int*>(meta + m.o_slot);
  a.tables = reinterpret_cast<const int*>(meta + m.o_tab);
  a.seqs = reinterpret_cast<const SeqDesc*>(meta + m.o_seqs);
  a.rope = s.rope;
  a.ctx = ctx.data();
  if (g->capture && s.cap) {  // test-only: every layer's output rows (decode: one chunk, rows 0..N-1)
    a.cap_stride = (int64_t)g->kv.max_tokens * c.hidden;
    a.cap = s.cap + (size_t)(2 * s.lb + 1) * a.cap_stride;  // point 2 lb + 1: h of the range's first layer
    for (int pt = 2 * s.lb + 1; pt <= 2 * s.le; ++pt) g->cap_owner[pt] = s.idx;
  }
  {
    const double H = c.hidden, F = c.ffn;
    const double wbytes = (double)nl * 2.0 * (4 * H * H + 3 * F * H + 2 * H);
    const double kv = (double)nl * 2.0 * 2 * H * (m.kv_tokens + m.n);
    ProfScope ps(g, s, PK_DSTACK, true, wbytes + kv, 2.0 * m.n * (wbytes / 2) + 4.0 * H * m.attn_pairs * nl);
    HS_TRY(dstack_launch(s.ds, a, s.comp));
  }
  *used = true;
  *fin_done = model_last;
  return HS_OK;
}

// Enqueues one call (prefill or decode) on every owned stage; returns after the tokens of
// the call are on the host.
//
// Prefill through s > 1 stages is micro-batched (PAPER.md:399, 405-406:
// the t_p terms of Eq. 1): every sequence's tokens are cut into m chunks (chunked prefill:
// chunk c attends to the KV of chunks < c already in the cache), each stage hands chunk c to
// the next stage as soon as it is through its layers, so stage k+1 works on chunk c while
// stage k works on chunk c+1.  A stage whose weights are still streaming in runs layer-major
// (every chunk of layer l as soon as layer l lands: it keeps pace with its PCIe link); a
// resident stage runs chunk-major (hands chunk 0 on first).  Chunk c of the residual stream
// lives in rows [R_c, R_c + T_c) of the stage buffers; hand-off flags carry epoch base + c.
struct Chunk {
  CallMeta m;
  size_t meta_off = 0;
  int row0 = 0;
};

static hs_status run_call(hs_group* g, const CallMeta& m0, const std::vector<int64_t>& ids,
                          const std::vector<int>& host_tokens, bool feedback, int32_t* out_tokens,
                          float* out_logits) {
  const auto t_call = std::chrono::steady_clock::now();
  const hs_model_cfg& c = g->cfg;
  const int first = g->active.front(), last = g->active.back();
  // ---- chunking of prefill: depends on the shapes only (never on the number of stages), so
  // PP = s stays bitwise equal to PP = 1.  A chunk keeps >= kChunkTokens tokens: below that a
  // chunk's GEMMs fall under the B200 ridge point (every chunk re-reads the layer's weights;
  // ~210 flop/byte needs ~210 tokens per weight read), and micro-batching would cost more than
  // the pipelining saves (measured: 4 x 128-token chunks of a 512-token prompt made PP=2 TTFT
  // 6 ms slower).
  int nchunks = 1;
  if (!m0.decode) {
    int min_len = 1 << 30;
    for (int i = 0; i < m0.n; ++i) min_len = std::min(min_len, g->seqs[ids[i]].ctx);
    static const int chunk_tokens = [] {
      const char* e = getenv("HS_CHUNK_TOKENS");
      return e && atoi(e) > 0 ? atoi(e) : kChunkTokens;
    }();
    const int ct = g->chunk_tokens > 0 ? g->chunk_tokens : chunk_tokens;
    const int mc = g->max_chunks > 0 ? std::min(g->max_chunks, kMaxChunks) : kMaxChunks;
    nchunks = std::max(1, std::min<int>({mc, min_len / 16, m0.T / ct}));
  }
  std::vector<int> dctx;  // decode: keys per sequence after this step (decode-stack item split)
  if (m0.decode)
    for (int i = 0; i < m0.n; ++i) dctx.push_back(g->seqs[ids[i]].ctx);
  const unsigned ep0 = g->epoch + 1;   // chunk c is handed over with flag value ep0 + c
  g->epoch += nchunks;
  const unsigned ep = g->epoch;        // the call's final epoch (token broadcast)
  std::vector<Chunk> ch(nchunks);
  {
    size_t off = 0;
    int row = 0;
    for (int cidx = 0; cidx < nchunks; ++cidx) {
      CallMeta m = m0;
      m.T = 0;
      m.max_nq = 0;
      m.kv_tokens = 0;
      m.attn_pairs = 0;
      for (int i = 0; i < m0.n; ++i) {
        const SeqState& ss = g->seqs[ids[i]];
        const int n_new = m0.decode ? 1 : ss.ctx;
        const int b = (int)((int64_t)n_new * cidx / nchunks), e = (int)((int64_t)n_new * (cidx + 1) / nchunks);
        m.T += e - b;
        m.max_nq = std::max(m.max_nq, e - b);
        m.kv_tokens += (ss.ctx - n_new) + e;
        m.attn_pairs += m0.decode ? ss.ctx : 0.5 * (double)(e - b) * (2.0 * ((ss.ctx - n_new) + b) + (e - b) + 1);
      }
      layout_meta(m, g->max_blocks);
      ch[cidx].m = m;
      ch[cidx].meta_off = off;
      ch[cidx].row0 = row;
      off += align_up(m.bytes, 256);
      row += m.T;
    }
  }
  if (g->capture) {  // test-only: buffer row of every token of the call, in call order
    std::vector<int> start(m0.n + 1, 0);
    for (int i = 0; i < m0.n; ++i) start[i + 1] = start[i] + (m0.decode ? 1 : g->seqs[ids[i]].ctx);
    g->cap_rowmap.assign(start[m0.n], 0);
    for (int cidx = 0; cidx < nchunks; ++cidx) {
      int qs = 0;
      for (int i = 0; i < m0.n; ++i) {
        const int n_new = m0.decode ? 1 : g->seqs[ids[i]].ctx;
        const int b = (int)((int64_t)n_new * cidx / nchunks), e = (int)((int64_t)n_new * (cidx + 1) / nchunks);
        for (int j = b; j < e; ++j) g->cap_rowmap[start[i] + j] = ch[cidx].row0 + qs + (j - b);
        qs += e - b;
      }
    }
    g->cap_owner.assign(2 * c.n_layers + 1, -1);
  }
  for (size_t ai = 0; ai < g->active.size(); ++ai) {
    const int k = g->active[ai];
    Stage& s = g->st[k];
    if (!s.owned) continue;
    if (!s.load_issued) HS_FAIL(HS_E_STATE, "stage %d: no load issued (call hs_load_stage_async first)", k);
    if (ch.back().meta_off + ch.back().m.bytes > s.meta_bytes) HS_FAIL(HS_E_INVAL, "call metadata too large");
    DeviceGuard dg(s.device);
    cudaStream_t st = s.comp;
    // host metadata (identical on every stage: centralised block manager), one block per chunk
    int tglob = 0;
    for (int cidx = 0; cidx < nchunks; ++cidx) {
      const CallMeta& m = ch[cidx].m;
      uint8_t* hm = s.h_meta + ch[cidx].meta_off;
      int* tok = reinterpret_cast<int*>(hm + m.o_tok);
      int* pos = reinterpret_cast<int*>(hm + m.o_pos);
      int* slot = reinterpret_cast<int*>(hm + m.o_slot);
      int* lastr = reinterpret_cast<int*>(hm + m.o_last);
      SeqDesc* sd = reinterpret_cast<SeqDesc*>(hm + m.o_seqs);
      int* tab = reinterpret_cast<int*>(hm + m.o_tab);
      int t = 0;
      for (int i = 0; i < m.n; ++i) {
        const SeqState& ss = g->seqs[ids[i]];
        const int n_new = m.decode ? 1 : ss.ctx;  // prefill: ctx == prompt length
        const int b = (int)((int64_t)n_new * cidx / nchunks), e = (int)((int64_t)n_new * (cidx + 1) / nchunks);
        const int p0 = ss.ctx - n_new + b;
        sd[i].q_start = t;
        sd[i].n_q = e - b;
        sd[i].pos0 = p0;
        sd[i].table = i;
        // host tokens are packed per sequence: sequence i's token j is at offset start_i + j
        int start_i = 0;
        if (!host_tokens.empty())
          for (int q = 0; q < i; ++q) start_i += m.decode ? 1 : g->seqs[ids[q]].ctx;
        for (int j = b; j < e; ++j) {
          const int pp = ss.ctx - n_new + j;
          pos[t] = pp;
          slot[t] = ss.blocks[pp / kBlock] * kBlock + pp % kBlock;
          tok[t] = host_tokens.empty() ? 0 : host_tokens[start_i + j];
          ++t;
        }
        lastr[i] = t - 1;
        for (int bb = 0; bb < g->max_blocks; ++bb)
          tab[(size_t)i * g->max_blocks + bb] = bb < (int)ss.blocks.size() ? ss.blocks[bb] : 0;
      }
      tglob += t;
    }
    (void)tglob;
    HS_CUDA(cudaEventRecord(s.ev_c0, st));
    launch_small_copy(s.h_meta, s.d_meta, ch.back().meta_off + ch.back().m.bytes, st);
    const bool dec = m0.decode;
    const bool is_first = k == first, is_last = k == last;
    Stage* nx = is_last ? nullptr : &g->st[g->active[ai + 1]];
    const int H = c.hidden;
    auto meta_of = [&](int cidx) { return s.d_meta + ch[cidx].meta_off; };
    auto xrows = [&](int cidx) { return s.xa + (size_t)ch[cidx].row0 * H; };
    auto in_rows = [&](int cidx) { return reinterpret_cast<bf16*>(s.comm + g->cl.x_in) + (size_t)ch[cidx].row0 * H; };
    // stage input of chunk cidx: embedding (first stage) or the hand-off buffer
    auto stage_input = [&](int cidx) -> hs_status {
      if (is_first) {
        const bf16* E = reinterpret_cast<const bf16*>(s.wptr(g->hdr.embed_off));
        // prefill while the table is still streaming: read the prompt's rows from the image
        const bool from_host = !dec && s.host_embed && cudaEventQuery(s.ev_embed) == cudaErrorNotReady;
        cudaGetLastError();
        if (from_host) {  // the prompt's rows are read from the host image: once fetched
          E = s.host_embed;
          HS_TRY(stream_wait_watermark(st, s.img->fetched_end, g->hdr.embed_off + g->hdr.embed_bytes));
        }
        else if (cidx == 0 && s.lb == 0) HS_CUDA(cudaStreamWaitEvent(st, s.ev_embed, 0));
        const int* d_tok = reinterpret_cast<const int*>(meta_of(cidx) + ch[cidx].m.o_tok);
        if (feedback) {
          ProfScope ps(g, s, PK_WAIT, dec, 0, 0);
          launch_wait(s.flag_tok(), ep0 - 1, s.err(), st);
          d_tok = reinterpret_cast<const int*>(s.comm + g->cl.tok_in);
        }
        ProfScope ps(g, s, PK_EMBED, dec, 4.0 * ch[cidx].m.T * H, 0);
        launch_embed(d_tok, E, xrows(cidx), ch[cidx].m.T, H, c.vocab, st);
      } else {
        ProfScope ps(g, s, PK_WAIT, dec, 0, 0);
        launch_wait(s.flag_x(), ep0 + cidx, s.err(), st);
      }
      return HS_OK;
    };
    auto hand_off = [&](int cidx) {
      ProfScope ps(g, s, PK_SEND, dec, 2.0 * ch[cidx].m.T * H, 0);
      launch_send(xrows(cidx), reinterpret_cast<uint8_t*>(nx->comm + g->cl.x_in) + (size_t)ch[cidx].row0 * H * 2,
                  (uint64_t)ch[cidx].m.T * H * 2, s.done(), nx->flag_x(), ep0 + cidx, kSendCtas, st);
    };
    // test-only capture: point pt's rows of chunk cidx (pt = 2l: the input of layer l, 0 = the
    // embedding rows, 2L = the last layer's output; pt = 2l + 1: layer l's h, which run_layer
    // leaves in s.xb rows 0..T_c-1), on the compute stream right behind their producer
    auto capture = [&](int pt, int cidx) -> hs_status {
      if (!g->capture || !s.cap) return HS_OK;
      const bf16* src = (pt & 1) ? s.xb : xrows(cidx);
      HS_CUDA(cudaMemcpyAsync(s.cap + ((size_t)pt * g->kv.max_tokens + ch[cidx].row0) * H, src,
                              (size_t)ch[cidx].m.T * H * 2, cudaMemcpyDeviceToDevice, st));
      g->cap_owner[pt] = k;
      return HS_OK;
    };
    auto capture_layer = [&](int l, int cidx) -> hs_status {
      HS_TRY(capture(2 * l + 1, cidx));
      return capture(2 * l + 2, cidx);
    };
    bool normed = false, fin_done = false;
    // layer-major while this stage's weights are still arriving, chunk-major once resident
    const bool loading = nchunks > 1 && is_first && cudaEventQuery(s.ev_l1) == cudaErrorNotReady;
    cudaGetLastError();
    if (nchunks == 1 || !loading) {
      for (int cidx = 0; cidx < nchunks; ++cidx) {
        HS_TRY(stage_input(cidx));
        if (is_first && s.lb == 0) HS_TRY(capture(0, cidx));
        normed = false;
        bool used = false;
        if (dec) {
          for (int l = s.lb; l < s.le; ++l) HS_CUDA(cudaStreamWaitEvent(st, s.ev_layer[l], 0));
          if (s.le == c.n_layers) HS_CUDA(cudaStreamWaitEvent(st, s.ev_final, 0));  // fused final norm
          HS_TRY(run_dstack(g, s, ch[cidx].m, meta_of(cidx), is_first ? xrows(cidx) : in_rows(cidx), xrows(cidx),
                            dctx, &used, &fin_done));
        }
        for (int l = s.lb; l < s.le && !used; ++l) {
          HS_CUDA(cudaStreamWaitEvent(st, s.ev_layer[l], 0));
          if (dec && l + 1 == c.n_layers) HS_CUDA(cudaStreamWaitEvent(st, s.ev_final, 0));  // fused final norm
          const bf16* xin = (l == s.lb && !is_first) ? in_rows(cidx) : xrows(cidx);
          HS_TRY(run_layer(g, s, l, xin, xrows(cidx), ch[cidx].m, meta_of(cidx), normed, fin_done));
          HS_TRY(capture_layer(l, cidx));
        }
        if (!is_last) hand_off(cidx);
      }
    } else {
      for (int cidx = 0; cidx < nchunks; ++cidx) {
        HS_TRY(stage_input(cidx));
        if (is_first && s.lb == 0) HS_TRY(capture(0, cidx));
      }
      for (int l = s.lb; l < s.le; ++l) {
        HS_CUDA(cudaStreamWaitEvent(st, s.ev_layer[l], 0));
        for (int cidx = 0; cidx < nchunks; ++cidx) {
          bool nrm = false, fd = false;
          const bf16* xin = (l == s.lb && !is_first) ? in_rows(cidx) : xrows(cidx);
          HS_TRY(run_layer(g, s, l, xin, xrows(cidx), ch[cidx].m, meta_of(cidx), nrm, fd));
          HS_TRY(capture_layer(l, cidx));
          if (l + 1 == s.le && !is_last) hand_off(cidx);
        }
      }
    }
    if (is_last) {
      const Chunk& lc = ch.back();
      const CallMeta& m = lc.m;
      if (s.le == c.n_layers) HS_CUDA(cudaStreamWaitEvent(st, s.ev_final, 0));
      const int* d_last = reinterpret_cast<const int*>(meta_of(nchunks - 1) + m.o_last);
      if (!fin_done) {
        ProfScope ps(g, s, PK_RMSNORM, dec, 4.0 * m.n * c.hidden, 0);
        launch_rmsnorm(xrows(nchunks - 1), d_last,
                       reinterpret_cast<const bf16*>(s.wptr(g->hdr.final_off + g->hdr.t_final_norm)), s.fin, m.n,
                       c.hidden, c.rms_eps, st);
      }
      GemmArgs a{};
      a.A = &s.lm; a.B = s.b_fin; a.M = c.vocab; a.N = m.n; a.K = c.hidden; a.epi = EPI_F32; a.out = s.logits;
      a.ldo = c.vocab; a.workspace = s.ws; a.workspace_bytes = kWorkspace; a.counters = s.ctr;
      {
        ProfScope ps(g, s, PK_LM_HEAD, dec, 2.0 * c.vocab * c.hidden + 2.0 * m.n * c.hidden + 4.0 * m.n * c.vocab,
                     2.0 * c.vocab * m.n * c.hidden);
        HS_TRY(gemm(a, st));
      }
      {
        ProfScope ps(g, s, PK_ARGMAX, dec, 4.0 * m.n * c.vocab, 0);
        launch_argmax(s.logits, c.vocab, m.n, s.d_tok_out, st);
      }
      const uint64_t tb = align_up((uint64_t)m.n * 4, 16);
      // token feedback to the first stage (the next decode embeds it on the device); in SPMD
      // mode to every stage, so that every rank can return the tokens
      // (local mode: also every full-memory stage, a possible consolidation target that then
      // embeds the fed-back tokens of the next decode step itself)
      for (int kk : g->active) {
        if (!g->spmd && kk != first && !g->st[kk].full_memory) continue;
        Stage& d = g->st[kk];
        launch_send(s.d_tok_out, d.comm + g->cl.tok_in, tb, s.done(), d.flag_tok(), ep, 1, st);
      }
      launch_small_copy(s.d_tok_out, s.h_out, align_up((uint64_t)m.n * 4, 16), st);
      if (out_logits)
        HS_CUDA(cudaMemcpyAsync(out_logits, s.logits, (size_t)m.n * c.vocab * 4, cudaMemcpyDeviceToHost, st));
    }
    if (!is_last && g->spmd) {  // non-last SPMD ranks read the broadcast tokens
      launch_wait(s.flag_tok(), ep, s.err(), st);
      launch_small_copy(s.comm + g->cl.tok_in, s.h_out, align_up((uint64_t)m0.n * 4, 16), st);
    }
    launch_small_copy(s.comm, s.h_out + align_up((uint64_t)m0.n, 4), 16, st);  // flags + err word
    HS_CUDA(cudaEventRecord(s.ev_c1, st));
    s.called = true;
  }
  // wait for the result on the stage(s) this process owns
  const auto t_enq = std::chrono::steady_clock::now();
  const int n = m0.n;
  int err = 0;
  bool got = false;
  for (int k : g->active) {
    Stage& s = g->st[k];
    if (!s.owned) continue;
    DeviceGuard dg(s.device);
    cudaError_t e = cudaStreamSynchronize(s.comp);
    if (e != cudaSuccess) {
      g->dead = true;
      HS_FAIL(HS_E_CUDA, "stage %d: %s", k, cudaGetErrorString(e));
    }
    err |= s.h_out[align_up((uint64_t)n, 4) + CommLayout::ERR / 4];
    if (k == last || (g->spmd && !got)) {
      memcpy(out_tokens, s.h_out, (size_t)n * 4);
      got = true;
    }
  }
  if (err) {
    g->dead = true;
    HS_FAIL(HS_E_TIMEOUT, "a cross-stage wait timed out (peer never signalled)");
  }
  for (int k : g->active) {
    if (!g->st[k].owned) continue;
    DeviceGuard dg(g->st[k].device);
    const unsigned bad = debug_bad_bits(true);
    if (bad) {
      g->dead = true;
      HS_FAIL(HS_E_CUDA, "device range check failed (bits 0x%x: 1 token id, 2 KV slot, 4 block id)", bad);
    }
  }
  g->last_ids = ids;
  static const bool dbg = getenv("HS_DEBUG_CALL") != nullptr;
  if (dbg) {
    const auto t_end = std::chrono::steady_clock::now();
    fprintf(stderr, "[hs] call stage %d: enqueue %.1f us, wait %.1f us\n", g->owned_stage,
            1e6 * std::chrono::duration<double>(t_enq - t_call).count(),
            1e6 * std::chrono::duration<double>(t_end - t_enq).count());
  }
  return HS_OK;
}

static hs_status alloc_tokens(hs_group* g, int64_t id, int n_new) {
  SeqState& ss = g->seqs[id];
  const int need = (ss.ctx + n_new + kBlock - 1) / kBlock;
  if (ss.ctx + n_new > g->cfg.max_seq) HS_FAIL(HS_E_INVAL, "sequence exceeds max_seq");
  while ((int)ss.blocks.size() < need) {
    if (g->free_blocks.empty()) HS_FAIL(HS_E_OOM, "KV blocks exhausted");
    ss.blocks.push_back(*g->free_blocks.begin());  // lowest free id first
    g->free_blocks.erase(g->free_blocks.begin());
  }
  ss.ctx += n_new;
  return HS_OK;
}

static void release(hs_group* g, int64_t id) {
  auto it = g->seqs.find(id);
  if (it == g->seqs.end()) return;
  for (int b : it->second.blocks) g->free_blocks.insert(b);
  g->seqs.erase(it);
}

static hs_status prefill(hs_group* g, int n, const int64_t* ids, const int32_t* tokens, const int32_t* lens,
                         int32_t* out_tokens, float* out_logits) {
  if (g->dead) HS_FAIL(HS_E_CUDA, "group is dead after a CUDA error");
  if (n <= 0 || n > g->kv.max_seqs || !ids || !tokens || !lens || !out_tokens) HS_FAIL(HS_E_INVAL, "bad prefill args");
  if (g->spmd && std::find(g->active.begin(), g->active.end(), g->owned_stage) == g->active.end())
    HS_FAIL(HS_E_STATE, "this rank's stage was released by consolidation");
  int T = 0, maxnq = 0;
  std::set<int64_t> uniq;
  for (int i = 0; i < n; ++i) {
    if (lens[i] <= 0) HS_FAIL(HS_E_INVAL, "empty prompt");
    if (g->seqs.count(ids[i]) || !uniq.insert(ids[i]).second) HS_FAIL(HS_E_INVAL, "sequence id already live");
    T += lens[i];
    maxnq = std::max(maxnq, (int)lens[i]);
  }
  if (T > g->kv.max_tokens) HS_FAIL(HS_E_INVAL, "prefill of %d tokens exceeds max_tokens %d", T, g->kv.max_tokens);
  for (int i = 0; i < T; ++i)
    if (tokens[i] < 0 || tokens[i] >= g->cfg.vocab) HS_FAIL(HS_E_INVAL, "token id out of range");
  std::vector<int64_t> v(ids, ids + n);
  for (int i = 0; i < n; ++i) {
    hs_status r = alloc_tokens(g, ids[i], lens[i]);
    if (r != HS_OK) {
      for (int j = 0; j <= i; ++j) release(g, ids[j]);
      return r;
    }
  }
  CallMeta m;
  m.T = T; m.n = n; m.max_nq = maxnq; m.decode = false;
  for (int i = 0; i < n; ++i) {
    m.kv_tokens += lens[i];
    m.attn_pairs += 0.5 * (double)lens[i] * (lens[i] + 1);
  }
  std::vector<int> ht(tokens, tokens + T);
  hs_status r = run_call(g, m, v, ht, false, out_tokens, out_logits);
  if (r != HS_OK && r != HS_E_CUDA && r != HS_E_TIMEOUT)
    for (int i = 0; i < n; ++i) release(g, ids[i]);
  return r;
}

static hs_status decode(hs_group* g, int n, const int64_t* ids, const int32_t* in_tokens, int32_t* out_tokens,
                        float* out_logits) {
  if (g->dead) HS_FAIL(HS_E_CUDA, "group is dead after a CUDA error");
  if (n <= 0 || n > g->kv.max_seqs || !ids || !out_tokens) HS_FAIL(HS_E_INVAL, "bad decode args");
  if (g->spmd && std::find(g->active.begin(), g->active.end(), g->owned_stage) == g->active.end())
    HS_FAIL(HS_E_STATE, "this rank's stage was released by consolidation");
  std::vector<int64_t> v(ids, ids + n);
  std::set<int64_t> uniq(v.begin(), v.end());
  if ((int)uniq.size() != n) HS_FAIL(HS_E_INVAL, "duplicate sequence ids");
  int maxctx = 0;
  for (int i = 0; i < n; ++i) {
    auto it = g->seqs.find(ids[i]);
    if (it == g->seqs.end()) HS_FAIL(HS_E_INVAL, "sequence %lld was never prefilled", (long long)ids[i]);
    if (it->second.ctx + 1 > g->cfg.max_seq) HS_FAIL(HS_E_INVAL, "sequence exceeds max_seq");
  }
  const bool feedback = in_tokens == nullptr;
  if (feedback && v != g->last_ids) HS_FAIL(HS_E_INVAL, "device token feedback needs the previous call's seq order");
  std::vector<int> ht;
  if (!feedback) {
    ht.assign(in_tokens, in_tokens + n);
    for (int t : ht) if (t < 0 || t >= g->cfg.vocab) HS_FAIL(HS_E_INVAL, "token id out of range");
  }
  for (int i = 0; i < n; ++i) {
    hs_status r = alloc_tokens(g, ids[i], 1);
    if (r != HS_OK) return r;
    maxctx = std::max(maxctx, g->seqs[ids[i]].ctx);
  }
  CallMeta m;
  m.T = n; m.n = n; m.max_nq = 1; m.max_ctx = maxctx; m.decode = true;
  for (int i = 0; i < n; ++i) {
    m.kv_tokens += g->seqs[ids[i]].ctx;
    m.attn_pairs += g->seqs[ids[i]].ctx;
  }
  return run_call(g, m, v, ht, feedback, out_tokens, out_logits);
}

// ------------------------------------------------------------------ pipelined decode -----
// hs_decode_steps: n_steps greedy steps with the batch split into micro-batches ("virtual
// engines") that flow through the stages concurrently (the t_d and t_n
// terms of Eq. 2, are per-stage and overlap across micro-batches).  Every stage
// works through items (step t, micro-batch j) in order; a stage hands micro-batch j of step t to
// the next stage as soon as its layers are done (hand-off flag epoch e(t, j), rows s0_j..), and
// the first stage starts micro-batch j of step t + 1 as soon as the last stage has sampled its
// tokens (token flag e(t, j)), so with m >= s micro-batches every stage streams its weights
// continuously.  Epochs: e(t, j) = base + t * m + j + 1, monotone in every stage's order.
static hs_status ve_reserve(hs_group* g, Stage& s, VeBuffers& b, size_t slot_bytes, int slots, size_t tok_ints) {
  DeviceGuard dg(s.device);
  if (b.slot_bytes < slot_bytes || b.slots < slots) {
    if (b.h) cudaFreeHost(b.h);
    if (b.d) cudaFree(b.d);
    for (auto e : b.ev) cudaEventDestroy(e);
    b.ev.clear();
    b.slot_bytes = std::max(b.slot_bytes, slot_bytes);
    b.slots = std::max(b.slots, slots);
    HS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&b.h), b.slot_bytes * b.slots, cudaHostAllocMapped | cudaHostAllocPortable));
    HS_CUDA(cudaMalloc(reinterpret_cast<void**>(&b.d), b.slot_bytes * b.slots));
    b.ev.assign(b.slots, nullptr);
    for (auto& e : b.ev) HS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (b.tok_cap < tok_ints) {
    if (b.h_tok) cudaFreeHost(b.h_tok);
    b.tok_cap = tok_ints;
    HS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&b.h_tok), b.tok_cap * 4 + 64, cudaHostAllocMapped | cudaHostAllocPortable));
  }
  (void)g;
  return HS_OK;
}

static void ve_free(VeBuffers& b) {
  if (b.h) cudaFreeHost(b.h);
  if (b.d) cudaFree(b.d);
  for (auto e : b.ev) cudaEventDestroy(e);
  if (b.h_tok) cudaFreeHost(b.h_tok);
  b = VeBuffers{};
}

static hs_status decode_steps(hs_group* g, int n, const int64_t* ids, const int32_t* in_tokens, int n_steps, int m_req,
                              int32_t* out_tokens) {
  if (g->dead) HS_FAIL(HS_E_CUDA, "group is dead after a CUDA error");
  if (n <= 0 || n > g->kv.max_seqs || !ids || !out_tokens || n_steps <= 0 || m_req <= 0)
    HS_FAIL(HS_E_INVAL, "bad decode_steps args");
  if (g->spmd && std::find(g->active.begin(), g->active.end(), g->owned_stage) == g->active.end())
    HS_FAIL(HS_E_STATE, "this rank's stage was released by consolidation");
  const hs_model_cfg& c = g->cfg;
  std::vector<int64_t> v(ids, ids + n);
  if ((int)std::set<int64_t>(v.begin(), v.end()).size() != n) HS_FAIL(HS_E_INVAL, "duplicate sequence ids");
  int need = 0;
  for (int i = 0; i < n; ++i) {
    auto it = g->seqs.find(ids[i]);
    if (it == g->seqs.end()) HS_FAIL(HS_E_INVAL, "sequence %lld was never prefilled", (long long)ids[i]);
    if (it->second.ctx + n_steps > c.max_seq) HS_FAIL(HS_E_INVAL, "sequence exceeds max_seq");
    need += (it->second.ctx + n_steps + kBlock - 1) / kBlock - (int)it->second.blocks.size();
  }
  if (need > (int)g->free_blocks.size()) HS_FAIL(HS_E_OOM, "KV blocks exhausted");
  const bool feedback = in_tokens == nullptr;
  if (feedback && v != g->last_ids) HS_FAIL(HS_E_INVAL, "device token feedback needs the previous call's seq order");
  if (!feedback)
    for (int i = 0; i < n; ++i)
      if (in_tokens[i] < 0 || in_tokens[i] >= c.vocab) HS_FAIL(HS_E_INVAL, "token id out of range");
  // layer-boundary capture covers hs_prefill / hs_decode_step calls only (one row layout per call)
  struct CaptureOff {
    hs_group* g; bool was;
    ~CaptureOff() { g->capture = was; }
  } capture_off{g, g->capture};
  g->capture = false;
  g->cap_rowmap.clear();
  // micro-batches on 4-sequence boundaries (token hand-offs move 16-byte words)
  const int quads = (n + 3) / 4;
  const int m = std::max(1, std::min({m_req, quads, kMaxMicro}));
  std::vector<int> s0(m + 1);
  for (int j = 0; j <= m; ++j) s0[j] = std::min(n, 4 * (int)((int64_t)quads * j / m));
  const int first = g->active.front(), last = g->active.back();
  const unsigned ep_prev = g->epoch;
  const unsigned base = g->epoch;
  auto ep = [&](int t, int j) { return base + (unsigned)(t * m + j) + 1; };
  const int H = c.hidden;
  const size_t row_ints = align_up((size_t)n, 4);
  CallMeta mx;
  mx.T = s0[1] - s0[0];
  for (int j = 0; j < m; ++j) mx.T = std::max(mx.T, s0[j + 1] - s0[j]);
  mx.n = mx.T;
  layout_meta(mx, g->max_blocks);
  const size_t slot_bytes = align_up(mx.bytes, 256);
  const int R = 2 * m;
  for (size_t ai = 0; ai < g->active.size(); ++ai) {
    Stage& s = g->st[g->active[ai]];
    if (!s.owned) continue;
    if (!s.load_issued) HS_FAIL(HS_E_STATE, "stage %d: no load issued", s.idx);
    HS_TRY(ve_reserve(g, s, g->ve[s.idx], slot_bytes, R, (size_t)n_steps * row_ints));
  }
  g->epoch += (unsigned)(n_steps * m);  // (no failure path left before the items are enqueued)
  // every step's KV slot, up front (capacity checked above; nothing can fail after this but CUDA)
  std::vector<int> ctx0(n);
  for (int i = 0; i < n; ++i) {
    ctx0[i] = g->seqs[ids[i]].ctx;
    HS_TRY(alloc_tokens(g, ids[i], n_steps));
  }
  int item = 0;
  for (int t = 0; t < n_steps; ++t)
    for (int j = 0; j < m; ++j, ++item) {
      const int a = s0[j], nb = s0[j + 1] - s0[j];
      CallMeta mm;
      mm.T = nb; mm.n = nb; mm.max_nq = 1; mm.decode = true;
      for (int i = a; i < a + nb; ++i) {
        mm.max_ctx = std::max(mm.max_ctx, ctx0[i] + t + 1);
        mm.kv_tokens += ctx0[i] + t + 1;
        mm.attn_pairs += ctx0[i] + t + 1;
      }
      layout_meta(mm, g->max_blocks);
      std::vector<int> dctx(nb);
      for (int i = 0; i < nb; ++i) dctx[i] = ctx0[a + i] + t + 1;
      for (size_t ai = 0; ai < g->active.size(); ++ai) {
        const int k = g->active[ai];
        Stage& s = g->st[k];
        if (!s.owned) continue;
        VeBuffers& vb = g->ve[k];
        DeviceGuard dg(s.device);
        cudaStream_t st = s.comp;
        const int slot = item % R;
        if (item >= R) HS_CUDA(cudaEventSynchronize(vb.ev[slot]));  // staging slot free again
        uint8_t* hm = vb.h + (size_t)slot * vb.slot_bytes;
        int* tok = reinterpret_cast<int*>(hm + mm.o_tok);
        int* pos = reinterpret_cast<int*>(hm + mm.o_pos);
        int* sl = reinterpret_cast<int*>(hm + mm.o_slot);
        int* lastr = reinterpret_cast<int*>(hm + mm.o_last);
        SeqDesc* sd = reinterpret_cast<SeqDesc*>(hm + mm.o_seqs);
        int* tab = reinterpret_cast<int*>(hm + mm.o_tab);
        for (int i = 0; i < nb; ++i) {
          const SeqState& ss = g->seqs[ids[a + i]];
          const int p = ctx0[a + i] + t;
          pos[i] = p;
          sl[i] = ss.blocks[p / kBlock] * kBlock + p % kBlock;
          tok[i] = (!feedback && t == 0) ? in_tokens[a + i] : 0;
          lastr[i] = i;
          sd[i].q_start = i; sd[i].n_q = 1; sd[i].pos0 = p; sd[i].table = i;
          for (int bb = 0; bb < g->max_blocks; ++bb)
            tab[(size_t)i * g->max_blocks + bb] = bb < (int)ss.blocks.size() ? ss.blocks[bb] : 0;
        }
        uint8_t* meta = vb.d + (size_t)slot * vb.slot_bytes;
        if (t == 0 && j == 0) HS_CUDA(cudaEventRecord(s.ev_c0, st));
        launch_small_copy(hm, meta, mm.bytes, st);
        HS_CUDA(cudaEventRecord(vb.ev[slot], st));
        const bool is_first = k == first, is_last = k == last;
        Stage* nx = is_last ? nullptr : &g->st[g->active[ai + 1]];
        bf16* x_in_rows = reinterpret_cast<bf16*>(s.comm + g->cl.x_in) + (size_t)a * H;
        int* tok_in = reinterpret_cast<int*>(s.comm + g->cl.tok_in) + a;
        // stage input
        if (is_first) {
          const int* d_tok = reinterpret_cast<const int*>(meta + mm.o_tok);
          if (t > 0 || feedback) {
            launch_wait(s.flag_tok(), t > 0 ? ep(t - 1, j) : ep_prev, s.err(), st);
            d_tok = tok_in;
            // the tokens of step t - 1 (this micro-batch) into the host token log
            if (t > 0) launch_small_copy(tok_in, vb.h_tok + (size_t)(t - 1) * row_ints + a, align_up((uint64_t)nb * 4, 16), st);
          }
          if (t == 0 && j == 0) HS_CUDA(cudaStreamWaitEvent(st, s.ev_embed, 0));
          launch_embed(d_tok, reinterpret_cast<const bf16*>(s.wptr(g->hdr.embed_off)), s.xa, nb, H, c.vocab, st);
        } else {
          launch_wait(s.flag_x(), ep(t, j), s.err(), st);
        }
        // this stage's layers: the decode stack (or the per-kernel path)
        if (t == 0 && j == 0) {
          for (int l = s.lb; l < s.le; ++l) HS_CUDA(cudaStreamWaitEvent(st, s.ev_layer[l], 0));
          if (s.le == c.n_layers) HS_CUDA(cudaStreamWaitEvent(st, s.ev_final, 0));
        }
        bool used = false, fin_done = false, normed = false;
        HS_TRY(run_dstack(g, s, mm, meta, is_first ? s.xa : x_in_rows, s.xa, dctx, &used, &fin_done));
        for (int l = s.lb; l < s.le && !used; ++l) {
          const bf16* xin = (l == s.lb && !is_first) ? x_in_rows : s.xa;
          HS_TRY(run_layer(g, s, l, xin, s.xa, mm, meta, normed, fin_done));
        }
        if (!is_last) {
          launch_send(s.xa, nx->comm + g->cl.x_in + (size_t)a * H * 2, (uint64_t)nb * H * 2, s.done(), nx->flag_x(), ep(t, j),
                      kSendCtas, st);
        } else {
          if (!fin_done)
            launch_rmsnorm(s.xa, reinterpret_cast<const int*>(meta + mm.o_last),
                           reinterpret_cast<const bf16*>(s.wptr(g->hdr.final_off + g->hdr.t_final_norm)), s.fin, nb, H,
                           c.rms_eps, st);
          GemmArgs ga{};
          ga.A = &s.lm; ga.B = s.b_fin; ga.M = c.vocab; ga.N = nb; ga.K = H; ga.epi = EPI_F32; ga.out = s.logits;
          ga.ldo = c.vocab; ga.workspace = s.ws; ga.workspace_bytes = kWorkspace; ga.counters = s.ctr;
          HS_TRY(gemm(ga, st));
          launch_argmax(s.logits, c.vocab, nb, s.d_tok_out + a, st);
          const uint64_t tb = align_up((uint64_t)nb * 4, 16);
          for (int kk : g->active) {  // token feedback (SPMD: every stage; local: first + full-memory)
            if (!g->spmd && kk != first && !g->st[kk].full_memory) continue;
            launch_send(s.d_tok_out + a, g->st[kk].comm + g->cl.tok_in + (size_t)a * 4, tb, s.done(), g->st[kk].flag_tok(),
                        ep(t, j), 1, st);
          }
          launch_small_copy(s.d_tok_out + a, vb.h_tok + (size_t)t * row_ints + a, tb, st);
        }
      }
    }
  // every stage's tail, after all items are enqueued (stages on one device share a stream): the
  // first stage collects the last step's tokens once sampled; the flags + error word to the host
  for (size_t ai = 0; ai < g->active.size(); ++ai) {
    const int k = g->active[ai];
    Stage& s = g->st[k];
    if (!s.owned) continue;
    DeviceGuard dg(s.device);
    cudaStream_t st = s.comp;
    if (k == first && k != last)
      for (int jj = 0; jj < m; ++jj) {
        launch_wait(s.flag_tok(), ep(n_steps - 1, jj), s.err(), st);
        launch_small_copy(reinterpret_cast<int*>(s.comm + g->cl.tok_in) + s0[jj],
                          g->ve[k].h_tok + (size_t)(n_steps - 1) * row_ints + s0[jj],
                          align_up((uint64_t)(s0[jj + 1] - s0[jj]) * 4, 16), st);
      }
    launch_small_copy(s.comm, s.h_out + align_up((uint64_t)n, 4), 16, st);  // flags + err word
    HS_CUDA(cudaEventRecord(s.ev_c1, st));
    s.called = true;
  }
  int err = 0;
  bool got = false;
  for (int k : g->active) {
    Stage& s = g->st[k];
    if (!s.owned) continue;
    DeviceGuard dg(s.device);
    cudaError_t e = cudaStreamSynchronize(s.comp);
    if (e != cudaSuccess) {
      g->dead = true;
      HS_FAIL(HS_E_CUDA, "stage %d: %s", k, cudaGetErrorString(e));
    }
    err |= s.h_out[align_up((uint64_t)n, 4) + CommLayout::ERR / 4];
    if (!got && (k == first || k == last)) {
      for (int t = 0; t < n_steps; ++t) memcpy(out_tokens + (size_t)t * n, g->ve[k].h_tok + (size_t)t * row_ints, (size_t)n * 4);
      got = true;
    }
  }
  if (err) {
    g->dead = true;
    HS_FAIL(HS_E_TIMEOUT, "a cross-stage wait timed out (peer never signalled)");
  }
  g->last_ids = v;
  return HS_OK;
}

// ------------------------------------------------------------------ consolidation (a17) --
static hs_status open_peer_memory(hs_group* g, Stage& s) {
  if (s.owned || s.ipc_arena_open || !g->spmd) return HS_OK;
  void* p = nullptr;
  HS_CUDA(cudaIpcOpenMemHandle(&p, s.share.arena, cudaIpcMemLazyEnablePeerAccess));
  s.arena = reinterpret_cast<uint8_t*>(p);
  HS_CUDA(cudaIpcOpenMemHandle(&p, s.share.kv, cudaIpcMemLazyEnablePeerAccess));
  s.kv_mem = reinterpret_cast<uint8_t*>(p);
  s.ipc_arena_open = true;
  for (void* q : {static_cast<void*>(s.arena), static_cast<void*>(s.kv_mem)}) {  // mapped as device memory
    cudaPointerAttributes at{};
    HS_CUDA(cudaPointerGetAttributes(&at, q));
    if (at.type != cudaMemoryTypeDevice) HS_FAIL(HS_E_CUDA, "peer mapping %p is not device memory", q);
  }
  return HS_OK;
}

// Appends {src, dst, bytes} to a copy list in pieces of at most `piece` bytes.  copy_list_kernel
// moves 16-byte words: every address and size must be a multiple of 16 (weight slices are
// HS_IMAGE_ALIGN aligned, KV blocks are 16 * 2 * H * 2 bytes), checked here rather than
// silently dropping a tail.
static hs_status add_copy(std::vector<CopyDesc>& list, uint64_t src, uint64_t dst, uint64_t bytes, uint64_t piece) {
  if ((src | dst | bytes | piece) & 15)
    HS_FAIL(HS_E_INVAL, "copy list: src 0x%llx dst 0x%llx bytes %llu not 16-byte aligned", (unsigned long long)src,
            (unsigned long long)dst, (unsigned long long)bytes);
  for (uint64_t o = 0; o < bytes; o += piece) list.push_back({src + o, dst + o, std::min(piece, bytes - o)});
  return HS_OK;
}

static hs_status consolidate(hs_group* g, int tgt, hs_consolidate_stats* out) {
  using clk = std::chrono::steady_clock;
  const auto t_enter = clk::now();
  if (g->dead) HS_FAIL(HS_E_CUDA, "group is dead");
  if (tgt < 0 || tgt >= (int)g->st.size() || std::find(g->active.begin(), g->active.end(), tgt) == g->active.end())
    HS_FAIL(HS_E_INVAL, "target stage %d is not active", tgt);
  if (!g->st[tgt].full_memory) HS_FAIL(HS_E_INVAL, "target stage %d is not a full-memory worker", tgt);
  const hs_model_cfg& c = g->cfg;
  hs_consolidate_stats stats{};
  // 1. drain: "stop scheduling ... wait for all on-the-fly batches".  Only this
  //    process's streams: no cross-rank barrier is needed in SPMD mode, because the previous call
  //    returned on every rank only after the last stage's token broadcast, and each stage hands
  //    off (release, system scope) only after all its layers (KV writes included) completed, so
  //    every source's KV and weights are final and visible before the target's copy starts; and
  //    the released memory is freed only at hs_release_peer_memory / destroy, behind a barrier
  //    that the target reaches after its copy.
  for (int k : g->active) {
    Stage& s = g->st[k];
    if (!s.owned) continue;
    DeviceGuard dg(s.device);
    HS_CUDA(cudaStreamSynchronize(s.comp));
    HS_CUDA(cudaStreamSynchronize(s.copy));
  }
  const auto t_drained = clk::now();
  auto t_listed = t_drained, t_copied = t_drained;
  Stage& T = g->st[tgt];
  if (T.owned) {
    DeviceGuard dg(T.device);
    cudaSetDevice(T.device);
    cudaStream_t s2 = T.comp;
    // 2. one copy list, pulled over NVLink by the target's SMs (16-byte loads, many in flight):
    //    (a) the weight regions the target lacks (each owner's stage slice; prebuilt at create),
    //    (b) the used KV blocks of every live sequence for those layers, placed at the same block
    //    ids ("collect these blocks from all workers with a gather operation ... placed at
    //    different layers, according to which worker it comes from")
    for (int k : g->active)
      if (k != tgt) HS_TRY(open_peer_memory(g, g->st[k]));
    HS_TRY(prepare_consolidation(g, T));
    std::vector<CopyDesc> kv;
    kv.reserve((size_t)g->kv.num_blocks * c.n_layers);
    for (int k : g->active) {
      if (k == tgt) continue;
      Stage& S = g->st[k];
      if (!T.bg_issued) stats.weight_bytes += g->plan.stage_bytes[k];
      for (int l = S.lb; l < S.le; ++l)
        for (auto& kvp : g->seqs)
          for (int b : kvp.second.blocks) {
            HS_TRY(add_copy(kv, reinterpret_cast<uint64_t>(S.kv_pool(l, g->kv_layer_bytes)) + (uint64_t)b * g->kv_block_bytes,
                            reinterpret_cast<uint64_t>(T.kv_pool(l, g->kv_layer_bytes)) + (uint64_t)b * g->kv_block_bytes,
                            g->kv_block_bytes, g->kv_block_bytes));
            stats.kv_bytes += g->kv_block_bytes;
          }
    }
    if ((int)kv.size() > T.cons_cap - T.cons_nw) HS_FAIL(HS_E_INVAL, "consolidation list overflow");
    if (!kv.empty()) {
      memcpy(T.cons_h + T.cons_nw, kv.data(), kv.size() * sizeof(CopyDesc));
      HS_CUDA(cudaMemcpyAsync(T.cons_d + T.cons_nw, T.cons_h + T.cons_nw, kv.size() * sizeof(CopyDesc),
                              cudaMemcpyHostToDevice, s2));
    }
    // with the background host path the weights came over the target's own PCIe link: only KV
    const int first = T.bg_issued ? T.cons_nw : 0;
    const int n = T.cons_nw + (int)kv.size() - first;
    if (T.bg_issued) {
      HS_CUDA(cudaStreamWaitEvent(s2, T.ev_bg, 0));  // the background load must be complete
      if (T.bg_from_peers) stats.weight_bytes_background = T.bg_bytes;
      else stats.weight_bytes_host = T.bg_bytes;
    }
    t_listed = clk::now();
    if (getenv("HS_DEBUG_CONS_SYNC")) {
      cudaError_t pe = cudaDeviceSynchronize();
      if (pe != cudaSuccess) HS_FAIL(HS_E_CUDA, "consolidate: fault before the copy list: %s", cudaGetErrorString(pe));
    }
    HS_CUDA(cudaEventRecord(T.ev_cons0, s2));
    launch_copy_list(T.cons_d + first, n, 8 * num_sms(T.device), s2);
    HS_CUDA(cudaEventRecord(T.ev_cons1, s2));
    HS_CUDA(cudaEventSynchronize(T.ev_cons1));
    float ms = 0;
    HS_CUDA(cudaEventElapsedTime(&ms, T.ev_cons0, T.ev_cons1));
    stats.seconds = ms / 1e3;
    t_copied = clk::now();
    // 3. rebind the target to every layer (maps already exist for a full-memory arena)
    T.lb = 0;
    T.le = c.n_layers;
    for (int l = 0; l < c.n_layers; ++l)
      if (!T.layers[l].maps) HS_TRY(make_layer_maps(g, T, l));
    // every layer is resident now: readiness events must not gate on stale loads
    for (int l = 0; l < c.n_layers; ++l) HS_CUDA(cudaEventRecord(T.ev_layer[l], T.copy));
    HS_CUDA(cudaEventRecord(T.ev_embed, T.copy));
    HS_CUDA(cudaEventRecord(T.ev_final, T.copy));
    T.load_issued = true;
  }
  const auto t_rebound = clk::now();
  // 4. release the other stages ("other workers are terminated"); a stage
  //    sharing the target's device hands its streams over first
  for (int k : g->active)
    if (k != tgt && g->st[k].owned && g->st[k].owns_streams && g->st[k].device == T.device && T.owned &&
        !T.owns_streams) {
      g->st[k].owns_streams = false;
      T.owns_streams = true;
    }
  for (int k : g->active)
    if (k != tgt) {
      Stage& S = g->st[k];
      if (!S.owned && S.ipc_arena_open) {  // unmapping ~GBs costs ~100 ms: defer it
        g->ipc_deferred.push_back(S.arena);
        g->ipc_deferred.push_back(S.kv_mem);
        S.ipc_arena_open = false;
        S.arena = nullptr;
        S.kv_mem = nullptr;
      }
      if (S.owned && g->spmd) {  // exported: peers may still map it; freed at the release point
        for (void* p : {static_cast<void*>(S.arena), static_cast<void*>(S.kv_mem), static_cast<void*>(S.comm)})
          if (p) g->exp_deferred.push_back({S.device, p});
        S.arena = nullptr;
        S.kv_mem = nullptr;
        S.comm = nullptr;
      }
      // the rest of the teardown (driver frees of GBs: tens of ms) waits for the release point
      g->stage_deferred.push_back(S);
      S = Stage{};
    }
  g->active = {tgt};
  g->st[tgt].lb = 0;
  g->st[tgt].le = c.n_layers;
  g->plan.pp = 1;
  const auto t_end = clk::now();
  stats.pause_seconds = std::chrono::duration<double>(t_end - t_enter).count();
  if (getenv("HS_DEBUG_CONS")) {
    auto ms = [](clk::time_point a, clk::time_point b) { return 1e3 * std::chrono::duration<double>(b - a).count(); };
    fprintf(stderr, "[hs] consolidate (stage %d): drain %.2f ms, KV list build + upload %.2f ms, copy %.2f ms "
            "(device %.2f ms), rebind %.2f ms, release %.2f ms, pause %.2f ms\n", g->owned_stage,
            ms(t_enter, t_drained), ms(t_drained, t_listed), ms(t_listed, t_copied), 1e3 * stats.seconds,
            ms(t_copied, t_rebound), ms(t_rebound, t_end), 1e3 * stats.pause_seconds);
  }
  if (out) *out = stats;
  return HS_OK;
}


// ------------------------------------------------------------------ scale-up ---------------
static hs_status scale_up(hs_group* g, const int32_t* owner_in, int32_t n_live, hs_group** out,
                          hs_consolidate_stats* out_stats) {
  const auto t_enter = std::chrono::steady_clock::now();
  if (g->dead) HS_FAIL(HS_E_CUDA, "group is dead");
  if (!out) HS_FAIL(HS_E_INVAL, "null out");
  const hs_model_cfg& c = g->cfg;
  const int np = (int)g->active.size();
  for (int k : g->active)
    if (!g->st[k].full_memory) HS_FAIL(HS_E_INVAL, "stage %d is not a full-memory worker", k);
  // live sequences in ascending id order -> owner endpoint
  std::vector<int64_t> live;
  for (auto& kv : g->seqs) live.push_back(kv.first);
  if (owner_in && n_live != (int)live.size()) HS_FAIL(HS_E_INVAL, "n_live %d != %zu live sequences", n_live, live.size());
  std::map<int64_t, int> owner;
  for (size_t i = 0; i < live.size(); ++i) {
    const int o = owner_in ? owner_in[i] : g->active[i % np];
    if (std::find(g->active.begin(), g->active.end(), o) == g->active.end()) HS_FAIL(HS_E_INVAL, "bad owner %d", o);
    owner[live[i]] = o;
  }
  // drain every stage ("wait for all on-the-fly batches")
  for (int k : g->active) {
    Stage& s = g->st[k];
    if (!s.owned) continue;
    DeviceGuard dg(s.device);
    HS_CUDA(cudaStreamSynchronize(s.comp));
    HS_CUDA(cudaStreamSynchronize(s.copy));
  }
  if (!comm_barrier(g)) HS_FAIL(HS_E_STATE, "barrier failed");
  hs_consolidate_stats tot{};
  const uint64_t piece = 64ull << 10;
  struct Pending { int k; CopyDesc* d; cudaEvent_t e0, e1; };
  std::vector<Pending> pend;
  for (int t : g->active) {  // every stage pulls what it lacks, all GPUs concurrently
    Stage& T = g->st[t];
    if (!T.owned) continue;
    DeviceGuard dg(T.device);
    std::vector<CopyDesc> list;
    auto add = [&](uint64_t src, uint64_t dst, uint64_t bytes) -> hs_status {
      return add_copy(list, src, dst, bytes, piece);
    };
    for (int k : g->active) {
      if (k == t) continue;
      Stage& S = g->st[k];
      HS_TRY(open_peer_memory(g, S));
      HS_TRY(add(reinterpret_cast<uint64_t>(S.arena + (S.slice_begin - S.arena_off0)),
                 reinterpret_cast<uint64_t>(T.wptr(S.slice_begin)), S.slice_end - S.slice_begin));
      tot.weight_bytes += g->plan.stage_bytes[k];
      for (int l = S.lb; l < S.le; ++l)
        for (auto& kvp : g->seqs) {
          if (owner[kvp.first] != t) continue;
          for (int b : kvp.second.blocks) {
            HS_TRY(add(reinterpret_cast<uint64_t>(S.kv_pool(l, g->kv_layer_bytes)) + (uint64_t)b * g->kv_block_bytes,
                       reinterpret_cast<uint64_t>(T.kv_pool(l, g->kv_layer_bytes)) + (uint64_t)b * g->kv_block_bytes,
                       g->kv_block_bytes));
            tot.kv_bytes += g->kv_block_bytes;
          }
        }
    }
    Pending p{t, nullptr, nullptr, nullptr};
    HS_CUDA(cudaEventCreate(&p.e0));
    HS_CUDA(cudaEventCreate(&p.e1));
    if (!list.empty()) {
      HS_CUDA(cudaMalloc(&p.d, list.size() * sizeof(CopyDesc)));
      HS_CUDA(cudaMemcpy(p.d, list.data(), list.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
    }
    HS_CUDA(cudaEventRecord(p.e0, T.comp));
    launch_copy_list(p.d, (int)list.size(), 8 * num_sms(T.device), T.comp);
    HS_CUDA(cudaEventRecord(p.e1, T.comp));
    pend.push_back(p);
  }
  double secs = 0;
  for (auto& p : pend) {
    DeviceGuard dg(g->st[p.k].device);
    HS_CUDA(cudaEventSynchronize(p.e1));
    float ms = 0;
    HS_CUDA(cudaEventElapsedTime(&ms, p.e0, p.e1));
    secs = std::max(secs, (double)ms / 1e3);
    cudaEventDestroy(p.e0);
    cudaEventDestroy(p.e1);
    if (p.d) cudaFree(p.d);
  }
  tot.seconds = secs;
  if (!comm_barrier(g)) HS_FAIL(HS_E_STATE, "barrier failed");
  // split: each owned stage becomes a single-stage group with its sequences
  int n_out = 0;
  std::vector<int> owned_stages;
  for (int k : g->active)
    if (g->st[k].owned) owned_stages.push_back(k);
  for (int k : owned_stages) {
    Stage& S = g->st[k];
    std::unique_ptr<hs_group> ng(new hs_group());
    ng->cfg = g->cfg;
    ng->hdr = g->hdr;
    ng->kv = g->kv;
    ng->cl = g->cl;
    ng->kv_layer_bytes = g->kv_layer_bytes;
    ng->kv_block_bytes = g->kv_block_bytes;
    ng->max_blocks = g->max_blocks;
    ng->plan = g->plan;
    ng->plan.pp = 1;
    ng->plan.device[0] = S.device;
    ng->plan.layer_begin[0] = 0;
    ng->plan.layer_end[0] = c.n_layers;
    ng->plan.full_memory[0] = 1;
    ng->plan.stage_bytes[0] = g->hdr.param_bytes;
    ng->plan.slice_begin[0] = g->hdr.embed_off;
    ng->plan.slice_end[0] = g->hdr.total_bytes;
    ng->st.resize(1);
    ng->st[0] = std::move(S);
    S = Stage{};  // the old group no longer owns anything of this stage
    S.owned = false;
    Stage& T = ng->st[0];
    T.idx = 0;
    T.lb = 0;
    T.le = c.n_layers;
    T.slice_begin = g->hdr.embed_off;
    T.slice_end = g->hdr.total_bytes;
    if (!T.owns_streams) {  // stages that shared a device's streams get their own
      DeviceGuard dg(T.device);
      int lo = 0, hi = 0;
      HS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      HS_CUDA(cudaStreamCreateWithPriority(&T.comp, cudaStreamNonBlocking, hi));
      HS_CUDA(cudaStreamCreateWithPriority(&T.copy, cudaStreamNonBlocking, lo));
      T.owns_streams = true;
    }
    for (int l = 0; l < c.n_layers; ++l)
      if (!T.layers[l].maps) HS_TRY(make_layer_maps(ng.get(), T, l));
    {
      DeviceGuard dg(T.device);
      for (int l = 0; l < c.n_layers; ++l) HS_CUDA(cudaEventRecord(T.ev_layer[l], T.copy));
      HS_CUDA(cudaEventRecord(T.ev_embed, T.copy));
      HS_CUDA(cudaEventRecord(T.ev_final, T.copy));
      HS_CUDA(cudaMemset(T.comm, 0, 16));  // flags restart with the new group's epochs
      HS_CUDA(cudaDeviceSynchronize());
    }
    T.load_issued = true;
    ng->active = {0};
    for (int b = 0; b < g->kv.num_blocks; ++b) ng->free_blocks.insert(b);
    for (auto& kvp : g->seqs)
      if (owner[kvp.first] == k) {
        ng->seqs[kvp.first] = kvp.second;
        for (int b : kvp.second.blocks) ng->free_blocks.erase(b);
      }
    out[n_out++] = ng.release();
  }
  // the old group keeps only remote views (closed by destroy)
  g->active.clear();
  tot.pause_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_enter).count();
  if (out_stats) *out_stats = tot;
  return HS_OK;
}

}  // namespace hs

// ------------------------------------------------------------------ C ABI -----------------
using namespace hs;

extern "C" hs_status hs_group_create(const hs_model_cfg* cfg, const hs_plan* plan, const hs_image* image,
                                     const hs_image* stage_images, const hs_kv_cfg* kv, const hs_comm* comm,
                                     hs_group** out) {
  return create(cfg, plan, image, stage_images, kv, comm, out);
}

extern "C" hs_status hs_load_stage_async(hs_group* g, int32_t stage, uint64_t chunk_bytes) {
  if (!g) HS_FAIL(HS_E_INVAL, "null group");
  if (g->dead) HS_FAIL(HS_E_CUDA, "group is dead");
  if (stage == -1) {
    for (int k : g->active) HS_TRY(load_stage(g, k, chunk_bytes));
    return HS_OK;
  }
  if (std::find(g->active.begin(), g->active.end(), stage) == g->active.end()) HS_FAIL(HS_E_INVAL, "bad stage %d", stage);
  return load_stage(g, stage, chunk_bytes);
}

extern "C" hs_status hs_stage_load_stats(hs_group* g, int32_t stage, int32_t wait, hs_load_stats* out) {
  if (!g || !out || stage < 0 || stage >= (int)g->st.size()) HS_FAIL(HS_E_INVAL, "bad args");
  Stage& s = g->st[stage];
  if (!s.owned) HS_FAIL(HS_E_INVAL, "stage %d is not driven by this process", stage);
  if (!s.load_issued) HS_FAIL(HS_E_STATE, "no load issued");
  DeviceGuard dg(s.device);
  hs_load_stats r{};
  r.bytes = s.loaded_bytes;
  if (wait) HS_CUDA(cudaEventSynchronize(s.ev_l1));
  for (int l = s.lb; l < s.le; ++l) r.layers_ready += cudaEventQuery(s.ev_layer[l]) == cudaSuccess;
  cudaGetLastError();
  r.done = cudaEventQuery(s.ev_l1) == cudaSuccess;
  cudaGetLastError();
  if (r.done) HS_CUDA(cudaEventElapsedTime(&r.load_ms, s.ev_l0, s.ev_l1));
  *out = r;
  return HS_OK;
}

extern "C" hs_status hs_prefill(hs_group* g, int32_t n_seqs, const int64_t* seq_ids, const int32_t* tokens,
                                const int32_t* seq_lens, int32_t* out_tokens, float* out_logits) {
  if (!g) HS_FAIL(HS_E_INVAL, "null group");
  return prefill(g, n_seqs, seq_ids, tokens, seq_lens, out_tokens, out_logits);
}

extern "C" hs_status hs_decode_step(hs_group* g, int32_t n_seqs, const int64_t* seq_ids, const int32_t* in_tokens,
                                    int32_t* out_tokens, float* out_logits) {
  if (!g) HS_FAIL(HS_E_INVAL, "null group");
  return decode(g, n_seqs, seq_ids, in_tokens, out_tokens, out_logits);
}

extern "C" hs_status hs_release_seq(hs_group* g, int64_t seq_id) {
  if (!g) HS_FAIL(HS_E_INVAL, "null group");
  if (!g->seqs.count(seq_id)) HS_FAIL(HS_E_INVAL, "unknown sequence");
  release(g, seq_id);
  return HS_OK;
}

extern "C" hs_status hs_consolidate(hs_group* g, int32_t target_stage, hs_consolidate_stats* out) {
  if (!g) HS_FAIL(HS_E_INVAL, "null group");
  hs_status r = consolidate(g, target_stage, out);
  if (r == HS_E_CUDA) g->dead = true;
  return r;
}

extern "C" hs_status hs_scale_up(hs_group* g, const int32_t* seq_owner, int32_t n_live, hs_group** out,
                                 hs_consolidate_stats* stats) {
  if (!g) HS_FAIL(HS_E_INVAL, "null group");
  hs_status r = scale_up(g, seq_owner, n_live, out, stats);
  if (r == HS_E_CUDA) g->dead = true;
  return r;
}

// Collective (SPMD): close this rank's mappings of released peers' memory, meet, then free this
// rank's exported memory of released stages.  Every rank enters the barrier (a rank-local
// "dead" flag is not agreed on, so it must not decide who skips it); only a failed comm skips
// it, and then the exported memory stays allocated (a peer may still map it) while everything
// else is freed.  Safe to call any number of times.
static hs_status release_peer_memory(hs_group* g) {
  for (void* p : g->ipc_deferred)
    if (p) cudaIpcCloseMemHandle(p);
  g->ipc_deferred.clear();
  for (Stage& s : g->stage_deferred)  // importer side first: closes the comm mapping
    if (!s.owned) free_stage(s);
  const bool agreed = comm_barrier(g);
  if (agreed) {
    for (auto& dp : g->exp_deferred) {
      DeviceGuard dg(dp.first);
      cudaFree(dp.second);
    }
  }
  g->exp_deferred.clear();  // (without agreement: intentionally leaked, never freed under a peer)
  for (Stage& s : g->stage_deferred)
    if (s.owned) free_stage(s);
  g->stage_deferred.clear();
  if (!agreed) HS_FAIL(HS_E_STATE, "barrier failed: exported memory of released stages left allocated");
  return HS_OK;
}

extern "C" hs_status hs_release_peer_memory(hs_group* g) {
  if (!g) HS_FAIL(HS_E_INVAL, "null group");
  return release_peer_memory(g);
}

extern "C" hs_status hs_group_destroy(hs_group* g) {
  if (!g) return HS_OK;
  for (auto& s : g->st) {
    if (s.owned) {
      DeviceGuard dg(s.device);
      cudaDeviceSynchronize();
    }
  }
  prof_collect(g);
  for (auto& kv : g->ev_free) {
    DeviceGuard dg(kv.first);
    for (auto e : kv.second) cudaEventDestroy(e);
  }
  for (auto& kv : g->ve) {
    DeviceGuard dg(g->st[kv.first].device >= 0 ? g->st[kv.first].device : 0);
    ve_free(kv.second);
  }
  g->ve.clear();
  for (auto& s : g->st)
    if (!s.owned) free_stage(s);
  // SPMD: every importer closes its mappings of a peer's arena / KV / comm block before that
  // peer frees them (an exporter's cudaFree ahead of an importer's close is undefined), so the
  // ranks meet between the closes and the frees.  Without agreement (failed comm) the exported
  // regions stay allocated; every other resource is released either way.
  const hs_status r = release_peer_memory(g);
  const bool keep_exported = g->spmd && r != HS_OK;
  for (auto& s : g->st)
    if (s.owned) free_stage(s, keep_exported);
  delete g;
  return r;
}

extern "C" hs_status hs_group_info(hs_group* g, int32_t* pp, int32_t* owned) {
  if (!g) HS_FAIL(HS_E_INVAL, "null group");
  if (pp) *pp = (int32_t)g->active.size();
  if (owned) *owned = g->spmd ? g->owned_stage : -1;
  return HS_OK;
}

extern "C" hs_status hs_debug_read_kv(hs_group* g, int64_t seq_id, int32_t layer, int32_t pos0, int32_t n_pos,
                                      void* host_out) {
  if (!g || !host_out || layer < 0 || layer >= g->cfg.n_layers) HS_FAIL(HS_E_INVAL, "bad args");
  auto it = g->seqs.find(seq_id);
  if (it == g->seqs.end() || pos0 < 0 || pos0 + n_pos > it->second.ctx) HS_FAIL(HS_E_INVAL, "bad sequence/positions");
  int k = -1;
  HS_TRY(stage_of_layer(g, layer, &k));
  Stage& s = g->st[k];
  if (!s.owned) HS_FAIL(HS_E_INVAL, "layer %d lives on a stage of another process", layer);
  DeviceGuard dg(s.device);
  HS_CUDA(cudaStreamSynchronize(s.comp));
  const int nh = g->cfg.n_heads, d = g->cfg.head_dim;
  std::vector<uint16_t> blk(g->kv_block_bytes / 2);
  uint16_t* out = reinterpret_cast<uint16_t*>(host_out);
  int cur = -1;
  for (int p = pos0; p < pos0 + n_pos; ++p) {
    const int b = it->second.blocks[p / kBlock];
    if (b != cur) {
      HS_CUDA(cudaMemcpy(blk.data(), reinterpret_cast<uint8_t*>(s.kv_pool(layer, g->kv_layer_bytes)) +
                                          (uint64_t)b * g->kv_block_bytes,
                         g->kv_block_bytes, cudaMemcpyDeviceToHost));
      cur = b;
    }
    const int off = p % kBlock;
    for (int kv = 0; kv < 2; ++kv)
      for (int h = 0; h < nh; ++h)
        memcpy(out + (((size_t)(p - pos0) * 2 + kv) * nh + h) * d, blk.data() + (((size_t)kv * nh + h) * kBlock + off) * d,
               (size_t)d * 2);
  }
  return HS_OK;
}

extern "C" hs_status hs_debug_read_weights(hs_group* g, int32_t stage, uint64_t off, uint64_t bytes, void* host_out) {
  if (!g || stage < 0 || stage >= (int)g->st.size()) HS_FAIL(HS_E_INVAL, "bad args");
  Stage& s = g->st[stage];
  if (!s.owned || !s.arena) HS_FAIL(HS_E_INVAL, "stage not resident in this process");
  if (off < s.arena_off0 || off + bytes > s.arena_off0 + s.arena_bytes) HS_FAIL(HS_E_INVAL, "range outside arena");
  DeviceGuard dg(s.device);
  HS_CUDA(cudaDeviceSynchronize());
  HS_CUDA(cudaMemcpy(host_out, s.wptr(off), bytes, cudaMemcpyDeviceToHost));
  return HS_OK;
}

extern "C" hs_status hs_debug_poison_weights(hs_group* g, int32_t stage) {
  if (!g || stage < 0 || stage >= (int)g->st.size()) HS_FAIL(HS_E_INVAL, "bad args");
  Stage& s = g->st[stage];
  if (!s.owned || !s.arena) HS_FAIL(HS_E_INVAL, "stage not resident in this process");
  DeviceGuard dg(s.device);
  HS_CUDA(cudaDeviceSynchronize());
  HS_CUDA(cudaMemset(s.arena, 0xFF, s.arena_bytes));
  HS_CUDA(cudaDeviceSynchronize());
  return HS_OK;
}

extern "C" hs_status hs_debug_launch_count(hs_group* g, uint64_t* out) {
  (void)g;
  if (!out) HS_FAIL(HS_E_INVAL, "null out");
  *out = launch_total();
  return HS_OK;
}

extern "C" hs_status hs_stage_timing_get(hs_group* g, int32_t stage, hs_stage_timing* out) {
  if (!g || !out || stage < 0 || stage >= (int)g->st.size()) HS_FAIL(HS_E_INVAL, "bad args");
  Stage& s = g->st[stage];
  if (!s.owned || !s.comp) HS_FAIL(HS_E_INVAL, "stage %d is not driven by this process", stage);
  DeviceGuard dg(s.device);
  hs_stage_timing t{};
  if (s.load_issued && s.ev_l1) {
    HS_CUDA(cudaEventSynchronize(s.ev_l1));
    HS_CUDA(cudaEventElapsedTime(&t.load_ms, s.ev_l0, s.ev_l1));
  }
  if (s.called) {
    HS_CUDA(cudaEventSynchronize(s.ev_c1));
    HS_CUDA(cudaEventElapsedTime(&t.call_ms, s.ev_c0, s.ev_c1));
    if (s.load_issued) {
      cudaError_t e = cudaEventElapsedTime(&t.since_load_ms, s.ev_l0, s.ev_c1);
      if (e != cudaSuccess) { cudaGetLastError(); t.since_load_ms = -1; }
    }
  }
  *out = t;
  return HS_OK;
}

extern "C" hs_status hs_profile_enable(hs_group* g, int32_t on) {
  if (!g) HS_FAIL(HS_E_INVAL, "null group");
  g->prof_on = on != 0;
  return HS_OK;
}

extern "C" hs_status hs_profile_read(hs_group* g, hs_prof_entry* out, int32_t max_entries, int32_t* n, int32_t reset) {
  if (!g || !n) HS_FAIL(HS_E_INVAL, "bad args");
  HS_TRY(prof_collect(g));
  int i = 0;
  for (auto& kv : g->prof_acc) {
    if (out && i < max_entries) {
      hs_prof_entry& e = out[i];
      memset(&e, 0, sizeof(e));
      snprintf(e.name, sizeof(e.name), "%s.%s", kProfNames[kv.first / 2], (kv.first & 1) ? "decode" : "prefill");
      e.count = kv.second.count;
      e.ms = kv.second.ms;
      e.bytes = kv.second.bytes;
      e.flops = kv.second.flops;
    }
    ++i;
  }
  *n = i;
  if (reset) g->prof_acc.clear();
  return HS_OK;
}

extern "C" hs_status hs_debug_comm_selftest(const hs_comm* comm) {
  if (!comm || !comm->allgather || !comm->barrier || comm->world <= 0 || comm->rank < 0 || comm->rank >= comm->world)
    HS_FAIL(HS_E_INVAL, "bad comm");
  struct Msg { int32_t rank, world; uint64_t tag; char pad[48]; } me{};
  me.rank = comm->rank;
  me.world = comm->world;
  me.tag = 0x48535350ull * (uint64_t)(comm->rank + 1);
  std::vector<Msg> all(comm->world);
  if (comm->allgather(comm->ctx, &me, sizeof(Msg), all.data()) != 0) HS_FAIL(HS_E_STATE, "allgather failed");
  for (int r = 0; r < comm->world; ++r)
    if (all[r].rank != r || all[r].world != comm->world || all[r].tag != 0x48535350ull * (uint64_t)(r + 1))
      HS_FAIL(HS_E_STATE, "allgather returned wrong bytes for rank %d", r);
  if (comm->barrier(comm->ctx) != 0) HS_FAIL(HS_E_STATE, "barrier failed");
  return HS_OK;
}

extern "C" hs_status hs_load_background_async(hs_group* g, int32_t target_stage, uint64_t chunk_bytes) {
  if (!g) HS_FAIL(HS_E_INVAL, "null group");
  if (g->dead) HS_FAIL(HS_E_CUDA, "group is dead");
  if (std::find(g->active.begin(), g->active.end(), target_stage) == g->active.end())
    HS_FAIL(HS_E_INVAL, "stage %d is not active", target_stage);
  return load_background(g, target_stage, chunk_bytes);
}

extern "C" hs_status hs_debug_capture(hs_group* g, int32_t enable) {
  if (!g) HS_FAIL(HS_E_INVAL, "null group");
  const size_t bytes = (size_t)(2 * g->cfg.n_layers + 1) * g->kv.max_tokens * g->cfg.hidden * 2;
  for (int k : g->active) {
    Stage& s = g->st[k];
    if (!s.owned) continue;
    DeviceGuard dg(s.device);
    if (enable && !s.cap) HS_ALLOC(s.cap, bytes);
    if (!enable && s.cap) {
      HS_CUDA(cudaDeviceSynchronize());
      HS_CUDA(cudaFree(s.cap));
      s.cap = nullptr;
    }
  }
  g->capture = enable != 0;
  g->cap_rowmap.clear();
  g->cap_owner.clear();
  return HS_OK;
}

extern "C" hs_status hs_debug_read_hidden(hs_group* g, int32_t boundary, int32_t row0, int32_t n_rows, void* host_out) {
  if (!g || !host_out || n_rows < 0) HS_FAIL(HS_E_INVAL, "bad args");
  if (!g->capture) HS_FAIL(HS_E_STATE, "capture is not enabled");
  if (boundary < 0 || boundary > 2 * g->cfg.n_layers || boundary >= (int)g->cap_owner.size())
    HS_FAIL(HS_E_INVAL, "bad boundary %d", boundary);
  if (row0 < 0 || row0 + n_rows > (int)g->cap_rowmap.size()) HS_FAIL(HS_E_INVAL, "rows outside the latest call");
  const int k = g->cap_owner[boundary];
  if (k < 0 || k >= (int)g->st.size() || !g->st[k].owned || !g->st[k].cap)
    HS_FAIL(HS_E_INVAL, "boundary %d was not captured by this process in the latest call", boundary);
  Stage& s = g->st[k];
  DeviceGuard dg(s.device);
  HS_CUDA(cudaStreamSynchronize(s.comp));
  const size_t H = g->cfg.hidden;
  const bf16* base = s.cap + (size_t)boundary * g->kv.max_tokens * H;
  uint8_t* out = static_cast<uint8_t*>(host_out);
  for (int r = row0; r < row0 + n_rows;) {  // contiguous runs of buffer rows
    int e = r + 1;
    while (e < row0 + n_rows && g->cap_rowmap[e] == g->cap_rowmap[e - 1] + 1) ++e;
    HS_CUDA(cudaMemcpy(out + (size_t)(r - row0) * H * 2, base + (size_t)g->cap_rowmap[r] * H, (size_t)(e - r) * H * 2,
                       cudaMemcpyDeviceToHost));
    r = e;
  }
  return HS_OK;
}

extern "C" hs_status hs_debug_set_prefill_chunking(hs_group* g, int32_t min_chunk_tokens, int32_t max_chunks) {
  if (!g || min_chunk_tokens < 0 || max_chunks < 0) HS_FAIL(HS_E_INVAL, "bad args");
  g->chunk_tokens = min_chunk_tokens;
  g->max_chunks = max_chunks;
  return HS_OK;
}

extern "C" hs_status hs_decode_steps(hs_group* g, int32_t n_seqs, const int64_t* seq_ids, const int32_t* in_tokens,
                                     int32_t n_steps, int32_t n_micro, int32_t* out_tokens) {
  if (!g) HS_FAIL(HS_E_INVAL, "null group");
  return decode_steps(g, n_seqs, seq_ids, in_tokens, n_steps, n_micro, out_tokens);
}

extern "C" hs_status hs_pull_background_async(hs_group* g, int32_t target_stage, uint64_t chunk_bytes) {
  if (!g) HS_FAIL(HS_E_INVAL, "null group");
  if (g->dead) HS_FAIL(HS_E_CUDA, "group is dead");
  if (std::find(g->active.begin(), g->active.end(), target_stage) == g->active.end())
    HS_FAIL(HS_E_INVAL, "stage %d is not active", target_stage);
  return pull_background(g, target_stage, chunk_bytes);
}
