// plan.cc — stage planning (a1) and the paper's predictors; host-only, no CUDA calls.
//
// PAPER.md §4.1: Eq. 1 (line 398), Eq. 2 (line 417), server selection (lines 408-413),
// Algorithm 1 (lines 420-452); §5.2 Eq. 5 (lines 579-584).  DESIGN.md readings R2 (contiguous
// split, remainder to the earliest stages) and R9 (Eq. 5 specialised to one box).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hs.h"

namespace hs {
static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }
const std::string& get_error() { return g_err; }
}  // namespace hs

using hs::set_error;

static inline uint64_t aup(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

static bool cfg_ok(const hs_model_cfg* c) {
  return c && c->n_layers > 0 && c->n_layers <= HS_MAX_LAYERS && c->n_heads > 0 &&
         c->n_kv_heads == c->n_heads && (c->head_dim == 64 || c->head_dim == 128) &&
         c->hidden == c->n_heads * c->head_dim && c->hidden % 128 == 0 && c->ffn % 64 == 0 &&
         (2 * c->ffn) % 128 == 0 && c->vocab % 128 == 0 && c->vocab > 0 && c->max_seq > 0 &&
         c->rms_eps > 0.f && c->rope_theta > 0.f;
}

extern "C" hs_status hs_image_layout(const hs_model_cfg* c, hs_image_header* h) {
  if (!cfg_ok(c) || !h) {
    set_error("hs_image_layout: unsupported model cfg");
    return HS_E_INVAL;
  }
  memset(h, 0, sizeof(*h));
  const uint64_t H = c->hidden, F = c->ffn, V = c->vocab;
  h->magic = HS_IMAGE_MAGIC;
  h->version = 2; /* 2: tiled weight matrices */
  h->gu_interleave = HS_GU_INTERLEAVE;
  h->cfg = *c;
  uint64_t o = 0;
  h->t_attn_norm = o; o = aup(o + 2 * H, HS_TENSOR_ALIGN);
  h->t_wqkv = o;      o = aup(o + 6 * H * H, HS_TENSOR_ALIGN);
  h->t_wo = o;        o = aup(o + 2 * H * H, HS_TENSOR_ALIGN);
  h->t_ffn_norm = o;  o = aup(o + 2 * H, HS_TENSOR_ALIGN);
  h->t_wgu = o;       o = aup(o + 4 * F * H, HS_TENSOR_ALIGN);
  h->t_wd = o;        o += 2 * H * F;
  h->layer_bytes = aup(o, HS_IMAGE_ALIGN);
  uint64_t p = HS_IMAGE_HEADER_BYTES;
  h->embed_off = p;
  h->embed_bytes = aup(2 * V * H, HS_IMAGE_ALIGN);
  p += h->embed_bytes;
  for (int l = 0; l < c->n_layers; ++l) { h->layer_off[l] = p; p += h->layer_bytes; }
  h->final_off = p;
  h->t_final_norm = 0;
  h->t_lm_head = aup(2 * H, HS_TENSOR_ALIGN);
  h->final_bytes = aup(h->t_lm_head + 2 * V * H, HS_IMAGE_ALIGN);
  p += h->final_bytes;
  h->total_bytes = p;
  h->param_bytes = 2 * (2 * V * H + H + (uint64_t)c->n_layers * (2 * H + 4 * H * H + 3 * F * H));
  return HS_OK;
}

extern "C" double hs_predict_ttft_eq1(double t_c, double M, int32_t s, int32_t w, const double* b,
                                      const double* p, double t_p, double t_n) {
  double mr = 0;
  for (int i = 0; i < s; ++i) mr = std::max(mr, 1.0 / b[i] + 1.0 / p[i]);
  return t_c + (M / s) * mr + t_p * (s - w + (double)w / s) + t_n * s;
}

extern "C" double hs_predict_tpot_eq2(double t_d, int32_t s, int32_t w, double t_n) {
  return t_d * (s - w + (double)w / s) + t_n * s;
}

extern "C" double hs_predict_ttft_eq5(double t_cc, double t_cu, double t_l, double M, int32_t s,
                                      int32_t w, const double* b, const double* p, double t_p,
                                      double t_n) {
  double f = 0;
  for (int i = 0; i < s; ++i)
    f = std::max(f, std::max(t_cc + t_cu + std::max((M / s) / p[i], t_l), (M / s) / b[i]));
  return f + t_p * (s - w + (double)w / s) + t_n * s;
}

// Bytes of one decoder layer / the embedding / the final norm + lm_head (no padding).
static uint64_t layer_params(const hs_model_cfg* c) {
  const uint64_t H = c->hidden, F = c->ffn;
  return 2 * (2 * H + 4 * H * H + 3 * F * H);
}

extern "C" hs_status hs_plan_stages(const hs_model_cfg* cfg, const hs_gpu* gpus, int32_t n_gpus,
                                    int32_t pp, int32_t full_memory_stages, double t_prefill_s,
                                    double t_hop_s, hs_plan* out) {
  if (!cfg_ok(cfg) || !gpus || !out || n_gpus <= 0) {
    set_error("hs_plan_stages: bad arguments");
    return HS_E_INVAL;
  }
  if (pp < 1 || pp > HS_MAX_STAGES || pp > cfg->n_layers) {
    set_error("hs_plan_stages: pp must be in [1, min(8, n_layers)] (pp = 0 is not implemented)");
    return HS_E_INVAL;
  }
  hs_image_header h;
  hs_image_layout(cfg, &h);
  const uint64_t H = cfg->hidden, V = cfg->vocab;
  const uint64_t emb = 2 * V * H, fin = 2 * (H + V * H), lay = layer_params(cfg);
  const uint64_t model = emb + fin + lay * (uint64_t)cfg->n_layers;
  hs_plan P;
  memset(&P, 0, sizeof(P));
  P.pp = pp;
  const int base = cfg->n_layers / pp, rem = cfg->n_layers % pp;
  uint64_t maxb = 0;
  for (int k = 0, b = 0; k < pp; ++k) {
    const int e = b + base + (k < rem ? 1 : 0);
    P.layer_begin[k] = b;
    P.layer_end[k] = e;
    uint64_t bytes = (uint64_t)(e - b) * lay;
    if (k == 0) bytes += emb;
    if (k == pp - 1) bytes += fin;
    P.stage_bytes[k] = bytes;
    P.slice_begin[k] = k == 0 ? h.embed_off : h.layer_off[b];
    P.slice_end[k] = k == pp - 1 ? h.final_off + h.final_bytes : h.layer_off[e];
    maxb = std::max(maxb, bytes);
    b = e;
  }
  // Selection rule with ratio 1/p_i (remote fetch absent: 1/b_i = 0).
  const int w = std::max(0, std::min<int>(full_memory_stages, pp));
  // ties in 1/p_i -> GPUs with fewer running workers first ("prioritizes free GPUs",
  // PAPER.md:421; R18), then device id
  struct Cand { double r; int nw; int dev; };
  std::vector<Cand> full, low;
  for (int i = 0; i < n_gpus; ++i) {
    if (gpus[i].h2d_gbps <= 0) { set_error("hs_plan_stages: h2d_gbps must be > 0"); return HS_E_INVAL; }
    const double r = 1.0 / gpus[i].h2d_gbps;
    if (gpus[i].free_bytes >= model) full.push_back({r, gpus[i].n_workers, gpus[i].device});
    else if (gpus[i].free_bytes >= maxb) low.push_back({r, gpus[i].n_workers, gpus[i].device});
  }
  auto less = [](const Cand& a, const Cand& b) {
    return a.r < b.r || (a.r == b.r && (a.nw < b.nw || (a.nw == b.nw && a.dev < b.dev)));
  };
  std::stable_sort(full.begin(), full.end(), less);
  if ((int)full.size() < w) { set_error("hs_plan_stages: not enough full-memory GPUs"); return HS_E_INFEASIBLE; }
  std::vector<Cand> rest(full.begin() + w, full.end());
  rest.insert(rest.end(), low.begin(), low.end());
  std::stable_sort(rest.begin(), rest.end(), less);
  if ((int)rest.size() < pp - w) { set_error("hs_plan_stages: not enough GPUs"); return HS_E_INFEASIBLE; }
  double pred = 0;
  for (int k = 0; k < pp; ++k) {
    const Cand& c = k < w ? full[k] : rest[k - w];
    P.device[k] = c.dev;
    P.full_memory[k] = k < w ? 1 : 0;
    pred = std::max(pred, (double)P.stage_bytes[k] * c.r / 1e9);
  }
  P.pred_ttft_s = pred + t_prefill_s * (pp - w + (double)w / pp) + t_hop_s * pp;
  *out = P;
  return HS_OK;
}

extern "C" const char* hs_last_error(void) { return hs::get_error().c_str(); }
