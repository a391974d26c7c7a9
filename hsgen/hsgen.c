/* hsgen.c — seeded synthetic-input generator (see include/hsgen.h).
 * Shared by tests/oracle and the benchmark; contains no arithmetic of the method. */
#define _GNU_SOURCE
#include "hsgen.h"

#include <math.h>
#include <omp.h>
#include <string.h>

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint64_t hash3(uint64_t seed, uint64_t tensor, uint64_t i) {
  return mix64(mix64(seed) ^ mix64(tensor * 0xD1B54A32D192ED03ull ^ mix64(i)));
}

/* Box-Muller: one hash per pair of indices (2j, 2j+1) -> (r cos t, r sin t). */
static inline void normal_pair(uint64_t seed, uint32_t tensor_id, uint64_t pair, double* z0,
                               double* z1) {
  uint64_t h = hash3(seed, tensor_id, pair);
  /* single-precision transcendentals: ~4x faster than double; the draws stay a pure
   * function of (seed, tensor, index) on a given libm */
  float u1 = ((float)(uint32_t)(h >> 40) + 0.5f) * (1.0f / 16777216.0f);
  float u2 = ((float)(uint32_t)(h & 0xffffffull) + 0.5f) * (1.0f / 16777216.0f);
  float r = sqrtf(-2.0f * logf(u1)), s, c;
  sincosf(6.2831853f * u2, &s, &c);
  *z0 = (double)(r * c);
  *z1 = (double)(r * s);
}

double hsgen_normal(uint64_t seed, uint32_t tensor_id, uint64_t index) {
  double z0, z1;
  normal_pair(seed, tensor_id, index >> 1, &z0, &z1);
  return (index & 1) ? z1 : z0;
}

/* float -> bf16 bits, round to nearest even, NaN kept quiet. */
static inline uint16_t to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

int32_t hsgen_tensor_spec(const hs_model_cfg* c, uint32_t id, int64_t* rows, int64_t* cols,
                          double* scale, double* offset) {
  int64_t H = c->hidden, F = c->ffn, V = c->vocab;
  int64_t r = 0, k = 0;
  double sc = 1.0, off = 0.0;
  if (id == HSGEN_EMBED) { r = V; k = H; sc = 1.0; }
  else if (id == HSGEN_FINAL_NORM) { r = 1; k = H; sc = 0.1; off = 1.0; }
  else if (id == HSGEN_LM_HEAD) { r = V; k = H; sc = 1.0 / sqrt((double)H); }
  else if (id >= 16) {
    uint32_t l = (id - 16) / 16, t = (id - 16) % 16;
    if ((int32_t)l >= c->n_layers) return -1;
    switch (t) {
      case HSGEN_ATTN_NORM: case HSGEN_FFN_NORM: r = 1; k = H; sc = 0.1; off = 1.0; break;
      case HSGEN_WQ: case HSGEN_WK: case HSGEN_WV: case HSGEN_WO: r = H; k = H; break;
      case HSGEN_WG: case HSGEN_WU: r = F; k = H; break;
      case HSGEN_WD: r = H; k = F; break;
      default: return -1;
    }
    if (t != HSGEN_ATTN_NORM && t != HSGEN_FFN_NORM) sc = 1.0 / sqrt((double)k);
  } else {
    return -1;
  }
  if (rows) *rows = r;
  if (cols) *cols = k;
  if (scale) *scale = sc;
  if (offset) *offset = off;
  return 0;
}

static inline uint16_t draw(uint64_t seed, uint32_t id, uint64_t i, double sc, double off) {
  return to_bf16((float)(off + sc * hsgen_normal(seed, id, i)));
}

void hsgen_tensor_bf16(const hs_model_cfg* cfg, uint64_t seed, uint32_t id, uint64_t start,
                       uint64_t count, uint16_t* out, int32_t nthreads) {
  double sc = 1, off = 0;
  if (hsgen_tensor_spec(cfg, id, 0, 0, &sc, &off) != 0) return;
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads) if (count > 65536)
  for (int64_t i = 0; i < (int64_t)count; ++i) {
    uint64_t g = start + (uint64_t)i;
    if ((g & 1) == 0 && i + 1 < (int64_t)count) continue; /* written with its odd partner */
    if (g & 1) {
      double z0, z1;
      normal_pair(seed, id, g >> 1, &z0, &z1);
      out[i] = to_bf16((float)(off + sc * z1));
      if (i > 0) out[i - 1] = to_bf16((float)(off + sc * z0));
    } else {
      out[i] = draw(seed, id, g, sc, off);
    }
  }
}

static inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

uint64_t hsgen_image_layout(const hs_model_cfg* c, hs_image_header* h) {
  if (!c || !h || c->n_layers <= 0 || c->n_layers > HS_MAX_LAYERS || c->hidden <= 0 ||
      c->ffn <= 0 || c->vocab <= 0 || c->ffn % HS_GU_INTERLEAVE)
    return 0;
  memset(h, 0, sizeof(*h));
  uint64_t H = (uint64_t)c->hidden, F = (uint64_t)c->ffn, V = (uint64_t)c->vocab;
  h->magic = HS_IMAGE_MAGIC;
  h->version = 2; /* 2: tiled weight matrices */
  h->gu_interleave = HS_GU_INTERLEAVE;
  h->cfg = *c;
  uint64_t o = 0;
  h->t_attn_norm = o; o = align_up(o + 2 * H, HS_TENSOR_ALIGN);
  h->t_wqkv = o;      o = align_up(o + 2 * 3 * H * H, HS_TENSOR_ALIGN);
  h->t_wo = o;        o = align_up(o + 2 * H * H, HS_TENSOR_ALIGN);
  h->t_ffn_norm = o;  o = align_up(o + 2 * H, HS_TENSOR_ALIGN);
  h->t_wgu = o;       o = align_up(o + 2 * 2 * F * H, HS_TENSOR_ALIGN);
  h->t_wd = o;        o = o + 2 * H * F;
  h->layer_bytes = align_up(o, HS_IMAGE_ALIGN);
  uint64_t p = HS_IMAGE_HEADER_BYTES;
  h->embed_off = p;
  h->embed_bytes = align_up(2 * V * H, HS_IMAGE_ALIGN);
  p += h->embed_bytes;
  for (int l = 0; l < c->n_layers; ++l) { h->layer_off[l] = p; p += h->layer_bytes; }
  h->final_off = p;
  h->t_final_norm = 0;
  h->t_lm_head = align_up(2 * H, HS_TENSOR_ALIGN);
  h->final_bytes = align_up(h->t_lm_head + 2 * V * H, HS_IMAGE_ALIGN);
  p += h->final_bytes;
  h->total_bytes = p;
  h->param_bytes = 2 * (V * H * 2 + H + (uint64_t)c->n_layers * (2 * H + 4 * H * H + 3 * F * H));
  return p;
}

/* Byte offset of element (row r, col k) of a [rows, cols] matrix: row-major, or the tiled
 * weight layout of include/hs.h ([rows/128][cols/64][128][64], each block contiguous). */
static inline uint64_t elem_off(int64_t r, int64_t k, int64_t cols, int tiled) {
  if (!tiled) return ((uint64_t)r * (uint64_t)cols + (uint64_t)k) * 2;
  const uint64_t blk = (uint64_t)(r >> 7) * (uint64_t)(cols >> 6) + (uint64_t)(k >> 6);
  return (blk * 8192 + (uint64_t)(r & 127) * 64 + (uint64_t)(k & 63)) * 2;
}

/* Enumerates the physical rows of tensor region [off, off + rows*cols*2). */
static void fill_rows(const hs_model_cfg* c, uint64_t seed, uint8_t* dst, uint64_t begin,
                      uint64_t end, uint64_t base, int64_t nrows, int64_t cols, int kind,
                      uint32_t id0, uint32_t id1, int nthreads, int tiled) {
  /* kind 0: plain tensor id0; kind 1: stacked q,k,v (id0..id0+2, H rows each);
   * kind 2: gate/up interleaved (id0 = gate, id1 = up).  tiled: weight-matrix layout. */
  uint64_t tb = base, te = base + (uint64_t)nrows * (uint64_t)cols * 2;
  if (te <= begin || tb >= end) return;
  int64_t r0 = (int64_t)((begin > tb ? begin - tb : 0) / (uint64_t)(cols * 2));
  int64_t r1 = (int64_t)(((end < te ? end : te) - tb + (uint64_t)cols * 2 - 1) / (uint64_t)(cols * 2));
  if (tiled) { r0 = 0; r1 = nrows; } /* a tile mixes rows: test every element's own offset */
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads)
  for (int64_t pr = r0; pr < r1; ++pr) {
    uint32_t id = id0;
    int64_t lr = pr;
    if (kind == 1) { int64_t H = c->hidden; id = id0 + (uint32_t)(pr / H); lr = pr % H; }
    else if (kind == 2) {
      int64_t G = HS_GU_INTERLEAVE, b = pr / (2 * G), j = pr % (2 * G);
      if (j < G) { id = id0; lr = b * G + j; } else { id = id1; lr = b * G + j - G; }
    }
    double sc, off;
    hsgen_tensor_spec(c, id, 0, 0, &sc, &off);
    double z0 = 0, z1 = 0;
    uint64_t have = ~0ull; /* pair index currently in (z0, z1) */
    for (int64_t k = 0; k < cols; ++k) {
      uint64_t ob = tb + elem_off(pr, k, cols, tiled);
      if (ob + 2 <= begin || ob >= end) continue;
      uint64_t li = (uint64_t)lr * (uint64_t)cols + (uint64_t)k;
      if ((li >> 1) != have) { normal_pair(seed, id, li >> 1, &z0, &z1); have = li >> 1; }
      uint16_t v = to_bf16((float)(off + sc * ((li & 1) ? z1 : z0)));
      /* bytes of v that fall inside [begin,end) */
      if (ob >= begin && ob + 2 <= end) memcpy(dst + (ob - begin), &v, 2);
      else if (ob < begin) dst[0] = (uint8_t)(v >> 8);
      else dst[ob - begin] = (uint8_t)(v & 0xff);
    }
  }
}

int32_t hsgen_image_fill(const hs_image_header* h, uint64_t seed, void* dstv, uint64_t begin,
                         uint64_t end, int32_t nthreads) {
  if (!h || h->magic != HS_IMAGE_MAGIC || end < begin || end > h->total_bytes) return -1;
  if (nthreads <= 0) nthreads = omp_get_max_threads();
  uint8_t* dst = (uint8_t*)dstv;
  const hs_model_cfg* c = &h->cfg;
  int64_t H = c->hidden, F = c->ffn, V = c->vocab;
  /* zero everything first (padding), then header, then tensors */
  uint64_t n = end - begin;
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t i = 0; i < (int64_t)((n + 4095) / 4096); ++i) {
    uint64_t a = (uint64_t)i * 4096, b = a + 4096 < n ? a + 4096 : n;
    memset(dst + a, 0, b - a);
  }
  if (begin < sizeof(hs_image_header)) {
    uint64_t e = end < sizeof(hs_image_header) ? end : sizeof(hs_image_header);
    memcpy(dst, (const uint8_t*)h + begin, e - begin);
  }
  fill_rows(c, seed, dst, begin, end, h->embed_off, V, H, 0, HSGEN_EMBED, 0, nthreads, 0);
  for (int l = 0; l < c->n_layers; ++l) {
    uint64_t L0 = h->layer_off[l];
    if (L0 >= end || L0 + h->layer_bytes <= begin) continue;
    fill_rows(c, seed, dst, begin, end, L0 + h->t_attn_norm, 1, H, 0, hsgen_layer_tensor(l, HSGEN_ATTN_NORM), 0, nthreads, 0);
    fill_rows(c, seed, dst, begin, end, L0 + h->t_wqkv, 3 * H, H, 1, hsgen_layer_tensor(l, HSGEN_WQ), 0, nthreads, 1);
    fill_rows(c, seed, dst, begin, end, L0 + h->t_wo, H, H, 0, hsgen_layer_tensor(l, HSGEN_WO), 0, nthreads, 1);
    fill_rows(c, seed, dst, begin, end, L0 + h->t_ffn_norm, 1, H, 0, hsgen_layer_tensor(l, HSGEN_FFN_NORM), 0, nthreads, 0);
    fill_rows(c, seed, dst, begin, end, L0 + h->t_wgu, 2 * F, H, 2, hsgen_layer_tensor(l, HSGEN_WG), hsgen_layer_tensor(l, HSGEN_WU), nthreads, 1);
    fill_rows(c, seed, dst, begin, end, L0 + h->t_wd, H, F, 0, hsgen_layer_tensor(l, HSGEN_WD), 0, nthreads, 1);
  }
  fill_rows(c, seed, dst, begin, end, h->final_off + h->t_final_norm, 1, H, 0, HSGEN_FINAL_NORM, 0, nthreads, 0);
  fill_rows(c, seed, dst, begin, end, h->final_off + h->t_lm_head, V, H, 0, HSGEN_LM_HEAD, 0, nthreads, 1);
  return 0;
}

void hsgen_tokens(uint64_t seed, int64_t n, int32_t vocab, int32_t* out) {
  for (int64_t i = 0; i < n; ++i)
    out[i] = (int32_t)(hash3(seed, 0xFFFFFFFFull, (uint64_t)i) % (uint64_t)vocab);
}
