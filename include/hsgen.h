/* hsgen.h — seeded synthetic-input generator shared by the oracle (tests) and the CUDA path.
 *
 * Holds none of the method's arithmetic: it only draws random numbers and writes them in
 * the host-image byte layout documented in hs.h.  Values are a pure function of
 * (seed, tensor_id, element index) — a counter-based generator — so any slice of any size
 * is reproducible independently (each rank can generate only its own stage slice).
 *
 * Initialisation recipe (SURVEY §8(c) reading 14):
 *   embed ~ N(0,1); W ~ N(0, 1/fan_in); norm weights ~ 1 + 0.1 N(0,1); all rounded to bf16
 *   (round-to-nearest-even).  Prompts: iid uniform token ids in [0, vocab).
 */
#ifndef HSGEN_H_
#define HSGEN_H_
#include <stdint.h>
#include "hs.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Tensor ids. */
enum {
  HSGEN_EMBED = 0, HSGEN_FINAL_NORM = 1, HSGEN_LM_HEAD = 2,
  /* layer l tensor k: 16 + 16*l + k */
  HSGEN_ATTN_NORM = 0, HSGEN_WQ = 1, HSGEN_WK = 2, HSGEN_WV = 3, HSGEN_WO = 4,
  HSGEN_FFN_NORM = 5, HSGEN_WG = 6, HSGEN_WU = 7, HSGEN_WD = 8
};
static inline uint32_t hsgen_layer_tensor(int layer, int k) { return 16u + 16u * (uint32_t)layer + (uint32_t)k; }

/* Logical shape and init distribution of a tensor id (rows x cols, value = offset + scale*z).
 * Returns 0 on success, -1 for an unknown id. */
int32_t hsgen_tensor_spec(const hs_model_cfg* cfg, uint32_t tensor_id, int64_t* rows,
                          int64_t* cols, double* scale, double* offset);

/* Elements [start, start+count) of a tensor in logical row-major order, as bf16 bits. */
void hsgen_tensor_bf16(const hs_model_cfg* cfg, uint64_t seed, uint32_t tensor_id,
                       uint64_t start, uint64_t count, uint16_t* out, int32_t nthreads);

/* Standard normal draw for (seed, tensor_id, index) (double, before scaling/rounding). */
double hsgen_normal(uint64_t seed, uint32_t tensor_id, uint64_t index);

/* Layout of the image (same rules as hs.h); returns total bytes (0 on invalid cfg). */
uint64_t hsgen_image_layout(const hs_model_cfg* cfg, hs_image_header* out);

/* Writes image bytes [begin, end) into dst (dst[0] == image byte `begin`), including the
 * header when [0, HS_IMAGE_HEADER_BYTES) intersects.  Padding bytes are zero.
 * Returns 0 on success. */
int32_t hsgen_image_fill(const hs_image_header* hdr, uint64_t seed, void* dst, uint64_t begin,
                         uint64_t end, int32_t nthreads);

/* n prompt tokens, uniform in [0, vocab), stream `seed`. */
void hsgen_tokens(uint64_t seed, int64_t n, int32_t vocab, int32_t* out);

#ifdef __cplusplus
}
#endif
#endif
