/* hs_probes.h — test-only hardware probes, built into libhs_probe.so (never into libhs.so).
 * They measured design alternatives of the decode stack and are kept so the
 * measurement can be repeated; no product path calls them. */
#ifndef HS_PROBES_H_
#define HS_PROBES_H_
#include <stdint.h>

#include "hs.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Test-only probe of the tcgen05 A-operand-in-TMEM path: one 128 x 16 tile, K a multiple of
 * 64; A [128][K], B [16][K] bf16 device pointers; out_ss / out_ts [16][128] fp32 device
 * pointers receive D = A.B^T computed with A from shared memory / A copied to TMEM
 * (tcgen05.cp.128x256b) respectively.  Synchronous. */
hs_status hs_debug_tmem_a_gemm(const void* A, const void* B, int32_t K, float* out_ss, float* out_ts);

/* Test-only probe of TMA weight streaming in the decode stack's pattern (every SM streams a
 * contiguous range of 16 KiB k-blocks of an [M, K] bf16 matrix through a ring of `slots` (8 or
 * 12) shared-memory slots), `iters` passes: layout 0 = row-major [M, K] (128-byte row segments
 * per box row, the image layout), layout 1 = tiled (each 128 x 64 block contiguous); layout + 2:
 * the consumer issues the decode stack's MMAs on each slot (4 x M=128 N=16 K=16, slot released
 * by tcgen05.commit) instead of releasing it at once.
 * *gbs = achieved HBM GB/s of the timed launch.  Allocates and frees its own matrix. */
hs_status hs_debug_stream_probe(int32_t layout, int64_t M, int64_t K, int32_t slots, int32_t iters, double* gbs);

#ifdef __cplusplus
}
#endif
#endif
