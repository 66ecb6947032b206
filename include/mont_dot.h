/*
 * mont_dot.h -- fused multiply-accumulate mod P with lazy reduction
 * (SURVEY.md §8(f) NEXT #4): the paper's "long sequences of modular
 * arithmetic" as batched dot products against one shared
 * vector -- a modular matrix-vector product.  Same conventions as mont.h.
 */
#ifndef MONT_DOT_H_
#define MONT_DOT_H_

#include "mont.h"

#ifdef __cplusplus
extern "C" {
#endif

/* out[r] = sum_{j<len} A[r*len + j] * x[j] * R^-1  mod P, canonical, for r < batch.
 * With x in Montgomery form (to_mont) this is the plain dot product A_r . x mod P.
 * Lazy reduction: each term is one signed REDC left in (-P, P) and the terms
 * are summed exactly in 64-bit integers (|sum| < len * P < 2^63), reduced once
 * per row at the end -- no per-term canonicalisation.  A, x canonical
 * residues.  One CTA per row, x read through the read-only cache; 4 B of HBM
 * per element of A.  len >= 1 when batch > 0; len < 2^32. */
mont_status_t mont_dot(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *A, const uint32_t *x, size_t batch,
                       size_t len, cudaStream_t stream);

/* mont_dot with an explicit launch (measurement): cfg->variant 0 = the
 * default (= 1, measured fastest); 1 = one CTA per row,
 * 4 x 16 B per thread per trip; 2 = 8 x 16 B; 3 = 4 x 16 B with the next
 * trip's loads issued before this trip's products;
 * 4 = 8 x 16 B prefetched; 5 = rows split into cfg->chunk-element pieces
 * (multiple of 1024, 0 = 4096; needs len % 4 == 0, 16-byte aligned A and x,
 * len >= 2 chunks, else variant 1), one CTA each, whose canonical partials
 * are added into out[r] mod P by atomic compare-and-swap after the library
 * zeroes out (out must not overlap A or x); 6 / 7 = 2 / 4 rows per CTA
 * against one load of x (len % 4 == 0, 16-byte aligned A and x, else 1);
 * 8 = a persistent grid (cfg->ctas_per_sm x SMs CTAs, 0 = 2) streaming each
 * CTA's rows through a cfg->unroll-stage (2, 4 or 8; 0 = 4, or 2 if 4 do
 * not fit) shared-memory
 * ring of cfg->chunk-element tiles of A and x (0 = 4096) filled by bulk
 * copies (len % 4 == 0, 16-byte aligned A and x, else 1; at most 200 KiB of
 * ring).  cfg may be NULL.  Errors as mont_dot, plus MONT_EINVAL_ARG for
 * another variant, chunk, stage count or CTA count. */
struct mont_launch;
mont_status_t mont_dot_ex(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *A, const uint32_t *x, size_t batch,
                          size_t len, const struct mont_launch *cfg, cudaStream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* MONT_DOT_H_ */
