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

#ifdef __cplusplus
}
#endif

#endif /* MONT_DOT_H_ */
