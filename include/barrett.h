/*
 * barrett.h -- Barrett reduction on B200, the
 * comparison point the paper argues against (§3.1: Alg. 1 at :71-85,
 * "three multiplications, at most four subtractions, and two bitwise shifts";
 * Montgomery needs "fewer addition/subtractions", :93, and is chosen for the
 * library, :119).  Plain domain: no residue-class conversion.  Same conventions
 * as mont.h.
 */
#ifndef BARRETT_H_
#define BARRETT_H_

#include "mont.h"

#ifdef __cplusplus
extern "C" {
#endif

/* k = ceil(log2 P), P' = floor(2^(2k) / P) */
typedef struct barrett_ctx {
    uint32_t p;
    uint32_t k;
    uint32_t pprime;  /* < 2^32 for odd 3 <= P < 2^31 */
    uint32_t pad;
} barrett_ctx_t;

/* host only; MONT_EINVAL_P for even P, P < 3, P >= 2^31 */
mont_status_t barrett_ctx_init(barrett_ctx_t *ctx, uint32_t p);

/* c[i] = a[i] * b[i] mod P by Alg. 1: m = floor(ab / 2^k), q = floor(m P' / 2^k),
 * t = ab - qP < 4P, then the "while t >= P" loop as two branch-free
 * corrections.  Canonical inputs (< P) required.  12 B of HBM per element. */
mont_status_t barrett_mul_vec(const barrett_ctx_t *ctx, uint32_t *c, const uint32_t *a, const uint32_t *b, size_t n,
                              cudaStream_t stream);

/* out[i] = base[i]^exp[i] mod P with the same 2-bit fixed-window ladder as
 * mont_pow_vec but Barrett products on plain values (base any uint32). */
mont_status_t barrett_pow_vec(const barrett_ctx_t *ctx, uint32_t *out, const uint32_t *base, const uint32_t *exp,
                              size_t n, cudaStream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* BARRETT_H_ */
