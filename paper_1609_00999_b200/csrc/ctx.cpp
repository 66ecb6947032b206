// ctx.cpp -- host-side Montgomery context.
//
// PAPER.md:89 defines P' by R R^-1 - P P' = 1, i.e. P' = -P^-1 mod R, and says
// it "can be computed using the extended Euclidean algorithm".  For R = 2^32
// this library instead lifts the 2-adic inverse by Newton's iteration
// x <- x (2 - P x) mod 2^32: P*P = 1 (mod 8) for odd P, so x0 = P is correct to
// 3 bits and four steps give 3 -> 6 -> 12 -> 24 -> 48 >= 32 bits.  The oracle
// uses extended Euclid; the two code paths share nothing.
#include <stdint.h>

#include "../../include/mont.h"

extern "C" mont_status_t mont_ctx_init(mont_ctx_t *ctx, uint32_t p) {
    if (!ctx) return MONT_EINVAL_ARG;
    if ((p & 1u) == 0u || p < 3u || p >= 0x80000000u) return MONT_EINVAL_P;
    uint32_t x = p;
    for (int i = 0; i < 4; ++i) x *= 2u - p * x;  // all mod 2^32
    // x = p^-1 mod 2^32 now; p * x == 1
    const uint32_t r1 = (uint32_t)((uint64_t{1} << 32) % p);
    ctx->p = p;
    ctx->pneg = 0u - x;
    ctx->r1 = r1;
    ctx->r2 = (uint32_t)(((uint64_t)r1 * r1) % p);
    return MONT_OK;
}

extern "C" const char *mont_strerror(mont_status_t s) {
    switch (s) {
        case MONT_OK: return "ok";
        case MONT_EINVAL_P: return "invalid modulus (need odd 3 <= P < 2^31)";
        case MONT_EINVAL_ARG: return "invalid argument (NULL pointer, bad context or size)";
        case MONT_ECUDA: return "CUDA runtime error during launch";
        case MONT_EUNSUPPORTED: return "unsupported request";
    }
    return "unknown status";
}

extern "C" int mont_build_arch(void) { return MONT_BUILD_ARCH; }
