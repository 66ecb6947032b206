/*
 * mont.h -- C ABI of the B200 (sm_100a) batched 32-bit Montgomery multiplication
 * library (libmont.so), the data-parallel hot path of arxiv 1609.00999,
 * "Automatic Generation of Vectorized Montgomery Algorithm".
 *
 * Arithmetic.  R = 2^32 and P is an odd modulus 3 <= P < 2^31 (DESIGN.md
 * reading G16; primality is not required, REDC needs only gcd(R, P) = 1,
 * PAPER.md:89).  REDC(a, b) = a*b*R^-1 mod P, computed with the paper's three
 * integer multiplications (Alg. 2 at PAPER.md:95-99) on the
 * integer-multiply (FMAHeavy) pipe -- T = a*b and m*P as 32x32->64 IMAD.WIDE,
 * the short product m as one IMAD -- and returned in the canonical range
 * [0, P).
 *
 * Conventions shared by every entry point below:
 *   - Array pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors),
 *     caller-owned; the library never frees or retains them.  Any 4-byte
 *     alignment is accepted; the 128-bit vector path is taken when all
 *     operands share the same address mod 16 (a scalar head is peeled),
 *     otherwise a 32-bit path runs.  out may alias an input exactly (in-place);
 *     partial overlap is undefined.
 *   - Element counts are size_t and may exceed 2^31 (64-bit indexing).
 *     n == 0 returns MONT_OK without launching anything.
 *   - Inputs must be canonical residues (< P) unless stated otherwise.  The
 *     exact REDC precondition is a*b < R*P, so one canonical
 *     operand suffices; with both operands >= P the output is unspecified
 *     (never a fault).
 *   - Every launcher is asynchronous on `stream` (0 = legacy default stream)
 *     and returns after enqueueing.  Synchronous argument validation returns
 *     MONT_EINVAL_*; a failed launch returns MONT_ECUDA.  Faults inside a
 *     kernel surface at the caller's next synchronisation (CUDA convention).
 *     No exceptions cross this boundary.
 *   - No global state, no allocation, re-entrant: concurrent calls on
 *     different streams are safe.  mont_ctx_t is a caller-owned immutable POD
 *     passed by value into every kernel.
 */
#ifndef MONT_H_
#define MONT_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Montgomery context for one modulus.
 *   p    : the modulus P
 *   pneg : P' = -P^-1 mod 2^32, the P' of "R R^-1 - P P' = 1"
 *   r1   : R mod P, the residue of 1 (1-bar)
 *   r2   : R^2 mod P, used by to_mont (x-bar = REDC(x, R^2 mod P))           */
typedef struct mont_ctx {
    uint32_t p;
    uint32_t pneg;
    uint32_t r1;
    uint32_t r2;
} mont_ctx_t;

typedef enum mont_status {
    MONT_OK = 0,
    MONT_EINVAL_P = 1,    /* modulus even, < 3 or >= 2^31                        */
    MONT_EINVAL_ARG = 2,  /* NULL pointer with n > 0, NULL ctx, bad size           */
    MONT_ECUDA = 3,       /* the CUDA runtime rejected a launch / attribute call   */
    MONT_EUNSUPPORTED = 4 /* request outside what this build implements            */
} mont_status_t;

/* Host only, no CUDA call.  Fills *ctx for modulus p: P' by Newton iteration
 * on the 2-adic inverse (x <- x(2 - p x) mod 2^32), r1 = 2^32 mod p,
 * r2 = r1^2 mod p.  PAPER.md:89 ("R^-1 and P' ... can be computed using the
 * extended Euclidean algorithm"; Newton reaches the same P').
 * Errors: MONT_EINVAL_ARG if ctx is NULL; MONT_EINVAL_P for even p, p < 3,
 * p >= 2^31 (ctx left untouched). */
mont_status_t mont_ctx_init(mont_ctx_t *ctx, uint32_t p);

/* out[i] = in[i] * R mod P (residue class i-bar = iR mod P),
 * computed as REDC(in[i], R^2 mod P) (PAPER.md:101 conversion).
 * in[i] may be any uint32 (REDC precondition holds since R^2 mod P < P).
 * 8 bytes of HBM traffic per element. */
mont_status_t to_mont(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *in, size_t n,
                      cudaStream_t stream);

/* out[i] = in[i] * R^-1 mod P = REDC(in[i], 1) (inverse map, PAPER.md:89,
 * :101).  in[i] may be any uint32.  8 bytes of HBM traffic per element. */
mont_status_t from_mont(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *in, size_t n,
                        cudaStream_t stream);

/* c[i] = REDC(a[i], b[i]) = a[i] * b[i] * R^-1 mod P, canonical in [0, P)
 * (Alg. 2, vectorised over the array as in §3.2 /
 * PAPER.md:121-139).  Raw REDC whatever the domain: Montgomery x Montgomery
 * gives Montgomery, plain x Montgomery gives plain.  12 bytes of HBM traffic
 * per element.  (BASELINE configs[0], [1], [4].) */
mont_status_t mont_mul_vec(const mont_ctx_t *ctx, uint32_t *c, const uint32_t *a, const uint32_t *b,
                           size_t n, cudaStream_t stream);

/* out[r*len + j] = REDC(x[r*len + j], tw[j]) for r < batch, j < len: every
 * row of a row-major batch x len matrix times one broadcast twiddle vector
 * (the NTT-stage twiddle multiply of the paper's modular FFTs, PAPER.md:19,
 * :189; BASELINE configs[2]).  With tw[j] = to_mont(w^j) this is
 * x * w^j mod P in the plain domain.  Each CTA stages its chunk of the table
 * into shared memory with the bulk-copy (TMA) engine, cp.async.bulk + mbarrier,
 * while its first x loads are in flight (mont_mul_twiddle_ex variant 2 instead
 * treats a power-of-two-len batch as one flat stream and reads the table
 * through L1; DESIGN.md §6 has both measured).  len not a multiple of 4 or
 * misaligned operands take a scalar path.  Requires len >= 1 when batch > 0.  x and out are batch*len
 * elements; out may alias x.  8 bytes of HBM traffic per element. */
mont_status_t mont_mul_twiddle(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *x,
                               const uint32_t *tw, size_t batch, size_t len, cudaStream_t stream);

/* out[i] = base[i]^exp[i] mod P, plain in / plain out (BASELINE configs[3];
 * DESIGN.md reading G10: 0^0 = 1, exponents are full 32-bit and not
 * reduced).  Internally: x-bar = to_mont(base), a left-to-right fixed-window
 * square-and-multiply ladder of Montgomery products held in registers, then
 * from_mont.  base[i] may be any uint32 (reduced mod P first).  12 bytes of
 * HBM traffic per element; bound by the integer-multiply pipe. */
mont_status_t mont_pow_vec(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *base,
                           const uint32_t *exp, size_t n, cudaStream_t stream);

/* *acc += sum_i x[i] (64-bit, device pointer, caller zeroes it), the
 * per-rank partial of the sum-mod-P checksum of BASELINE configs[4]
 * (SURVEY.md §8(a) A11).  Exact while the running total stays < 2^64
 * (n < 2^33 canonical residues).  acc must be 8-byte aligned.  Reduce mod P
 * on the host or after the cross-rank all-reduce.  4 bytes per element. */
mont_status_t mont_checksum(const mont_ctx_t *ctx, unsigned long long *acc, const uint32_t *x,
                            size_t n, cudaStream_t stream);

/* Fused A7 + A11: c[i] = REDC(a[i], b[i]) exactly as mont_mul_vec, and
 * *acc += sum_i c[i] (64-bit, device pointer, caller zeroes it) in the same
 * pass, so the checksum of configs[4] costs no second read of c.  One 64-bit
 * atomic per CTA.  Same argument rules as mont_mul_vec and mont_checksum. */
mont_status_t mont_mul_vec_checksum(const mont_ctx_t *ctx, uint32_t *c, const uint32_t *a, const uint32_t *b,
                                    size_t n, unsigned long long *acc, cudaStream_t stream);

/* tw[j] = to_mont(w^j mod P) for j < len: the Montgomery-form twiddle table of
 * BASELINE configs[2] (w a root of unity mod P).  Each element is an
 * independent square-and-multiply on the GPU. */
mont_status_t mont_twiddle_table(const mont_ctx_t *ctx, uint32_t *tw, uint32_t w, size_t len,
                                 cudaStream_t stream);

/* Human-readable text for a status code (static storage, never NULL). */
const char *mont_strerror(mont_status_t status);

/* Library build identification: returns the compiled SM target, e.g. 100. */
int mont_build_arch(void);

#ifdef __cplusplus
}
#endif

#endif /* MONT_H_ */
