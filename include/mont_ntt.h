/*
 * mont_ntt.h -- number-theoretic transform on top of the Montgomery product
 * (SURVEY.md §8(f) NEXT #1): the consumer of the paper's vectorised Montgomery
 * multiplication, its "modular FFT" libraries.  Same
 * conventions as mont.h (device pointers, asynchronous on `stream`, status
 * codes, no global state, no allocation).
 */
#ifndef MONT_NTT_H_
#define MONT_NTT_H_

#include "mont.h"

#ifdef __cplusplus
extern "C" {
#endif

/* In-place batched NTT of `batch` rows of N = 2^log_n canonical residues
 * (row r at data + r*N, natural order in and out):
 *     X[k] = s * sum_{j<N} x[j] w^(j k)  mod P
 * tw    : the stage-major twiddle table of N - 1 Montgomery-form entries built
 *         by mont_ntt_twiddles(ctx, tw, w, log_n): for stage s = 1..log_n
 *         (pair distance h = 2^(s-1)) the h twiddles w^(pos N / 2h), pos < h,
 *         are contiguous at tw[h - 1 + pos], so the threads of a warp read
 *         consecutive words.  w a primitive N-th root of unity mod P; the
 *         table of w^-1 gives the inverse transform.
 * scale : the output factor s in Montgomery form (to_mont(s)); ctx->r1 means
 *         s = 1 (no extra multiply); to_mont(N^-1) with the w^-1 table makes
 *         the normalised inverse.
 * Radix-2 Gentleman-Sande (decimation in frequency) with each butterfly
 * (u, v) -> (u + v, REDC(u - v, tw)) on plain residues, mod add/sub by one
 * conditional correction ("straightforward"); 32 elements per
 * thread, five stages per trip through shared memory.  A row is read from and
 * written to HBM once: 8 bytes per element.  1 <= log_n <= 15 (N <= 32768 words = 128 KiB
 * of shared memory), else MONT_EUNSUPPORTED.  data 4-byte aligned; tw, data
 * device pointers; rows may not overlap. */
mont_status_t mont_ntt(const mont_ctx_t *ctx, uint32_t *data, size_t batch, int log_n, const uint32_t *tw,
                       uint32_t scale, cudaStream_t stream);

/* mont_ntt with an explicit kernel: variant 0 = decimation in frequency (the
 * default: natural-order input read straight into registers, shared memory in
 * a padded layout with the bit reversal done by the last trip's stores),
 * 1 = decimation in time (bit-reversed load, XOR-swizzled layout),
 * 2 = one butterfly per thread per stage in shared memory (reference),
 * 3 = variant 0 with precomputed-quotient twiddle products: `tw` is then the
 * PAIR table of mont_ntt_twiddles_pq (8-byte aligned, else MONT_EINVAL_ARG)
 * and each butterfly computes x w mod P as x w - hi(x w') P (Shoup), one high
 * product instead of REDC's two,
 * 4 / 5 = variants 0 / 3 with the XOR-swizzled shared layout (bit reversal in
 * the final gather; for measurement),
 * 6 / 7 = variants 0 / 3 as a persistent grid (resident CTAs x SMs looping over
 * the rows; the next row's loads are issued before this row's stores).  At
 * log_n = 15 (one CTA per SM) variants 0 / 3 run these kernels.  Variants 3-7
 * need log_n >= 5, else MONT_EUNSUPPORTED.  At log_n = 14 variants 0 / 3 also
 * prefetch the rows one wave ahead into L2 (cp.async.bulk.prefetch; the
 * environment variable MONT_NTT_NO_PF=1, read once, turns that off for
 * measurement).  For P < 2^30 variants 0, 3, 6 and 7 keep values between stages
 * in [0, 2P) (lazy butterflies, one correction fewer each; the environment
 * variable MONT_NTT_NO_LAZY=1, read once, turns that off for measurement).
 * All variants give identical outputs. */
mont_status_t mont_ntt_ex(const mont_ctx_t *ctx, uint32_t *data, size_t batch, int log_n, const uint32_t *tw,
                          uint32_t scale, int variant, cudaStream_t stream);

/* tw[2^(s-1) - 1 + pos] = to_mont(w^(pos * 2^(log_n - s))) for s = 1..log_n,
 * pos < 2^(s-1): N - 1 entries (device pointer), each an independent
 * square-and-multiply on the GPU.  1 <= log_n <= 30. */
mont_status_t mont_ntt_twiddles(const mont_ctx_t *ctx, uint32_t *tw, uint32_t w, int log_n, cudaStream_t stream);

/* Pair table for mont_ntt_ex variant 3: for each entry e of the table above
 * (same index e, same exponent), tw2[2e] = w^x mod P (plain, canonical) and
 * tw2[2e + 1] = floor(w^x 2^32 / P) -- which equals to_mont(w^x) * P' mod 2^32,
 * so it comes from the Montgomery context with one multiply.  2 (N - 1) words,
 * device pointer, 8-byte aligned.  1 <= log_n <= 30. */
mont_status_t mont_ntt_twiddles_pq(const mont_ctx_t *ctx, uint32_t *tw2, uint32_t w, int log_n,
                                   cudaStream_t stream);

/* ---- large transforms, 2^16 <= N <= 2^30 ----
 * (An N-point transform needs N | P - 1; for odd P < 2^31 that allows at most
 * N = 2^27, P = 15 * 2^27 + 1 = 2013265921: no prime c 2^k + 1 < 2^31 has k >= 28.)
 * N = N1 N2, x viewed as the N1 x N2 row-major matrix x[n1][n2].
 * 2^22 <= N <= 2^27: three passes over HBM.  (1) N2 column transforms of
 *   length N1 = 2^11 (2^12 for N = 2^22 and 2^27) straight down the matrix
 *   (8 adjacent columns per CTA, so
 *   every row access is one full 32-byte sector; no transpose), each output
 *   (k1, n2) times the 2-D twiddle w^(n2 k1) (the configs[2] "twiddle multiply
 *   of one NTT stage", generated from two half tables), in place; (2) N1 row
 *   transforms of length N2 = N / N1; (3) one transpose to natural order.
 *   Both transform passes multiply by their twiddles with precomputed
 *   quotients (the pair tables of mont_ntt_twiddles_pq).  HBM traffic 3 x 8
 *   bytes per element.
 * otherwise: six-step -- N1 = 2^floor(log_n/2), N2 = 2^ceil(log_n/2): transpose,
 *   N2 transforms of length N1 with the 2-D twiddle in their epilogue,
 *   transpose, N1 transforms of length N2, transpose to natural order (both
 *   transform passes with precomputed-quotient twiddles too).  HBM traffic
 *   5 x 8 bytes per element.
 *
 * plan: device buffer of mont_ntt_plan_words(log_n) words, 8-byte aligned, filled by
 *       mont_ntt_plan_init for a primitive N-th root w (w^-1: inverse).
 * in  : the N inputs (canonical); DESTROYED (used as scratch).
 * out : the N outputs, natural order; must not overlap `in`.
 * scale as in mont_ntt. */
size_t mont_ntt_plan_words(int log_n);   /* 0 if log_n is outside [16, 30] */
mont_status_t mont_ntt_plan_init(const mont_ctx_t *ctx, uint32_t *plan, uint32_t w, int log_n,
                                 cudaStream_t stream);
mont_status_t mont_ntt_large(const mont_ctx_t *ctx, uint32_t *out, uint32_t *in, int log_n,
                             const uint32_t *plan, uint32_t scale, cudaStream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* MONT_NTT_H_ */
