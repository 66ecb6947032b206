/*
 * mont_ext.h -- extended entry points of libmont.so: explicit launch
 * configuration for the hot kernels (used by bench.py and the tuning sweeps),
 * the counter-based synthetic input generator (device side of synth/), and
 * the two measurement microbenchmarks that provide the roofline denominators
 * (SURVEY.md §2.3 K7, K8).  Same conventions as mont.h (device pointers,
 * asynchronous on `stream`, status codes, no global state).
 */
#ifndef MONT_EXT_H_
#define MONT_EXT_H_

#include "mont.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Launch configuration.  Zero fields select the library default.
 *   threads   : threads per CTA (multiple of 32, <= 1024)
 *   ctas_per_sm: CTAs per SM for the persistent grid (grid = SMs * ctas_per_sm)
 *   unroll    : 128-bit chunks per thread per loop trip (1, 2, 4 or 8)
 *   variant   : kernel variant (kernel-specific; 0 = default).
 *                 mont_mul_vec_ex, mont_mul_vec_checksum_ex, to_mont_ex,
 *                 from_mont_ex, mb_triad, mb_copy : 0 = flat grid (one
 *                                   tile of threads*unroll uint4 per CTA),
 *                                   1 = persistent grid-stride over tiles
 *                                   with grid = SMs * ctas_per_sm,
 *                                   2 = flat grid, each CTA's tile staged by
 *                                   cp.async.bulk (chunk words per operand,
 *                                   default 8192),
 *                                   3 = persistent bulk-copy pipeline: grid =
 *                                   SMs * ctas_per_sm, a 4-stage TMA load
 *                                   ring + TMA stores of chunk-word tiles
 *                                   (default 2048), threads <= 256, so few
 *                                   warps stream at full bandwidth
 *                                   (variants 2 and 3: 16-byte co-aligned
 *                                   operands, else the 32-bit path)
 *                 mont_pow_vec_ex : 0 = 2-bit fixed window, table in
 *                                   registers; 1 = binary ladder with
 *                                   selects; 2 = 3-bit window, registers;
 *                                   3 = 2-bit window, table in shared memory;
 *                                   4 = 3-bit window, shared memory;
 *                                   5/6/7/8 = 2-bit window with 3/2/1/0 of
 *                                   each 4 lanes on the IMAD pipe and the
 *                                   rest as FP64 Barrett products on the
 *                                   FP64 pipe; 9 = 2-bit window with
 *                                   Fourier-prime REDC products (PAPER.md
 *                                   Alg. 3; P = c 2^n + 1, 2n >= 32,
 *                                   3P < 2^32, 16-byte aligned operands,
 *                                   else MONT_EUNSUPPORTED / EINVAL_ARG);
 *                                   10 = variant 0 with 8 lanes (two uint4)
 *                                   per thread.
 *                                   ctas_per_sm = 0 selects a flat grid.
 *                 mont_mul_twiddle_ex : 0 = bulk-copy (TMA) staged table,
 *                                   1 = table read through L1/L2 (no smem),
 *                                   2 = flat stream (power-of-two len; else 0),
 *                                   3 = whole table staged once per CTA
 *                                   by TMA + cluster-launch-control work
 *                                   stealing over 2-row items (4 len <=
 *                                   200 KiB; else 0)
 *   chunk     : mont_mul_twiddle_ex only: table columns staged per CTA
 *               (multiple of 4; 0 = min(len, 4096)).                       */
typedef struct mont_launch {
    int threads;
    int ctas_per_sm;
    int unroll;
    int variant;
    int chunk;
} mont_launch_t;

mont_status_t mont_mul_vec_ex(const mont_ctx_t *ctx, uint32_t *c, const uint32_t *a, const uint32_t *b,
                              size_t n, const mont_launch_t *cfg, cudaStream_t stream);
mont_status_t mont_mul_vec_checksum_ex(const mont_ctx_t *ctx, uint32_t *c, const uint32_t *a,
                                       const uint32_t *b, size_t n, unsigned long long *acc,
                                       const mont_launch_t *cfg, cudaStream_t stream);
mont_status_t to_mont_ex(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *in, size_t n,
                         const mont_launch_t *cfg, cudaStream_t stream);
mont_status_t from_mont_ex(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *in, size_t n,
                           const mont_launch_t *cfg, cudaStream_t stream);
mont_status_t mont_mul_twiddle_ex(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *x,
                                  const uint32_t *tw, size_t batch, size_t len,
                                  const mont_launch_t *cfg, cudaStream_t stream);
mont_status_t mont_pow_vec_ex(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *base,
                              const uint32_t *exp, size_t n, const mont_launch_t *cfg,
                              cudaStream_t stream);

/* Device side of the seeded generator of synth/ (SURVEY.md Appendix B):
 *   h(seed, stream, i) = splitmix64_mix(seed + (stream * 2^40 + i + 1) * GAMMA)
 * for i = start .. start + n - 1, mapped by `mode`:
 *   0 : floor(h * p / 2^64)              uniform in [0, p)
 *   1 : 1 + floor(h * (p - 1) / 2^64)    uniform in [1, p)
 *   2 : h >> 33                          31-bit exponent (p ignored)
 * If `specials` is nonzero, index i is then overwritten with 0, 1 or p-1 when
 * h(seed, stream + 16, i) mod 300 is 0, 1 or 2 (BASELINE configs[1] "1 % of
 * entries set to 0, 1 or P-1"; reading G13).  No modular
 * arithmetic of the method happens here. */
mont_status_t synth_fill(uint32_t *out, size_t n, uint64_t seed, uint32_t stream, uint64_t start,
                         uint32_t p, int mode, int specials, cudaStream_t stream_);

/* Microbenchmarks (roofline denominators, not part of the method).
 * mb_triad: c[i] = a[i] ^ b[i] over n uint32 with the same launch shape as
 *   mont_mul_vec: 12 bytes per element, the achievable 2-read/1-write HBM rate.
 * mb_copy: out[i] = in[i], 8 bytes per element.
 * mb_imad: every thread runs `iters` trips of 8 ops on each of 8 independent
 *   dependency chains of one kind (0 = IMAD mul.lo, 1 = IMAD.HI mul.hi,
 *   2 = IMAD.WIDE mad.wide, 3 = the library's signed chain REDC, 4 = its
 *   canonical REDC, 5 = REDC from mul.lo/mul.hi, 6 = REDC with an IMAD.HI
 *   64-bit addend, 7 = DFMA, 8 = the FP64 Barrett product, 9 = IADD,
 *   10 = LOP3, 11 = 3 Montgomery : 1 FP64 chains, 12 = 1 : 1, 13 = VIMNMX,
 *   14 = SHF, 15 = PAPER.md Alg. 3 for P = 7 2^26 + 1 with c = 7 as shifts,
 *   16 = 7 Montgomery : 1 Alg.-3 chains, 17 = 3 : 1; kind > 17 is
 *   MONT_EINVAL_ARG), writing one word per thread to sink[] (which must hold
 *   SMs * ctas_per_sm * 256 words); the caller times it and divides the
 *   executed count (threads * iters * 64) by the time.
 *   grid = SMs * ctas_per_sm, 256 threads (cfg may be NULL: 8 CTAs/SM). */
mont_status_t mb_triad(uint32_t *c, const uint32_t *a, const uint32_t *b, size_t n,
                       const mont_launch_t *cfg, cudaStream_t stream);
mont_status_t mb_copy(uint32_t *out, const uint32_t *in, size_t n, const mont_launch_t *cfg,
                      cudaStream_t stream);
mont_status_t mb_imad(uint32_t *sink, int kind, int iters, const mont_launch_t *cfg, cudaStream_t stream,
                      unsigned long long *threads_launched);

/* Number of SMs of the current device (cached per device), or -1. */
int mont_sm_count(void);

#ifdef __cplusplus
}
#endif

#endif /* MONT_EXT_H_ */
