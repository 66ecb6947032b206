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
 *   variant   : kernel variant (kernel-specific; 0 = the library default, which
 *               is variant 0 itself except for mont_pow_vec_ex and
 *               mont_mul_twiddle_ex, where 0 selects another variant below).
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
 *                                   operands, else the 32-bit path),
 *                                   4 (mont_mul_vec_ex and _checksum_ex only)
 *                                   = flat grid with every product on the
 *                                   FP64 pipe (two FP64 Barrett products per
 *                                   element, a b mod P then times R^-1 mod P;
 *                                   no FMAHeavy instruction; both operands
 *                                   canonical)
 *                 mont_pow_vec_ex : 0 = library default: 11 when base, exp
 *                                   and out share their address mod 16, else
 *                                   17;  1 = binary ladder with selects;
 *                                   2 = 3-bit window, registers;
 *                                   3 = 2-bit window, table in shared memory;
 *                                   4 = 3-bit window, shared memory;
 *                                   5/6/7/8 = 2-bit window with 3/2/1/0 of
 *                                   each 4 lanes on the IMAD pipe and the
 *                                   rest as FP64 Barrett products on the
 *                                   FP64 pipe; 9 = 2-bit window with
 *                                   Fourier-prime REDC products (PAPER.md
 *                                   Alg. 3; P = c 2^n + 1, 2n >= 32, with
 *                                   t held in 33 bits when 3P >= 2^32 --
 *                                   DESIGN.md G8; 16-byte aligned operands,
 *                                   else MONT_EUNSUPPORTED / EINVAL_ARG);
 *                                   10 = variant 17 with 8 lanes (two uint4)
 *                                   per thread; 11 = 2-bit window, 8 lanes
 *                                   per thread, P a compile-time constant for
 *                                   the config primes 469762049, 998244353,
 *                                   2013265921 (run time otherwise);
 *                                   12 = 11 with 2 of the 8 lanes as FP64
 *                                   Barrett products; 13 = 11 with
 *                                   precomputed-quotient (Shoup) window
 *                                   multiplies; 14 = 13 + 2 FP64 lanes;
 *                                   15 / 16 = 11 / 13 with P at run time;
 *                                   (11-16 need 16-byte co-aligned operands,
 *                                   else they run 17; they take threads =
 *                                   64, 128 (their default) or 256, the
 *                                   others 256); 17 = 2-bit fixed
 *                                   window, 4 lanes per thread, table in
 *                                   registers (any alignment).
 *                                   ctas_per_sm = 0 selects a flat grid.
 *                 mont_mul_twiddle_ex : 0 = library default: 4 (the table
 *                                   staged in shared memory by TMA);
 *                                   1 = table read through L1/L2 (no smem),
 *                                   2 = flat stream (power-of-two len; else 4),
 *                                   3 = whole table staged once per CTA
 *                                   by TMA + cluster-launch-control work
 *                                   stealing over 2-row items (4 len <=
 *                                   200 KiB; else 4),
 *                                   4 = table chunk staged per CTA by the
 *                                   bulk-copy (TMA) engine, cp.async.bulk +
 *                                   mbarrier (any len; 256 threads unless
 *                                   threads is set)
 *   chunk     : mont_mul_twiddle_ex: table columns staged per CTA
 *               (multiple of 4; 0 = min(len, 2048)).  mont_pow_vec_ex
 *               variants 11-16: bytes of dynamic shared memory reserved
 *               (never touched) per CTA, an occupancy cap that keeps a
 *               flat pow grid to a few CTAs per SM while other kernels
 *               co-run (0 = none, at most 227 KiB).                        */
typedef struct mont_launch {
    int threads;
    int ctas_per_sm;
    int unroll;
    int variant;
    int chunk;
    int flags;
} mont_launch_t;

/* mont_launch_t.flags.  MONT_LAUNCH_OVERLAP_PREV (mont_mul_vec_ex / _checksum_ex default flat grid,
 * mont_mul_twiddle_ex variants 0 / 1 / 4, mont_run_ex; ignored elsewhere): the launch may start
 * while the previous kernel on the stream is still running (programmatic dependent launch: its
 * CTAs fill the SMs that kernel's tail leaves idle).  The CALLER guarantees that this operation
 * neither reads what the previous kernel writes nor writes what it reads or writes.  The
 * operation still completes only after the previous kernel has completed, so everything launched
 * after it keeps plain stream order.  Inside a CUDA graph capture it becomes a programmatic edge. */
#define MONT_LAUNCH_OVERLAP_PREV 1

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

/* mb_pipe: per-instruction issue-rate microbenchmark (csrc/k_pipes.cu).  Every thread runs 8
 *   independent dependency chains in which each instruction consumes the previous result as a
 *   register operand (nothing loop-invariant for ptxas to hoist), `iters` loop trips of
 *   mb_pipe_ops_per_iter(kind) = 128 timed instructions.  kind: 0 IMAD R,R,R; 1 IMAD R,R,imm;
 *   2 IMAD R,R,UR (kernel parameter); 3 IMAD.HI R,R,R; 4 IMAD.HI R,R,imm; 5 IMAD.WIDE R,R,R;
 *   6 IMAD.WIDE + IMAD.HI 1:1; 7 IMAD.WIDE + IMAD 1:1; 8 add.u32 (ptxas: half IADD3 on the ALU,
 *   half IMAD.IADD on FMAHeavy); 9 LOP3; 10 SEL; 11 VIMNMX; 12 SHF; 13 FFMA R,R,R;
 *   14 FFMA R,R,imm; 15 DFMA; mixes 1:1 -- 16 IMAD.WIDE + FFMA, 17 IMAD.WIDE + IADD3,
 *   18 IMAD.WIDE + DFMA, 19 IMAD.WIDE + IMAD imm, 20 IMAD + FFMA, 21 IMAD + IADD3,
 *   22 IMAD.WIDE + LOP3, 23 IMAD + IMAD imm, 24 IMAD + DFMA, 25 IMAD.WIDE + DMUL,
 *   26 IMAD.WIDE + DADD; modular products (counted as products, not instructions) --
 *   27 the library's chain REDC (sredc), 28 the FP64 Barrett product (fmulmod), 29 REDC +
 *   fmulmod 1:1, 30 REDC + fmulmod 3:1; 31 DMUL, 32 DADD, 33 IMAD + DMUL; warp-specialised
 *   products, warps 4-7 of each CTA on fmulmod and 0-3 on REDC (one of each per SMSP) -- 34 equal
 *   trip counts; 35, 36, 37: the FP64 warps run 2/3, 1/2, 1/3 of the trips, so their products are
 *   2/5, 1/3, 1/4 of the total (the caller counts threads * (iters + fp_iters) / 2 * 128).
 *   Warp-specialised instruction pairs (by hardware warp slot, %warpid, so both kinds share
 *   every SMSP; equal trips): 38 IMAD.WIDE / DFMA, 39 IMAD.WIDE / DMUL, 40 REDC / DFMA,
 *   41 IMAD.WIDE / fmulmod (counted as instructions; 40 and 41 count one REDC or fmulmod as
 *   one).  42: no work; sink[t] = the %warpid of thread t's warp.  43-48: NI REDC + NF
 *   fmulmod chains per thread interleaved instruction by instruction, (NI, NF) = (1,1), (3,1),
 *   (6,2), (2,0), (0,2), (4,0); mb_pipe_ops_per_iter = 32 (NI + NF) products.  49: IMAD.HI
 *   R,R,R with an RZ addend (mul.hi.u32, as in __umulhi).  kind outside [0, 50) is
 *   MONT_EINVAL_ARG.
 *   grid = SMs * ctas_per_sm (cfg may be NULL: 8), 256 threads; sink holds one word per
 *   thread.  Executed instructions = threads * iters * 128.  If clk (a DEVICE pointer to 2
 *   uint64) is not NULL, CTA 0 stores its elapsed SM cycles (clock64) and nanoseconds
 *   (%globaltimer) there: their ratio is the SM clock the kernel actually ran at. */
mont_status_t mb_pipe(uint32_t *sink, int kind, int iters, const mont_launch_t *cfg, cudaStream_t stream,
                      unsigned long long *threads_launched, unsigned long long *clk);
int mb_pipe_ops_per_iter(int kind);

/* mb_sm_clock: one warp spins `cycles` SM clocks (clock64) and stores out[0] = cycles elapsed,
 * out[1] = nanoseconds elapsed (%globaltimer); out is a DEVICE pointer to 2 uint64.  Their ratio
 * is the SM clock of the moment -- launched right after a kernel on the same stream, the clock
 * that kernel ran at (the power-managed clock changes on a millisecond scale). */
mont_status_t mb_sm_clock(unsigned long long *out, long long cycles, cudaStream_t stream);

/* Number of SMs of the current device (cached per device), or -1. */
int mont_sm_count(void);

#ifdef __cplusplus
}
#endif

#endif /* MONT_EXT_H_ */
