/*
 * mont_run.h -- several HBM-bound operations of mont.h in ONE launch (device buffers).
 *
 * A step of the path issues several independent streaming operations (BASELINE configs[1]'s
 * three mul_vec, the to_mont / from_mont pair, configs[2]'s twiddle multiply).  Issued one by
 * one, every launch pays its own ramp (CTAs reaching the SMs) and tail (the last partial wave)
 * with the memory system idle in between.  mont_run runs a list of such jobs as one flat grid:
 * the tiles of all jobs back to back, each CTA one 512-thread x 2 x 16 B tile of one job, so the
 * memory stream never drains between jobs.  A from_mont job whose input is exactly the output of
 * an earlier to_mont job (same n, same modulus) is fused into it: from_mont(x-bar) is computed
 * from the register that to_mont just produced (the conversions bracket a chain),
 * so x-bar is written once and never read back -- 12 instead of 16 bytes of HBM traffic per
 * element of the pair.  Results are bit-identical to the individual calls (same REDC code,
 * mont_core.cuh).  Same conventions as mont.h.
 */
#ifndef MONT_RUN_H_
#define MONT_RUN_H_

#include "mont.h"

#ifdef __cplusplus
extern "C" {
#endif

#define MONT_RUN_MAX_JOBS 16

typedef enum mont_run_op {
    MONT_RUN_MUL = 0,      /* out[i] = REDC(in0[i], in1[i])   (mont_mul_vec), optional checksum */
    MONT_RUN_TO = 1,       /* out[i] = in0[i] R mod P         (to_mont)                         */
    MONT_RUN_FROM = 2,     /* out[i] = in0[i] R^-1 mod P      (from_mont)                       */
    MONT_RUN_TWIDDLE = 3   /* out[r len + j] = REDC(in0[r len + j], in1[j])  (mont_mul_twiddle) */
} mont_run_op_t;

/* One job.  All pointers are DEVICE pointers, 16-byte aligned; n is a multiple of 4.
 *   op   : mont_run_op_t
 *   ctx  : HOST pointer to an initialised context (copied at the call)
 *   out  : n words written
 *   in0  : n words read (may equal out: in place)
 *   in1  : MUL: n words; TWIDDLE: the len-word table; else ignored
 *   n    : elements (TWIDDLE: batch * len)
 *   len  : TWIDDLE row length, a power of two >= 4 dividing n; else ignored
 *   acc  : MUL only, optional (NULL = none): *acc += sum_i out[i], 64-bit, 8-byte aligned,
 *          as mont_mul_vec_checksum (the caller zeroes it)                                  */
typedef struct mont_run_job {
    int op;
    const mont_ctx_t *ctx;
    uint32_t *out;
    const uint32_t *in0;
    const uint32_t *in1;
    size_t n;
    size_t len;
    unsigned long long *acc;
} mont_run_job_t;

/* Runs jobs[0 .. njobs) as one launch on `stream` (asynchronous; returns after enqueueing).
 * The jobs must be independent: no job may read or write a range another job writes, except
 * that a FROM job whose in0 is exactly the out of an earlier TO job with the same n and the
 * same modulus consumes that job's result (fused, see above).  Jobs with n == 0 are skipped.
 * Errors: MONT_EINVAL_ARG for njobs outside [0, MONT_RUN_MAX_JOBS], a NULL or misaligned
 * pointer, n % 4 != 0, a bad op / len, or a dependency other than the fused pair;
 * MONT_EINVAL_P for a context that was not initialised; MONT_ECUDA for a failed launch. */
mont_status_t mont_run(const mont_run_job_t *jobs, int njobs, cudaStream_t stream);

/* mont_run with an explicit tile shape (measurement): cfg->threads 256 or 512 (0 = 512),
 * cfg->unroll 1, 2 or 4 uint4 per thread per tile (0 = 2); other fields ignored; cfg may be
 * NULL.  MONT_EINVAL_ARG for another shape. */
struct mont_launch;
mont_status_t mont_run_ex(const mont_run_job_t *jobs, int njobs, const struct mont_launch *cfg,
                          cudaStream_t stream);

/* Bytes of HBM traffic the run moves by plan (after fusion): the algorithmic bytes of the
 * launch (reads + writes of every job, a fused pair counted once), for the roofline. */
mont_status_t mont_run_bytes(const mont_run_job_t *jobs, int njobs, unsigned long long *bytes);

#ifdef __cplusplus
}
#endif

#endif /* MONT_RUN_H_ */
