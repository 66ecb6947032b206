/*
 * mont_host.h -- host-buffer entry points of libmont.so (the end-to-end path).
 *
 * Same operations as mont.h, but every array is in HOST memory.  The library
 * streams the arrays through a caller-supplied device workspace in chunks with
 * a 3-stage pipeline: the host->device copy of chunk i+1, the kernel on chunk i
 * and the device->host copy of chunk i-1 run concurrently on three internal
 * streams (two copy engines + the SMs), so a call costs ~max(bytes in, bytes
 * out) / PCIe bandwidth instead of their sum.  Host memory must be page-locked
 * (cudaHostAlloc / torch pin_memory) for the copies to overlap; pageable memory
 * works but serialises.
 *
 * Ordering: the pipeline starts after all work previously enqueued on `stream`
 * and `stream` waits for its completion, so the call is asynchronous like the
 * device-pointer forms: outputs (and *acc_host) are valid once `stream` has
 * synchronised.  Several calls may run concurrently on different streams if
 * each has its own workspace.  The library creates and releases its internal
 * streams/events per call; it allocates no memory.
 *
 * Workspace: `ws` is a device buffer of `ws_bytes`; the chunk size is derived
 * from it (3 slots of in+out buffers).  It must hold at least
 * mont_host_min_workspace(op) bytes.  Errors as in mont.h; MONT_EINVAL_ARG for a
 * too-small or misaligned (16 B) workspace.
 */
#ifndef MONT_HOST_H_
#define MONT_HOST_H_

#include "mont.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum mont_host_op {
    MONT_HOST_MUL_VEC = 0,      /* 2 in, 1 out (+ optional checksum)          */
    MONT_HOST_TO_MONT = 1,      /* 1 in, 1 out                                */
    MONT_HOST_FROM_MONT = 2,    /* 1 in, 1 out                                */
    MONT_HOST_POW_VEC = 3,      /* 2 in, 1 out                                */
    MONT_HOST_TWIDDLE = 4,      /* 1 in, 1 out (+ the table, copied once)     */
    MONT_HOST_NTT = 5           /* rows in, rows out (+ the table, copied once); mont_host_run only */
} mont_host_op_t;

/* Smallest workspace (bytes) accepted for `op`; len = twiddle row length or
 * NTT transform length (ignored otherwise). */
size_t mont_host_min_workspace(mont_host_op_t op, size_t len);

/* c = REDC(a, b) elementwise (mont_mul_vec); if acc_host != NULL also
 * *acc_host = sum_i c[i] (64-bit, overwritten, not accumulated). */
mont_status_t mont_mul_vec_host(const mont_ctx_t *ctx, uint32_t *c_host, const uint32_t *a_host,
                                const uint32_t *b_host, size_t n, unsigned long long *acc_host, void *ws,
                                size_t ws_bytes, cudaStream_t stream);
mont_status_t to_mont_host(const mont_ctx_t *ctx, uint32_t *out_host, const uint32_t *in_host, size_t n,
                           void *ws, size_t ws_bytes, cudaStream_t stream);
mont_status_t from_mont_host(const mont_ctx_t *ctx, uint32_t *out_host, const uint32_t *in_host, size_t n,
                             void *ws, size_t ws_bytes, cudaStream_t stream);
mont_status_t mont_pow_vec_host(const mont_ctx_t *ctx, uint32_t *out_host, const uint32_t *base_host,
                                const uint32_t *exp_host, size_t n, void *ws, size_t ws_bytes,
                                cudaStream_t stream);
/* chunks are whole rows; the len-word table tw_host is copied once */
mont_status_t mont_mul_twiddle_host(const mont_ctx_t *ctx, uint32_t *out_host, const uint32_t *x_host,
                                    const uint32_t *tw_host, size_t batch, size_t len, void *ws,
                                    size_t ws_bytes, cudaStream_t stream);

/* ---- one pipelined run over many jobs (the e2e executor) ----
 *
 * The calls above pipeline one operation each; several of them share the PCIe
 * link only as well as concurrent streams interleave.  mont_host_run streams
 * the chunks of ALL jobs, in job order, through ONE ring of workspace slots:
 * one H2D stream, one compute stream and one D2H stream, so the host->device
 * direction stays busy from the first chunk to the last while results flow
 * back concurrently -- the step costs ~max(total bytes in, total bytes out) /
 * PCIe bandwidth.
 *
 * Fusion: consecutive elementwise jobs (MUL_VEC, TO_MONT, FROM_MONT, POW_VEC)
 * with the same n form one group when each later job reads a host buffer of the
 * group (an input of an earlier job, or an earlier job's output) and writes
 * none of them.  A group streams chunk by chunk: each distinct host input is
 * uploaded once per chunk, a job reading an earlier group job's output takes
 * that device chunk (no trip through host memory), and every job's output is
 * downloaded.  Results are those of running the jobs one after another.
 *
 * Chunk order: groups stream in job order, but up to 3 consecutive groups
 * are interleaved chunk by chunk so that the H2D and D2H byte counts stay
 * balanced (a download-heavy group beside upload-heavy ones keeps both
 * directions of the link busy).  Groups whose host buffers overlap (one writes
 * what the other reads or writes) are never interleaved: job order decides.
 *
 * Dependencies: jobs in different groups are independent unless `depends_on`
 * >= 0: then the job's group starts its input copies only after job
 * `depends_on` (an earlier index) has all its outputs in host memory -- needed
 * when a job reads a host buffer an earlier job of ANOTHER group writes; put
 * independent jobs in between to hide the wait.  Inside a group it is implied.
 * Workspace: 16-byte aligned; it holds the twiddle tables and checksum
 * accumulators of the jobs plus 4 slots of max(3, group inputs + outputs)
 * chunk buffers; the chunk size is derived from what is left (MONT_EINVAL_ARG
 * if that is < one row / 256 words). */
typedef struct mont_host_job {
    int op;                        /* mont_host_op_t                                       */
    const mont_ctx_t *ctx;
    uint32_t *out;                 /* host                                                 */
    const uint32_t *in0;           /* host: a / x / base / the NTT rows                    */
    const uint32_t *in1;           /* host: b / exp / the len-word twiddle table (TWIDDLE) /
                                      the (len - 1)-word mont_ntt_twiddles table (NTT)     */
    size_t n;                      /* elements (TWIDDLE, NTT: rows)                        */
    size_t len;                    /* TWIDDLE: row length; NTT: transform length 2^k,
                                      2 <= 2^k <= 2^15; else ignored                       */
    unsigned long long *acc_host;  /* MUL_VEC: optional sum of out (overwritten)           */
    int depends_on;                /* index of an earlier job whose outputs this reads, or -1 */
    uint32_t scale;                /* NTT: output factor in Montgomery form as in mont_ntt
                                      (0 selects R mod P, i.e. no scaling); else ignored   */
} mont_host_job_t;

mont_status_t mont_host_run(const mont_host_job_t *jobs, int njobs, void *ws, size_t ws_bytes,
                            cudaStream_t stream);

/* Host<->device bytes one mont_host_run(jobs, njobs, ...) copies (after fusion):
 * *h2d_bytes = uploaded inputs + twiddle tables, *d2h_bytes = outputs + 8 per
 * checksum.  Validates like mont_host_run; host only, no CUDA call. */
mont_status_t mont_host_run_bytes(const mont_host_job_t *jobs, int njobs, unsigned long long *h2d_bytes,
                                  unsigned long long *d2h_bytes);

#ifdef __cplusplus
}
#endif

#endif /* MONT_HOST_H_ */
