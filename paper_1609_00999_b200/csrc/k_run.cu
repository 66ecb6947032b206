// k_run.cu -- mont_run (include/mont_run.h): a list of HBM-bound jobs of the path (mul_vec with
// an optional fused checksum, to_mont, from_mont, twiddle multiply) as ONE flat grid.
//
// Tile space: job j owns tiles [tile0_j, tile0_j + ntiles_j); CTA b finds its job by a scan of
// the (<= 16) tile offsets in the kernel parameters and processes one tile of 256 threads x 2
// uint4 -- the launch shape of mont_mul_vec_checksum inside bench.py's step.
// Because the block scheduler hands out the tiles of job j+1 while job j's last tiles are still
// streaming, the memory pipeline never drains between jobs (one ramp and one tail per run instead
// of one per operation).  A to_mont job whose output feeds a later from_mont job (same n, same
// modulus) is fused with it: from_mont is applied to the register to_mont just produced and both
// outputs are stored, so x-bar is never read back.  Arithmetic: the REDC forms of mont_core.cuh,
// identical to the single-operation kernels (bit-identical results, tests/test_gpu_run.py).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mont_ext.h"
#include "../../include/mont_run.h"
#include "abi_util.h"

namespace mont {

// tile = THREADS x U uint4 per operand; the default (512 x 2, as mont_mul_vec_checksum's) and
// the alternatives are measured in profiles/r02_probe_run.jsonl
constexpr int kRunThreadsMax = 512;

struct RunJob {
    uint32_t op, fused;      // fused: TO job whose from_mont consumer writes out2
    uint32_t p, pinv, r2;    // context (pinv = P^-1 mod 2^32)
    uint32_t tmask4;         // TWIDDLE: len / 4 - 1 (row length in uint4, a power of two)
    uint32_t *out, *out2;
    const uint32_t *in0, *in1;
    unsigned long long *acc;
    size_t n4;               // uint4 chunks
    size_t tile0;            // first tile of this job
};

struct RunParams {
    int njobs;
    RunJob job[MONT_RUN_MAX_JOBS];
};

__device__ __forceinline__ unsigned long long run_warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

template <int kRunThreads, int kRunU>
__global__ void __launch_bounds__(kRunThreads) k_run(const __grid_constant__ RunParams P) {
    pdl_trigger();
    constexpr size_t kRunTile = (size_t)kRunU * kRunThreads;  // uint4 per tile
    const size_t t = blockIdx.x;
    int j = 0;
#pragma unroll 1
    for (int k = 1; k < P.njobs; ++k)
        if (P.job[k].tile0 <= t) j = k;
    const RunJob &J = P.job[j];
    const size_t base = (t - J.tile0) * kRunTile + threadIdx.x;
    const uint4 *a4 = reinterpret_cast<const uint4 *>(J.in0);
    uint4 *o4 = reinterpret_cast<uint4 *>(J.out);
    if (J.op == MONT_RUN_MUL) {
        const uint4 *b4 = reinterpret_cast<const uint4 *>(J.in1);
        uint4 va[kRunU], vb[kRunU];
        unsigned long long s = 0;
#pragma unroll
        for (int k = 0; k < kRunU; ++k) {
            const size_t i = base + (size_t)k * kRunThreads;
            if (i < J.n4) va[k] = ld_stream(a4 + i);
        }
#pragma unroll
        for (int k = 0; k < kRunU; ++k) {
            const size_t i = base + (size_t)k * kRunThreads;
            if (i < J.n4) vb[k] = ld_stream(b4 + i);
        }
#pragma unroll
        for (int k = 0; k < kRunU; ++k) {
            const size_t i = base + (size_t)k * kRunThreads;
            if (i < J.n4) {
                const uint4 r = make_uint4(redc(va[k].x, vb[k].x, J.p, J.pinv), redc(va[k].y, vb[k].y, J.p, J.pinv),
                                           redc(va[k].z, vb[k].z, J.p, J.pinv), redc(va[k].w, vb[k].w, J.p, J.pinv));
                st_stream(o4 + i, r);
                s += (unsigned long long)r.x + r.y + (unsigned long long)r.z + r.w;
            }
        }
        if (J.acc) {  // block-uniform branch: the CTA's sum, one 64-bit atomic
            __shared__ unsigned long long part[kRunThreadsMax / 32];
            s = run_warp_sum(s);
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
            if (lane == 0) part[wid] = s;
            __syncthreads();
            if (wid == 0) {
                s = lane < kRunThreads / 32 ? part[lane] : 0ull;
                s = run_warp_sum(s);
                if (lane == 0 && s) atomicAdd(J.acc, s);
            }
        }
    } else if (J.op == MONT_RUN_TWIDDLE) {
        const uint4 *w4 = reinterpret_cast<const uint4 *>(J.in1);
        uint4 va[kRunU];
#pragma unroll
        for (int k = 0; k < kRunU; ++k) {
            const size_t i = base + (size_t)k * kRunThreads;
            if (i < J.n4) va[k] = ld_stream(a4 + i);
        }
#pragma unroll
        for (int k = 0; k < kRunU; ++k) {
            const size_t i = base + (size_t)k * kRunThreads;
            if (i < J.n4) {
                const uint4 w = __ldg(w4 + (i & J.tmask4));  // the table stays L1-resident
                st_stream(o4 + i, make_uint4(redc(va[k].x, w.x, J.p, J.pinv), redc(va[k].y, w.y, J.p, J.pinv),
                                             redc(va[k].z, w.z, J.p, J.pinv), redc(va[k].w, w.w, J.p, J.pinv)));
            }
        }
    } else {  // TO (possibly fused with its FROM consumer) or FROM
        uint4 va[kRunU];
#pragma unroll
        for (int k = 0; k < kRunU; ++k) {
            const size_t i = base + (size_t)k * kRunThreads;
            if (i < J.n4) va[k] = ld_stream(a4 + i);
        }
        uint4 *o24 = reinterpret_cast<uint4 *>(J.out2);
#pragma unroll
        for (int k = 0; k < kRunU; ++k) {
            const size_t i = base + (size_t)k * kRunThreads;
            if (i < J.n4) {
                if (J.op == MONT_RUN_TO) {
                    const uint4 r = make_uint4(redc(va[k].x, J.r2, J.p, J.pinv), redc(va[k].y, J.r2, J.p, J.pinv),
                                               redc(va[k].z, J.r2, J.p, J.pinv), redc(va[k].w, J.r2, J.p, J.pinv));
                    st_stream(o4 + i, r);
                    if (J.fused)
                        st_stream(o24 + i, make_uint4(redc1(r.x, J.p, J.pinv), redc1(r.y, J.p, J.pinv),
                                                      redc1(r.z, J.p, J.pinv), redc1(r.w, J.p, J.pinv)));
                } else {
                    st_stream(o4 + i, make_uint4(redc1(va[k].x, J.p, J.pinv), redc1(va[k].y, J.p, J.pinv),
                                                 redc1(va[k].z, J.p, J.pinv), redc1(va[k].w, J.p, J.pinv)));
                }
            }
        }
    }
    pdl_wait();
}

struct Range {
    uintptr_t lo, hi;
};
static bool overlap(const Range &a, const Range &b) { return a.lo < b.hi && b.lo < a.hi; }

// validates the jobs and builds the plan; returns the total tile count through *tiles
static mont_status_t run_plan(const mont_run_job_t *jobs, int njobs, RunParams &P, size_t *tiles,
                              unsigned long long *bytes, size_t kRunTile) {
    if (njobs < 0 || njobs > MONT_RUN_MAX_JOBS || (njobs > 0 && !jobs)) return MONT_EINVAL_ARG;
    int fused_into[MONT_RUN_MAX_JOBS];
    for (int i = 0; i < njobs; ++i) fused_into[i] = -1;
    Range wr[MONT_RUN_MAX_JOBS], rd0[MONT_RUN_MAX_JOBS], rd1[MONT_RUN_MAX_JOBS];
    for (int i = 0; i < njobs; ++i) {
        const mont_run_job_t &J = jobs[i];
        if (!J.ctx) return MONT_EINVAL_ARG;
        if (!ctx_ok(J.ctx)) return MONT_EINVAL_P;
        if (J.op < MONT_RUN_MUL || J.op > MONT_RUN_TWIDDLE || (J.n & 3u)) return MONT_EINVAL_ARG;
        if (J.n == 0) {
            wr[i] = rd0[i] = rd1[i] = Range{0, 0};
            continue;
        }
        if (!J.out || !J.in0 || (((uintptr_t)J.out | (uintptr_t)J.in0) & 15u)) return MONT_EINVAL_ARG;
        const bool has_in1 = J.op == MONT_RUN_MUL || J.op == MONT_RUN_TWIDDLE;
        if (has_in1 && (!J.in1 || ((uintptr_t)J.in1 & 15u))) return MONT_EINVAL_ARG;
        if (J.op == MONT_RUN_TWIDDLE &&
            (J.len < 4 || (J.len & (J.len - 1)) || J.n % J.len || J.len / 4 - 1 > 0xffffffffull))
            return MONT_EINVAL_ARG;
        if (J.acc && (J.op != MONT_RUN_MUL || ((uintptr_t)J.acc & 7u))) return MONT_EINVAL_ARG;
        const size_t nb = J.n * 4;
        wr[i] = Range{(uintptr_t)J.out, (uintptr_t)J.out + nb};
        rd0[i] = Range{(uintptr_t)J.in0, (uintptr_t)J.in0 + nb};
        const size_t n1 = J.op == MONT_RUN_MUL ? nb : J.op == MONT_RUN_TWIDDLE ? J.len * 4 : 0;
        rd1[i] = Range{(uintptr_t)J.in1, (uintptr_t)J.in1 + n1};
    }
    // the one allowed dependency: FROM reading exactly an earlier TO's output (same n, same P)
    for (int j = 0; j < njobs; ++j) {
        const mont_run_job_t &J = jobs[j];
        if (J.n == 0 || J.op != MONT_RUN_FROM) continue;
        for (int i = 0; i < j; ++i) {
            const mont_run_job_t &I = jobs[i];
            if (I.n == J.n && I.op == MONT_RUN_TO && I.out == J.in0 && I.ctx->p == J.ctx->p && fused_into[i] < 0) {
                fused_into[i] = j;
                break;
            }
        }
    }
    auto consumer = [&](int j) {
        for (int i = 0; i < njobs; ++i)
            if (fused_into[i] == j) return i;
        return -1;
    };
    for (int i = 0; i < njobs; ++i) {
        for (int j = 0; j < njobs; ++j) {
            if (i == j || jobs[i].n == 0 || jobs[j].n == 0) continue;
            // j reads what i writes: only the fused pair (i = TO producer, j = its FROM)
            if ((overlap(wr[i], rd0[j]) || overlap(wr[i], rd1[j])) && !(consumer(j) == i && rd0[j].lo == wr[i].lo))
                return MONT_EINVAL_ARG;
            if (i < j && overlap(wr[i], wr[j])) return MONT_EINVAL_ARG;
        }
        // within a job, out may alias in0 / in1 exactly (in place) but not partially
        if (jobs[i].n && ((overlap(wr[i], rd0[i]) && wr[i].lo != rd0[i].lo) ||
                          (overlap(wr[i], rd1[i]) && !(wr[i].lo == rd1[i].lo && wr[i].hi == rd1[i].hi))))
            return MONT_EINVAL_ARG;
    }
    size_t t = 0;
    unsigned long long by = 0;
    int k = 0;
    for (int i = 0; i < njobs; ++i) {
        const mont_run_job_t &J = jobs[i];
        if (J.n == 0 || consumer(i) >= 0) continue;  // empty, or computed by its TO producer
        RunJob &R = P.job[k++];
        const uint32_t pinv = 0u - J.ctx->pneg;
        R.op = (uint32_t)J.op;
        R.fused = fused_into[i] >= 0 ? 1u : 0u;
        R.p = J.ctx->p;
        R.pinv = pinv;
        R.r2 = J.ctx->r2;
        R.tmask4 = J.op == MONT_RUN_TWIDDLE ? (uint32_t)(J.len / 4 - 1) : 0u;
        R.out = J.out;
        R.out2 = fused_into[i] >= 0 ? jobs[fused_into[i]].out : nullptr;
        R.in0 = J.in0;
        R.in1 = J.in1;
        R.acc = J.acc;
        R.n4 = J.n / 4;
        R.tile0 = t;
        t += (R.n4 + kRunTile - 1) / kRunTile;
        const unsigned long long nb = 4ull * J.n;
        by += J.op == MONT_RUN_MUL ? 3 * nb : J.op == MONT_RUN_TWIDDLE ? 2 * nb + 4ull * J.len : 2 * nb;
        if (R.fused) by += nb;  // the second output
    }
    P.njobs = k;
    *tiles = t;
    if (bytes) *bytes = by;
    return MONT_OK;
}

}  // namespace mont

using namespace mont;

extern "C" mont_status_t mont_run_ex(const mont_run_job_t *jobs, int njobs, const mont_launch_t *cfg,
                                     cudaStream_t stream) {
    const int threads = cfg && cfg->threads ? cfg->threads : 512;
    const int unroll = cfg && cfg->unroll ? cfg->unroll : 2;
    if (!((threads == 256 || threads == 512) && (unroll == 1 || unroll == 2 || unroll == 4))) return MONT_EINVAL_ARG;
    RunParams P{};
    size_t tiles = 0;
    const mont_status_t st = run_plan(jobs, njobs, P, &tiles, nullptr, (size_t)threads * unroll);
    if (st != MONT_OK) return st;
    if (tiles == 0) return MONT_OK;
    if (tiles > 0x7fffffffu) return MONT_EUNSUPPORTED;
    const dim3 g((unsigned)tiles), b((unsigned)threads);
    const int flags = cfg ? cfg->flags : 0;
    if (threads == 512) {
        if (unroll == 1) return launch_k(k_run<512, 1>, g, b, 0, stream, flags, P);
        if (unroll == 2) return launch_k(k_run<512, 2>, g, b, 0, stream, flags, P);
        return launch_k(k_run<512, 4>, g, b, 0, stream, flags, P);
    }
    if (unroll == 1) return launch_k(k_run<256, 1>, g, b, 0, stream, flags, P);
    if (unroll == 2) return launch_k(k_run<256, 2>, g, b, 0, stream, flags, P);
    return launch_k(k_run<256, 4>, g, b, 0, stream, flags, P);
}

extern "C" mont_status_t mont_run(const mont_run_job_t *jobs, int njobs, cudaStream_t stream) {
    return mont_run_ex(jobs, njobs, nullptr, stream);
}

extern "C" mont_status_t mont_run_bytes(const mont_run_job_t *jobs, int njobs, unsigned long long *bytes) {
    if (!bytes) return MONT_EINVAL_ARG;
    RunParams P{};
    size_t tiles = 0;
    return run_plan(jobs, njobs, P, &tiles, bytes, 1024);
}
