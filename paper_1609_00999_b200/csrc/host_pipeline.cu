// host_pipeline.cu -- host-buffer entry points (include/mont_host.h): the
// end-to-end path.  A chunked 3-stage pipeline over a caller-supplied device
// workspace: H2D(i+1) on one copy stream, the library kernel on chunk i on a
// compute stream and D2H(i-1) on a second copy stream, with per-slot events
// enforcing buffer reuse.  Host<->device traffic is the bound (PCIe), so the
// goal is simply that both copy directions and the SMs are busy at once.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mont_ext.h"
#include "../../include/mont_host.h"
#include "abi_util.h"

namespace mont {
namespace {

constexpr int kSlots = 3;
constexpr size_t kAlign = 256;

inline size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

struct Streams {
    cudaStream_t h2d = nullptr, krn = nullptr, d2h = nullptr;
    cudaEvent_t start = nullptr, done_k = nullptr, done_d = nullptr;
    cudaEvent_t h2d_done[kSlots] = {}, k_done[kSlots] = {}, d2h_done[kSlots] = {};
    bool ok = true;

    Streams() {
        ok &= cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking) == cudaSuccess;
        ok &= cudaStreamCreateWithFlags(&krn, cudaStreamNonBlocking) == cudaSuccess;
        ok &= cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking) == cudaSuccess;
        ok &= cudaEventCreateWithFlags(&start, cudaEventDisableTiming) == cudaSuccess;
        ok &= cudaEventCreateWithFlags(&done_k, cudaEventDisableTiming) == cudaSuccess;
        ok &= cudaEventCreateWithFlags(&done_d, cudaEventDisableTiming) == cudaSuccess;
        for (int s = 0; s < kSlots; ++s) {
            ok &= cudaEventCreateWithFlags(&h2d_done[s], cudaEventDisableTiming) == cudaSuccess;
            ok &= cudaEventCreateWithFlags(&k_done[s], cudaEventDisableTiming) == cudaSuccess;
            ok &= cudaEventCreateWithFlags(&d2h_done[s], cudaEventDisableTiming) == cudaSuccess;
        }
    }
    // Destroying streams/events with work still queued is legal: the driver
    // releases them when the work completes, so the call stays asynchronous.
    ~Streams() {
        for (int s = 0; s < kSlots; ++s) {
            if (h2d_done[s]) cudaEventDestroy(h2d_done[s]);
            if (k_done[s]) cudaEventDestroy(k_done[s]);
            if (d2h_done[s]) cudaEventDestroy(d2h_done[s]);
        }
        if (start) cudaEventDestroy(start);
        if (done_k) cudaEventDestroy(done_k);
        if (done_d) cudaEventDestroy(done_d);
        if (h2d) cudaStreamDestroy(h2d);
        if (krn) cudaStreamDestroy(krn);
        if (d2h) cudaStreamDestroy(d2h);
    }
};

// Streams `units` units of `unit_words` uint32 each: nin host inputs -> 1 host
// output.  `reserved` bytes at the front of the workspace are left to the
// caller (pre/post hooks).  launch(dev_in[], dev_out, units_in_chunk, first_unit,
// stream) runs the kernel for one chunk.
template <class Pre, class Launch, class Post>
mont_status_t pipeline(int nin, const uint32_t *const *host_in, uint32_t *host_out, size_t units, size_t unit_words,
                       void *ws, size_t ws_bytes, size_t reserved, cudaStream_t user, Pre pre, Launch launch,
                       Post post) {
    if (((uintptr_t)ws & 15u) || ws_bytes < align_up(reserved) + kAlign) return MONT_EINVAL_ARG;
    const size_t nbuf = (size_t)nin + 1;
    const size_t per_unit = unit_words * 4;
    const size_t avail = ws_bytes - align_up(reserved);
    size_t cap = avail / (kSlots * nbuf);  // bytes per buffer
    cap = cap > kAlign ? (cap / kAlign) * kAlign : 0;
    size_t chunk = cap / per_unit;
    if (chunk == 0) return MONT_EINVAL_ARG;
    // at least ~8 chunks so the three stages overlap, but not tiny chunks
    const size_t min_chunk = unit_words >= (1u << 20) ? 1 : ((size_t)1 << 20) / unit_words;
    size_t want = (units + 7) / 8;
    if (want < min_chunk) want = min_chunk;
    if (chunk > want) chunk = want;
    const size_t buf_bytes = align_up(chunk * per_unit);
    char *base = (char *)ws + align_up(reserved);
    auto dev_buf = [&](int slot, int k) { return (uint32_t *)(base + ((size_t)slot * nbuf + k) * buf_bytes); };

    Streams S;
    if (!S.ok) return MONT_ECUDA;
    if (cudaEventRecord(S.start, user) != cudaSuccess) return MONT_ECUDA;
    cudaStreamWaitEvent(S.h2d, S.start, 0);
    cudaStreamWaitEvent(S.krn, S.start, 0);
    cudaStreamWaitEvent(S.d2h, S.start, 0);
    mont_status_t st = pre(S.h2d, S.krn);
    if (st != MONT_OK) return st;
    const size_t nchunks = (units + chunk - 1) / chunk;
    for (size_t i = 0; i < nchunks; ++i) {
        const int slot = (int)(i % kSlots);
        const size_t u0 = i * chunk;
        const size_t nu = units - u0 < chunk ? units - u0 : chunk;
        const size_t off = u0 * unit_words, bytes = nu * per_unit;
        if (i >= (size_t)kSlots) cudaStreamWaitEvent(S.h2d, S.k_done[slot], 0);  // inputs of chunk i-3 consumed
        uint32_t *din[2] = {nullptr, nullptr};
        for (int k = 0; k < nin; ++k) {
            din[k] = dev_buf(slot, k);
            if (cudaMemcpyAsync(din[k], host_in[k] + off, bytes, cudaMemcpyHostToDevice, S.h2d) != cudaSuccess)
                return MONT_ECUDA;
        }
        cudaEventRecord(S.h2d_done[slot], S.h2d);
        cudaStreamWaitEvent(S.krn, S.h2d_done[slot], 0);
        if (i >= (size_t)kSlots) cudaStreamWaitEvent(S.krn, S.d2h_done[slot], 0);  // output of chunk i-3 drained
        uint32_t *dout = dev_buf(slot, nin);
        st = launch(din, dout, nu, u0, S.krn);
        if (st != MONT_OK) return st;
        cudaEventRecord(S.k_done[slot], S.krn);
        cudaStreamWaitEvent(S.d2h, S.k_done[slot], 0);
        if (cudaMemcpyAsync(host_out + off, dout, bytes, cudaMemcpyDeviceToHost, S.d2h) != cudaSuccess)
            return MONT_ECUDA;
        cudaEventRecord(S.d2h_done[slot], S.d2h);
    }
    st = post(S.krn, S.d2h);
    if (st != MONT_OK) return st;
    cudaEventRecord(S.done_k, S.krn);
    cudaEventRecord(S.done_d, S.d2h);
    cudaStreamWaitEvent(user, S.done_k, 0);
    cudaStreamWaitEvent(user, S.done_d, 0);
    return launch_status();
}

inline mont_status_t no_hook(cudaStream_t, cudaStream_t) { return MONT_OK; }

size_t min_ws(int nin, size_t unit_words, size_t reserved) {
    return align_up(reserved) + (size_t)kSlots * (nin + 1) * align_up(unit_words * 4 * 1024) + kAlign;
}

}  // namespace
}  // namespace mont

using namespace mont;

extern "C" size_t mont_host_min_workspace(mont_host_op_t op, size_t len) {
    switch (op) {
        case MONT_HOST_MUL_VEC: return min_ws(2, 1, 8);
        case MONT_HOST_POW_VEC: return min_ws(2, 1, 0);
        case MONT_HOST_TO_MONT:
        case MONT_HOST_FROM_MONT: return min_ws(1, 1, 0);
        case MONT_HOST_TWIDDLE: return align_up(len * 4) + (size_t)kSlots * 2 * align_up(len * 4) + kAlign;
    }
    return 0;
}

extern "C" mont_status_t mont_mul_vec_host(const mont_ctx_t *ctx, uint32_t *c_host, const uint32_t *a_host,
                                           const uint32_t *b_host, size_t n, unsigned long long *acc_host, void *ws,
                                           size_t ws_bytes, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (n == 0) {
        if (acc_host) *acc_host = 0;
        return MONT_OK;
    }
    if (!c_host || !a_host || !b_host || !ws) return MONT_EINVAL_ARG;
    const uint32_t *in[2] = {a_host, b_host};
    unsigned long long *dacc = (unsigned long long *)ws;  // reserved 8 bytes
    auto pre = [&](cudaStream_t, cudaStream_t k) -> mont_status_t {
        if (acc_host && cudaMemsetAsync(dacc, 0, 8, k) != cudaSuccess) return MONT_ECUDA;
        return MONT_OK;
    };
    auto launch = [&](uint32_t **din, uint32_t *dout, size_t nu, size_t, cudaStream_t s) {
        return acc_host ? mont_mul_vec_checksum(ctx, dout, din[0], din[1], nu, dacc, s)
                        : mont_mul_vec(ctx, dout, din[0], din[1], nu, s);
    };
    auto post = [&](cudaStream_t k, cudaStream_t) -> mont_status_t {
        if (acc_host && cudaMemcpyAsync(acc_host, dacc, 8, cudaMemcpyDeviceToHost, k) != cudaSuccess)
            return MONT_ECUDA;
        return MONT_OK;
    };
    return pipeline(2, in, c_host, n, 1, ws, ws_bytes, 8, stream, pre, launch, post);
}

extern "C" mont_status_t to_mont_host(const mont_ctx_t *ctx, uint32_t *out_host, const uint32_t *in_host, size_t n,
                                      void *ws, size_t ws_bytes, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (n == 0) return MONT_OK;
    if (!out_host || !in_host || !ws) return MONT_EINVAL_ARG;
    const uint32_t *in[1] = {in_host};
    auto launch = [&](uint32_t **din, uint32_t *dout, size_t nu, size_t, cudaStream_t s) {
        return to_mont(ctx, dout, din[0], nu, s);
    };
    return pipeline(1, in, out_host, n, 1, ws, ws_bytes, 0, stream, no_hook, launch, no_hook);
}

extern "C" mont_status_t from_mont_host(const mont_ctx_t *ctx, uint32_t *out_host, const uint32_t *in_host, size_t n,
                                        void *ws, size_t ws_bytes, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (n == 0) return MONT_OK;
    if (!out_host || !in_host || !ws) return MONT_EINVAL_ARG;
    const uint32_t *in[1] = {in_host};
    auto launch = [&](uint32_t **din, uint32_t *dout, size_t nu, size_t, cudaStream_t s) {
        return from_mont(ctx, dout, din[0], nu, s);
    };
    return pipeline(1, in, out_host, n, 1, ws, ws_bytes, 0, stream, no_hook, launch, no_hook);
}

extern "C" mont_status_t mont_pow_vec_host(const mont_ctx_t *ctx, uint32_t *out_host, const uint32_t *base_host,
                                           const uint32_t *exp_host, size_t n, void *ws, size_t ws_bytes,
                                           cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (n == 0) return MONT_OK;
    if (!out_host || !base_host || !exp_host || !ws) return MONT_EINVAL_ARG;
    const uint32_t *in[2] = {base_host, exp_host};
    auto launch = [&](uint32_t **din, uint32_t *dout, size_t nu, size_t, cudaStream_t s) {
        return mont_pow_vec(ctx, dout, din[0], din[1], nu, s);
    };
    return pipeline(2, in, out_host, n, 1, ws, ws_bytes, 0, stream, no_hook, launch, no_hook);
}

extern "C" mont_status_t mont_mul_twiddle_host(const mont_ctx_t *ctx, uint32_t *out_host, const uint32_t *x_host,
                                               const uint32_t *tw_host, size_t batch, size_t len, void *ws,
                                               size_t ws_bytes, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (batch == 0) return MONT_OK;
    if (len == 0 || !out_host || !x_host || !tw_host || !ws) return MONT_EINVAL_ARG;
    uint32_t *dtw = (uint32_t *)ws;  // reserved: the table
    const uint32_t *in[1] = {x_host};
    auto pre = [&](cudaStream_t h, cudaStream_t) -> mont_status_t {
        return cudaMemcpyAsync(dtw, tw_host, len * 4, cudaMemcpyHostToDevice, h) == cudaSuccess ? MONT_OK
                                                                                              : MONT_ECUDA;
    };
    auto launch = [&](uint32_t **din, uint32_t *dout, size_t rows, size_t, cudaStream_t s) {
        return mont_mul_twiddle(ctx, dout, din[0], dtw, rows, len, s);
    };
    return pipeline(1, in, out_host, batch, len, ws, ws_bytes, len * 4, stream, pre, launch, no_hook);
}

// ------------------------------------------------------------ mont_host_run
namespace mont {
namespace {

constexpr int kRing = 4;

struct JobPlan {
    int nin;            // streamed inputs (1 or 2)
    size_t units;       // chunkable units
    size_t unit_words;  // words per unit
    size_t chunk;       // units per chunk
    uint32_t *dtab;     // device twiddle table (TWIDDLE)
    unsigned long long *dacc;  // device accumulator (MUL_VEC with acc_host)
};

struct Ring {
    cudaStream_t h2d = nullptr, krn = nullptr, d2h = nullptr;
    cudaEvent_t start = nullptr, done_k = nullptr, done_d = nullptr;
    cudaEvent_t job_out[64] = {};
    cudaEvent_t h2d_done[kRing] = {}, k_done[kRing] = {}, d2h_done[kRing] = {};
    bool ok = true;
    Ring() {
        ok &= cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking) == cudaSuccess;
        ok &= cudaStreamCreateWithFlags(&krn, cudaStreamNonBlocking) == cudaSuccess;
        ok &= cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking) == cudaSuccess;
        cudaEvent_t *evs[] = {&start, &done_k, &done_d};
        for (cudaEvent_t *e : evs) ok &= cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
        for (int s = 0; s < kRing; ++s) {
            ok &= cudaEventCreateWithFlags(&h2d_done[s], cudaEventDisableTiming) == cudaSuccess;
            ok &= cudaEventCreateWithFlags(&k_done[s], cudaEventDisableTiming) == cudaSuccess;
            ok &= cudaEventCreateWithFlags(&d2h_done[s], cudaEventDisableTiming) == cudaSuccess;
        }
    }
    ~Ring() {
        for (int s = 0; s < kRing; ++s) {
            if (h2d_done[s]) cudaEventDestroy(h2d_done[s]);
            if (k_done[s]) cudaEventDestroy(k_done[s]);
            if (d2h_done[s]) cudaEventDestroy(d2h_done[s]);
        }
        cudaEvent_t evs[] = {start, done_k, done_d};
        for (cudaEvent_t e : evs)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : job_out)
            if (e) cudaEventDestroy(e);
        if (h2d) cudaStreamDestroy(h2d);
        if (krn) cudaStreamDestroy(krn);
        if (d2h) cudaStreamDestroy(d2h);
    }
};

}  // namespace
}  // namespace mont

extern "C" mont_status_t mont_host_run(const mont_host_job_t *jobs, int njobs, void *ws, size_t ws_bytes,
                                       cudaStream_t stream) {
    if (njobs < 0 || (njobs > 0 && !jobs) || (njobs > 0 && (!ws || ((uintptr_t)ws & 15u)))) return MONT_EINVAL_ARG;
    if (njobs == 0) return MONT_OK;
    // plan: reserved area (tables, accumulators), then the ring
    JobPlan plan[64];
    if (njobs > 64) return MONT_EUNSUPPORTED;
    size_t reserved = 0;
    for (int j = 0; j < njobs; ++j) {
        const mont_host_job_t &J = jobs[j];
        if (!ctx_ok(J.ctx)) return J.ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
        JobPlan &P = plan[j];
        P.dtab = nullptr;
        P.dacc = nullptr;
        switch (J.op) {
            case MONT_HOST_MUL_VEC: P.nin = 2; P.unit_words = 1; P.units = J.n; break;
            case MONT_HOST_POW_VEC: P.nin = 2; P.unit_words = 1; P.units = J.n; break;
            case MONT_HOST_TO_MONT:
            case MONT_HOST_FROM_MONT: P.nin = 1; P.unit_words = 1; P.units = J.n; break;
            case MONT_HOST_TWIDDLE:
                if (J.len == 0 && J.n) return MONT_EINVAL_ARG;
                P.nin = 1; P.unit_words = J.len; P.units = J.n;
                P.dtab = (uint32_t *)((char *)ws + reserved);
                reserved += align_up(J.len * 4);
                break;
            default: return MONT_EINVAL_ARG;
        }
        if (J.n && (!J.out || !J.in0 || (P.nin == 2 && !J.in1) || (J.op == MONT_HOST_TWIDDLE && !J.in1)))
            return MONT_EINVAL_ARG;
        if (J.depends_on >= j || J.depends_on < -1) return MONT_EINVAL_ARG;
        if (J.op == MONT_HOST_MUL_VEC && J.acc_host) {
            P.dacc = (unsigned long long *)((char *)ws + reserved);
            reserved += kAlign;
        }
    }
    if (ws_bytes < reserved + kRing * 3 * kAlign) return MONT_EINVAL_ARG;
    const size_t buf_bytes = ((ws_bytes - reserved) / (kRing * 3)) / kAlign * kAlign;
    char *ring = (char *)ws + reserved;
    auto slot_buf = [&](int slot, int k) { return (uint32_t *)(ring + ((size_t)slot * 3 + k) * buf_bytes); };
    for (int j = 0; j < njobs; ++j) {
        plan[j].chunk = buf_bytes / (plan[j].unit_words * 4);
        if (plan[j].chunk == 0 && jobs[j].n) return MONT_EINVAL_ARG;
    }

    Ring R;
    if (!R.ok) return MONT_ECUDA;
    for (int j = 0; j < njobs; ++j) {  // completion events only for jobs someone depends on
        const int d = jobs[j].depends_on;
        if (d >= 0 && !R.job_out[d] && cudaEventCreateWithFlags(&R.job_out[d], cudaEventDisableTiming) != cudaSuccess)
            return MONT_ECUDA;
    }
    if (cudaEventRecord(R.start, stream) != cudaSuccess) return MONT_ECUDA;
    cudaStreamWaitEvent(R.h2d, R.start, 0);
    cudaStreamWaitEvent(R.krn, R.start, 0);
    cudaStreamWaitEvent(R.d2h, R.start, 0);
    // prologue: tables in, accumulators zeroed
    for (int j = 0; j < njobs; ++j) {
        if (plan[j].dtab &&
            cudaMemcpyAsync(plan[j].dtab, jobs[j].in1, jobs[j].len * 4, cudaMemcpyHostToDevice, R.h2d) != cudaSuccess)
            return MONT_ECUDA;
        if (plan[j].dacc && cudaMemsetAsync(plan[j].dacc, 0, 8, R.krn) != cudaSuccess) return MONT_ECUDA;
    }
    size_t g = 0;  // global chunk counter -> ring slot
    for (int j = 0; j < njobs; ++j) {
        const mont_host_job_t &J = jobs[j];
        const JobPlan &P = plan[j];
        if (J.depends_on >= 0) cudaStreamWaitEvent(R.h2d, R.job_out[J.depends_on], 0);
        for (size_t u0 = 0; u0 < P.units; u0 += P.chunk, ++g) {
            const int slot = (int)(g % kRing);
            const size_t nu = P.units - u0 < P.chunk ? P.units - u0 : P.chunk;
            const size_t off = u0 * P.unit_words, bytes = nu * P.unit_words * 4;
            if (g >= (size_t)kRing) cudaStreamWaitEvent(R.h2d, R.k_done[slot], 0);
            uint32_t *d0 = slot_buf(slot, 0), *d1 = slot_buf(slot, 1), *dout = slot_buf(slot, 2);
            if (cudaMemcpyAsync(d0, J.in0 + off, bytes, cudaMemcpyHostToDevice, R.h2d) != cudaSuccess)
                return MONT_ECUDA;
            if (P.nin == 2 &&
                cudaMemcpyAsync(d1, J.in1 + off, bytes, cudaMemcpyHostToDevice, R.h2d) != cudaSuccess)
                return MONT_ECUDA;
            cudaEventRecord(R.h2d_done[slot], R.h2d);
            cudaStreamWaitEvent(R.krn, R.h2d_done[slot], 0);
            if (g >= (size_t)kRing) cudaStreamWaitEvent(R.krn, R.d2h_done[slot], 0);
            mont_status_t st;
            switch (J.op) {
                case MONT_HOST_MUL_VEC:
                    st = P.dacc ? mont_mul_vec_checksum(J.ctx, dout, d0, d1, nu, P.dacc, R.krn)
                                : mont_mul_vec(J.ctx, dout, d0, d1, nu, R.krn);
                    break;
                case MONT_HOST_POW_VEC: st = mont_pow_vec(J.ctx, dout, d0, d1, nu, R.krn); break;
                case MONT_HOST_TO_MONT: st = to_mont(J.ctx, dout, d0, nu, R.krn); break;
                case MONT_HOST_FROM_MONT: st = from_mont(J.ctx, dout, d0, nu, R.krn); break;
                default: st = mont_mul_twiddle(J.ctx, dout, d0, P.dtab, nu, J.len, R.krn); break;
            }
            if (st != MONT_OK) return st;
            cudaEventRecord(R.k_done[slot], R.krn);
            cudaStreamWaitEvent(R.d2h, R.k_done[slot], 0);
            if (cudaMemcpyAsync(J.out + off, dout, bytes, cudaMemcpyDeviceToHost, R.d2h) != cudaSuccess)
                return MONT_ECUDA;
            cudaEventRecord(R.d2h_done[slot], R.d2h);
        }
        if (P.dacc) {
            cudaStreamWaitEvent(R.d2h, R.k_done[(g + kRing - 1) % kRing], 0);
            if (cudaMemcpyAsync(J.acc_host, P.dacc, 8, cudaMemcpyDeviceToHost, R.d2h) != cudaSuccess)
                return MONT_ECUDA;
        }
        if (R.job_out[j]) cudaEventRecord(R.job_out[j], R.d2h);  // this job's outputs are in host memory
    }
    cudaEventRecord(R.done_k, R.krn);
    cudaEventRecord(R.done_d, R.d2h);
    cudaStreamWaitEvent(stream, R.done_k, 0);
    cudaStreamWaitEvent(stream, R.done_d, 0);
    return launch_status();
}
