// host_pipeline.cu -- host-buffer entry points (include/mont_host.h): the
// end-to-end path.  A chunked 3-stage pipeline over a caller-supplied device
// workspace: H2D(i+1) on one copy stream, the library kernel on chunk i on a
// compute stream and D2H(i-1) on a second copy stream, with per-slot events
// enforcing buffer reuse.  Host<->device traffic is the bound (PCIe), so the
// goal is simply that both copy directions and the SMs are busy at once.
// mont_host_run runs many jobs through one such ring: jobs sharing host buffers
// form fusion groups (a shared input goes up once, a chained result is read on
// the device), and consecutive groups are interleaved chunk by chunk to keep
// both link directions loaded (see include/mont_host.h).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mont_ext.h"
#include "../../include/mont_host.h"
#include "../../include/mont_ntt.h"
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
        case MONT_HOST_NTT:  // mont_host_run: the table + 4 ring slots of 3 one-row buffers
            return len < 2 ? 0 : align_up((len - 1) * 4) + (size_t)4 * 3 * align_up(len * 4) + kAlign;
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

namespace mont {
namespace {

// A fusion group: consecutive elementwise jobs over the same n that share host
// buffers.  Each distinct host input is uploaded once per chunk; a job whose
// input is an earlier group job's output reads that job's device chunk (no
// round trip through host memory); every job's output is downloaded.
constexpr int kMaxBufs = 16;
struct Group {
    int j0 = 0, j1 = 0;                    // jobs [j0, j1)
    int nbuf_in = 0;                       // distinct uploaded inputs: buffers [0, nbuf_in)
    const uint32_t *in_host[kMaxBufs];     // their host pointers
    int src[64][2];                        // per job input k: buffer index
    int dst[64];                           // per job: output buffer index
    int nbuf = 0;                          // inputs + outputs
};

bool elementwise(int op) { return op == MONT_HOST_MUL_VEC || op == MONT_HOST_TO_MONT || op == MONT_HOST_FROM_MONT ||
                                  op == MONT_HOST_POW_VEC; }

}  // namespace
}  // namespace mont

namespace mont {
namespace {

// Validates the jobs and plans the run: per-job units and reserved workspace
// (twiddle tables, checksum accumulators; ws may be null when only counting),
// then the fusion groups.
mont_status_t plan_run(const mont_host_job_t *jobs, int njobs, void *ws, JobPlan *plan, Group *groups, int &ng,
                       size_t &reserved) {
    // plan: reserved area (tables, accumulators), then the ring
    if (njobs > 64) return MONT_EUNSUPPORTED;
    reserved = 0;
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
            case MONT_HOST_NTT:  // rows of len = 2^k words, transformed in place in the slot
                if (J.len < 2 || J.len > 32768 || (J.len & (J.len - 1)) || (J.scale && J.scale >= J.ctx->p))
                    return MONT_EINVAL_ARG;
                P.nin = 1; P.unit_words = J.len; P.units = J.n;
                P.dtab = (uint32_t *)((char *)ws + reserved);
                reserved += align_up((J.len - 1) * 4);
                break;
            default: return MONT_EINVAL_ARG;
        }
        if (J.n && (!J.out || !J.in0 || (P.nin == 2 && !J.in1) ||
                    ((J.op == MONT_HOST_TWIDDLE || J.op == MONT_HOST_NTT) && !J.in1)))
            return MONT_EINVAL_ARG;
        if (J.depends_on >= j || J.depends_on < -1) return MONT_EINVAL_ARG;
        if (J.op == MONT_HOST_MUL_VEC && J.acc_host) {
            P.dacc = (unsigned long long *)((char *)ws + reserved);
            reserved += kAlign;
        }
    }
    // fusion groups (see Group): job j joins the group of job j-1 when both are elementwise over
    // the same n, j reads at least one buffer of the group (an input, or an output it then takes
    // from the device), and j's output aliases no buffer of the group
    ng = 0;
    for (int j = 0; j < njobs; ++j) {
        const mont_host_job_t &J = jobs[j];
        const uint32_t *ins[2] = {J.in0, plan[j].nin == 2 ? J.in1 : nullptr};
        bool join = false;
        if (ng > 0 && elementwise(J.op)) {
            Group &G = groups[ng - 1];
            const mont_host_job_t &F = jobs[G.j0];
            if (elementwise(F.op) && F.n == J.n && G.nbuf + 3 <= kMaxBufs) {
                bool shares = false, clash = false;
                for (int q = G.j0; q < j; ++q) {
                    const mont_host_job_t &Q = jobs[q];
                    const uint32_t *qb[3] = {Q.in0, plan[q].nin == 2 ? Q.in1 : nullptr, Q.out};
                    for (int k = 0; k < 2; ++k)
                        for (int b = 0; b < 3; ++b) shares |= ins[k] && ins[k] == qb[b];
                    for (int b = 0; b < 3; ++b) clash |= qb[b] && (const uint32_t *)J.out == qb[b];
                }
                join = shares && !clash;
            }
        }
        if (!join) {
            Group &G = groups[ng++];
            G.j0 = j;
            G.nbuf_in = 0;
            G.nbuf = 0;
        }
        Group &G = groups[ng - 1];
        G.j1 = j + 1;
        for (int k = 0; k < 2; ++k) {
            G.src[j - G.j0][k] = -1;
            if (!ins[k]) continue;
            for (int q = G.j0; q < j && G.src[j - G.j0][k] < 0; ++q)  // an earlier job's output?
                if ((const uint32_t *)jobs[q].out == ins[k]) G.src[j - G.j0][k] = G.dst[q - G.j0];
            for (int b = 0; b < G.nbuf_in && G.src[j - G.j0][k] < 0; ++b)  // an input already uploaded?
                if (G.in_host[b] == ins[k]) G.src[j - G.j0][k] = b;
            if (G.src[j - G.j0][k] < 0) {  // a new uploaded input: inputs come first, so shift outputs
                for (int q = G.j0; q < j; ++q) {
                    ++G.dst[q - G.j0];
                    for (int kk = 0; kk < 2; ++kk)
                        if (G.src[q - G.j0][kk] >= G.nbuf_in) ++G.src[q - G.j0][kk];
                }
                if (k == 1 && G.src[j - G.j0][0] >= G.nbuf_in) ++G.src[j - G.j0][0];
                G.in_host[G.nbuf_in] = ins[k];
                G.src[j - G.j0][k] = G.nbuf_in++;
                ++G.nbuf;
            }
        }
        if (J.op == MONT_HOST_NTT) G.dst[j - G.j0] = G.src[j - G.j0][0];  // in place (never fused)
        else G.dst[j - G.j0] = G.nbuf++;
    }
    return MONT_OK;
}

}  // namespace
}  // namespace mont

extern "C" mont_status_t mont_host_run(const mont_host_job_t *jobs, int njobs, void *ws, size_t ws_bytes,
                                       cudaStream_t stream) {
    if (njobs < 0 || (njobs > 0 && !jobs) || (njobs > 0 && (!ws || ((uintptr_t)ws & 15u)))) return MONT_EINVAL_ARG;
    if (njobs == 0) return MONT_OK;
    static thread_local JobPlan plan[64];
    static thread_local Group groups[64];
    int ng = 0;
    size_t reserved = 0;
    const mont_status_t pst = plan_run(jobs, njobs, ws, plan, groups, ng, reserved);
    if (pst != MONT_OK) return pst;
    int kb = 3;
    for (int gi = 0; gi < ng; ++gi) kb = groups[gi].nbuf > kb ? groups[gi].nbuf : kb;
    if (ws_bytes < reserved + (size_t)kRing * kb * kAlign) return MONT_EINVAL_ARG;
    const size_t buf_bytes = ((ws_bytes - reserved) / ((size_t)kRing * kb)) / kAlign * kAlign;
    char *ring = (char *)ws + reserved;
    auto slot_buf = [&](int slot, int k) { return (uint32_t *)(ring + ((size_t)slot * kb + k) * buf_bytes); };
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
        const size_t tab_words = jobs[j].op == MONT_HOST_NTT ? jobs[j].len - 1 : jobs[j].len;
        if (plan[j].dtab && jobs[j].n &&
            cudaMemcpyAsync(plan[j].dtab, jobs[j].in1, tab_words * 4, cudaMemcpyHostToDevice, R.h2d) != cudaSuccess)
            return MONT_ECUDA;
        if (plan[j].dacc && cudaMemsetAsync(plan[j].dacc, 0, 8, R.krn) != cudaSuccess) return MONT_ECUDA;
    }
    size_t g = 0;  // global chunk counter -> ring slot
    int slot_out0[kRing];  // per slot: first output buffer of the chunk that used it last
    // one chunk of group gi at unit offset u0 through ring slot g % kRing
    auto issue = [&](int gi, size_t u0) -> mont_status_t {
        const Group &G = groups[gi];
        const JobPlan &P = plan[G.j0];  // all jobs of a group share n, unit size and chunk
        const int slot = (int)(g % kRing);
        const size_t nu = P.units - u0 < P.chunk ? P.units - u0 : P.chunk;
        const size_t off = u0 * P.unit_words, bytes = nu * P.unit_words * 4;
        // the slot's previous chunk must be done with the buffers this upload overwrites: its
        // kernels, and also its downloads when some of them were outputs there (a group with
        // more inputs than the one before it)
        if (g >= (size_t)kRing)
            cudaStreamWaitEvent(R.h2d, G.nbuf_in > slot_out0[slot] ? R.d2h_done[slot] : R.k_done[slot], 0);
        slot_out0[slot] = jobs[G.j0].op == MONT_HOST_NTT ? 0 : G.nbuf_in;  // NTT: in place in buffer 0
        for (int b = 0; b < G.nbuf_in; ++b)
            if (cudaMemcpyAsync(slot_buf(slot, b), G.in_host[b] + off, bytes, cudaMemcpyHostToDevice, R.h2d) !=
                cudaSuccess)
                return MONT_ECUDA;
        cudaEventRecord(R.h2d_done[slot], R.h2d);
        cudaStreamWaitEvent(R.krn, R.h2d_done[slot], 0);
        if (g >= (size_t)kRing) cudaStreamWaitEvent(R.krn, R.d2h_done[slot], 0);
        for (int j = G.j0; j < G.j1; ++j) {
            const mont_host_job_t &J = jobs[j];
            const JobPlan &Pj = plan[j];
            uint32_t *d0 = slot_buf(slot, G.src[j - G.j0][0]);
            uint32_t *d1 = Pj.nin == 2 ? slot_buf(slot, G.src[j - G.j0][1]) : nullptr;
            uint32_t *dout = slot_buf(slot, G.dst[j - G.j0]);
            mont_status_t st;
            switch (J.op) {
                case MONT_HOST_MUL_VEC:
                    st = Pj.dacc ? mont_mul_vec_checksum(J.ctx, dout, d0, d1, nu, Pj.dacc, R.krn)
                                 : mont_mul_vec(J.ctx, dout, d0, d1, nu, R.krn);
                    break;
                case MONT_HOST_POW_VEC: st = mont_pow_vec(J.ctx, dout, d0, d1, nu, R.krn); break;
                case MONT_HOST_TO_MONT: st = to_mont(J.ctx, dout, d0, nu, R.krn); break;
                case MONT_HOST_FROM_MONT: st = from_mont(J.ctx, dout, d0, nu, R.krn); break;
                case MONT_HOST_NTT: {
                    int log_n = 0;
                    while ((1ull << log_n) < J.len) ++log_n;
                    st = mont_ntt(J.ctx, dout, nu, log_n, Pj.dtab, J.scale ? J.scale : J.ctx->r1, R.krn);
                    break;
                }
                default: st = mont_mul_twiddle(J.ctx, dout, d0, Pj.dtab, nu, J.len, R.krn); break;
            }
            if (st != MONT_OK) return st;
        }
        cudaEventRecord(R.k_done[slot], R.krn);
        cudaStreamWaitEvent(R.d2h, R.k_done[slot], 0);
        for (int j = G.j0; j < G.j1; ++j)
            if (cudaMemcpyAsync(jobs[j].out + off, slot_buf(slot, G.dst[j - G.j0]), bytes, cudaMemcpyDeviceToHost,
                                R.d2h) != cudaSuccess)
                return MONT_ECUDA;
        cudaEventRecord(R.d2h_done[slot], R.d2h);
        ++g;
        return MONT_OK;
    };
    // after a group's last chunk: checksums and completion events (kernels run in issue order on
    // R.krn, so the latest k_done covers every kernel of the group)
    auto finish = [&](int gi) -> mont_status_t {
        const Group &G = groups[gi];
        for (int j = G.j0; j < G.j1; ++j) {
            if (plan[j].dacc) {
                cudaStreamWaitEvent(R.d2h, R.k_done[(g + kRing - 1) % kRing], 0);
                if (cudaMemcpyAsync(jobs[j].acc_host, plan[j].dacc, 8, cudaMemcpyDeviceToHost, R.d2h) != cudaSuccess)
                    return MONT_ECUDA;
            }
        }
        for (int j = G.j0; j < G.j1; ++j)
            if (R.job_out[j]) cudaEventRecord(R.job_out[j], R.d2h);  // the group's outputs are in host memory
        return MONT_OK;
    };
    // Chunk order: groups stream in job order, but up to kWin consecutive ready groups are
    // interleaved chunk by chunk, each step taking the chunk that keeps the H2D and D2H byte
    // counts closest (the link is duplex: a download-heavy group next to upload-heavy ones keeps
    // both directions busy).  A group that depends on an earlier group's host outputs becomes
    // ready only after that group's last chunk (its completion event) has been issued.
    constexpr int kWin = 3;
    static thread_local size_t next_u0[64];
    static thread_local bool started[64], done[64];
    static thread_local int group_of[64];
    for (int gi = 0; gi < ng; ++gi) {
        next_u0[gi] = 0;
        started[gi] = done[gi] = false;
        for (int j = groups[gi].j0; j < groups[gi].j1; ++j) group_of[j] = gi;
    }
    // groups whose host buffers overlap (one writes what the other reads or writes) keep job
    // order: the later one starts only after the earlier one has issued its last chunk
    auto overlap = [](const void *p, size_t pb, const void *q, size_t qb) {
        const char *a = (const char *)p, *b = (const char *)q;
        return p && q && pb && qb && a < b + qb && b < a + pb;
    };
    auto conflict = [&](int ga, int gb) {
        const Group &A = groups[ga], &B = groups[gb];
        const size_t ba = plan[A.j0].units * plan[A.j0].unit_words * 4, bb = plan[B.j0].units * plan[B.j0].unit_words * 4;
        for (int ja = A.j0; ja < A.j1; ++ja)
            for (int jb = B.j0; jb < B.j1; ++jb) {
                const void *ra[3] = {jobs[ja].in0, plan[ja].nin == 2 ? jobs[ja].in1 : nullptr, jobs[ja].out};
                const void *rb[3] = {jobs[jb].in0, plan[jb].nin == 2 ? jobs[jb].in1 : nullptr, jobs[jb].out};
                for (int x = 0; x < 3; ++x)
                    if (overlap(jobs[ja].out, ba, rb[x], bb) || overlap(jobs[jb].out, bb, ra[x], ba)) return true;
            }
        return false;
    };
    unsigned long long cum_in = 0, cum_out = 0;
    int remaining = ng;
    while (remaining > 0) {
        int cand[kWin], nc = 0;
        for (int gi = 0; gi < ng && nc < kWin; ++gi) {
            if (done[gi]) continue;
            bool ready = true;
            for (int j = groups[gi].j0; j < groups[gi].j1; ++j) {
                const int d = jobs[j].depends_on;
                if (d >= 0 && group_of[d] != gi && !done[group_of[d]]) ready = false;
            }
            for (int c = 0; c < nc && ready; ++c) ready = !conflict(cand[c], gi);
            if (!ready) break;  // keep job order: nothing past a group still waiting
            cand[nc++] = gi;
        }
        int best = cand[0];
        unsigned long long best_cost = ~0ull;
        for (int c = 0; c < nc; ++c) {
            const Group &G = groups[cand[c]];
            const JobPlan &P = plan[G.j0];
            const size_t nu = P.units - next_u0[cand[c]] < P.chunk ? P.units - next_u0[cand[c]] : P.chunk;
            const unsigned long long b = (unsigned long long)nu * P.unit_words * 4;
            const unsigned long long in = cum_in + b * G.nbuf_in, out = cum_out + b * (G.j1 - G.j0);
            const unsigned long long cost = in > out ? in : out;
            if (cost < best_cost) best_cost = cost, best = cand[c];
        }
        const Group &G = groups[best];
        const JobPlan &P = plan[G.j0];
        if (!started[best]) {
            started[best] = true;
            for (int j = G.j0; j < G.j1; ++j) {  // dependencies on earlier groups' host outputs
                const int d = jobs[j].depends_on;
                if (d >= 0 && d < G.j0) cudaStreamWaitEvent(R.h2d, R.job_out[d], 0);
            }
        }
        mont_status_t st;
        if (P.units > 0) {
            const size_t u0 = next_u0[best];
            const size_t nu = P.units - u0 < P.chunk ? P.units - u0 : P.chunk;
            if ((st = issue(best, u0)) != MONT_OK) return st;
            next_u0[best] = u0 + nu;
            cum_in += (unsigned long long)nu * P.unit_words * 4 * G.nbuf_in;
            cum_out += (unsigned long long)nu * P.unit_words * 4 * (G.j1 - G.j0);
        }
        if (next_u0[best] >= P.units) {
            if ((st = finish(best)) != MONT_OK) return st;
            done[best] = true;
            --remaining;
        }
    }
    cudaEventRecord(R.done_k, R.krn);
    cudaEventRecord(R.done_d, R.d2h);
    cudaStreamWaitEvent(stream, R.done_k, 0);
    cudaStreamWaitEvent(stream, R.done_d, 0);
    return launch_status();
}

extern "C" mont_status_t mont_host_run_bytes(const mont_host_job_t *jobs, int njobs, unsigned long long *h2d_bytes,
                                             unsigned long long *d2h_bytes) {
    if (njobs < 0 || (njobs > 0 && !jobs) || !h2d_bytes || !d2h_bytes) return MONT_EINVAL_ARG;
    *h2d_bytes = *d2h_bytes = 0;
    if (njobs == 0) return MONT_OK;
    static thread_local JobPlan plan[64];
    static thread_local Group groups[64];
    int ng = 0;
    size_t reserved = 0;
    const mont_status_t st = plan_run(jobs, njobs, nullptr, plan, groups, ng, reserved);
    if (st != MONT_OK) return st;
    for (int j = 0; j < njobs; ++j) {
        const size_t bytes = plan[j].units * plan[j].unit_words * 4;
        if (jobs[j].op == MONT_HOST_TWIDDLE) *h2d_bytes += jobs[j].len * 4;  // the table, once
        if (jobs[j].op == MONT_HOST_NTT && jobs[j].n) *h2d_bytes += (jobs[j].len - 1) * 4;
        *d2h_bytes += bytes + (jobs[j].op == MONT_HOST_MUL_VEC && jobs[j].acc_host ? 8 : 0);
    }
    for (int gi = 0; gi < ng; ++gi)
        *h2d_bytes += (unsigned long long)groups[gi].nbuf_in * plan[groups[gi].j0].units * plan[groups[gi].j0].unit_words * 4;
    return MONT_OK;
}
