// k_pow.cu -- K3 mont_pow_vec: out[i] = base[i]^exp[i] mod P (SURVEY.md §8(a) A9,
// BASELINE configs[3]); K-twiddle-table: tw[j] = to_mont(w^j).
//
// The ladder is the "long sequence of modular arithmetic" for which the paper
// argues the residue-class conversion cost becomes negligible:
// one to_mont, ~46 Montgomery products held in registers, one from_mont.
// The kernel is bound by the integer-multiply (FMAHeavy) pipe, not HBM
// (12 B per ~48 REDCs).  B200 design choices:
//   * signed lazy REDC (mont_core.cuh sredc): 3 FMAHeavy ops per product
//     (IMAD.WIDE, IMAD, IMAD.WIDE), values stay in (-P, P) with no correction
//     inside the chain;
//   * per-lane exponents would make a bitwise if() diverge inside a warp, so
//     the ladder is a fixed 2-bit window (variant 0): every lane executes the
//     same 2 + 15*3 = 47 products and picks its multiplier x^d (d in 0..3,
//     x^0 = 1-bar) with selects on the ALU pipe; variant 2 is the 3-bit window
//     (6 + 10*4 = 46 products, 8-way select); variant 1 the binary ladder with
//     selects (64 products, reference point);
//   * each thread runs the 4 independent ladders of one uint4 interleaved
//     (instruction-level parallelism covers the ~20-cycle dependent latency).
#include <cuda_runtime.h>
#include <stdint.h>

#include "abi_util.h"

namespace mont {

struct PowParams {
    int32_t p, negp, pinv;  // negp = -P, pinv = P^-1 mod 2^32 = -pneg
    uint32_t pneg, r1, r2;
};

// ---- one lane's ladder, written for L lanes in lock-step so the compiler
// interleaves the L independent dependency chains.
template <int L>
__device__ __forceinline__ void pow_window2(const PowParams &q, const uint32_t (&base)[L], const uint32_t (&e)[L],
                                            uint32_t (&out)[L]) {
    int32_t t1[L], t2[L], t3[L], acc[L];
    const int32_t one = (int32_t)q.r1;
#pragma unroll
    for (int l = 0; l < L; ++l) {
        t1[l] = (int32_t)redc(base[l], q.r2, (uint32_t)q.p, q.pneg);  // x-bar, canonical
        t2[l] = sredc(t1[l], t1[l], q.negp, q.pinv);
        t3[l] = sredc(t2[l], t1[l], q.negp, q.pinv);
        const uint32_t d = e[l] >> 30;
        acc[l] = d == 0 ? one : d == 1 ? t1[l] : d == 2 ? t2[l] : t3[l];
    }
#pragma unroll 1
    for (int sh = 28; sh >= 0; sh -= 2) {
#pragma unroll
        for (int l = 0; l < L; ++l) {
            int32_t a = sredc(acc[l], acc[l], q.negp, q.pinv);
            a = sredc(a, a, q.negp, q.pinv);
            const uint32_t d = (e[l] >> sh) & 3u;
            const int32_t lo = (d & 1u) ? t1[l] : one;
            const int32_t hi = (d & 1u) ? t3[l] : t2[l];
            acc[l] = sredc(a, (d & 2u) ? hi : lo, q.negp, q.pinv);
        }
    }
#pragma unroll
    for (int l = 0; l < L; ++l) {
        // from_mont: REDC(acc * 1) in signed form, then canonicalise
        out[l] = canon(sredc1(acc[l], q.negp, q.pinv), q.p);
    }
}

template <int L>
__device__ __forceinline__ void pow_window3(const PowParams &q, const uint32_t (&base)[L], const uint32_t (&e)[L],
                                            uint32_t (&out)[L]) {
    int32_t t[L][8], acc[L];
#pragma unroll
    for (int l = 0; l < L; ++l) {
        t[l][0] = (int32_t)q.r1;
        t[l][1] = (int32_t)redc(base[l], q.r2, (uint32_t)q.p, q.pneg);
#pragma unroll
        for (int k = 2; k < 8; ++k) t[l][k] = sredc(t[l][k - 1], t[l][1], q.negp, q.pinv);
        const uint32_t d = e[l] >> 30;  // top 2 bits
        const int32_t s01 = (d & 1u) ? t[l][1] : t[l][0];
        const int32_t s23 = (d & 1u) ? t[l][3] : t[l][2];
        acc[l] = (d & 2u) ? s23 : s01;
    }
#pragma unroll 1
    for (int sh = 27; sh >= 0; sh -= 3) {
#pragma unroll
        for (int l = 0; l < L; ++l) {
            int32_t a = sredc(acc[l], acc[l], q.negp, q.pinv);
            a = sredc(a, a, q.negp, q.pinv);
            a = sredc(a, a, q.negp, q.pinv);
            const uint32_t d = (e[l] >> sh) & 7u;
            const bool b0 = d & 1u, b1 = d & 2u, b2 = d & 4u;
            const int32_t s01 = b0 ? t[l][1] : t[l][0];
            const int32_t s23 = b0 ? t[l][3] : t[l][2];
            const int32_t s45 = b0 ? t[l][5] : t[l][4];
            const int32_t s67 = b0 ? t[l][7] : t[l][6];
            const int32_t s03 = b1 ? s23 : s01;
            const int32_t s47 = b1 ? s67 : s45;
            acc[l] = sredc(a, b2 ? s47 : s03, q.negp, q.pinv);
        }
    }
#pragma unroll
    for (int l = 0; l < L; ++l) {
        out[l] = canon(sredc1(acc[l], q.negp, q.pinv), q.p);
    }
}

template <int L>
__device__ __forceinline__ void pow_binary(const PowParams &q, const uint32_t (&base)[L], const uint32_t (&e)[L],
                                           uint32_t (&out)[L]) {
    int32_t x[L], acc[L];
#pragma unroll
    for (int l = 0; l < L; ++l) {
        x[l] = (int32_t)redc(base[l], q.r2, (uint32_t)q.p, q.pneg);
        acc[l] = (int32_t)q.r1;
    }
#pragma unroll 1
    for (int sh = 31; sh >= 0; --sh) {
#pragma unroll
        for (int l = 0; l < L; ++l) {
            int32_t a = sredc(acc[l], acc[l], q.negp, q.pinv);
            int32_t m = sredc(a, x[l], q.negp, q.pinv);
            acc[l] = ((e[l] >> sh) & 1u) ? m : a;
        }
    }
#pragma unroll
    for (int l = 0; l < L; ++l) {
        out[l] = canon(sredc1(acc[l], q.negp, q.pinv), q.p);
    }
}

template <int V>
__device__ __forceinline__ void pow_lanes(const PowParams &q, const uint32_t (&b)[4], const uint32_t (&e)[4],
                                          uint32_t (&o)[4]) {
    if (V == 0) pow_window2<4>(q, b, e, o);
    else if (V == 1) pow_binary<4>(q, b, e, o);
    else pow_window3<4>(q, b, e, o);
}

template <int V>
__device__ __forceinline__ uint32_t pow_one(const PowParams &q, uint32_t b, uint32_t e) {
    uint32_t bb[1] = {b}, ee[1] = {e}, oo[1];
    if (V == 0) pow_window2<1>(q, bb, ee, oo);
    else if (V == 1) pow_binary<1>(q, bb, ee, oo);
    else pow_window3<1>(q, bb, ee, oo);
    return oo[0];
}

// head/tail scalars by CTA 0; vector body over n4 uint4 chunks (grid-stride)
template <int V>
__global__ void __launch_bounds__(256) k_pow(PowParams q, uint32_t *out, const uint32_t *base, const uint32_t *exp,
                                              uint32_t head, size_t n4, uint32_t tail) {
    if (blockIdx.x == 0 && threadIdx.x < head + tail) {
        size_t i = threadIdx.x < head ? threadIdx.x : head + 4 * n4 + (threadIdx.x - head);
        out[i] = pow_one<V>(q, base[i], exp[i]);
    }
    const uint4 *b4 = reinterpret_cast<const uint4 *>(base + head);
    const uint4 *e4 = reinterpret_cast<const uint4 *>(exp + head);
    uint4 *o4 = reinterpret_cast<uint4 *>(out + head);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const uint4 bv = ld_stream(b4 + i), ev = ld_stream(e4 + i);
        uint32_t b[4] = {bv.x, bv.y, bv.z, bv.w}, e[4] = {ev.x, ev.y, ev.z, ev.w}, o[4];
        pow_lanes<V>(q, b, e, o);
        st_stream(o4 + i, make_uint4(o[0], o[1], o[2], o[3]));
    }
}

template <int V>
__global__ void __launch_bounds__(256) k_pow_scalar(PowParams q, uint32_t *out, const uint32_t *base,
                                                     const uint32_t *exp, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = pow_one<V>(q, base[i], exp[i]);
}

// tw[j] = to_mont(w^j): binary ladder on the bits of j, canonical output
__global__ void __launch_bounds__(256) k_twiddle_table(Ctx c, uint32_t *tw, uint32_t w, size_t len) {
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < len; j += (size_t)gridDim.x * blockDim.x) {
        const uint32_t x = redc(w, c.r2, c.p, c.pneg);
        uint32_t acc = c.r1;
        unsigned long long e = j;
        for (int sh = 63 - __clzll(e | 1ull); sh >= 0; --sh) {
            acc = redc(acc, acc, c.p, c.pneg);
            if ((e >> sh) & 1ull) acc = redc(acc, x, c.p, c.pneg);
        }
        tw[j] = acc;
    }
}

static const Launch kPowDefault{256, 8, 1, 0, 0};

}  // namespace mont

using namespace mont;

extern "C" mont_status_t mont_pow_vec_ex(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *base,
                                         const uint32_t *exp, size_t n, const mont_launch_t *cfg,
                                         cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (n == 0) return MONT_OK;
    if (!out || !base || !exp || ((uintptr_t)out | (uintptr_t)base | (uintptr_t)exp) & 3u) return MONT_EINVAL_ARG;
    Launch L = resolve(cfg, kPowDefault);
    if (L.threads != 256 || L.variant < 0 || L.variant > 2) return MONT_EINVAL_ARG;
    const int sms = sm_count();
    if (sms <= 0) return MONT_ECUDA;
    PowParams q{(int32_t)ctx->p, -(int32_t)ctx->p, (int32_t)(0u - ctx->pneg), ctx->pneg, ctx->r1, ctx->r2};
    const uintptr_t pb = (uintptr_t)base, pe = (uintptr_t)exp, po = (uintptr_t)out;
    const int threads = 256;
    if (same_mod16(pb, pe) && same_mod16(pb, po)) {
        const uint32_t head = head_elems(pb, n);
        const size_t n4 = (n - head) / 4;
        const uint32_t tail = (uint32_t)((n - head) % 4);
        size_t grid = (size_t)sms * L.ctas_per_sm;
        const size_t need = (n4 + threads - 1) / threads;
        if (grid > need) grid = need;
        if (grid == 0) grid = 1;
        switch (L.variant) {
            case 0: k_pow<0><<<(unsigned)grid, threads, 0, stream>>>(q, out, base, exp, head, n4, tail); break;
            case 1: k_pow<1><<<(unsigned)grid, threads, 0, stream>>>(q, out, base, exp, head, n4, tail); break;
            default: k_pow<2><<<(unsigned)grid, threads, 0, stream>>>(q, out, base, exp, head, n4, tail); break;
        }
    } else {
        size_t grid = (size_t)sms * L.ctas_per_sm;
        const size_t need = (n + threads - 1) / threads;
        if (grid > need) grid = need;
        switch (L.variant) {
            case 0: k_pow_scalar<0><<<(unsigned)grid, threads, 0, stream>>>(q, out, base, exp, n); break;
            case 1: k_pow_scalar<1><<<(unsigned)grid, threads, 0, stream>>>(q, out, base, exp, n); break;
            default: k_pow_scalar<2><<<(unsigned)grid, threads, 0, stream>>>(q, out, base, exp, n); break;
        }
    }
    return launch_status();
}

extern "C" mont_status_t mont_pow_vec(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *base,
                                      const uint32_t *exp, size_t n, cudaStream_t stream) {
    return mont_pow_vec_ex(ctx, out, base, exp, n, nullptr, stream);
}

extern "C" mont_status_t mont_twiddle_table(const mont_ctx_t *ctx, uint32_t *tw, uint32_t w, size_t len,
                                            cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (len == 0) return MONT_OK;
    if (!tw || ((uintptr_t)tw & 3u)) return MONT_EINVAL_ARG;
    const int sms = sm_count();
    if (sms <= 0) return MONT_ECUDA;
    size_t grid = (len + 255) / 256;
    if (grid > (size_t)sms * 8) grid = (size_t)sms * 8;
    k_twiddle_table<<<(unsigned)grid, 256, 0, stream>>>(to_dev(ctx), tw, w, len);
    return launch_status();
}
