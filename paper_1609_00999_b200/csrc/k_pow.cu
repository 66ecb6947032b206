// k_pow.cu -- K3 mont_pow_vec: out[i] = base[i]^exp[i] mod P (SURVEY.md §8(a) A9,
// BASELINE configs[3]); K-twiddle-table: tw[j] = to_mont(w^j).
//
// The ladder is the "long sequence of modular arithmetic" for which the paper
// argues the residue-class conversion cost becomes negligible:
// one to_mont, ~46 Montgomery products held in registers, one from_mont.
// The kernel is bound by the integer-multiply (FMAHeavy) pipe, not HBM
// (12 B per ~48 REDCs).  B200 design choices:
//   * signed lazy REDC (mont_core.cuh sredc): 3 FMAHeavy instructions per
//     product (IMAD.WIDE, IMAD, IMAD.WIDE = 5 issue slots: high-word products
//     are half rate on B200), values stay in (-P, P) with no correction inside
//     the chain;
//   * per-lane exponents would make a bitwise if() diverge inside a warp, so
//     the ladder is a fixed 2-bit window (variant 0): every lane executes the
//     same 2 + 15*3 = 47 products and picks its multiplier x^d (d in 0..3,
//     x^0 = 1-bar) with selects on the ALU pipe; variant 2 is the 3-bit window
//     (6 + 10*4 = 46 products, 8-way select); variant 1 the binary ladder with
//     selects (64 products, reference point);
//   * each thread runs the 4 independent ladders of one uint4 interleaved
//     (instruction-level parallelism covers the ~20-cycle dependent latency);
//     variant 10 runs 8 (two uint4), which saturates the pipe with fewer
//     resident CTAs -- bench.py's two-lane step uses it at 2 CTAs/SM;
//   * measured alternatives kept as variants: 3/4 = the window table in shared
//     memory, 5-8 = some lanes as FP64 Barrett products on the FP64 pipe,
//     9 = PAPER.md Alg. 3 (Fourier-prime REDC) products.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/barrett.h"
#include "abi_util.h"

namespace mont {

struct PowParams {
    int32_t p, pinv;  // pinv = P^-1 mod 2^32 = -pneg
    uint32_t r1, r2;
    double pd, pdinv;  // P and fl(1/P) for the FP64 lanes
};

// x-bar = to_mont(base) = REDC(base, R^2 mod P): canonical, valid for any uint32 base
__device__ __forceinline__ int32_t pow_entry(const PowParams &q, uint32_t base) {
    return (int32_t)redc(base, q.r2, (uint32_t)q.p, (uint32_t)q.pinv);
}
// out = from_mont(acc) canonical
__device__ __forceinline__ uint32_t pow_exit(const PowParams &q, int32_t acc) {
    return canon(sredc1(acc, q.p, q.pinv), q.p);
}

// ---- W-bit fixed-window ladder over the 32 exponent bits, L lanes in
// lock-step (the compiler interleaves the L independent chains).  The first
// window takes the top (32 mod W, or W) bits and needs no squaring.  Table
// x^0..x^(2^W - 1) in Montgomery form, held in registers (multiplier picked by
// a select tree on the ALU pipe) or, with SMEM, in a per-thread slice of
// shared memory (one LDS per window on the LSU pipe).
template <int W, int L, bool SMEM>
__device__ __forceinline__ void pow_window(const PowParams &q, const uint32_t (&base)[L], const uint32_t (&e)[L],
                                           uint32_t (&out)[L], int32_t *s_tab) {
    constexpr int K = 1 << W;
    constexpr int TOP = (32 % W) ? (32 % W) : W;  // bits in the first window
    int32_t t[L][SMEM ? 2 : K], acc[L];
    const uint32_t bd = blockDim.x;
#pragma unroll
    for (int l = 0; l < L; ++l) {
        int32_t x = pow_entry(q, base[l]);
        int32_t prev = (int32_t)q.r1;
        int32_t first = prev;
        const uint32_t d0 = e[l] >> (32 - TOP);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int32_t v = k == 0 ? (int32_t)q.r1 : k == 1 ? x : sredc(prev, x, q.p, q.pinv);
            if (SMEM) s_tab[(k * L + l) * bd + threadIdx.x] = v;
            else t[l][k] = v;
            if (k < (1 << TOP)) first = (d0 == (uint32_t)k) ? v : first;
            prev = v;
        }
        acc[l] = first;
    }
#pragma unroll
    for (int sh = 32 - TOP - W; sh >= 0; sh -= W) {
#pragma unroll
        for (int l = 0; l < L; ++l) {
            int32_t a = acc[l];
#pragma unroll
            for (int r = 0; r < W; ++r) a = sredc(a, a, q.p, q.pinv);
            const uint32_t d = (e[l] >> sh) & (uint32_t)(K - 1);
            int32_t mlt;
            if (SMEM) {
                mlt = s_tab[(d * L + l) * bd + threadIdx.x];
            } else if (W == 2) {
                const int32_t lo = (d & 1u) ? t[l][1] : t[l][0];
                const int32_t hi = (d & 1u) ? t[l][3] : t[l][2];
                mlt = (d & 2u) ? hi : lo;
            } else {
                int32_t cur = t[l][0];
#pragma unroll
                for (int k = 1; k < K; ++k) cur = (d == (uint32_t)k) ? t[l][k] : cur;
                mlt = cur;
            }
            acc[l] = sredc(a, mlt, q.p, q.pinv);
        }
    }
#pragma unroll
    for (int l = 0; l < L; ++l) out[l] = pow_exit(q, acc[l]);
}

// binary ladder with selects: 32 squarings + 32 multiplies, reference point
template <int L>
__device__ __forceinline__ void pow_binary(const PowParams &q, const uint32_t (&base)[L], const uint32_t (&e)[L],
                                           uint32_t (&out)[L]) {
    int32_t x[L], acc[L];
#pragma unroll
    for (int l = 0; l < L; ++l) {
        x[l] = pow_entry(q, base[l]);
        acc[l] = (int32_t)q.r1;
    }
#pragma unroll 4
    for (int sh = 31; sh >= 0; --sh) {
#pragma unroll
        for (int l = 0; l < L; ++l) {
            const int32_t a = sredc(acc[l], acc[l], q.p, q.pinv);
            const int32_t mm = sredc(a, x[l], q.p, q.pinv);
            acc[l] = ((e[l] >> sh) & 1u) ? mm : a;
        }
    }
#pragma unroll
    for (int l = 0; l < L; ++l) out[l] = pow_exit(q, acc[l]);
}

// ---- hybrid 2-bit window: of the 4 lanes of a uint4, NI run the integer
// Montgomery ladder on the IMAD (FMAHeavy) pipe and 4 - NI run the same
// ladder as FP64 Barrett products (mont_core.cuh fmulmod) on the otherwise
// idle FP64 pipe, on plain residues (no residue-class conversion needed).
// Both instruction streams interleave in one thread, so the two multiplier
// arrays of the SM work at once.  Results are identical: both compute
// base^exp mod P exactly and canonicalise.
template <int NI>
__device__ __forceinline__ void pow_hybrid(const PowParams &q, const uint32_t (&base)[4], const uint32_t (&e)[4],
                                           uint32_t (&out)[4]) {
    constexpr int NF = 4 - NI;
    int32_t ti[NI > 0 ? NI : 1][4], ai[NI > 0 ? NI : 1];
    double tf[NF > 0 ? NF : 1][4], af[NF > 0 ? NF : 1];
#pragma unroll
    for (int l = 0; l < NI; ++l) {
        const int32_t x = pow_entry(q, base[l]);
        ti[l][0] = (int32_t)q.r1;
        ti[l][1] = x;
        ti[l][2] = sredc(x, x, q.p, q.pinv);
        ti[l][3] = sredc(ti[l][2], x, q.p, q.pinv);
        const uint32_t d0 = e[l] >> 30;
        ai[l] = (d0 & 2u) ? ((d0 & 1u) ? ti[l][3] : ti[l][2]) : ((d0 & 1u) ? ti[l][1] : ti[l][0]);
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        const double x = fmulmod((double)base[NI + f], 1.0, q.pd, q.pdinv);  // base mod P, in (-P/2, P/2]
        tf[f][0] = 1.0;
        tf[f][1] = x;
        tf[f][2] = fmulmod(x, x, q.pd, q.pdinv);
        tf[f][3] = fmulmod(tf[f][2], x, q.pd, q.pdinv);
        const uint32_t d0 = e[NI + f] >> 30;
        af[f] = (d0 & 2u) ? ((d0 & 1u) ? tf[f][3] : tf[f][2]) : ((d0 & 1u) ? tf[f][1] : tf[f][0]);
    }
#pragma unroll
    for (int sh = 28; sh >= 0; sh -= 2) {
#pragma unroll
        for (int l = 0; l < NI; ++l) {
            int32_t a = sredc(ai[l], ai[l], q.p, q.pinv);
            a = sredc(a, a, q.p, q.pinv);
            const uint32_t d = (e[l] >> sh) & 3u;
            const int32_t lo = (d & 1u) ? ti[l][1] : ti[l][0];
            const int32_t hi = (d & 1u) ? ti[l][3] : ti[l][2];
            ai[l] = sredc(a, (d & 2u) ? hi : lo, q.p, q.pinv);
        }
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            double a = fmulmod(af[f], af[f], q.pd, q.pdinv);
            a = fmulmod(a, a, q.pd, q.pdinv);
            const uint32_t d = (e[NI + f] >> sh) & 3u;
            const double lo = (d & 1u) ? tf[f][1] : tf[f][0];
            const double hi = (d & 1u) ? tf[f][3] : tf[f][2];
            af[f] = fmulmod(a, (d & 2u) ? hi : lo, q.pd, q.pdinv);
        }
    }
#pragma unroll
    for (int l = 0; l < NI; ++l) out[l] = pow_exit(q, ai[l]);
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        const double r = af[f] < 0.0 ? af[f] + q.pd : af[f];
        out[NI + f] = (uint32_t)__double2uint_rn(r);
    }
}

// variant: 0 = 2-bit window, registers; 1 = binary; 2 = 3-bit window, registers;
//          3 = 2-bit window, smem table; 4 = 3-bit window, smem table;
//          5/6/7/8 = hybrid 2-bit window with 3/2/1/0 of 4 lanes on the IMAD
//          pipe and the rest on the FP64 pipe
template <int V, int L>
__device__ __forceinline__ void pow_lanes(const PowParams &q, const uint32_t (&b)[L], const uint32_t (&e)[L],
                                          uint32_t (&o)[L], int32_t *s_tab) {
    if (V == 0) pow_window<2, L, false>(q, b, e, o, s_tab);
    else if (V == 1) pow_binary<L>(q, b, e, o);
    else if (V == 2) pow_window<3, L, false>(q, b, e, o, s_tab);
    else if (V == 3) pow_window<2, L, true>(q, b, e, o, s_tab);
    else if (V == 4) pow_window<3, L, true>(q, b, e, o, s_tab);
    else pow_hybrid<8 - V>(q, b, e, o);
}

template <int V>
constexpr int pow_smem_words() { return V == 3 ? 4 * 4 : V == 4 ? 8 * 4 : 0; }  // per thread, 4 lanes

// Vector body over n4 uint4 chunks; head/tail scalars by CTA 0 (1 lane each,
// using the same table slice layout with L = 4 so the smem footprint matches).
template <int V>
__global__ void __launch_bounds__(256) k_pow(PowParams q, uint32_t *out, const uint32_t *base, const uint32_t *exp,
                                              uint32_t head, size_t n4, uint32_t tail) {
    extern __shared__ int32_t s_tab[];
    if (blockIdx.x == 0 && threadIdx.x < head + tail) {
        size_t i = threadIdx.x < head ? threadIdx.x : head + 4 * n4 + (threadIdx.x - head);
        uint32_t b[4] = {base[i], 0u, 0u, 0u}, e[4] = {exp[i], 0u, 0u, 0u}, o[4];
        pow_lanes<V, 4>(q, b, e, o, s_tab);
        out[i] = o[0];
    }
    const uint4 *b4 = reinterpret_cast<const uint4 *>(base + head);
    const uint4 *e4 = reinterpret_cast<const uint4 *>(exp + head);
    uint4 *o4 = reinterpret_cast<uint4 *>(out + head);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const uint4 bv = ld_stream(b4 + i), ev = ld_stream(e4 + i);
        uint32_t b[4] = {bv.x, bv.y, bv.z, bv.w}, e[4] = {ev.x, ev.y, ev.z, ev.w}, o[4];
        pow_lanes<V, 4>(q, b, e, o, s_tab);
        st_stream(o4 + i, make_uint4(o[0], o[1], o[2], o[3]));
    }
}

// 8 lanes per thread (two uint4): twice the independent chains per thread, so a
// smaller grid saturates the IMAD pipe and leaves thread slots to co-running
// HBM-bound kernels (variant 10)
__global__ void __launch_bounds__(256) k_pow8(PowParams q, uint32_t *out, const uint32_t *base, const uint32_t *exp,
                                               uint32_t head, size_t n4, uint32_t tail) {
    if (blockIdx.x == 0 && threadIdx.x < head + tail) {
        size_t i = threadIdx.x < head ? threadIdx.x : head + 4 * n4 + (threadIdx.x - head);
        uint32_t b[1] = {base[i]}, e[1] = {exp[i]}, o[1];
        pow_window<2, 1, false>(q, b, e, o, nullptr);
        out[i] = o[0];
    }
    const uint4 *b4 = reinterpret_cast<const uint4 *>(base + head);
    const uint4 *e4 = reinterpret_cast<const uint4 *>(exp + head);
    uint4 *o4 = reinterpret_cast<uint4 *>(out + head);
    const size_t n8 = n4 / 2;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x) {
        const uint4 b0 = ld_stream(b4 + 2 * i), b1 = ld_stream(b4 + 2 * i + 1);
        const uint4 e0 = ld_stream(e4 + 2 * i), e1 = ld_stream(e4 + 2 * i + 1);
        uint32_t b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        uint32_t e[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w}, o[8];
        pow_window<2, 8, false>(q, b, e, o, nullptr);
        st_stream(o4 + 2 * i, make_uint4(o[0], o[1], o[2], o[3]));
        st_stream(o4 + 2 * i + 1, make_uint4(o[4], o[5], o[6], o[7]));
    }
    if ((n4 & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {  // odd last uint4
        const uint4 bv = ld_stream(b4 + n4 - 1), ev = ld_stream(e4 + n4 - 1);
        uint32_t b[4] = {bv.x, bv.y, bv.z, bv.w}, e[4] = {ev.x, ev.y, ev.z, ev.w}, o[4];
        pow_window<2, 4, false>(q, b, e, o, nullptr);
        st_stream(o4 + n4 - 1, make_uint4(o[0], o[1], o[2], o[3]));
    }
}

template <int V>
__global__ void __launch_bounds__(256) k_pow_scalar(PowParams q, uint32_t *out, const uint32_t *base,
                                                     const uint32_t *exp, size_t n) {
    extern __shared__ int32_t s_tab[];
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t b[4] = {base[i], 0u, 0u, 0u}, e[4] = {exp[i], 0u, 0u, 0u}, o[4];
        pow_lanes<V, 4>(q, b, e, o, s_tab);
        out[i] = o[0];
    }
}

// ---- Barrett ladder (include/barrett.h): the same 2-bit window on plain values
template <int L>
__device__ __forceinline__ void pow_barrett(const BarrettDev &c, const uint32_t (&base)[L], const uint32_t (&e)[L],
                                            uint32_t (&out)[L]) {
    uint32_t t1[L], t2[L], t3[L], acc[L];
#pragma unroll
    for (int l = 0; l < L; ++l) {
        t1[l] = base[l] % c.p;
        t2[l] = barrett(t1[l], t1[l], c);
        t3[l] = barrett(t2[l], t1[l], c);
        const uint32_t d = e[l] >> 30;
        acc[l] = d == 0 ? 1u : d == 1 ? t1[l] : d == 2 ? t2[l] : t3[l];
    }
#pragma unroll
    for (int sh = 28; sh >= 0; sh -= 2) {
#pragma unroll
        for (int l = 0; l < L; ++l) {
            uint32_t a = barrett(acc[l], acc[l], c);
            a = barrett(a, a, c);
            const uint32_t d = (e[l] >> sh) & 3u;
            const uint32_t lo = (d & 1u) ? t1[l] : 1u;
            const uint32_t hi = (d & 1u) ? t3[l] : t2[l];
            acc[l] = barrett(a, (d & 2u) ? hi : lo, c);
        }
    }
#pragma unroll
    for (int l = 0; l < L; ++l) out[l] = acc[l];  // barrett() outputs are canonical, and 1 < P
}

__global__ void __launch_bounds__(256) k_pow_barrett(BarrettDev c, uint32_t *out, const uint32_t *base,
                                                      const uint32_t *exp, size_t n) {
    const size_t n4 = n / 4;
    const uint4 *b4 = reinterpret_cast<const uint4 *>(base);
    const uint4 *e4 = reinterpret_cast<const uint4 *>(exp);
    uint4 *o4 = reinterpret_cast<uint4 *>(out);
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n4) {
        const uint4 bv = ld_stream(b4 + i), ev = ld_stream(e4 + i);
        uint32_t b[4] = {bv.x, bv.y, bv.z, bv.w}, e[4] = {ev.x, ev.y, ev.z, ev.w}, o[4];
        pow_barrett<4>(c, b, e, o);
        st_stream(o4 + i, make_uint4(o[0], o[1], o[2], o[3]));
    } else if (i < n4 + (n & 3)) {
        const size_t j = 4 * n4 + (i - n4);
        uint32_t b[1] = {base[j]}, e[1] = {exp[j]}, o[1];
        pow_barrett<1>(c, b, e, o);
        out[j] = o[0];
    }
}

// ---- Fourier-prime REDC ladder (variant 9): the same 2-bit window with every
// product an Alg. 3 REDC (identical results to the Montgomery ladder); WIDE = the 33-bit-t
// form for 3P >= 2^32 (mont_core.cuh fredc33)
template <int L, bool WIDE>
__device__ __forceinline__ void pow_fourier(const PowParams &q, const FourierDev &f, const uint32_t (&base)[L],
                                            const uint32_t (&e)[L], uint32_t (&out)[L]) {
    uint32_t t1[L], t2[L], t3[L], acc[L];
#pragma unroll
    for (int l = 0; l < L; ++l) {
        t1[l] = redc(base[l], q.r2, (uint32_t)q.p, (uint32_t)q.pinv);  // to_mont, any uint32 base
        t2[l] = WIDE ? fredc33(t1[l], t1[l], f) : fredc(t1[l], t1[l], f);
        t3[l] = WIDE ? fredc33(t2[l], t1[l], f) : fredc(t2[l], t1[l], f);
        const uint32_t d = e[l] >> 30;
        acc[l] = d == 0 ? q.r1 : d == 1 ? t1[l] : d == 2 ? t2[l] : t3[l];
    }
#pragma unroll
    for (int sh = 28; sh >= 0; sh -= 2) {
#pragma unroll
        for (int l = 0; l < L; ++l) {
            uint32_t a = WIDE ? fredc33(acc[l], acc[l], f) : fredc(acc[l], acc[l], f);
            a = WIDE ? fredc33(a, a, f) : fredc(a, a, f);
            const uint32_t d = (e[l] >> sh) & 3u;
            const uint32_t lo = (d & 1u) ? t1[l] : q.r1;
            const uint32_t hi = (d & 1u) ? t3[l] : t2[l];
            acc[l] = WIDE ? fredc33(a, (d & 2u) ? hi : lo, f) : fredc(a, (d & 2u) ? hi : lo, f);
        }
    }
#pragma unroll
    for (int l = 0; l < L; ++l) out[l] = redc1(acc[l], (uint32_t)q.p, (uint32_t)q.pinv);
}

template <bool WIDE>
__global__ void __launch_bounds__(256) k_pow_fourier(PowParams q, FourierDev f, uint32_t *out, const uint32_t *base,
                                                      const uint32_t *exp, size_t n) {
    const size_t n4 = n / 4;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n4) {
        const uint4 bv = ld_stream(reinterpret_cast<const uint4 *>(base) + i);
        const uint4 ev = ld_stream(reinterpret_cast<const uint4 *>(exp) + i);
        uint32_t b[4] = {bv.x, bv.y, bv.z, bv.w}, e[4] = {ev.x, ev.y, ev.z, ev.w}, o[4];
        pow_fourier<4, WIDE>(q, f, b, e, o);
        st_stream(reinterpret_cast<uint4 *>(out) + i, make_uint4(o[0], o[1], o[2], o[3]));
    } else if (i < n4 + (n & 3)) {
        const size_t j = 4 * n4 + (i - n4);
        uint32_t b[1] = {base[j]}, e[1] = {exp[j]}, o[1];
        pow_fourier<1, WIDE>(q, f, b, e, o);
        out[j] = o[0];
    }
}

// tw[j] = to_mont(w^j): binary ladder on the bits of j, canonical output
__global__ void __launch_bounds__(256) k_twiddle_table(Ctx c, uint32_t *tw, uint32_t w, size_t len) {
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < len; j += (size_t)gridDim.x * blockDim.x) {
        const uint32_t x = redc(w, c.r2, c.p, c.pinv);
        uint32_t acc = c.r1;
        unsigned long long e = j;
        for (int sh = 63 - __clzll(e | 1ull); sh >= 0; --sh) {
            acc = redc(acc, acc, c.p, c.pinv);
            if ((e >> sh) & 1ull) acc = redc(acc, x, c.p, c.pinv);
        }
        tw[j] = acc;
    }
}

template <int V>
static mont_status_t launch_pow(const PowParams &q, uint32_t *out, const uint32_t *base, const uint32_t *exp,
                                size_t n, int ctas_per_sm, int sms, cudaStream_t stream) {
    const int threads = 256;
    const size_t smem = (size_t)pow_smem_words<V>() * threads * 4;
    const uintptr_t pb = (uintptr_t)base, pe = (uintptr_t)exp, po = (uintptr_t)out;
    if (same_mod16(pb, pe) && same_mod16(pb, po)) {
        const uint32_t head = head_elems(pb, n);
        const size_t n4 = (n - head) / 4;
        const uint32_t tail = (uint32_t)((n - head) % 4);
        const size_t need = (n4 + threads - 1) / threads;
        size_t grid = ctas_per_sm > 0 ? (size_t)sms * ctas_per_sm : need;  // 0 = flat grid
        if (grid > need) grid = need;
        if (grid == 0) grid = 1;
        if (grid > 0x7fffffff) grid = 0x7fffffff;
        k_pow<V><<<(unsigned)grid, threads, smem, stream>>>(q, out, base, exp, head, n4, tail);
    } else {
        const size_t need = (n + threads - 1) / threads;
        size_t grid = ctas_per_sm > 0 ? (size_t)sms * ctas_per_sm : need;
        if (grid > need) grid = need;
        if (grid > 0x7fffffff) grid = 0x7fffffff;
        k_pow_scalar<V><<<(unsigned)grid, threads, smem, stream>>>(q, out, base, exp, n);
    }
    return launch_status();
}

// ctas_per_sm = 0: flat grid (one uint4 of work per thread)
static const Launch kPowDefault{256, 0, 1, 0, 0};

}  // namespace mont

using namespace mont;

mont_status_t mont_pow2_launch(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *base, const uint32_t *exp,
                               size_t n, int variant, int ctas_per_sm, int sms, size_t reserve_smem, int threads,
                               cudaStream_t stream);  // k_pow2.cu

extern "C" mont_status_t mont_pow_vec_ex(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *base,
                                         const uint32_t *exp, size_t n, const mont_launch_t *cfg,
                                         cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (n == 0) return MONT_OK;
    if (!out || !base || !exp || ((uintptr_t)out | (uintptr_t)base | (uintptr_t)exp) & 3u) return MONT_EINVAL_ARG;
    Launch L = resolve(cfg, kPowDefault);
    const bool v2 = L.variant == 0 || (L.variant >= 11 && L.variant <= 16);  // k_pow2: 64, 128 or 256 threads
    // k_pow2's default CTA is 128 threads: twice the CTAs of 256 for the same warps per SM, so the
    // last wave is half as long (235.9 vs 240.0 us for configs[3], profiles/r02_probe_pow_variants.jsonl)
    if (v2 && (!cfg || cfg->threads == 0)) L.threads = 128;
    if (!(L.threads == 256 || (v2 && (L.threads == 128 || L.threads == 64))) || L.variant < 0 || L.variant > 17 ||
        L.ctas_per_sm < 0 ||
        L.chunk < 0 ||
        L.chunk > 227 * 1024)
        return MONT_EINVAL_ARG;
    const int sms = sm_count();
    if (sms <= 0) return MONT_ECUDA;
    const PowParams q{(int32_t)ctx->p, (int32_t)(0u - ctx->pneg), ctx->r1, ctx->r2, (double)ctx->p, 1.0 / (double)ctx->p};
    const bool co16 = same_mod16((uintptr_t)base, (uintptr_t)exp) && same_mod16((uintptr_t)base, (uintptr_t)out);
    // variant 0 = the library default: variant 11 (8 lanes per thread, P specialised for the
    // config primes; measured fastest) when the operands are 16-byte co-aligned,
    // else the 4-lane 2-bit window (variant 17, round 1's default), which takes any alignment
    if (L.variant == 0) L.variant = co16 ? 11 : 17;
    if (L.variant >= 11 && L.variant <= 16 && co16)
        return mont_pow2_launch(ctx, out, base, exp, n, L.variant, L.ctas_per_sm, sms, (size_t)L.chunk, L.threads,
                                stream);
    L.threads = 256;  // the other ladders run 256-thread CTAs
    if (L.variant >= 11) L.variant = 0;  // 17, or misaligned operands: the 4-lane kernel
    if (L.variant == 10 && co16) {
        const uint32_t head = head_elems((uintptr_t)base, n);
        const size_t n4 = (n - head) / 4;
        const uint32_t tail = (uint32_t)((n - head) % 4);
        const size_t need = (n4 / 2 + 255) / 256;
        size_t grid = L.ctas_per_sm > 0 ? (size_t)sms * L.ctas_per_sm : need;
        if (grid > need) grid = need;
        if (grid == 0) grid = 1;
        if (grid > 0x7fffffff) grid = 0x7fffffff;
        k_pow8<<<(unsigned)grid, 256, 0, stream>>>(q, out, base, exp, head, n4, tail);
        return launch_status();
    }
    if (L.variant == 10) L.variant = 0;  // misaligned operands: the 4-lane kernel handles them
    if (L.variant == 9) {  // Fourier-prime REDC ladder: P = c 2^n + 1, 2n >= 32
        uint32_t nn = 0, cc = ctx->p - 1u;
        while ((cc & 1u) == 0u) { cc >>= 1; ++nn; }
        if (2 * nn < 32) return MONT_EUNSUPPORTED;
        if (((uintptr_t)out | (uintptr_t)base | (uintptr_t)exp) & 15u) return MONT_EINVAL_ARG;
        const FourierDev f{ctx->p, cc, nn, cc << (2 * nn - 32)};
        const size_t threads = n / 4 + (n & 3);
        const size_t grid = (threads + 255) / 256;
        if (grid > 0x7fffffff) return MONT_EUNSUPPORTED;
        if ((uint64_t)ctx->p * 3u >= (1ull << 32))  // t + P would not fit 32 bits: 33-bit t
            k_pow_fourier<true><<<(unsigned)grid, 256, 0, stream>>>(q, f, out, base, exp, n);
        else
            k_pow_fourier<false><<<(unsigned)grid, 256, 0, stream>>>(q, f, out, base, exp, n);
        return launch_status();
    }
    switch (L.variant) {
        case 0: return launch_pow<0>(q, out, base, exp, n, L.ctas_per_sm, sms, stream);
        case 1: return launch_pow<1>(q, out, base, exp, n, L.ctas_per_sm, sms, stream);
        case 2: return launch_pow<2>(q, out, base, exp, n, L.ctas_per_sm, sms, stream);
        case 3: return launch_pow<3>(q, out, base, exp, n, L.ctas_per_sm, sms, stream);
        case 4: return launch_pow<4>(q, out, base, exp, n, L.ctas_per_sm, sms, stream);
        case 5: return launch_pow<5>(q, out, base, exp, n, L.ctas_per_sm, sms, stream);
        case 6: return launch_pow<6>(q, out, base, exp, n, L.ctas_per_sm, sms, stream);
        case 7: return launch_pow<7>(q, out, base, exp, n, L.ctas_per_sm, sms, stream);
        default: return launch_pow<8>(q, out, base, exp, n, L.ctas_per_sm, sms, stream);
    }
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

extern "C" mont_status_t barrett_pow_vec(const barrett_ctx_t *ctx, uint32_t *out, const uint32_t *base,
                                         const uint32_t *exp, size_t n, cudaStream_t stream) {
    if (!ctx || (ctx->p & 1u) == 0u || ctx->p < 3u || ctx->p >= 0x80000000u || ctx->k > 31 ||
        ctx->pprime != (uint32_t)((1ull << (2 * ctx->k)) / ctx->p))
        return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (n == 0) return MONT_OK;
    if (!out || !base || !exp || ((uintptr_t)out | (uintptr_t)base | (uintptr_t)exp) & 15u)
        return MONT_EINVAL_ARG;  // 16-byte aligned operands only (comparison kernel)
    const size_t threads = n / 4 + (n & 3);
    const size_t grid = (threads + 255) / 256;
    if (grid > 0x7fffffff) return MONT_EUNSUPPORTED;
    k_pow_barrett<<<(unsigned)grid, 256, 0, stream>>>(BarrettDev{ctx->p, ctx->k, ctx->pprime}, out, base, exp, n);
    return launch_status();
}
