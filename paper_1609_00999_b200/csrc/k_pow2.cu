// k_pow2.cu -- round-2 K3 ladders for mont_pow_vec_ex variants 11-16 (include/mont_ext.h):
// out[i] = base[i]^exp[i] mod P, plain in / plain out (BASELINE configs[3], G10).
//
// Same left-to-right 2-bit fixed window as k_pow.cu variant 0 (every lane executes 2 table
// products + 15 windows of 2 squarings and 1 multiply, selects on the ALU pipe), with three
// B200-specific changes measured by mb_pipe (csrc/k_pipes.cu, profiles/r02_pipes*.jsonl):
//   * modulus specialisation: for the three config primes the kernel is instantiated with P
//     as a compile-time constant (the paper's generator emits code per modulus, §4),
//     so P and P^-1 are instruction immediates (IMAD R, R, imm) instead of uniform-register
//     operands; any other odd P < 2^31 runs the same code with P at run time;
//   * precomputed-quotient (Shoup) window multiplies (variants 13, 14, 16): the multiplier
//     x^d of each window is fixed per element, so with w' = floor(w 2^32 / P) the product is
//     q = hi(a w'), r = a w - q P (low words) in [0, 2P): IMAD.HI + 2 IMAD = 8 FMAHeavy
//     cycles per warp instead of REDC's 10.  w' needs no division: w 2^32 = w' P + w-bar gives
//     w' = w-bar * P' mod 2^32 (P' = -P^-1), one IMAD from the Montgomery form the table
//     already holds, and w = hi(w' P) + [w-bar != 0];
//   * FP64 lanes (variants 12, 14): 2 of each thread's 8 lanes run the same ladder as FP64
//     Barrett products (mont_core.cuh fmulmod) on the DFMA pipe, interleaved instruction by
//     instruction with the integer lanes (few chains per thread so ptxas interleaves them).
// Values: the squarings are signed lazy REDCs in (-P, P) (mont_core.cuh sredc); the second
// squaring of a window adds P in its final IADD3 (free) so the Shoup multiply sees a
// non-negative a < 2P; Shoup returns [0, 2P), which the next squaring accepts when 4P^2 <
// 2^31 P, i.e. P < 2^29 (P1 = 469762049); for larger P one min-subtract canonicalises it.
#include <cuda_runtime.h>
#include <stdint.h>

#include "abi_util.h"

namespace mont {

struct Pow2Params {
    int32_t p, pinv;    // pinv = P^-1 mod 2^32
    uint32_t r1, r2;    // R mod P, R^2 mod P
    uint32_t pneg;      // P' = -P^-1 mod 2^32
    uint32_t pad;
    double pd, pdinv;   // P and fl(1/P) for the FP64 lanes
};

__host__ __device__ constexpr uint32_t inv32(uint32_t p) {
    uint32_t x = p;  // p * p = 1 mod 8: 3 correct bits, doubling per Newton step
    for (int i = 0; i < 5; ++i) x *= 2u - p * x;
    return x;
}

template <uint32_t PC>
__device__ __forceinline__ Pow2Params fix(const Pow2Params &q) {
    if constexpr (PC == 0) {
        return q;
    } else {
        constexpr uint32_t pinv = inv32(PC);
        constexpr uint32_t r1 = (uint32_t)((1ull << 32) % PC);
        constexpr uint32_t r2 = (uint32_t)(((uint64_t)r1 * r1) % PC);
        return Pow2Params{(int32_t)PC, (int32_t)pinv, r1, r2, 0u - pinv, 0u, (double)PC, 1.0 / (double)PC};
    }
}

// signed lazy REDC returning t + P in (0, 2P): the paper's t before its
// correction, for a non-negative Shoup operand
__device__ __forceinline__ uint32_t sredc_pp(int32_t a, int32_t b, int32_t p, int32_t pinv) {
    const int64_t T = mul_wide_s32(a, b);
    const int32_t m = (int32_t)T * pinv;
    return (uint32_t)(hi32s(T) - hi32s(mul_wide_s32(m, p)) + p);
}

// Shoup product a w mod P for a < 2^32, w < P, wq = floor(w 2^32 / P): result in [0, 2P)
__device__ __forceinline__ uint32_t shoup(uint32_t a, uint32_t w, uint32_t wq, uint32_t p) {
    const uint32_t q = __umulhi(a, wq);
    return a * w - q * p;
}

template <uint32_t PC, int L, int NF, bool SH, bool BIGP>
__device__ __forceinline__ void pow2_lanes(const Pow2Params &q0, const uint32_t (&base)[L], const uint32_t (&e)[L],
                                           uint32_t (&out)[L]) {
    const Pow2Params q = fix<PC>(q0);
    constexpr int NI = L - NF;
    // integer lanes: table t[d] = x-bar^d (canonical), Shoup pairs (w, w') when SH
    int32_t ti[NI][4];
    uint32_t tw[SH ? NI : 1][4], tq[SH ? NI : 1][4];
    int32_t ai[NI];
    double tf[NF > 0 ? NF : 1][4], af[NF > 0 ? NF : 1];
#pragma unroll
    for (int l = 0; l < (NI > NF ? NI : NF); ++l) {
        if (l < NI) {
            const uint32_t x = redc(base[l], q.r2, (uint32_t)q.p, (uint32_t)q.pinv);  // to_mont, canonical
            ti[l][0] = (int32_t)q.r1;
            ti[l][1] = (int32_t)x;
            ti[l][2] = (int32_t)canon(sredc((int32_t)x, (int32_t)x, q.p, q.pinv), q.p);
            ti[l][3] = (int32_t)canon(sredc(ti[l][2], (int32_t)x, q.p, q.pinv), q.p);
            if (SH) {
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const uint32_t wb = (uint32_t)ti[l][d];
                    tq[l][d] = wb * q.pneg;                                      // floor(w 2^32 / P)
                    tw[l][d] = __umulhi(tq[l][d], (uint32_t)q.p) + (wb != 0u);    // w = x^d mod P
                }
            }
            const uint32_t d0 = e[l] >> 30;
            const int32_t lo = (d0 & 1u) ? ti[l][1] : ti[l][0];
            const int32_t hi = (d0 & 1u) ? ti[l][3] : ti[l][2];
            ai[l] = (d0 & 2u) ? hi : lo;
        }
        if (l < NF) {
            const double x = fmulmod((double)base[NI + l], 1.0, q.pd, q.pdinv);  // base mod P in (-P/2, P/2]
            tf[l][0] = 1.0;
            tf[l][1] = x;
            tf[l][2] = fmulmod(x, x, q.pd, q.pdinv);
            tf[l][3] = fmulmod(tf[l][2], x, q.pd, q.pdinv);
            const uint32_t d0 = e[NI + l] >> 30;
            const double lo = (d0 & 1u) ? tf[l][1] : tf[l][0];
            const double hi = (d0 & 1u) ? tf[l][3] : tf[l][2];
            af[l] = (d0 & 2u) ? hi : lo;
        }
    }
#pragma unroll
    for (int sh = 28; sh >= 0; sh -= 2) {
#pragma unroll
        for (int l = 0; l < (NI > NF ? NI : NF); ++l) {
            if (l < NI) {
                const uint32_t d = (e[l] >> sh) & 3u;
                const int32_t a1 = sredc(ai[l], ai[l], q.p, q.pinv);
                if (SH) {
                    const uint32_t a2 = sredc_pp(a1, a1, q.p, q.pinv);  // (0, 2P)
                    const uint32_t wlo = (d & 1u) ? tw[l][1] : tw[l][0], whi = (d & 1u) ? tw[l][3] : tw[l][2];
                    const uint32_t qlo = (d & 1u) ? tq[l][1] : tq[l][0], qhi = (d & 1u) ? tq[l][3] : tq[l][2];
                    uint32_t r = shoup(a2, (d & 2u) ? whi : wlo, (d & 2u) ? qhi : qlo, (uint32_t)q.p);  // [0, 2P)
                    if (BIGP) r = umin(r, r - (uint32_t)q.p);
                    ai[l] = (int32_t)r;
                } else {
                    const int32_t a2 = sredc(a1, a1, q.p, q.pinv);
                    const int32_t lo = (d & 1u) ? ti[l][1] : ti[l][0];
                    const int32_t hi = (d & 1u) ? ti[l][3] : ti[l][2];
                    ai[l] = sredc(a2, (d & 2u) ? hi : lo, q.p, q.pinv);
                }
            }
            if (l < NF) {
                double a = fmulmod(af[l], af[l], q.pd, q.pdinv);
                a = fmulmod(a, a, q.pd, q.pdinv);
                const uint32_t d = (e[NI + l] >> sh) & 3u;
                const double lo = (d & 1u) ? tf[l][1] : tf[l][0];
                const double hi = (d & 1u) ? tf[l][3] : tf[l][2];
                af[l] = fmulmod(a, (d & 2u) ? hi : lo, q.pd, q.pdinv);
            }
        }
    }
#pragma unroll
    for (int l = 0; l < NI; ++l) out[l] = canon(sredc1(ai[l], q.p, q.pinv), q.p);  // from_mont
#pragma unroll
    for (int l = 0; l < NF; ++l) {
        const double r = af[l] < 0.0 ? af[l] + q.pd : af[l];
        out[NI + l] = (uint32_t)__double2uint_rn(r);
    }
}

// 8 lanes per thread (two uint4 of base / exp); head, tail and an odd last uint4 run one lane per
// thread of CTA 0 / the last CTA through the runtime-P integer ladder.  ctas_per_sm > 0: a
// persistent grid-stride grid, else one 8-lane item per thread (flat grid).
template <uint32_t PC, int NF, bool SH, bool BIGP>
__global__ void __launch_bounds__(256) k_pow2(Pow2Params q, uint32_t *out, const uint32_t *base, const uint32_t *exp,
                                               uint32_t head, size_t n4, uint32_t tail) {
    if (blockIdx.x == 0 && threadIdx.x < head + tail) {
        const size_t i = threadIdx.x < head ? threadIdx.x : head + 4 * n4 + (threadIdx.x - head);
        uint32_t b[1] = {base[i]}, e[1] = {exp[i]}, o[1];
        pow2_lanes<PC, 1, 0, SH, BIGP>(q, b, e, o);
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
        pow2_lanes<PC, 8, NF, SH, BIGP>(q, b, e, o);
        st_stream(o4 + 2 * i, make_uint4(o[0], o[1], o[2], o[3]));
        st_stream(o4 + 2 * i + 1, make_uint4(o[4], o[5], o[6], o[7]));
    }
    if ((n4 & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x < 4) {  // odd last uint4: 4 threads x 1 lane
        const size_t j = head + 4 * (n4 - 1) + threadIdx.x;
        uint32_t b[1] = {base[j]}, e[1] = {exp[j]}, o[1];
        pow2_lanes<PC, 1, 0, SH, BIGP>(q, b, e, o);
        out[j] = o[0];
    }
}

template <uint32_t PC, int NF, bool SH, bool BIGP>
static void launch_pow2(const Pow2Params &q, uint32_t *out, const uint32_t *base, const uint32_t *exp, uint32_t head,
                        size_t n4, uint32_t tail, unsigned grid, size_t smem, int threads, cudaStream_t s) {
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_pow2<PC, NF, SH, BIGP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_pow2<PC, NF, SH, BIGP><<<grid, threads, smem, s>>>(q, out, base, exp, head, n4, tail);
}

template <int NF, bool SH, bool BIGP>
static void dispatch_p(uint32_t p, bool specialise, const Pow2Params &q, uint32_t *out, const uint32_t *base,
                       const uint32_t *exp, uint32_t head, size_t n4, uint32_t tail, unsigned grid, size_t smem,
                       int threads, cudaStream_t s) {
    if (specialise && p == 469762049u && !BIGP)
        launch_pow2<469762049u, NF, SH, false>(q, out, base, exp, head, n4, tail, grid, smem, threads, s);
    else if (specialise && p == 998244353u && BIGP)
        launch_pow2<998244353u, NF, SH, true>(q, out, base, exp, head, n4, tail, grid, smem, threads, s);
    else if (specialise && p == 2013265921u && BIGP)
        launch_pow2<2013265921u, NF, SH, true>(q, out, base, exp, head, n4, tail, grid, smem, threads, s);
    else
        launch_pow2<0u, NF, SH, BIGP>(q, out, base, exp, head, n4, tail, grid, smem, threads, s);
}

}  // namespace mont

using namespace mont;

// Called by mont_pow_vec_ex (k_pow.cu) for variants 11-16 with 16-byte co-aligned operands.
//   11: REDC multiplies, P specialised for the config primes   12: 11 + 2 of 8 lanes on FP64
//   13: Shoup multiplies, specialised                          14: 13 + 2 FP64 lanes
//   15: 11 with P at run time (no specialisation)              16: 13 with P at run time
// reserve_smem: dynamic shared memory requested per CTA and never touched -- an occupancy cap
// (e.g. 100 KiB: at most 2 pow CTAs per SM), so that a flat pow grid co-running with the
// HBM-bound launches keeps taking only a few CTA slots per SM while the block scheduler still
// balances it dynamically (bench.py's two-lane step)
mont_status_t mont_pow2_launch(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *base, const uint32_t *exp,
                               size_t n, int variant, int ctas_per_sm, int sms, size_t reserve_smem,
                               int threads, cudaStream_t stream) {
    const uint32_t p = ctx->p;
    const Pow2Params q{(int32_t)p, (int32_t)(0u - ctx->pneg), ctx->r1, ctx->r2, ctx->pneg, 0u, (double)p,
                       1.0 / (double)p};
    const uint32_t head = head_elems((uintptr_t)base, n);
    const size_t n4 = (n - head) / 4;
    const uint32_t tail = (uint32_t)((n - head) % 4);
    const size_t need = (n4 / 2 + threads - 1) / threads;
    size_t grid = ctas_per_sm > 0 ? (size_t)sms * ctas_per_sm : need;
    if (grid > need) grid = need;
    if (grid == 0) grid = 1;
    if (grid > 0x7fffffff) grid = 0x7fffffff;
    const bool bigp = p >= (1u << 29);  // Shoup outputs in [0, 2P) feed a squaring only if P < 2^29
    const bool spec = variant <= 14;
    const int v = variant == 15 ? 11 : variant == 16 ? 13 : variant;
    const unsigned g = (unsigned)grid;
#define P2(NF, SH)                                                                                \
    do {                                                                                          \
        if (bigp) dispatch_p<NF, SH, true>(p, spec, q, out, base, exp, head, n4, tail, g, reserve_smem, threads, stream); \
        else dispatch_p<NF, SH, false>(p, spec, q, out, base, exp, head, n4, tail, g, reserve_smem, threads, stream);     \
    } while (0)
    switch (v) {
        case 11: P2(0, false); break;
        case 12: P2(2, false); break;
        case 13: P2(0, true); break;
        default: P2(2, true); break;
    }
#undef P2
    return launch_status();
}
