// mont_core.cuh -- device-side Montgomery REDC for R = 2^32 on sm_100a.
//
// PAPER.md Alg. 2 (REDC, :95-99) with the GPU refinement of the §3.2 dataflow
// (:121-139): the paper gathers high and low 32-bit halves of 2-way 64-bit
// products with shuffles because SSE has no high-half multiply; sm_100a has
// one (mul.hi.u32 -> IMAD.HI) and a 32x32->64 multiply (mul.wide.u32 ->
// IMAD.WIDE), so the three integer multiplications become three
// FMAHeavy-pipe instructions (two of them half rate, below) and no gather
// exists.  The textbook add form reads:
//
//   T  = a*b                 mul.lo + mul.hi       (A3, "needs twice the width", :123)
//   m  = lo(T) * P' mod 2^32 mul.lo                (A4, the "short product", :93, :129)
//   t  = (T + m P) / 2^32    mul.hi + carry        (A5, the "2-way addition ... carries", :137)
//   t >= P ? t - P : t       min(t, t - P)         (A6, "selectively subtracting P", :139)
//
// The low half of m*P is never formed: lo(T) + lo(mP) = 0 (mod 2^32) by the
// choice of m, so the carry into the high word is exactly [lo(T) != 0].
// With P < 2^31 and a*b < R*P the pre-subtract t lies in [0, 2P)
// and fits 32 bits, so min(t, t-P) on unsigned words is the single conditional
// subtract.
//
// A second, "signed" form (used by the pow ladder) keeps values in the open
// interval (-P, P) as int32 and needs no correction between products:
//   m = lo(T) * P^-1 mod 2^32 ; t = (T - m P) / 2^32   (exact, arithmetic shift)
// T - mP = 0 (mod 2^32) exactly, and |t| <= (|T| + 2^31 P) / 2^32 < P whenever
// |a*b| < 2^31 P, which holds for |a|, |b| < P < 2^31.  It differs from the
// paper's P' only in sign (P^-1 = -P'), reading G2.
#pragma once
#include <stdint.h>

namespace mont {

struct Ctx {  // device view of mont_ctx_t (by value in kernel params); pinv = -pneg
    uint32_t p, pinv, r1, r2;
};

__device__ __forceinline__ uint32_t umin(uint32_t x, uint32_t y) { return x < y ? x : y; }

// Programmatic dependent launch (mont_launch_t.flags & MONT_LAUNCH_OVERLAP_PREV): a kernel lets the
// next overlap-flagged launch on its stream start as soon as all of its CTAs are running
// (pdl_trigger, at the top), and waits at its very end for the launch before it to complete
// (pdl_wait), so that its own completion still implies its predecessor's -- stream order holds for
// everything launched after it.  Both are no-ops for a launch without the attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// 32 x 32 -> 64 products (IMAD.WIDE): both halves of the paper's "2l-bit" product
// in one register pair.  (A 64-bit addend is not fused: ptxas splits mad.wide with a
// register-pair addend into IMAD.WIDE + IADD3 + IADD3.X, so the carry form of Alg. 2 costs ALU
// ops the subtract form below does not.)
__device__ __forceinline__ uint64_t mul_wide_u32(uint32_t a, uint32_t b) {
    uint64_t r;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ int64_t mul_wide_s32(int32_t a, int32_t b) {
    int64_t r;
    asm("mul.wide.s32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t hi32(uint64_t x) { return (uint32_t)(x >> 32); }
__device__ __forceinline__ int32_t hi32s(int64_t x) { return (int32_t)(x >> 32); }

// Measured on B200 with dependent chains nothing can hoist (mb_pipe, csrc/k_pipes.cu;
// profiles/r02_pipes.jsonl): IMAD issues at 64 lanes/clk/SM (register, immediate
// or uniform-register operand alike), IMAD.WIDE at 32 (half rate), IMAD.HI at 32 (~26 when
// all three sources are registers: mad.hi with a register addend).  So the high halves are taken from
// IMAD.WIDE results, never from mul.hi, and the REDC is written in the "subtract" form, which
// needs no carry:
//   T = a b (IMAD.WIDE);  m = lo(T) P^-1 mod 2^32 (IMAD);  M = m P (IMAD.WIDE)
//   lo(M) = lo(T) exactly, so (T - M) / 2^32 = hi(T) - hi(M)  (IADD3), in (-P, P)
// = 4 + 2 + 4 = 10 FMAHeavy cycles per warp on an SMSP ("5 issue slots" of the 64-lane IMAD
// rate) + 1 ALU op.  It is Alg. 2 with m' = -m:
// t' = (T - m'P)/R = (T + mP)/R - P, i.e. the paper's t shifted by -P, so the
// final "if t >= P then t - P" becomes "if t' < 0 then t' + P".
// pinv = P^-1 mod 2^32 = -P' (reading G2).

// canonical REDC: a*b < 2^32 P required; returns [0, P).  2 ALU ops
// (IADD3 + VIADDMNMX for the sign fix-up).
__device__ __forceinline__ uint32_t redc(uint32_t a, uint32_t b, uint32_t p, uint32_t pinv) {
    const uint64_t T = mul_wide_u32(a, b);
    const uint32_t m = (uint32_t)T * pinv;
    const uint64_t M = mul_wide_u32(m, p);
    const uint32_t t = hi32(T) - hi32(M);  // in (-P, P) as a signed value
    return umin(t, t + p);                 // t < 0 (wrapped) -> t + P
}

// REDC(x * 1) = x R^-1 mod P (A10): T = x, hi(T) = 0, so t = -hi(m P) and the canonical value
// is P - hi(m P), or 0 when hi(m P) = 0.  Written as a select, not as min(t, t + P): for that
// form NVVM emits neg / sub / min.u32, and ptxas 12.9 fused it in one kernel (k_run) into a
// VIADDMNMX that added +hi instead of -hi (wrong results; tests/test_gpu_run.py caught it).
__device__ __forceinline__ uint32_t redc1(uint32_t x, uint32_t p, uint32_t pinv) {
    const uint32_t m = x * pinv;
    const uint32_t h = hi32(mul_wide_u32(m, p));
    return h ? p - h : 0u;
}

// signed lazy form for chains: |a|, |b| < P  ->  result in (-P, P),
// congruent to a b R^-1 (mod P).  |T - M| < 2^31 P + 2^31 P, so |t| < P.
__device__ __forceinline__ int32_t sredc(int32_t a, int32_t b, int32_t p, int32_t pinv) {
    const int64_t T = mul_wide_s32(a, b);
    const int32_t m = (int32_t)T * pinv;
    return hi32s(T) - hi32s(mul_wide_s32(m, p));
}

// signed REDC(x * 1) for |x| < P -> (-P, P)
__device__ __forceinline__ int32_t sredc1(int32_t x, int32_t p, int32_t pinv) {
    const int32_t m = x * pinv;
    return (x >> 31) - hi32s(mul_wide_s32(m, p));
}

// Reference forms kept for the K8 microbenchmark only (k_micro.cu):
// mul.hi-based (IMAD.HI, half rate) and the IMAD.HI-with-64-bit-addend form.
__device__ __forceinline__ int32_t sredc_mulhi(int32_t a, int32_t b, int32_t p, int32_t pinv) {
    int32_t lo = a * b;
    int32_t hi = __mulhi(a, b);
    int32_t m = lo * pinv;
    return hi - __mulhi(m, p);
}
__device__ __forceinline__ int32_t sredc_hiadd(int32_t a, int32_t b, int32_t negp, int32_t pinv) {
    const int64_t T = mul_wide_s32(a, b);
    const int32_t m = (int32_t)T * pinv;
    return (int32_t)(((int64_t)m * negp + T) >> 32);
}

// (-P, P) -> [0, P)
__device__ __forceinline__ uint32_t canon(int32_t t, int32_t p) {
    uint32_t u = (uint32_t)t;
    return umin(u, u + (uint32_t)p);
}

// streaming 128-bit loads / stores: read-only path, no L1 allocation, 256B L2
// prefetch hint; stores evict-first (each byte is touched exactly once)
__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream(uint4 *p, const uint4 &v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint32_t ld_stream1(const uint32_t *p) {
    uint32_t r;
    asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream1(uint32_t *p, uint32_t v) {
    asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace mont

namespace mont {

// ---- FP64 reduction (Barrett, Alg. 1, with a floating
// reciprocal instead of the integer P' = floor(2^2k / P)).  Plain residues
// held as doubles in (-P, P):
//   h = fl(a b); l = fma(a, b, -h)       a b = h + l exactly (FMA error term)
//   q = rint(h / P)                       fma(h, 1/P, 1.5*2^52) - 1.5*2^52
//   r = fma(-q, P, h) + l                 = a b - q P exactly (|.| < 2^53)
// |a b / P - q| <= 1/2 + 2^-21, so |r| < P(1/2 + 2^-21): the chain needs no
// correction.  6 FP64-pipe instructions, no integer pipe use: this is the
// second multiplier array of the SM, idle in the IMAD-only ladder.
__device__ __forceinline__ double fmulmod(double a, double b, double P, double Pinv) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    const double h = a * b;
    const double l = fma(a, b, -h);
    const double q = fma(h, Pinv, M) - M;
    return fma(-q, P, h) + l;
}

}  // namespace mont

namespace mont {

// ---- Barrett (Alg. 1, :71-85) for the comparison kernels of
// include/barrett.h.  ab < P^2 < 2^(2k); m < 2^k; m P' < 2^63; t = ab - qP < 4P
// (PAPER.md:85), which can exceed 2^32 for P > 2^30, so t is 64-bit until the
// first correction.
struct BarrettDev {
    uint32_t p, k, pp;
};

__device__ __forceinline__ uint32_t barrett(uint32_t a, uint32_t b, const BarrettDev &c) {
    const uint64_t T = mul_wide_u32(a, b);
    const uint32_t m = (uint32_t)(T >> c.k);                           // floor(ab / 2^k)
    const uint32_t q = (uint32_t)(mul_wide_u32(m, c.pp) >> c.k);       // floor(m P' / 2^k)
    uint64_t t = T - mul_wide_u32(q, c.p);                             // < 4P
    const uint64_t t2 = t - 2ull * c.p;
    t = (int64_t)t2 >= 0 ? t2 : t;                                     // < 2P
    const uint32_t r = (uint32_t)t;
    return umin(r, r - c.p);                                           // < P
}

}  // namespace mont

namespace mont {

// ---- Fourier-prime REDC (Alg. 3, :105-117)
// for P = c 2^n + 1 with 2n >= 32 (all three config primes), R = 2^32:
//   q1 = T >> 32, r1 = T mod R, q2 = c 2^n r1 / R, r2 = c 2^n r1 mod R,
//   q3 = c 2^n r2 / R (r3 = 0, :117), t = q1 - q2 + q3 in [-(P-1), 2(P-1)].
// With u = c r1: q2 = u >> (32-n), r2 = (u mod 2^(32-n)) << n, and
// q3 = c (u mod 2^(32-n)) 2^(2n-32) exactly.  Here t + P is formed directly
// (the +P folded into the q3 multiply-add) and lies in [1, 3P-1]; two unsigned
// min-subtracts canonicalise, replacing the paper's three sign-mask steps (:108).
// Requires 3P < 2^32 (P < 2^30.58); canonical inputs.  Cost on B200: IMAD.WIDE
// (T) + IMAD.WIDE (u) + IMAD (q3) = 5 FMAHeavy slots, as many as Montgomery,
// plus 5 ALU ops -- measured in k_pow variant 9.
struct FourierDev {
    uint32_t p, c, n, c_sh;  // c_sh = c << (2n - 32)
};

__device__ __forceinline__ uint32_t fredc(uint32_t a, uint32_t b, const FourierDev &f) {
    const uint64_t T = mul_wide_u32(a, b);
    const uint32_t q1 = hi32(T), r1 = (uint32_t)T;
    const uint64_t u = mul_wide_u32(r1, f.c);
    const uint32_t q2 = (uint32_t)(u >> (32 - f.n));
    const uint32_t v = (uint32_t)u & ((1u << (32 - f.n)) - 1u);
    const uint32_t q3p = v * f.c_sh + f.p;      // q3 + P
    uint32_t t = q1 - q2 + q3p;                  // t + P in [1, 3P-1]
    t = umin(t, t - f.p);
    return umin(t, t - f.p);
}

// The same Alg. 3 product for any P = c 2^n + 1 < 2^31 with 2n >= 32, including 3P >= 2^32
// (P0 = 15 2^27 + 1), where t = q1 - q2 + q3 in [-(P-1), 2(P-1)] spans more than
// 2^32 values: t is held as a 33-bit quantity, the non-negative part s = q1 + q3 in [0, 2P)
// (q1 = hi(ab) < P, q3 = c v 2^(2n-32) < c 2^n < P) and the sign of s - q2 (DESIGN.md reading
// G8: the paper's 32-bit signed t with the mask step t + (t >> 31) & P is
// wrong for P > 2^30).  s < q2: t = s - q2 in (-P, 0), canonical t + P; else t in [0, 2P),
// one conditional subtract.
__device__ __forceinline__ uint32_t fredc33(uint32_t a, uint32_t b, const FourierDev &f) {
    const uint64_t T = mul_wide_u32(a, b);
    const uint32_t q1 = hi32(T), r1 = (uint32_t)T;
    const uint64_t u = mul_wide_u32(r1, f.c);
    const uint32_t q2 = (uint32_t)(u >> (32 - f.n));
    const uint32_t v = (uint32_t)u & ((1u << (32 - f.n)) - 1u);
    const uint32_t s = q1 + v * f.c_sh;          // q1 + q3 in [0, 2P)
    const uint32_t d = s - q2;                   // t mod 2^32
    return s < q2 ? d + f.p : umin(d, d - f.p);
}

}  // namespace mont

namespace mont {

// ---- Alg. 3 for P1 = 7 * 2^26 + 1 with the multiplications by c = 7 written as shifts and
// subtracts in PTX (so neither NVVM nor ptxas turns them back into IMADs): one IMAD.WIDE (a b)
// on the FMAHeavy pipe, everything else on the ALU.  Canonical in and out.  Exploratory: the
// K8 microbenchmark measures it alone and in a lane mix with the Montgomery chain.
__device__ __forceinline__ uint32_t fredc_p1(uint32_t a, uint32_t b, uint32_t p) {
    const uint64_t T = mul_wide_u32(a, b);
    const uint32_t q1 = hi32(T), r1 = (uint32_t)T;
    uint32_t q2, v;
    // u = 7 r1 = (r1 << 3) - r1 (35 bits); q2 = u >> 6; v = u mod 64
    asm("{\n\t.reg .u32 s, lo, hi;\n\t"
        "shl.b32 s, %2, 3;\n\t"
        "sub.cc.u32 lo, s, %2;\n\t"
        "shr.u32 hi, %2, 29;\n\t"
        "subc.u32 hi, hi, 0;\n\t"
        "shf.r.clamp.b32 %0, lo, hi, 6;\n\t"
        "and.b32 %1, lo, 63;\n\t}"
        : "=r"(q2), "=r"(v)
        : "r"(r1));
    uint32_t q3p;  // 7 v 2^20 + P = (v << 23) - (v << 20) + P
    asm("{\n\t.reg .u32 x, y;\n\t"
        "shl.b32 x, %1, 23;\n\t"
        "shl.b32 y, %1, 20;\n\t"
        "sub.u32 x, x, y;\n\t"
        "add.u32 %0, x, %2;\n\t}"
        : "=r"(q3p)
        : "r"(v), "r"(p));
    uint32_t t = q1 - q2 + q3p;  // t + P in [1, 3P - 1]
    t = umin(t, t - p);
    return umin(t, t - p);
}

}  // namespace mont
