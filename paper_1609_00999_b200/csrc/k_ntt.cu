// k_ntt.cu -- batched radix-2 NTT with Montgomery twiddle products
// (include/mont_ntt.h).
//
// Every row is read from and written to HBM once -- 8 B of traffic per element
// and (N/2) log_n twiddle products per row.  Kernels:
//   k_ntt_dif  (default) decimation in frequency, 32 elements per thread, five
//              stages per trip through shared memory, padded additive layout
//              (the bit reversal happens in the last trip's stores);
//   k_ntt_r32  decimation in time, XOR-swizzled layout (variant 1);
//   k_ntt_smem one butterfly per thread per stage, the reference (variant 2);
//   k_ntt_col  the large transform's column pass (8 columns per CTA);
// plus the twiddle-table builders and the transpose of the large transform.
// Twiddles come from the caller's table through the read-only path (L1-resident
// across the CTAs of an SM).  The butterfly multiplies a PLAIN residue by a
// Montgomery-form twiddle, so REDC(v, w-bar) = v w mod P stays plain
// (REDC(x-bar, y-bar) of two residues is the residue of xy; one
// plain operand makes the product plain); variant 3 instead multiplies by the
// plain twiddle with its precomputed quotient (Shoup).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "../../include/mont_ntt.h"
#include "abi_util.h"
#include "tma.cuh"

namespace mont {

__device__ __forceinline__ uint32_t mod_add(uint32_t a, uint32_t b, uint32_t p) {
    const uint32_t r = a + b;  // < 2P < 2^32
    return umin(r, r - p);
}
__device__ __forceinline__ uint32_t mod_sub(uint32_t a, uint32_t b, uint32_t p) {
    const uint32_t r = a - b;  // wraps when a < b
    return umin(r, r + p);
}

__global__ void __launch_bounds__(1024) k_ntt_smem(Ctx c, uint32_t *data, int log_n, const uint32_t *__restrict__ tw,
                                                    uint32_t scale) {
    extern __shared__ uint32_t s[];
    const uint32_t N = 1u << log_n, half_n = N >> 1;
    uint32_t *row = data + (size_t)blockIdx.x * N;
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) s[__brev(i) >> (32 - log_n)] = row[i];
    __syncthreads();
    for (int st = 1; st <= log_n; ++st) {
        const uint32_t hmask = (1u << (st - 1)) - 1u;
        for (uint32_t t = threadIdx.x; t < half_n; t += blockDim.x) {
            const uint32_t pos = t & hmask;
            const uint32_t i = ((t >> (st - 1)) << st) | pos;
            const uint32_t j = i + hmask + 1u;
            const uint32_t v = redc(s[j], __ldg(tw + hmask + pos), c.p, c.pinv);
            const uint32_t u = s[i];
            s[i] = mod_add(u, v, c.p);
            s[j] = mod_sub(u, v, c.p);
        }
        __syncthreads();
    }
    if (scale == c.r1) {
        for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) row[i] = s[i];
    } else {
        for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) row[i] = redc(s[i], scale, c.p, c.pinv);
    }
}

// ---- register-blocked radix-2 NTT: 32 elements per thread, 5 stages per
// trip through shared memory.
//
// Thread t of a row owns, in trip g, the 32 elements whose index bits
// [ws, ws+5) vary and whose other bits are fixed by t (ws = min(5g, log_n-5));
// the 5 butterfly stages whose pair distance is one of those bits run entirely
// in registers, so a row of N = 2^log_n crosses shared memory only
// ceil(log_n / 5) + 1 times instead of log_n.  Shared memory addresses are
// XOR-swizzled, a ^ (((a >> 5) ^ (a >> 10)) & 31): a bijection on [0, 2^15)
// that makes every access pattern used here (coalesced natural order, the
// bit-reversed scatter of the load, and each trip's gather) bank-conflict free
// (checked exhaustively for log_n = 10..15 offline; scripts/ntt_swizzle.py).
__device__ __forceinline__ uint32_t swz(uint32_t a) { return a ^ (((a >> 5) ^ (a >> 10)) & 31u); }

// optional 2-D twiddle epilogue of the six-step large transform: element
// (row, idx) is multiplied by w^(row * idx mod N) = lo[e mod 2^shift] * hi[e >> shift]
struct Tw2D {
    const uint32_t *lo, *hi;
    uint64_t mask;      // N - 1 of the large transform
    uint32_t lomask;    // 2^shift - 1
    int shift;
    size_t row0;        // global index of row 0 of this launch
};

// LOG_N is a template parameter so every shift, window position and twiddle
// stride is a compile-time constant.  Because the swizzle is linear over
// GF(2) and the per-thread bits and the per-k bits of an index are disjoint,
// swz(base | k << ws) = swz(base) ^ swz(k << ws): one LOP3 per shared-memory
// access, and twiddle addresses become (per-thread base) + (constant offset).
template <int LOG_N>
__global__ void __launch_bounds__(LOG_N == 15 ? 1024 : 512, LOG_N == 15 ? 1 : 2)
    k_ntt_r32(Ctx c, uint32_t *data, size_t batch, const uint32_t *__restrict__ tw, uint32_t scale, Tw2D t2) {
    constexpr uint32_t N = 1u << LOG_N, T = N >> 5;
    extern __shared__ uint32_t sm[];
    const uint32_t rl = threadIdx.x / T, t = threadIdx.x % T;
    const size_t row = (size_t)blockIdx.x * (blockDim.x / T) + rl;
    const bool live = row < batch;
    uint32_t *s = sm + (size_t)rl * N;
    uint32_t *g = data + row * N;
    uint32_t v[32];
    if (live) {
        // element t + k T goes to bit-reversed position brev(t) | brev(k T)
        const uint32_t bt = swz(__brev(t) >> (32 - LOG_N));
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = ld_stream1(g + t + (uint32_t)k * T);
#pragma unroll
        for (int k = 0; k < 32; ++k) s[bt ^ swz(__brev((uint32_t)k * T) >> (32 - LOG_N))] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int s0 = 0; s0 < LOG_N; s0 += 5) {
        const int ws = s0 < LOG_N - 5 ? s0 : LOG_N - 5;
        const uint32_t tl = t & ((1u << ws) - 1u);
        const uint32_t base = tl | ((t >> ws) << (ws + 5));
        const uint32_t sb = swz(base);
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = s[sb ^ swz((uint32_t)k << ws)];
#pragma unroll
        for (int lb = 0; lb < 5; ++lb) {
            const int st = ws + lb + 1;  // stage: pair distance 2^(st-1)
            if (st <= s0) continue;      // done by the previous trip (last, overlapping window)
            // stage-major table: this stage's twiddle for pos = tl | j << ws is at
            // tw[2^(st-1) - 1 + pos]; consecutive lanes (consecutive tl) read consecutive words
            const uint32_t *twb = tw + ((1u << (st - 1)) - 1u) + tl;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int k0 = ((q >> lb) << (lb + 1)) | (q & ((1 << lb) - 1));
                const int k1 = k0 | (1 << lb);
                const uint32_t w = __ldg(twb + ((uint32_t)(k0 & ((1 << lb) - 1)) << ws));
                const uint32_t x1 = redc(v[k1], w, c.p, c.pinv);
                const uint32_t u = v[k0];
                v[k0] = mod_add(u, x1, c.p);
                v[k1] = mod_sub(u, x1, c.p);
            }
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) s[sb ^ swz((uint32_t)k << ws)] = v[k];
        __syncthreads();
    }
    if (live) {
        const uint32_t st0 = swz(t);
        const uint64_t rowg = (uint64_t)(row + t2.row0);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const uint32_t idx = t + (uint32_t)k * T;
            uint32_t x = s[st0 ^ swz((uint32_t)k * T)];
            if (t2.lo) {  // six-step twiddle w^(row * idx), from two half tables
                const uint64_t e = (rowg * idx) & t2.mask;
                const uint32_t we = redc(__ldg(t2.hi + (e >> t2.shift)), __ldg(t2.lo + (e & t2.lomask)), c.p, c.pinv);
                x = redc(x, we, c.p, c.pinv);
            }
            if (scale != c.r1) x = redc(x, scale, c.p, c.pinv);
            st_stream1(g + idx, x);
        }
    }
}

// ---- decimation-in-frequency form (Gentleman-Sande), natural-order input:
// trip 0 reads its 32 elements per thread straight from global memory
// (window = the TOP five index bits, so lanes read consecutive words) and the
// bit-reversed result is unscrambled by the final shared-memory gather -- one
// shared-memory pass fewer than the DIT kernel above.  Butterfly:
// (u, v) -> (u + v, (u - v) w^pos), stages from pair distance N/2 down to 1.
// PQ = true (mont_ntt_ex variant 3): tw is the pair table of mont_ntt_twiddles_pq and each
// butterfly multiplies by the precomputed-quotient (Shoup) product: q = hi(x w'), x w - q P in
// [0, 2P) from LOW words only -- one high product instead of REDC's two (4 FMAHeavy issue slots
// instead of 5, one ALU op fewer); w' = floor(w 2^32 / P) is the Montgomery form of w times P'
// mod 2^32.
// Shared-memory layouts of the DIF kernel.  XOR swizzle (default): word a at swz(a), combined per
// access with one LOP3.  PADDED (PAD = true): word a at a + (a >> 5), one pad word per 32; because
// every access address splits into a per-thread part and a per-k part with disjoint bits, the
// layout is additive -- f(base | k) = f(base) + f(k) -- so the per-k part is an immediate offset of
// the LDS/STS and the LOP3s disappear.  The padded layout is conflict-free for every pattern only
// if the bit reversal happens in the LAST trip's stores (results land in natural order) instead of
// in the final gather (checked exhaustively for log N = 5..15 by tests/test_ntt_layout.py).
template <bool PAD>
__device__ __forceinline__ uint32_t lay(uint32_t a) { return PAD ? a + (a >> 5) : swz(a); }
template <bool PAD>
__device__ __forceinline__ uint32_t lay_comb(uint32_t thread_part, uint32_t k_part) {
    return PAD ? thread_part + k_part : thread_part ^ k_part;
}
template <int BITS>
__host__ __device__ constexpr uint32_t brev_bits(uint32_t x) {
    uint32_t r = 0;
    for (int i = 0; i < BITS; ++i) r |= ((x >> i) & 1u) << (BITS - 1 - i);
    return r;
}

// LAZY (P < 2^30, so 4P < 2^32): values between stages live in [0, 2P) instead of [0, P)
// (Harvey's lazy butterfly): the sum is folded to [0, 2P) with one min against 2P, the difference
// a - d + 2P < 4P goes into the product unreduced, and the product's own final correction is
// dropped (REDC and the precomputed-quotient product both return [0, 2P) before it) -- one ALU op
// fewer per butterfly; outputs are canonicalised once at the end.
// L2 prefetch of the row group `grp` (rpc rows of N words, contiguous) in 4 KiB pieces, one per
// thread of the first warps: issued at the start of a CTA for the group a CTA will take about one
// wave later, so that group's first-trip loads come from L2 instead of HBM
__device__ __forceinline__ void prefetch_group(const uint32_t *data, size_t batch, size_t grp, uint32_t rpc,
                                               uint32_t N) {
    const size_t r0 = grp * rpc;
    if (r0 >= batch) return;
    const size_t rows = batch - r0 < rpc ? batch - r0 : rpc;
    const size_t bytes = rows * N * 4;
    const size_t off = (size_t)threadIdx.x * 4096;
    if (off < bytes) {
        const size_t len = bytes - off < 4096 ? bytes - off : 4096;
        bulk_prefetch_l2(data + r0 * N + off / 4, (uint32_t)len);
    }
}

// The butterflies of one DIF trip (window bits [wlo, wlo + 5), stages with pair distance < 2^top)
// on the 32 values v[] of one thread; tl = the thread's index bits below the window.  (Writing the
// REDC's last step as one three-input add hi T - hi M + P and min(r, r - P), to keep it off the
// FMAHeavy pipe, compiles to the same SASS: ptxas canonicalises both forms.)
template <int LOG_N, bool PQ, bool LAZY>
__device__ __forceinline__ void dif_trip(const Ctx &c, uint32_t (&v)[32], const int top, const int wlo,
                                         const uint32_t tl, const uint32_t *__restrict__ tw) {
#pragma unroll
    for (int lb = 4; lb >= 0; --lb) {
        const int b = wlo + lb;  // pair distance 2^b
        if (b >= top) continue;  // done by an earlier trip
        const uint32_t *twb = tw + ((1u << b) - 1u) + tl;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int k0 = ((q >> lb) << (lb + 1)) | (q & ((1 << lb) - 1));
            const int k1 = k0 | (1 << lb);
            const uint32_t j = (uint32_t)(k0 & ((1 << lb) - 1));
            const uint32_t a = v[k0], d = v[k1];
            const uint32_t p2 = 2u * c.p;
            if (LAZY) {
                const uint32_t sum = a + d;  // [0, 4P)
                v[k0] = umin(sum, sum - p2);  // [0, 2P)
            } else {
                v[k0] = mod_add(a, d, c.p);
            }
            if (wlo == 0 && j == 0) {
                // pos = 0 (tl is empty when wlo = 0): the twiddle is w^0 = 1, so the product is
                // skipped (a compile-time decision; 30 of the last trip's 64 butterflies at 2^14)
                if (LAZY) {
                    const uint32_t x = a - d + p2;
                    v[k1] = umin(x, x - p2);
                } else {
                    v[k1] = mod_sub(a, d, c.p);
                }
            } else if (PQ) {
                const uint2 wq = __ldg(reinterpret_cast<const uint2 *>(tw) + ((1u << b) - 1u) + tl + (j << wlo));
                const uint32_t x = a - d + (LAZY ? p2 : c.p);  // (0, 2P) or (0, 4P): any x < 2^32 is allowed
                const uint32_t qq = __umulhi(x, wq.y);         // floor(x w' / 2^32)
                const uint32_t r = x * wq.x - qq * c.p;        // x w - q P in [0, 2P), exact mod 2^32
                v[k1] = LAZY ? r : umin(r, r - c.p);
            } else if (LAZY) {
                // (a - d + 2P) w < 4P P < 2^32 P: REDC's precondition holds; keep t' + P in (0, 2P)
                const uint64_t T = mul_wide_u32(a - d + p2, __ldg(twb + (j << wlo)));
                const uint32_t m = (uint32_t)T * c.pinv;
                v[k1] = hi32(T) - hi32(mul_wide_u32(m, c.p)) + c.p;
            } else {
                // REDC needs only (a - d) w < 2^32 P, so a - d + P in (0, 2P) goes in unreduced:
                // the subtraction's correction is folded into the multiply
                const uint32_t w = __ldg(twb + (j << wlo));
                v[k1] = redc(a - d + c.p, w, c.p, c.pinv);
            }
        }
    }
}

// Persistent, software-pipelined form of k_ntt_dif<LOG_N, PQ, PAD = true, LAZY> (variants 6 / 7):
// a grid of (resident CTAs per SM) x SMs loops over the row groups, and the first trip's HBM loads
// of the NEXT group are issued right after the last trip's bit-reversed store -- before this group's
// final gather and its HBM stores -- so their latency hides behind that phase instead of leaving
// the SM with half its warps waiting at the start of every CTA.  Same arithmetic, same outputs.
template <int LOG_N, bool PQ, bool LAZY>
__global__ void __launch_bounds__(LOG_N == 15 ? 1024 : 512, LOG_N == 15 ? 1 : 2)
    k_ntt_difp(Ctx c, uint32_t *data, size_t batch, const uint32_t *__restrict__ tw, uint32_t scale, Tw2D t2,
               uint32_t pf) {
    constexpr uint32_t N = 1u << LOG_N, T = N >> 5;
    constexpr uint32_t NP = N + (N >> 5);
    constexpr int NTRIP = (LOG_N + 4) / 5;
    constexpr int WLO0 = LOG_N - 5 > 0 ? LOG_N - 5 : 0;
    extern __shared__ uint32_t sm[];
    const uint32_t rpc = blockDim.x / T;
    const uint32_t rl = threadIdx.x / T, t = threadIdx.x % T;
    uint32_t *s = sm + (size_t)rl * NP;
    const uint32_t base0 = (t & ((1u << WLO0) - 1u)) | ((t >> WLO0) << (WLO0 + 5));
    uint32_t v[32];
    size_t grp = blockIdx.x;
    {
        const size_t row = grp * rpc + rl;
        if (row < batch) {
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = ld_stream1(data + row * N + base0 + ((uint32_t)k << WLO0));
        }
    }
    for (; grp * rpc < batch; grp += gridDim.x) {  // uniform over the CTA
        const size_t row = grp * rpc + rl;
        const bool live = row < batch;
        if (pf) prefetch_group(data, batch, grp + gridDim.x, rpc, N);
#pragma unroll
        for (int trip = 0; trip < NTRIP; ++trip) {
            const int top = LOG_N - 5 * trip;
            const int wlo = top - 5 > 0 ? top - 5 : 0;
            const uint32_t tl = t & ((1u << wlo) - 1u);
            const uint32_t base = tl | ((t >> wlo) << (wlo + 5));
            const uint32_t sb = lay<true>(base);
            if (trip > 0) {
#pragma unroll
                for (int k = 0; k < 32; ++k) v[k] = s[lay_comb<true>(sb, lay<true>((uint32_t)k << wlo))];
            }
            dif_trip<LOG_N, PQ, LAZY>(c, v, top, wlo, tl, tw);
            if (trip == NTRIP - 1) {
                if (NTRIP > 1) __syncthreads();
                const uint32_t bb = lay<true>(brev_bits<LOG_N>(base));
#pragma unroll
                for (int k = 0; k < 32; ++k) s[bb + lay<true>(brev_bits<LOG_N>((uint32_t)k << wlo))] = v[k];
            } else {
#pragma unroll
                for (int k = 0; k < 32; ++k) s[lay_comb<true>(sb, lay<true>((uint32_t)k << wlo))] = v[k];
            }
            __syncthreads();
        }
        // next group's first-trip loads, in flight during this group's gather and stores
        const size_t nrow = row + (size_t)gridDim.x * rpc;
        if (nrow < batch) {
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = ld_stream1(data + nrow * N + base0 + ((uint32_t)k << WLO0));
        }
        if (live) {
            uint32_t *g = data + row * N;
            const uint32_t bt = lay<true>(t);
            const uint64_t rowg = (uint64_t)(row + t2.row0);
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const uint32_t idx = t + (uint32_t)k * T;
                uint32_t x = s[bt + lay<true>((uint32_t)k * T)];
                if (LAZY) x = umin(x, x - c.p);
                if (t2.lo) {
                    const uint64_t e = (rowg * idx) & t2.mask;
                    const uint32_t we = redc(__ldg(t2.hi + (e >> t2.shift)), __ldg(t2.lo + (e & t2.lomask)), c.p, c.pinv);
                    x = redc(x, we, c.p, c.pinv);
                }
                if (scale != c.r1) x = redc(x, scale, c.p, c.pinv);
                st_stream1(g + idx, x);
            }
        }
        __syncthreads();  // the next group's first trip overwrites s
    }
}

template <int LOG_N, bool PQ = false, bool PAD = false, bool LAZY = false>
__global__ void __launch_bounds__(LOG_N == 15 ? 1024 : 512, LOG_N == 15 ? 1 : 2)
    k_ntt_dif(Ctx c, uint32_t *data, size_t batch, const uint32_t *__restrict__ tw, uint32_t scale, Tw2D t2,
              uint32_t pf) {
    constexpr uint32_t N = 1u << LOG_N, T = N >> 5;
    constexpr uint32_t NP = PAD ? N + (N >> 5) : N;  // words per row in shared memory
    extern __shared__ uint32_t sm[];
    if (pf) prefetch_group(data, batch, (size_t)blockIdx.x + pf, blockDim.x / T, N);
    const uint32_t rl = threadIdx.x / T, t = threadIdx.x % T;
    const size_t row = (size_t)blockIdx.x * (blockDim.x / T) + rl;
    const bool live = row < batch;
    uint32_t *s = sm + (size_t)rl * NP;
    uint32_t *g = data + row * N;
    uint32_t v[32];
    constexpr int NTRIP = (LOG_N + 4) / 5;
#pragma unroll
    for (int trip = 0; trip < NTRIP; ++trip) {
        // window of this trip: bits [wlo, wlo + 5); stages done: bits >= hi_done
        const int top = LOG_N - 5 * trip;               // bits >= top already processed
        const int wlo = top - 5 > 0 ? top - 5 : 0;
        const uint32_t tl = t & ((1u << wlo) - 1u);
        const uint32_t base = tl | ((t >> wlo) << (wlo + 5));
        const uint32_t sb = lay<PAD>(base);
        if (trip == 0) {
            if (live) {
#pragma unroll
                for (int k = 0; k < 32; ++k) v[k] = ld_stream1(g + base + ((uint32_t)k << wlo));
            }
        } else {
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = s[lay_comb<PAD>(sb, lay<PAD>((uint32_t)k << wlo))];
        }
        dif_trip<LOG_N, PQ, LAZY>(c, v, top, wlo, tl, tw);
        if (PAD && trip == NTRIP - 1) {
            // last trip: the transform's outputs are in bit-reversed order; store each at its
            // natural index brev(pos) (other threads' words: everyone must have loaded first)
            if (NTRIP > 1) __syncthreads();
            const uint32_t bb = lay<PAD>(brev_bits<LOG_N>(base));
#pragma unroll
            for (int k = 0; k < 32; ++k) s[bb + lay<PAD>(brev_bits<LOG_N>((uint32_t)k << wlo))] = v[k];
        } else {
#pragma unroll
            for (int k = 0; k < 32; ++k) s[lay_comb<PAD>(sb, lay<PAD>((uint32_t)k << wlo))] = v[k];
        }
        __syncthreads();
    }
    if (live) {
        // X[idx] sits at the bit-reversed position (swizzled layout) or at idx (padded layout)
        const uint32_t bt = PAD ? lay<PAD>(t) : swz(__brev(t) >> (32 - LOG_N));
        const uint64_t rowg = (uint64_t)(row + t2.row0);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const uint32_t idx = t + (uint32_t)k * T;
            uint32_t x = PAD ? s[bt + lay<PAD>((uint32_t)k * T)] : s[bt ^ swz(__brev((uint32_t)k * T) >> (32 - LOG_N))];
            if (LAZY) x = umin(x, x - c.p);  // [0, 2P) -> [0, P)
            if (t2.lo) {
                const uint64_t e = (rowg * idx) & t2.mask;
                const uint32_t we = redc(__ldg(t2.hi + (e >> t2.shift)), __ldg(t2.lo + (e & t2.lomask)), c.p, c.pinv);
                x = redc(x, we, c.p, c.pinv);
            }
            if (scale != c.r1) x = redc(x, scale, c.p, c.pinv);
            st_stream1(g + idx, x);
        }
    }
}

// ---- column-mode DIF transform: the first pass of the 3-pass large transform.
// The data is an R x ld row-major matrix; CTA b transforms the C adjacent
// columns [b C, b C + C), each a length-N = 2^LOG_N transform down the rows
// (stride ld), in place, then multiplies element (k1, col) by the 2-D twiddle
// w^(col k1) of the large transform (Tw2D).  Two thread->(column, t) maps:
//   G (global phases: the trip-0 load, the final store): lanes span the C
//     columns of 32/C consecutive rows, so every warp access is 32/C fully used
//     segments of C*4 contiguous bytes (no transpose pass needed);
//   S (the shared-memory trips): lanes span 32 consecutive t of one column, as
//     in k_ntt_dif.
// Column col keeps its N words at sm[col N + (swz(a) ^ (col << CSH))]: the XOR
// moves the C columns of a G-mode warp access onto different banks (checked
// exhaustively for every access pattern by scripts/ntt_col_banks.py).
// PAD = true (the default): column c keeps its words at c (N + N/32 + 4) + a + (a >> 5) -- the
// padded, additive layout of k_ntt_dif<.., PAD> with a 4-word column skew; the last trip stores
// in natural order and the final gather (map G) reads natural order (all patterns conflict-free:
// tests/test_ntt_layout.py).
template <int LOG_N, int C>
constexpr uint32_t col_stride(bool pad) { return pad ? (1u << LOG_N) + (1u << (LOG_N - 5)) + 4u : (1u << LOG_N); }

template <int LOG_N, int C, bool PQ, bool PAD = true, bool LAZY = false>
__global__ void __launch_bounds__(C * (1 << LOG_N) / 32, C * (1 << LOG_N) / 32 <= 512 ? 2 : 1)
    k_ntt_col(Ctx c, uint32_t *data, size_t ld, const uint32_t *__restrict__ tw, Tw2D t2) {
    constexpr uint32_t N = 1u << LOG_N, T = N >> 5;
    constexpr uint32_t NPC = col_stride<LOG_N, C>(PAD);
    constexpr int CSH = (C == 16) ? 1 : (C == 8) ? 2 : 3;  // log2(32 / C)
    static_assert(C == 4 || C == 8 || C == 16, "C: 4, 8 or 16 columns per CTA");
    constexpr int NTRIP = (LOG_N + 4) / 5;
    extern __shared__ uint32_t sm[];
    const size_t col0 = (size_t)blockIdx.x * C;
    const uint32_t cg = threadIdx.x % C, tg = threadIdx.x / C;  // map G
    const uint32_t cs = threadIdx.x / T, ts = threadIdx.x % T;  // map S
    uint32_t v[32];
#pragma unroll
    for (int trip = 0; trip < NTRIP; ++trip) {
        const uint32_t col = trip == 0 ? cg : cs, t = trip == 0 ? tg : ts;
        uint32_t *s = sm + col * NPC;
        const uint32_t fx = (col << CSH) & 31u;
        const int top = LOG_N - 5 * trip;
        const int wlo = top - 5 > 0 ? top - 5 : 0;
        const uint32_t tl = t & ((1u << wlo) - 1u);
        const uint32_t base = tl | ((t >> wlo) << (wlo + 5));
        const uint32_t sb = PAD ? lay<true>(base) : (swz(base) ^ fx);
        if (trip == 0) {
            // running pointer: one 64-bit add per load instead of 32 live 64-bit addresses
            const uint32_t *g = data + col0 + col + (size_t)base * ld;
            const size_t step = ld << wlo;
#pragma unroll
            for (int k = 0; k < 32; ++k, g += step) v[k] = ld_stream1(g);
        } else {
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = s[lay_comb<PAD>(sb, lay<PAD>((uint32_t)k << wlo))];
        }
#pragma unroll
        for (int lb = 4; lb >= 0; --lb) {
            const int b = wlo + lb;
            if (b >= top) continue;
            const uint32_t *twb = tw + ((1u << b) - 1u) + tl;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int k0 = ((q >> lb) << (lb + 1)) | (q & ((1 << lb) - 1));
                const int k1 = k0 | (1 << lb);
                const uint32_t j = (uint32_t)(k0 & ((1 << lb) - 1));
                const uint32_t a = v[k0], d = v[k1];
                const uint32_t p2 = 2u * c.p;  // LAZY: values in [0, 2P), as in k_ntt_dif<.., LAZY>
                if (LAZY) {
                    const uint32_t sum = a + d;
                    v[k0] = umin(sum, sum - p2);
                } else {
                    v[k0] = mod_add(a, d, c.p);
                }
                if (wlo == 0 && j == 0) {
                    if (LAZY) {
                        const uint32_t x = a - d + p2;
                        v[k1] = umin(x, x - p2);
                    } else {
                        v[k1] = mod_sub(a, d, c.p);
                    }
                } else if (PQ) {  // precomputed-quotient product, as in k_ntt_dif<.., true>
                    const uint2 wq = __ldg(reinterpret_cast<const uint2 *>(tw) + ((1u << b) - 1u) + tl + (j << wlo));
                    const uint32_t x = a - d + (LAZY ? p2 : c.p);
                    const uint32_t r = x * wq.x - __umulhi(x, wq.y) * c.p;
                    v[k1] = LAZY ? r : umin(r, r - c.p);
                } else if (LAZY) {
                    const uint64_t T = mul_wide_u32(a - d + p2, __ldg(twb + (j << wlo)));
                    const uint32_t m = (uint32_t)T * c.pinv;
                    v[k1] = hi32(T) - hi32(mul_wide_u32(m, c.p)) + c.p;
                } else {
                    v[k1] = redc(a - d + c.p, __ldg(twb + (j << wlo)), c.p, c.pinv);
                }
            }
        }
        if (PAD && trip == NTRIP - 1) {
            // last trip: store each result at its natural index (other threads' words: barrier first)
            if (NTRIP > 1) __syncthreads();
            const uint32_t bb = lay<true>(brev_bits<LOG_N>(base));
#pragma unroll
            for (int k = 0; k < 32; ++k) s[bb + lay<true>(brev_bits<LOG_N>((uint32_t)k << wlo))] = v[k];
        } else {
            // each thread writes back exactly the 32 words it read this trip: no barrier before the store
#pragma unroll
            for (int k = 0; k < 32; ++k) s[lay_comb<PAD>(sb, lay<PAD>((uint32_t)k << wlo))] = v[k];
        }
        __syncthreads();
    }
    // final gather in map H: lanes span the C columns of 32/C rows as in map G, but those rows
    // are T/(32/C) apart (t = j T/(32/C) + warp), so their bit-reversed positions differ in
    // the bits the swizzle folds onto the low banks and the column XOR keeps all 32 lanes apart.
    // X[idx] of column cg sits at the bit-reversed position.
    {
        constexpr uint32_t R = 32 / C;                 // rows per warp
        const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
        // padded layout: map G (natural order is conflict-free there); swizzled: map H
        const uint32_t ch = PAD ? cg : lane % C, th = PAD ? tg : (lane / C) * (T / R) + wid;
        const uint32_t *s = sm + ch * NPC;
        const uint32_t fx = (ch << CSH) & 31u;
        const uint32_t bt = PAD ? lay<true>(th) : (swz(__brev(th) >> (32 - LOG_N)) ^ fx);
        const uint64_t colg = (uint64_t)(col0 + ch);
        uint32_t *g = data + col0 + ch + (size_t)th * ld;
        const size_t step = ld * T;
        uint64_t e = (colg * th) & t2.mask;            // exponent col * idx, idx = th + k T
        const uint64_t de = (colg * T) & t2.mask;
#pragma unroll
        for (int k = 0; k < 32; ++k, g += step, e = (e + de) & t2.mask) {
            // (LAZY: x in [0, 2P); the REDC with the 2-D twiddle below still returns [0, P))
            const uint32_t x = PAD ? s[bt + lay<true>((uint32_t)k * T)] : s[bt ^ swz(__brev((uint32_t)k * T) >> (32 - LOG_N))];
            const uint32_t we = redc(__ldg(t2.hi + (e >> t2.shift)), __ldg(t2.lo + (e & t2.lomask)), c.p, c.pinv);
            st_stream1(g, redc(x, we, c.p, c.pinv));
        }
    }
}

// L2 prefetch of the row group one wave ahead in the row kernels; MONT_NTT_NO_PF=1 turns it off
// (measurement)
static bool ntt_pf() {
    static const bool on = !(getenv("MONT_NTT_NO_PF") && getenv("MONT_NTT_NO_PF")[0] == '1');
    return on;
}

template <int LOG_N, int C, bool PQ, bool LAZY = false>
static mont_status_t launch_ntt_col(const Ctx &c, uint32_t *data, size_t ld, const uint32_t *tw, Tw2D t2,
                                    cudaStream_t stream) {
    const size_t smem = (size_t)C * col_stride<LOG_N, C>(true) * 4;
    if (ld % C) return MONT_EUNSUPPORTED;
    const size_t grid = ld / C;
    if (grid > 0x7fffffffu) return MONT_EUNSUPPORTED;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(k_ntt_col<LOG_N, C, PQ, true, LAZY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
        return MONT_ECUDA;
    k_ntt_col<LOG_N, C, PQ, true, LAZY><<<(unsigned)grid, C * ((1u << LOG_N) >> 5), smem, stream>>>(c, data, ld, tw, t2);
    return launch_status();
}

template <int LOG_N, bool PQ = false, bool PAD = false, bool LAZY = false>
static mont_status_t launch_ntt_dif(const Ctx &c, uint32_t *data, size_t batch, const uint32_t *tw, uint32_t scale,
                                    cudaStream_t stream, Tw2D t2) {
    constexpr uint32_t N = 1u << LOG_N, T = N >> 5;
    constexpr uint32_t rpc = T >= 256 ? 1u : 256u / T;
    const size_t smem = (size_t)rpc * (PAD ? N + (N >> 5) : N) * 4;
    const size_t grid = (batch + rpc - 1) / rpc;
    if (grid > 0x7fffffffu) return MONT_EUNSUPPORTED;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(k_ntt_dif<LOG_N, PQ, PAD, LAZY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
        return MONT_ECUDA;
    // L2 prefetch one wave of resident CTAs ahead (2 per SM at 2^14): 2^14 rows 221.7 -> 217.6 us;
    // for shorter rows it measured 2 % slower, so it is off there
    // (profiles/r02_probe_ntt_persistent.jsonl)
    const int sms = sm_count();
    const uint32_t pf = LOG_N == 14 && ntt_pf() && sms > 0 ? (uint32_t)sms * 2u : 0u;
    k_ntt_dif<LOG_N, PQ, PAD, LAZY><<<(unsigned)grid, rpc * T, smem, stream>>>(c, data, batch, tw, scale, t2, pf);
    return launch_status();
}

template <int LOG_N, bool PQ, bool LAZY>
static mont_status_t launch_ntt_difp(const Ctx &c, uint32_t *data, size_t batch, const uint32_t *tw, uint32_t scale,
                                     cudaStream_t stream, Tw2D t2) {
    constexpr uint32_t N = 1u << LOG_N, T = N >> 5;
    constexpr uint32_t rpc = T >= 256 ? 1u : 256u / T;
    const size_t smem = (size_t)rpc * (N + (N >> 5)) * 4;
    static int resident = 0;  // CTAs per SM, once per instantiation
    if (resident == 0) {
        if (smem > 48 * 1024 &&
            cudaFuncSetAttribute(k_ntt_difp<LOG_N, PQ, LAZY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess)
            return MONT_ECUDA;
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_ntt_difp<LOG_N, PQ, LAZY>, (int)(rpc * T), smem) !=
                cudaSuccess ||
            nb < 1)
            return MONT_ECUDA;
        resident = nb;
        if (getenv("MONT_NTT_DEBUG")) fprintf(stderr, "k_ntt_difp<%d>: %d CTAs/SM\n", LOG_N, nb);
    }
    const int sms = sm_count();
    if (sms <= 0) return MONT_ECUDA;
    const size_t groups = (batch + rpc - 1) / rpc;
    size_t grid = (size_t)resident * (size_t)sms;
    if (grid > groups) grid = groups;
    k_ntt_difp<LOG_N, PQ, LAZY><<<(unsigned)grid, rpc * T, smem, stream>>>(c, data, batch, tw, scale, t2,
                                                                          ntt_pf() ? 1u : 0u);
    return launch_status();
}

template <int LOG_N>
static mont_status_t launch_ntt_r32(const Ctx &c, uint32_t *data, size_t batch, const uint32_t *tw, uint32_t scale,
                                    cudaStream_t stream, Tw2D t2 = Tw2D{nullptr, nullptr, 0, 0, 0, 0}) {
    constexpr uint32_t N = 1u << LOG_N, T = N >> 5;
    constexpr uint32_t rpc = T >= 256 ? 1u : 256u / T;  // rows per CTA
    const size_t smem = (size_t)rpc * N * 4;
    const size_t grid = (batch + rpc - 1) / rpc;
    if (grid > 0x7fffffffu) return MONT_EUNSUPPORTED;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(k_ntt_r32<LOG_N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return MONT_ECUDA;
    k_ntt_r32<LOG_N><<<(unsigned)grid, rpc * T, smem, stream>>>(c, data, batch, tw, scale, t2);
    return launch_status();
}

__global__ void __launch_bounds__(256) k_ntt_twiddles(Ctx c, uint32_t *tw, uint32_t w, int log_n) {
    const size_t total = ((size_t)1 << log_n) - 1;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        // e = 2^(s-1) - 1 + pos  ->  s - 1 = floor(log2(e + 1)), pos = e + 1 - 2^(s-1)
        const int sm1 = 63 - __clzll((unsigned long long)(e + 1));
        const size_t pos = e + 1 - ((size_t)1 << sm1);
        const unsigned long long ex = (unsigned long long)pos << (log_n - 1 - sm1);  // pos * N / 2^s
        const uint32_t x = redc(w, c.r2, c.p, c.pinv);
        uint32_t acc = c.r1;
        for (int sh = 63 - __clzll(ex | 1ull); sh >= 0; --sh) {
            acc = redc(acc, acc, c.p, c.pinv);
            if ((ex >> sh) & 1ull) acc = redc(acc, x, c.p, c.pinv);
        }
        tw[e] = acc;
    }
}

// pair table for variant 3: tw2[2e] = w^x (plain), tw2[2e + 1] = floor(w^x 2^32 / P) = to_mont(w^x) P'
// mod 2^32, with e and x as in k_ntt_twiddles
__global__ void __launch_bounds__(256) k_ntt_twiddles_pq(Ctx c, uint32_t *tw2, uint32_t w, int log_n) {
    const size_t total = ((size_t)1 << log_n) - 1;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int sm1 = 63 - __clzll((unsigned long long)(e + 1));
        const size_t pos = e + 1 - ((size_t)1 << sm1);
        const unsigned long long ex = (unsigned long long)pos << (log_n - 1 - sm1);
        const uint32_t x = redc(w, c.r2, c.p, c.pinv);
        uint32_t acc = c.r1;
        for (int sh = 63 - __clzll(ex | 1ull); sh >= 0; --sh) {
            acc = redc(acc, acc, c.p, c.pinv);
            if ((ex >> sh) & 1ull) acc = redc(acc, x, c.p, c.pinv);
        }
        // acc = w^x 2^32 mod P (canonical): w^x 2^32 = q P + acc, so q = -acc P^-1 mod 2^32
        tw2[2 * e] = redc1(acc, c.p, c.pinv);
        tw2[2 * e + 1] = acc * (0u - c.pinv);
    }
}

// tiled transpose of an R x C row-major uint32 matrix (32 x 32 tiles through
// padded shared memory; coalesced 128-byte rows on both sides)
__global__ void __launch_bounds__(256) k_transpose(uint32_t *dst, const uint32_t *src, size_t R, size_t C) {
    __shared__ uint32_t tile[32][33];
    const size_t c0 = (size_t)blockIdx.x * 32, r0 = (size_t)blockIdx.y * 32;
    const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const size_t r = r0 + ty + k, cc = c0 + tx;
        if (r < R && cc < C) tile[ty + k][tx] = ld_stream1(src + r * C + cc);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const size_t cc = c0 + ty + k, r = r0 + tx;  // dst is C x R
        if (r < R && cc < C) st_stream1(dst + cc * R + r, tile[tx][ty + k]);
    }
}

static mont_status_t transpose(uint32_t *dst, const uint32_t *src, size_t R, size_t C, cudaStream_t s) {
    const size_t gx = (C + 31) / 32, gy = (R + 31) / 32;
    if (gx > 0x7fffffffu || gy > 65535) return MONT_EUNSUPPORTED;
    k_transpose<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, s>>>(dst, src, R, C);
    return launch_status();
}

// 2^15 rows (one 1024-thread CTA per SM): variants 0 / 3 run the persistent kernel (variants 6 / 7),
// which hides the next row's HBM loads behind this row's stores (297 -> 275 us REDC, 252 -> 234 us
// precomputed-quotient for 2048 rows); with 2 or more CTAs per SM the other CTA already covers
// that phase and the persistent form measured slower (2^14: 222 -> 258 us),
// profiles/r02_probe_ntt_persistent.jsonl
#define MONT_NTT_CASE(L)                                                                           \
    case L:                                                                                        \
        if (L == 15 && (kind == 0 || kind == 3)) kind = kind == 0 ? 6 : 7;                          \
        return kind == 0   ? (lazy ? launch_ntt_dif<L, false, true, true>(c, data, batch, tw, scale, s, t2)   \
                                   : launch_ntt_dif<L, false, true>(c, data, batch, tw, scale, s, t2))      \
               : kind == 3 ? (lazy ? launch_ntt_dif<L, true, true, true>(c, data, batch, tw, scale, s, t2)    \
                                   : launch_ntt_dif<L, true, true>(c, data, batch, tw, scale, s, t2))       \
               : kind == 4 ? launch_ntt_dif<L, false, false>(c, data, batch, tw, scale, s, t2)    \
               : kind == 5 ? launch_ntt_dif<L, true, false>(c, data, batch, tw, scale, s, t2)     \
               : kind == 6 ? (lazy ? launch_ntt_difp<L, false, true>(c, data, batch, tw, scale, s, t2) \
                                   : launch_ntt_difp<L, false, false>(c, data, batch, tw, scale, s, t2)) \
               : kind == 7 ? (lazy ? launch_ntt_difp<L, true, true>(c, data, batch, tw, scale, s, t2) \
                                   : launch_ntt_difp<L, true, false>(c, data, batch, tw, scale, s, t2)) \
                           : launch_ntt_r32<L>(c, data, batch, tw, scale, s, t2);

// lazy [0, 2P) butterflies when 4P < 2^32 (P < 2^30); MONT_NTT_NO_LAZY=1 turns them off (measurement)
static bool ntt_lazy(uint32_t p) {
    static const bool ok = !(getenv("MONT_NTT_NO_LAZY") && getenv("MONT_NTT_NO_LAZY")[0] == '1');
    return ok && p < (1u << 30);
}

// kind: 0 = DIF (REDC twiddles), 1 = DIT, 3 = DIF with precomputed-quotient twiddles (both in the
// padded shared layout); 4 / 5 = 0 / 3 in the XOR-swizzled layout (kept for measurement)
static mont_status_t ntt_rows(const Ctx &c, uint32_t *data, size_t batch, int log_n, const uint32_t *tw,
                              uint32_t scale, cudaStream_t s, Tw2D t2, int kind = 0) {
    const bool lazy = ntt_lazy(c.p);
    switch (log_n) {
        MONT_NTT_CASE(5)
        MONT_NTT_CASE(6)
        MONT_NTT_CASE(7)
        MONT_NTT_CASE(8)
        MONT_NTT_CASE(9)
        MONT_NTT_CASE(10)
        MONT_NTT_CASE(11)
        MONT_NTT_CASE(12)
        MONT_NTT_CASE(13)
        MONT_NTT_CASE(14)
        MONT_NTT_CASE(15)
        default: return MONT_EUNSUPPORTED;
    }
}
#undef MONT_NTT_CASE

// split of a large transform: N = N1 * N2.  2^22..2^27: the 3-pass form (column pass over
// N1 = 2^11 or 2^12 rows, 8 columns = one 32-byte sector per row per CTA; row pass over
// N2 = 2^10..2^15; one transpose); otherwise the six-step form with N1 = 2^floor(log_n / 2)
// (both <= 2^15).
static bool ntt_three_pass(int log_n) { return log_n >= 22 && log_n <= 27; }
// Column length: 2^11 (8 x 8 KiB per CTA, 2 CTAs/SM) for 2^23..2^26, 2^12 (1 CTA/SM) for 2^22
// (where 2^11 leaves only 2^11 / 8 = 256 column CTAs) and 2^27 (rows are capped at 2^15);
// measured per size, profiles/r01_probe_ntt_large_3pass.jsonl.
static void ntt_split(int log_n, int &a, int &b, int &sh) {
    a = ntt_three_pass(log_n) ? ((log_n == 22 || log_n == 27) ? 12 : 11) : log_n / 2;
    b = log_n - a;
    sh = (log_n + 1) / 2;  // two-level table split of the exponent
}

static uint32_t host_powmod(uint32_t x, uint64_t e, uint32_t p) {
    uint64_t r = 1 % p, b = x % p;
    while (e) {
        if (e & 1) r = r * b % p;
        b = b * b % p;
        e >>= 1;
    }
    return (uint32_t)r;
}

}  // namespace mont

using namespace mont;

// plan layout: [column table][row table][2-D low table 2^sh][2-D high table 2^(log_n - sh)];
// the column and row tables are pair tables (mont_ntt_twiddles_pq, 2 words per entry, 8-byte
// aligned); the 2-D tables hold Montgomery forms (REDC of two of them gives the factor)
struct PlanLayout {
    int a, b, sh;
    bool pq;
    size_t tw1, tw2, tlo, thi, words;
};
static PlanLayout plan_layout(int log_n) {
    PlanLayout L;
    ntt_split(log_n, L.a, L.b, L.sh);
    L.pq = true;  // both forms multiply by precomputed-quotient twiddles
    const size_t e = L.pq ? 2 : 1;
    L.tw1 = 0;
    L.tw2 = L.tw1 + e * (((size_t)1 << L.a) - 1);
    L.tlo = L.tw2 + e * (((size_t)1 << L.b) - 1);
    L.thi = L.tlo + ((size_t)1 << L.sh);
    L.words = L.thi + ((size_t)1 << (log_n - L.sh));
    return L;
}

extern "C" size_t mont_ntt_plan_words(int log_n) {
    if (log_n < 16 || log_n > 30) return 0;
    return plan_layout(log_n).words;
}

extern "C" mont_status_t mont_ntt_plan_init(const mont_ctx_t *ctx, uint32_t *plan, uint32_t w, int log_n,
                                            cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (log_n < 16 || log_n > 30) return MONT_EUNSUPPORTED;
    if (!plan || ((uintptr_t)plan & 7u)) return MONT_EINVAL_ARG;
    const PlanLayout L = plan_layout(log_n);
    const int a = L.a, b = L.b, sh = L.sh;
    const uint32_t p = ctx->p;
    uint32_t *tw1 = plan + L.tw1, *tw2 = plan + L.tw2, *tlo = plan + L.tlo, *thi = plan + L.thi;
    mont_status_t st;
    // column transforms have length N1 = 2^a: root w^(N2); row transforms N2 = 2^b: root w^(N1)
    auto table = L.pq ? mont_ntt_twiddles_pq : mont_ntt_twiddles;
    if ((st = table(ctx, tw1, host_powmod(w, 1ull << b, p), a, stream)) != MONT_OK) return st;
    if ((st = table(ctx, tw2, host_powmod(w, 1ull << a, p), b, stream)) != MONT_OK) return st;
    if ((st = mont_twiddle_table(ctx, tlo, w, (size_t)1 << sh, stream)) != MONT_OK) return st;
    return mont_twiddle_table(ctx, thi, host_powmod(w, 1ull << sh, p), (size_t)1 << (log_n - sh), stream);
}

extern "C" mont_status_t mont_ntt_large(const mont_ctx_t *ctx, uint32_t *out, uint32_t *in, int log_n,
                                        const uint32_t *plan, uint32_t scale, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (log_n < 16 || log_n > 30) return MONT_EUNSUPPORTED;
    if (!out || !in || !plan || out == in || (((uintptr_t)out | (uintptr_t)in) & 3u) || ((uintptr_t)plan & 7u) ||
        scale >= ctx->p)
        return MONT_EINVAL_ARG;
    const PlanLayout L = plan_layout(log_n);
    const int a = L.a, b = L.b, sh = L.sh;
    const size_t N1 = (size_t)1 << a, N2 = (size_t)1 << b;
    const uint32_t *tw1 = plan + L.tw1, *tw2 = plan + L.tw2, *tlo = plan + L.tlo, *thi = plan + L.thi;
    const Ctx c = to_dev(ctx);
    const Tw2D none{nullptr, nullptr, 0, 0, 0, 0};
    const Tw2D t2{tlo, thi, ((uint64_t)1 << log_n) - 1, (1u << sh) - 1u, sh, 0};
    mont_status_t st;
    if (ntt_three_pass(log_n)) {
        // x as N1 x N2 [n1][n2]: N2 column transforms of length N1 down the rows, in place, each
        // output (k1, n2) times w^(n2 k1) -> [k1][n2]; then N1 row transforms of length N2 with
        // the output scale -> [k1][k2]; X[k1 + N1 k2] = [k1][k2]: one transpose to natural order
        // (both passes multiply by the twiddles with precomputed quotients: pair tables)
        const bool lazy = ntt_lazy(c.p);
        st = a == 11 ? (lazy ? launch_ntt_col<11, 8, true, true>(c, in, N2, tw1, t2, stream)
                             : launch_ntt_col<11, 8, true>(c, in, N2, tw1, t2, stream))
                     : (lazy ? launch_ntt_col<12, 8, true, true>(c, in, N2, tw1, t2, stream)
                             : launch_ntt_col<12, 8, true>(c, in, N2, tw1, t2, stream));
        if (st != MONT_OK) return st;
        if ((st = ntt_rows(c, in, N1, b, tw2, scale, stream, none, 3)) != MONT_OK) return st;
        return transpose(out, in, N1, N2, stream);
    }
    // x as N1 x N2 [n1][n2] -> out as N2 x N1 [n2][n1]
    if ((st = transpose(out, in, N1, N2, stream)) != MONT_OK) return st;
    // N2 column transforms of length N1, then the twiddle w^(n2 k1)
    if ((st = ntt_rows(c, out, N2, a, tw1, c.r1, stream, t2, 3)) != MONT_OK) return st;
    // back to N1 x N2 [k1][n2]
    if ((st = transpose(in, out, N2, N1, stream)) != MONT_OK) return st;
    // N1 row transforms of length N2 -> [k1][k2], with the output scale
    if ((st = ntt_rows(c, in, N1, b, tw2, scale, stream, none, 3)) != MONT_OK) return st;
    // X[k1 + N1 k2] = [k1][k2]: transpose to N2 x N1 -> natural order in out
    return transpose(out, in, N1, N2, stream);
}

extern "C" mont_status_t mont_ntt_twiddles(const mont_ctx_t *ctx, uint32_t *tw, uint32_t w, int log_n,
                                           cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (log_n < 1 || log_n > 30) return MONT_EUNSUPPORTED;
    if (!tw || ((uintptr_t)tw & 3u)) return MONT_EINVAL_ARG;
    const int sms = sm_count();
    if (sms <= 0) return MONT_ECUDA;
    size_t grid = ((((size_t)1 << log_n) - 1) + 255) / 256;
    if (grid > (size_t)sms * 8) grid = (size_t)sms * 8;
    if (grid == 0) grid = 1;
    k_ntt_twiddles<<<(unsigned)grid, 256, 0, stream>>>(to_dev(ctx), tw, w, log_n);
    return launch_status();
}

extern "C" mont_status_t mont_ntt_ex(const mont_ctx_t *ctx, uint32_t *data, size_t batch, int log_n,
                                     const uint32_t *tw, uint32_t scale, int variant, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (log_n < 1 || log_n > 15) return MONT_EUNSUPPORTED;
    if (batch == 0) return MONT_OK;
    if (!data || !tw || ((uintptr_t)data & 3u) || ((uintptr_t)tw & 3u) || scale >= ctx->p) return MONT_EINVAL_ARG;
    if (batch > 0x7fffffffu || variant < 0 || variant > 7) return variant < 0 || variant > 7 ? MONT_EINVAL_ARG
                                                                                             : MONT_EUNSUPPORTED;
    const bool pair = variant == 3 || variant == 5 || variant == 7;
    if (pair && ((uintptr_t)tw & 7u)) return MONT_EINVAL_ARG;  // pair table: 8-byte entries
    const uint32_t N = 1u << log_n;
    if (variant >= 3 && log_n < 5) return MONT_EUNSUPPORTED;  // the 32-per-thread kernels
    if (log_n >= 5 && variant != 2)
        return ntt_rows(to_dev(ctx), data, batch, log_n, tw, scale, stream, Tw2D{nullptr, nullptr, 0, 0, 0, 0},
                        variant);
    int threads = (int)(N / 2 < 1024 ? N / 2 : 1024);
    if (threads < 32) threads = 32;
    const size_t smem = (size_t)N * 4;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(k_ntt_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return MONT_ECUDA;
    k_ntt_smem<<<(unsigned)batch, threads, smem, stream>>>(to_dev(ctx), data, log_n, tw, scale);
    return launch_status();
}

extern "C" mont_status_t mont_ntt(const mont_ctx_t *ctx, uint32_t *data, size_t batch, int log_n, const uint32_t *tw,
                                  uint32_t scale, cudaStream_t stream) {
    return mont_ntt_ex(ctx, data, batch, log_n, tw, scale, 0, stream);
}

extern "C" mont_status_t mont_ntt_twiddles_pq(const mont_ctx_t *ctx, uint32_t *tw2, uint32_t w, int log_n,
                                              cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (log_n < 1 || log_n > 30) return MONT_EUNSUPPORTED;
    if (!tw2 || ((uintptr_t)tw2 & 7u)) return MONT_EINVAL_ARG;
    const int sms = sm_count();
    if (sms <= 0) return MONT_ECUDA;
    size_t grid = ((((size_t)1 << log_n) - 1) + 255) / 256;
    if (grid > (size_t)sms * 8) grid = (size_t)sms * 8;
    if (grid == 0) grid = 1;
    k_ntt_twiddles_pq<<<(unsigned)grid, 256, 0, stream>>>(to_dev(ctx), tw2, w, log_n);
    return launch_status();
}
