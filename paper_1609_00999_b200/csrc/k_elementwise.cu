// k_elementwise.cu -- the HBM-bound streaming kernels of the path:
//   K1 mont_mul_vec  c[i] = REDC(a[i], b[i])         12 B/elem
//   K4 to_mont       out[i] = REDC(in[i], R^2 mod P)  8 B/elem  (A2)
//   K5 from_mont     out[i] = REDC(in[i], 1)          8 B/elem  (A10)
//   K6 mont_checksum *acc += sum x[i]                 4 B/elem  (A11)
// plus the triad/copy microbenchmarks that share K1's launch shape.
//
// B200 design: the paper vectorises REDC across the 4 lanes of
// a 128-bit SSE register (§3.2, :125).  Here each thread owns whole
// 128-bit chunks (4 residues = one uint4), loaded with LDG.E.128 on the
// non-coherent path and stored evict-first.  Default shape: a flat grid, one
// tile of threads * U chunks per CTA (the block scheduler balances fast and
// slow SMs); variant 1 deals tiles round-robin to a persistent grid of
// SMs * k CTAs, variant 2 stages each CTA's tiles with cp.async.bulk (TMA),
// variant 3 is a persistent bulk-copy pipeline (TMA load ring + bulk stores).
// All U loads of a tile are issued before any arithmetic (memory-level
// parallelism); the REDC is 5 FMAHeavy issue slots + 2 ALU ops per residue and
// hides under the HBM stream (~25 % FMAHeavy at full bandwidth).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/barrett.h"
#include "abi_util.h"
#include "tma.cuh"

namespace mont {

struct OpMul {
    uint32_t p, pinv;
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return redc(a, b, p, pinv); }
};
struct OpTo {
    uint32_t p, pinv, r2;
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const { return redc(x, r2, p, pinv); }
};
struct OpFrom {
    uint32_t p, pinv;
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const { return redc1(x, p, pinv); }
};
// REDC(a, b) = a b R^-1 mod P computed on the FP64 pipe (mul_vec variant 4): two FP64 Barrett
// products (mont_core.cuh fmulmod, 6 FP64 ops each: a b mod P, then times R^-1 mod P), no
// FMAHeavy instruction -- for streaming next to an IMAD-bound kernel.  Both operands canonical.
struct OpFmont {
    double pd, pdinv, rinv;
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const {
        const double x = fmulmod(__uint2double_rn(a), __uint2double_rn(b), pd, pdinv);  // (-P, P)
        double y = fmulmod(x, rinv, pd, pdinv);
        y = y < 0.0 ? y + pd : y;
        return __double2uint_rn(y);
    }
};
struct OpBarrett {
    BarrettDev c;
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return barrett(a, b, c); }
};
struct OpXor {  // triad microbenchmark: no modular math
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a ^ b; }
};
struct OpCopy {
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const { return x; }
};

template <class Op>
__device__ __forceinline__ uint4 apply4(const Op &op, const uint4 &a, const uint4 &b) {
    return make_uint4(op(a.x, b.x), op(a.y, b.y), op(a.z, b.z), op(a.w, b.w));
}
template <class Op>
__device__ __forceinline__ uint4 apply4(const Op &op, const uint4 &a) {
    return make_uint4(op(a.x), op(a.y), op(a.z), op(a.w));
}

// ------------------------------------------------------------ block reduce
__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// adds the CTA's total of s into *acc with one 64-bit atomic
__device__ __forceinline__ void block_sum_to(unsigned long long *acc, unsigned long long s) {
    __shared__ unsigned long long warp_part[32];
    s = warp_sum(s);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) warp_part[wid] = s;
    __syncthreads();
    if (wid == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        s = lane < nw ? warp_part[lane] : 0ull;
        s = warp_sum(s);
        if (lane == 0 && s) atomicAdd(acc, s);
    }
}

__device__ __forceinline__ unsigned long long sum4(const uint4 &v) {
    return (unsigned long long)v.x + v.y + (unsigned long long)v.z + v.w;
}

// ---------------------------------------------------------------- binary map
// Vector body over n4 chunks of a4/b4/c4 (16-byte aligned), plus `head`
// scalar elements before it and `tail` after it, handled by CTA 0.
// SUM: also add the sum of every output word into *acc (A7 fused with the
// A11 checksum: saves re-reading c, 4 B/elem).
template <int U, class Op, bool SUM>
__global__ void __launch_bounds__(512) k_map2(Op op, uint32_t *c, const uint32_t *a, const uint32_t *b,
                                                uint32_t head, size_t n4, uint32_t tail, unsigned long long *acc) {
    pdl_trigger();
    unsigned long long s = 0;
    if (blockIdx.x == 0 && threadIdx.x < head + tail) {
        size_t i = threadIdx.x < head ? threadIdx.x : head + 4 * n4 + (threadIdx.x - head);
        const uint32_t r = op(a[i], b[i]);
        c[i] = r;
        s += r;
    }
    const uint4 *a4 = reinterpret_cast<const uint4 *>(a + head);
    const uint4 *b4 = reinterpret_cast<const uint4 *>(b + head);
    uint4 *c4 = reinterpret_cast<uint4 *>(c + head);
    const size_t tile = (size_t)U * blockDim.x;
    const size_t ntiles_full = n4 / tile;
    size_t t = blockIdx.x;
    for (; t < ntiles_full; t += gridDim.x) {
        const size_t base = t * tile + threadIdx.x;
        uint4 va[U], vb[U];
#pragma unroll
        for (int k = 0; k < U; ++k) va[k] = ld_stream(a4 + base + (size_t)k * blockDim.x);
#pragma unroll
        for (int k = 0; k < U; ++k) vb[k] = ld_stream(b4 + base + (size_t)k * blockDim.x);
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint4 r = apply4(op, va[k], vb[k]);
            st_stream(c4 + base + (size_t)k * blockDim.x, r);
            if (SUM) s += sum4(r);
        }
    }
    if (t == ntiles_full) {  // the one partial tile, owned by exactly one CTA
        for (size_t i = t * tile + threadIdx.x; i < n4; i += blockDim.x) {
            const uint4 r = apply4(op, ld_stream(a4 + i), ld_stream(b4 + i));
            st_stream(c4 + i, r);
            if (SUM) s += sum4(r);
        }
    }
    if (SUM) block_sum_to(acc, s);
    pdl_wait();
}

// Bulk-copy (TMA) variant: each CTA stages one tile of a and one of b into
// shared memory with two cp.async.bulk copies completing on one mbarrier, then
// computes from shared memory and stores c with 128-bit evict-first stores.
// Flat grid, one tile per CTA; several CTAs per SM keep copies in flight.
template <class Op, bool SUM>
__global__ void __launch_bounds__(256) k_map2_tma(Op op, uint32_t *c, const uint32_t *a, const uint32_t *b,
                                                   uint32_t head, size_t n4, uint32_t tail, unsigned long long *acc,
                                                   uint32_t tile4) {
    extern __shared__ __align__(128) uint4 sm[];
    __shared__ __align__(8) uint64_t bar;
    unsigned long long s = 0;
    const uint4 *a4 = reinterpret_cast<const uint4 *>(a + head);
    const uint4 *b4 = reinterpret_cast<const uint4 *>(b + head);
    uint4 *c4 = reinterpret_cast<uint4 *>(c + head);
    const size_t t0 = (size_t)blockIdx.x * tile4;
    const uint32_t cnt = (uint32_t)(n4 - t0 < tile4 ? n4 - t0 : tile4);
    if (threadIdx.x == 0 && cnt) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        mbar_expect_tx(&bar, cnt * 32u);
        bulk_g2s(sm, a4 + t0, cnt * 16u, &bar);
        bulk_g2s(sm + tile4, b4 + t0, cnt * 16u, &bar);
    }
    if (blockIdx.x == 0 && threadIdx.x < head + tail) {
        size_t i = threadIdx.x < head ? threadIdx.x : head + 4 * n4 + (threadIdx.x - head);
        const uint32_t r = op(a[i], b[i]);
        c[i] = r;
        s += r;
    }
    __syncthreads();
    if (cnt) {
        mbar_wait(&bar, 0);
        for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
            const uint4 r = apply4(op, sm[i], sm[tile4 + i]);
            st_stream(c4 + t0 + i, r);
            if (SUM) s += sum4(r);
        }
    }
    if (SUM) block_sum_to(acc, s);
}

// Persistent bulk-copy pipeline (variant 3): one or two CTAs per SM stream
// tiles through an S-stage shared-memory ring.  Thread 0 keeps S tile loads in
// flight with cp.async.bulk (each stage completes on its own mbarrier by
// transaction bytes) and writes each result tile back with a bulk store from
// one of two output buffers; the other threads only compute (LDS.128, REDC,
// STS.128).  Memory-level parallelism comes from the copy engine, not from
// resident warps, so the kernel streams with 4-8 warps per SM and leaves the
// SM's remaining warp slots and issue cycles to a co-running compute kernel
// (the pow ladder in bench.py's two-lane step).  Tile t goes to CTA
// t mod gridDim.x; one __syncthreads per tile.
template <int NIN, int S, class Op, bool SUM>
__global__ void __launch_bounds__(256) k_map_pipe(Op op, uint32_t *c, const uint32_t *a, const uint32_t *b,
                                                   uint32_t head, size_t n4, uint32_t tail, unsigned long long *acc,
                                                   uint32_t tile4) {
    extern __shared__ __align__(128) uint4 sm[];
    __shared__ __align__(8) uint64_t full[S];
    uint4 *sin = sm;                          // [S][NIN][tile4]
    uint4 *sout = sm + (size_t)S * NIN * tile4;  // [2][tile4]
    const uint4 *a4 = reinterpret_cast<const uint4 *>(a + head);
    const uint4 *b4 = reinterpret_cast<const uint4 *>((NIN == 2 ? b : a) + head);
    uint4 *c4 = reinterpret_cast<uint4 *>(c + head);
    const size_t ntiles = (n4 + tile4 - 1) / tile4;
    auto load = [&](size_t t, int st) {
        const uint32_t cnt = (uint32_t)(n4 - t * tile4 < tile4 ? n4 - t * tile4 : tile4);
        mbar_expect_tx(&full[st], cnt * 16u * NIN);
        bulk_g2s(sin + (size_t)st * NIN * tile4, a4 + t * tile4, cnt * 16u, &full[st]);
        if (NIN == 2) bulk_g2s(sin + ((size_t)st * NIN + 1) * tile4, b4 + t * tile4, cnt * 16u, &full[st]);
    };
    if (threadIdx.x == 0) {
        for (int st = 0; st < S; ++st) mbar_init(&full[st], 1);
        fence_mbar_init();
        for (int st = 0; st < S; ++st) {
            const size_t t = blockIdx.x + (size_t)st * gridDim.x;
            if (t < ntiles) load(t, st);
        }
    }
    unsigned long long s = 0;
    if (blockIdx.x == 0 && threadIdx.x < head + tail) {
        const size_t i = threadIdx.x < head ? threadIdx.x : head + 4 * n4 + (threadIdx.x - head);
        uint32_t r;
        if constexpr (NIN == 2) r = op(a[i], b[i]);
        else r = op(a[i]);
        c[i] = r;
        s += r;
    }
    __syncthreads();
    uint32_t it = 0;
    for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int st = (int)(it % S);
        const uint32_t cnt = (uint32_t)(n4 - t * tile4 < tile4 ? n4 - t * tile4 : tile4);
        mbar_wait(&full[st], (it / S) & 1u);
        const uint4 *ia = sin + (size_t)st * NIN * tile4, *ib = ia + tile4;
        uint4 *ob = sout + (size_t)(it & 1u) * tile4;
        for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
            uint4 r;
            if constexpr (NIN == 2) r = apply4(op, ia[i], ib[i]);
            else r = apply4(op, ia[i]);
            ob[i] = r;
            if (SUM) s += sum4(r);
        }
        fence_proxy_async_smem();
        // thread 0: the store issued last iteration (from the other output buffer) must have
        // finished reading it before anyone writes that buffer next iteration
        if (threadIdx.x == 0) bulk_wait_read0();
        __syncthreads();
        if (threadIdx.x == 0) {
            bulk_s2g(c4 + t * tile4, ob, cnt * 16u);
            bulk_commit();
            const size_t tn = t + (size_t)S * gridDim.x;  // refill this stage: everyone has read it
            if (tn < ntiles) load(tn, st);
        }
    }
    if (threadIdx.x == 0) bulk_wait0();  // the last stores read shared memory: finish before exit
    if (SUM) block_sum_to(acc, s);
}

// 32-bit path for operands that do not share an address mod 16
template <int U, class Op, bool SUM>
__global__ void __launch_bounds__(512) k_map2_scalar(Op op, uint32_t *c, const uint32_t *a, const uint32_t *b,
                                                       size_t n, unsigned long long *acc) {
    unsigned long long s = 0;
    const size_t tile = (size_t)U * blockDim.x;
    for (size_t t0 = (size_t)blockIdx.x * tile; t0 < n; t0 += (size_t)gridDim.x * tile) {
        uint32_t va[U], vb[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            size_t i = t0 + (size_t)k * blockDim.x + threadIdx.x;
            va[k] = i < n ? ld_stream1(a + i) : 0u;
            vb[k] = i < n ? ld_stream1(b + i) : 0u;
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            size_t i = t0 + (size_t)k * blockDim.x + threadIdx.x;
            if (i < n) {
                const uint32_t r = op(va[k], vb[k]);
                st_stream1(c + i, r);
                if (SUM) s += r;
            }
        }
    }
    if (SUM) block_sum_to(acc, s);
}

// ----------------------------------------------------------------- unary map
template <int U, class Op>
__global__ void __launch_bounds__(512) k_map1(Op op, uint32_t *out, const uint32_t *in, uint32_t head, size_t n4,
                                                uint32_t tail) {
    if (blockIdx.x == 0 && threadIdx.x < head + tail) {
        size_t i = threadIdx.x < head ? threadIdx.x : head + 4 * n4 + (threadIdx.x - head);
        out[i] = op(in[i]);
    }
    const uint4 *i4 = reinterpret_cast<const uint4 *>(in + head);
    uint4 *o4 = reinterpret_cast<uint4 *>(out + head);
    const size_t tile = (size_t)U * blockDim.x;
    const size_t ntiles_full = n4 / tile;
    size_t t = blockIdx.x;
    for (; t < ntiles_full; t += gridDim.x) {
        const size_t base = t * tile + threadIdx.x;
        uint4 v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) v[k] = ld_stream(i4 + base + (size_t)k * blockDim.x);
#pragma unroll
        for (int k = 0; k < U; ++k) st_stream(o4 + base + (size_t)k * blockDim.x, apply4(op, v[k]));
    }
    if (t == ntiles_full) {
        for (size_t i = t * tile + threadIdx.x; i < n4; i += blockDim.x) st_stream(o4 + i, apply4(op, ld_stream(i4 + i)));
    }
}

template <int U, class Op>
__global__ void __launch_bounds__(512) k_map1_scalar(Op op, uint32_t *out, const uint32_t *in, size_t n) {
    const size_t tile = (size_t)U * blockDim.x;
    for (size_t t0 = (size_t)blockIdx.x * tile; t0 < n; t0 += (size_t)gridDim.x * tile) {
        uint32_t v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            size_t i = t0 + (size_t)k * blockDim.x + threadIdx.x;
            v[k] = i < n ? ld_stream1(in + i) : 0u;
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            size_t i = t0 + (size_t)k * blockDim.x + threadIdx.x;
            if (i < n) st_stream1(out + i, op(v[k]));
        }
    }
}

// ------------------------------------------------------------------ checksum
template <int U>
__global__ void __launch_bounds__(512) k_sum(unsigned long long *acc, const uint32_t *x, uint32_t head, size_t n4,
                                               uint32_t tail) {
    unsigned long long s = 0;
    if (blockIdx.x == 0 && threadIdx.x < head + tail) {
        size_t i = threadIdx.x < head ? threadIdx.x : head + 4 * n4 + (threadIdx.x - head);
        s += x[i];
    }
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x + head);
    const size_t tile = (size_t)U * blockDim.x;
    for (size_t t0 = (size_t)blockIdx.x * tile; t0 < n4; t0 += (size_t)gridDim.x * tile) {
#pragma unroll
        for (int k = 0; k < U; ++k) {
            size_t i = t0 + (size_t)k * blockDim.x + threadIdx.x;
            if (i < n4) s += sum4(ld_stream(x4 + i));
        }
    }
    block_sum_to(acc, s);
}

// ------------------------------------------------------------------- helpers
template <bool SUM, class Op>
static mont_status_t launch_map2(const Op &op, uint32_t *c, const uint32_t *a, const uint32_t *b, size_t n,
                                 const Launch &L, cudaStream_t s, unsigned long long *acc = nullptr) {
    const int sms = sm_count();
    if (sms <= 0) return MONT_ECUDA;
    const uintptr_t pa = (uintptr_t)a, pb = (uintptr_t)b, pc = (uintptr_t)c;
    const bool flat = L.variant == 0;
    if (L.variant == 3 && same_mod16(pa, pb) && same_mod16(pa, pc)) {  // persistent bulk-copy pipeline
        const uint32_t head = head_elems(pa, n);
        const size_t n4 = (n - head) / 4;
        const uint32_t tail = (uint32_t)((n - head) % 4);
        const uint32_t tile4 = (uint32_t)((L.chunk > 0 ? L.chunk : 2048) / 4);
        constexpr int S = 4;
        const size_t smem = ((size_t)S * 2 + 2) * tile4 * 16;
        if (tile4 == 0 || smem > 227 * 1024 || L.threads > 256) return MONT_EINVAL_ARG;
        const size_t ntiles = (n4 + tile4 - 1) / tile4;
        size_t grid = (size_t)sms * (L.ctas_per_sm > 0 ? L.ctas_per_sm : 1);
        if (grid > ntiles) grid = ntiles;
        if (grid == 0) grid = 1;
        // (always set: the static mbarriers come on top of the dynamic size)
        if (cudaFuncSetAttribute(k_map_pipe<2, S, Op, SUM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return MONT_ECUDA;
        k_map_pipe<2, S, Op, SUM><<<(unsigned)grid, L.threads, smem, s>>>(op, c, a, b, head, n4, tail, acc, tile4);
        return launch_status();
    }
    if (L.variant == 2 && same_mod16(pa, pb) && same_mod16(pa, pc)) {  // bulk-copy (TMA) staged tiles
        const uint32_t head = head_elems(pa, n);
        const size_t n4 = (n - head) / 4;
        const uint32_t tail = (uint32_t)((n - head) % 4);
        const uint32_t tile4 = (uint32_t)((L.chunk > 0 ? L.chunk : 8192) / 4);
        const size_t smem = (size_t)tile4 * 32;
        if (tile4 == 0 || smem > 227 * 1024) return MONT_EINVAL_ARG;
        size_t grid = (n4 + tile4 - 1) / tile4;
        if (grid == 0) grid = 1;
        if (grid > 0x7fffffff) return MONT_EUNSUPPORTED;
        if (smem > 48 * 1024 &&
            cudaFuncSetAttribute(k_map2_tma<Op, SUM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
                cudaSuccess)
            return MONT_ECUDA;
        k_map2_tma<Op, SUM><<<(unsigned)grid, 256, smem, s>>>(op, c, a, b, head, n4, tail, acc, tile4);
        return launch_status();
    }
    if (same_mod16(pa, pb) && same_mod16(pa, pc)) {
        const uint32_t head = head_elems(pa, n);
        const size_t n4 = (n - head) / 4;
        const uint32_t tail = (uint32_t)((n - head) % 4);
        const size_t tile = (size_t)L.unroll * L.threads;
        size_t grid = flat ? (n4 + tile - 1) / tile : (size_t)sms * L.ctas_per_sm;
        const size_t need = (n4 + tile - 1) / tile;
        if (grid > need) grid = need;
        if (grid == 0) grid = 1;
        if (grid > 0x7fffffff) return MONT_EUNSUPPORTED;
        const dim3 g((unsigned)grid), bl((unsigned)L.threads);
        switch (L.unroll) {
            case 1: return launch_k(k_map2<1, Op, SUM>, g, bl, 0, s, L.flags, op, c, a, b, head, n4, tail, acc);
            case 2: return launch_k(k_map2<2, Op, SUM>, g, bl, 0, s, L.flags, op, c, a, b, head, n4, tail, acc);
            case 4: return launch_k(k_map2<4, Op, SUM>, g, bl, 0, s, L.flags, op, c, a, b, head, n4, tail, acc);
            default: return launch_k(k_map2<8, Op, SUM>, g, bl, 0, s, L.flags, op, c, a, b, head, n4, tail, acc);
        }
    } else {
        const size_t tile = (size_t)L.unroll * L.threads;
        size_t grid = (size_t)sms * L.ctas_per_sm;
        const size_t need = (n + tile - 1) / tile;
        if (grid > need) grid = need;
        switch (L.unroll) {
            case 1: k_map2_scalar<1, Op, SUM><<<(unsigned)grid, L.threads, 0, s>>>(op, c, a, b, n, acc); break;
            case 2: k_map2_scalar<2, Op, SUM><<<(unsigned)grid, L.threads, 0, s>>>(op, c, a, b, n, acc); break;
            case 4: k_map2_scalar<4, Op, SUM><<<(unsigned)grid, L.threads, 0, s>>>(op, c, a, b, n, acc); break;
            default: k_map2_scalar<8, Op, SUM><<<(unsigned)grid, L.threads, 0, s>>>(op, c, a, b, n, acc); break;
        }
    }
    return launch_status();
}

template <class Op>
static mont_status_t launch_map1(const Op &op, uint32_t *out, const uint32_t *in, size_t n, const Launch &L,
                                 cudaStream_t s) {
    const int sms = sm_count();
    if (sms <= 0) return MONT_ECUDA;
    const uintptr_t pi = (uintptr_t)in, po = (uintptr_t)out;
    if (L.variant == 3 && same_mod16(pi, po)) {  // persistent bulk-copy pipeline
        const uint32_t head = head_elems(pi, n);
        const size_t n4 = (n - head) / 4;
        const uint32_t tail = (uint32_t)((n - head) % 4);
        const uint32_t tile4 = (uint32_t)((L.chunk > 0 ? L.chunk : 2048) / 4);
        constexpr int S = 4;
        const size_t smem = ((size_t)S + 2) * tile4 * 16;
        if (tile4 == 0 || smem > 227 * 1024 || L.threads > 256) return MONT_EINVAL_ARG;
        const size_t ntiles = (n4 + tile4 - 1) / tile4;
        size_t grid = (size_t)sms * (L.ctas_per_sm > 0 ? L.ctas_per_sm : 1);
        if (grid > ntiles) grid = ntiles;
        if (grid == 0) grid = 1;
        if (cudaFuncSetAttribute(k_map_pipe<1, S, Op, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess)
            return MONT_ECUDA;
        k_map_pipe<1, S, Op, false><<<(unsigned)grid, L.threads, smem, s>>>(op, out, in, nullptr, head, n4, tail,
                                                                            nullptr, tile4);
        return launch_status();
    }
    if (same_mod16(pi, po)) {
        const uint32_t head = head_elems(pi, n);
        const size_t n4 = (n - head) / 4;
        const uint32_t tail = (uint32_t)((n - head) % 4);
        const size_t tile = (size_t)L.unroll * L.threads;
        size_t grid = L.variant == 0 ? (n4 + tile - 1) / tile : (size_t)sms * L.ctas_per_sm;
        const size_t need = (n4 + tile - 1) / tile;
        if (grid > need) grid = need;
        if (grid == 0) grid = 1;
        if (grid > 0x7fffffff) return MONT_EUNSUPPORTED;
        switch (L.unroll) {
            case 1: k_map1<1><<<(unsigned)grid, L.threads, 0, s>>>(op, out, in, head, n4, tail); break;
            case 2: k_map1<2><<<(unsigned)grid, L.threads, 0, s>>>(op, out, in, head, n4, tail); break;
            case 4: k_map1<4><<<(unsigned)grid, L.threads, 0, s>>>(op, out, in, head, n4, tail); break;
            default: k_map1<8><<<(unsigned)grid, L.threads, 0, s>>>(op, out, in, head, n4, tail); break;
        }
    } else {
        const size_t tile = (size_t)L.unroll * L.threads;
        size_t grid = (size_t)sms * L.ctas_per_sm;
        const size_t need = (n + tile - 1) / tile;
        if (grid > need) grid = need;
        switch (L.unroll) {
            case 1: k_map1_scalar<1><<<(unsigned)grid, L.threads, 0, s>>>(op, out, in, n); break;
            case 2: k_map1_scalar<2><<<(unsigned)grid, L.threads, 0, s>>>(op, out, in, n); break;
            case 4: k_map1_scalar<4><<<(unsigned)grid, L.threads, 0, s>>>(op, out, in, n); break;
            default: k_map1_scalar<8><<<(unsigned)grid, L.threads, 0, s>>>(op, out, in, n); break;
        }
    }
    return launch_status();
}

// Defaults from the B200 sweep recorded in DESIGN.md §6: a flat grid (variant
// 0, one tile of `threads` uint4 per CTA, ~65k CTAs at 2^26) beats every
// persistent grid-stride shape by ~10 % -- the block scheduler balances the
// slow and fast SMs dynamically, a static round-robin deal does not.
static const Launch kMulVecDefault{256, 4, 1, 0, 0};

// R^-1 mod P from the context: R R^-1 - P P' = 1 with P' = pneg
static OpFmont fmont_op(const mont_ctx_t *ctx) {
    const uint32_t rinv = (uint32_t)((1ull + (unsigned long long)ctx->p * ctx->pneg) >> 32);
    return OpFmont{(double)ctx->p, 1.0 / (double)ctx->p, (double)rinv};
}
static const Launch kMap1Default{512, 4, 2, 0, 0};
// fused checksum: 2 uint4 per thread x 512 threads -> one atomic per 4096 words
static const Launch kMulVecSumDefault{512, 4, 2, 0, 0};

}  // namespace mont

using namespace mont;

extern "C" mont_status_t mont_mul_vec_ex(const mont_ctx_t *ctx, uint32_t *c, const uint32_t *a, const uint32_t *b,
                                         size_t n, const mont_launch_t *cfg, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (n == 0) return MONT_OK;
    if (!a || !b || !c || ((uintptr_t)a | (uintptr_t)b | (uintptr_t)c) & 3u) return MONT_EINVAL_ARG;
    Launch L = resolve(cfg, kMulVecDefault);
    if (L.variant == 4) {  // FP64-pipe products, flat grid
        L.variant = 0;
        if (!launch_ok(L)) return MONT_EINVAL_ARG;
        return launch_map2<false>(fmont_op(ctx), c, a, b, n, L, stream);
    }
    if (!launch_ok(L) || L.variant > 3) return MONT_EINVAL_ARG;
    return launch_map2<false>(OpMul{ctx->p, 0u - ctx->pneg}, c, a, b, n, L, stream);
}

extern "C" mont_status_t mont_mul_vec(const mont_ctx_t *ctx, uint32_t *c, const uint32_t *a, const uint32_t *b,
                                      size_t n, cudaStream_t stream) {
    return mont_mul_vec_ex(ctx, c, a, b, n, nullptr, stream);
}

extern "C" mont_status_t mont_mul_vec_checksum_ex(const mont_ctx_t *ctx, uint32_t *c, const uint32_t *a,
                                                  const uint32_t *b, size_t n, unsigned long long *acc,
                                                  const mont_launch_t *cfg, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (n == 0) return MONT_OK;
    if (!a || !b || !c || !acc || ((uintptr_t)a | (uintptr_t)b | (uintptr_t)c) & 3u || ((uintptr_t)acc & 7u))
        return MONT_EINVAL_ARG;
    Launch L = resolve(cfg, kMulVecSumDefault);
    if (L.variant == 4) {  // FP64-pipe products, flat grid
        L.variant = 0;
        if (!launch_ok(L)) return MONT_EINVAL_ARG;
        return launch_map2<true>(fmont_op(ctx), c, a, b, n, L, stream, acc);
    }
    if (!launch_ok(L) || L.variant > 3) return MONT_EINVAL_ARG;
    return launch_map2<true>(OpMul{ctx->p, 0u - ctx->pneg}, c, a, b, n, L, stream, acc);
}

extern "C" mont_status_t mont_mul_vec_checksum(const mont_ctx_t *ctx, uint32_t *c, const uint32_t *a,
                                               const uint32_t *b, size_t n, unsigned long long *acc,
                                               cudaStream_t stream) {
    return mont_mul_vec_checksum_ex(ctx, c, a, b, n, acc, nullptr, stream);
}

extern "C" mont_status_t to_mont_ex(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *in, size_t n,
                                    const mont_launch_t *cfg, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (n == 0) return MONT_OK;
    if (!in || !out || ((uintptr_t)in | (uintptr_t)out) & 3u) return MONT_EINVAL_ARG;
    const Launch L = resolve(cfg, kMap1Default);
    if (!launch_ok(L) || L.variant > 3) return MONT_EINVAL_ARG;
    return launch_map1(OpTo{ctx->p, 0u - ctx->pneg, ctx->r2}, out, in, n, L, stream);
}

extern "C" mont_status_t to_mont(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *in, size_t n,
                                 cudaStream_t stream) {
    return to_mont_ex(ctx, out, in, n, nullptr, stream);
}

extern "C" mont_status_t from_mont_ex(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *in, size_t n,
                                      const mont_launch_t *cfg, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (n == 0) return MONT_OK;
    if (!in || !out || ((uintptr_t)in | (uintptr_t)out) & 3u) return MONT_EINVAL_ARG;
    const Launch L = resolve(cfg, kMap1Default);
    if (!launch_ok(L) || L.variant > 3) return MONT_EINVAL_ARG;
    return launch_map1(OpFrom{ctx->p, 0u - ctx->pneg}, out, in, n, L, stream);
}

extern "C" mont_status_t from_mont(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *in, size_t n,
                                   cudaStream_t stream) {
    return from_mont_ex(ctx, out, in, n, nullptr, stream);
}

extern "C" mont_status_t mont_checksum(const mont_ctx_t *ctx, unsigned long long *acc, const uint32_t *x, size_t n,
                                       cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (n == 0) return MONT_OK;
    if (!acc || !x || ((uintptr_t)acc & 7u) || ((uintptr_t)x & 3u)) return MONT_EINVAL_ARG;
    const int sms = sm_count();
    if (sms <= 0) return MONT_ECUDA;
    const uint32_t head = head_elems((uintptr_t)x, n);
    const size_t n4 = (n - head) / 4;
    const uint32_t tail = (uint32_t)((n - head) % 4);
    const int threads = 256;
    const size_t tile = 4 * (size_t)threads;
    size_t grid = (n4 + tile - 1) / tile;  // flat grid
    if (grid == 0) grid = 1;
    if (grid > 0x7fffffff) grid = 0x7fffffff;
    k_sum<4><<<(unsigned)grid, threads, 0, stream>>>(acc, x, head, n4, tail);
    return launch_status();
}

extern "C" mont_status_t mb_triad(uint32_t *c, const uint32_t *a, const uint32_t *b, size_t n,
                                  const mont_launch_t *cfg, cudaStream_t stream) {
    if (n == 0) return MONT_OK;
    if (!a || !b || !c) return MONT_EINVAL_ARG;
    const Launch L = resolve(cfg, kMulVecDefault);
    if (!launch_ok(L) || L.variant > 3) return MONT_EINVAL_ARG;
    return launch_map2<false>(OpXor{}, c, a, b, n, L, stream);
}

extern "C" mont_status_t mb_copy(uint32_t *out, const uint32_t *in, size_t n, const mont_launch_t *cfg,
                                 cudaStream_t stream) {
    if (n == 0) return MONT_OK;
    if (!in || !out) return MONT_EINVAL_ARG;
    const Launch L = resolve(cfg, kMap1Default);
    if (!launch_ok(L) || L.variant > 3) return MONT_EINVAL_ARG;
    return launch_map1(OpCopy{}, out, in, n, L, stream);
}

extern "C" int mont_sm_count(void) { return sm_count(); }

extern "C" mont_status_t barrett_ctx_init(barrett_ctx_t *ctx, uint32_t p) {
    if (!ctx) return MONT_EINVAL_ARG;
    if ((p & 1u) == 0u || p < 3u || p >= 0x80000000u) return MONT_EINVAL_P;
    uint32_t k = 0;
    while ((1ull << k) < p) ++k;  // ceil(log2 P)
    ctx->p = p;
    ctx->k = k;
    ctx->pprime = (uint32_t)((1ull << (2 * k)) / p);
    ctx->pad = 0;
    return MONT_OK;
}

static bool barrett_ok(const barrett_ctx_t *c) {
    return c && (c->p & 1u) && c->p >= 3u && c->p < 0x80000000u && c->k <= 31 && (1ull << c->k) >= c->p &&
           c->pprime == (uint32_t)((1ull << (2 * c->k)) / c->p);
}

extern "C" mont_status_t barrett_mul_vec(const barrett_ctx_t *ctx, uint32_t *c, const uint32_t *a, const uint32_t *b,
                                         size_t n, cudaStream_t stream) {
    if (!barrett_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (n == 0) return MONT_OK;
    if (!a || !b || !c || ((uintptr_t)a | (uintptr_t)b | (uintptr_t)c) & 3u) return MONT_EINVAL_ARG;
    return launch_map2<false>(OpBarrett{BarrettDev{ctx->p, ctx->k, ctx->pprime}}, c, a, b, n, kMulVecDefault, stream);
}
