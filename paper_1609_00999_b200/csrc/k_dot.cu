// k_dot.cu -- batched modular dot products with lazy reduction (include/mont_dot.h;
// SURVEY.md §8(f) NEXT #4).  HBM-bound on reading A (4 B/elem); each term is
// one signed REDC (mont_core.cuh sredc, 5 FMAHeavy slots) and the terms are
// accumulated exactly in int64, so the canonicalising correction of Alg. 2
// is paid once per row instead of once per product.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mont_dot.h"
#include "../../include/mont_ext.h"
#include "abi_util.h"
#include "tma.cuh"

namespace mont {

// One CTA per row.  PF = true: software-pipelined -- the next trip's U uint4 of the row are
// loaded before this trip's products, so each thread always has a trip of A in flight (the row
// stream is latency-bound otherwise: every trip waits for its own loads).
template <int U, bool PF = false>
__global__ void __launch_bounds__(256) k_dot(Ctx c, uint32_t *out, const uint32_t *A, const uint32_t *x, size_t len,
                                              bool vec) {
    const uint32_t *row = A + (size_t)blockIdx.x * len;
    const int32_t p = (int32_t)c.p, pinv = (int32_t)c.pinv;
    long long s = 0;
    if (vec) {  // row and x 16-byte aligned, len % 4 == 0
        const uint4 *r4 = reinterpret_cast<const uint4 *>(row);
        const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
        const size_t n4 = len >> 2;
        const size_t stride = (size_t)U * blockDim.x;
        size_t i = threadIdx.x;
        if (PF) {
            uint4 an[U];
            const bool first = i + (U - 1) * blockDim.x < n4;
            if (first) {
#pragma unroll
                for (int k = 0; k < U; ++k) an[k] = ld_stream(r4 + i + k * blockDim.x);
            }
            for (; i + (U - 1) * blockDim.x < n4; i += stride) {
                uint4 a[U], b[U];
#pragma unroll
                for (int k = 0; k < U; ++k) a[k] = an[k];
                if (i + stride + (U - 1) * blockDim.x < n4) {
#pragma unroll
                    for (int k = 0; k < U; ++k) an[k] = ld_stream(r4 + i + stride + k * blockDim.x);
                }
#pragma unroll
                for (int k = 0; k < U; ++k) b[k] = __ldg(x4 + i + k * blockDim.x);
#pragma unroll
                for (int k = 0; k < U; ++k)
                    s += (long long)sredc((int32_t)a[k].x, (int32_t)b[k].x, p, pinv) +
                         (long long)sredc((int32_t)a[k].y, (int32_t)b[k].y, p, pinv) +
                         (long long)sredc((int32_t)a[k].z, (int32_t)b[k].z, p, pinv) +
                         (long long)sredc((int32_t)a[k].w, (int32_t)b[k].w, p, pinv);
            }
        } else {
            for (; i + (U - 1) * blockDim.x < n4; i += stride) {
                uint4 a[U], b[U];
#pragma unroll
                for (int k = 0; k < U; ++k) a[k] = ld_stream(r4 + i + k * blockDim.x);
#pragma unroll
                for (int k = 0; k < U; ++k) b[k] = __ldg(x4 + i + k * blockDim.x);
#pragma unroll
                for (int k = 0; k < U; ++k)
                    s += (long long)sredc((int32_t)a[k].x, (int32_t)b[k].x, p, pinv) +
                         (long long)sredc((int32_t)a[k].y, (int32_t)b[k].y, p, pinv) +
                         (long long)sredc((int32_t)a[k].z, (int32_t)b[k].z, p, pinv) +
                         (long long)sredc((int32_t)a[k].w, (int32_t)b[k].w, p, pinv);
            }
        }
        for (; i < n4; i += blockDim.x) {
            const uint4 a = ld_stream(r4 + i), b = __ldg(x4 + i);
            s += (long long)sredc((int32_t)a.x, (int32_t)b.x, p, pinv) + (long long)sredc((int32_t)a.y, (int32_t)b.y, p, pinv) +
                 (long long)sredc((int32_t)a.z, (int32_t)b.z, p, pinv) + (long long)sredc((int32_t)a.w, (int32_t)b.w, p, pinv);
        }
    } else {
        for (size_t j = threadIdx.x; j < len; j += blockDim.x)
            s += sredc((int32_t)ld_stream1(row + j), (int32_t)__ldg(x + j), p, pinv);
    }
    // block reduction of the exact int64 partial sums
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    __shared__ long long part[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) part[wid] = s;
    __syncthreads();
    if (wid == 0) {
        s = lane < (int)(blockDim.x >> 5) ? part[lane] : 0ll;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (lane == 0) {
            long long r = s % (long long)c.p;  // the single reduction of the row
            if (r < 0) r += c.p;
            out[blockIdx.x] = (uint32_t)r;
        }
    }
}

// R rows per CTA against the same x: each thread loads x[i] once and multiplies it into the R rows
// at the same positions (x's L1 traffic and its registers shrink by R per A byte).  Row-major A,
// len % 4 == 0 and 16-byte aligned A, x (the launcher checks; otherwise k_dot runs).
template <int R, int U>
__global__ void __launch_bounds__(256) k_dot_rows(Ctx c, uint32_t *out, const uint32_t *A, const uint32_t *x,
                                                   size_t batch, size_t len) {
    const size_t r0 = (size_t)blockIdx.x * R;
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
    const size_t n4 = len >> 2;
    const int32_t p = (int32_t)c.p, pinv = (int32_t)c.pinv;
    long long s[R];
#pragma unroll
    for (int r = 0; r < R; ++r) s[r] = 0;
    for (size_t i = threadIdx.x; i < n4; i += (size_t)U * blockDim.x) {
        uint4 a[R][U], b[U];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int k = 0; k < U; ++k)
                if (r0 + r < batch && i + k * blockDim.x < n4)
                    a[r][k] = ld_stream(reinterpret_cast<const uint4 *>(A + (r0 + r) * len) + i + k * blockDim.x);
                else
                    a[r][k] = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int k = 0; k < U; ++k) b[k] = i + k * blockDim.x < n4 ? __ldg(x4 + i + k * blockDim.x) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int k = 0; k < U; ++k)
                s[r] += (long long)sredc((int32_t)a[r][k].x, (int32_t)b[k].x, p, pinv) +
                        (long long)sredc((int32_t)a[r][k].y, (int32_t)b[k].y, p, pinv) +
                        (long long)sredc((int32_t)a[r][k].z, (int32_t)b[k].z, p, pinv) +
                        (long long)sredc((int32_t)a[r][k].w, (int32_t)b[k].w, p, pinv);
    }
    __shared__ long long part[R][8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        long long v = s[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) part[r][wid] = v;
    }
    __syncthreads();
    if (wid < R && r0 + wid < batch) {
        long long v = lane < (int)(blockDim.x >> 5) ? part[wid][lane] : 0ll;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) {
            long long rr = v % (long long)c.p;
            if (rr < 0) rr += c.p;
            out[r0 + wid] = (uint32_t)rr;
        }
    }
}

// Split rows (the default for rows of >= 2 chunks): CTA b computes chunk b % S of row b / S --
// `chunk` elements, all of a thread's loads issued before any product (a flat grid of short CTAs
// streams like mont_mul_vec's, instead of 4096 one-row CTAs in 3.5 waves) -- reduces its exact
// int64 partial to a canonical residue and adds it into out[row] (zeroed by the launcher) with a
// modular compare-and-swap loop.  Exact: every partial and every sum is reduced into [0, P).
template <int U>
__global__ void __launch_bounds__(256) k_dot_split(Ctx c, uint32_t *out, const uint32_t *A, const uint32_t *x,
                                                    size_t len, uint32_t S, uint32_t chunk) {
    const size_t row = blockIdx.x / S;
    const uint32_t part = blockIdx.x % S;
    const size_t j0 = (size_t)part * chunk;
    const size_t j1 = j0 + chunk < len ? j0 + chunk : len;
    const uint4 *r4 = reinterpret_cast<const uint4 *>(A + row * len + j0);
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x + j0);
    const size_t n4 = (j1 - j0) >> 2;  // len % 4 == 0 and chunk % 4 == 0 on this path
    const int32_t p = (int32_t)c.p, pinv = (int32_t)c.pinv;
    long long s = 0;
    size_t i = threadIdx.x;
    for (; i + (U - 1) * blockDim.x < n4; i += U * blockDim.x) {
        uint4 a[U], b[U];
#pragma unroll
        for (int k = 0; k < U; ++k) a[k] = ld_stream(r4 + i + k * blockDim.x);
#pragma unroll
        for (int k = 0; k < U; ++k) b[k] = __ldg(x4 + i + k * blockDim.x);
#pragma unroll
        for (int k = 0; k < U; ++k)
            s += (long long)sredc((int32_t)a[k].x, (int32_t)b[k].x, p, pinv) +
                 (long long)sredc((int32_t)a[k].y, (int32_t)b[k].y, p, pinv) +
                 (long long)sredc((int32_t)a[k].z, (int32_t)b[k].z, p, pinv) +
                 (long long)sredc((int32_t)a[k].w, (int32_t)b[k].w, p, pinv);
    }
    for (; i < n4; i += blockDim.x) {
        const uint4 a = ld_stream(r4 + i), b = __ldg(x4 + i);
        s += (long long)sredc((int32_t)a.x, (int32_t)b.x, p, pinv) + (long long)sredc((int32_t)a.y, (int32_t)b.y, p, pinv) +
             (long long)sredc((int32_t)a.z, (int32_t)b.z, p, pinv) + (long long)sredc((int32_t)a.w, (int32_t)b.w, p, pinv);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    __shared__ long long partw[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) partw[wid] = s;
    __syncthreads();
    if (wid == 0) {
        s = lane < (int)(blockDim.x >> 5) ? partw[lane] : 0ll;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (lane == 0) {
            long long r = s % (long long)c.p;
            if (r < 0) r += c.p;
            if (S == 1) {
                out[row] = (uint32_t)r;
            } else {
                uint32_t old = out[row], assumed;
                do {  // out[row] = (out[row] + r) mod P, both in [0, P)
                    assumed = old;
                    const uint32_t nv = assumed + (uint32_t)r;
                    old = atomicCAS(out + row, assumed, umin(nv, nv - c.p));
                } while (old != assumed);
            }
        }
    }
}


// Copy-engine streaming (variant 8): a persistent grid (ctas_per_sm x SMs CTAs of 256 threads);
// CTA b owns rows b, b + G, b + 2G, ... (G = gridDim.x) and streams them as tiles of tile4 uint4
// through an S-stage shared-memory ring filled by cp.async.bulk (one mbarrier per stage,
// transaction-byte completion): each stage holds a tile of A and the matching tile of x, so S
// tiles are always in flight whatever the warps are doing and x never competes with the ring for
// L1.  The partial sum of a row is reduced across the CTA when its last tile has been consumed
// (part[] double-buffered by row parity).
template <int S>
__global__ void __launch_bounds__(256) k_dot_pipe(Ctx c, uint32_t *out, const uint32_t *A, const uint32_t *x,
                                                   size_t batch, size_t len, uint32_t tile4) {
    extern __shared__ __align__(128) uint4 ring[];  // [S][2][tile4]: A tile, x tile
    __shared__ __align__(8) uint64_t full[S];
    __shared__ long long part[2][8];
    const size_t n4 = len >> 2;
    const uint32_t tpr = (uint32_t)((n4 + tile4 - 1) / tile4);  // tiles per row
    const size_t mine = batch > blockIdx.x ? (batch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const size_t ntiles = mine * tpr;
    // producer cursor (thread 0): the (row, tile) of the next load, advanced without divisions
    uint32_t pk = 0, prow = 0;
    auto load_next = [&](int st) {
        const size_t row = blockIdx.x + (size_t)prow * gridDim.x;
        const size_t c0 = (size_t)pk * tile4;
        const uint32_t cnt = (uint32_t)(n4 - c0 < tile4 ? n4 - c0 : tile4);
        mbar_expect_tx(&full[st], cnt * 32u);
        bulk_g2s(ring + (size_t)st * 2 * tile4, reinterpret_cast<const uint4 *>(A + row * len) + c0, cnt * 16u,
                 &full[st]);
        bulk_g2s(ring + ((size_t)st * 2 + 1) * tile4, reinterpret_cast<const uint4 *>(x) + c0, cnt * 16u, &full[st]);
        if (++pk == tpr) pk = 0, ++prow;
    };
    if (threadIdx.x == 0) {
        for (int st = 0; st < S; ++st) mbar_init(&full[st], 1);
        fence_mbar_init();
        for (int st = 0; st < S; ++st)
            if ((size_t)st < ntiles) load_next(st);
    }
    __syncthreads();
    const int32_t p = (int32_t)c.p, pinv = (int32_t)c.pinv;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long s = 0;
    uint32_t kin = 0, rk = 0, st = 0, phase = 0;  // consumer cursor
    for (size_t k = 0; k < ntiles; ++k) {
        const size_t c0 = (size_t)kin * tile4;
        const uint32_t cnt = (uint32_t)(n4 - c0 < tile4 ? n4 - c0 : tile4);
        mbar_wait(&full[st], phase);
        const uint4 *ta = ring + (size_t)st * 2 * tile4, *tx = ta + tile4;
        for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
            const uint4 a = ta[i], b = tx[i];
            s += (long long)sredc((int32_t)a.x, (int32_t)b.x, p, pinv) + (long long)sredc((int32_t)a.y, (int32_t)b.y, p, pinv) +
                 (long long)sredc((int32_t)a.z, (int32_t)b.z, p, pinv) + (long long)sredc((int32_t)a.w, (int32_t)b.w, p, pinv);
        }
        const bool row_end = kin == tpr - 1;
        if (row_end) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
            if (lane == 0) part[rk & 1][wid] = s;
            s = 0;
        }
        __syncthreads();  // stage st consumed by everyone (and part[] written)
        if (threadIdx.x == 0 && k + S < ntiles) load_next((int)st);
        if (row_end && wid == 0) {
            long long r = lane < (int)(blockDim.x >> 5) ? part[rk & 1][lane] : 0ll;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
            if (lane == 0) {
                r %= (long long)c.p;  // the single reduction of the row
                if (r < 0) r += c.p;
                out[blockIdx.x + (size_t)rk * gridDim.x] = (uint32_t)r;
            }
        }
        if (row_end) kin = 0, ++rk;
        else ++kin;
        if (++st == S) st = 0, phase ^= 1u;
    }
}

}  // namespace mont

using namespace mont;

extern "C" mont_status_t mont_dot_ex(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *A, const uint32_t *x,
                                     size_t batch, size_t len, const mont_launch_t *cfg, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (batch == 0) return MONT_OK;
    if (len == 0 || len >= (1ull << 32)) return MONT_EINVAL_ARG;
    if (!out || !A || !x || ((uintptr_t)out | (uintptr_t)A | (uintptr_t)x) & 3u) return MONT_EINVAL_ARG;
    if (batch > 0x7fffffffu) return MONT_EUNSUPPORTED;
    const int variant = cfg ? cfg->variant : 0;
    const int chunk_req = cfg ? cfg->chunk : 0;
    if (variant < 0 || variant > 8 || chunk_req < 0 || (chunk_req % 1024) != 0) return MONT_EINVAL_ARG;
    const bool vec = (len % 4 == 0) && (((uintptr_t)A | (uintptr_t)x) & 15u) == 0;
    if (variant == 8 && vec) {
        const int k = cfg && cfg->ctas_per_sm ? cfg->ctas_per_sm : 2;
        const uint32_t tile4 = (chunk_req ? (uint32_t)chunk_req : 4096u) / 4u;
        // default stage count: 4, or 2 where 4 would not fit
        const int stages = cfg && cfg->unroll ? cfg->unroll : ((size_t)4 * tile4 * 32 <= 200 * 1024 ? 4 : 2);
        if ((stages != 2 && stages != 4 && stages != 8) || k < 1 || k > 8) return MONT_EINVAL_ARG;
        const size_t smem = (size_t)stages * tile4 * 32;
        if (smem > 200 * 1024) return MONT_EINVAL_ARG;
        const int sms = sm_count();
        if (sms <= 0) return MONT_ECUDA;
        size_t grid = (size_t)sms * k;
        if (grid > batch) grid = batch;
        const Ctx c = to_dev(ctx);
#define MONT_DOT_PIPE(SS)                                                                                       \
    if (smem > 48 * 1024 &&                                                                                     \
        cudaFuncSetAttribute(k_dot_pipe<SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) \
        return MONT_ECUDA;                                                                                      \
    k_dot_pipe<SS><<<(unsigned)grid, 256, smem, stream>>>(c, out, A, x, batch, len, tile4);
        if (stages == 2) { MONT_DOT_PIPE(2) } else if (stages == 4) { MONT_DOT_PIPE(4) } else { MONT_DOT_PIPE(8) }
#undef MONT_DOT_PIPE
        return launch_status();
    }
    const uint32_t chunk = chunk_req ? (uint32_t)chunk_req : 4096u;  // 4 uint4 per thread of 256
    const size_t S = (len + chunk - 1) / chunk;
    if (variant == 5 && vec && S >= 2 && batch * S <= 0x7fffffffu) {
        if (cudaMemsetAsync(out, 0, batch * sizeof(uint32_t), stream) != cudaSuccess) return MONT_ECUDA;
        k_dot_split<4><<<(unsigned)(batch * S), 256, 0, stream>>>(to_dev(ctx), out, A, x, len, (uint32_t)S, chunk);
        return launch_status();
    }
    const Ctx c = to_dev(ctx);
    if ((variant == 6 || variant == 7) && vec) {
        if (variant == 6) k_dot_rows<2, 2><<<(unsigned)((batch + 1) / 2), 256, 0, stream>>>(c, out, A, x, batch, len);
        else k_dot_rows<4, 1><<<(unsigned)((batch + 3) / 4), 256, 0, stream>>>(c, out, A, x, batch, len);
        return launch_status();
    }
    switch (variant) {
        case 2: k_dot<8, false><<<(unsigned)batch, 256, 0, stream>>>(c, out, A, x, len, vec); break;
        case 3: k_dot<4, true><<<(unsigned)batch, 256, 0, stream>>>(c, out, A, x, len, vec); break;
        case 4: k_dot<8, true><<<(unsigned)batch, 256, 0, stream>>>(c, out, A, x, len, vec); break;
        default: k_dot<4, false><<<(unsigned)batch, 256, 0, stream>>>(c, out, A, x, len, vec); break;  // 0, 1, 5-8
    }
    return launch_status();
}

extern "C" mont_status_t mont_dot(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *A, const uint32_t *x,
                                  size_t batch, size_t len, cudaStream_t stream) {
    return mont_dot_ex(ctx, out, A, x, batch, len, nullptr, stream);
}
