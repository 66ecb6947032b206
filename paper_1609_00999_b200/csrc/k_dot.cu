// k_dot.cu -- batched modular dot products with lazy reduction (include/mont_dot.h;
// SURVEY.md §8(f) NEXT #4).  HBM-bound on reading A (4 B/elem); each term is
// one signed REDC (mont_core.cuh sredc, 5 FMAHeavy slots) and the terms are
// accumulated exactly in int64, so the canonicalising correction of Alg. 2
// is paid once per row instead of once per product.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mont_dot.h"
#include "abi_util.h"

namespace mont {

template <int U>
__global__ void __launch_bounds__(256) k_dot(Ctx c, uint32_t *out, const uint32_t *A, const uint32_t *x, size_t len,
                                              bool vec) {
    const uint32_t *row = A + (size_t)blockIdx.x * len;
    const int32_t p = (int32_t)c.p, pinv = (int32_t)c.pinv;
    long long s = 0;
    if (vec) {  // row and x 16-byte aligned, len % 4 == 0
        const uint4 *r4 = reinterpret_cast<const uint4 *>(row);
        const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
        const size_t n4 = len >> 2;
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

}  // namespace mont

using namespace mont;

extern "C" mont_status_t mont_dot(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *A, const uint32_t *x,
                                  size_t batch, size_t len, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (batch == 0) return MONT_OK;
    if (len == 0 || len >= (1ull << 32)) return MONT_EINVAL_ARG;
    if (!out || !A || !x || ((uintptr_t)out | (uintptr_t)A | (uintptr_t)x) & 3u) return MONT_EINVAL_ARG;
    if (batch > 0x7fffffffu) return MONT_EUNSUPPORTED;
    const bool vec = (len % 4 == 0) && (((uintptr_t)A | (uintptr_t)x) & 15u) == 0;
    k_dot<4><<<(unsigned)batch, 256, 0, stream>>>(to_dev(ctx), out, A, x, len, vec);
    return launch_status();
}
