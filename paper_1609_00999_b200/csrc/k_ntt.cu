// k_ntt.cu -- batched radix-2 NTT with Montgomery twiddle products
// (include/mont_ntt.h).
//
// One CTA per row: the row is loaded from HBM once in bit-reversed order into
// shared memory, all log_n butterfly stages run there (one __syncthreads per
// stage), and the row is written back once -- 8 B of HBM traffic per element
// and (N/2) log_n Montgomery products per row.  Twiddles come from the
// caller's Montgomery-form table through the read-only path (L1-resident
// across the CTAs of an SM).  The butterfly multiplies a PLAIN residue by a
// Montgomery-form twiddle, so REDC(v, w-bar) = v w mod P stays plain
// (REDC(x-bar, y-bar) of two residues is the residue of xy; one
// plain operand makes the product plain).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mont_ntt.h"
#include "abi_util.h"

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
        const int tshift = log_n - st;
        for (uint32_t t = threadIdx.x; t < half_n; t += blockDim.x) {
            const uint32_t pos = t & hmask;
            const uint32_t i = ((t >> (st - 1)) << st) | pos;
            const uint32_t j = i + hmask + 1u;
            const uint32_t v = redc(s[j], __ldg(tw + (pos << tshift)), c.p, c.pinv);
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

}  // namespace mont

using namespace mont;

extern "C" mont_status_t mont_ntt(const mont_ctx_t *ctx, uint32_t *data, size_t batch, int log_n, const uint32_t *tw,
                                  uint32_t scale, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (log_n < 1 || log_n > 15) return MONT_EUNSUPPORTED;
    if (batch == 0) return MONT_OK;
    if (!data || !tw || ((uintptr_t)data & 3u) || ((uintptr_t)tw & 3u) || scale >= ctx->p) return MONT_EINVAL_ARG;
    if (batch > 0x7fffffffu) return MONT_EUNSUPPORTED;
    const uint32_t N = 1u << log_n;
    int threads = (int)(N / 2 < 1024 ? N / 2 : 1024);
    if (threads < 32) threads = 32;
    const size_t smem = (size_t)N * 4;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(k_ntt_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return MONT_ECUDA;
    k_ntt_smem<<<(unsigned)batch, threads, smem, stream>>>(to_dev(ctx), data, log_n, tw, scale);
    return launch_status();
}
