// synth.cu -- device implementation of the seeded input generator (K7).
//
// The same counter-based function as synth/__init__.py:
// SplitMix64's output mix (Steele, Lea, Flood 2014) applied to
// seed + (stream * 2^40 + i + 1) * GAMMA.  Each side implements it on its own
// (no shared code); tests/test_gpu_synth.py checks they agree.  It lets the
// bench materialise multi-GiB inputs directly in HBM; no arithmetic of the
// Montgomery method happens here.
#include <cuda_runtime.h>
#include <stdint.h>

#include "abi_util.h"

namespace mont {

__device__ __forceinline__ uint64_t sm_mix(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

__device__ __forceinline__ uint64_t sm_h(uint64_t seed, uint32_t stream, uint64_t i) {
    return sm_mix(seed + (((uint64_t)stream << 40) + i + 1ull) * 0x9E3779B97F4A7C15ull);
}

__global__ void __launch_bounds__(256) k_synth(uint32_t *out, size_t n, uint64_t seed, uint32_t stream, uint64_t start,
                                                uint32_t p, int mode, int specials) {
    for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
        const uint64_t i = start + k;
        const uint64_t h = sm_h(seed, stream, i);
        uint32_t v;
        if (mode == 0) v = (uint32_t)__umul64hi(h, (uint64_t)p);
        else if (mode == 1) v = 1u + (uint32_t)__umul64hi(h, (uint64_t)(p - 1u));
        else v = (uint32_t)(h >> 33);
        if (specials) {
            const uint32_t s = (uint32_t)(sm_h(seed, stream + 16u, i) % 300ull);
            if (s == 0) v = 0u;
            else if (s == 1) v = 1u;
            else if (s == 2) v = p - 1u;
        }
        out[k] = v;
    }
}

}  // namespace mont

using namespace mont;

extern "C" mont_status_t synth_fill(uint32_t *out, size_t n, uint64_t seed, uint32_t stream, uint64_t start,
                                    uint32_t p, int mode, int specials, cudaStream_t s) {
    if (n == 0) return MONT_OK;
    if (!out || mode < 0 || mode > 2) return MONT_EINVAL_ARG;
    if (mode != 2 && p < 2) return MONT_EINVAL_ARG;
    const int sms = sm_count();
    if (sms <= 0) return MONT_ECUDA;
    size_t grid = (n + 255) / 256;
    if (grid > (size_t)sms * 16) grid = (size_t)sms * 16;
    k_synth<<<(unsigned)grid, 256, 0, s>>>(out, n, seed, stream, start, p, mode, specials);
    return launch_status();
}
