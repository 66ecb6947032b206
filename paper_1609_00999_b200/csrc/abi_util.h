// abi_util.h -- host-side helpers shared by the extern "C" launchers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mont.h"
#include "../../include/mont_ext.h"
#include "mont_core.cuh"

namespace mont {

inline Ctx to_dev(const mont_ctx_t *c) { return Ctx{c->p, 0u - c->pneg, c->r1, c->r2}; }

// a context is usable if it came from mont_ctx_init: odd p in [3, 2^31) and
// p * pneg = -1 (mod 2^32).  Cheap, catches uninitialised structs.
inline bool ctx_ok(const mont_ctx_t *c) {
    return c && (c->p & 1u) && c->p >= 3u && c->p < 0x80000000u && (uint32_t)(c->p * c->pneg) == 0xFFFFFFFFu &&
           c->r1 < c->p && c->r2 < c->p;
}

inline int sm_count() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return n;
}

inline mont_status_t launch_status() {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? MONT_OK : MONT_ECUDA;
}

inline bool same_mod16(uintptr_t a, uintptr_t b) { return ((a ^ b) & 15u) == 0; }

// elements to peel so that p + head is 16-byte aligned (p is 4-byte aligned)
inline uint32_t head_elems(uintptr_t p, size_t n) {
    uint32_t h = (uint32_t)(((16u - (p & 15u)) & 15u) >> 2);
    return (size_t)h > n ? (uint32_t)n : h;
}

struct Launch {
    int threads, ctas_per_sm, unroll, variant, chunk, flags;
};

inline Launch resolve(const mont_launch_t *cfg, Launch def) {
    if (!cfg) return def;
    Launch l = def;
    if (cfg->threads > 0) l.threads = cfg->threads;
    if (cfg->ctas_per_sm > 0) l.ctas_per_sm = cfg->ctas_per_sm;
    if (cfg->unroll > 0) l.unroll = cfg->unroll;
    if (cfg->variant > 0) l.variant = cfg->variant;
    if (cfg->chunk > 0) l.chunk = cfg->chunk;
    l.flags = cfg->flags;
    return l;
}

inline bool launch_ok(const Launch &l) {
    return l.threads >= 32 && l.threads <= 1024 && (l.threads % 32) == 0 && l.ctas_per_sm >= 1 && l.chunk >= 0 &&
           (l.chunk % 4) == 0 &&
           l.ctas_per_sm <= 32 && (l.unroll == 1 || l.unroll == 2 || l.unroll == 4 || l.unroll == 8);
}

// <<<>>> or, with MONT_LAUNCH_OVERLAP_PREV, cudaLaunchKernelEx with programmatic stream
// serialisation: the launch may begin while the previous kernel on the stream is still running
// (the kernel brackets itself with pdl_trigger / pdl_wait, mont_core.cuh)
template <typename... KArgs, typename... Args>
inline mont_status_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int flags,
                              Args... args) {
    if (!(flags & MONT_LAUNCH_OVERLAP_PREV)) {
        kern<<<grid, block, smem, s>>>(args...);
        return launch_status();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...) == cudaSuccess ? launch_status() : MONT_ECUDA;
}

}  // namespace mont
