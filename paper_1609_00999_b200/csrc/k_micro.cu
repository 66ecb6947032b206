// k_micro.cu -- K8 integer-multiply pipe microbenchmark (roofline denominator
// for the compute-bound pow kernel).  Each thread
// runs 8 independent dependency chains, 8 ops per chain per loop trip, of one
// instruction kind, so the FMAHeavy pipe (which executes IMAD / IMUL,
// Nsight Compute Profiling Guide "Pipelines") is the only limiter.
#include <cuda_runtime.h>
#include <stdint.h>

#include "abi_util.h"

namespace mont {

template <int KIND>
__device__ __forceinline__ void op(uint32_t &x, uint64_t &w, uint32_t c, int32_t p, int32_t pinv, double &d) {
    if (KIND == 0) {
        asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(x) : "r"(c));
    } else if (KIND == 1) {
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x) : "r"(c));
    } else if (KIND == 2) {
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w) : "r"(x), "r"(c));
    } else if (KIND == 3) {
        x = (uint32_t)sredc((int32_t)x, (int32_t)x, p, pinv);           // library chain form
    } else if (KIND == 4) {
        x = redc(x, x, (uint32_t)p, (uint32_t)pinv);                    // library canonical form
    } else if (KIND == 5) {
        x = (uint32_t)sredc_mulhi((int32_t)x, (int32_t)x, p, pinv);     // mul.hi reference
    } else if (KIND == 6) {
        x = (uint32_t)sredc_hiadd((int32_t)x, (int32_t)x, -p, pinv);    // IMAD.HI 64-bit addend
    } else if (KIND == 7) {
        asm volatile("fma.rn.f64 %0, %0, %0, %0;" : "+d"(d));           // DFMA
    } else if (KIND == 8) {
        d = fmulmod(d, d, (double)p, 1.0 / (double)p);                   // FP64 Barrett product
    } else if (KIND == 9) {
        asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(c));           // IADD (ALU)
    } else if (KIND == 10) {
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(c), "r"((uint32_t)p));  // LOP3 (ALU)
    } else if (KIND == 13) {
        asm volatile("min.u32 %0, %0, %1;" : "+r"(x) : "r"(c));             // VIMNMX (ALU)
    } else if (KIND == 15) {
        x = fredc_p1(x, x, (uint32_t)p);                                   // Alg. 3, c = 7 as shifts
    } else if (KIND == 14) {
        asm volatile("shf.l.wrap.b32 %0, %0, %0, %1;" : "+r"(x) : "r"(c));  // SHF (ALU)
    }
}

template <int KIND>
__global__ void __launch_bounds__(256) k_imad(uint32_t *sink, int iters, uint32_t c, int32_t p, int32_t pinv) {
    uint32_t x[8];
    uint64_t w[8];
    double d[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        x[k] = (threadIdx.x * 2654435761u + k * 40503u) % (uint32_t)p;
        w[k] = x[k];
        d[k] = (double)x[k] * (KIND == 7 ? 1e-300 : 1.0);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (KIND == 11) {  // 3 integer Montgomery chains : 1 FP64 Barrett chain
                    if (k % 4 == 3) op<8>(x[k], w[k], c, p, pinv, d[k]);
                    else op<3>(x[k], w[k], c, p, pinv, d[k]);
                } else if (KIND == 16) {  // 7 Montgomery chains : 1 shift-Fourier chain (canonical)
                    if (k == 7) op<15>(x[k], w[k], c, p, pinv, d[k]);
                    else op<3>(x[k], w[k], c, p, pinv, d[k]);
                } else if (KIND == 17) {  // 3 : 1
                    if (k % 4 == 3) op<15>(x[k], w[k], c, p, pinv, d[k]);
                    else op<3>(x[k], w[k], c, p, pinv, d[k]);
                } else if (KIND == 12) {  // 1 : 1
                    if (k % 2 == 1) op<8>(x[k], w[k], c, p, pinv, d[k]);
                    else op<3>(x[k], w[k], c, p, pinv, d[k]);
                } else {
                    op<KIND>(x[k], w[k], c, p, pinv, d[k]);
                }
            }
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= x[k] ^ (uint32_t)w[k] ^ (uint32_t)(w[k] >> 32) ^ (uint32_t)(long long)d[k];
    sink[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace mont

using namespace mont;

extern "C" mont_status_t mb_imad(uint32_t *sink, int kind, int iters, const mont_launch_t *cfg, cudaStream_t stream,
                                 unsigned long long *threads_launched) {
    if (!sink || kind < 0 || kind > 17 || iters < 1) return MONT_EINVAL_ARG;
    const int sms = sm_count();
    if (sms <= 0) return MONT_ECUDA;
    const int ctas = (cfg && cfg->ctas_per_sm > 0) ? cfg->ctas_per_sm : 8;
    const unsigned grid = (unsigned)(sms * ctas);
    const uint32_t p = 469762049u;  // a config prime (BASELINE configs[3])
    uint32_t pinv = p;
    for (int i = 0; i < 4; ++i) pinv *= 2u - p * pinv;  // 2-adic inverse by Newton
    const uint32_t c = 0x9E3779B9u;
    switch (kind) {
        case 0: k_imad<0><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 1: k_imad<1><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 2: k_imad<2><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 3: k_imad<3><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 4: k_imad<4><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 5: k_imad<5><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 6: k_imad<6><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 7: k_imad<7><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 8: k_imad<8><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 9: k_imad<9><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 10: k_imad<10><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 11: k_imad<11><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 12: k_imad<12><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 13: k_imad<13><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 14: k_imad<14><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 15: k_imad<15><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        case 16: k_imad<16><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
        default: k_imad<17><<<grid, 256, 0, stream>>>(sink, iters, c, (int32_t)p, (int32_t)pinv); break;
    }
    if (threads_launched) *threads_launched = (unsigned long long)grid * 256ull;
    return launch_status();
}
