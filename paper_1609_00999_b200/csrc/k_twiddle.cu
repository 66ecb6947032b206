// k_twiddle.cu -- K2 mont_mul_twiddle: out[r][j] = REDC(x[r][j], tw[j])
// (BASELINE configs[2]: batch 4096 x len 2^14, the
// twiddle multiply of one NTT stage of the paper's modular FFTs).
//
// B200 design, table paths, all measured:
//  * variant 4 (the library default, variant 0, since round 2): a 2-D grid,
//    blockIdx.x = a column chunk of the table, blockIdx.y = a block of rows;
//    each CTA stages its chunk ONCE into shared memory with the bulk-copy
//    engine (cp.async.bulk, completion counted on an mbarrier by transaction
//    bytes -- the TMA path, SASS UBLKCP) and reads it with conflict-free
//    LDS.128 (alone it ties variant 2; inside bench.py's two-lane step it is
//    faster);
//  * variant 2 (power-of-two rows): the batch as one flat 128-bit stream,
//    table quads read through the read-only path where the 64 KiB table
//    stays L1-resident per SM; variant 1: the 2-D grid with the table via L1;
//  * variant 3: the whole table staged once per CTA lifetime plus cluster
//    launch control work stealing.
// HBM traffic is the 8 B/elem of x and out in every case.
#include <cuda_runtime.h>
#include <stdint.h>

#include "abi_util.h"
#include "tma.cuh"

namespace mont {

__device__ __forceinline__ uint4 redc4(const uint4 &x, const uint4 &t, uint32_t p, uint32_t pinv) {
    return make_uint4(redc(x.x, t.x, p, pinv), redc(x.y, t.y, p, pinv), redc(x.z, t.z, p, pinv),
                      redc(x.w, t.w, p, pinv));
}

// Vector path: len % 4 == 0, x/out/tw 16-byte aligned.  TMA = stage the table
// chunk in smem with cp.async.bulk; otherwise read it through L1 (__ldg).
template <int U, bool TMA>
__global__ void __launch_bounds__(512) k_twiddle(Ctx c, uint32_t *out, const uint32_t *x, const uint32_t *tw,
                                                  size_t batch, size_t len, uint32_t chunk, size_t rows_per_cta) {
    extern __shared__ __align__(128) uint4 s_tw[];
    __shared__ __align__(8) uint64_t bar;
    pdl_trigger();
    const size_t c0 = (size_t)blockIdx.x * chunk;
    const size_t r0 = (size_t)blockIdx.y * rows_per_cta;
    if (r0 >= batch || c0 >= len) return;  // uniform per CTA
    const size_t cwz = len - c0 < chunk ? len - c0 : chunk;
    const uint32_t cw4 = (uint32_t)(cwz >> 2);
    const size_t nrows = batch - r0 < rows_per_cta ? batch - r0 : rows_per_cta;
    const uint4 *t4 = reinterpret_cast<const uint4 *>(tw + c0);
    if (TMA) {
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            fence_mbar_init();
            const uint32_t bytes = cw4 * 16u;
            mbar_expect_tx(&bar, bytes);
            const uint32_t piece = 16384u;
            for (uint32_t off = 0; off < bytes; off += piece) {
                const uint32_t nb = bytes - off < piece ? bytes - off : piece;
                bulk_g2s(reinterpret_cast<char *>(s_tw) + off, reinterpret_cast<const char *>(t4) + off, nb, &bar);
            }
        }
        __syncthreads();  // barrier initialised before anyone polls it
    }
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
    uint4 *o4 = reinterpret_cast<uint4 *>(out);
    const size_t len4 = len >> 2;
    const size_t col0 = c0 >> 2;
    // running (row, col) position of this thread in the CTA's rows x cw4 tile
    const uint32_t step_r = blockDim.x / cw4, step_c = blockDim.x % cw4;
    size_t row = threadIdx.x / cw4;
    uint32_t col = threadIdx.x % cw4;
    bool waited = !TMA;
    while (row < nrows) {
        uint4 v[U];
        size_t idx[U];
        uint32_t cc[U];
        bool ok[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            ok[k] = row < nrows;
            idx[k] = (r0 + row) * len4 + col0 + col;
            cc[k] = col;
            if (ok[k]) v[k] = ld_stream(x4 + idx[k]);
            col += step_c;
            row += step_r;
            if (col >= cw4) {
                col -= cw4;
                ++row;
            }
        }
        if (!waited) {  // first trip: the table copy overlapped the first loads
            mbar_wait(&bar, 0);
            waited = true;
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            if (ok[k]) {
                const uint4 t = TMA ? s_tw[cc[k]] : __ldg(t4 + cc[k]);
                st_stream(o4 + idx[k], redc4(v[k], t, c.p, c.pinv));
            }
        }
    }
    if (!waited) mbar_wait(&bar, 0);  // never leave with a copy in flight
    pdl_wait();
}

// Flat variant (variant 2) for power-of-two len: the batch is one flat stream
// of uint4 chunks (like k_map1), chunk i uses table quad i mod (len/4), read
// through the read-only path (the whole table stays L1/L2-resident).
template <int U>
__global__ void __launch_bounds__(512) k_twiddle_flat(Ctx c, uint32_t *out, const uint32_t *x, const uint32_t *tw,
                                                       size_t n4, size_t qmask) {
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
    const uint4 *t4 = reinterpret_cast<const uint4 *>(tw);
    uint4 *o4 = reinterpret_cast<uint4 *>(out);
    const size_t tile = (size_t)U * blockDim.x;
    const size_t base = (size_t)blockIdx.x * tile + threadIdx.x;
    uint4 v[U], t[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
        const size_t i = base + (size_t)k * blockDim.x;
        if (i < n4) {
            v[k] = ld_stream(x4 + i);
            t[k] = __ldg(t4 + (i & qmask));
        }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
        const size_t i = base + (size_t)k * blockDim.x;
        if (i < n4) st_stream(o4 + i, redc4(v[k], t[k], c.p, c.pinv));
    }
}

// Variant 3: the whole table staged ONCE per CTA lifetime by the bulk-copy
// engine, rows processed in blocks of `rows_per_item`, and the CTA keeps
// taking row blocks from not-yet-launched CTAs by cluster launch control
// (hardware work stealing) -- TMA staging without paying the table per block,
// with the dynamic balance of a flat grid.  len % 4 == 0, 4 len <= 227 KB.
__global__ void __launch_bounds__(512) k_twiddle_clc(Ctx c, uint32_t *out, const uint32_t *x, const uint32_t *tw,
                                                      size_t batch, size_t len, uint32_t rows_per_item) {
    extern __shared__ __align__(128) uint4 s_tw[];
    __shared__ __align__(8) uint64_t bar_tw;
    __shared__ __align__(8) uint64_t bar_clc;
    __shared__ __align__(16) uint4 clc_resp;
    const uint32_t len4 = (uint32_t)(len >> 2);
    if (threadIdx.x == 0) {
        mbar_init(&bar_tw, 1);
        mbar_init(&bar_clc, 1);
        fence_mbar_init();
        const uint32_t bytes = len4 * 16u;
        mbar_expect_tx(&bar_tw, bytes);
        for (uint32_t off = 0; off < bytes; off += 16384u)
            bulk_g2s(reinterpret_cast<char *>(s_tw) + off, reinterpret_cast<const char *>(tw) + off,
                     bytes - off < 16384u ? bytes - off : 16384u, &bar_tw);
    }
    __syncthreads();
    mbar_wait(&bar_tw, 0);
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
    uint4 *o4 = reinterpret_cast<uint4 *>(out);
    uint32_t item = blockIdx.x, phase = 0;
    while (true) {
        if (threadIdx.x == 0) {  // ask for the next item while this one streams
            fence_mbar_init();
            mbar_expect_tx(&bar_clc, 16u);
            clc_try_cancel(&clc_resp, &bar_clc);
        }
        const size_t r0 = (size_t)item * rows_per_item;
        const size_t nrows = batch - r0 < rows_per_item ? batch - r0 : rows_per_item;
        for (size_t r = 0; r < nrows; ++r) {
            const uint4 *xr = x4 + (r0 + r) * len4;
            uint4 *orow = o4 + (r0 + r) * len4;
            for (uint32_t c0 = threadIdx.x; c0 < len4; c0 += 4 * blockDim.x) {
                uint4 v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t cc = c0 + k * blockDim.x;
                    if (cc < len4) v[k] = ld_stream(xr + cc);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t cc = c0 + k * blockDim.x;
                    if (cc < len4) st_stream(orow + cc, redc4(v[k], s_tw[cc], c.p, c.pinv));
                }
            }
        }
        mbar_wait(&bar_clc, phase);
        phase ^= 1u;
        uint32_t next;
        const bool more = clc_query(clc_resp, next);
        __syncthreads();  // everyone has read clc_resp before it is overwritten
        if (!more) break;
        item = next;
    }
}

// Scalar fallback (len % 4 != 0 or misaligned operands)
__global__ void __launch_bounds__(256) k_twiddle_scalar(Ctx c, uint32_t *out, const uint32_t *x, const uint32_t *tw,
                                                         size_t batch, size_t len) {
    for (size_t r = blockIdx.y; r < batch; r += gridDim.y) {
        const uint32_t *xr = x + r * len;
        uint32_t *orow = out + r * len;
        for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < len; j += (size_t)gridDim.x * blockDim.x)
            st_stream1(orow + j, redc(ld_stream1(xr + j), __ldg(tw + j), c.p, c.pinv));
    }
}

// B200 sweeps: the bulk-copy (TMA) staged table (variant 4: 64 CTAs per SM of
// 256 threads, a few rows and a 2048-column chunk each) runs configs[2] in 84.35 us, the flat
// stream with the table through L1 (variant 2, 512 threads x 4 uint4) in 84.26 us
// (profiles/r02_probe_twiddle_paths.jsonl); inside bench.py's two-lane step the staged path is
// the faster one (0.5956 vs 0.5997 ms per step, profiles/r02_step_sweep.jsonl), so variant 0
// (the library default) is variant 4 for every row length.
static const Launch kTwDefault{512, 64, 4, 0, 2048};

template <int U, bool TMA>
static mont_status_t launch_tw(const Ctx &c, uint32_t *out, const uint32_t *x, const uint32_t *tw, size_t batch,
                               size_t len, const Launch &L, int sms, cudaStream_t s) {
    size_t chunk = (size_t)L.chunk;
    if (chunk > len) chunk = len;
    chunk = (chunk + 3) & ~(size_t)3;
    const size_t nchunks = (len + chunk - 1) / chunk;
    const size_t smem = TMA ? chunk * 4 : 0;
    if (smem > 227 * 1024) return MONT_EINVAL_ARG;
    if (nchunks > 0x7fffffff) return MONT_EUNSUPPORTED;
    const size_t target = (size_t)sms * L.ctas_per_sm;
    size_t gy = (target + nchunks - 1) / nchunks;
    if (gy > batch) gy = batch;
    if (gy > 65535) gy = 65535;
    const size_t rows_per_cta = (batch + gy - 1) / gy;
    gy = (batch + rows_per_cta - 1) / rows_per_cta;
    if (TMA && smem > 48 * 1024) {
        if (cudaFuncSetAttribute(k_twiddle<U, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return MONT_ECUDA;
    }
    dim3 grid((unsigned)nchunks, (unsigned)gy);
    return launch_k(k_twiddle<U, TMA>, grid, dim3((unsigned)L.threads), smem, s, L.flags, c, out, x, tw, batch, len,
                    (uint32_t)chunk, rows_per_cta);
}

}  // namespace mont

using namespace mont;

extern "C" mont_status_t mont_mul_twiddle_ex(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *x,
                                             const uint32_t *tw, size_t batch, size_t len,
                                             const mont_launch_t *cfg, cudaStream_t stream) {
    if (!ctx_ok(ctx)) return ctx ? MONT_EINVAL_P : MONT_EINVAL_ARG;
    if (batch == 0) return MONT_OK;
    if (len == 0) return MONT_EINVAL_ARG;
    if (!out || !x || !tw || ((uintptr_t)out | (uintptr_t)x | (uintptr_t)tw) & 3u) return MONT_EINVAL_ARG;
    if (batch > ((size_t)-1) / len) return MONT_EINVAL_ARG;
    Launch L = resolve(cfg, kTwDefault);
    if (L.threads < 32 || L.threads > 512 || (L.threads & 31) || L.ctas_per_sm < 1 || L.chunk < 4 ||
        (L.chunk & 3) || !(L.unroll == 1 || L.unroll == 2 || L.unroll == 4 || L.unroll == 8) || L.variant < 0 ||
        L.variant > 4)
        return MONT_EINVAL_ARG;
    const int sms = sm_count();
    if (sms <= 0) return MONT_ECUDA;
    const Ctx c = to_dev(ctx);
    const bool vec = (len % 4 == 0) && (((uintptr_t)out | (uintptr_t)x | (uintptr_t)tw) & 15u) == 0;
    if (!vec) {
        size_t gx = (len + 255) / 256;
        if (gx > (size_t)sms * 8) gx = (size_t)sms * 8;
        size_t gy = ((size_t)sms * 8 + gx - 1) / gx;
        if (gy > batch) gy = batch;
        if (gy > 65535) gy = 65535;
        k_twiddle_scalar<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, stream>>>(c, out, x, tw, batch, len);
        return launch_status();
    }
    const bool pow2 = (len & (len - 1)) == 0;
    int v = L.variant;
    if (v == 0) v = 4;  // library default: the TMA-staged table (ties the L1 path alone, wins in the step)
    if (v == 3 && len * 4 <= 200 * 1024) {  // staged once per CTA + CLC work stealing
        const uint32_t rows_per_item = 2u;
        const size_t items = (batch + rows_per_item - 1) / rows_per_item;
        const size_t smem = len * 4;
        if (items > 0x7fffffff) return MONT_EUNSUPPORTED;
        if (smem > 48 * 1024 &&
            cudaFuncSetAttribute(k_twiddle_clc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return MONT_ECUDA;
        k_twiddle_clc<<<(unsigned)items, 512, smem, stream>>>(c, out, x, tw, batch, len, rows_per_item);
        return launch_status();
    }
    if (v == 3) v = 4;
    if (v == 2 && pow2) {  // flat stream, power-of-two rows
        const size_t n4 = batch * len / 4;
        const size_t tile = (size_t)L.unroll * L.threads;
        const size_t grid = (n4 + tile - 1) / tile;
        if (grid > 0x7fffffff) return MONT_EUNSUPPORTED;
        switch (L.unroll) {
            case 1: k_twiddle_flat<1><<<(unsigned)grid, L.threads, 0, stream>>>(c, out, x, tw, n4, len / 4 - 1); break;
            case 2: k_twiddle_flat<2><<<(unsigned)grid, L.threads, 0, stream>>>(c, out, x, tw, n4, len / 4 - 1); break;
            case 4: k_twiddle_flat<4><<<(unsigned)grid, L.threads, 0, stream>>>(c, out, x, tw, n4, len / 4 - 1); break;
            default: k_twiddle_flat<8><<<(unsigned)grid, L.threads, 0, stream>>>(c, out, x, tw, n4, len / 4 - 1); break;
        }
        return launch_status();
    }
    if (v == 2) v = 4;  // not a power of two: the staged-table kernel
    if (v == 4) {       // table chunk staged per CTA by cp.async.bulk (TMA engine) + mbarrier
        if (!cfg || cfg->threads == 0) L.threads = 256;  // its own best shape
        switch (L.unroll) {
            case 1: return launch_tw<1, true>(c, out, x, tw, batch, len, L, sms, stream);
            case 2: return launch_tw<2, true>(c, out, x, tw, batch, len, L, sms, stream);
            case 4: return launch_tw<4, true>(c, out, x, tw, batch, len, L, sms, stream);
            default: return launch_tw<8, true>(c, out, x, tw, batch, len, L, sms, stream);
        }
    }
    // v == 1: table read through L1/L2, no shared memory
    switch (L.unroll) {
        case 1: return launch_tw<1, false>(c, out, x, tw, batch, len, L, sms, stream);
        case 2: return launch_tw<2, false>(c, out, x, tw, batch, len, L, sms, stream);
        case 4: return launch_tw<4, false>(c, out, x, tw, batch, len, L, sms, stream);
        default: return launch_tw<8, false>(c, out, x, tw, batch, len, L, sms, stream);
    }
}

extern "C" mont_status_t mont_mul_twiddle(const mont_ctx_t *ctx, uint32_t *out, const uint32_t *x,
                                          const uint32_t *tw, size_t batch, size_t len, cudaStream_t stream) {
    return mont_mul_twiddle_ex(ctx, out, x, tw, batch, len, nullptr, stream);
}
