/*
 * c_api_demo.c -- the C ABI of libmont.so used from plain C (no Python, no torch):
 * context precompute, to_mont / mont_mul_vec / from_mont / mont_pow_vec on device buffers, one
 * host-buffer run through mont_host_run, each result checked against a naive 64-bit '%' loop.
 *
 *   gcc -std=c11 -O2 examples/c_api_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1609_00999_b200 -lmont -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1609_00999_b200 -o build/c_api_demo && ./build/c_api_demo
 *
 * Prints "c_api_demo ok" and exits 0, or names the first mismatch and exits 1.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "mont.h"
#include "mont_host.h"

#define N 100003u
#define CHECK(call)                                                                   \
    do {                                                                              \
        mont_status_t st_ = (call);                                                   \
        if (st_ != MONT_OK) {                                                         \
            fprintf(stderr, "%s failed: %s\n", #call, mont_strerror(st_));          \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

static uint32_t powmod(uint64_t b, uint32_t e, uint32_t p) {
    uint64_t r = 1 % p;
    b %= p;
    while (e) {
        if (e & 1u) r = r * b % p;
        b = b * b % p;
        e >>= 1;
    }
    return (uint32_t)r;
}

int main(void) {
    const uint32_t P = 2013265921u; /* 15 * 2^27 + 1 */
    mont_ctx_t ctx;
    CHECK(mont_ctx_init(&ctx, P));
    const uint64_t rinv = powmod(powmod(2, 32, P), P - 2, P); /* R^-1 by Fermat (P is prime) */

    uint32_t *a = malloc(N * 4), *b = malloc(N * 4), *c = malloc(N * 4), *e = malloc(N * 4);
    uint64_t s = 88172645463325252ull;
    for (uint32_t i = 0; i < N; ++i) { /* xorshift64 inputs, canonical */
        s ^= s << 13, s ^= s >> 7, s ^= s << 17;
        a[i] = (uint32_t)(s % P);
        b[i] = (uint32_t)((s >> 32) % P);
        e[i] = (uint32_t)(s >> 33);
    }
    a[0] = 0, b[1] = 0, a[2] = b[2] = P - 1;

    uint32_t *da, *db, *dc, *dt;
    if (cudaMalloc((void **)&da, N * 4) || cudaMalloc((void **)&db, N * 4) || cudaMalloc((void **)&dc, N * 4) ||
        cudaMalloc((void **)&dt, N * 4)) {
        fprintf(stderr, "cudaMalloc failed (no GPU?)\n");
        return 1;
    }
    cudaMemcpy(da, a, N * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b, N * 4, cudaMemcpyHostToDevice);

    /* c = a b R^-1 mod P */
    CHECK(mont_mul_vec(&ctx, dc, da, db, N, 0));
    cudaMemcpy(c, dc, N * 4, cudaMemcpyDeviceToHost);
    for (uint32_t i = 0; i < N; ++i)
        if (c[i] != (uint64_t)a[i] * b[i] % P * rinv % P) { fprintf(stderr, "mont_mul_vec %u\n", i); return 1; }

    /* from_mont(REDC(to_mont(a), to_mont(b))) = a b mod P */
    CHECK(to_mont(&ctx, dt, da, N, 0));
    CHECK(to_mont(&ctx, dc, db, N, 0));
    CHECK(mont_mul_vec(&ctx, dc, dt, dc, N, 0));
    CHECK(from_mont(&ctx, dc, dc, N, 0));
    cudaMemcpy(c, dc, N * 4, cudaMemcpyDeviceToHost);
    for (uint32_t i = 0; i < N; ++i)
        if (c[i] != (uint64_t)a[i] * b[i] % P) { fprintf(stderr, "domain round trip %u\n", i); return 1; }

    /* a^e mod P, 31-bit exponents */
    cudaMemcpy(dt, e, N * 4, cudaMemcpyHostToDevice);
    CHECK(mont_pow_vec(&ctx, dc, da, dt, N, 0));
    cudaMemcpy(c, dc, N * 4, cudaMemcpyDeviceToHost);
    for (uint32_t i = 0; i < N; i += 7)
        if (c[i] != powmod(a[i], e[i], P)) { fprintf(stderr, "mont_pow_vec %u\n", i); return 1; }

    /* the same product from host buffers through the pipelined executor (+ its checksum) */
    unsigned long long acc = 0;
    size_t ws_bytes = 64u << 20;
    void *ws;
    if (cudaMalloc(&ws, ws_bytes)) return 1;
    mont_host_job_t job = {MONT_HOST_MUL_VEC, &ctx, c, a, b, N, 0, &acc, -1, 0};
    CHECK(mont_host_run(&job, 1, ws, ws_bytes, 0));
    cudaDeviceSynchronize();
    unsigned long long ref = 0;
    for (uint32_t i = 0; i < N; ++i) {
        const uint32_t r = (uint32_t)((uint64_t)a[i] * b[i] % P * rinv % P);
        if (c[i] != r) { fprintf(stderr, "mont_host_run %u\n", i); return 1; }
        ref += r;
    }
    if (acc != ref) { fprintf(stderr, "mont_host_run checksum\n"); return 1; }

    cudaFree(ws), cudaFree(da), cudaFree(db), cudaFree(dc), cudaFree(dt);
    free(a), free(b), free(c), free(e);
    printf("c_api_demo ok\n");
    return 0;
}
