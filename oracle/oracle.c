/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the batched 32-bit
 * Montgomery multiplication path of arxiv 1609.00999.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or constant generator with the CUDA library
 * under paper_1609_00999_b200/csrc/, and the product never calls it.
 *
 * What it computes: the DEFINITIONS the Montgomery method reaches exactly
 * (§3.1), written out with 64-bit naive '%' (the "naive
 * implementation" with "expensive integer division", §1):
 *
 *   Montgomery product  REDC(a,b) = a*b*R^-1 mod P,  R = 2^32
 *   residue class       to_mont(x) = x*R mod P
 *   inverse map         from_mont(x) = x*R^-1 mod P
 *   twiddle product     out[r][j] = x[r][j]*tw[j]*R^-1 mod P     (BASELINE configs[2])
 *   modular power       base^exp mod P, left-to-right square-and-multiply on
 *                       plain values over the 32 exponent bits   (BASELINE configs[3])
 *   checksum            (sum_i c[i]) mod P                       (BASELINE configs[4])
 *
 * R^-1 and P' come from the extended Euclidean algorithm, as PAPER.md:89 says
 * ("R R^-1 - P P' = 1, which can be computed using the extended Euclidean
 * algorithm").
 *
 * Self-test-only functions follow the paper's algorithms step by step with a
 * general R = 2^l (l <= 32) so the SPEC.md worked examples (which use small l)
 * can be replayed: Alg. 1 Barrett, Alg. 2 REDC
 * (PAPER.md:95-99), Alg. 3 Fourier-prime REDC (read with a
 * 64-bit signed t: DESIGN.md reading G8).
 *
 * Parity pins: every function here is pinned in tests/test_oracle.py against
 * something other than itself (brute force over all pairs for all odd primes
 * <= 257 via the Montgomery identity c*2^32 = a*b (mod P), the special case
 * P | 2^32-1, Python's built-in pow, Fermat, round trips, closed forms, the
 * SPEC.md worked examples).  No function is "parity unpinned".
 */
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#include <pthread.h>
#include <unistd.h>

/* --------------------------------------------------------------- context */

typedef struct {
    uint32_t P;       /* odd modulus, 3 <= P < 2^31                          */
    uint32_t l;       /* R = 2^l                                             */
    uint64_t R;       /* 2^l                                                 */
    uint32_t Rinv;    /* 0 < Rinv < P,  R*Rinv = 1 (mod P)    */
    uint32_t Pprime;  /* 0 < P' < R,    R*Rinv - P*P' = 1    */
    uint32_t r1;      /* R mod P   (the residue of 1)                        */
    uint32_t r2;      /* R^2 mod P                                           */
    uint32_t bk;      /* Barrett k = ceil(log2 P)  */
    uint64_t bPprime; /* Barrett P' = floor(2^(2k) / P)  */
} oracle_ctx_t;

/* Extended Euclid: returns x with (a*x) mod m == 1 for gcd(a,m) = 1, 0 <= x < m. */
static int64_t ext_euclid_inverse(int64_t a, int64_t m)
{
    int64_t old_r = a, r = m, old_s = 1, s = 0;
    while (r != 0) {
        int64_t q = old_r / r, t;
        t = old_r - q * r; old_r = r; r = t;
        t = old_s - q * s; old_s = s; s = t;
    }
    if (old_r != 1) return -1;               /* not invertible */
    old_s %= m;
    if (old_s < 0) old_s += m;
    return old_s;
}

/* Returns 0 on success, 1 for an invalid modulus (even, < 3, >= 2^31, or R <= P). */
int oracle_ctx_l(oracle_ctx_t *c, uint32_t P, uint32_t l)
{
    if ((P & 1u) == 0 || P < 3u || P >= 0x80000000u || l < 1 || l > 32) return 1;
    uint64_t R = (uint64_t)1 << l;
    if (R <= P) return 1;
    c->P = P;
    c->l = l;
    c->R = R;
    c->r1 = (uint32_t)(R % P);
    int64_t rinv = ext_euclid_inverse((int64_t)c->r1, (int64_t)P);
    if (rinv <= 0) return 1;
    c->Rinv = (uint32_t)rinv;
    uint64_t num = R * (uint64_t)c->Rinv - 1u;   /* < 2^32 * 2^31: fits */
    if (num % P != 0) return 1;                  /* Bezout identity must be exact */
    c->Pprime = (uint32_t)(num / P);
    c->r2 = (uint32_t)(((uint64_t)c->r1 * c->r1) % P);
    uint32_t k = 0;
    while (((uint64_t)1 << k) < P) k++;          /* ceil(log2 P) */
    c->bk = k;
    /* 2^(2k) / P with 2k <= 62: fits in 64 bits */
    c->bPprime = ((uint64_t)1 << (2 * k)) / P;
    return 0;
}

int oracle_ctx(oracle_ctx_t *c, uint32_t P) { return oracle_ctx_l(c, P, 32); }

/* ----------------------------------------------------------- scalar defs */

/* naive modular product, the oracle primitive */
static inline uint32_t mulmod_naive(uint32_t a, uint32_t b, uint32_t P)
{
    return (uint32_t)(((uint64_t)a * b) % P);
}

uint32_t oracle_mulmod(uint32_t a, uint32_t b, uint32_t P) { return mulmod_naive(a, b, P); }

/* a*b*R^-1 mod P, by definition */
uint32_t oracle_mont_mul1(const oracle_ctx_t *c, uint32_t a, uint32_t b)
{
    return mulmod_naive(mulmod_naive(a, b, c->P), c->Rinv, c->P);
}

/* x*R mod P */
uint32_t oracle_to_mont1(const oracle_ctx_t *c, uint32_t x)
{
    return (uint32_t)((((uint64_t)x % c->P) << c->l) % c->P);
}

/* x*R^-1 mod P */
uint32_t oracle_from_mont1(const oracle_ctx_t *c, uint32_t x)
{
    return mulmod_naive(x % c->P, c->Rinv, c->P);
}

/* base^exp mod P on plain values: left-to-right square-and-multiply over all
 * 32 exponent bits 31..0, naive '%' (BASELINE configs[3] draws 31-bit
 * exponents; the product's contract, include/mont.h, takes any uint32
 * exponent; reading G10: 0^0 = 1). */
uint32_t oracle_pow1(uint32_t P, uint32_t base, uint32_t exp)
{
    uint32_t acc = 1u % P;
    uint32_t x = base % P;
    for (int bit = 31; bit >= 0; --bit) {
        acc = mulmod_naive(acc, acc, P);
        if ((exp >> bit) & 1u) acc = mulmod_naive(acc, x, P);
    }
    return acc;
}

/* -------------------------------------------- array forms (std threads) */

typedef struct {
    int op;
    const oracle_ctx_t *c;
    uint32_t *out;
    const uint32_t *a, *b;
    size_t lo, hi;       /* element range */
    size_t len;          /* twiddle row length */
    uint64_t sum;
} job_t;

enum { OP_MUL = 0, OP_TO = 1, OP_FROM = 2, OP_TW = 3, OP_POW = 4, OP_SUM = 5, OP_MULMOD = 6 };

static void *run_job(void *arg)
{
    job_t *j = (job_t *)arg;
    const oracle_ctx_t *c = j->c;
    size_t i;
    switch (j->op) {
    case OP_MUL:
        for (i = j->lo; i < j->hi; ++i) j->out[i] = oracle_mont_mul1(c, j->a[i], j->b[i]);
        break;
    case OP_TO:
        for (i = j->lo; i < j->hi; ++i) j->out[i] = oracle_to_mont1(c, j->a[i]);
        break;
    case OP_FROM:
        for (i = j->lo; i < j->hi; ++i) j->out[i] = oracle_from_mont1(c, j->a[i]);
        break;
    case OP_TW:    /* a = x (row-major batch x len), b = tw[len] */
        for (i = j->lo; i < j->hi; ++i) j->out[i] = oracle_mont_mul1(c, j->a[i], j->b[i % j->len]);
        break;
    case OP_POW:
        for (i = j->lo; i < j->hi; ++i) j->out[i] = oracle_pow1(c->P, j->a[i], j->b[i]);
        break;
    case OP_MULMOD:   /* plain a*b mod P by definition (the result Barrett, Alg. 1, reaches) */
        for (i = j->lo; i < j->hi; ++i) j->out[i] = mulmod_naive(j->a[i] % c->P, j->b[i] % c->P, c->P);
        break;
    case OP_SUM: {
        uint64_t s = 0;
        for (i = j->lo; i < j->hi; ++i) s += j->a[i];
        j->sum = s;
        break;
    }
    }
    return NULL;
}

static int n_workers(int nthreads)
{
    if (nthreads > 0) return nthreads;
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

/* Splits [0,n) into contiguous slices, one per worker thread. Returns the sum
 * of job sums (used by OP_SUM). */
static uint64_t run_parallel(int op, const oracle_ctx_t *c, uint32_t *out, const uint32_t *a,
                             const uint32_t *b, size_t n, size_t len, int nthreads)
{
    int w = n_workers(nthreads);
    if ((size_t)w > n) w = n ? (int)n : 1;
    job_t *jobs = (job_t *)calloc((size_t)w, sizeof(job_t));
    pthread_t *th = (pthread_t *)calloc((size_t)w, sizeof(pthread_t));
    for (int t = 0; t < w; ++t) {
        jobs[t].op = op; jobs[t].c = c; jobs[t].out = out; jobs[t].a = a; jobs[t].b = b;
        jobs[t].len = len;
        jobs[t].lo = n * (size_t)t / (size_t)w;
        jobs[t].hi = n * (size_t)(t + 1) / (size_t)w;
    }
    for (int t = 1; t < w; ++t) pthread_create(&th[t], NULL, run_job, &jobs[t]);
    run_job(&jobs[0]);
    uint64_t s = jobs[0].sum;
    for (int t = 1; t < w; ++t) { pthread_join(th[t], NULL); s += jobs[t].sum; }
    free(jobs);
    free(th);
    return s;
}

void oracle_mont_mul(const oracle_ctx_t *c, uint32_t *out, const uint32_t *a, const uint32_t *b,
                     size_t n, int nthreads)
{ run_parallel(OP_MUL, c, out, a, b, n, 1, nthreads); }

void oracle_mulmod_vec(const oracle_ctx_t *c, uint32_t *out, const uint32_t *a, const uint32_t *b, size_t n,
                       int nthreads)
{ run_parallel(OP_MULMOD, c, out, a, b, n, 1, nthreads); }

void oracle_to_mont(const oracle_ctx_t *c, uint32_t *out, const uint32_t *x, size_t n, int nthreads)
{ run_parallel(OP_TO, c, out, x, NULL, n, 1, nthreads); }

void oracle_from_mont(const oracle_ctx_t *c, uint32_t *out, const uint32_t *x, size_t n, int nthreads)
{ run_parallel(OP_FROM, c, out, x, NULL, n, 1, nthreads); }

void oracle_twiddle(const oracle_ctx_t *c, uint32_t *out, const uint32_t *x, const uint32_t *tw,
                    size_t batch, size_t len, int nthreads)
{ if (len) run_parallel(OP_TW, c, out, x, tw, batch * len, len, nthreads); }

void oracle_pow(const oracle_ctx_t *c, uint32_t *out, const uint32_t *base, const uint32_t *exp,
                size_t n, int nthreads)
{ run_parallel(OP_POW, c, out, base, exp, n, 1, nthreads); }

/* plain sum of x (uint64; n*(P-1) < 2^63 for n <= 2^32); caller reduces mod P */
uint64_t oracle_sum(const uint32_t *x, size_t n, int nthreads)
{ return run_parallel(OP_SUM, NULL, NULL, x, NULL, n, 1, nthreads); }

/* (sum_i x[i]) mod P  (BASELINE configs[4]) */
uint32_t oracle_checksum(const oracle_ctx_t *c, const uint32_t *x, size_t n, int nthreads)
{ return (uint32_t)(oracle_sum(x, n, nthreads) % c->P); }

/* ------------------------------------------------------------- twiddles */

/* w = g^((P-1)/order) mod P by the plain ladder (BASELINE configs[2]; G11) */
uint32_t oracle_root_of_unity(uint32_t P, uint32_t g, uint32_t order)
{
    uint32_t e = (P - 1u) / order;
    /* plain repeated squaring on the full 32-bit exponent */
    uint32_t acc = 1u % P, x = g % P;
    for (int bit = 31; bit >= 0; --bit) {
        acc = mulmod_naive(acc, acc, P);
        if ((e >> bit) & 1u) acc = mulmod_naive(acc, x, P);
    }
    return acc;
}

/* tw[j] = to_mont(w^j mod P), w^j by repeated naive multiplication (BASELINE configs[2]) */
void oracle_twiddle_table(const oracle_ctx_t *c, uint32_t *tw, uint32_t w, size_t len)
{
    uint32_t wj = 1u % c->P;
    for (size_t j = 0; j < len; ++j) {
        tw[j] = oracle_to_mont1(c, wj);
        wj = mulmod_naive(wj, w, c->P);
    }
}

/* ---------------------------------------- paper algorithms, self-test only */

/* Alg. 2 REDC with R = 2^l, step by step.  Precondition
 * 0 <= T < R*P.  Reports through *flags: bit0 = the low l bits of
 * T + mP were nonzero (exact-division violated), bit1 = t >= 2P before the
 * subtract (violates "0 <= t < 2P"), bit2 = the subtract branch was taken. */
uint32_t oracle_redc_l(const oracle_ctx_t *c, uint64_t T, uint32_t *flags)
{
    uint64_t Rm1 = c->R - 1u;
    uint64_t m = ((T & Rm1) * (uint64_t)c->Pprime) & Rm1;      /* m <- (T mod R) P' mod R */
    /* T + mP < RP + RP < 2^64 */
    uint64_t s = T + m * (uint64_t)c->P;
    uint32_t f = 0;
    if (s & Rm1) f |= 1u;
    uint64_t t = s >> c->l;                                      /* t <- (T + mP)/R */
    if (t >= 2u * (uint64_t)c->P) f |= 2u;
    if (t >= c->P) { t -= c->P; f |= 4u; }                       /* if t >= P: t - P */
    if (flags) *flags = f;
    return (uint32_t)t;
}

/* Alg. 1 Barrett: returns ab mod P, *loops = while-loop trips. */
uint32_t oracle_barrett(const oracle_ctx_t *c, uint32_t a, uint32_t b, uint32_t *loops)
{
    uint64_t ab = (uint64_t)a * b;
    uint64_t m = ab >> c->bk;                                    /* floor(ab / 2^k) */
    /* m < 2^k (ab < P^2 < 2^(2k)) and P' <= 2^k (ceil log2 P = k): m P' < 2^(2k) <= 2^62 */
    uint64_t q = (m * c->bPprime) >> c->bk;                      /* floor(m P' / 2^k) */
    uint64_t t = ab - q * (uint64_t)c->P;
    uint32_t n = 0;
    while (t >= c->P) { t -= c->P; ++n; }
    if (loops) *loops = n;
    return (uint32_t)t;
}

/* Alg. 3 Fourier-prime REDC for P = c 2^n + 1, R = 2^l,
 * n >= l/2.  t is held in 64-bit signed arithmetic (reading G8: the
 * paper's 32-bit (t >> 31) mask overflows for P > 2^30).  The three
 * normalisation steps follow the paper with the sign mask taken at 64 bits.
 * *t_raw receives q1 - q2 + q3 before normalisation and *r3 the quantity the
 * paper proves zero. */
uint32_t oracle_fourier_redc(const oracle_ctx_t *c, uint32_t cc, uint32_t n, uint32_t a, uint32_t b,
                             int64_t *t_raw, uint64_t *r3_out)
{
    uint64_t R = c->R, Rm1 = R - 1u;
    uint64_t ab = (uint64_t)a * b;
    uint64_t q1 = ab >> c->l;                                    /* ab / R      */
    uint64_t r1 = ab & Rm1;                                      /* ab mod R    */
    /* c 2^n r1 < P R < 2^63: exact in 64 bits */
    uint64_t k = (uint64_t)cc << n;                              /* c 2^n       */
    uint64_t q2 = (k * r1) >> c->l;
    uint64_t r2 = (k * r1) & Rm1;
    uint64_t q3 = (k * r2) >> c->l;
    uint64_t r3 = (k * r2) & Rm1;
    int64_t t = (int64_t)q1 - (int64_t)q2 + (int64_t)q3;
    if (t_raw) *t_raw = t;
    if (r3_out) *r3_out = r3;
    int64_t P = (int64_t)c->P;
    t = t + ((t >> 63) & P);                                     /* t + (t>>31)&P, 64-bit */
    t = t - P;
    t = t + ((t >> 63) & P);
    return (uint32_t)t;
}

/* (a + b) mod P, (a - b) mod P by definition ("straightforward") */
uint32_t oracle_mod_add(uint32_t a, uint32_t b, uint32_t P) { return (uint32_t)(((uint64_t)a + b) % P); }
uint32_t oracle_mod_sub(uint32_t a, uint32_t b, uint32_t P)
{ return (uint32_t)(((uint64_t)a + P - (b % P)) % P); }

/* ------------------------------------------------ NTT
 *
 * The number-theoretic transform the paper's generated modular FFT libraries
 * compute, by DEFINITION: for a primitive N-th root of
 * unity w mod P,
 *     X[k] = sum_{j<N} x[j] * w^(j k)  mod P,    k < N            (O(N^2))
 * and the cyclic convolution c[k] = sum_j a[j] b[(k - j) mod N] mod P, also by
 * definition.  Powers w^e are taken from a table of w^0..w^(N-1) built by
 * repeated naive multiplication; exponents are reduced mod N (w^N = 1). */
void oracle_dft(uint32_t P, uint32_t w, const uint32_t *x, uint32_t *X, size_t N)
{
    uint32_t *pw = (uint32_t *)malloc(N * sizeof(uint32_t));
    uint32_t acc = 1u % P;
    for (size_t e = 0; e < N; ++e) { pw[e] = acc; acc = mulmod_naive(acc, w, P); }
    for (size_t k = 0; k < N; ++k) {
        uint64_t s = 0;
        for (size_t j = 0; j < N; ++j) {
            s += mulmod_naive(x[j] % P, pw[(j * k) % N], P);
            s %= P;
        }
        X[k] = (uint32_t)s;
    }
    free(pw);
}

void oracle_cyclic_conv(uint32_t P, const uint32_t *a, const uint32_t *b, uint32_t *c, size_t N)
{
    for (size_t k = 0; k < N; ++k) {
        uint64_t s = 0;
        for (size_t j = 0; j < N; ++j) {
            s += mulmod_naive(a[j] % P, b[(k + N - j) % N] % P, P);
            s %= P;
        }
        c[k] = (uint32_t)s;
    }
}

/* modular inverse by extended Euclid (P:89's tool), 0 if not invertible */
uint32_t oracle_inverse(uint32_t x, uint32_t P)
{
    int64_t r = ext_euclid_inverse((int64_t)(x % P), (int64_t)P);
    return r < 0 ? 0u : (uint32_t)r;
}

/* Batched modular dot product by definition:
 * out[r] = sum_j A[r][j] x[j] R^-1 mod P  =  (sum_j (A x mod P)) R^-1 mod P. */
void oracle_dot(const oracle_ctx_t *c, uint32_t *out, const uint32_t *A, const uint32_t *x, size_t batch, size_t len)
{
    for (size_t r = 0; r < batch; ++r) {
        uint64_t s = 0;
        for (size_t j = 0; j < len; ++j) {
            s += mulmod_naive(A[r * len + j] % c->P, x[j] % c->P, c->P);
            s %= c->P;
        }
        out[r] = mulmod_naive((uint32_t)s, c->Rinv, c->P);
    }
}

/* One output of the DFT by definition, X[k] = sum_j x[j] w^(j k) mod P, O(N):
 * for sampled checks of transforms too large for oracle_dft. */
uint32_t oracle_dft_at(uint32_t P, uint32_t w, const uint32_t *x, size_t N, size_t k)
{
    /* wk = w^k by repeated squaring on plain values */
    uint32_t wk = 1u % P, b = w % P;
    for (size_t e = k % N; e; e >>= 1) {
        if (e & 1u) wk = mulmod_naive(wk, b, P);
        b = mulmod_naive(b, b, P);
    }
    uint64_t s = 0;
    uint32_t pw = 1u % P;
    for (size_t j = 0; j < N; ++j) {
        s += mulmod_naive(x[j] % P, pw, P);
        s %= P;
        pw = mulmod_naive(pw, wk, P);
    }
    return (uint32_t)s;
}
