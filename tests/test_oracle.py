"""Pins for the CPU oracle (oracle/), each against something other than the oracle itself.

Pins used (DESIGN.md §4 lists which pin covers which oracle function):
  * the Montgomery identity c * 2^32 = a*b (mod P), 0 <= c < P, which fixes c
    uniquely without ever forming R^-1;
  * brute force over ALL pairs for ALL odd moduli 3 <= P <= 257;
  * the special case P | 2^32 - 1 where R = 1 (mod P) and REDC is the textbook
    a*b mod P;
  * the Bezout identity R R^-1 - P P' = 1 and the closed form
    P' = P - 2 for Fourier primes c 2^n + 1 with 2n >= 32;
  * Python's built-in three-argument pow (a library routine), Fermat's little
    theorem, multiplicativity and the exponent reduction a^e = a^(e mod P-1);
  * SPEC.md's worked examples (tests/golden/spec_worked_examples.json);
  * the internal invariants the paper proves: 0 <= t < 2P before the single
    subtract (Alg. 2), Barrett's <= 3 loop trips,
    r3 = 0 and t in [-(P-1), 2(P-1)] for Alg. 3.
"""
import json

import numpy as np
import pytest

import oracle
import synth

CONFIG_PRIMES = (2013265921, 469762049, 998244353)
FOURIER_FORMS = {2013265921: (15, 27), 469762049: (7, 26), 998244353: (119, 23)}
R = 1 << 32


def odd_moduli(lo=3, hi=257):
    return list(range(lo, hi + 1, 2))


def is_prime(n):
    if n < 2:
        return False
    i = 2
    while i * i <= n:
        if n % i == 0:
            return False
        i += 1
    return True


def identity_ok(P, a, b, c):
    """c*2^32 == a*b (mod P) and c < P, in exact Python-int-free uint64 numpy arithmetic."""
    a = a.astype(np.uint64)
    b = b.astype(np.uint64)
    c = c.astype(np.uint64)
    lhs = (c % np.uint64(P) << np.uint64(32)) % np.uint64(P)  # c < 2^31 so c<<32 < 2^63
    rhs = ((a % np.uint64(P)) * (b % np.uint64(P))) % np.uint64(P)
    return bool(np.all(c < np.uint64(P))) and bool(np.all(lhs == rhs))


# ------------------------------------------------------------------ context

@pytest.mark.parametrize("P", CONFIG_PRIMES + (3, 5, 17, 257, 65537, 2147483647, 12289))
def test_ctx_bezout_and_ranges(P):
    c = oracle.ctx(P)
    assert R * c.Rinv - P * c.Pprime == 1
    assert 0 < c.Rinv < P and 0 < c.Pprime < R
    assert (P * c.Pprime) % R == R - 1             # P' = -P^-1 mod 2^32
    assert c.r1 == R % P and c.r2 == (R * R) % P


@pytest.mark.parametrize("P", CONFIG_PRIMES)
def test_ctx_fourier_closed_form(P):
    # (P-1)^2 = c^2 2^(2n) = 0 mod 2^32 when 2n >= 32, so P (P-2) = (P-1)^2 - 1 = -1 mod 2^32
    cc, n = FOURIER_FORMS[P]
    assert cc * (1 << n) + 1 == P and 2 * n >= 32
    assert oracle.ctx(P).Pprime == P - 2


@pytest.mark.parametrize("P", [0, 1, 2, 4, 100, 1 << 31, (1 << 31) + 1, 0xFFFFFFFF])
def test_ctx_rejects_invalid(P):
    with pytest.raises(oracle.OracleError):
        oracle.ctx(P)


# ------------------------------------------------------------- brute force

def test_bruteforce_all_pairs_all_odd_moduli_le_257():
    """Every pair a, b in [0,P) for every odd 3 <= P <= 257 (54 of them prime)."""
    total = 0
    for P in odd_moduli():
        g = np.arange(P, dtype=np.uint32)
        a = np.repeat(g, P)
        b = np.tile(g, P)
        c = oracle.mont_mul(P, a, b, nthreads=1)
        assert identity_ok(P, a, b, c), P
        total += a.size
    assert sum(P * P for P in odd_moduli() if is_prime(P)) == 1061822
    assert total > 1061822


@pytest.mark.parametrize("P", [3, 5, 17, 257, 65537])
def test_special_case_R_is_one(P):
    """P | 2^32 - 1 => R = 1 (mod P) => REDC(a,b) = a*b mod P (textbook)."""
    assert (R - 1) % P == 0
    rng = np.random.default_rng(P)
    a = rng.integers(0, P, 4096, dtype=np.uint32)
    b = rng.integers(0, P, 4096, dtype=np.uint32)
    c = oracle.mont_mul(P, a, b)
    assert np.array_equal(c, ((a.astype(np.uint64) * b) % np.uint64(P)).astype(np.uint32))
    assert np.array_equal(oracle.to_mont(P, a), a)
    assert np.array_equal(oracle.from_mont(P, a), a)


@pytest.mark.parametrize("P", CONFIG_PRIMES + (2147483647, 1073741827))
def test_random_identity_large(P):
    rng = np.random.default_rng(1)
    a = rng.integers(0, P, 200_000, dtype=np.uint32)
    b = rng.integers(0, P, 200_000, dtype=np.uint32)
    a[:6] = [0, 1, P - 1, P - 2, oracle.ctx(P).r1, oracle.ctx(P).r2]
    b[:6] = [P - 1, P - 1, P - 1, 1, 7, P - 2]
    assert identity_ok(P, a, b, oracle.mont_mul(P, a, b))


@pytest.mark.parametrize("P", CONFIG_PRIMES)
def test_closed_forms(P):
    c = oracle.ctx(P)
    rng = np.random.default_rng(2)
    a = rng.integers(0, P, 50_000, dtype=np.uint32)
    full = lambda v: np.full_like(a, v)
    assert np.array_equal(oracle.mont_mul(P, a, full(c.r1)), a)              # 1-bar is the identity
    assert np.all(oracle.mont_mul(P, a, full(0)) == 0)
    assert np.array_equal(oracle.mont_mul(P, a, full(1)), oracle.from_mont(P, a))
    assert np.array_equal(oracle.mont_mul(P, a, full(c.r2)), oracle.to_mont(P, a))
    # (-1)(-1) R^-1 = R^-1, and R^-1 * R = 1 mod P
    rinv = int(oracle.mont_mul(P, np.array([P - 1], np.uint32), np.array([P - 1], np.uint32))[0])
    assert (rinv * R) % P == 1


@pytest.mark.parametrize("P", (17, 97, 257, 12289))
def test_round_trip_exhaustive_small(P):
    x = np.arange(P, dtype=np.uint32)
    tm = oracle.to_mont(P, x)
    assert np.array_equal(oracle.from_mont(P, tm), x)
    assert np.array_equal(np.sort(tm), x)                     # to_mont is a bijection
    assert identity_ok(P, x, np.ones_like(x), oracle.from_mont(P, x))  # from_mont(x)*R = x


@pytest.mark.parametrize("P", CONFIG_PRIMES)
def test_round_trip_random(P):
    rng = np.random.default_rng(3)
    x = rng.integers(0, P, 100_000, dtype=np.uint32)
    tm = oracle.to_mont(P, x)
    assert np.array_equal(oracle.from_mont(P, tm), x)
    # to_mont(x) = x*2^32 mod P <=> from_mont(to_mont(x)) = x and, through the identity,
    # to_mont(x) * 1 reduces to x: REDC(to_mont(x), 1) * R = to_mont(x)
    assert identity_ok(P, tm, np.ones_like(tm), x)
    assert oracle.to_mont(P, np.array([1], np.uint32))[0] == oracle.ctx(P).r1


# -------------------------------------------------------------- exponentiation

@pytest.mark.parametrize("P", CONFIG_PRIMES + (17, 257))
def test_pow_vs_python_pow(P):
    rng = np.random.default_rng(4)
    base = rng.integers(0, P, 20_000, dtype=np.uint32)
    exp = rng.integers(0, 1 << 31, 20_000, dtype=np.uint32)
    base[:4] = [0, 0, 1, P - 1]
    exp[:4] = [0, 5, 0, (1 << 31) - 1]
    out = oracle.power(P, base, exp)
    ref = np.array([pow(int(x), int(e), P) for x, e in zip(base, exp)], dtype=np.uint32)
    assert np.array_equal(out, ref)
    assert out[0] == 1 % P and out[1] == 0            # 0^0 = 1, 0^e = 0 (G10)


@pytest.mark.parametrize("P", CONFIG_PRIMES + (17, 257, 2147483647))
def test_pow_full_32bit_exponents(P):
    """The product's contract (include/mont.h) takes any uint32 exponent: bits 31..0.  Pinned by
    Python's built-in pow (a library routine), by Fermat with exponents >= 2^31 (e = k(P-1) for
    k >= 2), and by the reduction a^e = a^(e mod (P-1)) for e in [2^31, 2^32) -- an independent
    path that never sets bit 31."""
    rng = np.random.default_rng(41)
    base = rng.integers(0, P, 20_000, dtype=np.uint64).astype(np.uint32)
    exp = rng.integers(1 << 31, 1 << 32, 20_000, dtype=np.uint64).astype(np.uint32)
    base[:3] = [0, 1, P - 1]
    exp[:3] = [0xFFFFFFFF, 0x80000000, 0x80000001]
    out = oracle.power(P, base, exp)
    ref = np.array([pow(int(x), int(e), P) for x, e in zip(base, exp)], dtype=np.uint32)
    assert np.array_equal(out, ref)
    a = base[base != 0]
    e = exp[base != 0]
    assert np.array_equal(oracle.power(P, a, e), oracle.power(P, a, e % np.uint32(P - 1)))
    k = np.uint64((1 << 31) // (P - 1) + 1)
    fermat = np.full(a.shape, min(int(k) * (P - 1), 0xFFFFFFFF // (P - 1) * (P - 1)), dtype=np.uint32)
    assert int(fermat[0]) >= 1 << 31
    assert np.all(oracle.power(P, a, fermat) == 1)                     # Fermat: a^(k(P-1)) = 1
    assert oracle.pow1(P, 0, 0x80000000) == 0 and oracle.pow1(P, 5 % P, 0x80000000) == pow(5, 1 << 31, P)


@pytest.mark.parametrize("P", CONFIG_PRIMES)
def test_pow_fermat_and_laws(P):
    rng = np.random.default_rng(5)
    a = rng.integers(1, P, 5000, dtype=np.uint32)
    assert np.all(oracle.power(P, a, np.full_like(a, P - 1)) == 1)                 # Fermat
    assert np.all(oracle.power(P, a, np.zeros_like(a)) == 1)
    assert np.array_equal(oracle.power(P, a, np.ones_like(a)), a)
    e1 = rng.integers(0, 1 << 30, 5000, dtype=np.uint32)
    e2 = rng.integers(0, 1 << 30, 5000, dtype=np.uint32)
    lhs = oracle.power(P, a, e1 + e2)
    rhs = (oracle.power(P, a, e1).astype(np.uint64) * oracle.power(P, a, e2)) % np.uint64(P)
    assert np.array_equal(lhs, rhs.astype(np.uint32))                                # multiplicativity
    e = rng.integers(0, 1 << 31, 5000, dtype=np.uint32)
    assert np.array_equal(oracle.power(P, a, e), oracle.power(P, a, (e % np.uint32(P - 1))))


def test_pow_primitive_root_469762049():
    P = 469762049           # 7 * 2^26 + 1, primitive root 3
    assert oracle.pow1(P, 3, (P - 1) // 2) == P - 1
    for q in (2, 7):
        assert oracle.pow1(P, 3, (P - 1) // q) != 1


# ------------------------------------------------------------------- twiddles

def test_twiddle_root_and_table():
    P, L = 2013265921, 1 << 14
    w = oracle.root_of_unity(P, synth.G11_GENERATOR, L)
    assert pow(w, L, P) == 1 and pow(w, L // 2, P) == P - 1                    # primitive 2^14-th root
    assert w == pow(31, (P - 1) // L, P)
    tw = oracle.twiddle_table(P, w, L)
    c = oracle.ctx(P)
    assert tw[0] == c.r1
    js = np.array([0, 1, 2, 3, 8191, 8192, 16383])
    for j in js:                                                                  # tw[j] = w^j R mod P
        assert int(tw[j]) == (pow(w, int(j), P) * R) % P
    x = synth.c3_x(P, batch=8, length=L)
    out = oracle.twiddle(P, x, tw)
    assert np.array_equal(out[:, 0], x[:, 0])                                     # column 0: identity
    assert np.array_equal(out[:, L // 2], (np.uint32(P) - x[:, L // 2]) % np.uint32(P))  # w^(L/2) = -1
    for r, j in [(0, 1), (3, 77), (7, 16383), (5, 4096)]:
        assert int(out[r, j]) == (int(x[r, j]) * pow(w, j, P)) % P


def test_twiddle_matches_mont_mul():
    P, L = 998244353, 1000
    rng = np.random.default_rng(6)
    x = rng.integers(0, P, (7, L), dtype=np.uint32)
    tw = rng.integers(0, P, L, dtype=np.uint32)
    out = oracle.twiddle(P, x, tw)
    assert identity_ok(P, x.reshape(-1), np.tile(tw, 7), out.reshape(-1))


# ------------------------------------------------------------------- checksum

def test_checksum():
    P = 2013265921
    rng = np.random.default_rng(7)
    x = rng.integers(0, P, 1_000_003, dtype=np.uint32)
    assert oracle.checksum(P, x) == sum(int(v) for v in x) % P
    assert oracle.checksum(P, np.zeros(0, np.uint32)) == 0
    # partition invariance: slice sums combine to the whole
    parts = [oracle.raw_sum(s) for s in np.array_split(x, 7)]
    assert sum(parts) % P == oracle.checksum(P, x)


# ------------------------------------------------- SPEC worked examples (l small)

def test_spec_worked_examples(golden_dir):
    g = json.loads((golden_dir / "spec_worked_examples.json").read_text())
    for e in g["precompute"]:
        c = oracle.ctx(e["P"], e["l"])
        assert c.Rinv == e["Rinv"] and c.Pprime == e["Pprime"], e["cite"]
        if "R2modP" in e:
            assert c.r2 == e["R2modP"] and c.bk == e["k_barrett"] and c.bPprime == e["Pprime_barrett"]
    for e in g["mulmod_naive"]:
        assert oracle.mulmod(e["a"], e["b"], e["P"]) == e["out"], e["cite"]
    for e in g["barrett"]:
        assert oracle.barrett(e["P"], e["a"], e["b"]) == (e["out"], e["loops"]), e["cite"]
    for e in g["redc"]:
        t, flags = oracle.redc_l(e["P"], e["l"], e["T"])
        assert t == e["out"] and (flags & 3) == 0, e["cite"]
    for e in g["mont_mul"]:
        assert oracle.mont_mul1(e["P"], e["a"], e["b"], e["l"]) == e["out"], e["cite"]
    c = lambda e: oracle.ctx(e["P"], e["l"])
    for e in g["to_mont"]:
        assert oracle.lib().oracle_to_mont1(oracle.C.byref(c(e)), e["x"]) == e["out"], e["cite"]
    for e in g["from_mont"]:
        assert oracle.lib().oracle_from_mont1(oracle.C.byref(c(e)), e["x"]) == e["out"], e["cite"]
    for e in g["fourier_redc"]:
        t, traw, r3 = oracle.fourier_redc(e["P"], e["l"], e["c"], e["n"], e["a"], e["b"])
        assert (t, traw, r3) == (e["out"], e["t_raw"], 0), e["cite"]
    for e in g["mod_add"]:
        assert oracle.mod_add(e["a"], e["b"], e["P"]) == e["out"], e["cite"]
    for e in g["mod_sub"]:
        assert oracle.mod_sub(e["a"], e["b"], e["P"]) == e["out"], e["cite"]


# -------------------------------- paper algorithms step by step (self-test only)

@pytest.mark.parametrize("P,l", [(17, 5), (97, 7), (257, 9), (257, 32), (2013265921, 32), (469762049, 29)])
def test_alg2_redc_invariants(P, l):
    """Alg. 2: exact division by R and 0 <= t < 2P before the single subtract."""
    rng = np.random.default_rng(8)
    Rl = 1 << l
    for _ in range(3000):
        a, b = int(rng.integers(0, P)), int(rng.integers(0, P))
        T = a * b
        t, flags = oracle.redc_l(P, l, T)
        assert flags & 3 == 0
        assert (t * Rl - T) % P == 0 and 0 <= t < P


@pytest.mark.parametrize("P", CONFIG_PRIMES + (17, 97, 12289))
def test_alg1_barrett(P):
    rng = np.random.default_rng(9)
    for _ in range(5000):
        a, b = int(rng.integers(0, P)), int(rng.integers(0, P))
        t, loops = oracle.barrett(P, a, b)
        assert t == (a * b) % P and loops <= 3


@pytest.mark.parametrize("P,l", [(2013265921, 32), (469762049, 32), (998244353, 32), (97, 7), (469762049, 29)])
def test_alg3_fourier_redc(P, l):
    cc, n = {97: (3, 5), **FOURIER_FORMS}[P]
    assert 2 * n >= l
    rng = np.random.default_rng(10)
    for _ in range(5000):
        a, b = int(rng.integers(0, P)), int(rng.integers(0, P))
        t, traw, r3 = oracle.fourier_redc(P, l, cc, n, a, b)
        assert r3 == 0
        assert -(P - 1) <= traw <= 2 * (P - 1)                   # PAPER.md:117 (interval reading G7)
        assert (t * (1 << l) - a * b) % P == 0 and 0 <= t < P


# ------------------------------------------------------------- NTT (NEXT #1)

@pytest.mark.parametrize("P", CONFIG_PRIMES)
@pytest.mark.parametrize("N", [1, 2, 4, 8, 64, 256])
def test_dft_pins(P, N):
    """Pins for the definition-DFT: delta -> ones, ones -> N e0, e1 -> powers of w, inverse round trip,
    and the convolution theorem against the (independent) definition of cyclic convolution."""
    w = oracle.root_of_unity(P, {2013265921: 31, 469762049: 3, 998244353: 3}[P], N)
    assert pow(w, N, P) == 1 and (N == 1 or pow(w, N // 2, P) == P - 1)
    e0 = np.zeros(N, np.uint32)
    e0[0] = 1
    assert np.all(oracle.dft(P, w, e0) == 1)
    ones = np.ones(N, np.uint32)
    ref = np.zeros(N, np.uint32)
    ref[0] = N % P
    assert np.array_equal(oracle.dft(P, w, ones), ref)
    if N > 1:
        e1 = np.zeros(N, np.uint32)
        e1[1] = 1
        assert [int(v) for v in oracle.dft(P, w, e1)] == [pow(w, k, P) for k in range(N)]
    rng = np.random.default_rng(N)
    x = rng.integers(0, P, N, dtype=np.uint64).astype(np.uint32)
    X = oracle.dft(P, w, x)
    winv = oracle.inverse(w, P)
    assert (winv * w) % P == 1
    ninv = oracle.inverse(N, P)
    back = (oracle.dft(P, winv, X).astype(np.uint64) * ninv % P).astype(np.uint32)
    assert np.array_equal(back, x)
    a = rng.integers(0, P, N, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, P, N, dtype=np.uint64).astype(np.uint32)
    prod = (oracle.dft(P, w, a).astype(np.uint64) * oracle.dft(P, w, b) % P).astype(np.uint32)
    conv = (oracle.dft(P, winv, prod).astype(np.uint64) * ninv % P).astype(np.uint32)
    assert np.array_equal(conv, oracle.cyclic_conv(P, a, b))


def test_cyclic_conv_small_integers():
    """Cyclic convolution of small integers equals numpy's exact integer convolution folded mod N."""
    P, N = 998244353, 16
    rng = np.random.default_rng(3)
    a = rng.integers(0, 100, N).astype(np.uint32)
    b = rng.integers(0, 100, N).astype(np.uint32)
    full = np.convolve(a.astype(np.int64), b.astype(np.int64))
    folded = full[:N].copy()
    folded[:N - 1] += full[N:]
    assert np.array_equal(oracle.cyclic_conv(P, a, b), folded.astype(np.uint32))


def test_mulmod_vec_pins():
    """Plain products: brute force all pairs for small P against Python ints; the Barrett step-by-step
    oracle and the definition agree (Alg. 1 reaches a*b mod P)."""
    for P in (3, 17, 97, 257):
        g = np.arange(P, dtype=np.uint32)
        a, b = np.repeat(g, P), np.tile(g, P)
        c = oracle.mulmod_vec(P, a, b)
        assert all(int(x) == (int(y) * int(z)) % P for x, y, z in zip(c[::7], a[::7], b[::7]))
    P = 2013265921
    rng = np.random.default_rng(30)
    a = rng.integers(0, P, 3000, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, P, 3000, dtype=np.uint64).astype(np.uint32)
    c = oracle.mulmod_vec(P, a, b)
    for i in range(0, 3000, 17):
        assert int(c[i]) == oracle.barrett(P, int(a[i]), int(b[i]))[0] == (int(a[i]) * int(b[i])) % P


@pytest.mark.parametrize("P", CONFIG_PRIMES + (17,))
def test_dot_pins(P):
    """dot(A, to_mont(x)) is the plain dot product mod P (Python ints); the REDC-domain identity."""
    rng = np.random.default_rng(31)
    A = rng.integers(0, P, (5, 300), dtype=np.uint64).astype(np.uint32)
    x = rng.integers(0, P, 300, dtype=np.uint64).astype(np.uint32)
    got = oracle.dot(P, A, oracle.to_mont(P, x))
    for r in range(5):
        assert int(got[r]) == sum(int(a) * int(b) for a, b in zip(A[r], x)) % P
    raw = oracle.dot(P, A, x)
    for r in range(5):
        assert (int(raw[r]) << 32) % P == sum(int(a) * int(b) for a, b in zip(A[r], x)) % P


def test_dft_at_matches_dft():
    P = 998244353
    N = 512
    w = oracle.root_of_unity(P, 3, N)
    x = synth.uniform(42, 40, P, 0, N)
    X = oracle.dft(P, w, x)
    for k in (0, 1, 7, 255, 511, 513):
        assert oracle.dft_at(P, w, x, k) == int(X[k % N])
