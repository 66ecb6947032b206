"""GPU parity: every kernel through the C ABI vs the CPU oracle, bit-exact.

Sizes span several tiles and ragged tails; edge cases cover n = 0..9,
misaligned (4/8/12-byte offset) operands, mixed alignments, in-place calls,
the fixed-index edge values of configs[0] and the specials of configs[1].
Full-size configs are in tests/test_gpu_fullsize.py.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

PRIMES = (2013265921, 469762049, 998244353)
ODD_SMALL = (3, 5, 17, 97, 257, 65537, 12289, 2147483647, 1073741827)


@pytest.fixture(scope="module")
def m():
    import paper_1609_00999_b200 as mod
    return mod


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def offset_view(x: np.ndarray, off: int):
    """Device tensor holding x starting `off` uint32 elements into a fresh allocation."""
    buf = torch.empty(x.size + 8, dtype=torch.uint32, device="cuda")
    v = buf[off:off + x.size]
    v.copy_(dev(x))
    return v


# ------------------------------------------------------------------ mul_vec

@pytest.mark.parametrize("P", PRIMES)
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 8, 9, 31, 33, 1000, 4099, 65536, 262147, 1 << 20 | 5])
def test_mul_vec_parity(m, P, n):
    a, b = synth.c2_inputs(P, 0, n)
    ctx = m.ctx_init(P)
    c = m.mul_vec(ctx, dev(a), dev(b))
    assert np.array_equal(host(c), oracle.mont_mul(P, a, b))


def test_mul_vec_c1_config(m):
    P = 2013265921
    a, b = synth.c1_inputs(P)
    c = host(m.mul_vec(m.ctx_init(P), dev(a), dev(b)))
    ref = oracle.mont_mul(P, a, b)
    assert np.array_equal(c, ref)
    assert oracle.checksum(P, c) == oracle.checksum(P, ref)


@pytest.mark.parametrize("P", ODD_SMALL)
def test_mul_vec_other_moduli(m, P):
    rng = np.random.default_rng(P)
    n = 100_003
    a = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    a[:3] = [0, P - 1, P - 1]
    b[:3] = [P - 1, P - 1, 0]
    c = m.mul_vec(m.ctx_init(P), dev(a), dev(b))
    assert np.array_equal(host(c), oracle.mont_mul(P, a, b))


@pytest.mark.parametrize("P", (3, 5, 7, 17, 97, 251, 257))
def test_mul_vec_all_pairs_small(m, P):
    g = np.arange(P, dtype=np.uint32)
    a = np.repeat(g, P)
    b = np.tile(g, P)
    c = m.mul_vec(m.ctx_init(P), dev(a), dev(b))
    assert np.array_equal(host(c), oracle.mont_mul(P, a, b))


def test_mul_vec_one_operand_noncanonical(m):
    """REDC needs only a*b < R P: any uint32 a with b < P is valid."""
    P = 2013265921
    rng = np.random.default_rng(12)
    n = 50_001
    a = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    a[:2] = [0xFFFFFFFF, 0xFFFFFFFF]
    b[:2] = [P - 1, 0]
    c = host(m.mul_vec(m.ctx_init(P), dev(a), dev(b)))
    assert np.array_equal(c, oracle.mont_mul(P, a % np.uint32(P), b))


@pytest.mark.parametrize("oa,ob,oc", [(1, 1, 1), (2, 2, 2), (3, 3, 3), (0, 1, 2), (1, 0, 0), (3, 0, 1), (0, 0, 3)])
@pytest.mark.parametrize("n", [0, 1, 2, 3, 5, 6, 9, 1023, 40_000 + 3])
@pytest.mark.parametrize("variant", [0, 2, 3])
def test_mul_vec_alignment(m, oa, ob, oc, n, variant):
    P = 998244353
    a, b = synth.c2_inputs(P, 7, n)
    ta, tb = offset_view(a, oa), offset_view(b, ob)
    buf = dev(np.full(n + 8, 0xDEADBEEF, dtype=np.uint32))
    tc = buf[oc:oc + n]
    m.mul_vec(m.ctx_init(P), ta, tb, out=tc, cfg=m.Launch(variant=variant))
    full = host(buf)
    assert np.array_equal(full[oc:oc + n], oracle.mont_mul(P, a, b))
    # nothing outside [oc, oc+n) was written
    assert np.all(full[:oc] == 0xDEADBEEF) and np.all(full[oc + n:] == 0xDEADBEEF)


def test_mul_vec_in_place(m):
    P = 469762049
    a, b = synth.c2_inputs(P, 0, 100_001)
    ta, tb = dev(a), dev(b)
    m.mul_vec(m.ctx_init(P), ta, tb, out=ta)
    assert np.array_equal(host(ta), oracle.mont_mul(P, a, b))
    tb2 = dev(b)
    m.mul_vec(m.ctx_init(P), dev(a), tb2, out=tb2)
    assert np.array_equal(host(tb2), oracle.mont_mul(P, a, b))


@pytest.mark.parametrize("threads,ctas,unroll,variant,chunk", [(32, 1, 1, 0, 0), (128, 2, 2, 0, 0), (256, 8, 8, 0, 0),
                                                               (512, 4, 4, 1, 0), (512, 1, 8, 1, 0), (64, 32, 4, 0, 0),
                                                               (256, 4, 1, 2, 0), (256, 4, 1, 2, 1024),
                                                               (256, 4, 1, 2, 16384), (256, 4, 1, 2, 4),
                                                               (128, 1, 1, 3, 0), (256, 2, 1, 3, 0), (32, 1, 1, 3, 4),
                                                               (128, 1, 1, 3, 512), (256, 1, 1, 3, 4096)])
def test_mul_vec_launch_configs(m, threads, ctas, unroll, variant, chunk):
    P = 2013265921
    a, b = synth.c2_inputs(P, 0, 300_007)
    cfg = m.Launch(threads=threads, ctas_per_sm=ctas, unroll=unroll, variant=variant, chunk=chunk)
    c = m.mul_vec(m.ctx_init(P), dev(a), dev(b), cfg=cfg)
    assert np.array_equal(host(c), oracle.mont_mul(P, a, b))


def test_mul_vec_pipe_rejects(m):
    """variant 3: a tile ring that does not fit in shared memory, or more than 256 threads."""
    P = 2013265921
    a = dev(synth.c2_inputs(P, 0, 4096)[0])
    for cfg in (m.Launch(threads=256, ctas_per_sm=1, unroll=1, variant=3, chunk=8192),
                m.Launch(threads=512, ctas_per_sm=1, unroll=1, variant=3, chunk=1024)):
        with pytest.raises(m.MontError):
            m.mul_vec(m.ctx_init(P), a, a, cfg=cfg)


def test_mul_vec_empty(m):
    e = torch.empty(0, dtype=torch.uint32, device="cuda")
    assert m.mul_vec(m.ctx_init(17), e, e).numel() == 0


# ------------------------------------------------------------- to/from_mont

@pytest.mark.parametrize("P", PRIMES + (3, 17, 2147483647))
@pytest.mark.parametrize("n", [1, 3, 4, 5, 4096 + 3, 1 << 20])
def test_to_from_mont_parity(m, P, n):
    x = synth.uniform(42, 9, P, 0, n)
    ctx = m.ctx_init(P)
    tm = m.to_mont(ctx, dev(x))
    assert np.array_equal(host(tm), oracle.to_mont(P, x))
    fm = m.from_mont(ctx, dev(x))
    assert np.array_equal(host(fm), oracle.from_mont(P, x))
    assert np.array_equal(host(m.from_mont(ctx, tm)), x)


def test_to_from_mont_noncanonical_input(m):
    P = 2013265921
    rng = np.random.default_rng(13)
    x = rng.integers(0, 1 << 32, 10_001, dtype=np.uint64).astype(np.uint32)
    x[:2] = [0xFFFFFFFF, P]
    ctx = m.ctx_init(P)
    assert np.array_equal(host(m.to_mont(ctx, dev(x))), oracle.to_mont(P, x))
    assert np.array_equal(host(m.from_mont(ctx, dev(x))), oracle.from_mont(P, x))


@pytest.mark.parametrize("off_in,off_out", [(1, 1), (1, 2), (3, 0), (2, 2)])
def test_to_mont_alignment_in_place(m, off_in, off_out):
    P = 469762049
    x = synth.uniform(42, 9, P, 0, 1001)
    ti = offset_view(x, off_in)
    to = offset_view(np.zeros_like(x), off_out)
    ctx = m.ctx_init(P)
    m.to_mont(ctx, ti, out=to)
    assert np.array_equal(host(to), oracle.to_mont(P, x))
    m.from_mont(ctx, to, out=to)
    assert np.array_equal(host(to), x)


# --------------------------------------------------------------------- pow

@pytest.mark.parametrize("P", PRIMES + (17, 257, 2147483647, 3, 536870909, 536870923))
@pytest.mark.parametrize("variant", list(range(9)) + list(range(10, 18)))
def test_pow_parity(m, P, variant):
    """Every ladder variant vs the oracle; 536870909 / 536870923 straddle 2^29, where variants
    13, 14, 16 switch from lazy [0, 2P) Shoup outputs to one canonicalising subtract."""
    n = 20_003
    base = synth.uniform(42, synth.STREAM_BASE, P, 0, n, low=1) if P > 3 else \
        np.random.default_rng(0).integers(0, 3, n).astype(np.uint32)
    exp = synth.exponents(42, synth.STREAM_EXP, 0, n)
    base[:6] = [0, 0, 1, P - 1, P - 1, 2 % P]
    exp[:6] = [0, 7, 0, 0, (1 << 31) - 1, 0x7FFFFFFF]
    cfg = m.Launch(variant=variant)
    out = m.pow_vec(m.ctx_init(P), dev(base), dev(exp), cfg=cfg)
    assert np.array_equal(host(out), oracle.power(P, base, exp))


@pytest.mark.parametrize("P", [998244353, 469762049, 2013265921, 2147483647, 17])
def test_pow_full_32bit_exponents_and_big_bases(m, P):
    """Header contract: any uint32 base (reduced mod P) and full 32-bit exponents, every variant
    (incl. Alg. 3 = 9 for the Fourier primes) against the oracle, whose ladder covers bits 31..0
    (pinned by Python's pow and Fermat in tests/test_oracle.py)."""
    rng = np.random.default_rng(14)
    n = 9_999
    base = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    exp = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    exp[:4] = [0xFFFFFFFF, 1 << 31, 0, (1 << 31) + 1]
    base[:4] = [P - 1, 0xFFFFFFFF, 0, P]
    ref = oracle.power(P, base, exp)
    assert int(ref[0]) == pow(P - 1, 0xFFFFFFFF, P) and int(ref[1]) == pow(0xFFFFFFFF, 1 << 31, P)
    variants = list(range(9)) + list(range(10, 18)) + ([9] if P in (998244353, 469762049, 2013265921) else [])
    for variant in variants:
        out = m.pow_vec(m.ctx_init(P), dev(base), dev(exp), cfg=m.Launch(variant=variant))
        assert np.array_equal(host(out), ref), variant


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8, 9, 12, 1000, 1 << 16 | 3, (1 << 16) + 4])
@pytest.mark.parametrize("variant", [0, 5, 6, 10, 11, 12, 13, 14, 17])
def test_pow_ragged_and_misaligned(m, n, variant):
    P = 469762049
    base, exp = synth.c4_inputs(P, 5, n)
    ref = oracle.power(P, base, exp)
    ctx = m.ctx_init(P)
    cfg = m.Launch(variant=variant)
    assert np.array_equal(host(m.pow_vec(ctx, dev(base), dev(exp), cfg=cfg)), ref)
    tb, te = offset_view(base, 1), offset_view(exp, 1)
    to = offset_view(np.zeros_like(base), 1)
    m.pow_vec(ctx, tb, te, out=to, cfg=cfg)
    assert np.array_equal(host(to), ref)
    tb, te = offset_view(base, 1), offset_view(exp, 2)
    assert np.array_equal(host(m.pow_vec(ctx, tb, te, cfg=cfg)), ref)


# ----------------------------------------------------------------- twiddle

@pytest.mark.parametrize("L", [4, 16, 1000, 1024, 4096, 16384, 16388, 65536])
def test_twiddle_table_parity(m, L):
    P = 2013265921
    order = 1 << 14
    w = oracle.root_of_unity(P, synth.G11_GENERATOR, order)
    tw = m.twiddle_table(m.ctx_init(P), w, L)
    assert np.array_equal(host(tw), oracle.twiddle_table(P, w, L))


@pytest.mark.parametrize("batch,L", [(1, 4), (3, 8), (5, 1000), (17, 1024), (7, 16384), (3, 16388), (2, 40000),
                                     (1000, 64), (33, 4100), (513, 4), (4096, 2048)])
@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
def test_twiddle_parity(m, batch, L, variant):
    P = 2013265921
    x = synth.c3_x(P, batch=batch, length=L)
    rng = np.random.default_rng(L)
    tw = rng.integers(0, P, L, dtype=np.uint64).astype(np.uint32)
    out = m.mul_twiddle(m.ctx_init(P), dev(x), dev(tw), cfg=m.Launch(variant=variant))
    assert np.array_equal(host(out), oracle.twiddle(P, x, tw))


@pytest.mark.parametrize("batch,L", [(3, 5), (4, 7), (2, 1001), (9, 3)])
def test_twiddle_ragged_len(m, batch, L):
    P = 998244353
    x = synth.c3_x(P, batch=batch, length=L)
    tw = synth.uniform(42, 11, P, 0, L)
    out = m.mul_twiddle(m.ctx_init(P), dev(x), dev(tw))
    assert np.array_equal(host(out), oracle.twiddle(P, x, tw))


@pytest.mark.parametrize("chunk,ctas,unroll,threads", [(4, 1, 1, 32), (1024, 2, 2, 128), (4096, 8, 8, 512),
                                                       (16384, 3, 4, 512), (36, 3, 4, 256)])
def test_twiddle_launch_configs(m, chunk, ctas, unroll, threads):
    P = 469762049
    batch, L = 37, 8192
    x = synth.c3_x(P, batch=batch, length=L)
    tw = synth.uniform(42, 11, P, 0, L)
    # variant 4 (bulk-copy staged table): the one whose shape chunk / ctas_per_sm set
    cfg = m.Launch(threads=threads, ctas_per_sm=ctas, unroll=unroll, chunk=chunk, variant=4)
    out = m.mul_twiddle(m.ctx_init(P), dev(x), dev(tw), cfg=cfg)
    assert np.array_equal(host(out), oracle.twiddle(P, x, tw))


def test_twiddle_misaligned_and_in_place(m):
    P = 2013265921
    batch, L = 6, 1024
    x = synth.c3_x(P, batch=batch, length=L)
    tw = synth.uniform(42, 11, P, 0, L)
    ref = oracle.twiddle(P, x, tw)
    ctx = m.ctx_init(P)
    tx = offset_view(x.reshape(-1), 1).view(batch, L)
    ttw = offset_view(tw, 3)
    assert np.array_equal(host(m.mul_twiddle(ctx, tx, ttw)), ref)
    tx = dev(x)
    m.mul_twiddle(ctx, tx, dev(tw), out=tx)
    assert np.array_equal(host(tx), ref)


# ---------------------------------------------------------------- checksum

@pytest.mark.parametrize("n", [1, 3, 4, 5, 1000, 65536 + 7, 1 << 22])
@pytest.mark.parametrize("off", [0, 1, 2, 3])
def test_checksum(m, n, off):
    P = 2013265921
    x = synth.uniform(42, 1, P, 0, n)
    acc = m.checksum(m.ctx_init(P), offset_view(x, off))
    torch.cuda.synchronize()
    assert int(acc.item()) == oracle.raw_sum(x)


# ------------------------------------------------------- fused mul + checksum

@pytest.mark.parametrize("n", [1, 3, 5, 4096, 65536 + 5, 1 << 20 | 3])
@pytest.mark.parametrize("off", [0, 1])
def test_mul_vec_checksum_fused(m, n, off):
    P = 2013265921
    a, b = synth.c5_inputs(P, 1000, n)
    ref = oracle.mont_mul(P, a, b)
    ctx = m.ctx_init(P)
    ta, tb = offset_view(a, off), offset_view(b, off)
    tc = offset_view(np.zeros_like(a), off)
    c, acc = m.mul_vec_checksum(ctx, ta, tb, out=tc)
    assert np.array_equal(host(c), ref)
    assert int(acc.item()) == oracle.raw_sum(ref)
    # accumulates across calls; misaligned operands take the 32-bit path
    tb2 = offset_view(b, (off + 1) % 4)
    m.mul_vec_checksum(ctx, ta, tb2, acc=acc)
    assert int(acc.item()) == 2 * oracle.raw_sum(ref)


@pytest.mark.parametrize("threads,unroll,variant", [(256, 1, 0), (512, 4, 0), (128, 2, 1), (256, 8, 1), (256, 1, 2),
                                                    (128, 1, 3), (256, 1, 3)])
def test_mul_vec_checksum_configs(m, threads, unroll, variant):
    P = 998244353
    a, b = synth.c2_inputs(P, 0, 300_001)
    ref = oracle.mont_mul(P, a, b)
    cfg = m.Launch(threads=threads, unroll=unroll, variant=variant, ctas_per_sm=4)
    c, acc = m.mul_vec_checksum(m.ctx_init(P), dev(a), dev(b), cfg=cfg)
    assert np.array_equal(host(c), ref) and int(acc.item()) == oracle.raw_sum(ref)


@pytest.mark.parametrize("unroll,threads,variant", [(1, 256, 0), (2, 256, 0), (4, 512, 0), (2, 128, 1), (1, 128, 3),
                                                    (1, 256, 3)])
def test_to_from_mont_configs(m, unroll, threads, variant):
    P = 469762049
    x = synth.uniform(42, 9, P, 0, 123_457)
    cfg = m.Launch(threads=threads, unroll=unroll, variant=variant, ctas_per_sm=4)
    ctx = m.ctx_init(P)
    tm = m.to_mont(ctx, dev(x), cfg=cfg)
    assert np.array_equal(host(tm), oracle.to_mont(P, x))
    assert np.array_equal(host(m.from_mont(ctx, tm, cfg=cfg)), x)


# ------------------------------------------- out-of-bounds guards (no sanitizer on this pool)

GUARD = 64


def guarded(n, off):
    """A device buffer of n words at offset `off` inside GUARD canary words on each side."""
    buf = dev(np.full(n + 2 * GUARD, 0xA5A5A5A5, dtype=np.uint32))
    return buf, buf[GUARD + off:GUARD + off + n]


def canaries_intact(buf, n, off):
    h = host(buf)
    return bool(np.all(h[:GUARD + off] == 0xA5A5A5A5) and np.all(h[GUARD + off + n:] == 0xA5A5A5A5))


@pytest.mark.parametrize("n", [1, 3, 4, 5, 7, 33, 4099, 65537])
@pytest.mark.parametrize("off", [0, 1, 2, 3])
def test_guards_all_kernels(m, n, off):
    P = 469762049
    ctx = m.ctx_init(P)
    a, b = synth.c2_inputs(P, 0, n)
    for name, run, ref in [
        ("mul_vec", lambda o: m.mul_vec(ctx, dev(a), dev(b), out=o), oracle.mont_mul(P, a, b)),
        ("mul_vec_checksum", lambda o: m.mul_vec_checksum(ctx, dev(a), dev(b), out=o), oracle.mont_mul(P, a, b)),
        ("to_mont", lambda o: m.to_mont(ctx, dev(a), out=o), oracle.to_mont(P, a)),
        ("from_mont", lambda o: m.from_mont(ctx, dev(a), out=o), oracle.from_mont(P, a)),
        ("pow_vec", lambda o: m.pow_vec(ctx, dev(a), dev(b), out=o), oracle.power(P, a, b)),
    ]:
        buf, o = guarded(n, off)
        run(o)
        assert np.array_equal(host(o), ref), name
        assert canaries_intact(buf, n, off), name


@pytest.mark.parametrize("batch,L,off", [(3, 1000, 1), (5, 16, 0), (2, 4100, 3), (9, 7, 2)])
def test_guards_twiddle(m, batch, L, off):
    P = 2013265921
    x = synth.c3_x(P, batch=batch, length=L)
    tw = synth.uniform(42, 11, P, 0, L)
    buf, o = guarded(batch * L, off)
    m.mul_twiddle(m.ctx_init(P), dev(x), dev(tw), out=o.view(batch, L))
    assert np.array_equal(host(o).reshape(batch, L), oracle.twiddle(P, x, tw))
    assert canaries_intact(buf, batch * L, off)


@pytest.mark.parametrize("log_n", [1, 4, 5, 9, 12])
@pytest.mark.parametrize("batch", [1, 3, 7])
def test_guards_ntt(m, log_n, batch):
    P = 998244353
    N = 1 << log_n
    ctx = m.ctx_init(P)
    w = oracle.root_of_unity(P, 3, N)
    tw = m.ntt_twiddles(ctx, w, log_n)
    x = synth.uniform(42, 26, P, 0, batch * N).reshape(batch, N)
    buf, o = guarded(batch * N, 0)
    o.copy_(dev(x.reshape(-1)))
    m.ntt(ctx, o.view(batch, N), tw)
    assert np.array_equal(host(o).reshape(batch, N), oracle.dft(P, w, x))
    assert canaries_intact(buf, batch * N, 0)



# ------------------------------------------ NEXT #2: Fourier-prime REDC ladder (variant 9)

@pytest.mark.parametrize("P", [469762049, 998244353, 65537, 786433, 2013265921, 1811939329, 1711276033, 2113929217])
@pytest.mark.parametrize("n", [1, 4, 5, 20003])
def test_pow_fourier_variant(m, P, n):
    # 469762049 = 7*2^26+1, 998244353 = 119*2^23+1, 65537 = 2^16+1, 786433 = 3*2^18+1; with 3P >= 2^32
    # (33-bit t, reading G8): 2013265921 = 15*2^27+1, 1811939329 = 27*2^26+1, 1711276033 = 51*2^25+1,
    # 2113929217 = 63*2^25+1
    base = synth.uniform(42, 3, P, 0, n, low=1)
    e = synth.exponents(42, 4, 0, n)
    base[:min(n, 3)] = [P - 1, 1, P - 2][:min(n, 3)]
    out = m.pow_vec(m.ctx_init(P), dev(base), dev(e), cfg=m.Launch(variant=9))
    assert np.array_equal(host(out), oracle.power(P, base, e))


def test_pow_fourier_33bit_t_both_signs(m):
    """P0 = 15*2^27+1 (3P > 2^32): all pairs of a set of residues that drive t = q1 - q2 + q3 to
    both ends of [-(P-1), 2(P-1)], through a ladder whose every product is Alg. 3:
    x^e with e = 2 is one squaring; x^3 one squaring and one multiply."""
    P = 2013265921
    vals = np.array([0, 1, 2, P - 1, P - 2, (P - 1) // 2, (P + 1) // 2, 1 << 30, (1 << 31) - 1 - P % 7,
                     268435454, 1172168163, 943718400, 1 << 27, (1 << 27) + 1, 15, 16], dtype=np.uint64) % P
    base = np.repeat(vals, 4).astype(np.uint32)
    exp = np.tile(np.array([2, 3, 0xFFFFFFFF, 0x80000001], dtype=np.uint32), len(vals))
    rng = np.random.default_rng(33)
    base = np.concatenate([base, rng.integers(0, P, 40000, dtype=np.uint64).astype(np.uint32)])
    exp = np.concatenate([exp, rng.integers(0, 1 << 32, 40000, dtype=np.uint64).astype(np.uint32)])
    out = m.pow_vec(m.ctx_init(P), dev(base), dev(exp), cfg=m.Launch(variant=9))
    assert np.array_equal(host(out), oracle.power(P, base, exp))


def test_pow_fourier_unsupported(m):
    for P in (1000003, 12289):   # not a Fourier prime / 2n < 32
        with pytest.raises(m.MontError) as ei:
            m.pow_vec(m.ctx_init(P), dev(np.ones(8, np.uint32)), dev(np.ones(8, np.uint32)), cfg=m.Launch(variant=9))
        assert ei.value.status == 4


@pytest.mark.parametrize("ctas", [0, 1, 3, 5])
@pytest.mark.parametrize("n", [4, 8, 12, 4100, 1 << 20])
@pytest.mark.parametrize("variant", [10, 11, 13])
def test_pow_variant10_grids(m, ctas, n, variant):
    P = 469762049
    base, e = synth.c4_inputs(P, 0, n)
    out = m.pow_vec(m.ctx_init(P), dev(base), dev(e), cfg=m.Launch(variant=variant, ctas_per_sm=ctas))
    assert np.array_equal(host(out), oracle.power(P, base, e))


@pytest.mark.parametrize("threads", [64, 128, 256])
@pytest.mark.parametrize("variant", [0, 11, 12, 13, 16])
@pytest.mark.parametrize("n", [1, 7, 8, 9, 4100, 1 << 20])
def test_pow2_cta_sizes(m, threads, variant, n):
    """The k_pow2 ladders (default variant 11 at 128 threads) at every CTA size they accept."""
    P = 2013265921
    base, e = synth.c4_inputs(P, 3, n)
    out = m.pow_vec(m.ctx_init(P), dev(base), dev(e), cfg=m.Launch(variant=variant, threads=threads))
    assert np.array_equal(host(out), oracle.power(P, base, e))


def test_pow_rejects_thread_counts(m):
    P = 469762049
    b = dev(np.ones(64, np.uint32))
    for cfg in (m.Launch(variant=17, threads=128), m.Launch(variant=11, threads=96), m.Launch(variant=1, threads=64)):
        with pytest.raises(m.MontError):
            m.pow_vec(m.ctx_init(P), b, b, cfg=cfg)


@pytest.mark.parametrize("n", [1, 3, 4, 5, 7, 8, 9, 33, 4099, 65537])
@pytest.mark.parametrize("variant,threads", [(11, 64), (11, 128), (11, 256), (12, 128), (13, 128), (14, 256),
                                             (9, 256), (10, 256)])
def test_guards_pow_ladders(m, n, variant, threads):
    """Round-2 ladders (and Alg. 3 with the 33-bit t for P0) write exactly their n words: canary
    words on both sides of out (co-aligned operands, the only layout these variants take)."""
    P = 2013265921
    base, e = synth.c4_inputs(P, 9, n)
    buf, o = guarded(n, 0)
    m.pow_vec(m.ctx_init(P), dev(base), dev(e), out=o, cfg=m.Launch(variant=variant, threads=threads))
    assert np.array_equal(host(o), oracle.power(P, base, e))
    assert canaries_intact(buf, n, 0)


@pytest.mark.parametrize("n", [4, 8, 2044, 4100, 65540])
def test_guards_run(m, n):
    """mont_run writes exactly each job's n words (incl. the fused pair's two outputs)."""
    P = 998244353
    ctx = m.ctx_init(P)
    a, b = synth.c2_inputs(P, 0, n)
    bufs = [guarded(n, 0) for _ in range(4)]
    (b0, c), (b1, t), (b2, f), (b3, g) = bufs
    m.run([m.run_job("mul_vec", ctx, c, dev(a), dev(b)), m.run_job("to_mont", ctx, t, dev(a)),
           m.run_job("from_mont", ctx, f, t), m.run_job("from_mont", ctx, g, dev(b))])
    assert np.array_equal(host(c), oracle.mont_mul(P, a, b))
    assert np.array_equal(host(t), oracle.to_mont(P, a)) and np.array_equal(host(f), a)
    assert np.array_equal(host(g), oracle.from_mont(P, b))
    assert all(canaries_intact(buf, n, 0) for buf, _ in bufs)


@pytest.mark.parametrize("batch", [1, 5, 33])
@pytest.mark.parametrize("variant", [1, 2, 3, 4, 5, 6, 7])
def test_guards_dot(m, batch, variant):
    P = 2013265921
    L = 16384
    A = synth.uniform(42, 35, P, 0, batch * L).reshape(batch, L)
    x = synth.uniform(42, 36, P, 0, L)
    buf, o = guarded(batch, 0)
    m.dot(m.ctx_init(P), dev(A), dev(x), out=o, cfg=m.Launch(variant=variant))
    assert np.array_equal(host(o), oracle.dot(P, A, x))
    assert canaries_intact(buf, batch, 0)


@pytest.mark.parametrize("P", PRIMES + (3, 17, 2147483647, 1073741827))
@pytest.mark.parametrize("n", [1, 5, 4100, 1 << 18])
def test_mul_vec_fp64_variant(m, P, n):
    """mont_mul_vec_ex / _checksum_ex variant 4: the same REDC result from two FP64 Barrett
    products per element (a b mod P, then times R^-1 mod P), canonical inputs."""
    a, b = synth.c2_inputs(P, 0, n) if P > 257 else (np.arange(n, dtype=np.uint32) % P, (np.arange(n, dtype=np.uint32) * 7) % P)
    a, b = a.astype(np.uint32), b.astype(np.uint32)
    if n >= 3:
        a[:3], b[:3] = [P - 1, 0, P - 1], [P - 1, P - 1, 1]
    ref = oracle.mont_mul(P, a, b)
    cfg = m.Launch(variant=4)
    assert np.array_equal(host(m.mul_vec(m.ctx_init(P), dev(a), dev(b), cfg=cfg)), ref)
    c, acc = m.mul_vec_checksum(m.ctx_init(P), dev(a), dev(b), cfg=cfg)
    assert np.array_equal(host(c), ref) and int(acc.item()) == oracle.raw_sum(ref)
