"""Full-size parity at BASELINE.json's configs, in the launch configuration bench.py times
(the library defaults), through the C ABI.

Inputs are generated in HBM by the device generator (itself checked against synth/ in
test_gpu_synth.py).  Checks: (1) sampled outputs against the oracle computed element by
element from synth/ (the host generator) at the same indices; (2) properties that hold at any
size, checked on every element with torch int64 arithmetic on the GPU (independent of our
kernels): the Montgomery identity c*2^32 = a*b (mod P) with 0 <= c < P; (3) checksums against
an independent torch reduction.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

P0, P1, P2 = synth.CONFIG_PRIMES
SAMPLES = 20_000


@pytest.fixture(scope="module")
def m():
    import paper_1609_00999_b200 as mod
    return mod


def i64(t):
    return t.view(torch.int32).to(torch.int64) & 0xFFFFFFFF


def identity_all(P, a, b, c, chunk=1 << 24):
    for s in range(0, a.numel(), chunk):
        aa, bb, cc = i64(a[s:s + chunk]), i64(b[s:s + chunk]), i64(c[s:s + chunk])
        if not bool(((cc << 32) % P == (aa * bb) % P).all()) or not bool((cc < P).all()):
            return False
    return True


def sample_idx(n, k=SAMPLES, seed=0):
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([rng.integers(0, n, k), np.arange(8), np.arange(n - 8, n)]))
    return idx.astype(np.int64)


def gen(n, stream_id, P, mode=0, specials=False, start=0, m=None):
    t = torch.empty(n, dtype=torch.uint32, device="cuda")
    m.synth_fill(t, 42, stream_id, start, P, mode, specials)
    return t


@pytest.mark.parametrize("P", [P0, P1, P2])
def test_c2_fullsize(m, P):
    """configs[1]: n = 2^26, 1 % specials, fused mul+checksum (the bench launch)."""
    n = 1 << 26
    a = gen(n, 1, P, 0, True, m=m)
    b = gen(n, 2, P, 0, True, m=m)
    c, acc = m.mul_vec_checksum(m.ctx_init(P), a, b)
    torch.cuda.synchronize()
    idx = sample_idx(n)
    ha, hb = synth.c2_inputs_at(P, idx.astype(np.uint64))
    ref = oracle.mont_mul(P, ha, hb)
    assert np.array_equal(c.cpu().numpy()[idx], ref)
    assert identity_all(P, a, b, c)
    assert int(acc.item()) == int(i64(c).sum().item())
    # the plain mul_vec entry point gives the same array
    c2 = m.mul_vec(m.ctx_init(P), a, b)
    assert bool((c2.view(torch.int32) == c.view(torch.int32)).all())


@pytest.mark.parametrize("P", [P0, P1, P2])
def test_c2_fullsize_every_element(m, P):
    """configs[1] at full size, EVERY element against the oracle (host generator -> oracle on all
    host cores) -- no sampling."""
    n = 1 << 26
    ha, hb = synth.c2_inputs(P, 0, n)
    ref = oracle.mont_mul(P, ha, hb)
    a = gen(n, 1, P, 0, True, m=m)
    b = gen(n, 2, P, 0, True, m=m)
    c, acc = m.mul_vec_checksum(m.ctx_init(P), a, b)
    assert np.array_equal(a.cpu().numpy(), ha) and np.array_equal(b.cpu().numpy(), hb)
    assert np.array_equal(c.cpu().numpy(), ref)
    assert int(acc.item()) % P == oracle.checksum(P, ref)


def test_c3_c4_fullsize_every_element(m):
    """configs[2] and configs[3] at full size, every element against the oracle: the twiddle
    multiply in the default path (flat stream, table through L1) AND in the bulk-copy (TMA)
    staged-table path (mont_mul_twiddle_ex variant 4) -- north_star's "twiddle tables staged in
    shared memory via TMA" at the configs[2] shape."""
    batch, L = 4096, 1 << 14
    hx = synth.c3_x(P0, batch=batch, length=L)
    w = oracle.root_of_unity(P0, synth.G11_GENERATOR, L)
    tw_ref = oracle.twiddle_table(P0, w, L)
    ctx = m.ctx_init(P0)
    ref = oracle.twiddle(P0, hx, tw_ref)
    tx, ttw = torch.from_numpy(hx).cuda(), m.twiddle_table(ctx, w, L)
    out = m.mul_twiddle(ctx, tx, ttw)
    assert np.array_equal(out.cpu().numpy(), ref)
    for v in (4, 3, 1):
        out = m.mul_twiddle(ctx, tx, ttw, cfg=m.Launch(variant=v))
        assert np.array_equal(out.cpu().numpy(), ref), v
    hb, he = synth.c4_inputs(P1, 0, 1 << 24)
    outp = m.pow_vec(m.ctx_init(P1), torch.from_numpy(hb).cuda(), torch.from_numpy(he).cuda())
    assert np.array_equal(outp.cpu().numpy(), oracle.power(P1, hb, he))


def test_c1_full(m):
    """configs[0] exactly: full array vs the oracle, and its checksum."""
    a, b = synth.c1_inputs(P0)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    c, acc = m.mul_vec_checksum(m.ctx_init(P0), ta, tb)
    ref = oracle.mont_mul(P0, a, b)
    assert np.array_equal(c.cpu().numpy(), ref)
    assert int(acc.item()) % P0 == oracle.checksum(P0, ref)
    assert c[0].item() == 0 and c[1].item() == 0


def test_c3_fullsize(m):
    """configs[2]: 4096 x 2^14 against tw[j] = to_mont(w^j), w = 31^((P-1)/2^14)."""
    batch, L = 4096, 1 << 14
    x = gen(batch * L, 5, P0, m=m).view(batch, L)
    w = oracle.root_of_unity(P0, synth.G11_GENERATOR, L)
    tw_ref = oracle.twiddle_table(P0, w, L)
    ctx = m.ctx_init(P0)
    tw = m.twiddle_table(ctx, w, L)
    assert np.array_equal(tw.cpu().numpy(), tw_ref)
    out = m.mul_twiddle(ctx, x, tw)
    torch.cuda.synchronize()
    idx = sample_idx(batch * L)
    hx = synth.uniform_at(42, 5, P0, idx.astype(np.uint64))
    ref = oracle.mont_mul(P0, hx, tw_ref[idx % L])
    assert np.array_equal(out.view(-1).cpu().numpy()[idx], ref)
    # x * w^j in the plain domain for a few (r, j), via Python's pow
    ho = out.cpu().numpy()
    for r, j in [(0, 0), (0, 1), (4095, 16383), (77, 8192), (1234, 4321)]:
        assert int(ho[r, j]) == (int(x[r, j].item()) * pow(w, j, P0)) % P0
    twx = tw.view(torch.int32).view(1, -1).expand(512, -1).contiguous().view(torch.uint32).view(-1)
    for r in range(0, batch, 512):
        assert identity_all(P0, x[r:r + 512].reshape(-1), twx, out[r:r + 512].reshape(-1))


def test_c4_fullsize(m):
    """configs[3]: 2^24 bases in [1,P), 31-bit exponents, P = 469762049 (bench launch)."""
    n = 1 << 24
    base = gen(n, 3, P1, 1, m=m)
    e = gen(n, 4, P1, 2, m=m)
    out = m.pow_vec(m.ctx_init(P1), base, e)
    torch.cuda.synchronize()
    idx = sample_idx(n, 50_000)
    hb = synth.uniform_at(42, 3, P1, idx.astype(np.uint64), low=1)
    he = synth.exponents_at(42, 4, idx.astype(np.uint64))
    assert np.array_equal(out.cpu().numpy()[idx], oracle.power(P1, hb, he))


@pytest.mark.parametrize("variant,ctas", [(10, 1), (10, 2), (11, 1), (11, 2)])
def test_c4_fullsize_lane_launch(m, variant, ctas):
    """configs[3] in the launches bench.py's two-lane step can time (variants 10 / 11, 8 ladders
    per thread, persistent grid of 1 or 2 CTAs per SM; the bench default is variant 10 at 1):
    sampled outputs against the oracle, and every element equal to the 4-lane kernel's
    (variant 17, a different kernel)."""
    n = 1 << 24
    ctx = m.ctx_init(P1)
    base = gen(n, 3, P1, 1, m=m)
    e = gen(n, 4, P1, 2, m=m)
    out = m.pow_vec(ctx, base, e, cfg=m.Launch(ctas_per_sm=ctas, variant=variant))
    ref = m.pow_vec(ctx, base, e, cfg=m.Launch(variant=17))
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    idx = sample_idx(n, 20_000)
    hb = synth.uniform_at(42, 3, P1, idx.astype(np.uint64), low=1)
    he = synth.exponents_at(42, 4, idx.astype(np.uint64))
    assert np.array_equal(out.cpu().numpy()[idx], oracle.power(P1, hb, he))


def test_to_from_fullsize(m):
    n = 1 << 26
    a = gen(n, 1, P0, 0, True, m=m)
    ctx = m.ctx_init(P0)
    abar = m.to_mont(ctx, a)
    back = m.from_mont(ctx, abar)
    torch.cuda.synchronize()
    assert bool((back.view(torch.int32) == a.view(torch.int32)).all())
    idx = sample_idx(n)
    assert np.array_equal(abar.cpu().numpy()[idx], oracle.to_mont(P0, a.cpu().numpy()[idx]))
    one = torch.ones(n, dtype=torch.int32, device="cuda").view(torch.uint32)
    assert identity_all(P0, abar, one, a)


@pytest.mark.parametrize("P", [P0, P1, P2])
def test_exhaustive_closed_forms(m, P):
    """All a in [0, P) against b in {0, 1, 1-bar, R^2 mod P, P-1} (SURVEY §8(c) pins), on the GPU."""
    ctx = m.ctx_init(P)
    chunk = 1 << 28
    for s in range(0, P, chunk):
        n = min(chunk, P - s)
        a = torch.arange(s, s + n, dtype=torch.int64, device="cuda").to(torch.int32).view(torch.uint32)
        full = lambda v: torch.full((n,), v, dtype=torch.int64, device="cuda").to(torch.int32).view(torch.uint32)
        eq = lambda x, y: bool((x.view(torch.int32) == y.view(torch.int32)).all())
        assert eq(m.mul_vec(ctx, a, full(ctx.r1)), a)                         # 1-bar is the identity
        assert bool((m.mul_vec(ctx, a, full(0)).view(torch.int32) == 0).all())
        assert eq(m.mul_vec(ctx, a, full(1)), m.from_mont(ctx, a))
        tm = m.to_mont(ctx, a)
        assert eq(m.mul_vec(ctx, a, full(ctx.r2)), tm)
        assert eq(m.from_mont(ctx, tm), a)                                    # round trip, every x < P
        neg = m.mul_vec(ctx, a, full(P - 1))                                  # -a R^-1
        fa = i64(m.from_mont(ctx, a))
        assert bool(((i64(neg) + fa) % P == 0).all())
        del a, tm, neg, fa
        torch.cuda.empty_cache()


def test_c5_fullsize(m):
    """configs[4] at W = 1: n = 2^31 (64-bit indexing), fused mul + checksum, P = 2013265921."""
    n = 1 << 31
    free, _ = torch.cuda.mem_get_info()
    if free < 3 * 4 * n + (4 << 30):
        pytest.skip("not enough device memory for 3 x 8 GiB")
    a = gen(n, 1, P0, m=m)
    b = gen(n, 2, P0, m=m)
    c, acc = m.mul_vec_checksum(m.ctx_init(P0), a, b)
    torch.cuda.synchronize()
    idx = sample_idx(n)
    ha, hb = synth.c5_inputs(P0, 0, 8)
    assert np.array_equal(c[:8].cpu().numpy(), oracle.mont_mul(P0, ha, hb))
    ia = torch.from_numpy(idx).cuda()
    hs_a = synth.uniform_at(42, 1, P0, idx.astype(np.uint64))
    hs_b = synth.uniform_at(42, 2, P0, idx.astype(np.uint64))
    assert np.array_equal(c.view(torch.int32)[ia].cpu().numpy().view(np.uint32), oracle.mont_mul(P0, hs_a, hs_b))
    assert identity_all(P0, a, b, c, chunk=1 << 26)
    tot = 0
    for s in range(0, n, 1 << 28):
        tot += int(i64(c[s:s + (1 << 28)]).sum().item())
    assert int(acc.item()) == tot


def test_bench_hbm_launch_shapes_fullsize(m):
    """The HBM-bound launches in the shapes bench.py times (mul_vec+checksum 256 threads x 2 uint4,
    to/from_mont 256 x 4): every element of configs[1] at P0 identical to the default launch's and
    satisfying the Montgomery identity; the to/from round trip; the checksum."""
    n = 1 << 26
    ctx = m.ctx_init(P0)
    a = gen(n, 1, P0, 0, True, m=m)
    b = gen(n, 2, P0, 0, True, m=m)
    c, acc = m.mul_vec_checksum(ctx, a, b, cfg=m.Launch(threads=256, unroll=2))
    c0, acc0 = m.mul_vec_checksum(ctx, a, b)
    torch.cuda.synchronize()
    assert torch.equal(c, c0) and int(acc.item()) == int(acc0.item())
    assert identity_all(P0, a, b, c)
    t = m.to_mont(ctx, a, cfg=m.Launch(threads=256, unroll=4))
    assert torch.equal(t, m.to_mont(ctx, a))
    back = m.from_mont(ctx, t, cfg=m.Launch(threads=256, unroll=4))
    assert torch.equal(back, a)
    idx = sample_idx(n)
    ha, hb = synth.c2_inputs_at(P0, idx.astype(np.uint64))
    assert np.array_equal(c.cpu().numpy()[idx], oracle.mont_mul(P0, ha, hb))
    assert np.array_equal(t.cpu().numpy()[idx], oracle.to_mont(P0, ha))


def test_beyond_2_32_elements(m):
    """Maximum sizes: n = 2^32 + 1029 (more elements than a 32-bit count holds, and a misaligned
    head and ragged tail at offsets past 2^32) through mont_mul_vec_checksum, to_mont / from_mont
    and mont_pow_vec: the Montgomery identity and canonical range on every element, the round
    trip on every element, the checksum against a torch reduction, and samples around index 2^32
    against the oracle / Python pow."""
    n = (1 << 32) + 1029
    free, _ = torch.cuda.mem_get_info()
    if free < 4 * 4 * n + (8 << 30):
        pytest.skip("not enough device memory for 4 x 16 GiB")
    ctx = m.ctx_init(P0)
    buf = gen(n + 1, 1, P0, m=m)
    a = buf[1:]                                   # 4-byte aligned, not 16: the head is peeled
    b = gen(n, 2, P0, m=m)
    c, acc = m.mul_vec_checksum(ctx, a, b)
    torch.cuda.synchronize()
    assert identity_all(P0, a, b, c, chunk=1 << 27)
    tot = 0
    for s in range(0, n, 1 << 28):
        tot += int(i64(c[s:s + (1 << 28)]).sum().item())
    assert int(acc.item()) == tot
    idx = np.unique(np.concatenate([np.arange(8), np.arange((1 << 32) - 8, (1 << 32) + 8), np.arange(n - 8, n),
                                    np.random.default_rng(1).integers(0, n, 2000)])).astype(np.int64)
    ia = torch.from_numpy(idx).cuda()
    ha, hb = (a.view(torch.int32)[ia].cpu().numpy().view(np.uint32), b.view(torch.int32)[ia].cpu().numpy().view(np.uint32))
    assert np.array_equal(c.view(torch.int32)[ia].cpu().numpy().view(np.uint32), oracle.mont_mul(P0, ha, hb))
    del c
    # conversions: to_mont into b's storage (b is no longer needed), then back into a fresh buffer
    tm = m.to_mont(ctx, a, out=b)
    back = m.from_mont(ctx, tm)
    for s in range(0, n, 1 << 28):
        assert bool((a[s:s + (1 << 28)].view(torch.int32) == back[s:s + (1 << 28)].view(torch.int32)).all())
    assert np.array_equal(tm.view(torch.int32)[ia].cpu().numpy().view(np.uint32), oracle.to_mont(P0, ha))
    del back, tm
    # pow: exponents from the generator, results sampled around 2^32 against Python's pow
    e = gen(n, 4, P0, mode=2, m=m)
    out = m.pow_vec(ctx, a, e, out=b)
    torch.cuda.synchronize()
    he = e.view(torch.int32)[ia].cpu().numpy().view(np.uint32)
    got = out.view(torch.int32)[ia].cpu().numpy().view(np.uint32)
    assert all(int(g) == pow(int(x), int(y), P0) for g, x, y in zip(got, ha, he))
    del a, b, e, out, buf
    torch.cuda.empty_cache()


def test_twiddle_ntt_run_beyond_2_32_elements(m):
    """Maximum sizes for the batched forms: 2^18 + 3 rows of 2^14 (4.3 G elements, row offsets
    past 2^32) through mont_mul_twiddle (the TMA-staged default), one mont_run launch and the
    default NTT rows: the Montgomery identity of every twiddle product, the inverse-NTT round trip
    of every element, and NTT outputs of the last rows against the DFT evaluated one output at a
    time."""
    batch, L = (1 << 18) + 3, 1 << 14
    n = batch * L
    free, _ = torch.cuda.mem_get_info()
    if free < 3 * 4 * n + (8 << 30):
        pytest.skip("not enough device memory for 3 x 16 GiB")
    ctx = m.ctx_init(P0)
    w = oracle.root_of_unity(P0, 31, L)
    tw = m.twiddle_table(ctx, w, L)
    x = gen(n, 5, P0, m=m).view(batch, L)
    out = m.mul_twiddle(ctx, x, tw)
    torch.cuda.synchronize()
    t64 = i64(tw)
    rows = 1 << 12
    for r in range(0, batch, rows):
        xx, oo = i64(x[r:r + rows]), i64(out[r:r + rows])
        assert bool(((oo << 32) % P0 == (xx * t64) % P0).all()) and bool((oo < P0).all()), r
    # the same product as one mont_run job (out overwritten), bit-identical
    ref_last = out[-2:].clone()
    out.zero_()
    m.run([m.run_job("twiddle", ctx, out.view(-1), x.view(-1), tw)])
    assert torch.equal(out[-2:], ref_last)
    assert bool((out[:2].view(torch.int32) != 0).any())
    del out, ref_last
    torch.cuda.empty_cache()
    # NTT rows in place, then the inverse with the 1/N scale: back to x on every element
    x0 = x.clone()
    twn = m.ntt_twiddles(ctx, w, 14)
    winv = oracle.inverse(w, P0)
    twi = m.ntt_twiddles(ctx, winv, 14)
    ninv_m = int(oracle.to_mont(P0, np.array([oracle.inverse(L, P0)], np.uint32))[0])
    m.ntt(ctx, x, twn)
    torch.cuda.synchronize()
    last = [int(v) for v in x0[-1].cpu().numpy()]
    for k in (0, 1, L - 1, 12345):
        wk, acc, pw = pow(w, k, P0), 0, 1
        for v in last:
            acc = (acc + v * pw) % P0
            pw = pw * wk % P0
        assert int(x[-1, k]) == acc, k
    m.ntt(ctx, x, twi, scale=ninv_m)
    for r in range(0, batch, rows):
        assert torch.equal(x[r:r + rows], x0[r:r + rows]), r
    del x, x0
    torch.cuda.empty_cache()
