"""GPU NTT (include/mont_ntt.h) vs the oracle's definition-DFT, inverse and convolution."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
# 1073479681 = 4095 * 2^18 + 1 sits just under 2^30, the tight end of the lazy [0, 2P) butterflies'
# bound 4P < 2^32 (smallest primitive root 11); rows up to 2^15 and six-step transforms up to 2^18
GEN = {2013265921: 31, 469762049: 3, 998244353: 3, 1073479681: 11}


@pytest.fixture(scope="module")
def m():
    import paper_1609_00999_b200 as mod
    return mod


def tables(m, P, N):
    ctx = m.ctx_init(P)
    w = oracle.root_of_unity(P, GEN[P], N)
    winv = oracle.inverse(w, P)
    log_n = N.bit_length() - 1
    tw = m.ntt_twiddles(ctx, w, log_n)
    twi = m.ntt_twiddles(ctx, winv, log_n)
    ninv_m = int(oracle.to_mont(P, np.array([oracle.inverse(N, P)], np.uint32))[0])
    return ctx, w, winv, tw, twi, ninv_m


def pq_tables(m, ctx, w, winv, log_n):
    return m.ntt_twiddles_pq(ctx, w, log_n), m.ntt_twiddles_pq(ctx, winv, log_n)


@pytest.mark.parametrize("P", list(GEN))
@pytest.mark.parametrize("log_n", [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12])
@pytest.mark.parametrize("variant", [None, 1, 2, 3, 4, 5, 6, 7])
def test_ntt_vs_dft(m, P, log_n, variant):
    N = 1 << log_n
    batch = 3
    ctx, w, winv, tw, twi, ninv_m = tables(m, P, N)
    if variant in (3, 4, 5, 6, 7) and log_n < 5:
        pytest.skip("variants 3-7 need log_n >= 5")
    if variant in (3, 5, 7):
        tw, twi = pq_tables(m, ctx, w, winv, log_n)
    x = synth.uniform(42, 21, P, 0, batch * N).reshape(batch, N)
    x[0, :2] = [0, P - 1]
    d = torch.from_numpy(x).cuda()
    m.ntt(ctx, d, tw, variant=variant)
    X = d.cpu().numpy()
    assert np.array_equal(X, oracle.dft(P, w, x))
    m.ntt(ctx, d, twi, scale=ninv_m, variant=variant)
    assert np.array_equal(d.cpu().numpy(), x)


@pytest.mark.parametrize("P", list(GEN))
@pytest.mark.parametrize("log_n", [13, 14, 15])
def test_ntt_full_rows_vs_dft(m, P, log_n):
    """The 2^13..2^15 row kernels (their own instantiations, incl. the 2^14 rows the bench times) on
    4 full rows per size and prime against the oracle's O(N^2) definition-DFT, in the default
    (REDC twiddles) and the precomputed-quotient (variant 3) forms, plus the inverse round trip."""
    N = 1 << log_n
    rows = 4
    ctx, w, winv, tw, twi, ninv_m = tables(m, P, N)
    x = synth.uniform(42, 23, P, 0, rows * N).reshape(rows, N)
    x[0, :3] = [P - 1, 0, P - 1]
    x[1, -2:] = [P - 1, P - 1]
    ref = oracle.dft(P, w, x)
    pq = pq_tables(m, ctx, w, winv, log_n)
    for variant, (t, ti) in ((None, (tw, twi)), (3, pq), (6, (tw, twi)), (7, pq)):
        d = torch.from_numpy(x).cuda()
        m.ntt(ctx, d, t, variant=variant)
        assert np.array_equal(d.cpu().numpy(), ref), variant
        m.ntt(ctx, d, ti, scale=ninv_m, variant=variant)
        assert np.array_equal(d.cpu().numpy(), x), variant


@pytest.mark.parametrize("P", list(GEN))
@pytest.mark.parametrize("log_n", [5, 8, 10, 12, 13, 14, 15])
def test_ntt_persistent_rounds(m, P, log_n):
    """Variants 6 / 7 (persistent grid, next row group's loads issued before this group's stores) on a
    batch that takes every CTA through several row groups with a ragged last round: bit-exact
    against variants 0 / 3 (pinned to the definition-DFT above), sampled outputs of the last rows
    against the DFT evaluated one output at a time, and the inverse round trip."""
    N = 1 << log_n
    rows_per_cta = max(1, 256 // (N // 32))
    batch = (2 * 148 * 2 * 2 + 37) * rows_per_cta + 3 if log_n < 15 else 148 * 3 + 5
    ctx, w, winv, tw, twi, ninv_m = tables(m, P, N)
    pq, pqi = pq_tables(m, ctx, w, winv, log_n)
    x = torch.empty(batch * N, dtype=torch.uint32, device="cuda")
    m.synth_fill(x, 42, 24 + log_n, 0, P)
    x = x.view(batch, N)
    for ref_v, v, t, ti in ((None, 6, tw, twi), (3, 7, pq, pqi)):
        ref = x.clone()
        m.ntt(ctx, ref, t, variant=ref_v)
        d = x.clone()
        m.ntt(ctx, d, t, variant=v)
        assert torch.equal(d, ref), v
        last = [int(u) for u in x[-1].cpu().numpy()]
        for k in (0, 1, N - 1):
            wk, acc, pw = pow(w, k, P), 0, 1
            for u in last:
                acc = (acc + u * pw) % P
                pw = pw * wk % P
            assert int(d[-1, k]) == acc, (v, k)
        m.ntt(ctx, d, ti, scale=ninv_m, variant=v)
        assert torch.equal(d, x), v


def test_ntt_non_lazy_path(tmp_path):
    """MONT_NTT_NO_LAZY=1 (read once per process) forces the canonical butterflies for P < 2^30:
    run in a subprocess, rows and a large transform against the oracle."""
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    code = """
import numpy as np, torch, sys
sys.path.insert(0, %r)
import oracle, synth, paper_1609_00999_b200 as m
ok = True
for P, g in ((998244353, 3), (1073479681, 11), (469762049, 3)):
    ctx = m.ctx_init(P)
    for log_n in (5, 12, 14):
        N = 1 << log_n
        w = oracle.root_of_unity(P, g, N)
        x = synth.uniform(42, 24, P, 0, 3 * N).reshape(3, N)
        d = torch.from_numpy(x).cuda()
        m.ntt(ctx, d, m.ntt_twiddles(ctx, w, log_n))
        ok &= np.array_equal(d.cpu().numpy(), oracle.dft(P, w, x))
    N = 1 << 16
    w = oracle.root_of_unity(P, g, N)
    x = synth.uniform(42, 25, P, 0, N)
    X = m.ntt_large(ctx, torch.from_numpy(x).cuda(), m.ntt_plan(ctx, w, 16)).cpu().numpy()
    ok &= all(int(X[k]) == oracle.dft_at(P, w, x, k) for k in (0, 1, 777, N - 1))
sys.exit(0 if ok else 1)
""" % str(root)
    env = dict(__import__("os").environ, MONT_NTT_NO_LAZY="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("log_n", [13, 14, 15])
@pytest.mark.parametrize("variant", [None, 1, 3, 4, 5, 6, 7])
def test_ntt_large_properties(m, log_n, variant):
    P = 998244353
    N = 1 << log_n
    ctx, w, winv, tw, twi, ninv_m = tables(m, P, N)
    if variant in (3, 5, 7):
        tw, twi = pq_tables(m, ctx, w, winv, log_n)
    x = synth.uniform(42, 22, P, 0, 2 * N).reshape(2, N)
    d = torch.from_numpy(x).cuda()
    m.ntt(ctx, d, tw, variant=variant)
    X = d.cpu().numpy()
    xs = [int(v) for v in x[1]]
    for k in (0, 1, 2, N // 2, N - 1, 12345 % N):
        wk = pow(w, k, P)
        acc, pw = 0, 1
        for v in xs:
            acc = (acc + v * pw) % P
            pw = pw * wk % P
        assert int(X[1, k]) == acc
    m.ntt(ctx, d, twi, scale=ninv_m, variant=variant)
    assert np.array_equal(d.cpu().numpy(), x)


@pytest.mark.parametrize("log_n", [4, 9, 12])
def test_ntt_convolution(m, log_n):
    P = 2013265921
    N = 1 << log_n
    ctx, w, winv, tw, twi, ninv_m = tables(m, P, N)
    a = synth.uniform(42, 23, P, 0, N)
    b = synth.uniform(42, 24, P, 0, N)
    da, db = torch.from_numpy(a.reshape(1, N)).cuda(), torch.from_numpy(b.reshape(1, N)).cuda()
    m.ntt(ctx, da, tw)
    m.ntt(ctx, db, tw)
    # pointwise product of the transforms: REDC(A, to_mont(B)) = A B mod P, via the library
    prod = m.mul_vec(ctx, da.view(-1), m.to_mont(ctx, db.view(-1))).view(1, N)
    m.ntt(ctx, prod, twi, scale=ninv_m)
    assert np.array_equal(prod.cpu().numpy().reshape(-1), oracle.cyclic_conv(P, a, b))


def test_ntt_many_rows_and_validation(m):
    P = 469762049
    N = 1 << 10
    ctx, w, winv, tw, twi, ninv_m = tables(m, P, N)
    x = synth.uniform(42, 25, P, 0, 300 * N).reshape(300, N)
    d = torch.from_numpy(x).cuda()
    m.ntt(ctx, d, tw)
    X = d.cpu().numpy()
    for r in (0, 1, 150, 299):
        assert np.array_equal(X[r], oracle.dft(P, w, x[r]))
    import ctypes as C
    L = m.lib()
    assert L.mont_ntt(C.byref(ctx), d.data_ptr(), 1, 16, tw.data_ptr(), ctx.r1, None) == 4
    assert L.mont_ntt(C.byref(ctx), d.data_ptr(), 1, 0, tw.data_ptr(), ctx.r1, None) == 4
    assert L.mont_ntt(C.byref(ctx), d.data_ptr(), 0, 10, tw.data_ptr(), ctx.r1, None) == 0
    assert L.mont_ntt(C.byref(ctx), d.data_ptr(), 1, 10, tw.data_ptr(), P, None) == 2


@pytest.mark.parametrize("log_n", [1, 2, 5, 11, 16])
def test_ntt_twiddle_table_layout(m, log_n):
    """tw[2^(s-1) - 1 + pos] = to_mont(w^(pos N / 2^s)), checked against Python's pow."""
    P = 2013265921
    N = 1 << log_n
    ctx = m.ctx_init(P)
    w = oracle.root_of_unity(P, 31, N)
    tw = m.ntt_twiddles(ctx, w, log_n).cpu().numpy()
    assert tw.size == N - 1
    rng = np.random.default_rng(log_n)
    for e in set([0, N - 2] + [int(v) for v in rng.integers(0, N - 1, 200)]):
        s1 = int(e + 1).bit_length() - 1
        pos = e + 1 - (1 << s1)
        expo = pos * (N >> (s1 + 1))
        assert int(tw[e]) == (pow(w, expo, P) << 32) % P


@pytest.mark.parametrize("P", list(GEN))
@pytest.mark.parametrize("log_n", [16, 17, 20, 22, 23, 24, 26, 27])
def test_ntt_large(m, P, log_n):
    """Large transform (six-step for 2^16..2^21, 3-pass column/row/transpose for 2^22..2^27): sampled
    outputs by definition (oracle.dft_at), inverse round trip."""
    if (P - 1) % (1 << log_n):
        pytest.skip("no primitive 2^log_n-th root of unity mod P")
    N = 1 << log_n
    ctx = m.ctx_init(P)
    w = oracle.root_of_unity(P, GEN[P], N)
    winv = oracle.inverse(w, P)
    plan = m.ntt_plan(ctx, w, log_n)
    plan_inv = m.ntt_plan(ctx, winv, log_n)
    x = synth.uniform(42, 41, P, 0, N)
    x[:2] = [P - 1, 0]
    X = m.ntt_large(ctx, torch.from_numpy(x).cuda(), plan)
    Xh = X.cpu().numpy()
    rng = np.random.default_rng(log_n)
    for k in [0, 1, 2, N // 2, N - 1] + [int(v) for v in rng.integers(0, N, 6)]:
        assert int(Xh[k]) == oracle.dft_at(P, w, x, k), k
    ninv_m = int(oracle.to_mont(P, np.array([oracle.inverse(N % P, P)], np.uint32))[0])
    back = m.ntt_large(ctx, X, plan_inv, scale=ninv_m)
    assert np.array_equal(back.cpu().numpy(), x)


def test_ntt_large_matches_small_path(m):
    """2^16 six-step vs a single small-path row of the same length is impossible (small path <= 2^15),
    so check linearity and the delta: NTT(e0) = ones, NTT(e1) = powers of w."""
    P, log_n = 2013265921, 16
    N = 1 << log_n
    ctx = m.ctx_init(P)
    w = oracle.root_of_unity(P, 31, N)
    plan = m.ntt_plan(ctx, w, log_n)
    e = np.zeros(N, np.uint32)
    e[0] = 1
    assert np.all(m.ntt_large(ctx, torch.from_numpy(e.copy()).cuda(), plan).cpu().numpy() == 1)
    e[0], e[1] = 0, 1
    X = m.ntt_large(ctx, torch.from_numpy(e.copy()).cuda(), plan).cpu().numpy()
    for k in (0, 1, 2, 12345, N - 1):
        assert int(X[k]) == pow(w, k, P)


@pytest.mark.parametrize("P", list(GEN))
@pytest.mark.parametrize("log_n", [1, 5, 12])
def test_ntt_twiddles_pq_layout(m, P, log_n):
    """Pair table: entry e = (w^x, floor(w^x 2^32 / P)) with x the stage-major exponent, checked
    with Python big integers (pow, //), independent of the library's Montgomery derivation."""
    N = 1 << log_n
    ctx = m.ctx_init(P)
    w = oracle.root_of_unity(P, GEN[P], N)
    tw2 = m.ntt_twiddles_pq(ctx, w, log_n).cpu().numpy().reshape(-1, 2)
    for s_ in range(1, log_n + 1):
        h = 1 << (s_ - 1)
        for pos in range(h):
            x = pow(w, pos * (N // (2 * h)), P)
            assert int(tw2[h - 1 + pos, 0]) == x
            assert int(tw2[h - 1 + pos, 1]) == (x << 32) // P


def test_ntt_pq_rejects(m):
    P = 2013265921
    ctx, w, winv, tw, twi, ninv_m = tables(m, P, 64)
    tw2 = m.ntt_twiddles_pq(ctx, w, 6)
    d = torch.zeros((2, 64), dtype=torch.uint32, device="cuda")
    with pytest.raises(m.MontError):
        m.ntt(ctx, d, tw2[1:], variant=3)   # 4-byte aligned only
    d4 = torch.zeros((2, 16), dtype=torch.uint32, device="cuda")
    with pytest.raises(m.MontError):
        m.ntt(ctx, d4, m.ntt_twiddles_pq(ctx, pow(w, 4, P), 4), variant=3)  # log_n < 5
