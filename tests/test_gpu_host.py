"""Host-buffer entry points (include/mont_host.h): chunked H2D / kernel / D2H pipeline."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
P0, P1, P2 = synth.CONFIG_PRIMES


@pytest.fixture(scope="module")
def m():
    import paper_1609_00999_b200 as mod
    return mod


def host(x, pin=True):
    t = torch.from_numpy(np.ascontiguousarray(x))
    return t.pin_memory() if pin else t


def empty(n, pin=True):
    return torch.empty(n, dtype=torch.uint32, pin_memory=pin)


@pytest.mark.parametrize("n", [1, 5, 4097, 1 << 20, (1 << 22) + 3])
@pytest.mark.parametrize("ws_mb", [1, 64])
@pytest.mark.parametrize("pin", [True, False])
def test_mul_vec_host(m, n, ws_mb, pin):
    P = P2
    a, b = synth.c2_inputs(P, 0, n)
    ref = oracle.mont_mul(P, a, b)
    ws = m.host_workspace("mul_vec", min_bytes=ws_mb << 20)
    out = empty(n, pin)
    acc = m.mul_vec_host(m.ctx_init(P), host(a, pin), host(b, pin), out, ws, want_checksum=True)
    torch.cuda.synchronize()
    assert np.array_equal(out.numpy(), ref)
    assert int(acc.item()) == oracle.raw_sum(ref)


@pytest.mark.parametrize("n", [3, 1 << 20, (1 << 21) + 1])
def test_to_from_pow_host(m, n):
    ctx = m.ctx_init(P1)
    ws = m.host_workspace("pow_vec", min_bytes=4 << 20)
    x = synth.uniform(42, 9, P1, 0, n)
    o = empty(n)
    m.to_mont_host(ctx, host(x), o, ws)
    torch.cuda.synchronize()
    assert np.array_equal(o.numpy(), oracle.to_mont(P1, x))
    o2 = empty(n)
    m.from_mont_host(ctx, o, o2, ws)
    torch.cuda.synchronize()
    assert np.array_equal(o2.numpy(), x)
    base, e = synth.c4_inputs(P1, 0, n)
    o3 = empty(n)
    m.pow_vec_host(ctx, host(base), host(e), o3, ws)
    torch.cuda.synchronize()
    assert np.array_equal(o3.numpy(), oracle.power(P1, base, e))


@pytest.mark.parametrize("batch,L,ws_mb", [(7, 1024, 1), (300, 4096, 8), (64, 16384, 64), (5, 1000, 1)])
def test_twiddle_host(m, batch, L, ws_mb):
    x = synth.c3_x(P0, batch=batch, length=L)
    tw = synth.uniform(42, 11, P0, 0, L)
    ws = m.host_workspace("twiddle", L, min_bytes=ws_mb << 20)
    out = torch.empty((batch, L), dtype=torch.uint32, pin_memory=True)
    m.mul_twiddle_host(m.ctx_init(P0), host(x), host(tw), out, ws)
    torch.cuda.synchronize()
    assert np.array_equal(out.numpy(), oracle.twiddle(P0, x, tw))


def test_concurrent_streams(m):
    """Two host-buffer calls on two streams with separate workspaces."""
    n = 1 << 21
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs, refs = [], []
    for P, s in ((P0, s1), (P2, s2)):
        a, b = synth.c2_inputs(P, 0, n)
        refs.append(oracle.mont_mul(P, a, b))
        o = empty(n)
        m.mul_vec_host(m.ctx_init(P), host(a), host(b), o, m.host_workspace("mul_vec", min_bytes=8 << 20), stream=s)
        outs.append(o)
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        assert np.array_equal(o.numpy(), r)


def test_host_validation(m):
    L = m.lib()
    ctx = m.ctx_init(P0)
    import ctypes as C
    assert L.mont_mul_vec_host(C.byref(ctx), None, None, None, 0, None, None, 0, None) == 0
    assert L.mont_mul_vec_host(C.byref(ctx), None, None, None, 5, None, None, 0, None) == 2
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    a = empty(10)
    assert L.mont_mul_vec_host(C.byref(ctx), a.data_ptr(), a.data_ptr(), a.data_ptr(), 10, None, ws.data_ptr(),
                               16, None) == 2   # workspace too small
    assert m.lib().mont_host_min_workspace(4, 16384) > 6 * 65536


def test_host_run_many_jobs(m):
    """One ring over mul_vec (x2, one with checksum), to_mont -> from_mont (chained), pow, twiddle."""
    P, P1_ = 2013265921, 469762049
    ctx, ctx1 = m.ctx_init(P), m.ctx_init(P1_)
    n = (1 << 20) + 3
    a, b = synth.c2_inputs(P, 0, n)
    a2, b2 = synth.c2_inputs(P1_, 5, 777)
    base, e = synth.c4_inputs(P1_, 0, 4099)
    L = 4096
    x = synth.c3_x(P, batch=33, length=L)
    tw = synth.uniform(42, 11, P, 0, L)
    ha, hb, ha2, hb2, hbase, he, hx, htw = (host(v) for v in (a, b, a2, b2, base, e, x, tw))
    o1, o2, o3, o4, o5 = empty(n), empty(777), empty(n), empty(n), empty(4099)
    o6 = torch.empty((33, L), dtype=torch.uint32, pin_memory=True)
    o7 = empty(n)
    acc = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    jobs = [m.host_job("mul_vec", ctx, o1, ha, hb, acc=acc),
            m.host_job("mul_vec", ctx1, o2, ha2, hb2),
            m.host_job("to_mont", ctx, o3, ha),
            m.host_job("from_mont", ctx, o4, o3, depends_on=2),
            m.host_job("pow_vec", ctx1, o5, hbase, he),
            m.host_job("twiddle", ctx, o6, hx, htw),
            m.host_job("from_mont", ctx, o7, o3, depends_on=2)]
    for ws_mb in (1, 3, 64):
        for o in (o1, o2, o3, o4, o5, o6, o7):
            o.zero_()
        acc.zero_()
        m.host_run(jobs, m.host_workspace("twiddle", L, min_bytes=ws_mb << 20))
        torch.cuda.synchronize()
        ref1 = oracle.mont_mul(P, a, b)
        assert np.array_equal(o1.numpy(), ref1) and int(acc.item()) == oracle.raw_sum(ref1)
        assert np.array_equal(o2.numpy(), oracle.mont_mul(P1_, a2, b2))
        assert np.array_equal(o3.numpy(), oracle.to_mont(P, a))
        assert np.array_equal(o4.numpy(), a)
        assert np.array_equal(o5.numpy(), oracle.power(P1_, base, e))
        assert np.array_equal(o6.numpy(), oracle.twiddle(P, x, tw))
        assert np.array_equal(o7.numpy(), a)

def test_host_run_fused_group(m):
    """Jobs over the same n that share host buffers form one fusion group: a shared input is
    uploaded once per chunk and an output consumed by a later job is read from the device; every
    output still lands in host memory.  Also an in-place host job, which must not join."""
    P = 2013265921
    ctx = m.ctx_init(P)
    n = (1 << 20) + 5
    a, b = synth.c2_inputs(P, 0, n)
    ha, hb = host(a), host(b)
    o1, o3, o4, o8, o9 = empty(n), empty(n), empty(n), empty(n), empty(n)
    acc = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    hip = host(b)  # in-place target
    jobs = [m.host_job("mul_vec", ctx, o1, ha, hb, acc=acc),
            m.host_job("to_mont", ctx, o3, ha),
            m.host_job("from_mont", ctx, o4, o3),
            m.host_job("mul_vec", ctx, o8, o4, hb),
            m.host_job("to_mont", ctx, hip, hip),
            m.host_job("mul_vec", ctx, o9, ha, ha)]       # both operands one host buffer
    ref1 = oracle.mont_mul(P, a, b)
    for ws_mb in (1, 7, 64):
        for o in (o1, o3, o4, o8, o9):
            o.zero_()
        hip.copy_(torch.from_numpy(b))
        acc.zero_()
        m.host_run(jobs, m.host_workspace("mul_vec", 0, min_bytes=ws_mb << 20))
        torch.cuda.synchronize()
        assert np.array_equal(o1.numpy(), ref1) and int(acc.item()) == oracle.raw_sum(ref1)
        assert np.array_equal(o3.numpy(), oracle.to_mont(P, a))
        assert np.array_equal(o4.numpy(), a)
        assert np.array_equal(o8.numpy(), ref1)
        assert np.array_equal(hip.numpy(), oracle.to_mont(P, b))
        assert np.array_equal(o9.numpy(), oracle.mont_mul(P, a, a))


def test_host_run_interleaving_keeps_host_buffer_order(m):
    """Independent groups are interleaved chunk by chunk, but a group that overwrites a host
    buffer an earlier group reads (write after read) still sees job order; so does one that
    rewrites an earlier group's output (write after write)."""
    P = 2013265921
    ctx = m.ctx_init(P)
    n1, n2 = (1 << 20) + 7, (1 << 19) + 3
    a = synth.uniform(42, 31, P, 0, n1)
    c = synth.uniform(42, 32, P, 0, n2)
    x, y = synth.c2_inputs(P, 3, n2)
    hA, hC, hx, hy = host(a), host(c), host(x), host(y)
    hB, hD, hE = empty(n1), empty(n2), empty(n2)
    hA2 = hA[:n2]                                               # a view: the first n2 words of A
    jobs = [m.host_job("to_mont", ctx, hB, hA),                 # reads A
            m.host_job("mul_vec", ctx, hD, hx, hy),             # independent: may interleave
            m.host_job("from_mont", ctx, hA2, hC),              # then overwrites A's first n2 words
            m.host_job("mul_vec", ctx, hE, hC, hC),             # independent
            m.host_job("to_mont", ctx, hD, hy)]                 # rewrites D (after the mul_vec above)
    for ws_mb in (1, 5, 64):
        hA.copy_(torch.from_numpy(a))
        m.host_run(jobs, m.host_workspace("mul_vec", 0, min_bytes=ws_mb << 20))
        torch.cuda.synchronize()
        assert np.array_equal(hB.numpy(), oracle.to_mont(P, a))
        assert np.array_equal(hA.numpy()[:n2], oracle.from_mont(P, c))
        assert np.array_equal(hA.numpy()[n2:], a[n2:])
        assert np.array_equal(hE.numpy(), oracle.mont_mul(P, c, c))
        assert np.array_equal(hD.numpy(), oracle.to_mont(P, y))


def test_host_run_job_limit(m):
    """64 jobs in one run (the executor's limit), a mix of ops and sizes; 65 are refused."""
    P = 998244353
    ctx = m.ctx_init(P)
    rng = np.random.default_rng(7)
    jobs, refs, outs = [], [], []
    for j in range(64):
        n = int(rng.integers(1, 5000))
        a, b = synth.c2_inputs(P, 1000 * j, n)
        ha, hb, ho = host(a), host(b), empty(n)
        kind = j % 3
        if kind == 0:
            jobs.append(m.host_job("mul_vec", ctx, ho, ha, hb))
            refs.append(oracle.mont_mul(P, a, b))
        elif kind == 1:
            jobs.append(m.host_job("to_mont", ctx, ho, ha))
            refs.append(oracle.to_mont(P, a))
        else:
            jobs.append(m.host_job("from_mont", ctx, ho, ha))
            refs.append(oracle.from_mont(P, a))
        outs.append(ho)
    ws = m.host_workspace("mul_vec", 0, min_bytes=4 << 20)
    m.host_run(jobs, ws)
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        assert np.array_equal(o.numpy(), r)
    with pytest.raises(m.MontError):
        m.host_run(jobs + jobs[:1], ws)


@pytest.mark.parametrize("log_n", [1, 5, 10, 14])
def test_host_run_ntt(m, log_n):
    """NTT jobs from host buffers (rows streamed through the ring, transformed in place in the
    slot): forward vs the oracle's definition DFT, inverse round trip through a second job, and
    interleaved with an elementwise job."""
    P = 2013265921
    N = 1 << log_n
    batch = 37 if log_n < 14 else 3
    ctx = m.ctx_init(P)
    w = oracle.root_of_unity(P, 31, N)
    winv = oracle.inverse(w, P)
    tw = m.ntt_twiddles(ctx, w, log_n).cpu()
    twi = m.ntt_twiddles(ctx, winv, log_n).cpu()
    ninv_m = int(oracle.to_mont(P, np.array([oracle.inverse(N, P)], np.uint32))[0])
    x = synth.uniform(42, 51, P, 0, batch * N).reshape(batch, N)
    hx = host(x)
    hX = torch.empty((batch, N), dtype=torch.uint32, pin_memory=True)
    hback = torch.empty((batch, N), dtype=torch.uint32, pin_memory=True)
    a, b = synth.c2_inputs(P, 9, 3001)
    ha, hb, hc = host(a), host(b), empty(3001)
    jobs = [m.host_job("ntt", ctx, hX, hx, tw),
            m.host_job("mul_vec", ctx, hc, ha, hb),
            m.host_job("ntt", ctx, hback, hX, twi, depends_on=0, scale=ninv_m)]
    for ws_mb in (1, 64):
        m.host_run(jobs, m.host_workspace("ntt", N, min_bytes=ws_mb << 20))
        torch.cuda.synchronize()
        if log_n <= 10:
            assert np.array_equal(hX.numpy(), oracle.dft(P, w, x))
        else:
            for k in (0, 1, N - 1, 12345 % N):
                assert int(hX.numpy()[1, k]) == oracle.dft_at(P, w, x[1], k)
        assert np.array_equal(hback.numpy(), x)
        assert np.array_equal(hc.numpy(), oracle.mont_mul(P, a, b))
