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
