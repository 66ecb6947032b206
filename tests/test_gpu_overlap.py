"""MONT_LAUNCH_OVERLAP_PREV (include/mont_ext.h): a flagged launch may start while the previous
kernel on the stream still runs; the results must be those of the plain launches, and work
launched after a flagged operation must still see everything before it (the flagged kernel waits
for its predecessor before it completes)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

P0, P1, _ = synth.CONFIG_PRIMES


@pytest.fixture(scope="module")
def m():
    import paper_1609_00999_b200 as mod
    return mod


def gen(m, n, sid, P, mode=0):
    t = torch.empty(n, dtype=torch.uint32, device="cuda")
    m.synth_fill(t, 42, sid, 0, P, mode, False)
    return t


def u32(t):
    return t.view(torch.int32).cpu().numpy().view(np.uint32)


def sequence(m, ctx, bufs, flagged, stream):
    """to_mont(x -> y); mul_vec+checksum; twiddle; one mont_run job; from_mont(y -> z): the middle
    three independent of the first, the last dependent on the first."""
    x, y, z, a, b, c, acc, xt, tw, ot, ra, rb, rc = bufs
    ov = m.Launch(flags=m.OVERLAP_PREV) if flagged else None
    acc.zero_()
    m.to_mont(ctx, x, out=y, stream=stream)
    m.mul_vec_checksum(ctx, a, b, out=c, acc=acc, stream=stream, cfg=m.Launch(threads=256, unroll=2, flags=m.OVERLAP_PREV) if flagged else None)
    m.mul_twiddle(ctx, xt, tw, out=ot, stream=stream, cfg=ov)
    m.run([m.run_job("mul_vec", ctx, rc, ra, rb)], stream=stream, cfg=ov)
    m.from_mont(ctx, y, out=z, stream=stream)


def make_bufs(m, ctx, n, rows, L):
    x, a, b = gen(m, n, 1, P0), gen(m, n, 2, P0), gen(m, n, 3, P0)
    y, z, c = (torch.empty_like(x) for _ in range(3))
    acc = torch.zeros(1, dtype=torch.int64, device="cuda")
    xt = gen(m, rows * L, 5, P0).view(rows, L)
    tw = m.twiddle_table(ctx, oracle.root_of_unity(P0, 31, L), L)
    ot = torch.empty_like(xt)
    ra, rb = gen(m, n, 6, P0), gen(m, n, 7, P0)
    rc = torch.empty_like(ra)
    return (x, y, z, a, b, c, acc, xt, tw, ot, ra, rb, rc)


@pytest.mark.parametrize("graph", [False, True])
def test_overlap_flag_same_results(m, graph):
    ctx = m.ctx_init(P0)
    n, rows, L = (1 << 24) + 12, 1024, 1 << 14
    ref = make_bufs(m, ctx, n, rows, L)
    got = tuple(t.clone() for t in ref)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())   # inputs were generated on the current stream
    with torch.cuda.stream(s):
        sequence(m, ctx, ref, False, s)
        if graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                sequence(m, ctx, got, True, s)
            for _ in range(3):
                g.replay()
        else:
            for _ in range(3):
                sequence(m, ctx, got, True, s)
    torch.cuda.synchronize()
    for i in (1, 2, 5, 6, 9, 12):  # y, z, c, acc, ot, rc
        assert torch.equal(ref[i], got[i]), i
    assert torch.equal(got[2], got[0])  # the round trip through to_mont / from_mont
    idx = np.arange(0, n, 9973)
    assert np.array_equal(u32(got[5])[idx], oracle.mont_mul(P0, u32(got[3])[idx], u32(got[4])[idx]))


def test_overlap_flag_keeps_stream_order(m):
    """A long pow writes `out`; a short flagged mul_vec follows; a plain kernel then reads `out`.
    The flagged kernel may start early, but it completes only after the pow, so the reader sees
    the finished pow results, every time."""
    ctx = m.ctx_init(P1)
    n = 1 << 24
    base, e = gen(m, n, 3, P1, 1), gen(m, n, 4, P1, 2)
    out = torch.empty_like(base)
    a, b = gen(m, 1 << 16, 1, P1), gen(m, 1 << 16, 2, P1)
    c = torch.empty_like(a)
    ref = m.pow_vec(ctx, base, e)
    ref_m = m.to_mont(ctx, ref)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())   # inputs were generated on the current stream
    for _ in range(20):
        with torch.cuda.stream(s):
            out.zero_()                           # on s, ordered before the pow
            m.pow_vec(ctx, base, e, out=out, stream=s)
            m.mul_vec(ctx, a, b, out=c, stream=s, cfg=m.Launch(flags=m.OVERLAP_PREV))
            got = m.to_mont(ctx, out, stream=s)
        s.synchronize()
        assert torch.equal(got, ref_m)


def test_overlap_flag_without_a_predecessor(m):
    """A flagged launch that is the first work on a fresh stream (and the first node of a captured
    graph) behaves as a plain launch."""
    ctx = m.ctx_init(P0)
    n = (1 << 20) + 4
    a, b = gen(m, n, 1, P0), gen(m, n, 2, P0)
    ref = m.mul_vec(ctx, a, b)
    torch.cuda.synchronize()
    ov = m.Launch(flags=m.OVERLAP_PREV)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        c = torch.empty_like(a)
        m.mul_vec(ctx, a, b, out=c, stream=s, cfg=ov)
    s.synchronize()
    assert torch.equal(c, ref)
    g = torch.cuda.CUDAGraph()
    c2 = torch.empty_like(a)
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        with torch.cuda.graph(g, stream=s2):
            m.mul_vec(ctx, a, b, out=c2, stream=s2, cfg=ov)
            m.mul_twiddle(ctx, a[:4096 * 256].view(256, 4096), b[:4096], out=c[:4096 * 256].view(256, 4096),
                          stream=s2, cfg=ov)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(c2, ref)
    t = m.mul_twiddle(ctx, a[:4096 * 256].view(256, 4096), b[:4096])
    assert torch.equal(c[:4096 * 256].view(256, 4096), t)
