"""Batched lazy-reduction dot products (include/mont_dot.h, NEXT #4) vs the oracle."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    import paper_1609_00999_b200 as mod
    return mod


@pytest.mark.parametrize("P", list(synth.CONFIG_PRIMES) + [3, 17, 2147483647])
@pytest.mark.parametrize("batch,L", [(1, 1), (3, 7), (5, 1024), (17, 4100), (2, 65536 + 4), (64, 16384)])
def test_dot(m, P, batch, L):
    A = synth.uniform(42, 31, P, 0, batch * L).reshape(batch, L)
    x = synth.uniform(42, 32, P, 0, L)
    A[0, 0] = P - 1
    x[0] = P - 1
    out = m.dot(m.ctx_init(P), torch.from_numpy(A).cuda(), torch.from_numpy(x).cuda())
    assert np.array_equal(out.cpu().numpy(), oracle.dot(P, A, x))


def test_dot_misaligned_and_extremes(m):
    P = 2013265921
    L = 1001
    A = np.full((4, L), P - 1, np.uint32)
    x = np.full(L, P - 1, np.uint32)
    buf = torch.empty(4 * L + 1, dtype=torch.uint32, device="cuda")
    tA = buf[1:].view(4, L)
    tA.copy_(torch.from_numpy(A).cuda())
    out = m.dot(m.ctx_init(P), tA, torch.from_numpy(x).cuda())
    assert np.array_equal(out.cpu().numpy(), oracle.dot(P, A, x))


@pytest.mark.parametrize("P", [2013265921, 469762049, 3, 2147483647])
@pytest.mark.parametrize("cfg", [None, (1, 0), (2, 0), (3, 0), (4, 0), (5, 1024), (5, 2048), (5, 0), (5, 8192), (6, 0), (7, 0),
                                 (8, 0), (8, 1024), (8, 8192)])
@pytest.mark.parametrize("batch,L", [(3, 8192), (5, 16384), (2, 16384 + 1028), (7, 40000), (1, 1 << 20)])
def test_dot_split_rows(m, P, cfg, batch, L):
    """The split-row path (chunks per CTA, canonical partials added into out by modular CAS) and
    the one-CTA-per-row path against the oracle, incl. a ragged last chunk and a stale out."""
    A = synth.uniform(42, 33, P, 0, batch * L).reshape(batch, L)
    x = synth.uniform(42, 34, P, 0, L)
    A[:, -1] = P - 1
    x[-1] = P - 1
    launch = None if cfg is None else m.Launch(variant=cfg[0], chunk=cfg[1])
    out = torch.full((batch,), 12345, dtype=torch.int32, device="cuda").view(torch.uint32)  # stale
    m.dot(m.ctx_init(P), torch.from_numpy(A).cuda(), torch.from_numpy(x).cuda(), out=out, cfg=launch)
    assert np.array_equal(out.cpu().numpy(), oracle.dot(P, A, x))


def test_dot_ex_rejects(m):
    ctx = m.ctx_init(2013265921)
    A = torch.zeros((2, 8192), dtype=torch.int32, device="cuda").view(torch.uint32)
    x = torch.zeros(8192, dtype=torch.int32, device="cuda").view(torch.uint32)
    for cfg in (m.Launch(variant=9), m.Launch(chunk=1000), m.Launch(variant=8, unroll=3),
                m.Launch(variant=8, ctas_per_sm=9), m.Launch(variant=8, chunk=1 << 20)):
        with pytest.raises(m.MontError):
            m.dot(ctx, A, x, cfg=cfg)


@pytest.mark.parametrize("P", [2013265921, 998244353])
@pytest.mark.parametrize("stages,ctas,chunk", [(4, 2, 0), (2, 1, 1024), (8, 1, 2048), (8, 4, 2048), (4, 8, 1024), (2, 3, 4096)])
@pytest.mark.parametrize("batch,L", [(700, 4096), (301, 16384 + 1028), (1500, 12)])
def test_dot_pipe_many_rows(m, P, stages, ctas, chunk, batch, L):
    """Variant 8 (persistent CTAs streaming their rows through a bulk-copy ring): batches larger
    than the grid, so every CTA runs several rows (and its ring wraps many times), ragged last
    tiles, rows shorter than one tile; against the oracle's definition."""
    A = synth.uniform(42, 35, P, 0, batch * L).reshape(batch, L)
    x = synth.uniform(42, 36, P, 0, L)
    A[-1, :] = P - 1
    x[:] = np.where(np.arange(L) % 5 == 0, P - 1, x)
    out = torch.full((batch,), 7, dtype=torch.int32, device="cuda").view(torch.uint32)
    m.dot(m.ctx_init(P), torch.from_numpy(A).cuda(), torch.from_numpy(x).cuda(), out=out,
          cfg=m.Launch(variant=8, unroll=stages, ctas_per_sm=ctas, chunk=chunk))
    assert np.array_equal(out.cpu().numpy(), oracle.dot(P, A, x))


def test_dot_pipe_misaligned_falls_back(m):
    """Variant 8 needs 16-byte rows and operands; otherwise the one-CTA-per-row kernel runs."""
    P = 2013265921
    L = 1001
    A = synth.uniform(42, 37, P, 0, 4 * L).reshape(4, L)
    x = synth.uniform(42, 38, P, 0, L)
    out = m.dot(m.ctx_init(P), torch.from_numpy(A).cuda(), torch.from_numpy(x).cuda(), cfg=m.Launch(variant=8))
    assert np.array_equal(out.cpu().numpy(), oracle.dot(P, A, x))
