"""Barrett comparison kernels (include/barrett.h) vs the oracle."""
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


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("P", list(synth.CONFIG_PRIMES) + [3, 17, 257, 65537, 2147483647, 1073741827, 1073741825 | 1])
@pytest.mark.parametrize("n", [1, 7, 4096 + 3, 1 << 20])
def test_barrett_mul_vec(m, P, n):
    rng = np.random.default_rng(n + P)
    a = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    a[:1] = P - 1
    b[:1] = P - 1
    c = m.barrett_mul_vec(m.barrett_ctx_init(P), dev(a), dev(b))
    assert np.array_equal(c.cpu().numpy(), oracle.mulmod_vec(P, a, b))


@pytest.mark.parametrize("P", [3, 5, 17, 97, 251, 257])
def test_barrett_all_pairs(m, P):
    g = np.arange(P, dtype=np.uint32)
    a, b = np.repeat(g, P), np.tile(g, P)
    c = m.barrett_mul_vec(m.barrett_ctx_init(P), dev(a), dev(b))
    assert np.array_equal(c.cpu().numpy(), oracle.mulmod_vec(P, a, b))


@pytest.mark.parametrize("P", list(synth.CONFIG_PRIMES) + [17, 2147483647])
@pytest.mark.parametrize("n", [1, 5, 4096, 20003])
def test_barrett_pow(m, P, n):
    base = synth.uniform(42, 3, P, 0, n, low=1)
    e = synth.exponents(42, 4, 0, n)
    base[:2] = [0, P - 1][:n]
    e[:2] = [0, (1 << 31) - 1][:n]
    out = m.barrett_pow_vec(m.barrett_ctx_init(P), dev(base), dev(e))
    assert np.array_equal(out.cpu().numpy(), oracle.power(P, base, e))


def test_barrett_ctx(m):
    for P in (3, 17, 2013265921, 2147483647):
        c = m.barrett_ctx_init(P)
        o = oracle.ctx(P)
        assert c.k == o.bk and c.pprime == o.bPprime
    with pytest.raises(m.MontError):
        m.barrett_ctx_init(4)
