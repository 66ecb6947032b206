"""GPU parity across the whole modulus range: 48 seeded random odd moduli 3 <= P < 2^31 (primes
and composites alike -- REDC needs only gcd(R, P) = 1, reading G16), log-uniform so
that every bit length 2..31 appears, plus the extremes 3 and 2^31 - 1.  Every hot-path kernel
(mul_vec, the fused checksum, to/from_mont, pow in the default and the bench's lane launch,
the twiddle multiply) against the oracle on ragged sizes with the edge values 0 and P - 1."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _moduli():
    rng = np.random.default_rng(20161999)
    ps = {3, 2147483647, 2147483645}
    while len(ps) < 50:
        bits = int(rng.integers(2, 32))
        p = int(rng.integers(1 << (bits - 1), 1 << bits)) | 1
        if 3 <= p < (1 << 31):
            ps.add(p)
    return sorted(ps)


MODULI = _moduli()


@pytest.fixture(scope="module")
def m():
    import paper_1609_00999_b200 as mod
    return mod


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def inputs(P, n, seed):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    a[:4] = [0, P - 1, P - 1, 1]
    b[:4] = [P - 1, P - 1, 0, P - 1]
    a[-1], b[-1] = P - 1, P - 1
    return a, b


@pytest.mark.parametrize("P", MODULI)
def test_elementwise_any_modulus(m, P):
    n = 4099
    a, b = inputs(P, n, P)
    ctx = m.ctx_init(P)
    ref = oracle.mont_mul(P, a, b)
    assert np.array_equal(host(m.mul_vec(ctx, dev(a), dev(b))), ref)
    c, acc = m.mul_vec_checksum(ctx, dev(a), dev(b))
    assert np.array_equal(host(c), ref) and int(acc.item()) == oracle.raw_sum(ref)
    t = m.to_mont(ctx, dev(a))
    assert np.array_equal(host(t), oracle.to_mont(P, a))
    assert np.array_equal(host(m.from_mont(ctx, t)), a)


@pytest.mark.parametrize("P", MODULI)
def test_pow_any_modulus(m, P):
    n = 2053
    rng = np.random.default_rng(P + 1)
    base = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    exp = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)   # full 32-bit exponents
    base[:3], exp[:3] = [0, P - 1, 1], [0, 0xFFFFFFFF, 0x7FFFFFFF]
    ctx = m.ctx_init(P)
    ref = oracle.power(P, base, exp)
    assert np.array_equal(host(m.pow_vec(ctx, dev(base), dev(exp))), ref)
    for v, k in ((10, 1), (10, 2), (11, 1), (13, 2), (17, 2)):
        lane = m.Launch(ctas_per_sm=k, variant=v)
        assert np.array_equal(host(m.pow_vec(ctx, dev(base), dev(exp), cfg=lane)), ref), v


@pytest.mark.parametrize("P", MODULI[::5])
def test_twiddle_any_modulus(m, P):
    batch, L = 5, 384
    rng = np.random.default_rng(P + 2)
    x = rng.integers(0, P, batch * L, dtype=np.uint64).astype(np.uint32).reshape(batch, L)
    tw = rng.integers(0, P, L, dtype=np.uint64).astype(np.uint32)
    out = m.mul_twiddle(m.ctx_init(P), dev(x), dev(tw))
    assert np.array_equal(host(out), oracle.twiddle(P, x, tw))
