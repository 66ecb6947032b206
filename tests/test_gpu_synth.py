"""The device generator (synth_fill in libmont.so) reproduces synth/ exactly."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    import paper_1609_00999_b200 as mod
    return mod


@pytest.mark.parametrize("P", synth.CONFIG_PRIMES)
@pytest.mark.parametrize("stream,mode,specials", [(1, 0, False), (2, 0, True), (3, 1, False), (4, 2, False),
                                                  (5, 0, False)])
def test_synth_first_2_20(m, P, stream, mode, specials):
    n = 1 << 20
    t = torch.empty(n, dtype=torch.uint32, device="cuda")
    m.synth_fill(t, 42, stream, 0, P, mode, specials)
    torch.cuda.synchronize()
    if mode == 2:
        ref = synth.exponents(42, stream, 0, n)
    else:
        ref = synth.uniform(42, stream, P, 0, n, low=mode)
    if specials:
        synth.apply_specials(ref, 42, stream, P, 0)
    assert np.array_equal(t.cpu().numpy(), ref)


def test_synth_high_indices(m):
    P = 2013265921
    start = (1 << 31) - 12345
    t = torch.empty(100_000, dtype=torch.uint32, device="cuda")
    m.synth_fill(t, 42, 1, start, P, 0, False)
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy(), synth.uniform(42, 1, P, start, 100_000))
