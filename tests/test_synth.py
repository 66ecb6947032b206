"""Known-answer tests for the shared seeded input generator (synth/)."""
import json

import numpy as np

import synth


def test_generator_kat(golden_dir):
    g = json.loads((golden_dir / "generator_kat.json").read_text())
    seed = g["seed"]
    h = synth.splitmix_h(seed, 1, np.arange(4))
    assert [int(x) for x in h] == [int(x, 16) for x in g["h_stream1"]]
    for P, ab in g["uniform"].items():
        P = int(P)
        assert synth.uniform(seed, synth.STREAM_A, P, 0, 4).tolist() == ab["a"]
        assert synth.uniform(seed, synth.STREAM_B, P, 0, 4).tolist() == ab["b"]
    base, exp = synth.c4_inputs(g["c4"]["P"], 0, 4, seed)
    assert base.tolist() == g["c4"]["base"] and exp.tolist() == g["c4"]["exp"]
    x = synth.c3_x(g["c3"]["P"], batch=2, seed=seed)
    assert x[0, :4].tolist() == g["c3"]["x_row0"] and int(x[1, 0]) == g["c3"]["x_row1_col0"]
    k = synth.special_codes(seed, synth.STREAM_A, np.arange(65536))
    assert int((k < 3).sum()) == g["c2_specials_stream_a_first_65536"]


def test_ranges_and_sampled_access():
    P = 469762049
    a = synth.uniform(42, 1, P, 1000, 1 << 16)
    assert a.max() < P
    b = synth.uniform(42, 3, P, 0, 1 << 16, low=1)
    assert b.min() >= 1 and b.max() < P
    idx = np.array([1000, 1001, 5000, 65535 + 1000], dtype=np.uint64)
    assert np.array_equal(synth.uniform_at(42, 1, P, idx), a[(idx - 1000).astype(np.int64)])
    e = synth.exponents(42, 4, 0, 1 << 16)
    assert e.max() < (1 << 31)
    a2, b2 = synth.c2_inputs(P, 123, 4096)
    ia = np.arange(123, 123 + 4096, dtype=np.uint64)
    a3, b3 = synth.c2_inputs_at(P, ia)
    assert np.array_equal(a2, a3) and np.array_equal(b2, b3)
    assert set(np.unique(a2[synth.special_codes(42, 1, ia) < 3]).tolist()) <= {0, 1, P - 1}


def test_c1_edges():
    P = 2013265921
    a, b = synth.c1_inputs(P)
    n = a.size
    assert (a[0], b[1], a[2], b[2], a[3]) == (0, 0, P - 1, P - 1, P - 1)
    assert (a[n - 2], b[n - 2], a[n - 1], b[n - 1]) == (0, 0, P - 1, P - 1)
