"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO Montgomery / modular-multiplication arithmetic: it only
turns (seed, stream, element index) into uint32 residues, exponents and the
edge-value injections that DESIGN.md §5 ("input recipe") fixes.  Both the
oracle tests and the product bench draw their host inputs from here; the CUDA
library carries its own implementation of the same counter-based function
(`synth_*` in csrc/synth.cu), cross-checked against this one in
tests/test_gpu_synth.py.

Generator (SURVEY.md §8(c) "Seeded inputs", Appendix B): the SplitMix64 output
function (Steele, Lea, Flood 2014) applied to a counter,

    h(seed, stream, i) = mix(seed + (stream * 2**40 + i + 1) * GAMMA)  (mod 2**64)

and the value maps

    uniform[0, P)  = floor(h * P / 2**64)
    uniform[1, P)  = 1 + floor(h * (P - 1) / 2**64)
    exponent       = h >> 33                      (31-bit, BASELINE configs[3])

The paper fixes no input distribution (§3.1 works over "word-size
primes", arbitrary residues), so uniform residues with the edge values
0, 1, P-1 injected stand in for the paper's operands.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK32 = np.uint64(0xFFFFFFFF)

DEFAULT_SEED = 42

# stream ids
STREAM_A = 1
STREAM_B = 2
STREAM_BASE = 3
STREAM_EXP = 4
STREAM_TWX = 5
SPECIAL_OFFSET = 16          # special-value injection uses stream + 16
SPECIAL_MOD = 300            # k = h mod 300; k < 3 -> (0, 1, P-1)[k]  (~1 %)

# convention for the twiddle root: w = G11_GENERATOR^((P-1)/len)
G11_GENERATOR = 31

_CHUNK = 1 << 22


def _mix(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * _M1
    z = z ^ (z >> np.uint64(27))
    z = z * _M2
    z = z ^ (z >> np.uint64(31))
    return z


def splitmix_h(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """h(seed, stream, i) for a uint64 index array (wrapping mod 2**64)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        ctr = np.uint64((stream << 40) & 0xFFFFFFFFFFFFFFFF) + idx + np.uint64(1)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + ctr * GAMMA
        return _mix(z)


def _scale(h: np.ndarray, m: int) -> np.ndarray:
    """floor(h * m / 2**64) for m < 2**32, exact via a 32-bit split."""
    m64 = np.uint64(m)
    hi = h >> np.uint64(32)
    lo = h & _MASK32
    return ((hi * m64 + ((lo * m64) >> np.uint64(32))) >> np.uint64(32)).astype(np.uint32)


def _indices(start: int, count: int) -> np.ndarray:
    return np.arange(start, start + count, dtype=np.uint64)


def _chunked(fn, start: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint32)
    for off in range(0, count, _CHUNK):
        c = min(_CHUNK, count - off)
        out[off:off + c] = fn(_indices(start + off, c))
    return out


def uniform(seed: int, stream: int, P: int, start: int, count: int, low: int = 0) -> np.ndarray:
    """uint32 values uniform in [low, P), low in {0, 1}, for indices start..start+count-1."""
    if low not in (0, 1):
        raise ValueError("low must be 0 or 1")
    if low == 0:
        return _chunked(lambda i: _scale(splitmix_h(seed, stream, i), P), start, count)
    return _chunked(lambda i: (_scale(splitmix_h(seed, stream, i), P - 1) + np.uint32(1)).astype(np.uint32),
                    start, count)


def uniform_at(seed: int, stream: int, P: int, idx: np.ndarray, low: int = 0) -> np.ndarray:
    """Same as uniform() but at arbitrary (sampled) indices."""
    idx = np.asarray(idx, dtype=np.uint64)
    if low == 0:
        return _scale(splitmix_h(seed, stream, idx), P)
    return (_scale(splitmix_h(seed, stream, idx), P - 1) + np.uint32(1)).astype(np.uint32)


def exponents(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """31-bit exponents h >> 33, uniform in [0, 2**31)."""
    return _chunked(lambda i: (splitmix_h(seed, stream, i) >> np.uint64(33)).astype(np.uint32), start, count)


def exponents_at(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    return (splitmix_h(seed, stream, np.asarray(idx, dtype=np.uint64)) >> np.uint64(33)).astype(np.uint32)


def special_codes(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """k = h(seed, stream+16, i) mod 300 (values < 3 select 0, 1, P-1)."""
    h = splitmix_h(seed, stream + SPECIAL_OFFSET, np.asarray(idx, dtype=np.uint64))
    return (h % np.uint64(SPECIAL_MOD)).astype(np.uint32)


def apply_specials(vals: np.ndarray, seed: int, stream: int, P: int, start: int) -> np.ndarray:
    """configs[1] "1% of entries set to 0, 1 or P-1", in place."""
    for off in range(0, vals.size, _CHUNK):
        c = min(_CHUNK, vals.size - off)
        k = special_codes(seed, stream, _indices(start + off, c))
        seg = vals[off:off + c]
        seg[k == 0] = 0
        seg[k == 1] = 1
        seg[k == 2] = P - 1
    return vals


def apply_specials_at(vals: np.ndarray, seed: int, stream: int, P: int, idx: np.ndarray) -> np.ndarray:
    k = special_codes(seed, stream, idx)
    vals = vals.copy()
    vals[k == 0] = 0
    vals[k == 1] = 1
    vals[k == 2] = P - 1
    return vals


# ---------------------------------------------------------------- configs

def c1_inputs(P: int = 2013265921, n: int = 65536, seed: int = DEFAULT_SEED):
    """configs[0]: uniform a, b in [0,P) with 0 and P-1 forced at fixed indices (G12)."""
    a = uniform(seed, STREAM_A, P, 0, n)
    b = uniform(seed, STREAM_B, P, 0, n)
    force_c1_edges(a, b, P)
    return a, b


def force_c1_edges(a: np.ndarray, b: np.ndarray, P: int) -> None:
    n = a.size
    if n >= 1:
        a[0] = 0
    if n >= 2:
        b[1] = 0
    if n >= 3:
        a[2] = P - 1
        b[2] = P - 1
    if n >= 4:
        a[3] = P - 1
    if n >= 6:
        a[n - 2] = 0
        b[n - 2] = 0
        a[n - 1] = P - 1
        b[n - 1] = P - 1


def c2_inputs(P: int, start: int = 0, count: int = 1 << 26, seed: int = DEFAULT_SEED):
    """configs[1] / configs[4] slice: uniform pairs with 1 % specials (global index start..)."""
    a = apply_specials(uniform(seed, STREAM_A, P, start, count), seed, STREAM_A, P, start)
    b = apply_specials(uniform(seed, STREAM_B, P, start, count), seed, STREAM_B, P, start)
    return a, b


def c2_inputs_at(P: int, idx: np.ndarray, seed: int = DEFAULT_SEED):
    a = apply_specials_at(uniform_at(seed, STREAM_A, P, idx), seed, STREAM_A, P, idx)
    b = apply_specials_at(uniform_at(seed, STREAM_B, P, idx), seed, STREAM_B, P, idx)
    return a, b


def c5_inputs(P: int, start: int, count: int, seed: int = DEFAULT_SEED):
    """configs[4]: uniform pairs, no specials, generated from the GLOBAL index."""
    return uniform(seed, STREAM_A, P, start, count), uniform(seed, STREAM_B, P, start, count)


def c3_x(P: int = 2013265921, batch: int = 4096, length: int = 1 << 14, row0: int = 0,
         seed: int = DEFAULT_SEED) -> np.ndarray:
    """configs[2]: x[r][j] uniform in [0,P), flattened index i = r*length + j."""
    return uniform(seed, STREAM_TWX, P, row0 * length, batch * length).reshape(batch, length)


def c4_inputs(P: int = 469762049, start: int = 0, count: int = 1 << 24, seed: int = DEFAULT_SEED):
    """configs[3]: base uniform in [1,P), exp uniform 31-bit."""
    return (uniform(seed, STREAM_BASE, P, start, count, low=1),
            exponents(seed, STREAM_EXP, start, count))


CONFIG_PRIMES = (2013265921, 469762049, 998244353)
