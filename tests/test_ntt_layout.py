"""Shared-memory layouts of the NTT kernels (k_ntt.cu), checked offline: every warp access of the
row kernel k_ntt_dif (the five-bit trip windows and the final bit-reversed gather) and of the
large transform's column kernel k_ntt_col<12, 8> touches 32 distinct banks, and the address maps
are bijections.  Pure Python replay of the kernels' index arithmetic; no GPU."""
import importlib.util
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _load(name):
    spec = importlib.util.spec_from_file_location(name, ROOT / "scripts" / f"{name}.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def swz(a):
    return a ^ (((a >> 5) ^ (a >> 10)) & 31)


def brev(x, n):
    return int(bin(x)[2:].zfill(n)[::-1], 2)


def worst_conflict(accesses):
    banks = {}
    for w in set(accesses):
        banks.setdefault(w % 32, set()).add(w)
    return max(len(v) for v in banks.values())


@pytest.mark.parametrize("log_n", [10, 11, 12, 13, 14, 15])
def test_dif_row_kernel_conflict_free(log_n):
    N, T = 1 << log_n, (1 << log_n) >> 5
    assert len({swz(a) for a in range(N)}) == N
    worst = 1
    ntrip = (log_n + 4) // 5
    for trip in range(1, ntrip):          # trip 0 reads HBM; its smem store uses the same pattern
        top = log_n - 5 * trip
        wlo = max(top - 5, 0)
        for w in range(T // 32):
            for k in range(32):
                acc = []
                for lane in range(32):
                    t = w * 32 + lane
                    tl = t & ((1 << wlo) - 1)
                    base = tl | ((t >> wlo) << (wlo + 5))
                    acc.append(swz(base) ^ swz(k << wlo))
                worst = max(worst, worst_conflict(acc))
    wlo0 = log_n - 5                      # trip-0 store
    for w in range(T // 32):
        for k in range(32):
            acc = []
            for lane in range(32):
                t = w * 32 + lane
                tl = t & ((1 << wlo0) - 1)
                base = tl | ((t >> wlo0) << (wlo0 + 5))
                acc.append(swz(base) ^ swz(k << wlo0))
            worst = max(worst, worst_conflict(acc))
    for w in range(T // 32):              # final gather: X[t + kT] at brev(t + kT)
        for k in range(32):
            acc = [swz(brev(w * 32 + lane, log_n)) ^ swz(brev(k * T, log_n)) for lane in range(32)]
            worst = max(worst, worst_conflict(acc))
    assert worst == 1


@pytest.mark.parametrize("log_n", [11, 12])
def test_column_kernel_conflict_free(log_n):
    banks = _load("ntt_col_banks")
    assert banks.check(log_n, 8) == 1


def pad(a):
    return a + (a >> 5)


@pytest.mark.parametrize("log_n", list(range(5, 16)))
def test_dif_padded_layout_conflict_free(log_n):
    """The padded layout of k_ntt_dif<.., PAD = true> (the default): word a at a + (a >> 5); the
    last trip stores each result at its natural index brev(pos) and the final gather reads natural
    order.  Rows per CTA as the launcher picks them (lanes may span rows for N < 1024)."""
    N, T = 1 << log_n, (1 << log_n) >> 5
    rpc = 1 if T >= 256 else 256 // T
    NP = N + N // 32
    nthr = rpc * T
    ntrip = (log_n + 4) // 5
    worst = 1

    def lanes(w):
        for lane in range(32):
            tid = w * 32 + lane
            yield tid // T, tid % T

    for trip in range(ntrip):
        top = log_n - 5 * trip
        wlo = max(top - 5, 0)
        last = trip == ntrip - 1
        for w in range(nthr // 32):
            for k in range(32):
                ld, st = [], []
                for rl, t in lanes(w):
                    tl = t & ((1 << wlo) - 1)
                    pos = tl | ((t >> wlo) << (wlo + 5)) | (k << wlo)
                    ld.append(rl * NP + pad(pos))
                    st.append(rl * NP + pad(brev(pos, log_n) if last else pos))
                if trip > 0:
                    worst = max(worst, worst_conflict(ld))
                worst = max(worst, worst_conflict(st))
    for w in range(nthr // 32):
        for k in range(32):
            worst = max(worst, worst_conflict([rl * NP + pad(t + k * T) for rl, t in lanes(w)]))
    assert worst == 1
    # additive: f(base | kpart) = f(base) + f(kpart) for disjoint bit sets (immediate offsets)
    for base, kp in ((0b1010, 0b110000000), (0x1F, 0x3E0), (0x2A5, 0x1800)):
        assert base & kp == 0 and pad(base | kp) == pad(base) + pad(kp)


@pytest.mark.parametrize("log_n", [11, 12])
def test_column_kernel_padded_layout_conflict_free(log_n):
    """k_ntt_col<.., 8, PQ, PAD = true> (the default): column c at c (N + N/32 + 4) + a + (a >> 5);
    trip 0 stores in map G (lanes: 8 columns x 4 rows), later trips in map S (32 t of one column),
    the last trip stores in natural order, the final gather reads natural order in map G."""
    C = 8
    N, T = 1 << log_n, (1 << log_n) >> 5
    NPC = N + N // 32 + 4
    nthr = C * T
    ntrip = (log_n + 4) // 5
    addr = lambda col, a: col * NPC + pad(a)
    worst = 1
    for trip in range(ntrip):
        top = log_n - 5 * trip
        wlo = max(top - 5, 0)
        last = trip == ntrip - 1
        for w in range(nthr // 32):
            for k in range(32):
                ld, st = [], []
                for lane in range(32):
                    tid = w * 32 + lane
                    col, t = (tid % C, tid // C) if trip == 0 else (tid // T, tid % T)
                    tl = t & ((1 << wlo) - 1)
                    pos = tl | ((t >> wlo) << (wlo + 5)) | (k << wlo)
                    ld.append(addr(col, pos))
                    st.append(addr(col, brev(pos, log_n) if last else pos))
                if trip > 0:
                    worst = max(worst, worst_conflict(ld))
                worst = max(worst, worst_conflict(st))
    for w in range(nthr // 32):
        for k in range(32):
            worst = max(worst, worst_conflict([addr((w * 32 + l) % C, (w * 32 + l) // C + k * T)
                                               for l in range(32)]))
    assert worst == 1
