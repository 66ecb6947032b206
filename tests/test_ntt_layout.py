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
