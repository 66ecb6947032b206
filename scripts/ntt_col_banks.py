"""Bank-conflict check for k_ntt_col (k_ntt.cu): replays every shared-memory access pattern of the
column-mode DIF kernel (trip-0 stores in map G, the map-S trips, the final bit-reversed gather in
map G) for each warp and reports the worst number of distinct words that share a bank (1 = none).
Also checks that the per-column address map is a bijection.  Offline, no GPU."""
import sys


def swz(a):
    return a ^ (((a >> 5) ^ (a >> 10)) & 31)


def brev(x, n):
    return int(bin(x)[2:].zfill(n)[::-1], 2)


def check(LOG_N, C):
    N, T = 1 << LOG_N, (1 << LOG_N) >> 5
    CSH = {16: 1, 8: 2, 4: 3}[C]
    nthr = C * T
    addr = lambda col, a: col * N + (swz(a) ^ ((col << CSH) & 31))
    for col in range(C):
        assert len({addr(col, a) for a in range(N)}) == N
    worst = 1
    ntrip = (LOG_N + 4) // 5

    def account(accesses):  # accesses: per lane one word address
        nonlocal worst
        banks = {}
        for w in set(accesses):
            banks.setdefault(w % 32, set()).add(w)
        worst = max(worst, max(len(v) for v in banks.values()))

    for trip in range(ntrip):
        top = LOG_N - 5 * trip
        wlo = max(top - 5, 0)
        for warp in range(nthr // 32):
            for k in range(32):
                acc = []
                for lane in range(32):
                    tid = warp * 32 + lane
                    col, t = (tid % C, tid // C) if trip == 0 else (tid // T, tid % T)
                    tl = t & ((1 << wlo) - 1)
                    base = tl | ((t >> wlo) << (wlo + 5))
                    acc.append(addr(col, base | (k << wlo)))
                account(acc)
    R = 32 // C
    for warp in range(nthr // 32):  # final gather, map H
        for k in range(32):
            acc = []
            for lane in range(32):
                col, t = lane % C, (lane // C) * (T // R) + warp
                acc.append(addr(col, brev(t + k * T, LOG_N)))
            account(acc)
    # map H covers every (column, t) exactly once
    assert sorted((l % C, (l // C) * (T // R) + w) for w in range(nthr // 32) for l in range(32)) == \
        sorted((c, t) for c in range(C) for t in range(T))
    return worst


if __name__ == "__main__":
    bad = 0
    for LOG_N in (11, 12):  # the instantiated column kernels (k_ntt_col<11|12, 8, PQ>), and C = 4
        for C in (8, 4):
            w = check(LOG_N, C)
            print(f"log_n={LOG_N} C={C}: worst {w}-way")
            bad |= w > 1
    sys.exit(1 if bad else 0)
