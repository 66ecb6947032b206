"""Offline check (no GPU) of a 16-elements-per-thread NTT row layout (4-bit trip windows) --
DESIGN.md §11 item 3.  Replays the shared-memory accesses of every trip (the DIF kernel's pattern
with W = 4 instead of 5, last trip storing in natural order as k_ntt_dif<.., PAD> does) and the
final gather, and reports the worst bank conflict for candidate layouts: additive paddings
a + (a >> s), a + (a >> s1) + (a >> s2), and XOR swizzles.

    python scripts/ntt_layout16.py
"""


def brev(x, n):
    return int(bin(x)[2:].zfill(n)[::-1], 2)


def worst_conflict(acc):
    banks = {}
    for w in set(acc):
        banks.setdefault(w % 32, set()).add(w)
    return max(len(v) for v in banks.values())


def check(log_n, f, E=16, W=4):
    N = 1 << log_n
    T = N // E
    rpc = 1 if T >= 256 else 256 // T
    NP = f(N - 1) + 1
    nthr = rpc * T
    ntrip = (log_n + W - 1) // W
    worst = 1

    def lanes(w):
        for lane in range(32):
            tid = w * 32 + lane
            yield tid // T, tid % T

    for trip in range(ntrip):
        top = log_n - W * trip
        wlo = max(top - W, 0)
        last = trip == ntrip - 1
        for w in range(nthr // 32):
            for k in range(E):
                ld, st = [], []
                for rl, t in lanes(w):
                    tl = t & ((1 << wlo) - 1)
                    pos = tl | ((t >> wlo) << (wlo + W)) | (k << wlo)
                    ld.append(rl * NP + f(pos))
                    st.append(rl * NP + f(brev(pos, log_n) if last else pos))
                if trip > 0:
                    worst = max(worst, worst_conflict(ld))
                worst = max(worst, worst_conflict(st))
    for w in range(nthr // 32):
        for k in range(E):
            worst = max(worst, worst_conflict([rl * NP + f(t + k * T) for rl, t in lanes(w)]))
    return worst


def candidates():
    c = {}
    for s in range(3, 9):
        c[f"a + (a >> {s})"] = (lambda s: lambda a: a + (a >> s))(s)
    for s1 in range(3, 8):
        for s2 in range(s1 + 1, 11):
            c[f"a + (a >> {s1}) + (a >> {s2})"] = (lambda s1, s2: lambda a: a + (a >> s1) + (a >> s2))(s1, s2)
    c["a ^ (((a >> 5) ^ (a >> 10)) & 31)"] = lambda a: a ^ (((a >> 5) ^ (a >> 10)) & 31)
    c["a ^ (((a >> 4) ^ (a >> 8) ^ (a >> 12)) & 15)"] = lambda a: a ^ (((a >> 4) ^ (a >> 8) ^ (a >> 12)) & 15)
    return c


def main():
    free = []
    for name, f in candidates().items():
        w = max(check(ln, f) for ln in range(8, 16))
        print(f"{name:48s} worst conflict over 2^8..2^15: {w}-way")
        if w == 1:
            free.append(name)
    print("conflict-free:", free or "none")


if __name__ == "__main__":
    main()
