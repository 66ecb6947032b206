import itertools
def bitrev(x, n):
    r = 0
    for i in range(n):
        r = (r << 1) | ((x >> i) & 1)
    return r

def patterns(logN, B):
    T = 1 << (logN - B)
    pats = []
    # natural coalesced read/write: idx = t + k*T, and the bitrev scatter
    for k in [0, 1, (1 << B) - 1]:
        pats.append(("nat", [(t + k * T) for t in range(min(32, T))]))
        pats.append(("brev", [bitrev(t + k * T, logN) for t in range(min(32, T))]))
    s0 = 0
    while s0 < logN:
        ws = min(s0, logN - B)
        for k in [0, 1, (1 << B) - 1]:
            addrs = []
            for t in range(min(32, T)):
                tl = t & ((1 << ws) - 1); th = t >> ws
                addrs.append(tl | (k << ws) | (th << (ws + B)))
            pats.append((f"grp{s0}", addrs))
        s0 += B
    return pats

def conflicts(sw, addrs):
    banks = {}
    for a in addrs:
        b = sw(a) & 31
        banks[b] = banks.get(b, 0) + 1
    return max(banks.values())

def make_fold(logN):
    def sw(a):
        h = 0
        x = a >> 5
        while x:
            h ^= x & 31
            x >>= 5
        return a ^ h
    return sw

def make_fold_rev(logN):
    def sw(a):
        h = 0
        x = a >> 5
        while x:
            h ^= x & 31
            x >>= 5
        h ^= bitrev((a >> (logN - 5)) & 31, 5) if logN >= 10 else 0
        return a ^ h
    return sw

for name, mk in [("fold", make_fold), ("fold_rev", make_fold_rev)]:
    for logN in range(10, 16):
        for B in (4, 5):
            sw = mk(logN)
            # bijection check
            assert len({sw(a) for a in range(1 << logN)}) == 1 << logN
            worst = max((conflicts(sw, ad), nm) for nm, ad in patterns(logN, B))
            print(name, logN, B, worst)
