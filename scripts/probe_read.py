"""Read-only HBM rate (the roofline of mont_dot's A stream): mont_checksum (a flat-grid sum, 4 B read
per element, nothing written) over 2^26 and 2^28 words, vs mont_dot over the same 2^26 words."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_00999_b200 as m  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


P = 2013265921
ctx = m.ctx_init(P)
acc = torch.zeros(1, dtype=torch.int64, device="cuda")
for logn in (26, 28):
    x = torch.empty(1 << logn, dtype=torch.uint32, device="cuda")
    m.synth_fill(x, 42, 40, 0, P)
    t = timeit(lambda: m.checksum(ctx, x, acc=acc))
    print(json.dumps({"what": "read_only_checksum", "words": 1 << logn, "us": t * 1e6, "gbs": 4 * (1 << logn) / t / 1e9}))
    del x
A = torch.empty(1 << 26, dtype=torch.uint32, device="cuda")
m.synth_fill(A, 42, 41, 0, P)
xv = torch.empty(1 << 14, dtype=torch.uint32, device="cuda")
m.synth_fill(xv, 42, 42, 0, P)
o = torch.empty(4096, dtype=torch.uint32, device="cuda")
t = timeit(lambda: m.dot(ctx, A.view(4096, 1 << 14), xv, out=o))
print(json.dumps({"what": "mont_dot 4096 x 2^14", "us": t * 1e6, "gbs": 4 * (1 << 26) / t / 1e9}))
