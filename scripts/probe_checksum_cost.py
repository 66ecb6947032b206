"""Cost of the fused checksum (A11) in mont_mul_vec_checksum at configs[1]'s size: the same launch
with and without the per-CTA reduction + 64-bit atomic, in the bench's lane shape and the default."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_00999_b200 as m  # noqa: E402


def timeit(fn, reps=30):
    for _ in range(5):
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
n = 1 << 26
ctx = m.ctx_init(P)
a, b, c = (torch.empty(n, dtype=torch.uint32, device="cuda") for _ in range(3))
m.synth_fill(a, 42, 1, 0, P)
m.synth_fill(b, 42, 2, 0, P)
acc = torch.zeros(1, dtype=torch.int64, device="cuda")
for name, cfg in (("default", None), ("256x2", m.Launch(threads=256, unroll=2)), ("512x2", m.Launch(threads=512, unroll=2)),
                  ("256x4", m.Launch(threads=256, unroll=4)), ("512x4", m.Launch(threads=512, unroll=4))):
    t0 = timeit(lambda: m.mul_vec(ctx, a, b, out=c, cfg=cfg))
    t1 = timeit(lambda: m.mul_vec_checksum(ctx, a, b, out=c, acc=acc, cfg=cfg))
    print(json.dumps({"what": "mul_vec vs mul_vec_checksum, 2^26", "launch": name, "us_plain": t0 * 1e6,
                      "us_checksum": t1 * 1e6, "gbs_plain": 12 * n / t0 / 1e9, "gbs_checksum": 12 * n / t1 / 1e9}))
