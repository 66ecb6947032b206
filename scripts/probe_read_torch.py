"""Reference read-only rates from torch reductions (library kernels, for the mont_dot roofline only)."""
import torch, json
def timeit(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); ts=[]
    for _ in range(reps):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1)*1e-3)
    ts.sort(); return ts[len(ts)//2]
for logn in (26, 28):
    x = torch.randint(0, 1000, (1 << logn,), dtype=torch.int32, device="cuda")
    t = timeit(lambda: torch.sum(x))
    print(json.dumps({"what": "torch.sum int32", "words": 1<<logn, "us": t*1e6, "gbs": 4*(1<<logn)/t/1e9}))
    xf = x.float()
    t = timeit(lambda: torch.sum(xf))
    print(json.dumps({"what": "torch.sum f32", "words": 1<<logn, "us": t*1e6, "gbs": 4*(1<<logn)/t/1e9}))
    t = timeit(lambda: torch.amax(x))
    print(json.dumps({"what": "torch.amax int32", "words": 1<<logn, "us": t*1e6, "gbs": 4*(1<<logn)/t/1e9}))
