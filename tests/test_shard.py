"""The N>1 path on CPU: world_size-2 gloo process group, contiguous global-index
slices, per-rank partials combined by one SUM all-reduce.
Each rank computes its slice with the oracle (the kernels need a GPU); what is
tested here is the shard arithmetic and the collective plumbing of
paper_1609_00999_b200.shard."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1609_00999_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import oracle
    import synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard.slice_bounds(n, world, rank)
        sums, Ps = [], list(synth.CONFIG_PRIMES)
        for P in Ps:
            a, b = synth.c2_inputs(P, lo, hi - lo)     # GLOBAL index -> world-size independent
            sums.append(oracle.raw_sum(oracle.mont_mul(P, a, b, nthreads=1)))
        box = shard.combine_checksums(sums, Ps)
        tmax = shard.max_over_ranks(float(rank + 1))
        shard.barrier()
        q.put((rank, lo, hi, box, tmax))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_checksum_matches_single(world):
    n = 100_003
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    import oracle
    import synth
    # slices tile [0, n) exactly
    assert res[0][1] == 0 and res[-1][2] == n
    assert all(res[i][2] == res[i + 1][1] for i in range(world - 1))
    want = []
    for P in synth.CONFIG_PRIMES:
        a, b = synth.c2_inputs(P, 0, n)
        want.append(oracle.checksum(P, oracle.mont_mul(P, a, b)))
    for r in res:
        assert r[3] == want            # every rank sees the box checksum
        assert r[4] == float(world)    # max over ranks


def test_slice_bounds():
    for n in (0, 1, 7, 2 ** 31):
        for w in (1, 2, 3, 8):
            b = [shard.slice_bounds(n, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1
    assert shard.slice_bounds(2 ** 31, 8, 3) == (3 * 2 ** 28, 4 * 2 ** 28)
    with pytest.raises(ValueError):
        shard.slice_bounds(10, 2, 2)


def test_single_process_passthrough():
    assert shard.combine_checksums(12345, 17) == 12345 % 17
    assert shard.combine_checksums([5, 40], [7, 11]) == [5, 40 % 11]
    assert shard.max_over_ranks(3.5) == 3.5
    shard.barrier()
    assert np.isfinite(shard.max_over_ranks(1.0))
