"""mont_run (include/mont_run.h): lists of HBM-bound jobs in one launch, bit-identical to the
single-operation entry points and to the oracle, incl. the fused to_mont -> from_mont pair, the
fused checksum, ragged tiles and the step's own job list at full size."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
P0, P1, P2 = synth.CONFIG_PRIMES


@pytest.fixture(scope="module")
def m():
    import paper_1609_00999_b200 as mod
    return mod


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def u32(n):
    return torch.empty(n, dtype=torch.uint32, device="cuda")


@pytest.mark.parametrize("n", [4, 8, 2044, 2048, 2052, 4096, 100_004, 1 << 20])
def test_run_each_op_vs_oracle(m, n):
    rng = np.random.default_rng(n)
    jobs, checks = [], []
    for P in (P0, P1, P2, 3, 2147483647):
        ctx = m.ctx_init(P)
        a = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
        b = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
        ta, tb = dev(a), dev(b)
        c, acc = u32(n), torch.zeros(1, dtype=torch.int64, device="cuda")
        t, f = u32(n), u32(n)
        jobs += [m.run_job("mul_vec", ctx, c, ta, tb, acc=acc), m.run_job("to_mont", ctx, t, ta),
                 m.run_job("from_mont", ctx, f, tb)]
        ref = oracle.mont_mul(P, a, b)
        checks += [(c, ref), (t, oracle.to_mont(P, a)), (f, oracle.from_mont(P, b)),
                   (acc, oracle.raw_sum(ref))]
    m.run(jobs)
    torch.cuda.synchronize()
    for got, want in checks:
        if isinstance(want, int):
            assert int(got.item()) == want
        else:
            assert np.array_equal(got.cpu().numpy(), want)


@pytest.mark.parametrize("batch,L", [(1, 4), (3, 8), (17, 1024), (5, 16384), (64, 64)])
def test_run_twiddle_vs_oracle(m, batch, L):
    P = P0
    ctx = m.ctx_init(P)
    x = synth.c3_x(P, batch=batch, length=L)
    tw = synth.uniform(42, 11, P, 0, L)
    out = u32(batch * L)
    m.run([m.run_job("twiddle", ctx, out, dev(x).view(-1), dev(tw))])
    assert np.array_equal(out.cpu().numpy().reshape(batch, L), oracle.twiddle(P, x, tw))


@pytest.mark.parametrize("n", [4, 2048, 5000, 1 << 20])
def test_run_fused_to_from_pair(m, n):
    """from_mont(to_mont(x)) in one job pair: to_mont's output is written, from_mont's consumes
    the register (bit-identical to the separate calls; the round trip returns x)."""
    P = P0
    ctx = m.ctx_init(P)
    x = synth.uniform(42, 1, P, 0, n)
    tx = dev(x)
    bar, back = u32(n), u32(n)
    jobs = [m.run_job("to_mont", ctx, bar, tx), m.run_job("from_mont", ctx, back, bar)]
    assert m.run_bytes(jobs) == 12 * n
    m.run(jobs)
    assert np.array_equal(bar.cpu().numpy(), oracle.to_mont(P, x))
    assert np.array_equal(back.cpu().numpy(), x)


def test_run_in_place_and_empty_jobs(m):
    P = P1
    ctx = m.ctx_init(P)
    a = synth.uniform(42, 1, P, 0, 4096)
    b = synth.uniform(42, 2, P, 0, 4096)
    ta, tb = dev(a), dev(b)
    e = u32(0)
    m.run([m.run_job("mul_vec", ctx, ta, ta, tb), m.run_job("to_mont", ctx, e, e)])
    assert np.array_equal(ta.cpu().numpy(), oracle.mont_mul(P, a, b))
    m.run([])


def test_run_rejects(m):
    ctx = m.ctx_init(P0)
    a, c = u32(1028), u32(1028)
    with pytest.raises(m.MontError):
        m.run([m.run_job("to_mont", ctx, c[1:1025], a[:1024])])        # misaligned out
    with pytest.raises(m.MontError):
        m.run([m.run_job("to_mont", ctx, c[:1026], a[:1026])])         # n % 4
    with pytest.raises(m.MontError):                                   # a job reading another's output
        m.run([m.run_job("to_mont", ctx, c, a), m.run_job("mul_vec", ctx, a, c, c)])


def test_run_step_job_list_fullsize(m):
    """The HBM lane of bench.py's step as ONE run at full size (configs[1] x 3 primes with fused
    checksums, the to/from pair on P0's operand a, configs[2]'s twiddle), every output equal to the
    single-operation kernels' and the checksums to the oracle's sampled identity."""
    n = 1 << 26
    jobs, singles = [], []
    accs = []
    abar = back = None
    for si, P in enumerate((P0, P1, P2)):
        ctx = m.ctx_init(P)
        a, b = u32(n), u32(n)
        m.synth_fill(a, 42, 1, 0, P, 0, True)
        m.synth_fill(b, 42, 2, 0, P, 0, True)
        c = u32(n)
        acc = torch.zeros(1, dtype=torch.int64, device="cuda")
        jobs.append(m.run_job("mul_vec", ctx, c, a, b, acc=acc))
        singles.append((c, lambda ctx=ctx, a=a, b=b: m.mul_vec_checksum(ctx, a, b)))
        accs.append(acc)
        if P == P0:
            abar, back = u32(n), u32(n)
            jobs += [m.run_job("to_mont", ctx, abar, a), m.run_job("from_mont", ctx, back, abar)]
            a0 = a
    ctx0 = m.ctx_init(P0)
    L = 1 << 14
    x = u32(4096 * L)
    m.synth_fill(x, 42, 5, 0, P0, 0, False)
    tw = m.twiddle_table(ctx0, oracle.root_of_unity(P0, 31, L), L)
    o = u32(4096 * L)
    jobs.append(m.run_job("twiddle", ctx0, o, x, tw))
    m.run(jobs)
    torch.cuda.synchronize()
    for (c, single), acc in zip(singles, accs):
        c2, acc2 = single()
        assert torch.equal(c, c2) and int(acc.item()) == int(acc2.item())
    assert torch.equal(abar, m.to_mont(ctx0, a0)) and torch.equal(back, a0)
    assert torch.equal(o, m.mul_twiddle(ctx0, x.view(4096, L), tw).view(-1))
