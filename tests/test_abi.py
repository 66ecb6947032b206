"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/*.h
declares, and its host-side logic (context precompute, argument validation)
behaves as documented.  No kernel is launched here."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_1609_00999_b200 as m

ROOT = Path(__file__).resolve().parent.parent
HEADERS = sorted((ROOT / "include").glob("*.h"))


def declared_functions():
    names = []
    for h in HEADERS:
        text = h.read_text()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for mt in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_ ]*?[\s\*]+([A-Za-z_][A-Za-z0-9_]*)\s*\(",
                              text, flags=re.M):
            name = mt.group(1)
            if name not in ("if", "while", "for", "sizeof", "return"):
                names.append(name)
    return sorted(set(names))


def test_headers_declare_the_north_star_api():
    names = declared_functions()
    for required in ("mont_ctx_init", "to_mont", "from_mont", "mont_mul_vec", "mont_mul_twiddle",
                     "mont_pow_vec", "mont_checksum", "mont_strerror"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(str(m.LIB_PATH))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the binding knows every one of them
    assert set(declared_functions()) == set(m.SIGNATURES)


def test_build_arch():
    assert m.lib().mont_build_arch() == 100


@pytest.mark.parametrize("P", list(range(3, 258, 2)) + [2013265921, 469762049, 998244353, 2147483647,
                                                         1073741827, 65537, 12289])
def test_ctx_matches_oracle(P):
    """Newton-lifted P' (library) vs extended Euclid (oracle), plus r1, r2."""
    c = m.ctx_init(P)
    o = oracle.ctx(P)
    assert (c.p, c.pneg, c.r1, c.r2) == (o.P, o.Pprime, o.r1, o.r2)


def test_ctx_random_odd_moduli():
    rng = np.random.default_rng(11)
    for P in rng.integers(3, 1 << 31, 2000):
        P = int(P) | 1
        if P >= 1 << 31:
            continue
        c = m.ctx_init(P)
        assert (c.p * c.pneg) % (1 << 32) == (1 << 32) - 1
        assert c.r1 == (1 << 32) % P and c.r2 == (1 << 64) % P


@pytest.mark.parametrize("P", [0, 1, 2, 4, 1 << 30, 1 << 31, (1 << 31) + 1, 0xFFFFFFFF])
def test_ctx_rejects(P):
    with pytest.raises(m.MontError) as e:
        m.ctx_init(P)
    assert e.value.status == 1


def test_null_ctx_and_strerror():
    L = m.lib()
    assert L.mont_ctx_init(None, 17) == 2
    for s in range(5):
        assert L.mont_strerror(s)
    assert L.mont_strerror(99) == b"unknown status"


def test_validation_without_launch():
    """Synchronous validation paths return before touching CUDA (safe without a GPU)."""
    L = m.lib()
    ctx = m.ctx_init(2013265921)
    bad = m.Ctx(2013265921, 1, 0, 0)           # pneg wrong: not from mont_ctx_init
    pc = C.byref(ctx)
    assert L.mont_mul_vec(pc, None, None, None, 0, None) == 0          # n == 0: OK, no launch
    assert L.mont_mul_vec(pc, None, None, None, 5, None) == 2          # NULL with n > 0
    assert L.mont_mul_vec(C.byref(bad), None, None, None, 5, None) == 1
    assert L.mont_mul_vec(None, None, None, None, 5, None) == 2
    assert L.mont_mul_vec(pc, 0x1002, 0x2000, 0x3000, 5, None) == 2   # not 4-byte aligned
    assert L.to_mont(pc, None, None, 0, None) == 0
    assert L.from_mont(pc, None, None, 3, None) == 2
    assert L.mont_pow_vec(pc, None, None, None, 0, None) == 0
    assert L.mont_pow_vec(pc, None, None, None, 1, None) == 2
    assert L.mont_mul_twiddle(pc, None, None, None, 0, 16, None) == 0  # batch == 0
    assert L.mont_mul_twiddle(pc, 0x1000, 0x2000, 0x3000, 4, 0, None) == 2  # len == 0
    assert L.mont_mul_twiddle(pc, 0x1000, 0x2000, 0x3000, 1 << 40, 1 << 40, None) == 2  # overflow
    assert L.mont_checksum(pc, None, None, 0, None) == 0
    assert L.mont_checksum(pc, 0x1004, 0x2000, 8, None) == 2           # acc not 8-byte aligned
    assert L.mont_twiddle_table(pc, None, 5, 0, None) == 0
    cfg = m.Launch(threads=100)
    assert L.mont_mul_vec_ex(pc, 0x1000, 0x2000, 0x3000, 8, C.byref(cfg), None) == 2  # threads % 32
    cfg = m.Launch(unroll=3)
    assert L.mont_mul_vec_ex(pc, 0x1000, 0x2000, 0x3000, 8, C.byref(cfg), None) == 2
    assert L.synth_fill(None, 4, 1, 1, 0, 17, 0, 0, None) == 2
    assert L.synth_fill(0x1000, 4, 1, 1, 0, 17, 7, 0, None) == 2
    # variants outside each entry point's documented set are refused, not silently remapped
    for v, fn in ((5, L.mont_mul_vec_ex), (4, L.to_mont_ex), (4, L.from_mont_ex)):
        cfg = m.Launch(variant=v)
        args = (pc, 0x1000, 0x2000, 0x3000, 8) if fn is L.mont_mul_vec_ex else (pc, 0x1000, 0x2000, 8)
        assert fn(*args, C.byref(cfg), None) == 2, v
    cfg = m.Launch(variant=18)
    assert L.mont_pow_vec_ex(pc, 0x1000, 0x2000, 0x3000, 8, C.byref(cfg), None) == 2
    cfg = m.Launch(variant=5)
    assert L.mont_mul_twiddle_ex(pc, 0x1000, 0x2000, 0x3000, 4, 16, C.byref(cfg), None) == 2


def test_host_run_bytes_fusion_plan():
    """mont_host_run_bytes (host only): the executor's fusion plan, as bytes copied.
    mul_vec(a, b) -> to_mont(a) -> from_mont(to_mont's out) is one group: a and b go up once each,
    all three outputs come back; an unrelated job, a different n, or a job writing a buffer the
    group already uses starts a new group."""
    import torch
    ctx = m.ctx_init(2013265921)
    n = 1000
    u = lambda k=n: torch.zeros(k, dtype=torch.uint32)
    a, b, c, t, f, x, y = u(), u(), u(), u(), u(), u(), u()
    acc = torch.zeros(1, dtype=torch.int64)
    jobs = [m.host_job("mul_vec", ctx, c, a, b, acc=acc), m.host_job("to_mont", ctx, t, a),
            m.host_job("from_mont", ctx, f, t)]
    assert m.host_run_bytes(jobs) == (2 * 4 * n, 3 * 4 * n + 8)
    # an unrelated job over the same n: its own group (its input is uploaded)
    assert m.host_run_bytes(jobs + [m.host_job("to_mont", ctx, y, x)]) == (3 * 4 * n, 4 * 4 * n + 8)
    # writing a buffer the group reads: not fused, so a is uploaded again for it
    assert m.host_run_bytes(jobs + [m.host_job("to_mont", ctx, a, a)]) == (3 * 4 * n, 4 * 4 * n + 8)
    # a different n never fuses: the half-length from_mont uploads its input
    h = u(n // 2)
    assert m.host_run_bytes(jobs[:1] + [m.host_job("from_mont", ctx, h, u(n // 2))]) == (2 * 4 * n + 2 * n,
                                                                                         4 * n + 2 * n + 8)
    # twiddle: table once + rows; never fused
    tx, to, tw = torch.zeros((3, 64), dtype=torch.uint32), torch.zeros((3, 64), dtype=torch.uint32), u(64)
    assert m.host_run_bytes([m.host_job("twiddle", ctx, to, tx, tw)]) == (3 * 64 * 4 + 64 * 4, 3 * 64 * 4)
    # NTT rows: the (N - 1)-word table once, the rows up and back; never fused with others
    rows, rows_out, ttab = torch.zeros((5, 256), dtype=torch.uint32), torch.zeros((5, 256), dtype=torch.uint32), u(255)
    assert m.host_run_bytes([m.host_job("ntt", ctx, rows_out, rows, ttab)]) == (5 * 256 * 4 + 255 * 4, 5 * 256 * 4)
    with pytest.raises(m.MontError):  # not a power of two
        m.host_run_bytes([m.host_job("ntt", ctx, u(0).reshape(0, 0), torch.zeros((2, 96), dtype=torch.uint32),
                                     u(95))])
    # the same host buffer as both operands (a squaring) is uploaded once
    assert m.host_run_bytes([m.host_job("mul_vec", ctx, c, a, a)]) == (4 * n, 4 * n)
    with pytest.raises(m.MontError):
        m.host_run_bytes([m.host_job("from_mont", ctx, f, t, depends_on=0)])  # depends on itself


def _run_job(op, ctx, out, in0, in1=0, n=0, length=0, acc=0):
    j = m.RunJob()
    j.op, j.ctx, j.out, j.in0, j.in1, j.n, j.len, j.acc = op, C.pointer(ctx), out, in0, in1 or None, n, length, acc or None
    return j


def test_run_plan_bytes_and_validation():
    """mont_run's planner on the host (fake, never dereferenced device addresses): the fused
    to_mont -> from_mont pair is counted once (12 B/element instead of 16), and every dependency
    other than that pair is refused before any launch."""
    lib = m.lib()
    c0 = m.ctx_init(2013265921)
    c1 = m.ctx_init(469762049)
    MB = 1 << 20
    A, B, Cc, D, E, F, T = (0x10000000 + k * 64 * MB for k in range(7))
    n = 1 << 20
    acc = 0x7f000000

    def bytes_of(jobs):
        arr = (m.RunJob * len(jobs))(*jobs)
        b = C.c_ulonglong(0)
        st = lib.mont_run_bytes(arr, len(jobs), C.byref(b))
        return st, b.value

    mul = _run_job(0, c0, Cc, A, B, n, acc=acc)
    to = _run_job(1, c0, D, A, n=n)
    frm = _run_job(2, c0, E, D, n=n)
    tw = _run_job(3, c0, F, T, A, n=n, length=4096)
    st, b = bytes_of([mul, to, frm, tw])
    assert st == 0 and b == 12 * n + 12 * n + (8 * n + 4 * 4096)
    assert bytes_of([mul])[1] == 12 * n and bytes_of([frm])[1] == 8 * n
    # the chain with a different modulus is not a fused pair: a dependency -> refused
    frm1 = _run_job(2, c1, E, D, n=n)
    assert bytes_of([to, frm1])[0] == 2
    # FROM before its producer, overlapping outputs, a job reading another's output, partial aliasing
    assert bytes_of([frm, to])[0] == 2
    assert bytes_of([mul, _run_job(1, c0, Cc, A, n=n)])[0] == 2
    assert bytes_of([mul, _run_job(0, c0, D, Cc, B, n=n)])[0] == 2
    assert bytes_of([_run_job(1, c0, A + 16, A, n=n)])[0] == 2
    # in place is fine; n % 4, alignment, op, twiddle len, acc on a non-mul job, too many jobs
    assert bytes_of([_run_job(1, c0, A, A, n=n)])[0] == 0
    assert bytes_of([_run_job(1, c0, D, A, n=n + 2)])[0] == 2
    assert bytes_of([_run_job(1, c0, D + 4, A, n=n)])[0] == 2
    assert bytes_of([_run_job(7, c0, D, A, n=n)])[0] == 2
    assert bytes_of([_run_job(3, c0, F, T, A, n=n, length=3000)])[0] == 2
    assert bytes_of([_run_job(1, c0, D, A, n=n, acc=acc)])[0] == 2
    assert bytes_of([to] * 17)[0] == 2
    bad = m.Ctx()
    assert bytes_of([_run_job(1, bad, D, A, n=n)])[0] == 1
    assert bytes_of([])[0] == 0 and bytes_of([])[1] == 0


def test_binding_structs_match_headers():
    """The ctypes mirrors of the C structs list the same fields in the same order as the headers
    (mont_launch_t in include/mont_ext.h, mont_run_job_t in include/mont_run.h), and the flag value
    matches MONT_LAUNCH_OVERLAP_PREV."""
    root = Path(__file__).resolve().parents[1] / "include"

    def fields(header, name):
        txt = (root / header).read_text()
        body = re.search(r"typedef struct " + name + r" \{(.*?)\}", txt, re.S).group(1)
        return [re.findall(r"(\w+)\s*;", line)[0] for line in body.splitlines() if ";" in line and "(" not in line]

    assert fields("mont_ext.h", "mont_launch") == [f for f, _ in m.Launch._fields_]
    assert C.sizeof(m.Launch) == 4 * len(m.Launch._fields_)
    assert fields("mont_run.h", "mont_run_job") == [f for f, *_ in m.RunJob._fields_]
    flag = re.search(r"#define MONT_LAUNCH_OVERLAP_PREV (\d+)", (root / "mont_ext.h").read_text()).group(1)
    assert int(flag) == m.OVERLAP_PREV
