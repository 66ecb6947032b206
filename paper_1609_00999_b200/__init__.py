"""Batched 32-bit Montgomery modular multiplication on B200 (sm_100a).

Thin Python binding over the C ABI of ``libmont.so`` (include/mont.h,
include/mont_ext.h).  Argument marshalling only: every step of the path runs
in the library's CUDA kernels; torch supplies device memory, streams and the
process group.  There is no CPU fallback -- importing this package on a box
whose library is missing raises, and every launcher raises on a non-OK
status.

Paper: arxiv 1609.00999, "Automatic Generation of Vectorized Montgomery
Algorithm".  REDC(a, b) = a*b*R^-1 mod P, R = 2^32 (Alg. 2,
PAPER.md:95-99).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libmont.so"
if os.environ.get("MONT_LIB_AB"):  # measurement only: an A/B build of the same library (scripts/ab_build.sh)
    LIB_PATH = _HERE / "csrc" / "build_ab" / f"libmont_{os.environ['MONT_LIB_AB']}.so"

__all__ = [
    "Ctx", "MontError", "ctx_init", "to_mont", "from_mont", "mul_vec", "mul_vec_checksum", "mul_twiddle", "pow_vec",
    "checksum", "twiddle_table", "synth_fill", "Launch", "lib", "LIB_PATH",
]


class MontError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {_strerror(status)} (status {status})")


class Ctx(C.Structure):
    """mont_ctx_t: {p, pneg = -p^-1 mod 2^32, r1 = 2^32 mod p, r2 = 2^64 mod p}."""
    _fields_ = [("p", C.c_uint32), ("pneg", C.c_uint32), ("r1", C.c_uint32), ("r2", C.c_uint32)]

    def __repr__(self):
        return f"Ctx(p={self.p}, pneg={self.pneg}, r1={self.r1}, r2={self.r2})"


class Launch(C.Structure):
    """mont_launch_t (include/mont_ext.h); zero fields = library default."""
    _fields_ = [("threads", C.c_int), ("ctas_per_sm", C.c_int), ("unroll", C.c_int),
                ("variant", C.c_int), ("chunk", C.c_int), ("flags", C.c_int)]


OVERLAP_PREV = 1  # mont_launch_t.flags: MONT_LAUNCH_OVERLAP_PREV (include/mont_ext.h)


_lib = None
_P = C.c_void_p
_S = C.c_size_t
_CTX = C.POINTER(Ctx)
_LAUNCH = C.POINTER(Launch)

# name -> (restype, argtypes); mirrors include/mont.h and include/mont_ext.h
SIGNATURES = {
    "mont_ctx_init": (C.c_int, [_CTX, C.c_uint32]),
    "to_mont": (C.c_int, [_CTX, _P, _P, _S, _P]),
    "from_mont": (C.c_int, [_CTX, _P, _P, _S, _P]),
    "mont_mul_vec": (C.c_int, [_CTX, _P, _P, _P, _S, _P]),
    "mont_mul_twiddle": (C.c_int, [_CTX, _P, _P, _P, _S, _S, _P]),
    "mont_pow_vec": (C.c_int, [_CTX, _P, _P, _P, _S, _P]),
    "mont_checksum": (C.c_int, [_CTX, _P, _P, _S, _P]),
    "mont_twiddle_table": (C.c_int, [_CTX, _P, C.c_uint32, _S, _P]),
    "mont_mul_vec_checksum": (C.c_int, [_CTX, _P, _P, _P, _S, _P, _P]),
    "mont_mul_vec_checksum_ex": (C.c_int, [_CTX, _P, _P, _P, _S, _P, _LAUNCH, _P]),
    "to_mont_ex": (C.c_int, [_CTX, _P, _P, _S, _LAUNCH, _P]),
    "from_mont_ex": (C.c_int, [_CTX, _P, _P, _S, _LAUNCH, _P]),
    "mont_strerror": (C.c_char_p, [C.c_int]),
    "mont_build_arch": (C.c_int, []),
    "mont_mul_vec_ex": (C.c_int, [_CTX, _P, _P, _P, _S, _LAUNCH, _P]),
    "mont_mul_twiddle_ex": (C.c_int, [_CTX, _P, _P, _P, _S, _S, _LAUNCH, _P]),
    "mont_pow_vec_ex": (C.c_int, [_CTX, _P, _P, _P, _S, _LAUNCH, _P]),
    "synth_fill": (C.c_int, [_P, _S, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int, C.c_int, _P]),
    "mb_triad": (C.c_int, [_P, _P, _P, _S, _LAUNCH, _P]),
    "mb_copy": (C.c_int, [_P, _P, _S, _LAUNCH, _P]),
    "mb_imad": (C.c_int, [_P, C.c_int, C.c_int, _LAUNCH, _P, C.POINTER(C.c_ulonglong)]),
    "mb_pipe": (C.c_int, [_P, C.c_int, C.c_int, _LAUNCH, _P, C.POINTER(C.c_ulonglong), _P]),
    "mb_pipe_ops_per_iter": (C.c_int, [C.c_int]),
    "mb_sm_clock": (C.c_int, [_P, C.c_longlong, _P]),
    "mont_sm_count": (C.c_int, []),
    # include/mont_host.h
    "mont_host_min_workspace": (C.c_size_t, [C.c_int, C.c_size_t]),
    "mont_mul_vec_host": (C.c_int, [_CTX, _P, _P, _P, _S, _P, _P, _S, _P]),
    "to_mont_host": (C.c_int, [_CTX, _P, _P, _S, _P, _S, _P]),
    "from_mont_host": (C.c_int, [_CTX, _P, _P, _S, _P, _S, _P]),
    "mont_pow_vec_host": (C.c_int, [_CTX, _P, _P, _P, _S, _P, _S, _P]),
    "mont_mul_twiddle_host": (C.c_int, [_CTX, _P, _P, _P, _S, _S, _P, _S, _P]),
}

SIGNATURES["mont_ntt"] = (C.c_int, [_CTX, _P, _S, C.c_int, _P, C.c_uint32, _P])
SIGNATURES["mont_ntt_twiddles"] = (C.c_int, [_CTX, _P, C.c_uint32, C.c_int, _P])
SIGNATURES["mont_ntt_twiddles_pq"] = (C.c_int, [_CTX, _P, C.c_uint32, C.c_int, _P])
SIGNATURES["mont_ntt_ex"] = (C.c_int, [_CTX, _P, _S, C.c_int, _P, C.c_uint32, C.c_int, _P])
SIGNATURES["mont_dot"] = (C.c_int, [_CTX, _P, _P, _P, _S, _S, _P])
SIGNATURES["mont_dot_ex"] = (C.c_int, [_CTX, _P, _P, _P, _S, _S, _LAUNCH, _P])
SIGNATURES["mont_ntt_plan_words"] = (C.c_size_t, [C.c_int])
SIGNATURES["mont_ntt_plan_init"] = (C.c_int, [_CTX, _P, C.c_uint32, C.c_int, _P])
SIGNATURES["mont_ntt_large"] = (C.c_int, [_CTX, _P, _P, C.c_int, _P, C.c_uint32, _P])


class BarrettCtx(C.Structure):
    """barrett_ctx_t (include/barrett.h): k = ceil(log2 P), P' = floor(2^2k / P)."""
    _fields_ = [("p", C.c_uint32), ("k", C.c_uint32), ("pprime", C.c_uint32), ("pad", C.c_uint32)]


_BCTX = C.POINTER(BarrettCtx)
SIGNATURES.update({
    "barrett_ctx_init": (C.c_int, [_BCTX, C.c_uint32]),
    "barrett_mul_vec": (C.c_int, [_BCTX, _P, _P, _P, _S, _P]),
    "barrett_pow_vec": (C.c_int, [_BCTX, _P, _P, _P, _S, _P]),
})

HOST_OPS = {"mul_vec": 0, "to_mont": 1, "from_mont": 2, "pow_vec": 3, "twiddle": 4, "ntt": 5}


class HostJob(C.Structure):
    """mont_host_job_t (include/mont_host.h)."""
    _fields_ = [("op", C.c_int), ("ctx", _CTX), ("out", C.c_void_p), ("in0", C.c_void_p), ("in1", C.c_void_p),
                ("n", C.c_size_t), ("len", C.c_size_t), ("acc_host", C.c_void_p), ("depends_on", C.c_int),
                ("scale", C.c_uint32)]


SIGNATURES["mont_host_run"] = (C.c_int, [C.POINTER(HostJob), C.c_int, _P, _S, _P])

RUN_OPS = {"mul_vec": 0, "to_mont": 1, "from_mont": 2, "twiddle": 3}


class RunJob(C.Structure):
    """mont_run_job_t (include/mont_run.h)."""
    _fields_ = [("op", C.c_int), ("ctx", _CTX), ("out", C.c_void_p), ("in0", C.c_void_p), ("in1", C.c_void_p),
                ("n", C.c_size_t), ("len", C.c_size_t), ("acc", C.c_void_p)]


SIGNATURES["mont_run"] = (C.c_int, [C.POINTER(RunJob), C.c_int, _P])
SIGNATURES["mont_run_ex"] = (C.c_int, [C.POINTER(RunJob), C.c_int, _LAUNCH, _P])
SIGNATURES["mont_run_bytes"] = (C.c_int, [C.POINTER(RunJob), C.c_int, C.POINTER(C.c_ulonglong)])
SIGNATURES["mont_host_run_bytes"] = (C.c_int, [C.POINTER(HostJob), C.c_int, C.POINTER(C.c_ulonglong),
                                               C.POINTER(C.c_ulonglong)])


def lib():
    """Load libmont.so (built in-tree by __graft_entry__.build() / make)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _strerror(status: int) -> str:
    try:
        return lib().mont_strerror(status).decode()
    except Exception:  # pragma: no cover
        return "unknown"


def _check(status: int, where: str) -> None:
    if status != 0:
        raise MontError(status, where)


def ctx_init(p: int) -> Ctx:
    """Host-only Montgomery context (mont_ctx_init)."""
    c = Ctx()
    _check(lib().mont_ctx_init(C.byref(c), p), "mont_ctx_init")
    return c


# ------------------------------------------------------------ tensor helpers

def _torch():
    import torch
    return torch


def _stream_handle(stream) -> int:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def _dev_u32(t, name):
    torch = _torch()
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the library takes device pointers only)")
    if t.dtype not in (torch.uint32, torch.int32):
        raise TypeError(f"{name} must be uint32 (or int32 bit pattern), got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _out_like(out, ref, name="out"):
    torch = _torch()
    if out is None:
        return torch.empty_like(ref, dtype=torch.uint32)
    _dev_u32(out, name)
    if out.numel() != ref.numel():
        raise ValueError(f"{name} has {out.numel()} elements, expected {ref.numel()}")
    return out


def _ptr(t) -> int:
    return t.data_ptr()


def mul_vec(ctx: Ctx, a, b, out=None, stream=None, cfg: Launch | None = None):
    """c[i] = a[i] b[i] R^-1 mod P (mont_mul_vec)."""
    _dev_u32(a, "a"), _dev_u32(b, "b")
    if a.numel() != b.numel():
        raise ValueError("a and b differ in length")
    out = _out_like(out, a)
    s = _stream_handle(stream)
    if cfg is None:
        _check(lib().mont_mul_vec(C.byref(ctx), _ptr(out), _ptr(a), _ptr(b), a.numel(), s), "mont_mul_vec")
    else:
        _check(lib().mont_mul_vec_ex(C.byref(ctx), _ptr(out), _ptr(a), _ptr(b), a.numel(), C.byref(cfg), s),
               "mont_mul_vec_ex")
    return out


def mul_vec_checksum(ctx: Ctx, a, b, out=None, acc=None, stream=None, cfg: Launch | None = None):
    """c = mul_vec(a, b) and acc += sum(c) in one pass (mont_mul_vec_checksum); returns (c, acc)."""
    torch = _torch()
    _dev_u32(a, "a"), _dev_u32(b, "b")
    if a.numel() != b.numel():
        raise ValueError("a and b differ in length")
    out = _out_like(out, a)
    if acc is None:
        acc = torch.zeros(1, dtype=torch.int64, device=a.device)
    s = _stream_handle(stream)
    if cfg is None:
        _check(lib().mont_mul_vec_checksum(C.byref(ctx), _ptr(out), _ptr(a), _ptr(b), a.numel(), _ptr(acc), s),
               "mont_mul_vec_checksum")
    else:
        _check(lib().mont_mul_vec_checksum_ex(C.byref(ctx), _ptr(out), _ptr(a), _ptr(b), a.numel(), _ptr(acc),
                                              C.byref(cfg), s), "mont_mul_vec_checksum_ex")
    return out, acc


def to_mont(ctx: Ctx, x, out=None, stream=None, cfg: Launch | None = None):
    _dev_u32(x, "x")
    out = _out_like(out, x)
    s = _stream_handle(stream)
    if cfg is None:
        _check(lib().to_mont(C.byref(ctx), _ptr(out), _ptr(x), x.numel(), s), "to_mont")
    else:
        _check(lib().to_mont_ex(C.byref(ctx), _ptr(out), _ptr(x), x.numel(), C.byref(cfg), s), "to_mont_ex")
    return out


def from_mont(ctx: Ctx, x, out=None, stream=None, cfg: Launch | None = None):
    _dev_u32(x, "x")
    out = _out_like(out, x)
    s = _stream_handle(stream)
    if cfg is None:
        _check(lib().from_mont(C.byref(ctx), _ptr(out), _ptr(x), x.numel(), s), "from_mont")
    else:
        _check(lib().from_mont_ex(C.byref(ctx), _ptr(out), _ptr(x), x.numel(), C.byref(cfg), s), "from_mont_ex")
    return out


def mul_twiddle(ctx: Ctx, x, tw, out=None, stream=None, cfg: Launch | None = None):
    """out[r][j] = x[r][j] tw[j] R^-1 mod P for x of shape (batch, len)."""
    _dev_u32(x, "x"), _dev_u32(tw, "tw")
    if x.dim() != 2 or tw.dim() != 1 or x.shape[1] != tw.shape[0]:
        raise ValueError("x must be (batch, len) and tw (len,)")
    out = _out_like(out, x)
    batch, length = x.shape
    s = _stream_handle(stream)
    if cfg is None:
        _check(lib().mont_mul_twiddle(C.byref(ctx), _ptr(out), _ptr(x), _ptr(tw), batch, length, s),
               "mont_mul_twiddle")
    else:
        _check(lib().mont_mul_twiddle_ex(C.byref(ctx), _ptr(out), _ptr(x), _ptr(tw), batch, length,
                                         C.byref(cfg), s), "mont_mul_twiddle_ex")
    return out


def pow_vec(ctx: Ctx, base, exp, out=None, stream=None, cfg: Launch | None = None):
    """out[i] = base[i]^exp[i] mod P, plain in/out (mont_pow_vec)."""
    _dev_u32(base, "base"), _dev_u32(exp, "exp")
    if base.numel() != exp.numel():
        raise ValueError("base and exp differ in length")
    out = _out_like(out, base)
    s = _stream_handle(stream)
    if cfg is None:
        _check(lib().mont_pow_vec(C.byref(ctx), _ptr(out), _ptr(base), _ptr(exp), base.numel(), s),
               "mont_pow_vec")
    else:
        _check(lib().mont_pow_vec_ex(C.byref(ctx), _ptr(out), _ptr(base), _ptr(exp), base.numel(),
                                     C.byref(cfg), s), "mont_pow_vec_ex")
    return out


def checksum(ctx: Ctx, x, acc=None, stream=None):
    """Adds sum(x) into the int64 device scalar `acc` (created zeroed if None); returns acc."""
    torch = _torch()
    _dev_u32(x, "x")
    if acc is None:
        acc = torch.zeros(1, dtype=torch.int64, device=x.device)
    _check(lib().mont_checksum(C.byref(ctx), _ptr(acc), _ptr(x), x.numel(), _stream_handle(stream)),
           "mont_checksum")
    return acc


def twiddle_table(ctx: Ctx, w: int, length: int, device="cuda", out=None, stream=None):
    """tw[j] = to_mont(w^j mod P) on the GPU (mont_twiddle_table)."""
    torch = _torch()
    if out is None:
        out = torch.empty(length, dtype=torch.uint32, device=device)
    _dev_u32(out, "out")
    _check(lib().mont_twiddle_table(C.byref(ctx), _ptr(out), w, length, _stream_handle(stream)),
           "mont_twiddle_table")
    return out


def synth_fill(out, seed: int, stream_id: int, start: int, p: int, mode: int = 0, specials: bool = False,
               stream=None):
    """Device side of synth/: counter-based inputs straight into HBM (include/mont_ext.h)."""
    _dev_u32(out, "out")
    _check(lib().synth_fill(_ptr(out), out.numel(), seed, stream_id, start, p, mode, int(bool(specials)),
                            _stream_handle(stream)), "synth_fill")
    return out


# ----------------------------------------------------- host-buffer forms (e2e)

def _host_u32(t, name):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or t.is_cuda:
        raise TypeError(f"{name} must be a CPU (ideally pinned) torch tensor")
    if t.dtype not in (torch.uint32, torch.int32) or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous uint32 CPU tensor")
    return t


def host_workspace(op: str, length: int = 0, min_bytes: int = 256 << 20, device="cuda"):
    """A device workspace for the host-buffer forms (include/mont_host.h)."""
    torch = _torch()
    need = int(lib().mont_host_min_workspace(HOST_OPS[op], length))
    return torch.empty(max(need, min_bytes), dtype=torch.uint8, device=device)


def mul_vec_host(ctx: Ctx, a, b, out, ws, want_checksum: bool = False, stream=None):
    """out = REDC(a, b) for HOST tensors, streamed through device workspace `ws`.
    Returns a pinned int64 scalar tensor holding sum(out) if want_checksum (valid after sync)."""
    torch = _torch()
    for t, nme in ((a, "a"), (b, "b"), (out, "out")):
        _host_u32(t, nme)
    if not (a.numel() == b.numel() == out.numel()):
        raise ValueError("length mismatch")
    acc = torch.zeros(1, dtype=torch.int64, pin_memory=True) if want_checksum else None
    _check(lib().mont_mul_vec_host(C.byref(ctx), _ptr(out), _ptr(a), _ptr(b), a.numel(),
                                   _ptr(acc) if acc is not None else None, _ptr(ws), ws.numel(),
                                   _stream_handle(stream)), "mont_mul_vec_host")
    return acc


def to_mont_host(ctx: Ctx, x, out, ws, stream=None):
    _host_u32(x, "x"), _host_u32(out, "out")
    _check(lib().to_mont_host(C.byref(ctx), _ptr(out), _ptr(x), x.numel(), _ptr(ws), ws.numel(),
                              _stream_handle(stream)), "to_mont_host")


def from_mont_host(ctx: Ctx, x, out, ws, stream=None):
    _host_u32(x, "x"), _host_u32(out, "out")
    _check(lib().from_mont_host(C.byref(ctx), _ptr(out), _ptr(x), x.numel(), _ptr(ws), ws.numel(),
                                _stream_handle(stream)), "from_mont_host")


def pow_vec_host(ctx: Ctx, base, exp, out, ws, stream=None):
    _host_u32(base, "base"), _host_u32(exp, "exp"), _host_u32(out, "out")
    _check(lib().mont_pow_vec_host(C.byref(ctx), _ptr(out), _ptr(base), _ptr(exp), base.numel(), _ptr(ws),
                                   ws.numel(), _stream_handle(stream)), "mont_pow_vec_host")


def mul_twiddle_host(ctx: Ctx, x, tw, out, ws, stream=None):
    _host_u32(x, "x"), _host_u32(tw, "tw"), _host_u32(out, "out")
    batch, length = x.shape
    _check(lib().mont_mul_twiddle_host(C.byref(ctx), _ptr(out), _ptr(x), _ptr(tw), batch, length, _ptr(ws),
                                       ws.numel(), _stream_handle(stream)), "mont_mul_twiddle_host")


def ntt_twiddles(ctx: Ctx, w: int, log_n: int, device="cuda", stream=None):
    """Stage-major NTT twiddle table (N - 1 Montgomery-form words) for mont_ntt."""
    torch = _torch()
    tw = torch.empty((1 << log_n) - 1, dtype=torch.uint32, device=device)
    _check(lib().mont_ntt_twiddles(C.byref(ctx), _ptr(tw), w, log_n, _stream_handle(stream)), "mont_ntt_twiddles")
    return tw


def ntt_twiddles_pq(ctx: Ctx, w: int, log_n: int, device="cuda", stream=None):
    """Pair table (plain w^x, floor(w^x 2^32 / P)) x (N - 1) for mont_ntt_ex variant 3."""
    torch = _torch()
    tw2 = torch.empty(2 * ((1 << log_n) - 1), dtype=torch.uint32, device=device)
    _check(lib().mont_ntt_twiddles_pq(C.byref(ctx), _ptr(tw2), w, log_n, _stream_handle(stream)),
           "mont_ntt_twiddles_pq")
    return tw2


def ntt(ctx: Ctx, data, tw, scale: int | None = None, stream=None, variant: int | None = None):
    """In-place batched NTT of the rows of `data` (batch, N), N = 2^k <= 32768 (include/mont_ntt.h).
    tw: stage-major table from ntt_twiddles(); scale: Montgomery form of the output factor."""
    _dev_u32(data, "data"), _dev_u32(tw, "tw")
    if data.dim() != 2:
        raise ValueError("data must be (batch, N)")
    batch, n = data.shape
    log_n = n.bit_length() - 1
    if n != 1 << log_n or tw.numel() < n - 1:
        raise ValueError("N must be a power of two and tw must hold the N-1 stage-major twiddles")
    sc = ctx.r1 if scale is None else scale
    if variant is None:
        _check(lib().mont_ntt(C.byref(ctx), _ptr(data), batch, log_n, _ptr(tw), sc, _stream_handle(stream)),
               "mont_ntt")
    else:
        _check(lib().mont_ntt_ex(C.byref(ctx), _ptr(data), batch, log_n, _ptr(tw), sc, variant,
                                 _stream_handle(stream)), "mont_ntt_ex")
    return data


def ntt_plan(ctx: Ctx, w: int, log_n: int, device="cuda", stream=None):
    """Device plan (tables) for mont_ntt_large of size 2^log_n, 16 <= log_n <= 30."""
    torch = _torch()
    words = int(lib().mont_ntt_plan_words(log_n))
    if words == 0:
        raise ValueError("log_n must be in [16, 30]")
    plan = torch.empty(words, dtype=torch.uint32, device=device)
    _check(lib().mont_ntt_plan_init(C.byref(ctx), _ptr(plan), w, log_n, _stream_handle(stream)), "mont_ntt_plan_init")
    return plan


def ntt_large(ctx: Ctx, x, plan, out=None, scale: int | None = None, stream=None):
    """Natural-order NTT of one vector of 2^k (16 <= k <= 30) words; x is destroyed (scratch)."""
    _dev_u32(x, "x"), _dev_u32(plan, "plan")
    n = x.numel()
    log_n = n.bit_length() - 1
    if n != 1 << log_n:
        raise ValueError("length must be a power of two")
    out = _out_like(out, x)
    _check(lib().mont_ntt_large(C.byref(ctx), _ptr(out), _ptr(x), log_n, _ptr(plan),
                                ctx.r1 if scale is None else scale, _stream_handle(stream)), "mont_ntt_large")
    return out


def dot(ctx: Ctx, A, x, out=None, stream=None, cfg: Launch | None = None):
    """out[r] = sum_j A[r][j] x[j] R^-1 mod P for A (batch, len) (include/mont_dot.h)."""
    torch = _torch()
    _dev_u32(A, "A"), _dev_u32(x, "x")
    if A.dim() != 2 or x.dim() != 1 or A.shape[1] != x.shape[0]:
        raise ValueError("A must be (batch, len) and x (len,)")
    if out is None:
        out = torch.empty(A.shape[0], dtype=torch.uint32, device=A.device)
    if cfg is None:
        _check(lib().mont_dot(C.byref(ctx), _ptr(out), _ptr(A), _ptr(x), A.shape[0], A.shape[1],
                              _stream_handle(stream)), "mont_dot")
    else:
        _check(lib().mont_dot_ex(C.byref(ctx), _ptr(out), _ptr(A), _ptr(x), A.shape[0], A.shape[1], C.byref(cfg),
                                 _stream_handle(stream)), "mont_dot_ex")
    return out


def barrett_ctx_init(p: int) -> BarrettCtx:
    c = BarrettCtx()
    _check(lib().barrett_ctx_init(C.byref(c), p), "barrett_ctx_init")
    return c


def barrett_mul_vec(ctx: BarrettCtx, a, b, out=None, stream=None):
    """c = a b mod P, plain domain, Barrett's Alg. 1 (comparison kernel, include/barrett.h)."""
    _dev_u32(a, "a"), _dev_u32(b, "b")
    out = _out_like(out, a)
    _check(lib().barrett_mul_vec(C.byref(ctx), _ptr(out), _ptr(a), _ptr(b), a.numel(), _stream_handle(stream)),
           "barrett_mul_vec")
    return out


def barrett_pow_vec(ctx: BarrettCtx, base, exp, out=None, stream=None):
    _dev_u32(base, "base"), _dev_u32(exp, "exp")
    out = _out_like(out, base)
    _check(lib().barrett_pow_vec(C.byref(ctx), _ptr(out), _ptr(base), _ptr(exp), base.numel(),
                                 _stream_handle(stream)), "barrett_pow_vec")
    return out


def host_job(op: str, ctx: Ctx, out, in0, in1=None, acc=None, depends_on: int = -1, scale: int = 0) -> HostJob:
    """Describe one operation on HOST tensors for host_run(); twiddle: in0 = x (batch, len), in1 = tw;
    ntt: in0 = rows (batch, N), in1 = the (N - 1)-word mont_ntt_twiddles table (a host copy), scale = the
    Montgomery-form output factor (0: none)."""
    j = HostJob()
    j.op = HOST_OPS[op]
    j.ctx = C.pointer(ctx)
    j.out, j.in0 = _ptr(_host_u32(out, "out")), _ptr(_host_u32(in0, "in0"))
    j.in1 = _ptr(_host_u32(in1, "in1")) if in1 is not None else None
    if op in ("twiddle", "ntt"):
        j.n, j.len = in0.shape[0], in0.shape[1]
    else:
        j.n, j.len = in0.numel(), 0
    j.scale = int(scale)
    j.acc_host = _ptr(acc) if acc is not None else None
    j.depends_on = int(depends_on)
    j._keep = (ctx, out, in0, in1, acc)  # keep the referenced objects alive
    return j


def run_job(op: str, ctx: Ctx, out, in0, in1=None, acc=None) -> RunJob:
    """Describe one operation on DEVICE tensors for run() (include/mont_run.h); twiddle: in0 = x
    (batch, len) or flat with in1 = the len-word table; mul_vec: acc = optional int64 tensor (1,)."""
    j = RunJob()
    j.op = RUN_OPS[op]
    j.ctx = C.pointer(ctx)
    j.out, j.in0 = _ptr(_dev_u32(out, "out")), _ptr(_dev_u32(in0, "in0"))
    j.in1 = _ptr(_dev_u32(in1, "in1")) if in1 is not None else None
    j.n = in0.numel()
    j.len = in1.numel() if op == "twiddle" else 0
    j.acc = _ptr(acc) if acc is not None else None
    j._keep = (ctx, out, in0, in1, acc)
    return j


def run(jobs, stream=None, cfg: Launch | None = None):
    """Run the jobs as one launch (mont_run): independent HBM-bound operations back to back in one
    flat grid; a from_mont reading an earlier to_mont's output is fused into it."""
    arr = (RunJob * len(jobs))(*jobs)
    if cfg is None:
        _check(lib().mont_run(arr, len(jobs), _stream_handle(stream)), "mont_run")
    else:
        _check(lib().mont_run_ex(arr, len(jobs), C.byref(cfg), _stream_handle(stream)), "mont_run_ex")


def run_bytes(jobs) -> int:
    arr = (RunJob * len(jobs))(*jobs)
    b = C.c_ulonglong(0)
    _check(lib().mont_run_bytes(arr, len(jobs), C.byref(b)), "mont_run_bytes")
    return int(b.value)


def host_run(jobs, ws, stream=None):
    """Stream all jobs' chunks through one H2D / kernel / D2H ring (mont_host_run)."""
    arr = (HostJob * len(jobs))(*jobs)
    _check(lib().mont_host_run(arr, len(jobs), _ptr(ws), ws.numel(), _stream_handle(stream)), "mont_host_run")


def host_run_bytes(jobs):
    """(h2d_bytes, d2h_bytes) that host_run(jobs, ...) copies, after fusion (mont_host_run_bytes)."""
    arr = (HostJob * len(jobs))(*jobs)
    h2d, d2h = C.c_ulonglong(0), C.c_ulonglong(0)
    _check(lib().mont_host_run_bytes(arr, len(jobs), C.byref(h2d), C.byref(d2h)), "mont_host_run_bytes")
    return int(h2d.value), int(d2h.value)


def sm_count() -> int:
    return int(lib().mont_sm_count())


if os.environ.get("MONT_EAGER_LOAD", "1") == "1":
    lib()
