"""CPU oracle for the batched 32-bit Montgomery multiplication path (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product library
(paper_1609_00999_b200) never imports it, and it imports nothing from the
product: it is a thin ctypes/numpy wrapper around oracle/oracle.c, which
computes the plain definitions with 64-bit naive '%' (see the header of
oracle.c for the passage each function follows).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "oracle.c"
_LIB = _HERE / "liboracle.so"


def build(force: bool = False) -> Path:
    """Compile oracle.c with gcc (plain -O2, no target-specific tuning)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".{os.getpid()}.tmp.so")
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread",
                               "-o", str(tmp), str(_SRC)])
        os.replace(tmp, _LIB)
    return _LIB


class Ctx(C.Structure):
    _fields_ = [("P", C.c_uint32), ("l", C.c_uint32), ("R", C.c_uint64), ("Rinv", C.c_uint32),
                ("Pprime", C.c_uint32), ("r1", C.c_uint32), ("r2", C.c_uint32),
                ("bk", C.c_uint32), ("bPprime", C.c_uint64)]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


_lib = None
_U32P = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")


def lib():
    global _lib
    if _lib is None:
        # test hook: tests/test_oracle_mutants.py points this at deliberately broken builds
        override = os.environ.get("ORACLE_LIB_OVERRIDE")
        L = C.CDLL(override if override else str(build()))
        L.oracle_ctx_l.argtypes = [C.POINTER(Ctx), C.c_uint32, C.c_uint32]
        L.oracle_ctx_l.restype = C.c_int
        L.oracle_mulmod.argtypes = [C.c_uint32] * 3
        L.oracle_mulmod.restype = C.c_uint32
        for name in ("oracle_mont_mul1",):
            getattr(L, name).argtypes = [C.POINTER(Ctx), C.c_uint32, C.c_uint32]
            getattr(L, name).restype = C.c_uint32
        for name in ("oracle_to_mont1", "oracle_from_mont1"):
            getattr(L, name).argtypes = [C.POINTER(Ctx), C.c_uint32]
            getattr(L, name).restype = C.c_uint32
        L.oracle_pow1.argtypes = [C.c_uint32] * 3
        L.oracle_pow1.restype = C.c_uint32
        L.oracle_mont_mul.argtypes = [C.POINTER(Ctx), _U32P, _U32P, _U32P, C.c_size_t, C.c_int]
        L.oracle_to_mont.argtypes = [C.POINTER(Ctx), _U32P, _U32P, C.c_size_t, C.c_int]
        L.oracle_mulmod_vec.argtypes = [C.POINTER(Ctx), _U32P, _U32P, _U32P, C.c_size_t, C.c_int]
        L.oracle_from_mont.argtypes = [C.POINTER(Ctx), _U32P, _U32P, C.c_size_t, C.c_int]
        L.oracle_twiddle.argtypes = [C.POINTER(Ctx), _U32P, _U32P, _U32P, C.c_size_t, C.c_size_t, C.c_int]
        L.oracle_pow.argtypes = [C.POINTER(Ctx), _U32P, _U32P, _U32P, C.c_size_t, C.c_int]
        L.oracle_sum.argtypes = [_U32P, C.c_size_t, C.c_int]
        L.oracle_sum.restype = C.c_uint64
        L.oracle_checksum.argtypes = [C.POINTER(Ctx), _U32P, C.c_size_t, C.c_int]
        L.oracle_checksum.restype = C.c_uint32
        L.oracle_root_of_unity.argtypes = [C.c_uint32] * 3
        L.oracle_root_of_unity.restype = C.c_uint32
        L.oracle_twiddle_table.argtypes = [C.POINTER(Ctx), _U32P, C.c_uint32, C.c_size_t]
        L.oracle_redc_l.argtypes = [C.POINTER(Ctx), C.c_uint64, C.POINTER(C.c_uint32)]
        L.oracle_redc_l.restype = C.c_uint32
        L.oracle_barrett.argtypes = [C.POINTER(Ctx), C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32)]
        L.oracle_barrett.restype = C.c_uint32
        L.oracle_fourier_redc.argtypes = [C.POINTER(Ctx), C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.POINTER(C.c_int64), C.POINTER(C.c_uint64)]
        L.oracle_fourier_redc.restype = C.c_uint32
        L.oracle_dft.argtypes = [C.c_uint32, C.c_uint32, _U32P, _U32P, C.c_size_t]
        L.oracle_cyclic_conv.argtypes = [C.c_uint32, _U32P, _U32P, _U32P, C.c_size_t]
        L.oracle_dot.argtypes = [C.POINTER(Ctx), _U32P, _U32P, _U32P, C.c_size_t, C.c_size_t]
        L.oracle_dft_at.argtypes = [C.c_uint32, C.c_uint32, _U32P, C.c_size_t, C.c_size_t]
        L.oracle_dft_at.restype = C.c_uint32
        L.oracle_inverse.argtypes = [C.c_uint32, C.c_uint32]
        L.oracle_inverse.restype = C.c_uint32
        L.oracle_mod_add.argtypes = [C.c_uint32] * 3
        L.oracle_mod_add.restype = C.c_uint32
        L.oracle_mod_sub.argtypes = [C.c_uint32] * 3
        L.oracle_mod_sub.restype = C.c_uint32
        _lib = L
    return _lib


class OracleError(ValueError):
    pass


def ctx(P: int, l: int = 32) -> Ctx:
    """Montgomery context by extended Euclid. Raises for invalid P."""
    c = Ctx()
    if lib().oracle_ctx_l(C.byref(c), P, l) != 0:
        raise OracleError(f"invalid modulus P={P} for l={l}")
    return c


def _u32(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.uint32)


def mont_mul(P: int, a, b, nthreads: int = 0) -> np.ndarray:
    """c[i] = a[i] b[i] R^-1 mod P."""
    a, b = _u32(a), _u32(b)
    assert a.shape == b.shape
    out = np.empty_like(a)
    c = ctx(P)
    lib().oracle_mont_mul(C.byref(c), out.reshape(-1), a.reshape(-1), b.reshape(-1), a.size, nthreads)
    return out


def mulmod_vec(P: int, a, b, nthreads: int = 0) -> np.ndarray:
    """c[i] = a[i] b[i] mod P (plain), by definition."""
    a, b = _u32(a), _u32(b)
    out = np.empty_like(a)
    c = ctx(P)
    lib().oracle_mulmod_vec(C.byref(c), out.reshape(-1), a.reshape(-1), b.reshape(-1), a.size, nthreads)
    return out


def to_mont(P: int, x, nthreads: int = 0) -> np.ndarray:
    x = _u32(x)
    out = np.empty_like(x)
    c = ctx(P)
    lib().oracle_to_mont(C.byref(c), out.reshape(-1), x.reshape(-1), x.size, nthreads)
    return out


def from_mont(P: int, x, nthreads: int = 0) -> np.ndarray:
    x = _u32(x)
    out = np.empty_like(x)
    c = ctx(P)
    lib().oracle_from_mont(C.byref(c), out.reshape(-1), x.reshape(-1), x.size, nthreads)
    return out


def twiddle(P: int, x, tw, nthreads: int = 0) -> np.ndarray:
    """out[r][j] = x[r][j] tw[j] R^-1 mod P for x of shape (batch, len)."""
    x, tw = _u32(x), _u32(tw)
    batch, length = x.shape
    assert tw.shape == (length,)
    out = np.empty_like(x)
    c = ctx(P)
    lib().oracle_twiddle(C.byref(c), out.reshape(-1), x.reshape(-1), tw, batch, length, nthreads)
    return out


def power(P: int, base, exp, nthreads: int = 0) -> np.ndarray:
    """out[i] = base[i]^exp[i] mod P, plain in/out (BASELINE configs[3])."""
    base, exp = _u32(base), _u32(exp)
    assert base.shape == exp.shape
    out = np.empty_like(base)
    c = ctx(P)
    lib().oracle_pow(C.byref(c), out.reshape(-1), base.reshape(-1), exp.reshape(-1), base.size, nthreads)
    return out


def checksum(P: int, x, nthreads: int = 0) -> int:
    """(sum x) mod P (BASELINE configs[4])."""
    x = _u32(x).reshape(-1)
    return int(lib().oracle_sum(x, x.size, nthreads)) % P


def raw_sum(x, nthreads: int = 0) -> int:
    x = _u32(x).reshape(-1)
    return int(lib().oracle_sum(x, x.size, nthreads))


def root_of_unity(P: int, g: int, order: int) -> int:
    return int(lib().oracle_root_of_unity(P, g, order))


def twiddle_table(P: int, w: int, length: int) -> np.ndarray:
    """tw[j] = to_mont(w^j mod P) (BASELINE configs[2])."""
    tw = np.empty(length, dtype=np.uint32)
    c = ctx(P)
    lib().oracle_twiddle_table(C.byref(c), tw, w, length)
    return tw


# scalar forms -------------------------------------------------------------

def mulmod(a: int, b: int, P: int) -> int:
    return int(lib().oracle_mulmod(a, b, P))


def mont_mul1(P: int, a: int, b: int, l: int = 32) -> int:
    c = ctx(P, l)
    return int(lib().oracle_mont_mul1(C.byref(c), a, b))


def pow1(P: int, base: int, exp: int) -> int:
    return int(lib().oracle_pow1(P, base, exp))


def redc_l(P: int, l: int, T: int):
    """Alg. 2 step by step with R = 2^l; returns (t, flags)."""
    c = ctx(P, l)
    f = C.c_uint32(0)
    t = lib().oracle_redc_l(C.byref(c), T, C.byref(f))
    return int(t), int(f.value)


def barrett(P: int, a: int, b: int):
    """Alg. 1; returns (ab mod P, while-loop trips)."""
    c = ctx(P, 32)
    n = C.c_uint32(0)
    t = lib().oracle_barrett(C.byref(c), a, b, C.byref(n))
    return int(t), int(n.value)


def fourier_redc(P: int, l: int, cc: int, n: int, a: int, b: int):
    """Alg. 3; returns (t, t_raw, r3)."""
    c = ctx(P, l)
    traw = C.c_int64(0)
    r3 = C.c_uint64(0)
    t = lib().oracle_fourier_redc(C.byref(c), cc, n, a, b, C.byref(traw), C.byref(r3))
    return int(t), int(traw.value), int(r3.value)


def mod_add(a: int, b: int, P: int) -> int:
    return int(lib().oracle_mod_add(a, b, P))


def mod_sub(a: int, b: int, P: int) -> int:
    return int(lib().oracle_mod_sub(a, b, P))


# NTT by definition -----------------------------------

def dft(P: int, w: int, x) -> np.ndarray:
    """X[k] = sum_j x[j] w^(jk) mod P for each row of x (O(N^2) per row).  Rows run on a thread
    pool (ctypes releases the GIL in the C call): slicing only, the arithmetic is oracle_dft's."""
    from concurrent.futures import ThreadPoolExecutor
    x = _u32(x)
    rows = np.ascontiguousarray(x.reshape(-1, x.shape[-1]))
    out = np.empty_like(rows)
    L = lib()

    def one(r):
        L.oracle_dft(P, w, rows[r], out[r], rows.shape[1])

    if rows.shape[0] == 1:
        one(0)
    else:
        with ThreadPoolExecutor(max_workers=min(rows.shape[0], os.cpu_count() or 1)) as ex:
            list(ex.map(one, range(rows.shape[0])))
    return out.reshape(x.shape)


def cyclic_conv(P: int, a, b) -> np.ndarray:
    a, b = _u32(a), _u32(b)
    out = np.empty_like(a)
    lib().oracle_cyclic_conv(P, a, b, out, a.size)
    return out


def inverse(x: int, P: int) -> int:
    return int(lib().oracle_inverse(x, P))


def dot(P: int, A, x) -> np.ndarray:
    """out[r] = sum_j A[r][j] x[j] R^-1 mod P (NEXT #4), by definition."""
    A, x = _u32(A), _u32(x)
    batch, length = A.shape
    out = np.empty(batch, dtype=np.uint32)
    c = ctx(P)
    lib().oracle_dot(C.byref(c), out, A.reshape(-1), x, batch, length)
    return out


def dft_at(P: int, w: int, x, k: int) -> int:
    """X[k] = sum_j x[j] w^(jk) mod P, one output by definition (O(N))."""
    x = _u32(x).reshape(-1)
    return int(lib().oracle_dft_at(P, w, x, x.size, k))
