"""Mutation check of the oracle's pins: each plausible mistake below (a dropped term, a wrong
sign or index, an off-by-one) is compiled into a copy of oracle/oracle.c, and the pin suite
tests/test_oracle.py must FAIL against it.  This is what makes the pins evidence: they are
chosen so that a mistake anywhere in the oracle is caught by something other than the oracle."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SRC = (ROOT / "oracle" / "oracle.c").read_text()

MUTANTS = {
    "mont_mul drops R^-1": ("return mulmod_naive(mulmod_naive(a, b, c->P), c->Rinv, c->P);",
                            "return mulmod_naive(a, b, c->P);"),
    "r1 off by one": ("c->r1 = (uint32_t)(R % P);", "c->r1 = (uint32_t)((R + 1) % P);"),
    "P' off by one": ("c->Pprime = (uint32_t)(num / P);", "c->Pprime = (uint32_t)(num / P + 1);"),
    "to_mont shift": ("return (uint32_t)((((uint64_t)x % c->P) << c->l) % c->P);",
                      "return (uint32_t)((((uint64_t)x % c->P) << (c->l - 1)) % c->P);"),
    "from_mont uses P'": ("return mulmod_naive(x % c->P, c->Rinv, c->P);",
                          "return mulmod_naive(x % c->P, c->Pprime % c->P, c->P);"),
    "pow drops bit 31": ("for (int bit = 31; bit >= 0; --bit) {\n        acc = mulmod_naive(acc, acc, P);\n"
                         "        if ((exp >> bit) & 1u) acc = mulmod_naive(acc, x, P);",
                         "for (int bit = 30; bit >= 0; --bit) {\n        acc = mulmod_naive(acc, acc, P);\n"
                         "        if ((exp >> bit) & 1u) acc = mulmod_naive(acc, x, P);"),
    "pow misses bit 30": ("for (int bit = 31; bit >= 0; --bit) {\n        acc = mulmod_naive(acc, acc, P);\n"
                          "        if ((exp >> bit) & 1u) acc = mulmod_naive(acc, x, P);",
                          "for (int bit = 31; bit >= 0; --bit) {\n        if (bit == 30) continue;\n"
                          "        acc = mulmod_naive(acc, acc, P);\n"
                          "        if ((exp >> bit) & 1u) acc = mulmod_naive(acc, x, P);"),
    "pow multiply before square": ("        acc = mulmod_naive(acc, acc, P);\n        if ((exp >> bit) & 1u) acc = mulmod_naive(acc, x, P);\n    }\n    return acc;\n}\n\n/* -",
                                   "        if ((exp >> bit) & 1u) acc = mulmod_naive(acc, x, P);\n        acc = mulmod_naive(acc, acc, P);\n    }\n    return acc;\n}\n\n/* -"),
    "twiddle column shifted": ("j->out[i] = oracle_mont_mul1(c, j->a[i], j->b[i % j->len]);",
                               "j->out[i] = oracle_mont_mul1(c, j->a[i], j->b[(i + 1) % j->len]);"),
    "checksum drops last": ("for (i = j->lo; i < j->hi; ++i) s += j->a[i];", "for (i = j->lo; i + 1 < j->hi; ++i) s += j->a[i];"),
    "table power off by one": ("        tw[j] = oracle_to_mont1(c, wj);\n        wj = mulmod_naive(wj, w, c->P);",
                               "        wj = mulmod_naive(wj, w, c->P);\n        tw[j] = oracle_to_mont1(c, wj);"),
    "dft exponent off": ("s += mulmod_naive(x[j] % P, pw[(j * k) % N], P);", "s += mulmod_naive(x[j] % P, pw[(j * k + j) % N], P);"),
    "conv index sign": ("s += mulmod_naive(a[j] % P, b[(k + N - j) % N] % P, P);", "s += mulmod_naive(a[j] % P, b[(k + j) % N] % P, P);"),
    "root exponent off": ("uint32_t e = (P - 1u) / order;", "uint32_t e = (P - 1u) / order + 1u;"),
    "barrett extra shift": ("uint64_t q = (m * c->bPprime) >> c->bk;", "uint64_t q = (m * c->bPprime) >> (c->bk + 1);"),
    "fourier sign": ("int64_t t = (int64_t)q1 - (int64_t)q2 + (int64_t)q3;", "int64_t t = (int64_t)q1 + (int64_t)q2 - (int64_t)q3;"),
}


@pytest.mark.parametrize("name", sorted(MUTANTS))
def test_pins_catch_mutant(name, tmp_path):
    old, new = MUTANTS[name]
    assert SRC.count(old) == 1, f"mutation anchor not found uniquely: {name}"
    src = tmp_path / "oracle_mutant.c"
    src.write_text(SRC.replace(old, new))
    so = tmp_path / "liboracle_mutant.so"
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread", "-o", str(so), str(src)])
    env = dict(os.environ, ORACLE_LIB_OVERRIDE=str(so))
    r = subprocess.run([sys.executable, "-m", "pytest", str(ROOT / "tests" / "test_oracle.py"), "-x", "-q",
                        "-p", "no:cacheprovider"], env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode != 0, f"pins did not catch mutant '{name}'"
