"""Known-answer pins (CPU): the oracle and the library's host-side context against values the
survey computed independently with Python big integers (tests/golden/survey_known_answers.json,
SURVEY.md Appendices A and B).  The GPU side of the same values: tests/test_gpu_known_answers.py."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_1609_00999_b200 as m
import synth

KA = json.loads((Path(__file__).resolve().parent / "golden" / "survey_known_answers.json").read_text())
GEN = json.loads((Path(__file__).resolve().parent / "golden" / "generator_kat.json").read_text())
PRIMES = [int(p) for p in KA["constants"]]


@pytest.mark.parametrize("P", PRIMES)
def test_constants_oracle_and_library(P):
    k = KA["constants"][str(P)]
    o = oracle.ctx(P)
    assert (o.Pprime, o.r1, o.r2, o.Rinv) == (k["Pprime"], k["r1"], k["r2"], k["Rinv"])
    c = m.ctx_init(P)                    # host-side Newton lift (no CUDA call)
    assert (c.pneg, c.r1, c.r2) == (k["Pprime"], k["r1"], k["r2"])
    assert (0x100000000 - c.pneg) % 0x100000000 == k["Pinv_mod_2_32"]
    assert P == k["c"] * 2 ** k["n"] + 1 and k["Pprime"] == P - 2          # Fourier closed form
    assert oracle.root_of_unity(P, k["g"], 1 << 14) == k["w"]
    assert int(oracle.to_mont(P, np.array([k["w"]], np.uint32))[0]) == k["to_mont_w"]


@pytest.mark.parametrize("P", PRIMES)
def test_mont_ab_first4(P):
    a = synth.uniform(42, 1, P, 0, 4)
    b = synth.uniform(42, 2, P, 0, 4)
    assert a.tolist() == GEN["uniform"][str(P)]["a"] and b.tolist() == GEN["uniform"][str(P)]["b"]
    assert oracle.mont_mul(P, a, b).tolist() == KA["mont_ab_first4"][str(P)]


def test_c1_end_to_end():
    k = KA["c1"]
    a, b = synth.c1_inputs(k["P"], n=k["n"])
    c = oracle.mont_mul(k["P"], a, b)
    assert oracle.checksum(k["P"], c) == k["checksum_mod_P"]
    assert c[:4].tolist() == k["c_first4"] and c[-2:].tolist() == k["c_last2"]


def test_c4_first4():
    k = KA["c4"]
    base, e = synth.c4_inputs(k["P"], 0, 4)
    assert oracle.power(k["P"], base, e).tolist() == k["out_first4"]


def test_c3_first4():
    k = KA["c3"]
    P, L = k["P"], k["len"]
    w = oracle.root_of_unity(P, KA["constants"][str(P)]["g"], L)
    tw = oracle.twiddle_table(P, w, L)
    assert tw[:4].tolist() == k["tw_first4"]
    x = synth.c3_x(P, batch=1, length=L)
    assert oracle.twiddle(P, x, tw)[0, :4].tolist() == k["out_row0_first4"]
