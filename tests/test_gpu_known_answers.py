"""Known-answer pins on the GPU (SURVEY.md Appendices A and B, tests/golden/
survey_known_answers.json): every hot-path kernel reproduces the survey's independently computed
values, in the default launch and in every variant that computes the same function."""
import json
from pathlib import Path

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

KA = json.loads((Path(__file__).resolve().parent / "golden" / "survey_known_answers.json").read_text())
PRIMES = [int(p) for p in KA["constants"]]


@pytest.fixture(scope="module")
def m():
    import paper_1609_00999_b200 as mod
    return mod


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("P", PRIMES)
def test_gpu_mont_ab_and_conversions(m, P):
    k = KA["constants"][str(P)]
    ctx = m.ctx_init(P)
    a, b = synth.uniform(42, 1, P, 0, 4), synth.uniform(42, 2, P, 0, 4)
    assert m.mul_vec(ctx, dev(a), dev(b)).cpu().tolist() == KA["mont_ab_first4"][str(P)]
    x = dev(np.array([1, k["w"], P - 1, 0], np.uint32))
    tm = m.to_mont(ctx, x).cpu().tolist()
    assert tm[0] == k["r1"] and tm[1] == k["to_mont_w"] and tm[3] == 0
    # mont(P-1, P-1) = R^-1 mod P (SURVEY §8(c) closed form), from_mont(1) = R^-1 too
    assert m.mul_vec(ctx, dev(np.array([P - 1], np.uint32)), dev(np.array([P - 1], np.uint32))).item() == k["Rinv"]
    assert m.from_mont(ctx, dev(np.array([1], np.uint32))).item() == k["Rinv"]


def test_gpu_c1_end_to_end(m):
    k = KA["c1"]
    a, b = synth.c1_inputs(k["P"], n=k["n"])
    c, acc = m.mul_vec_checksum(m.ctx_init(k["P"]), dev(a), dev(b))
    hc = c.cpu().numpy()
    assert int(acc.item()) % k["P"] == k["checksum_mod_P"]
    assert hc[:4].tolist() == k["c_first4"] and hc[-2:].tolist() == k["c_last2"]


@pytest.mark.parametrize("variant", list(range(18)))
def test_gpu_c4_first4(m, variant):
    k = KA["c4"]
    base, e = synth.c4_inputs(k["P"], 0, 4096)   # whole uint4s so every vector path runs
    out = m.pow_vec(m.ctx_init(k["P"]), dev(base), dev(e), cfg=m.Launch(variant=variant))
    assert out[:4].cpu().tolist() == k["out_first4"]


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
def test_gpu_c3_first4(m, variant):
    k = KA["c3"]
    P, L = k["P"], k["len"]
    ctx = m.ctx_init(P)
    tw = m.twiddle_table(ctx, KA["constants"][str(P)]["w"], L)
    assert tw[:4].cpu().tolist() == k["tw_first4"]
    x = synth.c3_x(P, batch=3, length=L)
    out = m.mul_twiddle(ctx, dev(x), tw, cfg=m.Launch(variant=variant))
    assert out[0, :4].cpu().tolist() == k["out_row0_first4"]
