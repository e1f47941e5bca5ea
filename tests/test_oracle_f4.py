"""Pins the C restatement of the baseline compressors and the generic
error-feedback wrapper (oracle/covap_oracle.c) to the
reference: its known-answer tests (test_compress.cpp:247-386) and the golden
fixtures generated from the reference library (tests/golden/make_golden_f4.py).
When oracle/_ref exists (the build container) it is also compared live."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT

from oracle.oracle import Oracle, OracleError

GOLD = os.path.join(ROOT, "tests", "golden")
KINDS = {"identity": 0, "covap": 1, "topk": 2, "randomk": 3, "fp16": 4}


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def ref_or_skip():
    from oracle.oracle import Ref, REF_SO
    if not os.path.exists(REF_SO) and not os.path.isdir("/root/reference/proj"):
        pytest.skip("reference library not built here")
    return Ref()


def test_known_answers(orc):
    # test_compress.cpp:247-260
    i, v = orc.topk(np.array([3, -5, 1, 2], float), 0.5)
    assert i.tolist() == [1, 0] and v.tolist() == [-5, 3]
    assert len(orc.topk(np.array([3, -5, 1, 2], float), 1.0)[0]) == 4
    assert orc.topk(np.array([2, -2, 2], float), 1 / 3)[0].tolist() == [0]
    with pytest.raises(OracleError):
        orc.topk(np.zeros(0), 0.5)
    # test_compress.cpp:290-300
    a = orc.randomk(10, 0.3, 99)
    assert a.tolist() == orc.randomk(10, 0.3, 99).tolist() and len(a) == 3
    assert len(set(a.tolist())) == 3 and max(a) < 10
    assert len(orc.randomk(10, 1.0, 1)) == 10
    # test_compress.cpp:317-328
    y, sat = orc.fp16_roundtrip(np.array([1.0, 2049.0, 70000.0, -70000.0, 0.0, 0.1]))
    assert y[:5].tolist() == [1.0, 2048.0, 65504.0, -65504.0, 0.0]
    assert abs(y[5] - 0.0999755859375) < 1e-12 and sat == 2
    for bad in (0.0, -0.1, 1.5):
        with pytest.raises(OracleError):
            orc.sparsifier_k(10, bad)


def test_randomk_uniform_over_seeds(orc):
    # test_compress.cpp:303-315
    hits = np.zeros(10)
    for seed in range(10000):
        for i in orc.randomk(10, 0.3, seed):
            hits[i] += 1
    assert np.all(np.abs(hits / 10000 - 0.3) <= 0.02)


def test_half_bits_match_reference_fixture(orc):
    z = np.load(os.path.join(GOLD, "half_bits.npz"))
    vals, half, sat, widened = z["values"], z["half"], z["saturated"], z["widened"]
    for i in range(64):  # the special values and a few random ones, bit by bit
        h, s = orc.half_bits(vals[i])
        assert h == half[i] and s == bool(sat[i]), (i, vals[i])
    for h in range(0, 65536, 257):
        assert np.float32(orc.float_from_half(h)).tobytes() == widened[h].tobytes(), h
    # every value: round trip == the reference's widened half, same clamp count
    y, nsat = orc.fp16_roundtrip(vals)
    assert y.tobytes() == widened[half].tobytes()
    assert nsat == int(sat.sum())


def test_sparsifiers_match_reference_fixture(orc):
    with open(os.path.join(GOLD, "sparsifiers.json")) as f:
        cases = json.load(f)
    for c in cases:
        if "x" in c:
            x = np.array(c["x"], float)
            assert orc.topk(x, c["k_fraction"])[0].tolist() == c["topk_indices"]
            assert orc.randomk(len(x), c["k_fraction"], c["seed"]).tolist() == c["randomk_indices"]
        elif "gen" in c:
            seed, n, kind = c["gen"]
            x = orc.generate(orc.stream_key(seed, n, kind), n, kind=kind, dtype=np.float64)
            assert orc.topk(x, c["k_fraction"])[0].tolist() == c["topk_indices"]
        else:
            assert orc.randomk(c["d"], c["k_fraction"], c["seed"]).tolist() == c["randomk_indices"]


def tensors_of(sizes):
    out, b = [], 0
    for s in sizes:
        out.append((len(out), b, b + s))
        b += s
    return out


def coeff_of(orc, ef, step):
    return orc.ef_coefficient(step, ef[1], ef[2], ef[3]) if ef[0] else 0.0


@pytest.mark.parametrize("case", json.load(open(os.path.join(GOLD, "feedback.json"))),
                         ids=lambda c: c["name"])
def test_feedback_matches_reference_trace_f64(orc, case):
    z = np.load(os.path.join(GOLD, f"feedback_{case['name']}.npz"))
    tensors = tensors_of(case["sizes"])
    r = np.zeros(sum(case["sizes"]))
    for step in range(case["steps"]):
        kept, sent, _ = orc.feedback_step(KINDS[case["kind"]], step, z["g"][step], r, tensors,
                                          case["ef"][0], coeff_of(orc, case["ef"], step),
                                          interval=case["interval"], k_fraction=case["k_fraction"],
                                          seed=case["seed"])
        assert kept.tobytes() == z["kept"][step].tobytes(), (case["name"], step)
        assert r.tobytes() == z["residual"][step].tobytes(), (case["name"], step)
        assert sent == z["transmitted"][step]


def test_feedback_conserves_mass_for_every_scheme(orc):
    # test_compress.cpp:338-360, integer inputs, full compensation
    sizes = [6, 6, 6]
    tensors = tensors_of(sizes)
    for kind in (1, 2, 3, 4, 0):
        for dt in (np.float64, np.float32):
            r = np.zeros(18, dt)
            gin = np.zeros(18, dt)
            sent = np.zeros(18, dt)
            for step in range(100):
                g = orc.generate(orc.stream_key(77, kind, step), 18, kind=1, dtype=dt)
                gin += g
                kept, _, _ = orc.feedback_step(kind, step, g, r, tensors, 1, 1.0, interval=3,
                                               k_fraction=0.25, seed=42)
                sent += kept
            assert np.array_equal(sent + r, gin), (kind, dt)


def test_oracle_matches_live_reference_on_random_cases(orc):
    ref = ref_or_skip()
    from oracle.oracle import RefFeedback
    rng = np.random.default_rng(11)
    for trial in range(12):
        sizes = rng.integers(1, 300, rng.integers(1, 6)).tolist()
        kind = int(trial % 5)
        kf = float(rng.choice([0.01, 0.1, 0.37, 1.0]))
        ef = (1, 0.3, 2, 0.2)
        fb = RefFeedback(ref, sizes, kind, interval=3, k_fraction=kf, seed=trial, ef=ef)
        r = np.zeros(sum(sizes))
        for step in range(5):
            g = rng.standard_normal(sum(sizes)) * (10.0 ** rng.integers(-8, 6))
            if trial % 3 == 0:
                g = np.round(g)  # ties
            kept_ref, res_ref, sent_ref, _ = fb.step(g)
            kept, sent, _ = orc.feedback_step(kind, step, g, r, tensors_of(sizes), 1,
                                              coeff_of(orc, ef, step), interval=3,
                                              k_fraction=kf, seed=trial)
            assert kept.tobytes() == kept_ref.tobytes()
            assert r.tobytes() == res_ref.tobytes()
            assert sent == sent_ref
        fb.close()
