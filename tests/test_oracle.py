"""Pin the CPU oracle (oracle/covap_oracle.c) before trusting it.

1. The reference's own known-answer tests, transcribed with their file:line.
2. The golden fixtures produced by the reference library itself
   (tests/golden/make_golden.py) — bit-exact.
3. Live cross-checks against oracle/_ref (the reference compiled from its
   sources) on fresh seeded inputs, where that library is present.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle.oracle import OracleError

CAP25 = 25 * 1024 * 1024
TABLE_V = [4101096, 16781312, 107480576, 7079424, 7669760, 555072]


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def layout_sizes(name):
    with open(os.path.join(os.path.dirname(GOLDEN), "..", "paper_2311_04499_b200", "layouts",
                           name + ".json")) as f:
        d = json.load(f)
    return [l["param_count"] for l in d["layers"]]


# ---------------------------------------------------------------- 1. known answers

def test_bucketing_known_answers(orc):
    # test_model.cpp:37-42, 44-48, 50-54, 56-58
    assert orc.allocate_buckets([1728, 36864], CAP25)[0] == [38592]
    assert orc.allocate_buckets([102760448], CAP25)[0] == [102760448]
    assert orc.allocate_buckets([6000000] * 3, CAP25)[0] == [6000000] * 3
    with pytest.raises(OracleError) as e:
        orc.allocate_buckets([], CAP25)
    assert e.value.code == 1
    # test_model.cpp:60-65: the Table V buckets reproduce from their own sizes
    assert orc.allocate_buckets(TABLE_V, CAP25)[0] == TABLE_V


def test_median_known_answers(orc):
    assert orc.median_twice(TABLE_V) == 2 * 5590260            # test_model.cpp:67-69
    assert orc.median_twice([5]) == 10                          # test_model.cpp:71-74
    b, _ = orc.allocate_buckets([1, 3, 100], 4)                 # test_model.cpp:76-80
    assert b == [1, 3, 100] and orc.median_twice(b) == 6


def test_sharding_known_answers(orc):
    # test_model.cpp:82-96 and acceptance.cpp:91-118
    ts = orc.effective_tensors(TABLE_V, 19, 1)
    assert sum(1 for t in ts if t[0] == 1) == 3
    assert sum(1 for t in ts if t[0] == 2) == 19
    assert len(ts) == 26
    assert len(orc.effective_tensors(TABLE_V, 2, 1)) == 8
    for K in (25, 64):
        assert len(orc.effective_tensors(TABLE_V, K, 1)) == 26
    # equal buckets never shard (test_model.cpp:98-105)
    for K in (1, 2, 7, 100):
        assert len(orc.effective_tensors([10, 10, 10], K, 1)) == 3


def test_selection_known_answers(orc):
    sel = lambda *a: np.flatnonzero(orc.select(*a)).tolist()  # noqa: E731
    assert sel(0, 4, 8) == [0, 4]                 # test_compress.cpp:62-66
    assert sel(1, 4, 8) == [1, 5]
    assert sel(123, 1, 5) == [0, 1, 2, 3, 4]
    assert sel(0, 4, 8, 1) == [0, 4]              # test_compress.cpp:68-71
    assert sel(1, 4, 8, 1) == [3, 7]
    with pytest.raises(OracleError):
        orc.select(0, 0, 4)
    with pytest.raises(OracleError):
        orc.select(0, 4, 0)


def test_ef_known_answers(orc):
    # test_compress.cpp:103-107
    assert orc.ef_coefficient(0, 0.2, 100, 0.1) == pytest.approx(0.2)
    assert orc.ef_coefficient(350, 0.2, 100, 0.1) == pytest.approx(0.5)
    assert orc.ef_coefficient(1000000, 0.2, 100, 0.1) == 1.0


def test_two_step_trace(orc):
    # test_compress.cpp:118-137 (K=2, coeff == 1)
    tensors = [(0, 0, 2), (1, 2, 4)]
    r = np.zeros(4)
    p0 = orc.compress(np.array([1., 2, 3, 4]), r, tensors, orc.select(0, 2, 2), 1, 1.0)
    assert p0.tolist() == [1, 2] and r.tolist() == [0, 0, 3, 4]
    p1 = orc.compress(np.array([5., 6, 7, 8]), r, tensors, orc.select(1, 2, 2), 1, 1.0)
    assert p1.tolist() == [10, 12] and r.tolist() == [5, 6, 0, 0]


def test_decompress_and_mean_known_answers(orc):
    tensors = [(0, 0, 2), (1, 2, 4)]
    assert orc.decompress([1., 2], tensors, [1, 0], 4, np.float64).tolist() == [1, 2, 0, 0]
    assert orc.decompress([], tensors, [0, 0], 4, np.float64).tolist() == [0, 0, 0, 0]
    assert orc.allreduce_mean(np.array([[1., 2], [3, 4]])).tolist() == [2, 3]   # test_trainer.cpp:45-49
    assert orc.allreduce_mean(np.array([[5., 6, 7]])).tolist() == [5, 6, 7]


def test_ccr_known_answers(orc):
    # test_perf.cpp:27-41, acceptance.cpp:120-124
    assert orc.ccr(280, 135) == pytest.approx(2.074, rel=1e-3)
    assert orc.ccr(842, 210) == pytest.approx(4.0095, rel=1e-3)
    assert orc.ccr(0, 100) == 0.0 and orc.ccr(0, 0) == 0.0
    with pytest.raises(OracleError) as e:
        orc.ccr(10, 0)
    assert e.value.code == 3
    for c, k in ((280 / 135, 3), (4.0, 4), (3.5, 4), (0.4, 1), (0.0, 1)):
        assert orc.choose_interval(c) == k


def test_profile_known_answers(orc):
    # test_sim.cpp:266-279: skew {0, 40, 0} on one 100 ms collective
    a, naive, c, k = orc.profile_ccr([[60.0], [100.0], [60.0]], [200.0], 50.0)  # arrivals, shared end
    assert a == 100.0 and naive == [140.0, 100.0, 140.0] and c == pytest.approx(2.0) and k == 2


def test_conservation_on_integers(orc):
    # test_compress.cpp:223-245: 200 integer steps, K=3, coeff 1 -> exact
    tensors = [(t, 8 * t, 8 * t + 8) for t in range(5)]
    r = np.zeros(40)
    inp = np.zeros(40)
    sent = np.zeros(40)
    for s in range(200):
        g = orc.generate(orc.stream_key(17, 0, s), 40, 1, 0, np.float64)
        inp += g
        keep = orc.select(s, 3, 5)
        p = orc.compress(g, r, tensors, keep, 1, 1.0)
        sent += orc.decompress(p, tensors, keep, 40, np.float64)
        for t in np.flatnonzero(keep):
            assert np.all(r[8 * t:8 * t + 8] == 0)
    assert np.array_equal(sent + r, inp)


def test_generator_properties(orc):
    g = orc.generate(orc.stream_key(1, 0, 0), 200000, 0, 0, np.float32)
    assert abs(g.mean()) < 0.01 and 1.0 < g.std() < 1.3 and np.abs(g).max() <= 4.0
    gi = orc.generate(orc.stream_key(1, 0, 0), 200000, 1, 0, np.float64)
    assert gi.min() >= -1000 and gi.max() <= 1000 and np.all(gi == np.round(gi))
    # counter-based: any window equals the same slice of the full stream
    full = orc.generate(12345, 1000, 0, 0, np.float64)
    assert np.array_equal(orc.generate(12345, 77, 0, 501, np.float64), full[501:578])
    assert np.array_equal(full.astype(np.float32), orc.generate(12345, 1000, 0, 0, np.float32))


# ---------------------------------------------------------------- 2. golden fixtures

def _plan_sizes(case):
    return case["layers"] if case["layers"] is not None else layout_sizes(case["layout"])


def test_oracle_plans_match_reference_fixtures(orc):
    for case in load("plans.json"):
        sizes = _plan_sizes(case)
        b, _ = orc.allocate_buckets(sizes, case["cap"])
        assert b == case["buckets"], case["case"]
        assert orc.median_twice(b) == case["twice_median"], case["case"]
        ts = orc.effective_tensors(b, case["K"], case["shard"])
        assert [list(t) for t in ts] == case["tensors"], (case["case"], case["K"])


def test_oracle_selection_ef_ccr_match_fixtures(orc):
    for c in load("selection.json"):
        assert np.flatnonzero(orc.select(c["step"], c["K"], c["count"], c["rule"])).tolist() == c["selected"]
    for c in load("ef.json"):
        assert orc.ef_coefficient(c["step"], *c["sched"]) == c["coeff"]
    d = load("ccr.json")
    for c in d["ccr"]:
        if "error" in c:
            with pytest.raises(OracleError) as e:
                orc.ccr(c["comm"], c["comp"])
            assert e.value.code == c["error"]
        else:
            assert orc.ccr(c["comm"], c["comp"]) == c["value"]
    for c in d["interval"]:
        if "error" in c:
            with pytest.raises(OracleError):
                orc.choose_interval(c["ccr"])
        else:
            assert orc.choose_interval(c["ccr"]) == c["value"]
    for c in d["profile"]:
        a, naive, cc, k = orc.profile_ccr(c["starts"], c["ends"], c["comp"])
        assert (a, naive, cc, k) == (c["aligned"], c["naive"], c["ccr"], c["interval"])


def _trace_cases():
    return load("manifest.json")["compress"]


@pytest.mark.parametrize("case", _trace_cases(), ids=lambda c: c["name"])
def test_oracle_compress_traces_bit_exact(orc, case):
    fx = np.load(os.path.join(GOLDEN, f"compress_{case['name']}.npz"))
    tensors = [tuple(int(x) for x in t) for t in fx["tensors"]]
    buckets, ts = orc.plan(case["sizes"], case["cap"], case["K"])
    assert [tuple(t) for t in ts] == tensors
    d = tensors[-1][2]
    r = np.zeros(d)
    en, init, asc, rng = case["ef"]
    for s in range(case["steps"]):
        g = orc.generate(orc.stream_key(case["seed"], 0, s), d, case["kind"], 0, np.float64)
        keep = orc.select(s, case["K"], len(tensors), case["rule"])
        assert np.flatnonzero(keep).tolist() == fx[f"selected_{s}"].tolist()
        coeff = orc.ef_coefficient(s, init, asc, rng)
        p = orc.compress(g, r, tensors, keep, en, coeff)
        assert np.array_equal(p, fx[f"payload_{s}"])
        assert np.array_equal(r, fx[f"residual_{s}"])
        dense = orc.decompress(p, tensors, keep, d, np.float64)
        assert np.array_equal(dense, fx[f"dense_{s}"])


@pytest.mark.parametrize("case", load("manifest.json")["session"], ids=lambda c: c["name"])
def test_oracle_sessions_bit_exact(orc, case):
    """The per-rank decomposition K1 -> sum -> K2(x1/P) reproduces the
    reference's in-process step (trainer.cpp:365-386) exactly."""
    fx = np.load(os.path.join(GOLDEN, f"session_{case['name']}.npz"))
    _, tensors = orc.plan(case["sizes"], case["cap"], case["K"])
    d = tensors[-1][2]
    P = case["P"]
    rs = [np.zeros(d) for _ in range(P)]
    en, init, asc, rng = case["ef"]
    for s in range(case["steps"]):
        keep = orc.select(s, case["K"], len(tensors), case["rule"])
        coeff = orc.ef_coefficient(s, init, asc, rng)
        payloads = []
        for w in range(P):
            g = orc.generate(orc.stream_key(case["seed"], w, s), d, case["kind"], 0, np.float64)
            payloads.append(orc.compress(g, rs[w], tensors, keep, en, coeff))
        mean = orc.allreduce_mean(np.stack(payloads)) if len(payloads[0]) else payloads[0]
        upd = orc.decompress(mean, tensors, keep, d, np.float64)
        assert np.array_equal(upd, fx[f"update_{s}"])
        assert np.array_equal(rs[0], fx[f"residual0_{s}"])


# ---------------------------------------------------------------- 3. live reference

def test_oracle_vs_live_reference_random(orc, ref):
    rng = np.random.default_rng(3)
    for trial in range(25):
        n = int(rng.integers(1, 12))
        sizes = [int(x) for x in rng.integers(1, 5000, n)]
        cap = 4 * int(rng.integers(1, 6000))
        K = int(rng.integers(1, 7))
        rb, tw, rts = ref.plan(sizes, cap, K)
        ob, ots = orc.plan(sizes, cap, K)
        assert ob == rb and [tuple(t) for t in ots] == [tuple(t) for t in rts]
        numels = [t[2] - t[1] for t in rts]
        d = sum(numels)
        r_ref, r_orc = np.zeros(d), np.zeros(d)
        ns = 0
        for s in range(2 * K + 1):
            g = orc.generate(orc.stream_key(trial, 0, s), d, 0, 0, np.float64)
            p_ref, sel, ns = ref.compress(g, numels, r_ref, ns, K, 0, (1, 0.4, 2, 0.15))
            keep = orc.select(s, K, len(numels))
            p_orc = orc.compress(g, r_orc, rts, keep, 1, orc.ef_coefficient(s, 0.4, 2, 0.15))
            assert np.array_equal(p_ref, p_orc) and np.array_equal(r_ref, r_orc)
