"""The "covap" settings of a run and the CCR controller in the library
(SURVEY.md §8 rows a14-a17), host-only: covap_settings_from_json
(config.cpp:27-38, 133-157), covap_resolve_interval (config.cpp:238-241) and
covap_ccr_decide with one rank (sim.cpp:164-216, perf.cpp:40-53).
Known answers from the reference's own tests (test_config.cpp:18-66,
test_perf.cpp:27-41, test_sim.cpp:254-317)."""
import json

import pytest

# test_config.cpp:18-39, the reference's minimal document
MINIMAL = {
    "name": "unit", "seed": 3,
    "model": {"layers": [{"name": "a", "param_count": 1000}, {"name": "b", "param_count": 1000}],
              "bucket_cap_bytes": 4000},
    "cluster": {"workers": 8, "bandwidth_bps": 3e10, "latency_ms": 1.0,
                "allreduce_efficiency": 0.5},
    "phases": {"before_ms": 10, "comp_ms": 20, "comm_ms": 50},
    "compressor": {"scheme": "covap"},
    "covap": {"interval": "auto",
              "ef": {"enabled": True, "init_value": 0.3, "ascend_steps": 10, "ascend_range": 0.1}},
}


def test_defaults(covap):
    s = covap.CovapSettings.from_json({})
    assert (s.interval, s.auto_interval, s.rule) == (1, False, covap.SelectionRule.kMatchStep)
    assert s.ef == covap.EfSchedule(True, 0.3, 100, 0.1)  # compress.hpp:27-30
    assert s.resolve_interval(5.5) == 1


def test_reference_document_and_auto_interval(covap):
    """test_config.cpp:43-66: "auto" resolves through the measured ratio,
    a fixed interval ignores it."""
    s = covap.settings_from_json(MINIMAL)
    assert s.auto_interval and s.ef.init_value == pytest.approx(0.3) and s.ef.ascend_steps == 10
    assert covap.resolve_interval(s, 2.5) == 3
    assert covap.resolve_interval(s, 0.2) == 1
    doc = json.loads(json.dumps(MINIMAL))
    doc["covap"]["interval"] = 7
    fixed = covap.settings_from_json(json.dumps(doc))
    assert not fixed.auto_interval and fixed.interval == 7
    assert fixed.resolve_interval(2.5) == 7
    doc["covap"]["selection"] = "formula"
    assert covap.settings_from_json(doc).rule == covap.SelectionRule.kPlusStep
    assert covap.settings_from_json(doc).config(7) == covap.CovapConfig(
        7, covap.SelectionRule.kPlusStep, covap.EfSchedule(True, 0.3, 10, 0.1))


@pytest.mark.parametrize("patch,path", [
    ({"interval": 0}, "covap.interval"),
    ({"interval": -3}, "covap.interval"),
    ({"interval": "sometimes"}, "covap.interval"),
    ({"interval": 2.5}, "covap.interval"),
    ({"selection": "sideways"}, "covap.selection"),
    ({"ef": 3}, "covap.ef"),
    ({"ef": {"init_value": 1.5}}, "covap.ef.init_value"),
    ({"ef": {"init_value": "x"}}, "init_value"),
    ({"ef": {"ascend_steps": 0}}, "covap.ef.ascend_steps"),
    ({"ef": {"ascend_range": -0.1}}, "covap.ef.ascend_range"),
])
def test_bad_fields_carry_their_path(covap, patch, path):
    """ConfigError with the field path in the message (config.cpp:17-19;
    test_config.cpp:68-87 for covap.interval)."""
    doc = json.loads(json.dumps(MINIMAL))
    doc["covap"].update(patch)
    with pytest.raises(covap.ConfigError) as e:
        covap.settings_from_json(doc)
    assert f"config field '{path}'" in str(e.value)


def test_malformed_documents(covap):
    with pytest.raises(covap.ConfigError):
        covap.settings_from_json("{not json")
    with pytest.raises(covap.ConfigError, match="root must be a JSON object"):
        covap.settings_from_json("[1, 2]")


@pytest.mark.parametrize("comm,comp,k", [([280.0], 135.0, 3), ([842.0], 210.0, 5),
                                         ([100.0, 300.0], 100.0, 4), ([0.0, -1.0], 50.0, 1)])
def test_ccr_decide_one_rank(covap, comm, comp, k):
    """ccr / choose_interval on the aligned communication time; a collective
    that did not run (negative duration) counts 0 (test_perf.cpp:27-41,
    test_sim.cpp:307-317)."""
    r = covap.ccr_decide(None, comm, comp)
    aligned = sum(max(0.0, x) for x in comm)
    assert r.comm_aligned_ms == aligned and r.comp_ms == comp
    assert r.ccr == covap.ccr(aligned, comp) and r.recommended_interval == k


def test_ccr_decide_errors(covap):
    with pytest.raises(covap.UndefinedRatio):
        covap.ccr_decide(None, [10.0], 0.0)  # x / 0 (perf.cpp:42-45)
    assert covap.ccr_decide(None, [0.0], 0.0).ccr == 0.0  # 0 / 0 -> 0
    with pytest.raises(covap.InvalidInput):
        covap.ccr_decide(None, [1.0], -1.0)
