"""The product's host planner, selection, EF and CCR logic — reached through
the C-ABI (libcovap_b200.so), no GPU needed — against the reference's golden
fixtures and known answers.  Integer outputs are bit-exact by contract."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from test_oracle import TABLE_V, CAP25, layout_sizes, load


def model(c, sizes, cap):
    return c.ModelSpec([c.LayerSpec(f"l{i}", int(n)) for i, n in enumerate(sizes)], cap)


def test_plans_match_reference(covap):
    for case in load("plans.json"):
        sizes = case["layers"] if case["layers"] is not None else layout_sizes(case["layout"])
        m = model(covap, sizes, case["cap"])
        p = covap.BucketPlan(m, interval=case["K"], shard=case["shard"])
        assert [b.numel for b in p.buckets] == case["buckets"], case["case"]
        assert p.twice_median == case["twice_median"]
        assert [[t.bucket, t.begin, t.end] for t in p.tensors] == case["tensors"], case["case"]
        # flat offsets are contiguous and cover [0, N)
        assert p.tensors[0].begin == 0 and p.tensors[-1].end == p.total_numel()
        assert all(a.end == b.begin for a, b in zip(p.tensors, p.tensors[1:]))


def test_reference_api_mirror(covap):
    plan = covap.allocate_buckets(model(covap, TABLE_V, CAP25))
    assert [b.numel for b in plan.buckets] == TABLE_V
    assert covap.median_numel(plan) == 5590260.0
    s19 = covap.shard_plan(plan, 19)
    assert sum(1 for t in s19.tensors if t.bucket == 1) == 3
    assert sum(1 for t in s19.tensors if t.bucket == 2) == 19
    assert len(covap.effective_tensors(s19)) == 26
    assert len(covap.effective_numels(covap.shard_plan(plan, 2))) == 8
    # plan_for mirrors train(): no sharding at K == 1
    assert not covap.plan_for(plan.model, covap.CovapConfig(interval=1)).sharded
    assert covap.plan_for(plan.model, covap.CovapConfig(interval=4)).sharded


def test_layouts_appendix_a(covap):
    """SURVEY.md Appendix A (numbers produced by the reference library)."""
    expect = {
        "resnet50": (161, 25557032, [6515688, 4462592, 6300160, 6112256, 2166336], [5, 5, 5, 5, 5],
                     [8682024, 4462592, 6300160, 6112256]),
        "vgg16": (32, 138357544, [4101096, 16777216, 4096, 102760448, 4720128, 4719616, 5274944],
                  [7, 9, 12, 16, 24], [29795304, 36002646, 36002133, 36557461]),
        "bert_large": (391, 335141888, None, [50, 51, 53, 53, 53],
                       [84987392, 83372544, 83409408, 83372544]),
    }
    for name, (nl, total, buckets, counts, payload) in expect.items():
        m = covap.load_layout(name)
        assert len(m.layers) == nl and m.total_params() == total
        p = covap.allocate_buckets(m)
        if buckets:
            assert [b.numel for b in p.buckets] == buckets
        assert [len(covap.plan_for(m, covap.CovapConfig(interval=K)).tensors)
                for K in (1, 2, 4, 8, 16)] == counts
        p4 = covap.plan_for(m, covap.CovapConfig(interval=4))
        assert [p4.payload_elements(s) for s in range(4)] == payload


def test_selection_ef_ccr_match_reference(covap):
    for c in load("selection.json"):
        assert covap.select_tensors(c["step"], c["K"], c["count"], c["rule"]) == c["selected"]
    for c in load("ef.json"):
        assert covap.ef_coefficient(c["step"], covap.EfSchedule(True, *c["sched"])) == c["coeff"]
    d = load("ccr.json")
    errs = {1: covap.InvalidInput, 3: covap.UndefinedRatio}
    for c in d["ccr"]:
        if "error" in c:
            with pytest.raises(errs[c["error"]]):
                covap.ccr(c["comm"], c["comp"])
        else:
            assert covap.ccr(c["comm"], c["comp"]) == c["value"]
    for c in d["interval"]:
        if "error" in c:
            with pytest.raises(errs[c["error"]]):
                covap.choose_interval(c["ccr"])
        else:
            assert covap.choose_interval(c["ccr"]) == c["value"]
    for c in d["profile"]:
        r = covap.profile_ccr(c["starts"], c["ends"], c["comp"], len(c["starts"]))
        assert (r.comm_aligned_ms, r.naive_comm_ms, r.ccr, r.recommended_interval) == \
            (c["aligned"], c["naive"], c["ccr"], c["interval"])


def test_profile_incomplete_and_skew(covap):
    # test_sim.cpp:266-279 and 319-326
    r = covap.profile_ccr([[60.0], [100.0], [60.0]], [200.0], 50.0, 3)
    assert r.comm_aligned_ms == 100.0 and r.naive_comm_ms == [140.0, 100.0, 140.0]
    assert r.recommended_interval == 2
    with pytest.raises(covap.IncompleteProfile):
        covap.profile_ccr([[60.0], [100.0]], [200.0], 50.0, 3)
    # zero communication -> K = 1 (test_sim.cpp:307-317)
    assert covap.profile_ccr([[], []], [], 40.0, 2).recommended_interval == 1


def test_errors_match_reference_taxonomy(covap):
    with pytest.raises(covap.InvalidInput):
        covap.allocate_buckets(covap.ModelSpec([]))                       # model.cpp:25
    with pytest.raises(covap.InvalidInput):
        covap.allocate_buckets(model(covap, [0, 5], CAP25))              # model.cpp:27-28
    with pytest.raises(covap.InvalidInput):
        covap.allocate_buckets(covap.ModelSpec([covap.LayerSpec("x", 5, 3)]))  # model.cpp:29-30
    with pytest.raises(covap.InvalidInput):
        covap.allocate_buckets(model(covap, [5], CAP25), cap_bytes=0)    # model.cpp:38
    with pytest.raises(covap.InvalidInput):
        covap.shard_plan(covap.allocate_buckets(model(covap, [5], CAP25)), 0)  # model.cpp:96
    with pytest.raises(covap.InvalidInput):
        covap.select_tensors(0, 0, 5)                                      # compress.cpp:15
    with pytest.raises(covap.InvalidInput):
        covap.select_tensors(0, 3, 0)                                      # compress.cpp:16
    with pytest.raises(covap.InvalidInput):
        covap.ef_coefficient(3, covap.EfSchedule(True, 0.3, 0, 0.1))       # compress.cpp:31
    with pytest.raises(covap.InvalidInput):
        covap.choose_interval(-1.0)                                        # perf.cpp:50


@pytest.mark.parametrize("name,K,rule", [("resnet50", 4, 0), ("resnet50", 8, 0), ("vgg16", 4, 0),
                                         ("vgg16", 3, 1), ("bert_large", 4, 0), ("tablev", 19, 0),
                                         ("tablev", 2, 1), ("bert_large", 1, 0)])
def test_send_layout_invariants(covap, name, K, rule):
    """The device send layout: runs of selected tensors, dst ≡ begin (mod
    align) so 16-byte vectors line up, disjoint destinations, at most one
    selected range per bucket, and a K-window transmits every element once
    (bytes per K-window = 4d, test_trainer.cpp:89-106)."""
    m = covap.load_layout(name)
    p = covap.plan_for(m, covap.CovapConfig(interval=K, rule=rule))
    align = p.info.align
    total_payload = 0
    seen = np.zeros(len(p.tensors), np.int64)
    for s in range(K):
        sel = p.selection(s)
        assert sel == covap.select_tensors(s, K, len(p.tensors), rule)
        seen[sel] += 1
        send_elems, payload = p.send_elems(s)
        assert payload == sum(p.tensors[t].numel() for t in sel)
        total_payload += payload
        spans = []
        for b in range(len(p.buckets)):
            br = p.bucket_range(s, b)
            assert br.bucket_end - br.bucket_begin == p.buckets[b].numel
            chosen = [t for t in sel if p.tensors[t].bucket == b]
            assert len(chosen) <= 1
            if chosen:
                t = p.tensors[chosen[0]]
                assert (br.sel_begin, br.sel_end) == (t.begin, t.end)
                assert br.send_offset % align == br.sel_begin % align
                spans.append((br.send_offset, br.send_offset + t.numel()))
            else:
                assert br.sel_begin == br.sel_end
        spans.sort()
        assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))
        assert not spans or spans[-1][1] == send_elems
        assert send_elems <= p.max_send_elems
        assert send_elems - payload <= align * len(spans)
    assert np.all(seen == 1)
    assert total_payload == p.total_numel()


@pytest.mark.parametrize("name,K", [("resnet50", 4), ("vgg16", 4), ("bert_large", 3), ("tablev", 19)])
def test_padded_device_layout(covap, name, K):
    """COVAP_PLAN_PAD_BUCKETS: flat coordinates (tensors, selection, payload
    sizes) are those of the unpadded plan; device offsets start every bucket
    on a 32-element boundary; send offsets stay vector-aligned."""
    m = covap.load_layout(name)
    flat = covap.plan_for(m, covap.CovapConfig(interval=K))
    pad = covap.plan_for(m, covap.CovapConfig(interval=K), pad=True)
    assert not flat.padded and pad.padded
    assert [(t.bucket, t.begin, t.end) for t in pad.tensors] == \
        [(t.bucket, t.begin, t.end) for t in flat.tensors]
    assert flat.device_numel() == flat.total_numel()
    dev = 0
    for b, bk in enumerate(pad.buckets):
        assert pad.device_begin(b) == dev and dev % 32 == 0
        dev = (dev + bk.numel + 31) // 32 * 32
    assert pad.device_numel() == pad.device_begin(len(pad.buckets) - 1) + pad.buckets[-1].numel
    for s in range(K):
        assert pad.selection(s) == flat.selection(s)
        assert pad.send_elems(s)[1] == flat.send_elems(s)[1]
        for b in range(len(pad.buckets)):
            br, bf = pad.bucket_range(s, b), flat.bucket_range(s, b)
            assert (br.sel_begin, br.sel_end) == (bf.sel_begin, bf.sel_end)
            if br.sel_end > br.sel_begin:
                dev_sel = br.sel_begin - br.bucket_begin + br.device_begin
                assert br.send_offset % 32 == dev_sel % 32


def test_overlap_schedule_matches_reference(covap):
    """overlap_schedule (perf.cpp:63-103) bit-exact against the reference's
    outputs on 24 random cases (with/without compress blocks and masks), and
    the reference's own test_perf.cpp:59-83 cases."""
    for c in load("ccr.json")["overlap"]:
        sc = covap.overlap_schedule(c["before"], c["comp"], c["compress"], c["comm"],
                                    None if c["communicated"] is None else [bool(x) for x in c["communicated"]])
        assert (sc.total_ms, sc.stream_end_ms, sc.unoverlapped_comm_ms) == \
            (c["total"], c["stream_end"], c["unoverlapped"])
        assert sc.comm_start_ms == c["comm_start"] and sc.comm_end_ms == c["comm_end"]
        assert sc.comm_tensor == c["comm_tensor"]
        assert [b[0] for b in sc.bubbles] == c["bubble_after"]
        assert [b[1] for b in sc.bubbles] == c["bubble_ms"]
    # test_perf.cpp:59-65: zero communication ends with the stream
    sc = covap.overlap_schedule(5, [10, 20], None, [0, 0])
    assert sc.total_ms == 35 and sc.unoverlapped_comm_ms == 0
    with pytest.raises(covap.InvalidInput):
        covap.overlap_schedule(0, [1, 2], None, [1])
