"""GPU parity of the baseline compressors under error feedback (SURVEY.md
§8(f4); covap_feedback.cu through the C-ABI) against the reference and the
oracle.

Bars:
  * fp64: kept gradient, residual and transmitted count bit-exact against the
    REFERENCE's ErrorFeedback::step traces (tests/golden/feedback_*.npz, made
    by oracle/_ref) for every filter kind;
  * fp32: bit-exact against the fp32 restatement (oc_feedback_step_f32) at
    BASELINE layout sizes;
  * the synchronised gradient (trainer.cpp:387-403) bit-exact against the
    rank-ordered allreduce_mean of every rank's kept gradient, P = 1..4
    (virtual ranks on one GPU) and through a one-rank NCCL communicator;
  * the standalone compressors against the reference fixtures (index order
    included) and the oracle.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)
KINDS = {"identity": 0, "covap": 1, "topk": 2, "randomk": 3, "fp16": 4}


def F():
    from paper_2311_04499_b200 import feedback
    return feedback


def make_filter(kind, interval=1, k_fraction=0.01, seed=0):
    f = F()
    return {0: lambda: f.IdentityFilter(), 1: lambda: f.CovapFilter(interval),
            2: lambda: f.TopkFilter(k_fraction), 3: lambda: f.RandomkFilter(k_fraction, seed),
            4: lambda: f.Fp16Filter()}[kind]()


def schedule(covap, ef):
    return covap.EfSchedule(bool(ef[0]), float(ef[1]), int(ef[2]), float(ef[3]))


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def tensors_of(sizes):
    out, b = [], 0
    for s in sizes:
        out.append((len(out), b, b + s))
        b += s
    return out


def coeff_of(orc, ef, step):
    return orc.ef_coefficient(step, ef[1], ef[2], ef[3]) if ef[0] else 0.0


# ------------------------------------------------- fp64 vs the reference

@pytest.mark.parametrize("case", json.load(open(os.path.join(GOLDEN, "feedback.json"))),
                         ids=lambda c: c["name"])
def test_fp64_matches_reference_trace(covap, case):
    z = np.load(os.path.join(GOLDEN, f"feedback_{case['name']}.npz"))
    fb = F().ErrorFeedback(case["sizes"], schedule(covap, case["ef"]),
                           make_filter(KINDS[case["kind"]], case["interval"], case["k_fraction"],
                                       case["seed"]), dtype=torch.float64)
    for step in range(case["steps"]):
        assert fb.transmitted_elements() == z["transmitted"][step]
        g = torch.from_numpy(z["g"][step]).to(DEV)
        kept = fb.step(g).cpu().numpy()
        np.testing.assert_array_equal(bits(kept), bits(z["kept"][step]), err_msg=f"step {step}")
        np.testing.assert_array_equal(bits(fb.residuals.cpu().numpy()), bits(z["residual"][step]))
    assert fb.num_steps == case["steps"]


def test_fp64_matches_live_reference(covap, orc, ref):
    from oracle.oracle import RefFeedback
    rng = np.random.default_rng(5)
    for trial in range(10):
        sizes = rng.integers(1, 5000, rng.integers(1, 5)).tolist()
        kind = trial % 5
        kf = float(rng.choice([0.001, 0.05, 0.3, 1.0]))
        ef = (1, 0.3, 2, 0.2)
        rf = RefFeedback(ref, sizes, kind, interval=3, k_fraction=kf, seed=trial + 1, ef=ef)
        fb = F().ErrorFeedback(sizes, schedule(covap, ef), make_filter(kind, 3, kf, trial + 1),
                               dtype=torch.float64)
        for step in range(4):
            g = rng.standard_normal(sum(sizes)) * 10.0 ** rng.integers(-6, 7)
            if trial % 2:
                g = np.round(g * 4) / 4  # heavy ties
            kref, rres, sent, _ = rf.step(g)
            kept = fb.step(torch.from_numpy(g).to(DEV)).cpu().numpy()
            np.testing.assert_array_equal(bits(kept), bits(kref))
            np.testing.assert_array_equal(bits(fb.residuals.cpu().numpy()), bits(rres))
        rf.close()


# --------------------------------------------------- fp32 vs the oracle

def layout_buckets(covap, name):
    plan = covap.allocate_buckets(covap.load_layout(name))
    return [b.numel for b in plan.buckets]


@pytest.mark.parametrize("kind,kf,layout,steps", [
    (4, 0.0, "resnet50", 3),
    (2, 0.01, "resnet50", 2),
    (3, 0.01, "resnet50", 2),
    (3, 0.5, "resnet50", 2),  # 12.8 M samples: the sort variant of the selection
    (2, 0.001, "tablev", 1),
    (3, 0.05, "tablev", 1),
    (1, 0.0, "resnet50", 3),
])
def test_fp32_full_layout_bit_exact(covap, orc, kind, kf, layout, steps):
    sizes = layout_buckets(covap, layout)
    n = sum(sizes)
    ef = (1, 0.3, 1, 0.1)
    fb = F().ErrorFeedback(sizes, schedule(covap, ef), make_filter(kind, 4, kf, 99))
    r = np.zeros(n, np.float32)
    for step in range(steps):
        key = orc.stream_key(17, 0, step)
        g = torch.empty(n, dtype=torch.float32, device=DEV)
        covap.generate(g, key, 0)
        kept = fb.step(g).cpu().numpy()
        gh = orc.generate(key, n, kind=0, dtype=np.float32)
        want, sent, _ = orc.feedback_step(kind, step, gh, r, tensors_of(sizes), 1,
                                          coeff_of(orc, ef, step), interval=4, k_fraction=kf,
                                          seed=99)
        np.testing.assert_array_equal(bits(kept), bits(want), err_msg=f"{layout} step {step}")
        np.testing.assert_array_equal(bits(fb.residuals.cpu().numpy()), bits(r))
        assert fb.transmitted_elements(step) == sent


@pytest.mark.parametrize("kind", [2, 3])
@pytest.mark.parametrize("inputs", ["zeros", "ints", "one_hot", "tiny"])
def test_sparsifier_edge_cases(covap, orc, kind, inputs):
    """Degenerate candidate sets: all-equal magnitudes (every element in the
    threshold bin), integer ties, a single large element, size-1 tensors."""
    sizes = [1, 2, 3, 1000, 70000, 1]
    n = sum(sizes)
    rng = np.random.default_rng(3)
    for dt, npd in ((torch.float32, np.float32), (torch.float64, np.float64)):
        for kf in (0.001, 0.25, 0.5, 1.0):
            fb = F().ErrorFeedback(sizes, covap.EfSchedule(True, 1.0, 1, 0.0),
                                   make_filter(kind, 1, kf, 5), dtype=dt)
            r = np.zeros(n, npd)
            for step in range(3):
                if inputs == "zeros":
                    g = np.zeros(n, npd) if step == 0 else -np.zeros(n, npd)
                elif inputs == "ints":
                    g = rng.integers(-3, 4, n).astype(npd)
                elif inputs == "one_hot":
                    g = np.zeros(n, npd)
                    g[rng.integers(0, n)] = 7.0
                else:
                    g = (rng.standard_normal(n) * 1e-30).astype(npd)
                kept = fb.step(torch.from_numpy(g).to(DEV)).cpu().numpy()
                want, _, _ = orc.feedback_step(kind, step, g, r, tensors_of(sizes), 1, 1.0,
                                               k_fraction=kf, seed=5)
                np.testing.assert_array_equal(bits(kept), bits(want), err_msg=f"{dt} {kf} {step}")
                np.testing.assert_array_equal(bits(fb.residuals.cpu().numpy()), bits(r))


def test_fp16_saturation_count(covap, orc):
    x = np.array([1.0, 2049.0, 70000.0, -70000.0, 0.0, 0.1, 1e9, -1e-9], np.float32)
    fb = F().ErrorFeedback([len(x)], covap.EfSchedule(False), F().Fp16Filter())
    kept = fb.step(torch.from_numpy(x).to(DEV)).cpu().numpy()
    want, sat = orc.fp16_roundtrip(x)
    np.testing.assert_array_equal(bits(kept), bits(want))
    assert fb.saturations() == sat == 3
    assert fb.wire_bytes() == 2 * len(x)


# ------------------------------------------------------------ sync step

def oracle_mean(orc, kept_rows):
    return orc.allreduce_mean(np.stack(kept_rows))


@pytest.mark.parametrize("kind", [2, 3, 4])
@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("sizes", [[4097, 1, 30000, 65536, 513], [4097, 1, 30000, 65536, 511, 1]],
                         ids=["ragged", "tail-tensor"])
def test_virtual_rank_sync_matches_rank_ordered_mean(covap, orc, kind, P, sizes):
    """The wire of every rank, combined in rank order.  'tail-tensor': 100 146
    elements end in a 1-element tensor, so random-k always samples inside the
    streaming pass's 2-element scalar tail (whose list slots follow every
    tile's)."""
    n = sum(sizes)
    ef = (1, 0.3, 2, 0.2)
    ranks = [F().ErrorFeedback(sizes, schedule(covap, ef), make_filter(kind, 1, 0.02, 11))
             for _ in range(P)]
    res = [np.zeros(n, np.float32) for _ in range(P)]
    for step in range(3):
        outs, kepts, wires = [], [], []
        for p in range(P):
            key = orc.stream_key(23, p, step)
            g = torch.empty(n, dtype=torch.float32, device=DEV)
            covap.generate(g, key, 0)
            out = torch.full((n,), float("nan"), device=DEV)
            ranks[p].pack(g, out)
            a, b = ranks[p].wire()
            wires.append((None if a is None else a.clone(), None if b is None else b.clone()))
            outs.append(out)
            k, _, _ = orc.feedback_step(kind, step, orc.generate(key, n, 0, dtype=np.float32),
                                        res[p], tensors_of(sizes), 1, coeff_of(orc, ef, step),
                                        k_fraction=0.02, seed=11)
            kepts.append(k)
        want = oracle_mean(orc, kepts)
        ra = None if wires[0][0] is None else torch.cat([w[0] for w in wires])
        rb = None if wires[0][1] is None else torch.cat([w[1] for w in wires])
        for p in range(P):
            ranks[p].combine(ra, rb, P, outs[p])
            np.testing.assert_array_equal(bits(outs[p].cpu().numpy()), bits(want))
            np.testing.assert_array_equal(bits(ranks[p].residuals.cpu().numpy()), bits(res[p]))


@pytest.mark.parametrize("kind", [2, 3, 4])
def test_sync_step_one_rank_nccl_and_local(covap, orc, kind):
    sizes = [100000, 3, 77777]
    n = sum(sizes)
    uid = covap.Communicator.unique_id()
    comm = covap.Communicator(uid, 1, 0, 0)
    ef = (1, 0.3, 100, 0.1)
    a = F().ErrorFeedback(sizes, schedule(covap, ef), make_filter(kind, 1, 0.01, 3))
    b = F().ErrorFeedback(sizes, schedule(covap, ef), make_filter(kind, 1, 0.01, 3))
    r = np.zeros(n, np.float32)
    for step in range(3):
        key = orc.stream_key(29, 0, step)
        g = torch.empty(n, dtype=torch.float32, device=DEV)
        covap.generate(g, key, 0)
        oa = torch.full((n,), float("nan"), device=DEV)
        ob = torch.full((n,), float("nan"), device=DEV)
        a.sync(g, oa, comm)
        b.sync(g, ob, None)
        k, _, _ = orc.feedback_step(kind, step, orc.generate(key, n, 0, dtype=np.float32), r,
                                    tensors_of(sizes), 1, coeff_of(orc, ef, step),
                                    k_fraction=0.01, seed=3)
        want = oracle_mean(orc, [k])
        np.testing.assert_array_equal(bits(oa.cpu().numpy()), bits(want))
        np.testing.assert_array_equal(bits(ob.cpu().numpy()), bits(want))
    comm.close()


def test_sync_rejects_dense_filters_and_bad_shapes(covap):
    fb = F().ErrorFeedback([10], covap.EfSchedule(), F().CovapFilter(2))
    g = torch.zeros(10, device=DEV)
    with pytest.raises(covap.InvalidInput):
        fb.sync(g, torch.zeros(10, device=DEV))
    with pytest.raises(covap.InvalidState):
        fb.step(torch.zeros(11, device=DEV))
    with pytest.raises(covap.InvalidInput):
        F().ErrorFeedback([10, 0], covap.EfSchedule(), F().TopkFilter(0.1))
    with pytest.raises(covap.InvalidInput):
        F().ErrorFeedback([10], covap.EfSchedule(), F().TopkFilter(0.0))
    with pytest.raises(covap.InvalidInput):
        F().ErrorFeedback([10], covap.EfSchedule(), F().RandomkFilter(1.5, 1))


# ------------------------------------------------ standalone compressors

def test_standalone_compressors_match_reference_fixtures(covap, orc):
    f = F()
    with open(os.path.join(GOLDEN, "sparsifiers.json")) as fh:
        cases = json.load(fh)
    for c in cases:
        if "x" in c:
            x = torch.tensor(c["x"], dtype=torch.float64, device=DEV)
            i, v = f.topk_compress(x, c["k_fraction"])
            assert i.tolist() == c["topk_indices"] and v.tolist() == c["topk_values"]
            assert f.randomk_compress(x, c["k_fraction"], c["seed"])[0].tolist() == \
                c["randomk_indices"]
        elif "gen" in c:
            seed, n, kind = c["gen"]
            x = orc.generate(orc.stream_key(seed, n, kind), n, kind=kind, dtype=np.float64)
            i, v = f.topk_compress(torch.from_numpy(x).to(DEV), c["k_fraction"])
            assert i.tolist() == c["topk_indices"]
            np.testing.assert_array_equal(v.cpu().numpy(), x[c["topk_indices"]])
        else:
            x = torch.ones(c["d"], dtype=torch.float64, device=DEV)
            i, _ = f.randomk_compress(x, c["k_fraction"], c["seed"])
            assert i.tolist() == c["randomk_indices"]


def test_standalone_against_oracle_large(covap, orc):
    f = F()
    for n, kf, kind in ((1_000_003, 0.01, 0), (300_000, 0.3, 1), (4096, 1.0, 1)):
        for dt, npd in ((torch.float32, np.float32), (torch.float64, np.float64)):
            x = orc.generate(orc.stream_key(31, n, kind), n, kind=kind, dtype=npd)
            i, v = f.topk_compress(torch.from_numpy(x).to(DEV), kf)
            wi, wv = orc.topk(x, kf)
            np.testing.assert_array_equal(i.cpu().numpy(), wi.astype(np.int64))
            np.testing.assert_array_equal(bits(v.cpu().numpy()), bits(wv))
            ri, _ = f.randomk_compress(torch.from_numpy(x).to(DEV), kf, n * 7 + kind)
            np.testing.assert_array_equal(ri.cpu().numpy(),
                                          orc.randomk(n, kf, n * 7 + kind).astype(np.int64))


def test_fp16_roundtrip_matches_reference_half_table(covap):
    z = np.load(os.path.join(GOLDEN, "half_bits.npz"))
    vals, half, sat, widened = z["values"], z["half"], z["saturated"], z["widened"]
    out, nsat = F().fp16_roundtrip(torch.from_numpy(vals).to(DEV))
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), widened[half].view(np.uint32))
    assert nsat == int(sat.sum())
    # fp64 input: double -> float -> half, as fp16_roundtrip does (compress.cpp:230)
    x = np.array([1.0, 2049.0, 70000.0, -70000.0, 0.0, 0.1])
    out, nsat = F().fp16_roundtrip(torch.from_numpy(x).to(DEV))
    assert out.cpu().tolist()[:5] == [1.0, 2048.0, 65504.0, -65504.0, 0.0]
    assert abs(out.cpu().tolist()[5] - 0.0999755859375) < 1e-12 and nsat == 2


def test_conservation_every_scheme_at_layout_size(covap, orc):
    """sent + residual == sum of inputs, exactly, with integer gradients and
    full compensation (test_compress.cpp:338-360) at BERT-bucket scale."""
    sizes = [6296576, 6299648, 31254528 // 8]
    n = sum(sizes)
    for kind in (1, 2, 3, 4):
        fb = F().ErrorFeedback(sizes, covap.EfSchedule(True, 1.0, 1, 0.0),
                               make_filter(kind, 3, 0.01, 8))
        gin = torch.zeros(n, dtype=torch.float64, device=DEV)
        sent = torch.zeros(n, dtype=torch.float64, device=DEV)
        g = torch.empty(n, dtype=torch.float32, device=DEV)
        for step in range(6):
            covap.generate(g, orc.stream_key(41, kind, step), 1)
            gin += g.double()
            sent += fb.step(g).double()
        assert torch.equal(sent + fb.residuals.double(), gin), kind


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("kind", [2, 3, 4])
def test_sync_one_rank_signed_zero_mean(covap, orc, kind, dtype):
    """One rank fuses the mean into the filter pass: kept -0.0 must still come
    out as +0.0, the (0.0 + x) of allreduce_mean (trainer.cpp:41)."""
    sizes = [4100, 7]
    n = sum(sizes)
    fb = F().ErrorFeedback(sizes, covap.EfSchedule(False, 0.3, 100, 0.1),
                           make_filter(kind, 1, 1.0, 5), dtype=dtype)
    g = torch.full((n,), -0.0, dtype=dtype, device=DEV)
    g[::3] = -2.5
    out = torch.full((n,), float("nan"), dtype=dtype, device=DEV)
    fb.sync(g, out, None)
    gh = g.cpu().numpy()
    npt = np.float64 if dtype == torch.float64 else np.float32
    k, _, _ = orc.feedback_step(kind, 0, gh, np.zeros(n, npt), tensors_of(sizes), 0,
                                npt(0), k_fraction=1.0, seed=5)
    want = oracle_mean(orc, [k])
    assert np.all(bits(want)[gh == 0] == 0)  # +0.0, not -0.0
    np.testing.assert_array_equal(bits(out.cpu().numpy()), bits(want))


@pytest.mark.parametrize("kind", [2, 3])
def test_unsynchronised_steps_and_step_jumps(covap, orc, kind):
    """Random-k draws step s + 1's selection on a side stream during step s
    (covap_feedback_capi.cpp, ef_step): consecutive steps issued without a
    host synchronisation, on a user stream, and after num_steps jumps
    (set_step forwards and back, reset) must all select exactly what the
    reference selects for that step.  Top-k runs the same sequence (its
    mark / expand collect pass keeps a per-chunk hit bitmap across launches)."""
    sizes = [3, 5000, 70001, 1, 123457]
    n = sum(sizes)
    ef = (1, 0.3, 2, 0.2)
    fb = F().ErrorFeedback(sizes, schedule(covap, ef), make_filter(kind, 1, 0.02, 11))
    r = np.zeros(n, np.float32)
    stream = torch.cuda.Stream()
    steps = [0, 1, 2, 3, 7, 8, 2, 3, 3, 0, 1]
    gs = []
    for i, s in enumerate(steps):
        key = orc.stream_key(23, 0, i)
        g = torch.empty(n, dtype=torch.float32, device=DEV)
        covap.generate(g, key, 0)
        gs.append((g, orc.generate(key, n, kind=0, dtype=np.float32)))
    torch.cuda.synchronize()
    kepts, res = [], []
    with torch.cuda.stream(stream):
        for i, s in enumerate(steps):
            if fb.num_steps != s:
                fb.num_steps = s
            kept = torch.empty(n, dtype=torch.float32, device=DEV)
            fb.step(gs[i][0], kept=kept, stream=stream)
            kepts.append(kept)
            res.append(fb.residuals.clone())
    torch.cuda.synchronize()
    for i, s in enumerate(steps):
        want, _, _ = orc.feedback_step(kind, s, gs[i][1], r, tensors_of(sizes), 1,
                                       coeff_of(orc, ef, s), k_fraction=0.02, seed=11)
        np.testing.assert_array_equal(bits(kepts[i].cpu().numpy()), bits(want), err_msg=f"#{i} step {s}")
        np.testing.assert_array_equal(bits(res[i].cpu().numpy()), bits(r), err_msg=f"#{i} step {s}")
    fb.reset()
    r[:] = 0
    for s in range(3):
        kept = fb.step(gs[s][0]).cpu().numpy()
        want, _, _ = orc.feedback_step(kind, s, gs[s][1], r, tensors_of(sizes), 1,
                                       coeff_of(orc, ef, s), k_fraction=0.02, seed=11)
        np.testing.assert_array_equal(bits(kept), bits(want), err_msg=f"after reset, step {s}")
