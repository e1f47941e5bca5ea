"""GPU parity of the sm_100a path against the oracle and the reference.

Bars (BASELINE.json north_star):
  * shard boundaries, selection masks, K: bit-exact (test_planner.py);
  * fp64 instantiation of K1/K2: bit-exact against the REFERENCE's own
    covap_compress / covap_decompress / allreduce_mean (golden fixtures made
    by oracle/_ref, and the live library when present);
  * fp32 path: residuals, payload and synchronised gradients bit-exact against
    the fp32 restatement at P = 1 (FMA contraction controlled by
    __fmul_rn/__fadd_rn in the kernel and -ffp-contract=off in the oracle);
  * at full BASELINE sizes: exact integer conservation and K-window coverage.
Every call goes through the C-ABI (libcovap_b200.so) via the Python mirror.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)


def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)


def mk_model(c, sizes, cap):
    return c.ModelSpec([c.LayerSpec(f"l{i}", int(n)) for i, n in enumerate(sizes)], cap)


def dev_gen(c, key, n, kind, dtype):
    t = torch.empty(n, dtype=dtype, device=DEV)
    c.generate(t, key, kind)
    return t


def payload_of(plan, send, step):
    """Concatenate the selected tensors out of the (gapped) send buffer."""
    parts = []
    for t in plan.selection(step):
        ts = plan.tensors[t]
        br = plan.bucket_range(step, ts.bucket)
        off = br.send_offset + (ts.begin - br.sel_begin)
        parts.append(send[off:off + ts.numel()])
    if not parts:
        return np.zeros(0, send.dtype)
    return np.concatenate(parts)


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


# ------------------------------------------------------------------ K0

@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("kind", [0, 1])
def test_generator_bit_identical_to_host_twin(covap, orc, dtype, kind):
    npd = np.float32 if dtype == torch.float32 else np.float64
    for n in (1, 3, 5, 1000, 1 << 20, 12345677):
        key = orc.stream_key(7, 3, n)
        assert covap.stream_key(7, 3, n) == key
        d = dev_gen(covap, key, n, kind, dtype).cpu().numpy()
        assert np.array_equal(bits(d), bits(orc.generate(key, n, kind, 0, npd)))


# ------------------------------------------------------------------ fp64 == reference

@pytest.mark.parametrize("case", manifest()["compress"], ids=lambda c: c["name"])
def test_fp64_kernels_bit_exact_vs_reference_fixtures(covap, orc, case):
    fx = np.load(os.path.join(GOLDEN, f"compress_{case['name']}.npz"))
    plan = covap.BucketPlan(mk_model(covap, case["sizes"], case["cap"]), interval=case["K"],
                            rule=case["rule"])
    assert [[t.bucket, t.begin, t.end] for t in plan.tensors] == fx["tensors"].tolist()
    en, init, asc, rng = case["ef"]
    st = covap.CompressorState(plan, torch.float64, 0, covap.EfSchedule(bool(en), init, asc, rng))
    d = plan.total_numel()
    out = torch.empty(d, dtype=torch.float64, device=DEV)
    for s in range(case["steps"]):
        g = dev_gen(covap, orc.stream_key(case["seed"], 0, s), d, case["kind"], torch.float64)
        upd = covap.covap_compress(g, st)
        assert upd.selected == fx[f"selected_{s}"].tolist() and upd.step == s
        covap.covap_decompress(upd, out)
        torch.cuda.synchronize()
        send = st.send.cpu().numpy()
        assert np.array_equal(bits(payload_of(plan, send, s)), bits(fx[f"payload_{s}"]))
        assert np.array_equal(bits(st.residuals.cpu().numpy()), bits(fx[f"residual_{s}"]))
        assert np.array_equal(bits(out.cpu().numpy()), bits(fx[f"dense_{s}"]))
    assert st.num_steps == case["steps"]


@pytest.mark.parametrize("case", manifest()["session"], ids=lambda c: c["name"])
def test_fp64_sync_steps_bit_exact_vs_reference(covap, orc, case):
    """The reference's whole P-worker step (trainer.cpp:365-386) vs P device
    states on one GPU: K1 per worker, a fixed-order device sum of the packed
    send buffers (the allreduce, rank order as trainer.cpp:41-43), K2 x 1/P."""
    fx = np.load(os.path.join(GOLDEN, f"session_{case['name']}.npz"))
    plan = covap.BucketPlan(mk_model(covap, case["sizes"], case["cap"]), interval=case["K"],
                            rule=case["rule"])
    en, init, asc, rng = case["ef"]
    P = case["P"]
    states = [covap.CompressorState(plan, torch.float64, 0,
                                    covap.EfSchedule(bool(en), init, asc, rng)) for _ in range(P)]
    d = plan.total_numel()
    out = torch.empty(d, dtype=torch.float64, device=DEV)
    for s in range(case["steps"]):
        for w in range(P):
            g = dev_gen(covap, orc.stream_key(case["seed"], w, s), d, case["kind"], torch.float64)
            states[w].filter_pack(g)
        total = torch.zeros_like(states[0].send)
        for w in range(P):
            total += states[w].send  # rank order 0..P-1 (trainer.cpp:41-43)
        states[0].unpack(out, 1.0 / P, recv=total)
        for w in range(P):
            states[w].step_end()
        torch.cuda.synchronize()
        # (((0 + v0) + v1) + ...) * 1/P in rank order: bit-exact for every P
        assert np.array_equal(bits(out.cpu().numpy()), bits(fx[f"update_{s}"]))
        assert np.array_equal(bits(states[0].residuals.cpu().numpy()), bits(fx[f"residual0_{s}"]))


def test_fp64_live_reference_random_layouts(covap, orc, ref):
    rng = np.random.default_rng(11)
    for trial in range(12):
        n = int(rng.integers(1, 14))
        sizes = [int(x) for x in rng.integers(1, 30000, n)]
        cap = 4 * int(rng.integers(100, 40000))
        K = int(rng.integers(1, 9))
        rb, _, rts = ref.plan(sizes, cap, K)
        plan = covap.BucketPlan(mk_model(covap, sizes, cap), interval=K)
        assert [[t.bucket, t.begin, t.end] for t in plan.tensors] == [list(t) for t in rts]
        numels = [t[2] - t[1] for t in rts]
        d = sum(numels)
        st = covap.CompressorState(plan, torch.float64, 0, covap.EfSchedule(True, 0.3, 2, 0.2))
        r_ref = np.zeros(d)
        ns = 0
        out = torch.empty(d, dtype=torch.float64, device=DEV)
        for s in range(2 * K + 1):
            key = orc.stream_key(100 + trial, 0, s)
            g = dev_gen(covap, key, d, 0, torch.float64)
            p_ref, sel, ns = ref.compress(g.cpu().numpy(), numels, r_ref, ns, K, 0, (1, 0.3, 2, 0.2))
            upd = covap.covap_compress(g, st)
            covap.covap_decompress(upd, out)
            torch.cuda.synchronize()
            assert upd.selected == sel
            assert np.array_equal(payload_of(plan, st.send.cpu().numpy(), s), p_ref)
            assert np.array_equal(st.residuals.cpu().numpy(), r_ref)
            assert np.array_equal(out.cpu().numpy(), ref.decompress(p_ref, sel, numels))


# ------------------------------------------------------------------ fp32 == restatement

F32_CASES = [("resnet50", 4, 0, (1, 0.3, 100, 0.1), 6), ("resnet50", 8, 0, (1, 0.4, 1, 0.2), 9),
             ("vgg16", 4, 0, (1, 0.3, 1, 0.25), 5), ("vgg16", 3, 1, (0, 0.3, 100, 0.1), 4),
             ("tablev", 19, 0, (1, 0.5, 2, 0.1), 3), ("bert_large", 4, 0, (1, 0.3, 1, 0.3), 2),
             ("resnet50", 1, 0, (1, 0.3, 100, 0.1), 2)]


@pytest.mark.parametrize("name,K,rule,ef,steps", F32_CASES,
                         ids=[f"{c[0]}-K{c[1]}-r{c[2]}" for c in F32_CASES])
def test_fp32_full_layouts_bit_exact_vs_oracle(covap, orc, name, K, rule, ef, steps):
    """Full BASELINE layouts, fp32: send payload, residual arena and the
    synchronised gradient (P = 1: (0 + x) * 1) bit-exact against the fp32
    restatement, step after step (residual carried)."""
    m = covap.load_layout(name)
    plan = covap.plan_for(m, covap.CovapConfig(interval=K, rule=rule))
    tensors = [(t.bucket, t.begin, t.end) for t in plan.tensors]
    _, ots = orc.plan([l.param_count for l in m.layers], m.bucket_cap_bytes, K)
    assert [tuple(t) for t in ots] == tensors
    st = covap.CompressorState(plan, torch.float32, 0, covap.EfSchedule(bool(ef[0]), *ef[1:]))
    sync = covap.CovapSync(plan, None, torch.float32, 0, covap.EfSchedule(bool(ef[0]), *ef[1:]))
    d = plan.total_numel()
    r = np.zeros(d, np.float32)
    out = torch.empty(d, dtype=torch.float32, device=DEV)
    out2 = torch.empty(d, dtype=torch.float32, device=DEV)
    for s in range(steps):
        key = orc.stream_key(5, 0, s)
        g = dev_gen(covap, key, d, 0, torch.float32)
        upd = covap.covap_compress(g, st)
        covap.covap_decompress(upd, out)
        sync.sync(g, out2)
        keep = orc.select(s, K, len(tensors), rule)
        coeff = np.float32(orc.ef_coefficient(s, *ef[1:]))
        p = orc.compress(orc.generate(key, d, 0, 0, np.float32), r, tensors, keep, ef[0], coeff)
        dense = orc.decompress(orc.allreduce_mean(p[None, :]) if len(p) else p, tensors, keep, d,
                               np.float32)
        torch.cuda.synchronize()
        assert np.array_equal(bits(payload_of(plan, st.send.cpu().numpy(), s)), bits(p))
        assert np.array_equal(bits(st.residuals.cpu().numpy()), bits(r))
        assert np.array_equal(bits(out.cpu().numpy()), bits(orc.decompress(p, tensors, keep, d, np.float32)))
        assert np.array_equal(bits(out2.cpu().numpy()), bits(dense))
        assert np.array_equal(bits(sync.state.residuals.cpu().numpy()), bits(r))


def test_overlapped_schedule_equals_standalone(covap):
    """bucket_ready()/finish() on the side stream gives exactly sync()'s
    results, and the dense path gives allreduce_mean at P = 1."""
    for name, K in (("resnet50", 4), ("vgg16", 4), ("bert_large", 2)):
        plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
        a = covap.CovapSync(plan, None, torch.float32, 0)
        b = covap.CovapSync(plan, None, torch.float32, 0)
        d = plan.total_numel()
        oa = torch.empty(d, device=DEV)
        ob = torch.empty(d, device=DEV)
        for s in range(K + 1):
            g = torch.empty(d, device=DEV)
            covap.generate(g, covap.stream_key(9, 0, s))
            a.sync(g, oa)
            for bk in range(len(plan.buckets)):
                b.bucket_ready(bk, g, ob)
            b.finish()
            torch.cuda.synchronize()
            assert torch.equal(oa, ob)
            assert torch.equal(a.state.residuals, b.state.residuals)
        durs = b.last_comm_ms()
        assert len(durs) == len(plan.buckets)
        # dense baseline: out = (0 + g) * 1 at P = 1, in place
        g = torch.randn(d, device=DEV)
        g[::7] = -0.0
        dense = g.clone()
        for bk in range(len(plan.buckets)):
            b.dense_bucket_ready(bk, dense, dense)
        b.finish()
        torch.cuda.synchronize()
        assert torch.equal(dense, g + 0.0)
        assert not torch.signbit(dense[::7]).any()


# ------------------------------------------------------------------ edge cases

def test_edge_cases_small_and_ragged(covap, orc):
    """Unaligned bucket boundaries, 1-element layers, K > tensor count (empty
    phases: no payload, residual still written, zero output), signed zeros."""
    for sizes, cap, K in (([1], 4, 1), ([1, 2, 3], 4, 4), ([5, 1, 7, 3, 9], 12, 3),
                          ([33, 1, 1, 65, 127, 4097], 132, 16), ([300, 300, 300], 1200, 8),
                          ([4096, 3, 5, 4093], 16388, 2)):
        plan = covap.BucketPlan(mk_model(covap, sizes, cap), interval=K)
        tensors = [(t.bucket, t.begin, t.end) for t in plan.tensors]
        _, ots = orc.plan(sizes, cap, K)
        assert [tuple(t) for t in ots] == tensors
        st = covap.CompressorState(plan, torch.float32, 0, covap.EfSchedule(True, 0.5, 1, 0.25))
        d = plan.total_numel()
        r = np.zeros(d, np.float32)
        out = torch.empty(d, device=DEV)
        for s in range(2 * K + 1):
            key = orc.stream_key(31, 0, s)
            gh = orc.generate(key, d, 0, 0, np.float32)
            gh[::3] = -0.0
            g = torch.from_numpy(gh.copy()).to(DEV)
            upd = covap.covap_compress(g, st)
            covap.covap_decompress(upd, out)
            keep = orc.select(s, K, len(tensors))
            p = orc.compress(gh, r, tensors, keep, 1, np.float32(orc.ef_coefficient(s, 0.5, 1, 0.25)))
            torch.cuda.synchronize()
            assert np.array_equal(bits(payload_of(plan, st.send.cpu().numpy(), s)), bits(p))
            assert np.array_equal(bits(st.residuals.cpu().numpy()), bits(r))
            assert np.array_equal(bits(out.cpu().numpy()),
                                  bits(orc.decompress(p, tensors, keep, d, np.float32)))


def test_errors_on_device_calls(covap):
    plan = covap.plan_for(covap.load_layout("resnet50"), covap.CovapConfig(interval=4))
    st = covap.CompressorState(plan, torch.float32, 0)
    d = plan.total_numel()
    with pytest.raises(covap.InvalidState):
        covap.covap_compress(torch.zeros(d - 1, device=DEV), st)
    with pytest.raises(covap.InvalidInput):
        covap.covap_compress(torch.zeros(d, dtype=torch.float64, device=DEV), st)
    big = torch.zeros(d + 1, device=DEV)
    with pytest.raises(covap.InvalidInput):  # 4-byte offset: not 16-byte aligned
        st.filter_pack(big[1:])
    with pytest.raises(covap.InvalidInput):
        st.filter_pack(big[:d], b0=3, b1=2)
    with pytest.raises(covap.InvalidState):
        covap.covap_compress(big[:d], st, covap.CovapConfig(interval=2))


# ------------------------------------------------------------------ full-size properties

@pytest.mark.parametrize("name,K", [("bert_large", 4), ("vgg16", 8), ("resnet50", 16)])
def test_full_size_integer_conservation(covap, name, K):
    """Size-independent property at BASELINE sizes: with integer gradients and
    coeff = 1 (test_compress.cpp:223-245, acceptance.cpp:273-327) the sum of
    transmitted updates plus the residual store equals the sum of inputs
    exactly (every element is transmitted once per K-window, so after K steps
    the residual holds only what was accumulated since its tensor was sent)."""
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
    sync = covap.CovapSync(plan, None, torch.float32, 0, covap.EfSchedule(True, 1.0, 1, 0.0))
    d = plan.total_numel()
    inp = torch.zeros(d, device=DEV)
    sent = torch.zeros(d, device=DEV)
    g = torch.empty(d, device=DEV)
    out = torch.empty(d, device=DEV)
    for s in range(K):
        covap.generate(g, covap.stream_key(1, 0, s), 1)
        inp += g
        sync.sync(g, out)
        sent += out
    torch.cuda.synchronize()
    assert torch.equal(sent + sync.state.residuals, inp)


@pytest.mark.parametrize("fused", [True, False], ids=["k1f", "k1_k2"])
def test_beyond_2pow32_elements(covap, fused):
    """Maximum sizes: a 2-bucket layout of 2^31 + 7 and 2^31 + 5 fp32
    elements (> 2^32 in total, 17 GB per array) at K = 2, integer gradients,
    coeff = 1.  Element by element, out + r_new == g + r_old (exact in fp32
    for integers), out is zero outside the selected bucket and r is zero
    inside it — so no 32-bit index wraps anywhere in K1F, K1 or K2."""
    free, _ = torch.cuda.mem_get_info()
    sizes = [(1 << 31) + 7, (1 << 31) + 5]
    d = sum(sizes)
    if free < 7 * 4 * d:
        pytest.skip("needs ~120 GB of free device memory")
    plan = covap.BucketPlan(mk_model(covap, sizes, 1), interval=2)
    assert plan.total_numel() == d and len(plan.tensors) == 2
    sync = covap.CovapSync(plan, None, torch.float32, 0, covap.EfSchedule(True, 1.0, 1, 0.0),
                           fuse_single_rank=fused)
    g = torch.empty(d, device=DEV)
    out = torch.empty(d, device=DEV)
    b0 = plan.tensors[1].begin
    for s in range(3):
        covap.generate(g, covap.stream_key(5, 0, s), 1)
        r_old = sync.state.residuals.clone()
        sync.sync(g, out)
        r_new = sync.state.residuals
        sel = (0, b0) if s % 2 == 0 else (b0, d)
        step = 1 << 28
        for a in range(0, d, step):  # chunked: bounded temporaries
            e = min(d, a + step)
            assert torch.equal(out[a:e] + r_new[a:e], g[a:e] + r_old[a:e]), (s, a)
            lo, hi = max(a, sel[0]), min(e, sel[1])
            if lo < hi:
                assert not torch.any(r_new[lo:hi]), (s, a)
            for x0, x1 in ((a, min(e, sel[0])), (max(a, sel[1]), e)):
                if x0 < x1:
                    assert not torch.any(out[x0:x1]), (s, a)
        del r_old
    torch.cuda.synchronize()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("name,K", [("resnet50", 4), ("vgg16", 3), ("tablev", 19), ("resnet50", 1)])
def test_fused_single_rank_pass_equals_k1_k2(covap, dtype, name, K):
    """K1F (the one-rank sync pass) is bit-identical to K1 -> K2(mean, 1/1),
    also when the output overwrites the gradient in place."""
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
    ef = covap.EfSchedule(True, 0.3, 1, 0.2)
    a = covap.CompressorState(plan, dtype, 0, ef)
    b = covap.CompressorState(plan, dtype, 0, ef)
    d = plan.total_numel()
    oa = torch.empty(d, dtype=dtype, device=DEV)
    for s in range(K + 2):
        g = torch.empty(d, dtype=dtype, device=DEV)
        covap.generate(g, covap.stream_key(3, 0, s))
        g[::11] = -0.0
        a.filter_pack(g)
        a.unpack(oa, 1.0, True)
        a.step_end()
        gb = g.clone()
        b.filter_unpack(gb, gb)  # in place: out aliases grad
        b.step_end()
        torch.cuda.synchronize()
        assert torch.equal(oa.view(torch.int32 if dtype == torch.float32 else torch.int64),
                           gb.view(torch.int32 if dtype == torch.float32 else torch.int64))
        assert torch.equal(a.residuals, b.residuals)


@pytest.mark.parametrize("name,K,chunk,alias", [("resnet50", 4, 0, True), ("resnet50", 1, 1 << 20, False),
                                                ("vgg16", 4, 3 << 20, True)])
def test_host_pipeline_back_to_back(covap, name, K, chunk, alias):
    """Consecutive covap_sync_step_host calls chain chunk by chunk (uploads of
    step s + 1 overlap downloads of step s): issued back to back with no host
    synchronisation, every step's host output still equals the device step's —
    with the staging buffers aliased (an upload must wait for that chunk's
    download) and separate."""
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
    a = covap.CovapSync(plan, None, torch.float32, 0)
    b = covap.CovapSync(plan, None, torch.float32, 0)
    d = plan.total_numel()
    steps = K + 3
    g = torch.empty(d, device=DEV)
    outs = [torch.empty(d, device=DEV) for _ in range(steps)]
    hins = [torch.empty(d, pin_memory=True) for _ in range(steps)]
    houts = [torch.empty(d, pin_memory=True) for _ in range(steps)]
    dg = torch.empty(d, device=DEV)
    do = dg if alias else torch.empty(d, device=DEV)
    for s in range(steps):
        covap.generate(g, covap.stream_key(29, 0, s))
        hins[s].copy_(g)
        a.sync(g, outs[s])
    torch.cuda.synchronize()
    for s in range(steps):  # back to back
        b.sync_host(hins[s], houts[s], dg, do, chunk_elems=chunk)
    torch.cuda.synchronize()
    for s in range(steps):
        assert torch.equal(outs[s].cpu(), houts[s]), s
    assert torch.equal(a.state.residuals, b.state.residuals)


@pytest.mark.parametrize("name,K,chunk", [("resnet50", 1, 0), ("resnet50", 4, 1 << 20),
                                          ("vgg16", 4, 3 << 20), ("tablev", 19, 1 << 21)])
def test_host_pipeline_equals_device_sync(covap, name, K, chunk):
    """covap_sync_step_host (chunked H2D / kernels / D2H on three streams)
    gives exactly the device-resident step's output and residuals."""
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
    a = covap.CovapSync(plan, None, torch.float32, 0)
    b = covap.CovapSync(plan, None, torch.float32, 0)
    d = plan.total_numel()
    g = torch.empty(d, device=DEV)
    out = torch.empty(d, device=DEV)
    hin = torch.empty(d, pin_memory=True)
    hout = torch.empty(d, pin_memory=True)
    for s in range(K + 1):
        covap.generate(g, covap.stream_key(21, 0, s))
        hin.copy_(g)
        a.sync(g, out)
        b.sync_host(hin, hout, chunk_elems=chunk)
        torch.cuda.synchronize()
        assert torch.equal(out.cpu(), hout)
        assert torch.equal(a.state.residuals, b.state.residuals)


@pytest.mark.parametrize("name,K", [("resnet50", 4), ("vgg16", 4), ("tablev", 19), ("bert_large", 2)])
def test_multi_rank_code_path_on_one_gpu(covap, name, K):
    """The K1 -> NCCL allreduce -> K2 path every P > 1 rank runs, exercised on
    one GPU through a 1-rank NCCL communicator (fusion switched off): sync(),
    the per-bucket overlapped schedule, the chunked host pipeline and the
    dense path give exactly the fused single-rank results; the per-bucket
    collective timings and the CCR exchange go through NCCL."""
    comm = covap.Communicator(covap.Communicator.unique_id(), 1, 0, 0)
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
    ref = covap.CovapSync(plan, None, torch.float32, 0)
    a = covap.CovapSync(plan, comm, torch.float32, 0, fuse_single_rank=False)
    b = covap.CovapSync(plan, comm, torch.float32, 0, fuse_single_rank=False)
    c = covap.CovapSync(plan, comm, torch.float32, 0, fuse_single_rank=False)
    e = covap.CovapSync(plan, comm, torch.float32, 0, fuse_single_rank=False, pipeline=3)
    # the overlapped schedules with SMs left free for the collective
    f = covap.CovapSync(plan, comm, torch.float32, 0, fuse_single_rank=False, free_sms=40)
    h = covap.CovapSync(plan, comm, torch.float32, 0, fuse_single_rank=False, pipeline=3,
                        free_sms=20)
    d = plan.total_numel()
    g = torch.empty(d, device=DEV)
    o_ref, o_a, o_b, o_e, o_f, o_h = (torch.empty(d, device=DEV) for _ in range(6))
    hin = torch.empty(d, pin_memory=True)
    hout = torch.empty(d, pin_memory=True)
    for s in range(K + 1):
        covap.generate(g, covap.stream_key(33, 0, s))
        hin.copy_(g)
        ref.sync(g, o_ref)
        a.sync(g, o_a)
        for bk in range(len(plan.buckets)):
            b.bucket_ready(bk, g, o_b)
        b.finish()
        c.sync_host(hin, hout, chunk_elems=1 << 20)
        e.sync(g, o_e)  # pipelined bucket groups
        for bk in range(len(plan.buckets)):
            f.bucket_ready(bk, g, o_f)
        f.finish()
        h.sync(g, o_h)
        torch.cuda.synchronize()
        for o in (o_a, o_b, hout.to(DEV), o_e, o_f, o_h):
            assert torch.equal(o, o_ref)
        for st in (a, b, c, e, f, h):
            assert torch.equal(st.state.residuals, ref.state.residuals)
        durs = b.last_comm_ms()
        for bk in range(len(plan.buckets)):
            sel = plan.bucket_range(s, bk)
            assert (durs[bk] >= 0) == (sel.sel_end > sel.sel_begin)
    aligned, comp = comm.profile_exchange([1.5, 0.25, 3.0], 7.0)
    assert aligned == [1.5, 0.25, 3.0] and comp == 7.0
    dense = g.clone()
    for bk in range(len(plan.buckets)):
        a.dense_bucket_ready(bk, dense, dense)
    a.finish()
    torch.cuda.synchronize()
    assert torch.equal(dense, g + 0.0)
    comm.close()


@pytest.mark.parametrize("name,K", [("resnet50", 4), ("vgg16", 3)])
def test_padded_plan_equals_flat(covap, name, K):
    """A padded plan on a padded arena gives the flat plan's results, element
    for element, through sync() and through the bucket-local entry points."""
    m = covap.load_layout(name)
    fp = covap.plan_for(m, covap.CovapConfig(interval=K))
    pp = covap.plan_for(m, covap.CovapConfig(interval=K), pad=True)
    a = covap.CovapSync(fp, None, torch.float32, 0)
    b = covap.CovapSync(pp, None, torch.float32, 0)
    c = covap.CovapSync(pp, None, torch.float32, 0)
    n, dn = fp.total_numel(), pp.device_numel()
    idx = torch.cat([torch.arange(pp.device_begin(i), pp.device_begin(i) + bk.numel)
                     for i, bk in enumerate(pp.buckets)]).to(DEV)
    g = torch.empty(n, device=DEV)
    oa = torch.empty(n, device=DEV)
    gp = torch.zeros(dn, device=DEV)
    ob = torch.empty(dn, device=DEV)
    for s in range(K + 1):
        covap.generate(g, covap.stream_key(44, 0, s))
        gp[idx] = g
        a.sync(g, oa)
        b.sync(gp, ob)
        bufs = [g[fp.buckets[i].begin:fp.buckets[i].begin + bk.numel].clone()
                for i, bk in enumerate(pp.buckets)]
        for i, buf in enumerate(bufs):
            c.bucket_ready_local(i, buf, buf)
        c.finish()
        torch.cuda.synchronize()
        assert torch.equal(ob[idx], oa)
        assert torch.equal(torch.cat(bufs), oa)
        assert torch.equal(b.state.residuals[idx], a.state.residuals)
        assert torch.equal(c.state.residuals[idx], a.state.residuals)


def _virtual_ranks(covap, plan, P, dtype, ef, fused=True):
    """P ranks of the peer collective inside one process on one GPU: each has
    its own state and send buffers, its kernels run on its own stream, and
    the grids are capped so all P collectives are resident together."""
    states = [covap.CompressorState(plan, dtype, 0, ef) for _ in range(P)]
    groups = [covap.PeerGroup(st, P, r) for r, st in enumerate(states)]
    covap.PeerGroup.attach_local(groups)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for g in groups:
        g.set_limits(max_ctas=max(1, sms // (2 * P)), timeout_s=10.0)
        g.set_fused(fused)
    streams = [torch.cuda.Stream() for _ in range(P)]
    return states, groups, streams


@pytest.mark.parametrize("fused", [1, 0, 2], ids=["fused", "gather", "step"])
@pytest.mark.parametrize("case", manifest()["session"], ids=lambda c: c["name"])
def test_peer_collective_bit_exact_vs_reference(covap, orc, case, fused):
    """The NVLink load/store allreduce sums in rank order, so the whole
    P-worker step equals the reference's (trainer.cpp:365-386) bit for bit —
    for P = 2, 3 and 4 (fp64 fixtures from the reference library)."""
    fx = np.load(os.path.join(GOLDEN, f"session_{case['name']}.npz"))
    plan = covap.BucketPlan(mk_model(covap, case["sizes"], case["cap"]), interval=case["K"],
                            rule=case["rule"])
    en, init, asc, rng = case["ef"]
    P = case["P"]
    states, groups, streams = _virtual_ranks(covap, plan, P, torch.float64,
                                             covap.EfSchedule(bool(en), init, asc, rng), fused)
    d = plan.total_numel()
    outs = [torch.empty(d, dtype=torch.float64, device=DEV) for _ in range(P)]
    for s in range(case["steps"]):
        grads = [dev_gen(covap, orc.stream_key(case["seed"], w, s), d, case["kind"], torch.float64)
                 for w in range(P)]
        torch.cuda.synchronize()
        for w in range(P):
            groups[w].sync(grads[w], outs[w], streams[w])
        torch.cuda.synchronize()
        for g in groups:
            g.check()
        for w in range(P):
            assert np.array_equal(bits(outs[w].cpu().numpy()), bits(fx[f"update_{s}"])), (s, w)
        assert np.array_equal(bits(states[0].residuals.cpu().numpy()), bits(fx[f"residual0_{s}"]))


@pytest.mark.parametrize("name,K,P,fused", [("resnet50", 4, 2, 1), ("vgg16", 4, 4, 1),
                                            ("resnet50", 1, 8, 1), ("vgg16", 3, 3, 0),
                                            ("tablev", 19, 2, 1), ("resnet50", 4, 2, 2),
                                            ("vgg16", 4, 4, 2), ("resnet50", 8, 3, 2),
                                            ("resnet50", 1, 8, 2), ("tablev", 19, 2, 2)])
def test_peer_collective_fp32_full_layouts(covap, orc, name, K, P, fused):
    """fp32 at BASELINE sizes, P virtual ranks: every rank's synchronised
    gradient equals the rank-ordered oracle mean, bit for bit."""
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
    ef = covap.EfSchedule(True, 0.3, 1, 0.2)
    states, groups, streams = _virtual_ranks(covap, plan, P, torch.float32, ef, fused)
    d = plan.total_numel()
    tensors = [(t.bucket, t.begin, t.end) for t in plan.tensors]
    rs = [np.zeros(d, np.float32) for _ in range(P)]
    outs = [torch.empty(d, device=DEV) for _ in range(P)]
    # K = 8 walks every phase, the empty ones (ResNet-50 phases 5-7) included,
    # and reuses each parity buffer several times
    for s in range(K + 1 if K == 8 else 3):
        keys = [orc.stream_key(9, w, s) for w in range(P)]
        grads = [dev_gen(covap, k, d, 0, torch.float32) for k in keys]
        torch.cuda.synchronize()
        for w in range(P):
            groups[w].sync(grads[w], outs[w], streams[w])
        keep = orc.select(s, K, len(tensors))
        coeff = np.float32(orc.ef_coefficient(s, 0.3, 1, 0.2))
        pays = [orc.compress(orc.generate(keys[w], d, 0, 0, np.float32), rs[w], tensors, keep, 1, coeff)
                for w in range(P)]
        want = orc.decompress(orc.allreduce_mean(np.stack(pays)), tensors, keep, d, np.float32)
        torch.cuda.synchronize()
        for g in groups:
            g.check()
        for w in range(P):
            assert np.array_equal(bits(outs[w].cpu().numpy()), bits(want)), (s, w)
            assert np.array_equal(bits(states[w].residuals.cpu().numpy()), bits(rs[w]))


@pytest.mark.parametrize("name,K,fuse", [("resnet50", 1, True), ("resnet50", 4, True),
                                         ("vgg16", 4, False), ("tablev", 19, True),
                                         ("vgg16", 3, True)])
def test_fused_sgd_step_bit_exact(covap, orc, name, K, fuse):
    """The sync step ending in the SGD update (trainer.cpp:408-409) — one rank
    K1F+SGD, or K1 -> K2+SGD — equals the oracle's synchronised gradient
    followed by params - lr * update (fp32, mul then sub), bit for bit, with
    the residual carried; unselected parameters are untouched."""
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
    ef = covap.EfSchedule(True, 0.3, 1, 0.2)
    sync = covap.CovapSync(plan, None, torch.float32, 0, ef, fuse_single_rank=fuse)
    d = plan.total_numel()
    tensors = [(t.bucket, t.begin, t.end) for t in plan.tensors]
    lr = 0.0625 * 1.1
    params = dev_gen(covap, 99, d, 0, torch.float32)
    p_ref = params.cpu().numpy().copy()
    r = np.zeros(d, np.float32)
    for s in range(K + 2):
        key = orc.stream_key(12, 0, s)
        g = dev_gen(covap, key, d, 0, torch.float32)
        sync.sync_sgd(g, params, lr)
        keep = orc.select(s, K, len(tensors))
        p = orc.compress(orc.generate(key, d, 0, 0, np.float32), r, tensors, keep, 1,
                         np.float32(orc.ef_coefficient(s, 0.3, 1, 0.2)))
        upd = orc.decompress(orc.allreduce_mean(p[None, :]) if len(p) else p, tensors, keep, d,
                             np.float32)
        with np.errstate(all="ignore"):
            p_ref = (p_ref - (np.float32(lr) * upd).astype(np.float32)).astype(np.float32)
        torch.cuda.synchronize()
        assert np.array_equal(bits(params.cpu().numpy()), bits(p_ref)), s
        assert np.array_equal(bits(sync.state.residuals.cpu().numpy()), bits(r)), s


def test_timeline_and_chrome_trace(covap, tmp_path):
    """The real-timeline profiler: per-bucket K1 / collective / K2 marks of an
    overlapped step are ordered and non-overlapping per stream; the Chrome
    trace is written; overlap_schedule over the measured times predicts the
    step."""
    import json
    from paper_2311_04499_b200 import trace
    comm = covap.Communicator(covap.Communicator.unique_id(), 1, 0, 0)
    plan = covap.plan_for(covap.load_layout("resnet50"), covap.CovapConfig(interval=4))
    for fuse in (True, False):
        sync = covap.CovapSync(plan, None if fuse else comm, torch.float32, 0, fuse_single_rank=fuse)
        d = plan.total_numel()
        g, out = torch.empty(d, device=DEV), torch.empty(d, device=DEV)
        covap.generate(g, 5)

        def step():
            for b in range(len(plan.buckets)):
                covap.spin(200.0)
                sync.bucket_ready(b, g, out)
            sync.finish()
        step()
        tl = trace.record_step(sync, step)
        assert len(tl) == len(plan.buckets) and tl[0]["k1_start"] == 0.0
        for b, r in enumerate(tl):
            assert r["k1_end"] >= r["k1_start"]
            if b:
                assert r["k1_start"] >= tl[b - 1]["k1_end"] + 0.15  # the 200 us spin in between
            if fuse:
                assert r["comm_start"] == -1.0
            else:
                assert r["k1_end"] <= r["comm_start"] + 1e-3 <= r["comm_end"] + 2e-3 <= r["k2_end"] + 3e-3
        trace.chrome_trace(str(tmp_path / "t.json"), tl)
        doc = json.load(open(tmp_path / "t.json"))
        assert len(doc["traceEvents"]) == len(plan.buckets) * (1 if fuse else 3)
        mc = trace.model_check(tl, [0.2] * len(tl), tl[-1]["k2_end"])
        assert mc["predicted_step_ms"] > 0.9
    comm.close()


@pytest.mark.parametrize("name,K", [("resnet50", 4), ("vgg16", 3)])
def test_checkpoint_resume_equals_uninterrupted(covap, name, K):
    """CompressorState is the residual arena plus num_steps (compress.hpp:42-47):
    saving both mid-run (host copy) and restoring them into a fresh state
    continues the run bit for bit — the EF coefficient schedule and the
    round-robin phase resume from num_steps."""
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
    ef = covap.EfSchedule(True, 0.3, 2, 0.2)
    a = covap.CovapSync(plan, None, torch.float32, 0, ef)
    d = plan.total_numel()
    g = torch.empty(d, device=DEV)
    oa, ob = torch.empty(d, device=DEV), torch.empty(d, device=DEV)
    for s in range(K + 1):
        covap.generate(g, covap.stream_key(41, 0, s))
        a.sync(g, oa)
    torch.cuda.synchronize()
    saved_r, saved_step = a.state.residuals.cpu(), a.state.num_steps  # the checkpoint
    b = covap.CovapSync(plan, None, torch.float32, 0, ef)
    b.state.residuals.copy_(saved_r.to(DEV))
    b.state.num_steps = saved_step
    for s in range(K + 1, 2 * K + 3):
        covap.generate(g, covap.stream_key(41, 0, s))
        a.sync(g, oa)
        b.sync(g, ob)
        torch.cuda.synchronize()
        assert torch.equal(oa, ob), s
        assert torch.equal(a.state.residuals, b.state.residuals), s


# ------------------------------------------------------------------ allreduce_mean (a11)

def _signed_zero_input(n, dtype, seed):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(n, generator=g, dtype=torch.float64).to(dtype)
    x[::7] = -0.0
    x[1::7] = 0.0
    x[2::11] = torch.tensor(-1e-30, dtype=torch.float64).to(dtype)
    return x


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_allreduce_mean_python_boundary(covap, orc, dtype):
    """covap.allreduce_mean (trainer.cpp:35-47) through covap_comm_allreduce_mean:
    (0 + sum) * (1/P) — with no communicator and with a 1-rank NCCL
    communicator, into a new tensor and in place; -0.0 comes out as +0.0 as
    in the reference (the sum starts from +0.0, trainer.cpp:41)."""
    npd = np.float32 if dtype == torch.float32 else np.float64
    comm = covap.Communicator(covap.Communicator.unique_id(), 1, 0, 0)
    for n in (1, 3, 17, 1000, 1 << 20, 5_000_001):
        x = _signed_zero_input(n, dtype, n)
        want = orc.allreduce_mean(x.numpy()[None, :].astype(npd))
        for c in (None, comm):
            buf = x.to(DEV)
            out = covap.allreduce_mean(buf, c)
            torch.cuda.synchronize()
            assert np.array_equal(bits(out.cpu().numpy()), bits(want)), (n, c)
            zeros = x.numpy() == 0
            assert not np.signbit(out.cpu().numpy()[zeros]).any()  # -0.0 -> +0.0
            inplace = x.to(DEV)
            covap.allreduce_mean(inplace, c, out=inplace)
            torch.cuda.synchronize()
            assert np.array_equal(bits(inplace.cpu().numpy()), bits(want))
    empty = torch.empty(0, dtype=dtype, device=DEV)
    assert covap.allreduce_mean(empty).numel() == 0
    with pytest.raises(covap.InvalidInput):
        covap.allreduce_mean(torch.zeros(4, dtype=dtype, device=DEV), None,
                             out=torch.zeros(3, dtype=dtype, device=DEV))
    comm.close()


def test_allreduce_mean_rows_bit_exact_vs_reference(covap, ref):
    """The kernel behind the C++ drop-in covap::allreduce_mean
    (covap_cxx.cpp -> covap_mean_rows): P = 1..8 in-process worker vectors,
    fp64, against the reference's own allreduce_mean, bit for bit; plus the
    reference's known answers (test_trainer.cpp:45-49)."""
    import ctypes
    from paper_2311_04499_b200 import _lib as L

    def mean_rows(rows):
        rows = np.ascontiguousarray(rows, np.float64)
        P, n = rows.shape
        d_rows = torch.from_numpy(rows.reshape(-1).copy()).to(DEV)
        d_out = torch.empty(n, dtype=torch.float64, device=DEV)
        L.lib().covap_mean_rows(0, L.F64, ctypes.c_void_p(d_rows.data_ptr()),
                                ctypes.c_void_p(d_out.data_ptr()), P, n, None)
        torch.cuda.synchronize()
        return d_out.cpu().numpy()

    assert mean_rows([[1, 2], [3, 4]]).tolist() == [2, 3]
    assert mean_rows([[5, 6, 7]]).tolist() == [5, 6, 7]
    for P in range(1, 9):
        for n in (1, 5, 4099, 300_007):
            rows = np.stack([_signed_zero_input(n, torch.float64, 100 * P + w).numpy()
                             * (10.0 ** (w - 3)) for w in range(P)])
            rows[:, 3::13] = -0.0  # all-negative-zero columns: the reference gives +0.0
            got, want = mean_rows(rows), ref.allreduce_mean(rows)
            assert np.array_equal(bits(got), bits(want)), (P, n)


# ------------------------------------------------------------------ fp32 vs the fp64 reference

@pytest.mark.parametrize("name,K", [("resnet50", 4), ("vgg16", 4), ("bert_large", 4)])
def test_fp32_path_normwise_vs_fp64_reference(covap, orc, name, K):
    """the fp32 sync path against the REFERENCE's fp64
    covap_compress / allreduce_mean / covap_decompress (compress.cpp:50-103,
    trainer.cpp:35-47; oracle/_ref, else its pinned fp64 restatement) on the
    same gradients widened to fp64, default EF schedule (0.3, 100, 0.1), full
    BASELINE layouts: ||a - b||_2 / ||b||_2 <= 1e-6 for the synchronised
    gradient and the residual arena at every step of a K + 1 step run.
    (Per-element relative error is unbounded — cancellation in g + c*r —
    so the north star's 1e-6 is normwise; SURVEY §7 hard part 1.)"""
    from oracle.oracle import REF_SO, Ref, RefSession
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
    sync = covap.CovapSync(plan, None, torch.float32, 0)  # default EfSchedule
    numels = [t.numel() for t in plan.tensors]
    tensors = [(t.bucket, t.begin, t.end) for t in plan.tensors]
    d = plan.total_numel()
    sess = RefSession(Ref(), numels, 1, K) if os.path.exists(REF_SO) else None
    r64 = np.zeros(d)
    g, out = torch.empty(d, device=DEV), torch.empty(d, device=DEV)

    def rel(a, b):
        nb = np.linalg.norm(b)
        return np.linalg.norm(a.astype(np.float64) - b) / (nb if nb > 0 else 1.0)

    worst = 0.0
    for s in range(K + 1):
        covap.generate(g, covap.stream_key(61, 0, s))
        sync.sync(g, out)
        g64 = g.cpu().numpy().astype(np.float64)
        if sess is not None:
            upd, res, _ = sess.step(g64[None, :], want_residual=True)
        else:
            keep = orc.select(s, K, len(tensors))
            p = orc.compress(g64, r64, tensors, keep, 1, orc.ef_coefficient(s))
            upd = orc.decompress(orc.allreduce_mean(p[None, :]) if len(p) else p, tensors, keep,
                                 d, np.float64)
            res = r64
        torch.cuda.synchronize()
        e_out = rel(out.cpu().numpy(), upd)
        e_res = rel(sync.state.residuals.cpu().numpy(), res)
        worst = max(worst, e_out, e_res)
        assert e_out <= 1e-6 and e_res <= 1e-6, (s, e_out, e_res)
    if sess is not None:
        sess.close()
    assert worst > 0.0  # fp32 really differs from fp64 (the comparison is not vacuous)


# ------------------------------------------------------------------ buffer parity

@pytest.mark.parametrize("fused", [0, 1], ids=["gather", "fused"])
def test_peer_back_to_back_across_empty_phases(covap, orc, fused):
    """ResNet-50 at K = 8 has empty phases 5-7 (no collective, no barrier):
    steps 4 and 12 and 8 and 16 must still not share a send buffer a slower
    peer may be reading.  Two virtual ranks run 17 steps back to back with
    no host synchronisation; every step's output (copied aside on each rank's
    stream) and the final residuals equal the rank-ordered oracle."""
    K, P, S = 8, 2, 17
    plan = covap.plan_for(covap.load_layout("resnet50"), covap.CovapConfig(interval=K))
    ef = covap.EfSchedule(True, 0.3, 1, 0.2)
    states, groups, streams = _virtual_ranks(covap, plan, P, torch.float32, ef, fused)
    d = plan.total_numel()
    tensors = [(t.bucket, t.begin, t.end) for t in plan.tensors]
    grads = [[dev_gen(covap, orc.stream_key(17, w, s), d, 0, torch.float32) for s in range(S)]
             for w in range(P)]
    outs = [[torch.empty(d, device=DEV) for _ in range(S)] for _ in range(P)]
    tmp = [torch.empty(d, device=DEV) for _ in range(P)]
    torch.cuda.synchronize()
    for s in range(S):
        for w in range(P):
            groups[w].sync(grads[w][s], tmp[w], streams[w])
            with torch.cuda.stream(streams[w]):
                outs[w][s].copy_(tmp[w])
        if s % 3 == 0:  # rank 1 falls behind: give rank 0 a head start
            streams[1].wait_stream(streams[1])
            covap.spin(300.0, 1, streams[1])
    torch.cuda.synchronize()
    for g in groups:
        g.check()
    rs = [np.zeros(d, np.float32) for _ in range(P)]
    for s in range(S):
        keep = orc.select(s, K, len(tensors))
        coeff = np.float32(orc.ef_coefficient(s, 0.3, 1, 0.2))
        pays = [orc.compress(grads[w][s].cpu().numpy(), rs[w], tensors, keep, 1, coeff)
                for w in range(P)]
        mean = orc.allreduce_mean(np.stack(pays)) if len(pays[0]) else pays[0]
        want = orc.decompress(mean, tensors, keep, d, np.float32)
        for w in range(P):
            assert np.array_equal(bits(outs[w][s].cpu().numpy()), bits(want)), (s, w)
    for w in range(P):
        assert np.array_equal(bits(states[w].residuals.cpu().numpy()), bits(rs[w]))


# ------------------------------------------------------------------ K1 zero fill + selected-only K2

@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("name,K", [("resnet50", 4), ("vgg16", 4), ("tablev", 19),
                                    ("resnet50", 8), ("bert_large", 2)])
def test_zero_filling_k1_and_selected_k2_equal_full_k2(covap, dtype, name, K):
    """The multi-rank step's split — K1 also writes out = 0 for unselected
    slots (compress.cpp:91 moved ahead of the allreduce), K2 then writes only
    the selected slots — equals K1 -> full K2 bit for bit at every phase
    (empty phases included), into a NaN-poisoned output and in place (out
    aliasing the gradient, the DDP-bucket case)."""
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
    ef = covap.EfSchedule(True, 0.3, 1, 0.2)
    a = covap.CompressorState(plan, dtype, 0, ef)
    b = covap.CompressorState(plan, dtype, 0, ef)
    c = covap.CompressorState(plan, dtype, 0, ef)
    d = plan.total_numel()
    g = torch.empty(d, dtype=dtype, device=DEV)
    oa = torch.empty(d, dtype=dtype, device=DEV)
    ob = torch.empty(d, dtype=dtype, device=DEV)
    for s in range(K + 1):
        covap.generate(g, covap.stream_key(71, 0, s))
        ob.fill_(float("nan"))
        gc = g.clone()
        a.filter_pack(g)
        a.unpack(oa, 0.5, True)
        b.filter_pack(g, out=ob)
        b.unpack(ob, 0.5, True, selected_only=True)
        c.filter_pack(gc, out=gc)  # in place
        c.unpack(gc, 0.5, True, selected_only=True)
        for st in (a, b, c):
            st.step_end()
        torch.cuda.synchronize()
        assert torch.equal(oa, ob), s
        assert torch.equal(oa, gc), s
        assert torch.equal(a.residuals, b.residuals) and torch.equal(a.residuals, c.residuals)
        se, _ = plan.send_elems(s)
        assert torch.equal(a.send[:se], b.send[:se])


@pytest.mark.parametrize("sizes,cap,K", [
    ([1001, 77, 65539, 3, 300007, 12345, 5, 777777], 1 << 20, 1),   # one run across odd buckets
    ([1001, 77, 65539, 3, 300007, 12345, 5, 777777], 1 << 20, 3),
    ([4099] * 7 + [1_000_003, 33, 250_001], 1 << 16, 2),             # sharded, tiny buckets
    ([2_000_001, 5, 9, 1_500_007], 4 << 20, 4),
])
def test_selected_unpack_per_bucket_ragged(covap, sizes, cap, K):
    """The send-space-tiled selected-only unpack clipped to one bucket at a
    time (covap_bucket_ready's K2) on layouts whose buckets start at odd
    offsets and whose runs span several buckets: every bucket-local K2 plus
    the zero-filling K1 equals the full K1 -> K2, bit for bit, fp32 and fp64."""
    for dtype in (torch.float32, torch.float64):
        plan = covap.BucketPlan(mk_model(covap, sizes, cap), interval=K)
        ef = covap.EfSchedule(True, 0.3, 1, 0.2)
        a = covap.CompressorState(plan, dtype, 0, ef)
        b = covap.CompressorState(plan, dtype, 0, ef)
        d = plan.total_numel()
        g = torch.empty(d, dtype=dtype, device=DEV)
        oa = torch.empty(d, dtype=dtype, device=DEV)
        ob = torch.empty(d, dtype=dtype, device=DEV)
        nb = len(plan.buckets)
        for s in range(K + 1):
            covap.generate(g, covap.stream_key(72, 0, s))
            ob.fill_(float("nan"))
            a.filter_pack(g)
            a.unpack(oa, 0.25, True)
            for bk in range(nb):
                b.filter_pack(g, bk, bk + 1, out=ob)
            for bk in reversed(range(nb)):
                b.unpack(ob, 0.25, True, bk, bk + 1, selected_only=True)
            a.step_end()
            b.step_end()
            torch.cuda.synchronize()
            assert torch.equal(oa, ob), (s, dtype)
            assert torch.equal(a.residuals, b.residuals)


@pytest.mark.parametrize("name,K", [("resnet50", 4), ("vgg16", 4)])
def test_symmetric_send_window_same_results(covap, name, K):
    """The send buffer moved to an NCCL symmetric window (ncclMemAlloc +
    ncclCommWindowRegister, the NVLS / symmetric-kernel path at P > 1) gives
    the same synchronised gradients and residuals as the plain buffer, through
    the multi-rank step on a 1-rank communicator; destroying the communicator
    before the state is safe."""
    comm = covap.Communicator(covap.Communicator.unique_id(), 1, 0, 0)
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
    a = covap.CovapSync(plan, comm, torch.float32, 0, fuse_single_rank=False)
    try:
        b = covap.CovapSync(plan, comm, torch.float32, 0, fuse_single_rank=False, symmetric=True)
    except covap.NcclError as e:  # reported, not hidden: NCCL builds without window support
        comm.close()
        pytest.skip(f"NCCL refused a symmetric window on this box: {e}")
    d = plan.total_numel()
    g = torch.empty(d, device=DEV)
    oa, ob = torch.empty(d, device=DEV), torch.empty(d, device=DEV)
    for s in range(K + 1):
        covap.generate(g, covap.stream_key(81, 0, s))
        a.sync(g, oa)
        b.sync(g, ob)
        torch.cuda.synchronize()
        assert torch.equal(oa, ob), s
        assert torch.equal(a.state.residuals, b.state.residuals), s
    comm.close()  # deregisters the window
    del b
    torch.cuda.synchronize()
