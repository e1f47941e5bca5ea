"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

Every number in the fixtures comes out of oracle/_ref/libcovap_ref.so, i.e.
the reference's own model.cpp / compress.cpp / trainer.cpp / perf.cpp /
sim.cpp compiled from its sources; inputs come from the splitmix64 stream
generator (oc_generate_f64), whose seeds are stored next to the outputs so
tests can regenerate them bit-identically on any host.

Outputs:
  plans.json       bucket plans / medians / effective tensors for the
                   BASELINE layouts and seeded random models at many K
  selection.json   select_tensors at many (step, K, count, rule)
  ef.json          ef_coefficient schedules
  ccr.json         ccr / choose_interval / profile_ccr cases
  compress_*.npz   multi-step covap_compress traces (payload, selected,
                   residual per step) on seeded fp64 gradients
  session_*.npz    whole P-worker sync steps (trainer.cpp:365-386)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, Ref, RefSession, OracleError  # noqa: E402

LAYOUTS = ["resnet50", "vgg16", "bert_large", "tablev"]
KS = [1, 2, 3, 4, 5, 8, 16, 19, 25, 64]


def layout(name):
    with open(os.path.join(ROOT, "paper_2311_04499_b200", "layouts", name + ".json")) as f:
        doc = json.load(f)
    return [l["param_count"] for l in doc["layers"]], doc["bucket_cap_bytes"]


def splitmix(seed):
    state = [seed & (2**64 - 1)]

    def nxt():
        state[0] = (state[0] + 0x9e3779b97f4a7c15) & (2**64 - 1)
        z = state[0]
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & (2**64 - 1)
        return z ^ (z >> 31)
    return nxt


def main():
    ref = Ref()
    orc = Oracle()

    # -- plans -------------------------------------------------------------
    plans = []
    for name in LAYOUTS:
        sizes, cap = layout(name)
        for K in KS:
            for shard in (0, 1):
                b, tw, ts = ref.plan(sizes, cap, K, shard)
                plans.append({"case": name, "layers": None, "layout": name, "cap": cap, "K": K,
                              "shard": shard, "buckets": b, "twice_median": tw, "tensors": ts})
    rng = splitmix(4242)
    for trial in range(80):
        n = 1 + rng() % 30
        sizes = [1 + rng() % 200000 for _ in range(n)]
        cap = 4 * (1 + rng() % 150000)
        K = 1 + rng() % 24
        for shard in (0, 1):
            b, tw, ts = ref.plan(sizes, cap, K, shard)
            plans.append({"case": f"random{trial}", "layers": sizes, "layout": None, "cap": cap,
                          "K": K, "shard": shard, "buckets": b, "twice_median": tw, "tensors": ts})
    # singleton buckets: exercise the even-count median quirk (n = 2, 4, 6 ...)
    for n in range(1, 13):
        sizes = [1000 + (rng() % 50000) for _ in range(n)]
        b, tw, ts = ref.plan(sizes, 4, 1000000, 1)
        plans.append({"case": f"singletons{n}", "layers": sizes, "layout": None, "cap": 4,
                      "K": 1000000, "shard": 1, "buckets": b, "twice_median": tw, "tensors": ts})
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(plans, f)

    # -- selection ---------------------------------------------------------
    sel = []
    for K in (1, 2, 3, 4, 7, 8, 16):
        for count in (1, 5, 8, 23, 53):
            for step in (0, 1, 2, 3, 5, 17, 123, 10**6 + 3):
                for rule in (0, 1):
                    sel.append({"step": step, "K": K, "count": count, "rule": rule,
                                "selected": ref.select(step, K, count, rule)})
    with open(os.path.join(HERE, "selection.json"), "w") as f:
        json.dump(sel, f)

    # -- EF schedule -------------------------------------------------------
    ef = []
    for sched in ((0.3, 100, 0.1), (0.2, 100, 0.1), (1.0, 1, 0.0), (0.4, 3, 0.2), (0.05, 7, 0.3)):
        for step in (0, 1, 2, 3, 99, 100, 101, 350, 699, 700, 1000, 10**6):
            ef.append({"sched": sched, "step": step,
                       "coeff": ref.ef_coefficient(step, 1, *sched)})
    with open(os.path.join(HERE, "ef.json"), "w") as f:
        json.dump(ef, f)

    # -- CCR ---------------------------------------------------------------
    ccr = {"ccr": [], "interval": [], "profile": []}
    for comm, comp in ((280, 135), (842, 210), (0, 100), (0, 0), (10, 0), (-1, 5), (3.5, 1.0),
                       (1e-9, 1.0), (7.0, 7.0)):
        try:
            ccr["ccr"].append({"comm": comm, "comp": comp, "value": ref.ccr(comm, comp)})
        except OracleError as e:
            ccr["ccr"].append({"comm": comm, "comp": comp, "error": e.code})
    for c in (280 / 135, 4.0, 3.5, 0.4, 0.0, 1.0, 1.0000001, 16.0, 15.2, -0.5):
        try:
            ccr["interval"].append({"ccr": c, "value": ref.choose_interval(c)})
        except OracleError as e:
            ccr["interval"].append({"ccr": c, "error": e.code})
    rng = splitmix(77)
    for trial in range(20):
        W = 1 + rng() % 6
        C = 1 + rng() % 9
        starts = [[(rng() % 4000) * 0.25 for _ in range(C)] for _ in range(W)]
        ends = [max(starts[w][c] for w in range(W)) + (1 + rng() % 400) * 0.25 for c in range(C)]
        comp = (1 + rng() % 800) * 0.25
        a, naive, cc, k = ref.profile_ccr(starts, ends, comp)
        ccr["profile"].append({"starts": starts, "ends": ends, "comp": comp, "aligned": a,
                               "naive": naive, "ccr": cc, "interval": k})
    # overlap_schedule (perf.cpp:63-103): random per-tensor times, with and
    # without compress blocks and with a communicated mask
    ccr["overlap"] = []
    for trial in range(24):
        n = 1 + rng() % 12
        comp = [(1 + rng() % 64) * 0.25 for _ in range(n)]
        comm = [(rng() % 128) * 0.25 for _ in range(n)]
        compress = [(rng() % 8) * 0.125 for _ in range(n)] if trial % 2 else None
        sent = [int(rng() % 3 != 0) for _ in range(n)] if trial % 3 else None
        before = (rng() % 40) * 0.5
        res = ref.overlap_schedule(before, comp, compress, comm, sent)
        ccr["overlap"].append({"before": before, "comp": comp, "compress": compress, "comm": comm,
                               "communicated": sent, **res})
    with open(os.path.join(HERE, "ccr.json"), "w") as f:
        json.dump(ccr, f)

    # -- compress traces (fp64, reference covap_compress) --------------------
    traces = [
        # name, layer sizes, cap bytes, K, rule, ef, kind, steps
        ("small_k3", [37, 5, 129, 64, 1, 300, 77, 2, 515], 600, 3, 0, (1, 0.3, 100, 0.1), 0, 12),
        ("small_k4_plus", [37, 5, 129, 64, 1, 300, 77, 2, 515], 600, 4, 1, (1, 0.4, 3, 0.2), 0, 12),
        ("sharded_k4", [4000, 12, 9000, 33, 700, 1500], 4 * 2000, 4, 0, (1, 0.4, 3, 0.2), 0, 10),
        ("ef_off_k2", [4000, 12, 9000, 33, 700, 1500], 4 * 2000, 2, 0, (0, 0.3, 100, 0.1), 0, 6),
        ("int_k3_full", [1000, 999, 1001, 17, 4096], 4 * 1100, 3, 0, (1, 1.0, 1, 0.0), 1, 30),
        ("k1_dense", [513, 77, 1030], 4 * 700, 1, 0, (1, 0.3, 100, 0.1), 0, 4),
        ("k8_empty_phases", [300, 300, 300], 4 * 300, 8, 0, (1, 0.5, 2, 0.25), 0, 16),
    ]
    manifest = []
    for name, sizes, cap, K, rule, efp, kind, steps in traces:
        buckets, tw, tensors = ref.plan(sizes, cap, K)
        numels = [t[2] - t[1] for t in tensors]
        d = sum(numels)
        residual = np.zeros(d)
        ns = 0
        out = {"numels": np.array(numels, np.uint64), "tensors": np.array(tensors, np.uint64)}
        seed = 1000 + len(manifest)
        for s in range(steps):
            g = orc.generate(orc.stream_key(seed, 0, s), d, kind, 0, np.float64)
            payload, selected, ns = ref.compress(g, numels, residual, ns, K, rule, efp)
            dense = ref.decompress(payload, selected, numels)
            out[f"payload_{s}"] = payload
            out[f"selected_{s}"] = np.array(selected, np.uint64)
            out[f"residual_{s}"] = residual.copy()
            out[f"dense_{s}"] = dense
        np.savez_compressed(os.path.join(HERE, f"compress_{name}.npz"), **out)
        manifest.append({"name": name, "sizes": sizes, "cap": cap, "K": K, "rule": rule,
                         "ef": efp, "kind": kind, "steps": steps, "seed": seed})

    # -- whole sync steps, P workers (trainer.cpp:365-386) -------------------
    sessions = [
        ("p2_k3", [37, 5, 129, 64, 1, 300, 77, 2, 515], 600, 3, 0, (1, 0.3, 100, 0.1), 0, 2, 9),
        ("p4_sharded_k4", [4000, 12, 9000, 33, 700, 1500], 8000, 4, 0, (1, 0.4, 3, 0.2), 0, 4, 8),
        ("p3_int_k2", [1000, 999, 1001, 17, 4096], 4400, 2, 1, (1, 1.0, 1, 0.0), 1, 3, 6),
        # eight workers (one B200 box), kPlusStep, five tensors
        ("p8_plus_k5", [513, 2048, 77, 1500, 4096, 9, 640, 3000, 1200], 9000, 5, 1,
         (1, 0.3, 2, 0.15), 0, 8, 11),
        # more phases than tensors: empty selections on some steps, five workers
        ("p5_k8_empty", [700, 5000, 300, 2500], 5200, 8, 0, (1, 0.5, 4, 0.1), 0, 5, 10),
    ]
    smanifest = []
    for name, sizes, cap, K, rule, efp, kind, P, steps in sessions:
        buckets, tw, tensors = ref.plan(sizes, cap, K)
        numels = [t[2] - t[1] for t in tensors]
        d = sum(numels)
        sess = RefSession(ref, numels, P, K, rule, efp)
        seed = 2000 + len(smanifest)
        out = {}
        for s in range(steps):
            grads = np.stack([orc.generate(orc.stream_key(seed, w, s), d, kind, 0, np.float64)
                              for w in range(P)])
            upd, res, _ = sess.step(grads, want_residual=True)
            out[f"update_{s}"] = upd
            out[f"residual0_{s}"] = res
        sess.close()
        np.savez_compressed(os.path.join(HERE, f"session_{name}.npz"), **out)
        smanifest.append({"name": name, "sizes": sizes, "cap": cap, "K": K, "rule": rule,
                          "ef": efp, "kind": kind, "P": P, "steps": steps, "seed": seed})
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump({"compress": manifest, "session": smanifest}, f, indent=1)
    print("golden fixtures written:", len(plans), "plans,", len(sel), "selections,",
          len(manifest), "traces,", len(smanifest), "sessions")


if __name__ == "__main__":
    main()
