"""Golden fixtures for the baseline compressors under error feedback
(SURVEY.md §8(f4)), generated from the REFERENCE itself.

Run in the build container, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden_f4.py

Every output comes from oracle/_ref/libcovap_ref.so (the reference's
compress.cpp compiled from its sources, probed through oracle/ref_shim.cpp):

  half_bits.npz      half_bits_from_float / float_from_half_bits
                     (compress.cpp:157-224) over special values and 200 000
                     random float32 bit patterns
  sparsifiers.json   topk_compress / randomk_compress (compress.cpp:119-155)
                     on small inputs with ties, plus the known answers of
                     test_compress.cpp:247-300
  feedback_*.npz     multi-step ErrorFeedback::step traces (compress.cpp:323-344)
                     for every GradientFilter kind: per step the input
                     gradient, kept output, residual and transmitted count
  feedback.json      the manifest of those traces
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, Ref, RefFeedback  # noqa: E402

KINDS = {"identity": 0, "covap": 1, "topk": 2, "randomk": 3, "fp16": 4}

# name, kind, sizes, steps, k_fraction, interval, seed, ef, input
FEEDBACK = [
    ("topk_small", "topk", [37, 5, 129, 64, 1, 300, 77, 2, 515], 8, 0.1, 1, 0, (1, 0.3, 100, 0.1), "ih"),
    ("topk_ties", "topk", [40, 40, 40, 7, 1000], 10, 0.25, 1, 0, (1, 1.0, 1, 0.0), "int"),
    ("topk_dense", "topk", [64, 33, 4096], 4, 1.0, 1, 0, (1, 0.3, 2, 0.25), "ih"),
    ("topk_tiny_frac", "topk", [3000, 5000, 1], 6, 0.001, 1, 0, (0, 0.3, 100, 0.1), "ih"),
    ("randomk_small", "randomk", [37, 5, 129, 64, 1, 300, 77, 2, 515], 8, 0.05, 1, 7, (1, 0.3, 100, 0.1), "ih"),
    ("randomk_half", "randomk", [1000, 2048, 3], 6, 0.5, 1, 99, (1, 1.0, 1, 0.0), "int"),
    ("fp16_range", "fp16", [37, 5, 129, 64, 1, 300, 77, 2, 515], 6, 0.01, 1, 0, (1, 0.3, 100, 0.1), "wide"),
    ("covap_k3", "covap", [37, 5, 129, 64, 1, 300, 77, 2, 515], 7, 0.01, 3, 0, (1, 0.4, 3, 0.2), "ih"),
    ("identity", "identity", [37, 5, 129], 3, 0.01, 1, 0, (1, 0.3, 100, 0.1), "ih"),
]


def inputs(orc, kind, n, step, seed):
    key = orc.stream_key(seed, 0, step)
    if kind == "int":
        return orc.generate(key, n, kind=1, dtype=np.float64)
    g = orc.generate(key, n, kind=0, dtype=np.float64)
    if kind == "wide":
        # magnitudes from 2^-30 to 2^20: subnormal halves, rounding, saturation
        e = orc.generate(orc.stream_key(seed, 1, step), n, kind=1, dtype=np.float64)
        g = g * np.exp2(np.round((e + 1000) / 2000 * 50) - 30)
    return g


def main():
    ref = Ref()
    orc = Oracle()

    # half conversion ---------------------------------------------------
    special = np.array([0.0, -0.0, 1.0, -1.0, 2049.0, 65504.0, 65505.0, 65519.99, 65520.0,
                        70000.0, -70000.0, np.inf, -np.inf, np.nan, 0.1, 2.0**-14, 2.0**-15,
                        2.0**-24, 2.0**-25, 1.5 * 2.0**-25, 2.0**-24 * 1.5, 2.0**-24 * 2.5,
                        3.0e-8, 6.0e-8, 5.96e-8, 1e-30, 1e30], np.float32)
    rng = np.random.default_rng(4499)
    bits = rng.integers(0, 2**32, 200_000, dtype=np.uint64).astype(np.uint32)
    vals = np.concatenate([special, bits.view(np.float32)])
    hb = np.zeros(len(vals), np.uint16)
    sat = np.zeros(len(vals), np.uint8)
    for i, v in enumerate(vals):
        hb[i], s = ref.half_bits(v)
        sat[i] = s
    back = np.array([ref.float_from_half(h) for h in range(65536)], np.float32)
    np.savez_compressed(os.path.join(HERE, "half_bits.npz"), values=vals, half=hb, saturated=sat,
                        widened=back)

    # sparsifiers -------------------------------------------------------
    cases = []
    for (x, kf, seed) in [([3, -5, 1, 2], 0.5, 0), ([3, -5, 1, 2], 1.0, 0), ([2, -2, 2], 1 / 3, 0),
                          ([0, 0, 0, -0.0, 1], 0.6, 3), ([1] * 10, 0.3, 99), ([1] * 10, 1.0, 1)]:
        ti, tv = ref.topk(np.array(x, float), kf)
        ri, rv = ref.randomk(np.array(x, float), kf, seed)
        cases.append({"x": x, "k_fraction": kf, "seed": seed, "topk_indices": ti.tolist(),
                      "topk_values": tv.tolist(), "randomk_indices": ri.tolist()})
    for d, kf, seed in [(10, 0.3, s) for s in range(50)] + [(1000, 0.01, 5), (4097, 0.25, 11),
                                                             (100000, 0.01, 2**63 + 5)]:
        ri, _ = ref.randomk(np.ones(d), kf, seed)
        cases.append({"d": d, "k_fraction": kf, "seed": seed, "randomk_indices": ri.tolist()})
    for n, kf, kind in [(1000, 0.1, 0), (1000, 0.1, 1), (513, 0.02, 1), (4096, 0.5, 0)]:
        x = orc.generate(orc.stream_key(77, n, kind), n, kind=kind, dtype=np.float64)
        ti, tv = ref.topk(x, kf)
        cases.append({"gen": [77, n, kind], "k_fraction": kf, "topk_indices": ti.tolist()})
    with open(os.path.join(HERE, "sparsifiers.json"), "w") as f:
        json.dump(cases, f)

    # feedback traces ---------------------------------------------------
    manifest = []
    for name, kind, sizes, steps, kf, K, seed, ef, inp in FEEDBACK:
        fb = RefFeedback(ref, sizes, KINDS[kind], interval=K, k_fraction=kf, seed=seed, ef=ef)
        n = sum(sizes)
        out = {"g": [], "kept": [], "residual": [], "transmitted": []}
        for step in range(steps):
            g = inputs(orc, inp, n, step, 3000 + len(manifest))
            kept, res, sent, _ = fb.step(g)
            out["g"].append(g)
            out["kept"].append(kept)
            out["residual"].append(res)
            out["transmitted"].append(sent)
        fb.close()
        np.savez_compressed(os.path.join(HERE, f"feedback_{name}.npz"),
                            **{k: np.array(v) for k, v in out.items()})
        manifest.append({"name": name, "kind": kind, "sizes": sizes, "steps": steps,
                         "k_fraction": kf, "interval": K, "seed": seed, "ef": list(ef),
                         "input": inp})
    with open(os.path.join(HERE, "feedback.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print("half_bits:", len(vals), "values; sparsifier cases:", len(cases), "; feedback traces:",
          len(manifest))


if __name__ == "__main__":
    main()
