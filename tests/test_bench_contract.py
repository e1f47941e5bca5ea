"""bench.py's contract, CPU side: the reference arm runs the reference's own
CPU path (oracle/_ref) without loading anything of the product, prints one
JSON line with the contract's keys, and its `config` is the very object the
GPU arm reports for the same command line (the driver's `same_config`)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

PROBE = r"""
import json, sys
sys.argv = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"] + sys.argv[1:]
sys.path.insert(0, ".")
import bench
bench.main()
bench._OUT.flush()
loaded = sorted(m for m in sys.modules if m.startswith("paper_2311_04499_b200"))
maps = [l for l in open("/proc/self/maps").read().splitlines() if "libcovap_b200" in l]
print(json.dumps({"loaded": loaded, "maps": len(maps)}), file=sys.stderr)
"""


def run_reference(args):
    from oracle.oracle import REF_SO
    if not os.path.exists(REF_SO):
        pytest.skip("reference library (oracle/_ref) not built here")
    p = subprocess.run([sys.executable, "-c", PROBE] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, p.stdout
    probe = json.loads(p.stderr.strip().splitlines()[-1])
    return json.loads(lines[0]), probe


@pytest.mark.parametrize("args", [[], ["--interval", "auto"]])
def test_reference_arm_is_clean_and_same_config(args):
    line, probe = run_reference(args)
    assert probe == {"loaded": [], "maps": 0}  # nothing of the product in the reference arm
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e", "impl"):
        assert k in line, k
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    ns = argparse.Namespace(layout="resnet50", interval=args[1] if args else "4", flush=False)
    assert line["config"] == bench.workload_config(ns, 1)
    want_k = 1 if args else 4  # "auto": the reference's train() runs its default K = 1
    assert line["reference_run"]["interval_used"] == want_k


@pytest.mark.gpu
def test_gpu_arm_line_has_the_contract_keys():
    """The GPU arm's one JSON line on a B200 (short run): the contract's keys,
    the roofline object with algorithmic bytes and a measured peak, the e2e
    object with the copied bytes, the clocks sample and the launch count."""
    p = subprocess.run([sys.executable, "bench.py", "--steps", "4", "--warmup", "3",
                        "--no-real-model", "--no-cpu-baseline", "--no-overhead"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, p.stdout
    line = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in line, k
    assert line["steps"] == 4 and line["warmup"] == 3 and line["n_gpus"] == 1
    assert line["config"]["workload"] and line["config"]["interval"] == 4
    r = line["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2
    assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-3
    assert r["algorithmic_bytes_per_launch"] == 16 * line["config"]["params"]
    e = line["e2e"]
    assert e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 4 * line["config"]["params"]
    assert 0 < e["value"] < line["value"]
    assert line["gpu_launches"] == line["steps"]
    assert line["clocks"]["sm_mhz"] and "reasons" in line["clocks"]
    u = r["unfused_p1"]
    assert 0 < u["k1_frac"] < 1.2 and 0 < u["k2_frac"] < 1.3 and "eager" in u and "graph" in u
