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
