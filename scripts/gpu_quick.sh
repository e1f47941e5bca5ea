#!/bin/bash
# tests + default bench + extra configs (no ncu)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
rm -f gpurun_out/bench_extra.json
for cfg in "--layout resnet50 --interval 4" "--layout vgg16 --interval 4" "--layout bert_large --interval 4" "--layout bert_large --interval 1"; do
  timeout 300 python bench.py $cfg --no-cpu-baseline --no-overhead --steps 12 --warmup 4 >> gpurun_out/bench_extra.json 2>> gpurun_out/bench.err
done
python - <<'PY'
import json
for f in ["gpurun_out/bench.json", "gpurun_out/bench_extra.json"]:
    for l in open(f):
        d = json.loads(l); r = d["roofline"]; u = r.get("unfused_p1", {})
        print(d["config"]["layout"], "K", d["config"]["interval"], "value", d["value"], "ms", d["ms_per_step"],
              "k1f", r["frac"], "k1", u.get("k1_frac"), "k2", u.get("k2_frac"), "e2e", d["e2e"]["value"])
PY
tail -3 gpurun_out/bench.err
