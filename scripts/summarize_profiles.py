"""Summarise a GPU session's artefacts (gpurun_out/) into profiles/ (committed).

    python scripts/summarize_profiles.py r1
writes profiles/<tag>_ncu.md, profiles/<tag>_launches.md, copies the launch
list CSV and the bench lines, and updates profiles/dram_traffic.json (the
per-launch DRAM bytes bench.py reports as roofline.traffic)."""
import csv
import glob
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size",
           "launch__shared_mem_per_block_dynamic", "lts__t_bytes.sum"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Kbyte/block": 1e3,
        "byte/block": 1, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9, "nsecond": 1,
        "usecond": 1e3, "msecond": 1e6}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    v = float(v) * UNIT.get(units[i], 1)
                except ValueError:
                    pass
                d[m] = (v, units[i])
        res.append(d)
    return res


lines = [f"# {tag}: ncu --set full captures (B200, --clock-control none)\n",
         "Captured with `scripts/gpu_check.sh` (`scripts/profile_step.py`, L2 flushed before each "
         "step; ncu's own cache control also flushes).  Per launch: duration, DRAM bytes, and "
         "the algorithmic bytes the bench uses (K1F 16N; multi-rank split: K1 16N with the output zero fill, K2 8S selected-only).  DRAM writes "
         "below the algorithmic figure are lines still dirty in the 126 MB L2 at kernel end.\n"]
traffic = {}
tpath = os.path.join(P, "dram_traffic.json")
if os.path.exists(tpath):
    traffic = json.load(open(tpath))
for rep in sorted(glob.glob(os.path.join(G, "prof_*.ncu-rep"))):
    if os.path.basename(rep)[5:].split("_")[0] not in ("r50", "bert", "vgg"):
        continue  # other studies' captures (f4, K2 traces) are summarised by hand
    name = os.path.basename(rep)[5:-8]
    lines.append(f"\n## {name}\n")
    lines.append("| kernel | µs | DRAM read MB | DRAM write MB | DRAM % peak | SM % | warps active % | regs | grid | dyn smem KB |")
    lines.append("|---|---|---|---|---|---|---|---|---|---|")
    per = defaultdict(list)
    for d in raw(rep):
        g = lambda m: d.get(m, (float("nan"), ""))[0]  # noqa: E731
        lines.append(f"| {d['kernel'][-40:]} | {g('gpu__time_duration.sum') / 1e3:.1f} | "
                     f"{g('dram__bytes_read.sum') / 1e6:.1f} | {g('dram__bytes_write.sum') / 1e6:.1f} | "
                     f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{g('sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
                     f"{g('launch__registers_per_thread'):.0f} | {g('launch__grid_size'):.0f} | "
                     f"{g('launch__shared_mem_per_block_dynamic') / 1e3:.0f} |")
        per[d["kernel"]].append(g("dram__bytes_read.sum") + g("dram__bytes_write.sum"))
    # traffic key: layout/K/kernel (profile names: r50_k1_fused, r50_k4_unfused, bert_k1_fused)
    lay = {"r50": "resnet50", "bert": "bert_large", "vgg": "vgg16"}[name.split("_")[0]]
    K = int(name.split("_")[1][1:])
    for k, v in per.items():
        kind = "K1F" if "filter_kernel<float, 1>" in k else ("K1" if "filter_kernel<float, 0>" in k else "K2")
        traffic[f"{lay}/K{K}/{kind}"] = int(sum(v) / len(v))
with open(os.path.join(P, f"{tag}_ncu.md"), "w") as f:
    f.write("\n".join(lines) + "\n")
with open(tpath, "w") as f:
    json.dump(traffic, f, indent=1, sort_keys=True)

# launch list (share of each kernel in the bench command's launches)
lc = os.path.join(G, "launches.csv")
if os.path.exists(lc):
    shutil.copy(lc, os.path.join(P, f"{tag}_launches.csv"))
    rows = list(csv.reader(open(lc)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[i], rows[i + 1:]
    ki, mi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in data:
        agg[r[ki].split("(")[0]][0] += 1
        agg[r[ki].split("(")[0]][1] += float(r[mi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    prod = {k: v for k, v in agg.items() if "spin_kernel" not in k and "busy_kernel" not in k
            and "generate_kernel" not in k and "at::" not in k}
    ptot = sum(v[1] for v in prod.values())
    out2 = ["", "Product kernels only (K3 spin / busy = the emulated backward of the CCR profile step, "
            "K0 generate = synthetic inputs):", "", "| kernel | launches | total µs | share |",
            "|---|---|---|---|"]
    for k, v in sorted(prod.items(), key=lambda x: -x[1][1]):
        out2.append(f"| {k[-60:]} | {v[0]} | {v[1] / 1e3:.1f} | {v[1] / ptot:.3f} |")
    out = [f"# {tag}: launch list of `python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-overhead`\n",
           "ncu `--metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: "
           "shares, not absolute times).  Raw list: `" + f"{tag}_launches.csv`.\n",
           "| kernel | launches | total µs | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {k[-60:]} | {v[0]} | {v[1] / 1e3:.1f} | {v[1] / tot:.3f} |")
    with open(os.path.join(P, f"{tag}_launches.md"), "w") as f:
        f.write("\n".join(out + out2) + "\n")
for b in ("bench.json", "bench_extra.json"):
    if os.path.exists(os.path.join(G, b)):
        shutil.copy(os.path.join(G, b), os.path.join(P, f"{tag}_{b.replace('.json', '.jsonl')}"))
print("profiles written:", sorted(os.listdir(P)))
