#!/bin/bash
timeout 900 python bench.py --net resnet18 --no-cpu --steps 20 > gpurun_out/r18_v10.json 2> gpurun_out/r18_v10.err
timeout 900 python bench.py --net resnet50 --mode wd --total-mib 2544 --no-cpu --steps 10 > gpurun_out/r50_v10.json 2> gpurun_out/r50_v10.err
python - <<'P'
import json
for f in ("gpurun_out/r18_v10.json","gpurun_out/r50_v10.json"):
    d=json.load(open(f)); print(f, d["value"], d.get("speedup_vs_undivided"), d["roofline"].get("kernel"), d["roofline"]["frac"], d["clocks"])
    pk=d.get("per_kernel_ms",{}); print(sorted(pk.items(), key=lambda x:-x[1])[:8])
P
