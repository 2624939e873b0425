#!/bin/bash
# algorithm 8: CTA pairs for >= 192-channel 3x3 / 5x5 BackwardFilter -- parity, benches
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_scale_gpu.py -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_v14.json 2> gpurun_out/bench_v14.err
timeout 900 python bench.py --net resnet18 --no-cpu --steps 20 > gpurun_out/r18_v13.json 2> gpurun_out/r18_v13.err
timeout 900 python bench.py --net resnet50 --mode wd --total-mib 2544 --no-cpu --steps 10 > gpurun_out/r50_v11.json 2> gpurun_out/r50_v11.err
python - <<'P'
import json
for f in ("gpurun_out/bench_v14.json","gpurun_out/r18_v13.json","gpurun_out/r50_v11.json"):
    d=json.load(open(f)); print(f, d["value"], d["undivided_ms_per_step"], d.get("speedup_vs_undivided"), d["e2e"]["value"], d["roofline"].get("kernel"), d["roofline"]["frac"], d["clocks"], d.get("plan_seconds"))
    pk=d.get("per_kernel_ms",{}); print(sorted(pk.items(), key=lambda x:-x[1])[:12])
P
