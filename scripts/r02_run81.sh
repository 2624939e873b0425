#!/bin/bash
# stepped ring positions in precomp / precomp2 / strip: parity, then the benches
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_scale_gpu.py -q -p no:cacheprovider -k "a5 or a7 or replayed or resnet18" 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_v12.json 2> gpurun_out/bench_v12.err
timeout 900 python bench.py --net resnet18 --no-cpu --steps 20 > gpurun_out/r18_v11.json 2> gpurun_out/r18_v11.err
python - <<'P'
import json
for f in ("gpurun_out/bench_v12.json","gpurun_out/r18_v11.json"):
    d=json.load(open(f)); print(f, d["value"], d.get("speedup_vs_undivided"), d["e2e"]["value"], d["roofline"].get("kernel"), d["roofline"]["frac"], d["clocks"], d.get("plan_seconds"))
    pk=d.get("per_kernel_ms",{}); print(sorted(pk.items(), key=lambda x:-x[1])[:16])
P
