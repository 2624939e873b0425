#!/bin/bash
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -k "knob and (fct_bf1 or 2-6)" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_scale_gpu.py -q -p no:cacheprovider -k "resnet18 and BF" 2>&1 | tail -2
timeout 300 python scripts/time_table.py 256,64,56,56,64,3,3,1,1 256,128,28,28,128,3,3,1,1 256,128,28,28,128,3,3,1,1 --ops 2 --algos 6 --batches 256,128
timeout 900 python bench.py --net resnet18 --no-cpu --steps 20 > gpurun_out/r18_v16.json 2> gpurun_out/r18_v16.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_v17.json 2> gpurun_out/bench_v17.err
python - <<'P'
import json
for f in ("gpurun_out/bench_v17.json","gpurun_out/r18_v16.json"):
    d=json.load(open(f)); print(f, d["value"], d["undivided_ms_per_step"], d.get("speedup_vs_undivided"), d["e2e"]["value"], d["roofline"].get("kernel"), d["roofline"]["frac"], d["clocks"])
P
