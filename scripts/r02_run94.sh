#!/bin/bash
# full GPU suite after the division-free loops / finalize kernels, then the benches
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_r94.txt 2>&1
tail -3 gpurun_out/pytest_r94.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_v16.json 2> gpurun_out/bench_v16.err
timeout 900 python bench.py --net resnet18 --no-cpu --steps 20 > gpurun_out/r18_v15.json 2> gpurun_out/r18_v15.err
python - <<'P'
import json
for f in ("gpurun_out/bench_v16.json","gpurun_out/r18_v15.json"):
    d=json.load(open(f)); print(f, d["value"], d.get("speedup_vs_undivided"), d["e2e"]["value"], d["roofline"].get("kernel"), d["roofline"]["frac"], d["clocks"], d.get("plan_seconds"))
    pk=d.get("per_kernel_ms",{}); print(sorted(pk.items(), key=lambda x:-x[1])[:16])
P
