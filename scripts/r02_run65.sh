#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/p65*.csv
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --db gpurun_out/p65a.csv > gpurun_out/b65a.json 2>/dev/null
timeout 1200 python bench.py --policy all --steps 20 --warmup 5 --no-cpu --db gpurun_out/p65b.csv > gpurun_out/b65b.json 2>/dev/null
for f in b65a b65b; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d.get('speedup_vs_undivided'), d['plan_seconds'])"; done
timeout 1500 python -m pytest tests/test_executor_gpu.py tests/test_dp_nccl_gpu.py -m gpu -q -p no:cacheprovider --timeout 900 2>&1 | tail -2
