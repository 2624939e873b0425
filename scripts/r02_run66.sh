#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_r66.txt 2>&1
tail -3 gpurun_out/pytest_r66.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_v11.json 2> gpurun_out/bench_v11.err
python -c "
import json; d=json.load(open('gpurun_out/bench_v11.json')); print(d['value'], d.get('speedup_vs_undivided'), d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks'], d['gpu_launches'], d['cpu_baseline']['value'])"
