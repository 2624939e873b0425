#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -x > gpurun_out/pytest_r37.txt 2>&1
tail -4 gpurun_out/pytest_r37.txt
timeout 900 python bench.py > gpurun_out/bench37.json 2> gpurun_out/bench37.err
cat gpurun_out/bench37.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('speedup_vs_undivided'), d['e2e']['value'], d['roofline'])"
