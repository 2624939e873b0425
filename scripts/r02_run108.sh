#!/bin/bash
# final tree: full GPU suite, smoke, and the four bench configurations
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_r108.txt 2>&1
tail -3 gpurun_out/pytest_r108.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_v18.json 2> gpurun_out/bench_v18.err
timeout 900 python bench.py --net resnet18 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_resnet18_v17.json 2> gpurun_out/bench_resnet18_v17.err
timeout 1200 python bench.py --net resnet50 --mode wd --total-mib 2544 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_resnet50_v13.json 2> gpurun_out/bench_resnet50_v13.err
timeout 1200 python bench.py --policy all --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_all_v9.json 2> gpurun_out/bench_all_v9.err
for f in bench_v18 bench_resnet18_v17 bench_resnet50_v13 bench_all_v9; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d['undivided_ms_per_step'], d.get('speedup_vs_undivided'), d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks'], d.get('plan_seconds'))"; done
python -c "
import json; d=json.load(open('gpurun_out/bench_v18.json')); pk=d['per_kernel_ms']; print(sorted(pk.items(), key=lambda x:-x[1])[:8])"
