#!/bin/bash
# checkpoint: fresh B200 cost tables + bench lines for the four configs on the current kernels
mkdir -p gpurun_out
rm -f gpurun_out/b200_*.csv
timeout 900 python bench.py --steps 20 --warmup 5 --db gpurun_out/b200_alexnet_pow2_64M.csv > gpurun_out/bench_v5.json 2> gpurun_out/bench_v5.err
timeout 900 python bench.py --net resnet18 --steps 10 --warmup 3 --no-cpu --db gpurun_out/b200_resnet18_pow2_64M.csv > gpurun_out/bench_resnet18_v5.json 2> gpurun_out/bench_resnet18_v5.err
timeout 1200 python bench.py --net resnet50 --mode wd --steps 10 --warmup 3 --no-cpu --db gpurun_out/b200_resnet50_wd_pow2_2544M.csv > gpurun_out/bench_resnet50_v5.json 2> gpurun_out/bench_resnet50_v5.err
timeout 1200 python bench.py --policy all --steps 20 --warmup 5 --no-cpu --db gpurun_out/b200_alexnet_all_64M.csv > gpurun_out/bench_all_v5.json 2> gpurun_out/bench_all_v5.err
for f in bench_v5 bench_resnet18_v5 bench_resnet50_v5 bench_all_v5; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d.get('speedup_vs_undivided'), d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks']['reasons'], d['config'].get('plan_seconds'))"; done
ls -la gpurun_out/b200_*.csv
