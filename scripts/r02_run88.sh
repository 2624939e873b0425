#!/bin/bash
# fresh B200 cost tables + bench lines (four configs) after the algorithm-8 pair default
mkdir -p gpurun_out
rm -f gpurun_out/b200_*.csv
timeout 900 python bench.py --steps 20 --warmup 5 --db gpurun_out/b200_alexnet_pow2_64M.csv > gpurun_out/bench_v15.json 2> gpurun_out/bench_v15.err
timeout 900 python bench.py --net resnet18 --steps 20 --warmup 5 --no-cpu --db gpurun_out/b200_resnet18_pow2_64M.csv > gpurun_out/bench_resnet18_v14.json 2> gpurun_out/bench_resnet18_v14.err
timeout 1200 python bench.py --net resnet50 --mode wd --total-mib 2544 --steps 10 --warmup 3 --no-cpu --db gpurun_out/b200_resnet50_wd_pow2_2544M.csv > gpurun_out/bench_resnet50_v12.json 2> gpurun_out/bench_resnet50_v12.err
timeout 1200 python bench.py --policy all --steps 20 --warmup 5 --no-cpu --db gpurun_out/b200_alexnet_all_64M.csv > gpurun_out/bench_all_v8.json 2> gpurun_out/bench_all_v8.err
for f in bench_v15 bench_resnet18_v14 bench_resnet50_v12 bench_all_v8; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d['undivided_ms_per_step'], d.get('speedup_vs_undivided'), d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks'], d.get('plan_seconds'))"; done
ls -la gpurun_out/b200_*.csv
