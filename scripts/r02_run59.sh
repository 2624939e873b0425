#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/b200_resnet*.csv
timeout 900 python bench.py --net resnet18 --steps 10 --warmup 3 --no-cpu --db gpurun_out/b200_resnet18_pow2_64M.csv > gpurun_out/bench_resnet18_v9.json 2> gpurun_out/bench_resnet18_v9.err
timeout 1200 python bench.py --net resnet50 --mode wd --steps 10 --warmup 3 --no-cpu --db gpurun_out/b200_resnet50_wd_pow2_2544M.csv > gpurun_out/bench_resnet50_v9.json 2> gpurun_out/bench_resnet50_v9.err
for f in bench_resnet18_v9 bench_resnet50_v9; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d.get('speedup_vs_undivided'), d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks']['reasons'])"; done
timeout 1200 python -m pytest tests/test_algos_gpu.py -m gpu -q -p no:cacheprovider --timeout 900 -k "knob" > gpurun_out/pytest_r61.txt 2>&1
tail -2 gpurun_out/pytest_r61.txt
