#!/bin/bash
# final-build tables, full GPU suite, benches
mkdir -p gpurun_out
rm -f gpurun_out/b200_*.csv
timeout 600 python bench.py --plan-only --db gpurun_out/b200_alexnet_pow2_64M.csv > gpurun_out/plan_alexnet.json 2>&1
timeout 600 python bench.py --net resnet18 --plan-only --db gpurun_out/b200_resnet18_pow2_64M.csv > gpurun_out/plan_resnet18.json 2>&1
timeout 900 python bench.py --policy all --plan-only --db gpurun_out/b200_alexnet_all_64M.csv > gpurun_out/plan_alexnet_all.json 2>&1
timeout 900 python bench.py --net resnet50 --mode wd --plan-only --db gpurun_out/b200_resnet50_wd_pow2_2544M.csv > gpurun_out/plan_resnet50_wd.json 2>&1
cp gpurun_out/b200_*.csv tests/golden/csv/
timeout 3600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_r19.txt 2>&1
tail -5 gpurun_out/pytest_r19.txt
timeout 900 python bench.py --steps 20 --warmup 5 --db gpurun_out/b200_alexnet_pow2_64M.csv > gpurun_out/bench19.json 2> gpurun_out/bench19.err
timeout 900 python bench.py --net resnet18 --no-cpu --steps 20 --db gpurun_out/b200_resnet18_pow2_64M.csv > gpurun_out/r18_19.json 2> gpurun_out/r18_19.err
timeout 900 python bench.py --net resnet50 --mode wd --total-mib 2544 --no-cpu --steps 10 --db gpurun_out/b200_resnet50_wd_pow2_2544M.csv > gpurun_out/r50_19.json 2> gpurun_out/r50_19.err
timeout 900 python bench.py --policy all --no-cpu --steps 20 --db gpurun_out/b200_alexnet_all_64M.csv > gpurun_out/alexall_19.json 2> gpurun_out/alexall_19.err
for f in bench19 r18_19 r50_19 alexall_19; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['value'], d['undivided_ms_per_step'], d['speedup_vs_undivided'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"; done
