#!/bin/bash
# regenerate the B200 cost tables with this build, then the whole GPU suite and the bench
mkdir -p gpurun_out
rm -f gpurun_out/b200_*.csv
timeout 600 python bench.py --plan-only --db gpurun_out/b200_alexnet_pow2_64M.csv > gpurun_out/plan_alexnet.json 2>&1
timeout 600 python bench.py --net resnet18 --plan-only --db gpurun_out/b200_resnet18_pow2_64M.csv > gpurun_out/plan_resnet18.json 2>&1
timeout 900 python bench.py --policy all --plan-only --db gpurun_out/b200_alexnet_all_64M.csv > gpurun_out/plan_alexnet_all.json 2>&1
timeout 900 python bench.py --net resnet50 --mode wd --plan-only --db gpurun_out/b200_resnet50_wd_pow2_2544M.csv > gpurun_out/plan_resnet50_wd.json 2>&1
cp gpurun_out/b200_*.csv tests/golden/csv/
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_r10.txt 2>&1
tail -5 gpurun_out/pytest_r10.txt
timeout 900 python bench.py --steps 20 --warmup 5 --db gpurun_out/b200_alexnet_pow2_64M.csv > gpurun_out/bench10.json 2> gpurun_out/bench10.err
cat gpurun_out/bench10.json
