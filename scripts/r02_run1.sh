#!/bin/bash
# round-2 GPU run 1: bench (writes the B200 cost tables), then the GPU suite
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py --steps 20 --warmup 5 --db gpurun_out/b200_alexnet_pow2_64M.csv > gpurun_out/bench_alexnet.json 2> gpurun_out/bench_alexnet.err
timeout 600 python bench.py --net resnet18 --plan-only --db gpurun_out/b200_resnet18_pow2_64M.csv > gpurun_out/plan_resnet18.json 2> gpurun_out/plan_resnet18.err
cp gpurun_out/b200_alexnet_pow2_64M.csv gpurun_out/b200_resnet18_pow2_64M.csv tests/golden/csv/
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=15 --timeout 900 -k "scale or nccl or torch_conv" > gpurun_out/pytest_new.txt 2>&1
tail -5 gpurun_out/pytest_new.txt
timeout 900 python bench.py --net alexnet --policy all --plan-only --db gpurun_out/b200_alexnet_all_64M.csv > gpurun_out/plan_alexnet_all.json 2> gpurun_out/plan_alexnet_all.err
timeout 900 python bench.py --net resnet50 --mode wd --plan-only --db gpurun_out/b200_resnet50_wd_pow2.csv > gpurun_out/plan_resnet50_wd.json 2> gpurun_out/plan_resnet50_wd.err
ls -la gpurun_out
