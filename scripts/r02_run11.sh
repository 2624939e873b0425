#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_deterministic_gpu.py tests/test_math_modes_gpu.py -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_r11.txt 2>&1
tail -15 gpurun_out/pytest_r11.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_step.py alexnet > gpurun_out/r02_memcheck_alexnet.txt 2>&1
tail -5 gpurun_out/r02_memcheck_alexnet.txt
rm -f gpurun_out/dball.csv
( time timeout 900 python bench.py --policy all --plan-only --db gpurun_out/dball.csv ) > gpurun_out/plan_all_r11.json 2>&1
tail -4 gpurun_out/plan_all_r11.json
timeout 900 python bench.py --net resnet18 --no-cpu --steps 20 --db tests/golden/csv/b200_resnet18_pow2_64M.csv > gpurun_out/r18_r11.json 2> gpurun_out/r18_r11.err
timeout 900 python bench.py --net resnet50 --mode wd --total-mib 2544 --no-cpu --steps 10 --db tests/golden/csv/b200_resnet50_wd_pow2_2544M.csv > gpurun_out/r50_r11.json 2> gpurun_out/r50_r11.err
timeout 900 python bench.py --policy all --no-cpu --steps 20 --db tests/golden/csv/b200_alexnet_all_64M.csv > gpurun_out/alexall_r11.json 2> gpurun_out/alexall_r11.err
for f in r18_r11 r50_r11 alexall_r11; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['value'], d['undivided_ms_per_step'], d['speedup_vs_undivided'], d['roofline']['kernel'], d['roofline']['frac'])"; done
