#!/bin/bash
# final: fresh B200 cost tables + bench lines (four configs), full GPU suite, smoke, launch list
mkdir -p gpurun_out
rm -f gpurun_out/b200_*.csv
timeout 900 python bench.py --steps 20 --warmup 5 --db gpurun_out/b200_alexnet_pow2_64M.csv > gpurun_out/bench_v7.json 2> gpurun_out/bench_v7.err
timeout 900 python bench.py --net resnet18 --steps 10 --warmup 3 --no-cpu --db gpurun_out/b200_resnet18_pow2_64M.csv > gpurun_out/bench_resnet18_v7.json 2> gpurun_out/bench_resnet18_v7.err
timeout 1200 python bench.py --net resnet50 --mode wd --steps 10 --warmup 3 --no-cpu --db gpurun_out/b200_resnet50_wd_pow2_2544M.csv > gpurun_out/bench_resnet50_v7.json 2> gpurun_out/bench_resnet50_v7.err
timeout 1200 python bench.py --policy all --steps 20 --warmup 5 --no-cpu --db gpurun_out/b200_alexnet_all_64M.csv > gpurun_out/bench_all_v7.json 2> gpurun_out/bench_all_v7.err
for f in bench_v7 bench_resnet18_v7 bench_resnet50_v7 bench_all_v7; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d.get('speedup_vs_undivided'), d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks']['reasons'])"; done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_r54.txt 2>&1
tail -3 gpurun_out/pytest_r54.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches54.csv python bench.py --steps 1 --warmup 3 --no-cpu --db gpurun_out/b200_alexnet_pow2_64M.csv > gpurun_out/ncu54.log 2>&1
python scripts/launch_times.py gpurun_out/launches54.csv > gpurun_out/launches54_summary.txt 2>&1; head -12 gpurun_out/launches54_summary.txt
