#!/bin/bash
# final validation: full GPU suite, smoke, default bench (fresh table), launch list of the bench command
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_r47.txt 2>&1
tail -3 gpurun_out/pytest_r47.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
rm -f gpurun_out/db47.csv
timeout 900 python bench.py --db gpurun_out/db47.csv > gpurun_out/bench47.json 2> gpurun_out/bench47.err
python -c "
import json; d=json.load(open('gpurun_out/bench47.json')); print(d['value'], d.get('speedup_vs_undivided'), d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks'], d['gpu_launches'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches47.csv python bench.py --steps 1 --warmup 3 --no-cpu --db gpurun_out/db47.csv > gpurun_out/ncu47.log 2>&1
python scripts/launch_times.py gpurun_out/launches47.csv > gpurun_out/launches47_summary.txt 2>&1; head -20 gpurun_out/launches47_summary.txt
