#!/bin/bash
# the bench's ncu launch list with planning served from the committed B200 table (no benchmarking launches)
mkdir -p gpurun_out
cp tests/golden/csv/b200_alexnet_pow2_64M.csv gpurun_out/db97.csv
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches97.csv python bench.py --steps 1 --warmup 3 --no-cpu --db gpurun_out/db97.csv > gpurun_out/ncu97.log 2>&1
python scripts/launch_times.py gpurun_out/launches97.csv > gpurun_out/r02_launches_bench_v16_summary.txt 2>&1; head -24 gpurun_out/r02_launches_bench_v16_summary.txt
bash scripts/r02_run96.sh
