#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list of the bench.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
rm -f gpurun_out/db.csv; timeout 900 python bench.py --db gpurun_out/db.csv > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --db gpurun_out/db.csv > gpurun_out/ncu_bench.log 2>&1
fi
