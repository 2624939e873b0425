#!/bin/bash
# final evidence: memcheck over one planned AlexNet / ResNet-18 step on the final kernels, and the bench's ncu launch list
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_step.py alexnet > gpurun_out/r02_memcheck_alexnet_v8.txt 2>&1
tail -3 gpurun_out/r02_memcheck_alexnet_v8.txt
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_step.py resnet18 > gpurun_out/r02_memcheck_resnet18_v8.txt 2>&1
tail -3 gpurun_out/r02_memcheck_resnet18_v8.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches95.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu95.log 2>&1
python scripts/launch_times.py gpurun_out/launches95.csv > gpurun_out/r02_launches_bench_v16_summary.txt 2>&1; head -16 gpurun_out/r02_launches_bench_v16_summary.txt
