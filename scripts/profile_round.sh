#!/bin/bash
# One gpurun call: bench (writes the cost table), launch list of a short bench
# reusing that table, and full ncu captures of the top kernels.
mkdir -p gpurun_out
rm -f gpurun_out/db.csv
timeout 900 python bench.py --db gpurun_out/db.csv > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --db gpurun_out/db.csv > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bfl2?_kernel" -s 1 -c 1 \
  -o gpurun_out/gather_conv2_bf python scripts/one_conv.py --layer a2 --op 2 --algo 6 --batch 256 --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bfl2?_kernel" -s 1 -c 1 \
  -o gpurun_out/gather_conv1_bf python scripts/one_conv.py --layer a1 --op 2 --algo 6 --batch 256 --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:precomp -s 1 -c 1 \
  -o gpurun_out/precomp_conv2_bd python scripts/one_conv.py --layer a2 --op 1 --algo 5 --batch 64 --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:precomp -s 1 -c 1 \
  -o gpurun_out/precomp_conv1_f python scripts/one_conv.py --layer a1 --op 0 --algo 5 --batch 64 --reps 2 > /dev/null 2>&1
timeout 600 python bench.py --net resnet18 --no-cpu --steps 20 > gpurun_out/r18.json 2> gpurun_out/r18.err
timeout 600 python bench.py --net resnet50 --mode wd --total-mib 2544 --no-cpu --steps 10 > gpurun_out/r50.json 2> gpurun_out/r50.err
timeout 600 python bench.py --policy all --no-cpu --steps 50 > gpurun_out/alex_all.json 2> gpurun_out/alex_all.err
ls -la gpurun_out
