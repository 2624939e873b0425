#!/bin/bash
# round-2 ncu evidence: tensor-pipe % of the implicit GEMMs, HBM GB/s of the
# transform / copy kernels, launch list of one bench step
mkdir -p gpurun_out
N="ncu --clock-control none"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
timeout 300 $N --set full --import-source on -k regex:precomp2 -s 1 -c 1 -o gpurun_out/r02_precomp2_conv2_f python scripts/one_conv.py --layer a2 --op 0 --algo 5 --batch 256 --reps 2 > /dev/null 2>&1
timeout 300 $N --set full --import-source on -k regex:precomp2 -s 1 -c 1 -o gpurun_out/r02_precomp2_conv3_f python scripts/one_conv.py --layer a3 --op 0 --algo 5 --batch 256 --reps 2 > /dev/null 2>&1
timeout 300 $N --set full --import-source on -k regex:precomp -s 1 -c 1 -o gpurun_out/r02_precomp_conv2_bd python scripts/one_conv.py --layer a2 --op 1 --algo 7 --batch 256 --reps 2 > /dev/null 2>&1
timeout 300 $N --set full --import-source on -k regex:bfn2 -s 1 -c 1 -o gpurun_out/r02_bfn2_conv4_bf python scripts/one_conv.py --layer a4 --op 2 --algo 8 --batch 128 --reps 2 > /dev/null 2>&1
for spec in "a3 0 4 64" "a3 0 1 64" "a3 1 4 64" "a2 0 2 32" "a3 0 2 32" "a3 0 3 32" "a3 1 3 32" "a2 0 5 256" "a1 0 5 64" "a1 1 5 64" "a2 2 8 64" "a2 1 7 256" "a1 2 6 256" "a4 2 8 128"; do
  set -- $spec
  timeout 300 $N $M --csv --log-file gpurun_out/r02_m_$1_op$2_a$3_b$4.csv python scripts/one_conv.py --layer $1 --op $2 --algo $3 --batch $4 --reps 2 > /dev/null 2>&1
done
rm -f gpurun_out/dbp.csv
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --db gpurun_out/dbp.csv > gpurun_out/benchp.json 2>&1
timeout 900 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-graph --db gpurun_out/dbp.csv > gpurun_out/ncu_bench.log 2>&1
ls gpurun_out | head -50
