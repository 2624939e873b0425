#!/bin/bash
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fct_bwdd -s 1 -c 1 -o gpurun_out/r02_fct_bwdd_conv1 python scripts/one_conv.py --shape 256,3,227,227,64,11,11,0,4 --op 1 --algo 0 --batch 256 --reps 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fct_fwd -s 1 -c 1 -o gpurun_out/r02_fct_fwd_conv1 python scripts/one_conv.py --shape 256,3,227,227,64,11,11,0,4 --op 0 --algo 0 --batch 256 --reps 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fct_bwdf_kernel -s 1 -c 1 -o gpurun_out/r02_fct_bwdf_conv1 python scripts/one_conv.py --shape 256,3,227,227,64,11,11,0,4 --op 2 --algo 6 --batch 256 --reps 2 > /dev/null 2>&1
ls gpurun_out | grep fct_
