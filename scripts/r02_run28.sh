#!/bin/bash
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fct_fwd -s 1 -c 1 -o gpurun_out/r02_fct_conv1_f python scripts/one_conv.py --shape 256,3,227,227,64,11,11,0,4 --op 0 --algo 0 --batch 256 --reps 2 > gpurun_out/ncu28.log 2>&1
tail -3 gpurun_out/ncu28.log
ls gpurun_out | grep fct
