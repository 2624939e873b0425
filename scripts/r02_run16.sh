#!/bin/bash
mkdir -p gpurun_out
L="256,64,56,56,64,1,1,0,1 256,64,56,56,256,1,1,0,1 256,256,56,56,64,1,1,0,1 256,512,28,28,128,1,1,0,1 256,1024,14,14,256,1,1,0,1 256,2048,7,7,512,1,1,0,1"
timeout 600 python scripts/time_table.py $L --ops 0,1,2 --algos 0,5,8 --batches 256 > gpurun_out/tt_r16.txt 2>&1
cat gpurun_out/tt_r16.txt
