#!/bin/bash
mkdir -p gpurun_out
for sp in "2 3 31 31 16 11 11 2 4" "2 3 36 36 70 7 7 3 2" "3 3 227 227 64 11 11 0 4" "2 3 224 224 64 7 7 3 2" "1 2 40 40 8 11 11 0 4" "3 4 30 30 24 5 5 2 2"; do
  timeout 60 python scripts/one_small.py $sp 0 0 2>&1 | tail -2 >> gpurun_out/fct_r27.txt
done
cat gpurun_out/fct_r27.txt
L="256,3,227,227,64,11,11,0,4 256,3,224,224,64,7,7,3,2"
for t in "" "fct=0"; do
  echo "== $t" >> gpurun_out/tt_r27.txt
  UCUDNN_TUNE=$t timeout 120 python scripts/time_table.py $L --ops 0 --algos 0,5 --batches 256,64 >> gpurun_out/tt_r27.txt 2>&1
done
cat gpurun_out/tt_r27.txt
