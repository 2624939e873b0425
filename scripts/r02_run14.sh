#!/bin/bash
mkdir -p gpurun_out
L="256,64,27,27,192,5,5,2,1"
C1="256,3,227,227,64,11,11,2,4"
for t in "" "pc_ksub=4" "pc_ksub=4,pc_cps=1" "pc_ksub=2,pc_cps=1" "pc_ksub=1" "pc_stages=4" "pc_ksub=3"; do
  echo "== $t" >> gpurun_out/tt_r14.txt
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $L --ops 1 --algos 7,5 --batches 256,64 >> gpurun_out/tt_r14.txt 2>&1
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $C1 --ops 0,1 --algos 5 --batches 64 >> gpurun_out/tt_r14.txt 2>&1
done
cat gpurun_out/tt_r14.txt
