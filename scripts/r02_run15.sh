#!/bin/bash
mkdir -p gpurun_out
L="256,64,27,27,192,5,5,2,1 256,192,13,13,384,3,3,1,1 256,384,13,13,256,3,3,1,1 256,256,13,13,256,3,3,1,1"
for t in "" "pc2_ksub=1" "pc2_ksub=1,pc2_stages=5" "pc2_ksub=2,pc2_stages=2" "two_sm_min_bn=64"; do
  echo "== $t" >> gpurun_out/tt_r15.txt
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $L --ops 0,1 --algos 5 --batches 256 >> gpurun_out/tt_r15.txt 2>&1
done
cat gpurun_out/tt_r15.txt
