#!/bin/bash
mkdir -p gpurun_out
L="256,3,227,227,64,11,11,0,4"
for t in "" "fct_dbg=4" "fct_dbg=8" "fct_dbg=12" "fct_dbg=15" ; do
  echo "== $t" >> gpurun_out/tt_r29.txt
  UCUDNN_TUNE=$t timeout 120 python scripts/time_table.py $L --ops 0 --algos 0 --batches 256 >> gpurun_out/tt_r29.txt 2>&1
done
cat gpurun_out/tt_r29.txt
