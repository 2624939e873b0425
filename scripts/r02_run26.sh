#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_algos_gpu.py -m gpu -q -p no:cacheprovider --timeout 300 -k "knob" > gpurun_out/pytest_r26.txt 2>&1
tail -15 gpurun_out/pytest_r26.txt
L="256,64,27,27,192,5,5,2,1 256,192,13,13,384,3,3,1,1 256,384,13,13,256,3,3,1,1 256,256,13,13,256,3,3,1,1 256,128,28,28,128,3,3,1,1 256,256,14,14,256,3,3,1,1"
for t in "" "pc2_msub=2" "pc2_msub=2,pc2_ksub=2"; do
  echo "== $t" >> gpurun_out/tt_r26.txt
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $L --ops 0,1 --algos 5 --batches 256,64 >> gpurun_out/tt_r26.txt 2>&1
done
cat gpurun_out/tt_r26.txt
