#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_algos_gpu.py -m gpu -q -p no:cacheprovider -x --timeout 600 -k "[0-" > gpurun_out/pytest_r5.txt 2>&1
tail -3 gpurun_out/pytest_r5.txt
L="256,3,227,227,64,11,11,2,4 256,64,27,27,192,5,5,2,1 256,192,13,13,384,3,3,1,1 256,384,13,13,256,3,3,1,1 256,256,13,13,256,3,3,1,1"
for t in "z_msub=1" "z_msub=2" "z_msub=2,z_stages=4" "z_msub=1,z_stages=6"; do
  echo "== $t" >> gpurun_out/tt_r5.txt
  UCUDNN_TUNE=$t timeout 600 python scripts/time_table.py $L --ops 0,1 --algos 0 --batches 256 >> gpurun_out/tt_r5.txt 2>&1
done
cat gpurun_out/tt_r5.txt
