#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_algos_gpu.py -m gpu -q -p no:cacheprovider --timeout 600 -k "BF and 6" -x > gpurun_out/pytest_r9a.txt 2>&1
tail -2 gpurun_out/pytest_r9a.txt
for t in "" "bfs_stages=2" "bfs_stages=3"; do
echo "== $t" >> gpurun_out/tt_r9.txt
UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,3,227,227,64,11,11,2,4 256,3,224,224,64,7,7,3,2 --ops 2 --algos 6 --batches 256,64 >> gpurun_out/tt_r9.txt 2>&1
done
cat gpurun_out/tt_r9.txt
