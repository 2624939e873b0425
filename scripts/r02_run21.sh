#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_algos_gpu.py -m gpu -q -p no:cacheprovider --timeout 600 -k "[0-" > gpurun_out/pytest_r21.txt 2>&1
tail -3 gpurun_out/pytest_r21.txt
L="256,256,56,56,512,1,1,0,2 256,512,28,28,1024,1,1,0,2 256,256,56,56,128,1,1,0,2 256,64,56,56,128,1,1,0,2"
timeout 600 python scripts/time_table.py $L --ops 0,1 --algos 0,5 --batches 256 > gpurun_out/tt_r21.txt 2>&1
cat gpurun_out/tt_r21.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29541 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu --db tests/golden/csv/b200_alexnet_pow2_64M.csv > gpurun_out/bench_dist2.json 2> gpurun_out/bench_dist2.err
head -c 200 gpurun_out/bench_dist2.json
