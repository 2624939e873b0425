#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_dp_nccl_gpu.py tests/test_scale_gpu.py -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_r20.txt 2>&1
tail -3 gpurun_out/pytest_r20.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29533 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu --db tests/golden/csv/b200_alexnet_pow2_64M.csv > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err
python -c "import json;d=json.load(open('gpurun_out/bench_dist1.json'));print(d['value'], d['config']['launch'], d['e2e']['value'])"
