#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_algos_gpu.py tests/test_scale_gpu.py tests/test_deterministic_gpu.py -m gpu -q -p no:cacheprovider --timeout 900 -x > gpurun_out/pytest_r34.txt 2>&1
tail -5 gpurun_out/pytest_r34.txt
