#!/bin/bash
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_step.py alexnet > gpurun_out/r02_memcheck_alexnet_v7.txt 2>&1
tail -4 gpurun_out/r02_memcheck_alexnet_v7.txt
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_step.py resnet18 > gpurun_out/r02_memcheck_resnet18_v7.txt 2>&1
tail -4 gpurun_out/r02_memcheck_resnet18_v7.txt
