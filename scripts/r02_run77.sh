#!/bin/bash
# AlexNet conv1 BackwardData (phase scatter, 48 phase-channels) through algorithm 5 at 64 images
timeout 300 python scripts/one_conv.py --layer a1 --op 1 --algo 5 --batch 64 --reps 1 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:precomp -s 1 -c 1 \
  -o gpurun_out/pc_conv1_bd python scripts/one_conv.py --layer a1 --op 1 --algo 5 --batch 64 --reps 2 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/pc_conv1_bd.ncu-rep
