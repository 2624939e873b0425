#!/bin/bash
# ncu full capture: strided 3x3 BackwardData (ResNet-18 l2b1c1) through precomp2 with the phase scatter
timeout 600 ncu --set full --clock-control none --import-source on -k regex:precomp -s 1 -c 1 \
  -o gpurun_out/pc2_phase_l2b1c1_bd python scripts/one_conv.py --shape 256,64,56,56,128,3,3,1,2 --op 1 --algo 5 --batch 64 --reps 2 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/pc2_phase_l2b1c1_bd.ncu-rep
