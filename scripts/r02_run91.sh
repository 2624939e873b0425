#!/bin/bash
# ncu full captures of the three AlexNet conv1 TMEM-operand kernels after the division-free loops
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fct_bwdd -s 1 -c 1 -o gpurun_out/fct_bwdd_a1 python scripts/one_conv.py --layer a1 --op 1 --algo 0 --batch 256 --reps 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fct_bwdf_kernel" -s 1 -c 1 -o gpurun_out/fct_bwdf_a1 python scripts/one_conv.py --layer a1 --op 2 --algo 6 --batch 256 --reps 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fct_fwd -s 1 -c 1 -o gpurun_out/fct_fwd_a1 python scripts/one_conv.py --layer a1 --op 0 --algo 0 --batch 256 --reps 2 > /dev/null 2>&1
for r in fct_bwdd_a1 fct_bwdf_a1 fct_fwd_a1; do python scripts/ncu_summary.py gpurun_out/$r.ncu-rep; done
