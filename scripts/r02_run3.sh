#!/bin/bash
# round-2 GPU run 3: gather BF with MN-major x rows (xmn) + ncu of zgemm
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_algos_gpu.py tests/test_scale_gpu.py -m gpu -q -p no:cacheprovider -x --timeout 600 -k "BF" > gpurun_out/pytest_r3.txt 2>&1
tail -3 gpurun_out/pytest_r3.txt
timeout 300 python scripts/time_table.py 256,3,227,227,64,11,11,2,4 256,3,224,224,64,7,7,3,2 --ops 2 --algos 0,6 --batches 256,64 > gpurun_out/tt_r3.txt 2>&1
UCUDNN_TUNE=bfl_xmn=0 timeout 300 python scripts/time_table.py 256,3,227,227,64,11,11,2,4 256,3,224,224,64,7,7,3,2 --ops 2 --algos 6 --batches 256 >> gpurun_out/tt_r3.txt 2>&1
cat gpurun_out/tt_r3.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zgemm -s 1 -c 1 \
  -o gpurun_out/r02_zgemm_conv2_f python scripts/one_conv.py --layer a2 --op 0 --algo 0 --batch 256 --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zgemm -s 1 -c 1 \
  -o gpurun_out/r02_zgemm_conv3_bd python scripts/one_conv.py --layer a3 --op 1 --algo 0 --batch 256 --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bfl_kernel" -s 1 -c 1 \
  -o gpurun_out/r02_bfl_xmn_conv1_bf python scripts/one_conv.py --layer a1 --op 2 --algo 6 --batch 256 --reps 2 > /dev/null 2>&1
ls gpurun_out
