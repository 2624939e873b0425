#!/bin/bash
# conv1 TMEM-operand kernels after the division-free loops: ring / strips / rows re-sweep (AlexNet and ResNet conv1)
A="256,3,224,224,64,11,11,2,4"; R="256,3,224,224,64,7,7,3,2"
for t in "" "fct_bd_strips=2" "fct_bd_strips=3" "fct_bd_ring=12"; do echo "== BD $t"; UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $A $R --ops 1 --algos 0 --batches 256; done
for t in "" "fct_ring=40" "fct_rows=1" "fct_epi=8" "fct_epi=4"; do echo "== F $t"; UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $A $R --ops 0 --algos 0 --batches 256; done
for t in "" "fct_bf_ring=12" "fct_bf_dtma=0"; do echo "== BF $t"; UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $A $R --ops 2 --algos 6 --batches 256; done
