#!/bin/bash
timeout 300 python scripts/time_table.py 256,64,56,56,64,3,3,1,1 256,128,28,28,128,3,3,1,1 --ops 2 --algos 0,5,6,8 --batches 256,128,64 2>&1
python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch
from paper_1804_04806_b200 import ConvShape, Handle, algorithm_workspace
from paper_1804_04806_b200.api import set_trace, take_trace
from tests.oracle_py import out_shape
dev=torch.device('cuda'); h=Handle()
for algo in (5,6,8):
  s=ConvShape(64,64,56,56,64,3,3,1,1,1,1)
  x=torch.randn(s.N,s.C,s.H,s.W,device=dev); dy=torch.randn(s.N,s.K,s.OH,s.OW,device=dev); dw=torch.empty(s.K,s.C,s.R,s.S,device=dev)
  wsb,ok=algorithm_workspace(2,s,algo,s.N)
  if not ok: print(algo,'infeasible'); continue
  ws=torch.empty(max(wsb,4)//4+1,device=dev)
  set_trace(True); h.run(2,s,x,dy,dw,algo,ws); torch.cuda.synchronize(); print(algo, take_trace())
PY
