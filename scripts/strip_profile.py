"""MMA-warp wait split of the strip implicit GEMM (UCUDNN_TUNE=strip=1,prof=1,...):
operand waits (strip + filter stage), filter-stage waits alone, accumulator waits, total."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1804_04806_b200 import Handle, algorithm_workspace, ConvShape
from paper_1804_04806_b200._lib import lib
from tests.oracle_py import out_shape
dev = torch.device("cuda")
h = Handle()
v = [int(t) for t in sys.argv[1].split(",")]
s = ConvShape(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[7], v[8], v[8])
op = int(sys.argv[2])
x = torch.randn(s.N, s.C, s.H, s.W, device=dev); w = torch.randn(s.K, s.C, s.R, s.S, device=dev)
dy = torch.randn(s.N, s.K, s.OH, s.OW, device=dev)
a, b = [(x, w), (dy, w)][op]
out = torch.empty(out_shape(op, s), device=dev)
wsb, ok = algorithm_workspace(op, s, 5, s.N)
ws = torch.empty(max(wsb, 4) // 4 + 1, device=dev)
for _ in range(2):
    h.run(op, s, a, b, out, 5, ws)
torch.cuda.synchronize()
r = (C.c_double * 4)()
lib().ucudnnDebugPrecompProfile(r)
tot = r[3] or 1
print(f"{sys.argv[1]} op{op} {os.environ.get('UCUDNN_TUNE')}: operand-wait {100*r[0]/tot:5.1f}% (stage {100*r[1]/tot:5.1f}%) acc-wait {100*r[2]/tot:5.1f}% total {r[3]/1.9e3:8.1f} us")
if os.environ.get("UCUDNN_TUNE", "").endswith("prof=2"):
    print(f"  prof=2: epilogue busy {r[0]/1.9e3:7.1f} us  last epilogue {r[1]/1.9e3:6.1f} us  tmem-ld {r[2]/1.9e3:6.1f} us  CTA {r[3]/1.9e3:7.1f} us")
