"""Runs IMPLICIT_PRECOMP_GEMM on the AlexNet layers with UCUDNN_TUNE=prof=1 and
prints the MMA warp's cycle split (operand wait / issue / accumulator wait)."""
import ctypes as C, os, sys
os.environ["UCUDNN_TUNE"] = os.environ.get("UCUDNN_TUNE", "prof=1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1804_04806_b200 import Handle, algorithm_workspace
from paper_1804_04806_b200._lib import lib
from paper_1804_04806_b200 import ConvShape
ALEXNET = [("conv1", ConvShape(256, 3, 224, 224, 64, 11, 11, 2, 2, 4, 4)),
           ("conv2", ConvShape(256, 64, 27, 27, 192, 5, 5, 2, 2, 1, 1)),
           ("conv3", ConvShape(256, 192, 13, 13, 384, 3, 3, 1, 1, 1, 1)),
           ("conv4", ConvShape(256, 384, 13, 13, 256, 3, 3, 1, 1, 1, 1)),
           ("conv5", ConvShape(256, 256, 13, 13, 256, 3, 3, 1, 1, 1, 1))]
from tests.oracle_py import out_shape
dev = torch.device("cuda")
h = Handle()
L = lib()
b = int(os.environ.get("BATCH", "64"))
for name, s in ALEXNET:
    s = s.with_batch(b)
    for op in (0, 1, 2):
        x = torch.randn(s.N, s.C, s.H, s.W, device=dev); w = torch.randn(s.K, s.C, s.R, s.S, device=dev)
        dy = torch.randn(s.N, s.K, s.OH, s.OW, device=dev)
        a, bb = [(x, w), (dy, w), (x, dy)][op]
        out = torch.empty(out_shape(op, s), device=dev)
        wsb, ok = algorithm_workspace(op, s, 5, s.N)
        ws = torch.empty(max(wsb, 4) // 4 + 1, device=dev)
        h.run(op, s, a, bb, out, 5, ws)
        torch.cuda.synchronize()
        r = (C.c_double * 4)()
        (L.ucudnnDebugBackwardFilterProfile if op == 2 else L.ucudnnDebugPrecompProfile)(r)
        tot = r[3] or 1
        print(f"{name} op{op}: data-wait {100*r[0]/tot:5.1f}%  issue {100*r[1]/tot:5.1f}%  acc-wait {100*r[2]/tot:5.1f}%  total {r[3]/1.9e3:8.1f} us@1.9GHz")
