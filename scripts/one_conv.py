"""Runs one convolution (op, layer, algo, batch) a few times -- for ncu captures."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1804_04806_b200 import ConvShape, Handle
from tests.oracle_py import out_shape

LAYERS = {"a1": ConvShape(256, 3, 224, 224, 64, 11, 11, 2, 2, 4, 4),
          "a2": ConvShape(256, 64, 27, 27, 192, 5, 5, 2, 2, 1, 1),
          "a3": ConvShape(256, 192, 13, 13, 384, 3, 3, 1, 1, 1, 1),
          "a4": ConvShape(256, 384, 13, 13, 256, 3, 3, 1, 1, 1, 1),
          "a5": ConvShape(256, 256, 13, 13, 256, 3, 3, 1, 1, 1, 1)}
ap = argparse.ArgumentParser()
ap.add_argument("--layer", default="a2"); ap.add_argument("--op", type=int, default=0)
ap.add_argument("--algo", type=int, default=0); ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--shape", default="", help="N,C,H,W,K,R,S,pad,stride (overrides --layer)")
a = ap.parse_args()
if a.shape:
    v = [int(t) for t in a.shape.split(",")]
    LAYERS["shape"] = ConvShape(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[7], v[8], v[8])
    a.layer = "shape"
s = LAYERS[a.layer].with_batch(a.batch)
dev = torch.device("cuda")
x = torch.randn(s.N, s.C, s.H, s.W, device=dev); w = torch.randn(s.K, s.C, s.R, s.S, device=dev)
dy = torch.randn(s.N, s.K, s.OH, s.OW, device=dev)
ins = [(x, w), (dy, w), (x, dy)][a.op]
out = torch.empty(out_shape(a.op, s), device=dev)
h = Handle()
from paper_1804_04806_b200 import algorithm_workspace
ws_b, _ = algorithm_workspace(a.op, s, a.algo, s.N)
ws = torch.empty(max(ws_b, 4) // 4 + 1, device=dev)
from paper_1804_04806_b200.api import set_trace, take_trace
set_trace(True)
for _ in range(a.reps):
    h.run(a.op, s, ins[0], ins[1], out, a.algo, ws)
torch.cuda.synchronize()
print("trace", take_trace()[:2])
print("ok")
