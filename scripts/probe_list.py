"""Runs a list of (layer, op, algo, batch) convolutions once each (after one
warm-up) -- for `ncu --metrics gpu__time_duration.sum` launch lists."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1804_04806_b200 import Handle, algorithm_workspace
from scripts.one_conv_shapes import LAYERS
from tests.oracle_py import out_shape

dev = torch.device("cuda")
h = Handle()
for spec in sys.argv[1:]:
    layer, op, algo, b = spec.split(":")
    op, algo, b = int(op), int(algo), int(b)
    s = LAYERS[layer].with_batch(b)
    x = torch.randn(s.N, s.C, s.H, s.W, device=dev); w = torch.randn(s.K, s.C, s.R, s.S, device=dev)
    dy = torch.randn(s.N, s.K, s.OH, s.OW, device=dev)
    ins = [(x, w), (dy, w), (x, dy)][op]
    out = torch.empty(out_shape(op, s), device=dev)
    ws_b, _ = algorithm_workspace(op, s, algo, b)
    ws = torch.empty(max(ws_b, 4) // 4 + 1, device=dev)
    for _ in range(2):
        h.run(op, s, ins[0], ins[1], out, algo, ws)
    torch.cuda.synchronize()
    print(spec, "done", flush=True)
