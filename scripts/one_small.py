"""Runs one small convolution through a concrete algorithm and compares with
the fp64 oracle (debug helper: python scripts/one_small.py N C H W K R S p s op algo)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1804_04806_b200 import ConvShape, Handle, algorithm_workspace
from paper_1804_04806_b200.api import set_trace, take_trace
from tests.oracle_py import conv_ref, inputs_for, out_shape
v = [int(t) for t in sys.argv[1:]]
s = ConvShape(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[7], v[8], v[8])
op, algo = v[9], v[10]
rng = np.random.default_rng(1)
a, b = inputs_for(op, s, rng, integer=True)
dev = torch.device("cuda")
ws_b, ok = algorithm_workspace(op, s, algo, s.N)
ws = torch.empty(max(ws_b, 4) // 4 + 1, device=dev)
out = torch.zeros(out_shape(op, s), device=dev)
set_trace(True)
Handle().run(op, s, torch.from_numpy(a).float().to(dev), torch.from_numpy(b).float().to(dev), out, algo, ws)
torch.cuda.synchronize()
got = out.cpu().double().numpy(); ref = conv_ref(op, s, a, b)
print("trace", take_trace())
print(s, "op", op, "algo", algo, "maxdiff", np.abs(got - ref).max(), "exact", np.array_equal(got, ref))
