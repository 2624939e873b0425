import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1804_04806_b200 import ConvShape, Handle, algorithm_workspace
from tests.oracle_py import conv_ref, inputs_for, out_shape
np.set_printoptions(linewidth=200, precision=1, suppress=True)
for s in [ConvShape(1, 32, 8, 8, 32, 1, 1, 0, 0, 1, 1), ConvShape(1, 32, 4, 8, 32, 1, 1, 0, 0, 1, 1)]:
    rng = np.random.default_rng(0)
    a, b = inputs_for(2, s, rng, integer=True)
    ref = conv_ref(2, s, a, b)
    ws_b, ok = algorithm_workspace(2, s, 5, s.N)
    dev = torch.device("cuda")
    out = torch.full(out_shape(2, s), 7.0, device=dev)
    ws = torch.zeros(ws_b // 4 + 64, device=dev)
    Handle().run(2, s, torch.from_numpy(a).float().to(dev), torch.from_numpy(b).float().to(dev), out, 5, ws)
    torch.cuda.synchronize()
    got = out.cpu().double().numpy().reshape(32, 32)
    ref = ref.reshape(32, 32)
    print("shape", s, "equal", np.array_equal(got, ref), "zeros", (got == 0).sum(), "nan", np.isnan(got).sum())
    print("got[:6,:8]\n", got[:6, :8]); print("ref[:6,:8]\n", ref[:6, :8])
    # is it transposed?
    print("transposed eq", np.array_equal(got, ref.T))
    # nhwc buffers
    xn = ws[: s.N * s.H * s.W * 32].view(s.N, s.H * s.W, 32).cpu().numpy()
    print("xn ok", np.array_equal(xn[0], a.reshape(32, -1).T))
