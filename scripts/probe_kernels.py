"""Per-kernel timing probe: every concrete algorithm on the AlexNet / ResNet-18
layer shapes at a given batch, via the C ABI benchmarker (CUDA events)."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_04806_b200 import ConvShape, Handle, algorithm_workspace, ALGOS

ALEXNET = [("conv1", ConvShape(256, 3, 224, 224, 64, 11, 11, 2, 2, 4, 4)),
           ("conv2", ConvShape(256, 64, 27, 27, 192, 5, 5, 2, 2, 1, 1)),
           ("conv3", ConvShape(256, 192, 13, 13, 384, 3, 3, 1, 1, 1, 1)),
           ("conv4", ConvShape(256, 384, 13, 13, 256, 3, 3, 1, 1, 1, 1)),
           ("conv5", ConvShape(256, 256, 13, 13, 256, 3, 3, 1, 1, 1, 1))]

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--algos", default="0")
ap.add_argument("--out", default=None)
a = ap.parse_args()
h = Handle()
h.set_benchmark_iterations(2, 5)
rows = []
for name, s in ALEXNET:
    s = s.with_batch(a.batch)
    for op in range(3):
        for algo in [int(x) for x in a.algos.split(",")]:
            t, ws, ok = h.time_algorithm(op, s, algo, a.batch)
            if not ok:
                continue
            tf = s.flops() / (t * 1e-6) / 1e12
            rows.append(dict(layer=name, op=op, algo=ALGOS[algo], us=round(t, 1), tflops=round(tf, 1), ws=ws))
            print(f"{name} op{op} {ALGOS[algo]:14s} {t:9.1f} us {tf:7.1f} TFLOP/s ws={ws}", flush=True)
tot = sum(r["us"] for r in rows)
print("total us", round(tot, 1))
if a.out:
    json.dump(rows, open(a.out, "w"), indent=1)
