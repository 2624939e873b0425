"""Prints the benchmarker's per-(algo, micro-batch) times for a few layers
(debug helper: python scripts/time_table.py "N,C,H,W,K,R,S,p,s" ... [--ops 0,1,2])."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_04806_b200 import ConvShape, Handle

ap = argparse.ArgumentParser()
ap.add_argument("shapes", nargs="+")
ap.add_argument("--ops", default="0,1,2")
ap.add_argument("--algos", default="0,1,2,3,4,5")
ap.add_argument("--batches", default="256,64,16")
a = ap.parse_args()
h = Handle()
for spec in a.shapes:
    v = [int(t) for t in spec.split(",")]
    s = ConvShape(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[7], v[8], v[8])
    for op in map(int, a.ops.split(",")):
        print(f"{spec} op={'F BD BF'.split()[op]}")
        for algo in map(int, a.algos.split(",")):
            row = []
            for b in map(int, a.batches.split(",")):
                try:
                    t, ws, ok = h.time_algorithm(op, s, algo, b)
                    row.append(f"{b}:{t * 256 / b:8.3f}ms/{ws >> 20}M" if ok else f"{b}:      --")
                except Exception as e:  # noqa: BLE001
                    row.append(f"{b}: err")
            print(f"  algo {algo}: " + "  ".join(row))
