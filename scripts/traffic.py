"""Per-call DRAM traffic of the planned AlexNet step, for bench.py's
roofline.traffic: run under ncu with dram__bytes_{read,write}.sum, each of
the 15 C-ABI calls preceded by a one-element fill (marker kernel), then
`--parse launches.csv plan.json out.json` sums each call's launches.

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \\
      --log-file gpurun_out/traffic.csv python scripts/traffic.py --db gpurun_out/db.csv
  python scripts/traffic.py --parse gpurun_out/traffic.csv gpurun_out/bench.json profiles/r01_traffic.json
"""
import argparse, csv, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--db", default="")
ap.add_argument("--net", default="alexnet")
ap.add_argument("--limit-mib", type=int, default=64)
ap.add_argument("--parse", nargs=3, metavar=("CSV", "BENCH_JSON", "OUT"))
a = ap.parse_args()
if a.parse:
    src, bj, out = a.parse
    rows = list(csv.DictReader(l for l in open(src) if not l.startswith("==")))
    launches = {}
    for r in rows:
        d = launches.setdefault(r["ID"], {"name": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    seq = [launches[k] for k in sorted(launches, key=int)]
    bench = json.load(open(bj))
    names = list(bench["plans"])
    calls, cur = [], None
    for L in seq:
        if "FillFunctor" in L["name"]:
            cur = {"bytes": 0.0, "ns": 0.0, "kernels": []}
            calls.append(cur)
        elif cur is not None:
            cur["bytes"] += L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
            cur["ns"] += L.get("gpu__time_duration.sum", 0)
            cur["kernels"].append(L["name"].split("(")[0].split("::")[-1])
    calls = calls[-len(names):]  # the last marked pass (earlier ones warm up)
    res = {n: {"plan": bench["plans"][n], "dram_bytes": int(c["bytes"]), "ncu_us": round(c["ns"] / 1e3, 1),
               "kernels": sorted(set(c["kernels"]))} for n, c in zip(names, calls)}
    json.dump({"source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum per C-ABI call ({os.path.basename(src)})",
               "calls": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))
    sys.exit(0)

import torch
from paper_1804_04806_b200 import Handle
from paper_1804_04806_b200.network import ConvStack
dev = torch.device("cuda", 0)
stack = ConvStack(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs",
                               a.net + ".net"), 256, dev)
h = Handle(policy="powerOfTwo", mode="wr", database=a.db or None)
stack.plan(h, a.limit_mib << 20)
mark = torch.zeros(1, device=dev)
for rep in range(2):
    for i, op in stack.kernels():
        mark.fill_(float(i * 3 + op))
        stack.run_kernel(h, i, op)
torch.cuda.synchronize()
print("ok")
