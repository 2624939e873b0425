"""Per-call roofline table of a bench JSON line: each planned call's
algorithmic FLOPs (2*N*K*C*R*S*OH*OW), its eager
device time (per_kernel_ms), achieved TFLOP/s and the fraction of the
line's measured TF32 peak, plus its plan.

  python scripts/roofline_table.py profiles/r02_bench_v10.json [configs/alexnet.net] > profiles/r02_alexnet_roofline.txt
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1804_04806_b200.network import parse_net  # noqa: E402


def main():
    line = json.load(open(sys.argv[1]))
    net = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "configs", line["config"]["net"] + ".net")
    _, layers = parse_net(net, 256)
    shapes = {L.name: L.shape for L in layers}
    peak = line["roofline"]["peak"]
    print(f"{sys.argv[1]}: {line['value']} ms/iter, TF32 peak {peak} TFLOP/s ({line['roofline']['peak_source']})")
    print(f"{'call':28s} {'ms':>7s} {'GFLOP':>7s} {'TFLOP/s':>8s} {'frac':>6s}  plan")
    total = 0.0
    for name, ms in sorted(line["per_kernel_ms"].items(), key=lambda kv: -kv[1]):
        s = shapes[name.split("/")[0]]
        gf = s.flops() / 1e9
        total += gf
        tf = gf / ms
        print(f"{name:28s} {ms:7.3f} {gf:7.1f} {tf:8.1f} {tf / peak:6.3f}  {line['plans'][name]}")
    print(f"step: {total:.1f} GFLOP in {line['value']} ms = {total / line['value']:.1f} TFLOP/s "
          f"({total / line['value'] / peak:.3f} of peak)")


if __name__ == "__main__":
    main()
