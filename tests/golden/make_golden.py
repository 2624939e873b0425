"""Regenerates the planner golden fixtures from the REFERENCE planner.

Runs oracle/_ref/ref_plan (the unmodified reference headers under
/root/reference/proj/include, compiled by `make -C oracle ref`) and stores
its machine reports / flushed cost tables. Committed outputs:
  reports/<case>.txt   machine report of the reference (builtin model)
  csv/<case>.csv       the reference's write-through cost table for the case
  random.jsonl         seeded random instances: net, model, args, report, csv
Run from the repo root:  python tests/golden/make_golden.py
"""
import json
import os
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "oracle", "_ref", "ref_plan")
OUT = os.path.dirname(os.path.abspath(__file__))
MiB = 1 << 20

# (case, net, batch, mode, policy, limit, keep_csv)
CASES = [
    ("alexnet_wr_pow2_64M", "alexnet", 256, "wr", "powerOfTwo", 64 * MiB, True),
    ("alexnet_wr_all_64M", "alexnet", 256, "wr", "all", 64 * MiB, False),
    ("alexnet_wr_undiv_64M", "alexnet", 256, "wr", "undivided", 64 * MiB, False),
    ("alexnet_wr_all_8M", "alexnet", 256, "wr", "all", 8 * MiB, False),
    ("alexnet_wr_pow2_512M", "alexnet", 256, "wr", "powerOfTwo", 512 * MiB, False),
    ("alexnet_wd_all_120M", "alexnet", 256, "wd", "all", 120 * MiB, False),
    ("alexnet_wd_pow2_120M", "alexnet", 256, "wd", "powerOfTwo", 120 * MiB, True),
    ("alexnet_wd_pow2_960M", "alexnet", 256, "wd", "powerOfTwo", 960 * MiB, False),
    ("resnet18_wr_all_64M", "resnet18", 256, "wr", "all", 64 * MiB, False),
    ("resnet18_wr_pow2_64M", "resnet18", 256, "wr", "powerOfTwo", 64 * MiB, True),
    ("resnet18_wr_undiv_64M", "resnet18", 256, "wr", "undivided", 64 * MiB, False),
    ("resnet18_wd_pow2_1G", "resnet18", 256, "wd", "powerOfTwo", 1024 * MiB, False),
    ("resnet50_wd_pow2_2544M", "resnet50", 256, "wd", "powerOfTwo", 2544 * MiB, True),
    ("resnet50_wd_all_2544M", "resnet50", 256, "wd", "all", 2544 * MiB, False),
    ("resnet50_wr_pow2_64M", "resnet50", 256, "wr", "powerOfTwo", 64 * MiB, False),
    ("resnet50_wd_pow2_32_2544M", "resnet50", 32, "wd", "powerOfTwo", 2544 * MiB, False),
]


def ref_optimize(net, batch, mode, policy, limit, cost="builtin", flush=None, jobs=8):
    args = [REF, "optimize", net, str(batch), mode, policy, str(limit), str(jobs), cost]
    if flush:
        args.append(flush)
    p = subprocess.run(args, capture_output=True, text=True)
    if p.returncode not in (0, 3):
        raise RuntimeError(p.stderr)
    return p.stdout


def main():
    os.makedirs(os.path.join(OUT, "reports"), exist_ok=True)
    os.makedirs(os.path.join(OUT, "csv"), exist_ok=True)
    for case, net, batch, mode, policy, limit, keep in CASES:
        netf = os.path.join(ROOT, "configs", net + ".net")
        with tempfile.TemporaryDirectory() as td:
            flush = os.path.join(td, "t.csv")
            rep = ref_optimize(netf, batch, mode, policy, limit, flush=flush)
            open(os.path.join(OUT, "reports", case + ".txt"), "w").write(rep)
            if keep:
                os.replace(flush, os.path.join(OUT, "csv", case + ".csv"))
        print(case, rep.splitlines()[-6] if rep else "")
    with tempfile.TemporaryDirectory() as td:
        subprocess.check_call([REF, "random", td, "300", "424242"])
        with open(os.path.join(OUT, "random.jsonl"), "w") as f:
            for i in range(300):
                b = os.path.join(td, str(i))
                rec = {k: open(b + "." + k).read() for k in ("net", "model", "args", "report", "csv")}
                f.write(json.dumps(rec) + "\n")
    print("random instances: 300")



# Measured B200 cost tables (written by bench.py's device benchmarker, nine
# algorithm ids, ns-resolution times) replayed through the REFERENCE planner:
# (case, net, batch, mode, policy, limit, csv file in csv/)
B200_CASES = [
    ("b200_alexnet_wr_pow2_64M", "alexnet", 256, "wr", "powerOfTwo", 64 * MiB, "b200_alexnet_pow2_64M"),
    ("b200_alexnet_wr_undiv_64M", "alexnet", 256, "wr", "undivided", 64 * MiB, "b200_alexnet_pow2_64M"),
    ("b200_alexnet_wr_pow2_8M", "alexnet", 256, "wr", "powerOfTwo", 8 * MiB, "b200_alexnet_pow2_64M"),
    ("b200_alexnet_wd_pow2_960M", "alexnet", 256, "wd", "powerOfTwo", 960 * MiB, "b200_alexnet_pow2_64M"),
    ("b200_alexnet_wd_pow2_240M", "alexnet", 256, "wd", "powerOfTwo", 240 * MiB, "b200_alexnet_pow2_64M"),
    ("b200_alexnet_wr_all_64M", "alexnet", 256, "wr", "all", 64 * MiB, "b200_alexnet_all_64M"),
    ("b200_alexnet_wd_all_960M", "alexnet", 256, "wd", "all", 960 * MiB, "b200_alexnet_all_64M"),
    ("b200_resnet18_wr_pow2_64M", "resnet18", 256, "wr", "powerOfTwo", 64 * MiB, "b200_resnet18_pow2_64M"),
    ("b200_resnet18_wd_pow2_1280M", "resnet18", 256, "wd", "powerOfTwo", 1280 * MiB, "b200_resnet18_pow2_64M"),
    ("b200_resnet50_wd_pow2_2544M", "resnet50", 256, "wd", "powerOfTwo", 2544 * MiB, "b200_resnet50_wd_pow2_2544M"),
]


def make_b200_golden():
    for case, net, batch, mode, policy, limit, csv in B200_CASES:
        rep = ref_optimize(os.path.join(ROOT, "configs", net + ".net"), batch, mode, policy, limit,
                           cost=os.path.join(OUT, "csv", csv + ".csv"))
        open(os.path.join(OUT, "reports", case + ".txt"), "w").write(rep)
        print(case, len(rep.splitlines()), "lines")


def make_conv_golden():
    """Small conv golden vectors from the reference's own execute_plan
    (oracle/_ref/ref_conv.so): integer inputs, one stride-2 and one padded
    case per op, a non-trivial micro-batch plan each."""
    import sys
    import numpy as np
    sys.path.insert(0, ROOT)
    from paper_1804_04806_b200.api import ConvShape
    from tests.oracle_py import conv_ref, inputs_for
    cases = [(ConvShape(5, 3, 9, 8, 4, 3, 3, 1, 1, 2, 2), [2, 2, 1]),
             (ConvShape(4, 2, 7, 7, 3, 5, 5, 2, 2, 1, 1), [3, 1]),
             (ConvShape(3, 4, 11, 11, 2, 11, 11, 2, 2, 4, 4), [1, 1, 1])]
    out = {}
    for i, (s, plan) in enumerate(cases):
        for op in range(3):
            a, b = inputs_for(op, s, np.random.default_rng(100 * i + op), integer=True)
            out[f"c{i}_op{op}_a"], out[f"c{i}_op{op}_b"] = a, b
            out[f"c{i}_op{op}_out"] = conv_ref(op, s, a, b, plan, use_reference=True)
        out[f"c{i}_shape"] = np.array([s.N, s.C, s.H, s.W, s.K, s.R, s.S, s.ph, s.pw, s.sh, s.sw])
        out[f"c{i}_plan"] = np.array(plan)
    np.savez_compressed(os.path.join(OUT, "conv_golden.npz"), **out)
    print("conv golden:", len(cases), "cases x 3 ops")


if __name__ == "__main__":
    import sys
    if sys.argv[1:] == ["b200"]:
        make_b200_golden()
    else:
        main()
        make_conv_golden()
        make_b200_golden()
