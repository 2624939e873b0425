"""One AlexNet bs256 training step of the bench's plan, eager, for
compute-sanitizer (memcheck / synccheck): the plan comes from the committed
B200 cost table (no benchmarking runs under the sanitizer), every one of the
15 planned calls runs once, BackwardFilter on the bench's two side streams.

  compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_step.py
"""
import os
import shutil
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1804_04806_b200 import Handle  # noqa: E402
from paper_1804_04806_b200.network import ConvStack  # noqa: E402


def main():
    net = sys.argv[1] if len(sys.argv) > 1 else "alexnet"
    csv = os.path.join(ROOT, "tests", "golden", "csv", f"b200_{net}_pow2_64M.csv")
    dev = torch.device("cuda:0")
    with tempfile.TemporaryDirectory() as td:
        db = os.path.join(td, "t.csv")
        shutil.copy(csv, db)
        stack = ConvStack(os.path.join(ROOT, "configs", net + ".net"), 256, dev)
        h = Handle(policy="powerOfTwo", database=db)
        stack.plan(h, 64 << 20)
        sides = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
        stack.step(h, bf_stream=sides)
        torch.cuda.synchronize()
        h.close()
    print("sanitize step ok:", net, "15 planned calls" if net == "alexnet" else "")


if __name__ == "__main__":
    main()
