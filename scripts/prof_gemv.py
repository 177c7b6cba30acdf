"""Runs one small-M LUT GEMM path a few times on a synthetic weight (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemv_probe import SHAPES, synthetic  # noqa: E402

from paper_2507_04610_b200 import anyq  # noqa: E402


def main():
    name, m, path = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    iters = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    n, k = SHAPES[name]
    dt = anyq.DeviceTensor(synthetic(n, k))
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(iters):
        dt.gemm(x, y, path=path)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
