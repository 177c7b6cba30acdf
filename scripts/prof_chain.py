"""Runs the 8B-layer chain a few times (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gemv_probe import synthetic  # noqa: E402
from trace_chain import LAYER  # noqa: E402

from paper_2507_04610_b200 import anyq  # noqa: E402

tens = [anyq.DeviceTensor(synthetic(n, k, seed=i)) for i, (_, n, k) in enumerate(LAYER)]
x = torch.randn(1, 4096, device="cuda").to(torch.bfloat16)
ys = [torch.empty(1, n, device="cuda", dtype=torch.bfloat16) for _, n, _ in LAYER]
xs = [x, x, x, ys[0], ys[3], ys[3], ys[5]]
for _ in range(4):
    anyq.gemm_chain(tens, xs, ys, wait_prev=[0, 0, 0, 1, 1, 0, 1])
torch.cuda.synchronize()
print("ok")
