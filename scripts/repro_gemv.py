"""Tiny single-problem GEMV launch (for compute-sanitizer)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemv_probe import synthetic  # noqa: E402

from paper_2507_04610_b200 import anyq  # noqa: E402

n, k, m = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (200, 384, 1)))
dt = anyq.DeviceTensor(synthetic(n, k))
x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
y = dt.gemm(x, path=1)
torch.cuda.synchronize()
print("ok", float(y.float().abs().sum()))
