"""Launch split of the dequant+cuBLAS path (run under ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04610_b200 import anyq  # noqa: E402
import bench  # noqa: E402

n, k, m = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dt = anyq.DeviceTensor(bench.synthetic_qtensor(n, k, 5))
x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    dt.gemm(x, y, None, path=3)
torch.cuda.synchronize()
