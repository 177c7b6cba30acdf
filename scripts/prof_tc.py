"""One tcgen05 LUT GEMM launch (path 2) for ncu: gate shape at M given on argv."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04610_b200 import anyq  # noqa: E402
import bench  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dt = anyq.DeviceTensor(bench.synthetic_qtensor(14336, 4096, 5))
x = torch.randn(m, 4096, device="cuda").to(torch.bfloat16)
y = torch.empty(m, 14336, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    dt.gemm(x, y, None, path=int(sys.argv[2]) if len(sys.argv) > 2 else 2)
torch.cuda.synchronize()
