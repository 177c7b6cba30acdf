"""Sliced K1t: in-place y32 running sum vs stream-scratch running sum (bf16 y)."""
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04610_b200 import anyq  # noqa: E402
from scripts.gemv_probe import synthetic  # noqa: E402

for (n, k, m) in [(14336, 4096, 9), (14336, 4096, 12), (14336, 4096, 16)]:
    qt = synthetic(n, k, seed=1)
    dt = anyq.DeviceTensor(qt)
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    ys = []
    for rep in range(4):
        y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        dt.gemm(x, y, None, path=5)
        torch.cuda.synchronize()
        ys.append(y.clone())
    ys32 = []
    for rep in range(4):
        y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        y32 = torch.zeros(m, n, device="cuda", dtype=torch.float32)
        dt.gemm(x, y, y32, path=5)
        torch.cuda.synchronize()
        ys32.append(y.clone())
    print(f"n={n} k={k} m={m}: scratch det={all(torch.equal(ys[0], o) for o in ys[1:])} "
          f"inplace det={all(torch.equal(ys32[0], o) for o in ys32[1:])} same={torch.equal(ys[0], ys32[0])}")
    dt.close()
