"""Sliced K1t (K-slices through the fp32 running sum) vs the fused-mma path:
agreement and run-to-run determinism on given shapes and M."""
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04610_b200 import anyq  # noqa: E402
from scripts.gemv_probe import synthetic  # noqa: E402

for (n, k, m) in [(14336, 4096, 9), (14336, 4096, 16), (4096, 4096, 9), (14336, 2048, 9), (14336, 4096, 12),
                  (2048, 4096, 9), (14336, 1024, 9)]:
    qt = synthetic(n, k, seed=1)
    dt = anyq.DeviceTensor(qt)
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    outs = []
    for rep in range(3):
        y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        y32 = torch.empty(m, n, device="cuda", dtype=torch.float32)
        dt.gemm(x, y, y32, path=5)
        torch.cuda.synchronize()
        outs.append(y32.clone())
    ref32 = torch.empty(m, n, device="cuda", dtype=torch.float32)
    dt.gemm(x, None, ref32, path=4)
    torch.cuda.synchronize()
    det = all(torch.equal(outs[0], o) for o in outs[1:])
    d = (outs[0] - ref32).abs()
    bad = (d > 1e-2 * ref32.abs().max()).nonzero()
    print(f"n={n} k={k} m={m}: det={det} maxdiff={d.max().item():.3e} scale={ref32.abs().max().item():.3e} "
          f"bad={bad.shape[0]} rows_m={sorted(set(bad[:, 0].tolist()))[:16]} first_cols={bad[:5, 1].tolist()}")
    dt.close()
