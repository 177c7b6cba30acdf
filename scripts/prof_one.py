"""Runs the tensor-core LUT GEMM a few times on one synthetic weight (for ncu).

usage: python scripts/prof_one.py N K M [iters]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04610_b200 import _abi, anyq  # noqa: E402
from paper_2507_04610_b200.qtensor import QuantizedTensor  # noqa: E402


def synthetic_tensor(n, k, seed=0, group=128):
    rng = np.random.default_rng(seed)
    cfg = _abi.default_config(codebook=_abi.CB_ANY, group_size=group)
    qt = QuantizedTensor.empty(n, k, cfg)
    qt.codes[:] = rng.integers(0, 256, qt.codes.size, dtype=np.uint8)
    qt.luts[:] = np.sort(rng.random((n, 16), dtype=np.float32) * 15, axis=1).ravel()
    qt.alphas[:] = 0.1 + rng.random(qt.alphas.size, dtype=np.float32)
    qt.betas[:] = -1.0
    return qt


def main():
    n, k, m = (int(a) for a in sys.argv[1:4])
    iters = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    dt = anyq.DeviceTensor(synthetic_tensor(n, k))
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(iters):
        dt.gemm(x, y)
    torch.cuda.synchronize()
    print("ok", float(y.float().abs().sum()))


if __name__ == "__main__":
    main()
