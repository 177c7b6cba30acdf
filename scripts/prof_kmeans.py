"""Timing probe of the device k-means quantizer: fixed cost vs per-row cost.

usage: python scripts/prof_kmeans.py [rows ...]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04610_b200 import _abi, anyq  # noqa: E402


def main():
    specs = sys.argv[1:] or ["148", "296", "1024", "4096", "8192"]
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    cfg = _abi.default_config(codebook=_abi.CB_ANY)
    for spec in specs:  # "ROWS" or "ROWSxCOLS"
        r, c = (int(v) for v in spec.split("x")) if "x" in spec else (int(spec), 4096)
        x = torch.randn(r, c, device=dev, generator=g)
        anyq.dev_quantize_any(x, cfg)  # warm (scratch pool)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            anyq.dev_quantize_any(x, cfg)
            e1.record()
            torch.cuda.synchronize()
            ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
        ev = min(t[0] for t in ts)
        wall = min(t[1] for t in ts)
        print(f"rows {r:6d} x {c:5d}: event {ev:8.2f} ms  wall {wall:8.2f} ms  -> {r / ev * 1e3:10.0f} rows/s")


if __name__ == "__main__":
    main()
