"""Quick device probe: correctness smoke + rough timings of the hot path.

Not the bench (see bench.py); used while iterating on kernels.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.refpy import bf16_round, oracle  # noqa: E402
from paper_2507_04610_b200 import _abi, anyq  # noqa: E402


def timed(fn, iters=50, warm=5):
    import time
    t_end = time.time() + 0.2  # let the SM clocks ramp up first
    while time.time() < t_end:
        fn()
        torch.cuda.synchronize()
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    orc = oracle()
    shapes = [(4096, 4096), (1024, 4096), (14336, 4096), (4096, 14336)]
    for (n, k) in shapes:
        w = orc.gaussian(n, k, 1)
        cfg = _abi.default_config(codebook=_abi.CB_ANY, max_iters=3)
        t0 = time.time()
        qt = anyq.quantize_any(w, cfg)
        t1 = time.time()
        dt = anyq.DeviceTensor(qt)
        for m in (1, 4, 16):
            x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
            y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
            ms = timed(lambda: dt.gemm(x, y))
            nbytes = dt.weight_bytes + m * k * 2 + m * n * 2
            print(f"{n}x{k} M={m}: {ms*1e3:8.2f} us  {nbytes/ms/1e6:8.1f} GB/s "
                  f"(quantize {t1-t0:.2f}s host-call)", flush=True)
        # correctness vs oracle at M=1
        x = bf16_round(orc.gaussian(1, k, 2))
        y32 = torch.empty(1, n, device="cuda")
        dt.gemm(torch.from_numpy(x).cuda().to(torch.bfloat16), y, y32)
        ref = orc.gemm_reference(x, orc.narrowed(qt))
        err = np.abs(y32.cpu().numpy() - ref).max()
        print(f"   max|dy| {err:.3e} max|y| {np.abs(ref).max():.3e}", flush=True)
        dt.close()


if __name__ == "__main__" and not os.environ.get("ROT"):
    main()


def rotating():
    """Back-to-back GEMMs over a rotating set of weights larger than L2."""
    rng = np.random.default_rng(0)
    for (n, k, copies) in [(4096, 4096, 20), (14336, 4096, 6), (1024, 4096, 64)]:
        dts = []
        for c in range(copies):
            cfg = _abi.default_config(codebook=_abi.CB_ANY)
            from paper_2507_04610_b200.qtensor import QuantizedTensor
            qt = QuantizedTensor.empty(n, k, cfg)
            qt.codes[:] = rng.integers(0, 256, qt.codes.size, dtype=np.uint8)
            qt.luts[:] = np.sort(rng.random((n, 16), dtype=np.float32) * 15, axis=1).ravel()
            qt.alphas[:] = 0.1 + rng.random(qt.alphas.size, dtype=np.float32)
            qt.betas[:] = -1.0
            dts.append(anyq.DeviceTensor(qt))
        for m in (1, 16):
            x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
            ys = [torch.empty(m, n, device="cuda", dtype=torch.bfloat16) for _ in dts]
            def run():
                for d, y in zip(dts, ys):
                    d.gemm(x, y)
            ms = timed(run, iters=10, warm=3) / copies
            nbytes = dts[0].weight_bytes + m * k * 2 + m * n * 2
            print(f"rotating {copies}x {n}x{k} M={m}: {ms*1e3:8.2f} us/GEMM  {nbytes/ms/1e6:8.1f} GB/s",
                  flush=True)
        for d in dts:
            d.close()


if __name__ == "__main__" and os.environ.get("ROT"):
    rotating()
