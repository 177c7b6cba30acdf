"""Per-CTA timeline of the CUDA-core LUT GEMV (debug hook anyq_debug_set_gemv_trace).

usage: python scripts/trace_gemv.py SHAPE M
"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gemv_probe import SHAPES, synthetic  # noqa: E402

from paper_2507_04610_b200 import anyq  # noqa: E402

# trace slots of gemv.cu (GV_TRACE)
NAMES = {0: "start", 1: "table0_built", **{2 + i: f"xprep_img{i}" for i in range(8)},
         **{16 + p: f"dep_wait_p{p}" for p in range(8)}, **{24 + p: f"dep_done_p{p}" for p in range(8)},
         **{32 + g: f"item{g}_done" for g in range(8)}, 63: "end"}


def main():
    name, m = sys.argv[1], int(sys.argv[2])
    n, k = SHAPES[name]
    L = anyq.lib()
    L.anyq_debug_set_gemv_trace.argtypes = [C.c_void_p]
    dt = anyq.DeviceTensor(synthetic(n, k))
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    tr = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
    t_end = time.time() + 0.3
    while time.time() < t_end:
        for _ in range(50):
            dt.gemm(x, y, path=1)
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        dt.gemm(x, y, path=1)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} M={m}: {e0.elapsed_time(e1) * 1e3 / 200:.2f} us per call, same tensor back to back")
    for rep in range(3):
        tr.zero_()
        L.anyq_debug_set_gemv_trace(C.c_void_p(tr.data_ptr()))
        dt.gemm(x, y, path=1)
        torch.cuda.synchronize()
        L.anyq_debug_set_gemv_trace(None)
        t = tr.cpu().numpy().reshape(148, 64)
        t0 = t[:, 0][t[:, 0] > 0].min()
        print(f"{name} M={m} rep {rep}: us after first CTA start: median / min / max")
        for s, nm in NAMES.items():
            col = t[:, s]
            col = col[col > 0]
            if col.size:
                rel = (col - t0) / 1e3
                print(f"  {nm:14s} med {np.median(rel):7.2f}  min {rel.min():7.2f}  max {rel.max():7.2f}")


if __name__ == "__main__":
    main()
