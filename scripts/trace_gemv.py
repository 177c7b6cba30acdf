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

NAMES = {0: "start", 1: "loads_issued", 2: "table0_built", 3: "dep_wait_done", 4: "xprep_done",
         5: "bar0", 6: "seg0_done", 7: "seg0_bar", 8: "seg1_done", 9: "seg1_bar", 10: "seg2_done",
         11: "seg2_bar", 12: "seg3_done", 13: "seg3_bar", 15: "end"}


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
    for rep in range(3):
        tr.zero_()
        L.anyq_debug_set_gemv_trace(C.c_void_p(tr.data_ptr()))
        dt.gemm(x, y, path=1)
        torch.cuda.synchronize()
        L.anyq_debug_set_gemv_trace(None)
        t = tr.cpu().numpy().reshape(148, 64)
        t0 = t[:, 0][t[:, 0] > 0].min()
        print(f"{name} M={m} rep {rep}: us after first CTA start: median / min / max")
        ghz = (t[:, 13] - t[:, 12]) / np.maximum(t[:, 15] - t[:, 0], 1)
        print(f"  SM clock during kernel: median {np.median(ghz):.3f} GHz")
        for s, nm in NAMES.items():
            col = t[:, s]
            col = col[col > 0]
            if col.size:
                rel = (col - t0) / 1e3
                print(f"  {nm:14s} med {np.median(rel):7.2f}  min {rel.min():7.2f}  max {rel.max():7.2f}")


if __name__ == "__main__":
    main()
