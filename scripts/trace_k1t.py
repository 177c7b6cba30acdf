"""Per-chunk-group timeline of K1t (gemv.cu TC_TRACE) on one shape.
usage: python scripts/trace_k1t.py SHAPE M [cta]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gemv_probe import SHAPES, synthetic  # noqa: E402

from paper_2507_04610_b200 import anyq  # noqa: E402

EV = ["dq0_top", "dq0_lookups_in", "dq0_got_afree", "dq0_arrived", "mma_got_a", "mma_issued",
      "epi_got_d", "dq3_arrived"]


def main():
    name, m = sys.argv[1], int(sys.argv[2])
    ctas = [int(c) for c in (sys.argv[3] if len(sys.argv) > 3 else "0,77").split(",")]
    n, k = SHAPES[name]
    L = anyq.lib()
    L.anyq_debug_set_gemv_trace.argtypes = [C.c_void_p]
    dt = anyq.DeviceTensor(synthetic(n, k))
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    tr = torch.zeros(148 * 64 + 148 * 8 * 64, dtype=torch.int64, device="cuda")
    for _ in range(20):
        dt.gemm(x, y, path=5)
    torch.cuda.synchronize()
    tr.zero_()
    L.anyq_debug_set_gemv_trace(C.c_void_p(tr.data_ptr()))
    dt.gemm(x, y, path=5)
    torch.cuda.synchronize()
    L.anyq_debug_set_gemv_trace(None)
    t = tr.cpu().numpy()[148 * 64:].reshape(148, 8, 64)
    t0 = t[t > 0].min()
    for b in ctas:
        print(f"CTA {b}: ns after the first stamp (chunk group index across)")
        for e, nm in enumerate(EV):
            row = t[b, e]
            v = [f"{(x - t0):6d}" if x > 0 else "     -" for x in row[:32]]
            print(f"  {nm:14s} " + " ".join(v))


if __name__ == "__main__":
    main()
