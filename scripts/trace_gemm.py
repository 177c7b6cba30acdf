"""Per-CTA timeline of the tensor-core LUT GEMM (debug hook anyq_debug_set_trace).

usage: python scripts/trace_gemm.py N K M
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from prof_one import synthetic_tensor  # noqa: E402

from paper_2507_04610_b200 import anyq  # noqa: E402

NAMES = {0: "start", 1: "prologue", 2: "prod_first_issue", 3: "prod_done", 4: "mma_first_full",
         5: "mma_done", 6: "epi_staged", 7: "epi_first_drain", 8: "epi_flush_full",
         9: "epi_flush_part", 10: "dq_table", 11: "dq_done", 12: "end",
         13: "flush1_begin", 14: "flush1_atomic_done", 15: "flush1_done"}


def main():
    n, k, m = (int(a) for a in sys.argv[1:4])
    L = anyq.lib()
    L.anyq_debug_set_trace.argtypes = [C.c_void_p]
    dt = anyq.DeviceTensor(synthetic_tensor(n, k))
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    tr = torch.zeros(148 * 16 + 9 * 256, dtype=torch.int64, device="cuda")
    # warm the SM clocks up (~0.2 s of back-to-back GEMMs) before tracing
    import time
    t_end = time.time() + 0.3
    while time.time() < t_end:
        for it in range(50):
            dt.gemm(x, y)
        torch.cuda.synchronize()
    L.anyq_debug_set_trace(C.c_void_p(tr.data_ptr()))
    dt.gemm(x, y)
    torch.cuda.synchronize()
    L.anyq_debug_set_trace(None)
    allt = tr.cpu().numpy().astype(np.int64)
    t = allt[:148 * 16].reshape(148, 16)
    ev = allt[148 * 16:].reshape(9, 256)
    t0 = t[:, 0][t[:, 0] > 0].min()
    print(f"{n}x{k} M={m}: per-CTA stamps (us after first CTA start): median / max")
    for s, name in NAMES.items():
        col = t[:, s]
        col = col[col > 0]
        if col.size:
            rel = (col - t0) / 1e3
            print(f"  {name:18s} med {np.median(rel):7.2f}  min {rel.min():7.2f}  max {rel.max():7.2f}")
    c0 = t[0, 0]
    names = ["mma_full_ok", "mma_afull_ok", "mma_accempty", "mma_committed", "epi_accfull_ok",
             "epi_drained", "dq_full_ok", "dq_aempty_ok", "dq_afull_arriv"]
    print("CTA0 per-chunk events (ns after CTA start):")
    print("  i " + " ".join(f"{n[:14]:>15s}" for n in names))
    for i in range(min(40, 256)):
        row = [ev[e, i] - c0 if ev[e, i] > 0 else -1 for e in range(9)]
        if all(r < 0 for r in row):
            continue
        print(f"{i:3d} " + " ".join(f"{r:15d}" for r in row))


if __name__ == "__main__":
    main()
