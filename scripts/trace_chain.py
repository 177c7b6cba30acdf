"""Per-CTA timeline of one 8B-layer chain launch (anyq_debug_set_gemv_trace)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gemv_probe import synthetic  # noqa: E402

from paper_2507_04610_b200 import anyq  # noqa: E402

LAYER = [("q", 4096, 4096), ("k", 1024, 4096), ("v", 1024, 4096), ("o", 4096, 4096),
         ("gate", 14336, 4096), ("up", 14336, 4096), ("down", 4096, 14336)]


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    L = anyq.lib()
    L.anyq_debug_set_gemv_trace.argtypes = [C.c_void_p]
    tens = [anyq.DeviceTensor(synthetic(n, k, seed=i)) for i, (_, n, k) in enumerate(LAYER)]
    x = torch.randn(m, 4096, device="cuda").to(torch.bfloat16)
    ys = [torch.empty(m, n, device="cuda", dtype=torch.bfloat16) for _, n, _ in LAYER]
    xs = [x, x, x, ys[0], ys[3], ys[3], ys[5]]
    waits = [0, 0, 0, 1, 1, 0, 1]
    tr = torch.zeros(148 * 64 + 15 * 16, dtype=torch.int64, device="cuda")
    t_end = time.time() + 0.3
    while time.time() < t_end:
        for _ in range(20):
            anyq.gemm_chain(tens, xs, ys, deps=[-1, -1, -1, 0, 3, 3, 5])
        torch.cuda.synchronize()
    L.anyq_debug_set_gemv_trace(C.c_void_p(tr.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    anyq.gemm_chain(tens, xs, ys, deps=[-1, -1, -1, 0, 3, 3, 5])
    e1.record()
    torch.cuda.synchronize()
    L.anyq_debug_set_gemv_trace(None)
    print(f"chain event time {e0.elapsed_time(e1)*1e3:.1f} us")
    allt = tr.cpu().numpy()
    t = allt[:148 * 64].reshape(148, 64)
    w = allt[148 * 64:].reshape(15, 16)
    t0 = t[:, 0][t[:, 0] > 0].min()
    names = {0: "start", 1: "prologue_done", 63: "end"}
    for p_ in range(7):
        names[2 + p_] = f"xbatch{p_}_ready"
        names[16 + p_] = f"wait{p_}_begin"
        names[24 + p_] = f"wait{p_}_end"
    for s_, nm in names.items():
        col = t[:, s_]
        col = col[col > 0]
        if col.size:
            rel = (col - t0) / 1e3
            print(f"  {nm:16s} med {np.median(rel):7.2f}  min {rel.min():7.2f}  max {rel.max():7.2f}")
    for b in (0, 1, 100):
        row = t[b, 32:63]
        print(f"  CTA {b} item ends: " + " ".join(f"{(v - t0) / 1e3:.1f}" for v in row if v > 0))
    return
    print("CTA 0 per warp (rows: seg g stage k; cols: warps 0..15):")
    for g in range(3):
        for k, nm in enumerate(["start", "chunk1", "consumed", "handed", "tbl_built"]):
            r = w[g * 5 + k]
            print(f"  seg{g} {nm:9s} " + " ".join(f"{(v - t0) / 1e3:5.2f}" if v > 0 else "  -  " for v in r))
    return
    for b in (0, 1, 100):
        row = t[b, 32:62]
        print(f"  CTA {b}: " + " ".join(f"{(v - t0) / 1e3:.1f}" for v in row if v > 0))


if __name__ == "__main__":
    main()


def stragglers():
    pass
