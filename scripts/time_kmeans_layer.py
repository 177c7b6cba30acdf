"""Time the device quantizer (anyq_dev_quantize_any) on one Llama-3-8B layer
(config 4 stratified, as bench.py); LIB=path selects the library build."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04610_b200 import _abi  # noqa: E402

L = C.CDLL(os.environ.get("LIB") or os.path.join(os.path.dirname(__file__), "..", "paper_2507_04610_b200", "_lib",
                                                  "libanyq_b200.so"))
vp = C.c_void_p
L.anyq_dev_quantize_any.restype = C.c_int
L.anyq_dev_quantize_any.argtypes = [vp, C.c_int64, C.c_int64, C.POINTER(_abi.Config), vp, C.c_int64, vp, vp, vp, vp, vp]
LAYER = [(4096, 4096), (1024, 4096), (1024, 4096), (4096, 4096), (14336, 4096), (14336, 4096), (4096, 14336)]
dev = torch.device("cuda")
cfg = _abi.default_config(codebook=_abi.CB_ANY)
mats = []
for i, (n, k) in enumerate(LAYER):
    g = torch.Generator(device=dev)
    g.manual_seed(1 + i)
    exj = torch.rand(k, device=dev, generator=g) + 0.05
    w = torch.randn(n, k, device=dev, generator=g)
    out = [torch.empty(n * k // 2, dtype=torch.uint8, device=dev), torch.empty(n * 16, device=dev),
           torch.empty(n * (k // 128), device=dev), torch.empty(n * (k // 128), device=dev)]
    mats.append((w, exj, out))
s = torch.cuda.current_stream().cuda_stream


def run(w, e, out):
    st = L.anyq_dev_quantize_any(w.data_ptr(), w.shape[0], w.shape[1], C.byref(cfg), e.data_ptr(), 0,
                                 out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(), out[3].data_ptr(), s)
    assert st == 0, st


for m in mats:
    run(*m)
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for m in mats:
        run(*m)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"layer {ms:.2f} ms  {43008 / ms * 1e3:.0f} rows/s", flush=True)
for i, m in enumerate(mats):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(*m)
    e1.record()
    torch.cuda.synchronize()
    print(i, LAYER[i], f"{e0.elapsed_time(e1):.2f} ms")
