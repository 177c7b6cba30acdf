"""Correctness + timing probe of the small-M LUT GEMM paths (GEMV and tcgen05).

usage: python scripts/gemv_probe.py [--paths 1,2] [--ms 1,2,4] [--shapes q,k,gate,down]

Weights rotate over enough copies to exceed 2x L2, so every call streams
from HBM. Times are CUDA-event device times of back-to-back graph replays.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04610_b200 import _abi, anyq  # noqa: E402
from paper_2507_04610_b200.qtensor import QuantizedTensor  # noqa: E402

SHAPES = {"q": (4096, 4096), "k": (1024, 4096), "gate": (14336, 4096), "down": (4096, 14336),
          "q70": (8192, 8192), "gate70": (28672, 8192)}


def synthetic(n, k, seed=0, group=128):
    rng = np.random.default_rng(seed)
    cfg = _abi.default_config(codebook=_abi.CB_ANY, group_size=group)
    qt = QuantizedTensor.empty(n, k, cfg)
    qt.codes[:] = rng.integers(0, 256, qt.codes.size, dtype=np.uint8)
    qt.luts[:] = np.sort(rng.random((n, 16), dtype=np.float32) * 15, axis=1).ravel()
    qt.alphas[:] = (0.01 + 0.04 * rng.random(qt.alphas.size)).astype(np.float32)
    qt.betas[:] = (-0.3 * rng.random(qt.betas.size)).astype(np.float32)
    return qt


def dequant_f16(qt, group=128):
    """fp32 weights of the fp16-narrowed tensor (what the GPU consumes)."""
    n, k = qt.rows, qt.cols
    p = qt.codes.reshape(n, -1)
    codes = np.empty((n, k), np.uint8)
    codes[:, 0::2] = p[:, : (k + 1) // 2] & 15
    codes[:, 1::2] = p[:, : k // 2] >> 4
    lut = qt.luts.reshape(n, 16).astype(np.float16).astype(np.float32)
    T = np.take_along_axis(lut, codes.astype(np.int64), axis=1)
    g = (k + group - 1) // group
    a = qt.alphas.reshape(n, g).astype(np.float16).astype(np.float32)
    b = qt.betas.reshape(n, g).astype(np.float16).astype(np.float32)
    a = np.repeat(a, group, axis=1)[:, :k]
    b = np.repeat(b, group, axis=1)[:, :k]
    return (a * T + b).astype(np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--paths", default="1,2")
    ap.add_argument("--ms", default="1,2,4")
    ap.add_argument("--shapes", default="q,k,gate,down")
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--chain", action="store_true", help="also time the 8B layer as one chain launch")
    ap.add_argument("--chain-paths", default="1", help="chain engines: 1 = GEMV (K1a), 5 = K1t")
    args = ap.parse_args()
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    out = {}
    for name in [s for s in args.shapes.split(",") if s]:
        n, k = SHAPES[name]
        qt = synthetic(n, k)
        w = dequant_f16(qt)
        wb = n * k // 2 + n * (k // 128) * 4 + n * 32
        ncopy = max(2, int(np.ceil(2 * 126e6 / wb)))
        dts = [anyq.DeviceTensor(qt) for _ in range(ncopy)]
        for m in (int(v) for v in args.ms.split(",")):
            x = torch.randn(m, k, device=dev).to(torch.bfloat16)
            xf = x.float().cpu().numpy().astype(np.float64)
            ref = xf @ w.astype(np.float64).T
            bound = np.abs(xf) @ np.abs(w.astype(np.float64)).T
            for path in (int(v) for v in args.paths.split(",")):
                if path == 1 and m > 4:
                    continue
                y = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
                y32 = torch.empty(m, n, device=dev, dtype=torch.float32)
                try:
                    dts[0].gemm(x, y, y32, path=path)
                    torch.cuda.synchronize()
                except Exception as e:  # noqa: BLE001
                    print(f"{name} m={m} path={path}: {e}")
                    continue
                err = np.abs(y32.cpu().numpy().astype(np.float64) - ref)
                rel = float((err / np.maximum(bound, 1e-30)).max())
                # determinism
                y32b = torch.empty_like(y32)
                dts[0].gemm(x, y, y32b, path=path)
                torch.cuda.synchronize()
                det = bool(torch.equal(y32, y32b))
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for d in dts:
                        d.gemm_ptr(x.data_ptr(), m, y.data_ptr(), None, stream.cuda_stream, path)
                reps = max(1, args.reps // ncopy)
                with torch.cuda.stream(stream):
                    for _ in range(3):
                        g.replay()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    for _ in range(reps):
                        g.replay()
                    e1.record(stream)
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / (reps * ncopy)
                nb = wb + m * k * 2 + m * n * 2
                gbs = nb / (us * 1e-6) / 1e9
                key = f"{name}_m{m}_p{path}"
                out[key] = {"us": round(us, 3), "GBps": round(gbs, 1), "pct": round(100 * gbs / peak, 1),
                            "max_rel_err": rel, "deterministic": det}
                print(key, out[key], flush=True)
        for d in dts:
            d.close()
    # the 8B decoder layer as ONE chain launch (q,k,v <- x; o <- y_q; gate,up <- y_o;
    # down <- y_up), weights rotated over enough layers to defeat L2
    if args.chain:
        layer = [("q", 4096, 4096), ("k", 1024, 4096), ("v", 1024, 4096), ("o", 4096, 4096),
                 ("gate", 14336, 4096), ("up", 14336, 4096), ("down", 4096, 14336)]
        nl = 4
        tens = [[anyq.DeviceTensor(synthetic(n, k, seed=10 * l + i)) for i, (_, n, k) in enumerate(layer)]
                for l in range(nl)]
        for m, cpath in ((int(v), int(c)) for v in args.ms.split(",") for c in args.chain_paths.split(",")):
            if m > (4 if cpath == 1 else 16):
                continue
            x = torch.randn(m, 4096, device=dev).to(torch.bfloat16)
            ys = [torch.empty(m, n, device=dev, dtype=torch.bfloat16) for _, n, _ in layer]
            xs = [x, x, x, ys[0], ys[3], ys[3], ys[5]]
            # natural order (q,k,v,o,gate,up,down) and the scheduled order of bench.py
            orders = {"": ([0, 1, 2, 3, 4, 5, 6], [-1, -1, -1, 0, 3, 3, 5]),
                      "_sched": ([0, 3, 1, 2, 5, 4, 6], [-1, 0, -1, -1, 1, 1, 4])}
            # extra orders to try: CHAIN_ORDERS="0,3,5,4,6,1,2;..." (indices of q,k,v,o,gate,up,down)
            x_src = [-1, -1, -1, 0, 3, 3, 5]
            for spec in filter(None, os.environ.get("CHAIN_ORDERS", "").split(";")):
                order = [int(v) for v in spec.split(",")]
                orders["_" + "".join(map(str, order))] = (
                    order, [-1 if x_src[j] < 0 else order.index(x_src[j]) for j in order])
            for tag, (order, deps) in orders.items():
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for l in range(nl):
                        anyq.gemm_chain([tens[l][j] for j in order], [xs[j] for j in order],
                                        [ys[j] for j in order], deps=deps, stream=stream, path=cpath)
                reps = 20
                with torch.cuda.stream(stream):
                    for _ in range(3):
                        g.replay()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    for _ in range(reps):
                        g.replay()
                    e1.record(stream)
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / (reps * nl)
                nb = sum(n * k // 2 + n * (k // 128) * 4 + n * 32 + m * k * 2 + m * n * 2 for _, n, k in layer)
                gbs = nb / (us * 1e-6) / 1e9
                key = f"layer_chain_m{m}_p{cpath}{tag}"
                out[key] = {"us": round(us, 3), "GBps": round(gbs, 1), "pct": round(100 * gbs / peak, 1)}
                print(key, out[key], flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/gemv_probe.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
