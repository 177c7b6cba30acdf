"""The reference's bench table (qgemm.cpp:154-218, schema qgemm.hpp:59:
shape,format,layout,median_ns,p10_ns,p90_ns,bytes_per_weight) with the B200
rows next to the reference's CPU rows, on the same shapes and formats.

layouts: dense / rowmajor   the reference build (oracle/_ref), host CPU, 1 thread
         b200-dense         fp32 gemm_dense on the GPU (kind 0)
         b200-exact         the bit-exact gemm_fused kernel on the GPU (kind 1)
         b200               the A16W4 LUT GEMM (bf16 x, the AUTO kernel for m; kind 2)
GPU times are device times of the library's own timing loop (anyq_bench_gemm).

usage: python scripts/bench_csv.py [out.csv] [--repeats R]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.refpy import have_ref, ref  # noqa: E402
from paper_2507_04610_b200 import _abi, anyq  # noqa: E402

SHAPES = [(1, 4096, 4096), (1, 14336, 4096), (16, 4096, 4096)]
FORMATS = ["int4", "nf4", "any4"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out", nargs="?", default="gpurun_out/bench_rows.csv")
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    rows = []
    if have_ref() and not args.no_cpu:
        rows += ref().bench(SHAPES, FORMATS, args.repeats, 1)
    rng = np.random.default_rng(1)
    for (m, n, k) in SHAPES:
        w = rng.standard_normal((n, k), dtype=np.float32)
        x = rng.standard_normal((m, k), dtype=np.float32)
        ns = anyq.bench_gemm(0, None, w, x, max(args.repeats, 10))
        rows.append(((m, n, k), "fp32", "b200-dense", *np.quantile(ns, [0.5, 0.1, 0.9]), 4.0))
        for fmt in FORMATS:
            c = _abi.default_config(group_size=min(128, k), seed=1)
            anyq.apply_format(c, fmt)
            qt = anyq.quantize_any(w, c) if c.codebook == _abi.CB_ANY else anyq.quantize_fixed(w, c)
            bpw = anyq.storage_bits_per_entry(c, n, k) / 8.0
            for kind, layout in ((1, "b200-exact"), (2, "b200")):
                ns = anyq.bench_gemm(kind, qt, None, x, max(args.repeats, 10))
                rows.append(((m, n, k), fmt, layout, *np.quantile(ns, [0.5, 0.1, 0.9]), bpw))
    lines = ["shape,format,layout,median_ns,p10_ns,p90_ns,bytes_per_weight"]
    for (m, n, k), fmt, layout, med, p10, p90, bpw in rows:
        lines.append(f"{m}x{n}x{k},{fmt},{layout},{int(med)},{int(p10)},{int(p90)},{bpw:g}")
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    with open(args.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
