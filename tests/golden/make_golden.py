"""Generates the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run here (where /root/reference exists and oracle/_ref/libanyq_ref.so was built
by `make -C oracle ref`):

    python tests/golden/make_golden.py

Outputs (committed; read by tests/test_oracle.py on CPU and by the GPU parity
tests on the B200 box, where /root/reference does not exist):

  golden.json   config-1 fingerprints (sha256 of the raw little-endian bytes)
                and spot values, fp16/bf16 known answers, bits-per-weight
  cases.npz     small quantize / GEMM / k-means cases: inputs are regenerated
                from the reference's own generators (tests/helpers.hpp) by seed,
                outputs are the reference's results

Every output below comes from oracle.refpy.ref() (proj/src compiled in place);
nothing here is computed by the repo's own code.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.refpy import have_ref, ref  # noqa: E402
from paper_2507_04610_b200 import _abi  # noqa: E402

FORMATS = {"int4": (0, 4), "fp4": (1, 4), "nf4": (2, 4), "any4": (3, 4), "any3": (3, 3),
           "any2": (3, 2), "int8": (0, 8), "int3": (0, 3)}

# (name, rows, cols, fmt, granularity, group, symmetric, stats, seed)
QUANT_CASES = [
    ("any4_g8", 24, 56, "any4", 3, 8, 0, False, 5),
    ("any4_g16_stats", 24, 64, "any4", 3, 16, 0, True, 6),
    ("any4_row", 9, 40, "any4", 1, 0, 0, False, 7),
    ("any4_sym", 12, 48, "any4", 3, 16, 1, False, 8),
    ("any4_ragged", 7, 33, "any4", 3, 8, 0, True, 9),
    ("any3_g8", 16, 40, "any3", 3, 8, 0, False, 10),
    ("any2_g8", 16, 40, "any2", 3, 8, 0, True, 11),
    ("int4_g8", 24, 56, "int4", 3, 8, 0, False, 12),
    ("int4_sym", 24, 56, "int4", 3, 8, 1, False, 13),
    ("nf4_g16", 20, 64, "nf4", 3, 16, 0, False, 14),
    ("fp4_g16", 20, 64, "fp4", 3, 16, 0, False, 15),
    ("int8_row", 10, 30, "int8", 1, 0, 0, False, 16),
    ("int3_g8", 10, 30, "int3", 3, 8, 0, False, 17),
    ("any4_k128", 64, 256, "any4", 3, 128, 0, True, 18),
]
GEMM_MS = (1, 5, 16)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_cfg(fmt, gran, group, sym, seed):
    cb, bits = FORMATS[fmt]
    c = _abi.default_config(codebook=cb, bits=bits, granularity=gran, symmetric=sym, seed=seed)
    if gran == 3:
        c.group_size = group
    return c


def main():
    if not have_ref():
        raise SystemExit("oracle/_ref/libanyq_ref.so missing: run `make -C oracle ref` first")
    R = ref()
    out = {"source": "oracle/_ref (reference proj/src compiled in place), tests/golden/make_golden.py"}

    # ---- config 1: W = gaussian(4096,4096,1), any4 g128 seed 0
    w = R.gaussian(4096, 4096, 1)
    cfg = _abi.default_config(codebook=_abi.CB_ANY)
    c1 = {}
    for tag, exj in (("nostats", None), ("stats", R.synthetic_stats(4096, 3))):
        qt = R.quantize(w, cfg, exj, threads=os.cpu_count() or 1)
        bpr = qt.codes.size // 4096
        d = {
            "codes": sha(qt.codes), "luts": sha(qt.luts), "alphas": sha(qt.alphas),
            "betas": sha(qt.betas),
            "codes_rows256": sha(qt.codes[: 256 * bpr]), "luts_rows256": sha(qt.luts[: 256 * 16]),
            "alphas_rows256": sha(qt.alphas[: 256 * 32]), "betas_rows256": sha(qt.betas[: 256 * 32]),
        }
        if tag == "nostats":
            x = R.gaussian(1, 4096, 2)
            y = R.gemm_fused(x, qt)
            d.update({
                "row0_lut": [float(v) for v in qt.luts[:16]],
                "row0_code_bytes": qt.codes[:8].tobytes().hex(),
                "alpha0": float(qt.alphas[0]), "beta0": float(qt.betas[0]),
                "y_first3": [float(v) for v in y[0, :3]], "y": sha(y),
            })
        c1[tag] = d
    out["config1"] = c1

    # ---- fp16 / bf16 known answers (pack.cpp:61-128), incl. subnormal/tie/overflow
    vals = [0.0, -0.0, 1.0, -2.5, 65504.0, 65519.0, 6.1035156e-05, 5.9604645e-08, 2.9802322e-08,
            1.0009765625, 1.00048828125, 0.1, 3.14159265, 1e-9, 123456.0]
    kat16, katb = [], []
    for v in vals:
        try:
            kat16.append([v, R.f32_to_f16(v)])
        except Exception as e:  # noqa: BLE001  (overflow -> IoError)
            kat16.append([v, str(type(e).__name__) + ":" + e.kind])
        katb.append([v, R.f32_to_bf16(v)])
    out["f16_kat"] = kat16
    out["bf16_kat"] = katb

    # ---- bits per weight (codebooks.cpp:99-121)
    bits = {}
    for fmt in ("any4", "int4", "nf4"):
        c = make_cfg(fmt, 3, 128, 0, 0)
        bits[fmt] = R.storage_bits_per_entry(c, 4096, 4096)
    out["bits_per_weight_4096"] = bits

    # ---- small cases
    arrays = {}
    meta = []
    for (name, n, k, fmt, gran, group, sym, stats, seed) in QUANT_CASES:
        c = make_cfg(fmt, gran, group, sym, seed)
        wq = R.gaussian(n, k, 100 + seed)
        exj = R.synthetic_stats(k, 200 + seed) if stats else None
        qt = R.quantize(wq, c, exj, threads=1)
        arrays[f"{name}.codes"] = qt.codes
        arrays[f"{name}.alphas"] = qt.alphas
        arrays[f"{name}.betas"] = qt.betas
        if qt.luts is not None:
            arrays[f"{name}.luts"] = qt.luts
        nq = R.narrowed(qt)
        arrays[f"{name}.narrowed_alphas"] = nq.alphas
        arrays[f"{name}.narrowed_betas"] = nq.betas
        if nq.luts is not None:
            arrays[f"{name}.narrowed_luts"] = nq.luts
        arrays[f"{name}.dequant"] = R.dequantize(qt)
        for m in GEMM_MS:
            x = R.gaussian(m, k, 300 + seed + m)
            arrays[f"{name}.y_fused_m{m}"] = R.gemm_fused(x, qt)
            arrays[f"{name}.y_ref_m{m}"] = R.gemm_reference(x, qt)
        meta.append({"name": name, "rows": n, "cols": k, "fmt": fmt, "granularity": gran,
                     "group_size": group, "symmetric": sym, "stats": stats, "seed": seed,
                     "w_seed": 100 + seed, "stats_seed": 200 + seed,
                     "x_seed": {str(m): 300 + seed + m for m in GEMM_MS}})
    out["quant_cases"] = meta

    # ---- k-means pieces on one row (learner.cpp:132-341)
    km = []
    for i, (n, k, seed) in enumerate(((64, 4, 3), (200, 16, 4), (33, 8, 5))):
        xs = R.gaussian(1, n, 400 + i)[0] * 3 + 7
        ws = np.abs(R.gaussian(1, n, 500 + i)[0]) + 0.1
        c = _abi.default_config(codebook=_abi.CB_ANY)
        init = R.kmeans_pp_init(xs, ws, k, seed, i)
        cen, asg, loss, iters = R.weighted_kmeans(xs, ws, k, c, seed, i)
        arrays[f"km{i}.x"] = xs
        arrays[f"km{i}.w"] = ws
        arrays[f"km{i}.init"] = init
        arrays[f"km{i}.centroids"] = cen
        arrays[f"km{i}.assign"] = asg
        km.append({"n": n, "k": k, "seed": seed, "row": i, "loss": loss, "iters": iters})
    out["kmeans_cases"] = km

    # ---- RNG stream (core.hpp:154-200)
    arrays["rng_u64_seed7_row3"] = R.rng_u64(7, 3, 16)
    arrays["rng_double_seed7_row3"] = R.rng_double(7, 3, 16)

    np.savez_compressed(os.path.join(HERE, "cases.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {len(arrays)} arrays and golden.json")


if __name__ == "__main__":
    main()
