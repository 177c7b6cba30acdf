"""profiles/roundN.md from the round's bench line, the reference arm and
profiles/ncu_summary.json.

usage: python scripts/make_round_report.py [N [bench.log [bench_ref.log]]]
(defaults: 1, gpurun_out/bench.log, gpurun_out/bench_ref.log)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def last_json(path):
    out = None
    if os.path.exists(path):
        for line in open(path):
            if line.startswith("{"):
                out = json.loads(line)
    return out


def main():
    rnd = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    b = last_json(sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "bench.log"))
    r = last_json(sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", "bench_ref.log"))
    n = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
    L = [f"# Round {rnd} — measured on one B200 (sm_100a, 148 SMs)", ""]
    L += ["Source: `python bench.py` (defaults: N=1, 500 steps, 5 warm-up, CUDA graphs, weights rotated "
          "over 4 layers > L2) and `python bench.py --impl reference`; ncu: "
          "`ncu --set full --clock-control none` of `scripts/prof_chain.py` (cold L2, serialised).", ""]
    L += ["## Headline (decoder-layer chain, M=1)", "", "| key | value |", "|---|---|"]
    L += [f"| value | {b['value']} {b['unit']} ({b['ms_per_step'] * 1e3:.1f} µs per layer) |",
          f"| roofline frac | {b['roofline']['frac']} of {b['roofline']['peak']} GB/s ({b['roofline']['peak_kind']}) |",
          f"| e2e (public API, H2D x + D2H y) | {b['e2e']['value']} {b['e2e']['unit']} |",
          f"| DRAM traffic per launch (ncu) | {b['roofline']['traffic']:.0f} B (algorithmic 117383168 B) |",
          f"| cpu_baseline (1 core, reference gemm_fused) | {b['cpu_baseline']['value']:.4f} GB/s |",
          f"| reference arm (all host threads) | {r['value'] if r else 'n/a'} GB/s, cores {r['cpu_baseline']['cores'] if r else 'n/a'} |",
          f"| clocks | {b['clocks']} |", ""]
    L += ["## Per-GEMM (M=1, single launches, AUTO path)", "", "| shape | N | K | µs | GB/s | % HBM |",
          "|---|---|---|---|---|---|"]
    for k, v in b["per_shape"].items():
        L.append(f"| {k} | {v['N']} | {v['K']} | {v['us']} | {v['GBps']} | {v['pct_hbm_peak']} |")
    if b.get("per_shape_70b_m1"):
        L += ["", "## Llama-3-70B shapes (config 3 slice at P=1), M=1", "", "| shape | N | K | µs | GB/s | % HBM |",
              "|---|---|---|---|---|---|"]
        for k, v in b["per_shape_70b_m1"].items():
            L.append(f"| {k} | {v['N']} | {v['K']} | {v['us']} | {v['GBps']} | {v['pct_hbm_peak']} |")
    L += ["", "## M sweep (AUTO path)", "", "| shape, M | µs | % HBM | TFLOP/s | path |",
          "|---|---|---|---|---|"]
    for k, v in b.get("m_sweep", {}).items():
        L.append(f"| {k} | {v['us']} | {v['pct_hbm_peak']} | {v['TFLOPs']} | {v['path']} |")
    km = b.get("kmeans")
    if km:
        L += ["", "## k-means quantizer", "", f"{km['rows_per_s']} rows/s on {km['matrix']} "
              f"({km['seconds']} s, median of 3, device-resident)."]
    L += ["", "## ncu — k_lutgemv chain", "", "| metric | value |", "|---|---|"]
    for k, v in n["metrics"].items():
        L.append(f"| {k} | {v['value']} {v['unit']} |")
    L += ["", "Stalls per issued instruction: " +
          ", ".join(f"{k} {v}" for k, v in sorted(n["stalls_per_issue"].items(), key=lambda kv: -kv[1])[:8])]
    kmp = os.path.join(ROOT, "profiles", "ncu_kmeans.json")
    if os.path.exists(kmp):  # scripts/make_kmeans_profile.py
        kn = json.load(open(kmp))
        L += ["", "## ncu — k_kmeans_warp (4096x4096, G = 4 warps per row)", "", "| metric | value |", "|---|---|"]
        for k, v in kn["metrics"].items():
            L.append(f"| {k} | {v['value']} {v['unit']} |")
        L += ["", "Stalls per issued instruction: " +
              ", ".join(f"{k} {v}" for k, v in sorted(kn["stalls_per_issue"].items(), key=lambda kv: -kv[1])[:8])]
    with open(os.path.join(ROOT, "profiles", f"round{rnd}.md"), "w") as f:
        f.write("\n".join(L) + "\n")


if __name__ == "__main__":
    main()
