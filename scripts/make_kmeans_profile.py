"""Write profiles/ncu_kmeans.json from the k-means ncu capture (gpurun_out/km_warp.ncu-rep,
made by scripts/gpu_kmeans_ncu.sh): key metrics, stall reasons per issue and the hottest
source lines (usage: python scripts/make_kmeans_profile.py)."""
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REP = os.path.join(ROOT, "gpurun_out", "km_warp.ncu-rep")
KEEP = ["gpu__time_duration.sum", "launch__block_size", "launch__grid_size", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed.avg.per_cycle_active", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct"]
STALLS = "smsp__average_warps_issue_stalled_"


def ncu(*args):
    return subprocess.run(["ncu", "-i", REP, *args], capture_output=True, text=True).stdout


def main():
    rows = list(csv.reader(ncu("--page", "raw", "--csv").splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    metrics = {k: {"value": x, "unit": un} for k, un, x in zip(h, u, v) if k in KEEP}
    stalls = {k[len(STALLS):].replace("_per_issue_active.ratio", ""): round(float(x), 3)
              for k, x in zip(h, v) if k.startswith(STALLS) and k.endswith("per_issue_active.ratio")
              and float(x) > 0.005}
    # the source page holds one section per function (kernel + called subroutines)
    hot, allrows = [], []
    sec, hdr = "", None
    for r in csv.reader(ncu("--page", "source", "--csv").splitlines()):
        if r and r[0] == "Kernel Name":
            sec, hdr = r[1], None
        elif hdr is None:
            hdr = r
        else:
            allrows.append((sec, dict(zip(hdr, r))))
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(float(d.get(key) or 0) for _, d in allrows) or 1.0
    for sec, d in sorted(allrows, key=lambda x: -float(x[1].get(key) or 0))[:14]:
        hot.append({"function": sec[:60], "sass": d["Source"].strip()[:80],
                    "share": round(float(d.get(key) or 0) / tot, 4)})
    out = {"kernel": "k_kmeans_warp (G=4 warps per row, 4096x4096 any4 g128, scripts/prof_kmeans.py)",
           "capture": "ncu --set full --import-source on --clock-control none -k regex:k_kmeans_warp -c 1",
           "metrics": metrics, "stalls_per_issue": stalls, "hot_source_lines": hot}
    with open(os.path.join(ROOT, "profiles", "ncu_kmeans.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("stalls_per_issue",)}, indent=0)[:800])
    for x in hot:
        print(x)


if __name__ == "__main__":
    main()
