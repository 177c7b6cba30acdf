"""One ncu report -> a compact JSON summary for profiles/ (key metrics, stall
reasons per issue, the hottest SASS lines).
usage: python scripts/ncu_summarize.py REPORT.ncu-rep OUT.json "kernel description" [algorithmic_bytes]"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

KEEP = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__block_size",
        "launch__grid_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.avg.per_cycle_active", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
STALLS = "smsp__average_warps_issue_stalled_"


def to_bytes(v, unit):
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    rep, out, desc = sys.argv[1], sys.argv[2], sys.argv[3]
    algo = float(sys.argv[4]) if len(sys.argv) > 4 else None
    rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                          text=True).stdout.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    m = {k: {"value": x, "unit": un} for k, un, x in zip(h, u, v) if k in KEEP}
    stalls = {k[len(STALLS):].replace("_per_issue_active.ratio", ""): round(float(x), 3)
              for k, x in zip(h, v) if k.startswith(STALLS) and k.endswith("per_issue_active.ratio")
              and x not in ("", "0")}
    src = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                         capture_output=True, text=True).stdout.splitlines()))
    hdr, hot, tot = None, [], 0
    for r in src:
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            try:
                sm = int(d["Warp Stall Sampling (All Samples)"] or 0)
            except ValueError:
                continue
            tot += sm
            hot.append((sm, d["Source"].strip()[:80]))
    hot.sort(reverse=True)
    rd = to_bytes(m["dram__bytes_read.sum"]["value"], m["dram__bytes_read.sum"]["unit"])
    wr = to_bytes(m["dram__bytes_write.sum"]["value"], m["dram__bytes_write.sum"]["unit"])
    summary = {"kernel": desc, "capture": f"ncu --set full --clock-control none --import-source on ({rep.split('/')[-1]})",
               "dram_bytes_per_launch": rd + wr, "algorithmic_bytes_per_launch": algo, "metrics": m,
               "stalls_per_issue": stalls,
               "hot_sass": [{"share": round(s / max(tot, 1), 4), "sass": t} for s, t in hot[:12]]}
    json.dump(summary, open(out, "w"), indent=1)
    print(out, rd + wr, m.get("gpu__time_duration.sum"))


if __name__ == "__main__":
    main()
