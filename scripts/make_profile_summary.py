"""Write profiles/ncu_summary.json (+ the launch-list share table) from the
round's ncu captures in gpurun_out/ (usage: python scripts/make_profile_summary.py)."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
KEEP = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "launch__block_size", "launch__grid_size", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.avg.per_cycle_active", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__shared_mem_per_block_dynamic"]
STALLS = "smsp__average_warps_issue_stalled_"


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    rep = os.path.join(OUT, sys.argv[1] if len(sys.argv) > 1 else "chain_full.ncu-rep")
    h, u, vals = raw(rep)
    v = vals[0]
    m = {k: {"value": x, "unit": un} for k, un, x in zip(h, u, v) if k in KEEP}
    stalls = {k[len(STALLS):].replace("_per_issue_active.ratio", ""): round(float(x), 3)
              for k, x in zip(h, v) if k.startswith(STALLS) and k.endswith("per_issue_active.ratio")
              and x not in ("", "0")}
    rd = to_bytes(m["dram__bytes_read.sum"]["value"], m["dram__bytes_read.sum"]["unit"])
    wr = to_bytes(m["dram__bytes_write.sum"]["value"], m["dram__bytes_write.sum"]["unit"])
    # launch list of the bench (per-launch times are cold-cache and serialised)
    share = {}
    lf = os.path.join(OUT, "launches_bench.csv")
    if os.path.exists(lf):
        hdr = None
        tot = 0.0
        for r in csv.reader(open(lf)):
            if "Kernel Name" in r:
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                name = d["Kernel Name"].split("(")[0].split("::")[-1]
                t = float(d["Metric Value"])
                share[name] = share.get(name, 0.0) + t
                tot += t
        share = {k: {"ns": round(t, 0), "share": round(t / tot, 4)} for k, t in
                 sorted(share.items(), key=lambda kv: -kv[1])}
    summary = {
        "round": 2,
        "kernel": "k_lutgemv<1> chain (one Llama-3-8B decoder layer, 7 GEMMs, M=1): 16 compute + writer + producer + builder + dependency warps",
        "capture": f"ncu --set full --clock-control none (cold L2, serialised) of scripts/prof_chain.py -> {os.path.basename(rep)}",
        "dram_bytes_per_launch_layer_chain": rd + wr,
        "algorithmic_bytes_per_launch": 117383168,
        "metrics": m,
        "stalls_per_issue": stalls,
        "bench_launch_list_share": share,
    }
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: summary[k] for k in ("dram_bytes_per_launch_layer_chain",)}), len(share))


if __name__ == "__main__":
    main()
