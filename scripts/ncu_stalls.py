"""Per-instruction stall attribution from an ncu report's source page.
usage: python scripts/ncu_stalls.py REPORT.ncu-rep [top]"""
import csv
import subprocess
import sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = None
    recs = []
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        recs.append(dict(zip(hdr, r)))
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = defaultdict(int)
    by_op = defaultdict(lambda: defaultdict(int))
    per = []
    for d in recs:
        src = d["Source"].split()
        op = (src[1] if src and src[0].startswith("@") else (src[0] if src else "?"))
        for k in reasons:
            try:
                v = int(d[k])
            except ValueError:
                v = 0
            tot[k] += v
            by_op[op][k] += v
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        per.append((s, d["Address"][-5:], d["Source"].strip()[:70],
                    {k[6:]: int(d[k]) for k in reasons if d[k] not in ("", "0")}))
    T = sum(tot.values()) or 1
    print("stall totals:", {k[6:]: round(100 * v / T, 1) for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v})
    print("by opcode (top reasons):")
    for op, dd in sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:15]:
        s = sum(dd.values())
        print(f"  {op:28s} {100*s/T:5.1f}%  " + ", ".join(f"{k[6:]}={100*v/T:.1f}" for k, v in sorted(dd.items(), key=lambda kv: -kv[1])[:4] if v))
    print("top instructions:")
    for s, a, src, dd in sorted(per, key=lambda t: -t[0])[:top]:
        print(f"  {100*s/T:5.2f}% {a} {src:70s} {dict(sorted(dd.items(), key=lambda kv: -kv[1])[:3])}")


if __name__ == "__main__":
    main()
