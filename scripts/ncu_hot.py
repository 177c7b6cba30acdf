"""Summarise an ncu report's source page: stall samples per opcode and the top
instructions (usage: python scripts/ncu_hot.py REPORT.ncu-rep [kernel-substring])."""
import csv
import subprocess
import sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    ksub = sys.argv[2] if len(sys.argv) > 2 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, hdr = None, None
    by_op = defaultdict(lambda: [0, 0])
    insts = []
    reasons = defaultdict(int)
    for r in rows:
        if len(r) >= 2 and r[0] == "Kernel Name":
            cur = r[1]
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr) or (ksub and ksub not in (cur or "")):
            continue
        d = dict(zip(hdr, r))
        try:
            s = int(d["Warp Stall Sampling (All Samples)"])
            ex = int(d["Instructions Executed"] or 0)
        except ValueError:
            continue
        op = d["Source"].split()[0] if d["Source"].split() else "?"
        if op.startswith("@"):
            op = d["Source"].split()[1]
        op = op.split(".")[0]
        by_op[op][0] += s
        by_op[op][1] += ex
        insts.append((s, d["Address"], d["Source"][:60]))
        for k, v in d.items():
            if k.startswith("stall_") or "Stall" in k and "Sampling" not in k:
                try:
                    reasons[k] += int(v)
                except ValueError:
                    pass
    tot = sum(v[0] for v in by_op.values()) or 1
    print(f"total stall samples {tot}")
    for op, (s, ex) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:20]:
        print(f"  {op:10s} samples {s:6d} ({100*s/tot:5.1f}%)  executed {ex}")
    print("top instructions:")
    for s, a, src in sorted(insts, reverse=True)[:25]:
        print(f"  {s:6d}  {src}")


if __name__ == "__main__":
    main()
