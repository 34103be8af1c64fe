#!/usr/bin/env python
"""Per-instruction stall attribution from an ncu --set full --import-source capture.

  ncu_hotloop.py <report.ncu-rep> [top_n]
Prints the total sample count by stall reason, the instructions with the most samples, and
the samples per opcode class -- the evidence for where a latency-bound loop waits.
"""
import csv
import subprocess
import sys
from collections import Counter, defaultdict


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    tot = Counter()
    per_op = defaultdict(Counter)
    scored = []
    for r in body:
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ex = int(r[ix["Instructions Executed"]] or 0)
        per_op[op]["samples"] += n
        per_op[op]["executed"] += ex
        for c in stall_cols:
            v = int(r[ix[c]] or 0)
            tot[c] += v
            per_op[op][c] += v
        scored.append((n, r[ix["Address"]][-5:], src, {c[6:]: int(r[ix[c]] or 0) for c in stall_cols if int(r[ix[c]] or 0)}))
    S = sum(tot.values())
    print(f"total samples {S}")
    for c, v in tot.most_common():
        if v:
            print(f"  {c:22s} {v:8d} {100.0 * v / S:5.1f}%")
    print("\nby opcode (samples, executed warp-instructions, top stalls):")
    for op, d in sorted(per_op.items(), key=lambda kv: -kv[1]["samples"])[:16]:
        st = sorted(((v, c[6:]) for c, v in d.items() if c.startswith("stall_")), reverse=True)[:3]
        print(f"  {op:10s} {d['samples']:8d} {d['executed']:12d}  " + ", ".join(f"{c} {v}" for v, c in st))
    print(f"\ntop {top} instructions:")
    for n, a, src, st in sorted(scored, key=lambda x: -x[0])[:top]:
        print(f"  {n:6d} {a} {src[:60]:60s} {dict(sorted(st.items(), key=lambda kv: -kv[1])[:3])}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
