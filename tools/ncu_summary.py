#!/usr/bin/env python
"""Summarise Nsight Compute output into profiles/ (committed evidence).

  ncu_summary.py launches <launches.csv> <out.md> [--dram-json profiles/ncu_dram.json --key c5_mixed_k3]
      <launches.csv> is the --csv --log-file output of
      `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none`
      (one row per kernel launch and metric).  Writes a per-launch table, each kernel family's
      share of the summed device time, and (optionally) the DRAM bytes per launch of every
      sweep dim into the JSON that bench.py reads for roofline.traffic.
  ncu_summary.py full <report.ncu-rep> <out.md>
      Key metrics of a `--set full` capture (throughput, DRAM bytes, issue/stall breakdown).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict, defaultdict


def short(name):
    n = name.split("(")[0]
    return n.replace("void ", "").replace("sldg::", "")


def launches(path, out, dram_json=None, key=None, pipe_json=None):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: i for i, h in enumerate(hdr)}
    per = OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        lid = int(r[ix["ID"]])
        d = per.setdefault(lid, {"name": r[ix["Kernel Name"]], "grid": r[ix["Grid Size"]], "block": r[ix["Block Size"]]})
        unit, val = r[ix["Metric Unit"]], float(r[ix["Metric Value"]].replace(",", ""))
        m = r[ix["Metric Name"]]
        if m == "gpu__time_duration.sum":
            d["ms"] = val * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        elif m.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d["read" if "read" in m else "write"] = val * scale
        elif m == "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active":
            d["fp64"] = val
        elif m == "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active":
            d["xu"] = val
    tot = sum(d.get("ms", 0) for d in per.values())
    fam = defaultdict(float)
    for d in per.values():
        fam[short(d["name"])] += d.get("ms", 0)
    lines = [f"# ncu launch list: `{os.path.basename(path)}`", "",
             "Cold-cache, serialised per-launch device times under ncu (compare SHARES, not absolutes).", "",
             "| # | kernel | grid x block | ms | DRAM read GB | DRAM write GB | GB/s (DRAM, under ncu) |",
             "|---|---|---|---|---|---|---|"]
    for lid, d in per.items():
        ms = d.get("ms", 0)
        rd, wr = d.get("read", 0) / 1e9, d.get("write", 0) / 1e9
        gbs = (rd + wr) / (ms * 1e-3) if ms else 0
        lines.append(f"| {lid} | {short(d['name'])} | {d['grid']} x {d['block']} | {ms:.3f} | {rd:.3f} | {wr:.3f} | {gbs:.0f} |")
    lines += ["", "| kernel family | total ms | share |", "|---|---|---|"]
    for f, ms in sorted(fam.items(), key=lambda x: -x[1]):
        lines.append(f"| {f} | {ms:.3f} | {ms / tot:.1%} |")
    open(out, "w").write("\n".join(lines) + "\n")
    if dram_json and key:
        db = json.load(open(dram_json)) if os.path.exists(dram_json) else {}
        sweeps = [d for d in per.values() if "sweep" in d["name"]]
        # sweeps are launched in dim order within each split step; take the first timed step
        # (after bench.py's default 3 warm-up steps), not the e2e / precision-comparison runs
        ndim = int(key.split("_D")[-1]) if "_D" in key else 4
        base = key.split("_D")[0]
        # a step is ndim sweep launches in dim order, or with the fused x pair (bench default)
        # sweep_fused01_kernel then dims 2 .. ndim-1
        fused = any("fused01" in d["name"] for d in sweeps)
        per_step = ndim - 1 if fused else ndim
        names = (["fused01"] + [f"dim{e}" for e in range(2, ndim)]) if fused else [f"dim{e}" for e in range(ndim)]
        first = sweeps[3 * per_step:4 * per_step]
        for nm, d in zip(names, first):
            db[f"{base}_{nm}"] = d.get("read", 0) + d.get("write", 0)
        json.dump(db, open(dram_json, "w"), indent=1, sort_keys=True)
        if pipe_json:  # secondary roofline: fp64-pipe and XU activity per sweep
            pb = json.load(open(pipe_json)) if os.path.exists(pipe_json) else {}
            for nm, d in zip(names, first):
                if "fp64" in d:
                    pb[f"{base}_{nm}"] = {"fp64_pipe_pct": d["fp64"], "xu_pct": d.get("xu")}
            json.dump(pb, open(pipe_json, "w"), indent=1, sort_keys=True)
    print(out)


def full(rep, out):
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    want = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
            ("dram__bytes_write.sum", "DRAM write"),
            ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
            ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
            ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
            ("launch__registers_per_thread", "registers/thread"),
            ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
            ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe % (F2F)"),
            ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
            ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
            ("lts__t_sector_hit_rate.pct", "L2 hit %")]
    stalls = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in h]
    lines = [f"# ncu --set full: `{os.path.basename(rep)}`", ""]
    for r in rows[2:]:
        lines.append(f"## {short(r[hdr.index('Kernel Name')])}  grid {r[hdr.index('Grid Size')]} x {r[hdr.index('Block Size')]}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for m, lab in want:
            if m in hdr:
                lines.append(f"| {lab} (`{m}`) | {r[hdr.index(m)]} | {rows[1][hdr.index(m)]} |")
        tot = sum(float(r[hdr.index(s)] or 0) for s in stalls)
        top = sorted(((float(r[hdr.index(s)] or 0), s) for s in stalls), reverse=True)[:6]
        lines.append("")
        lines.append("Warp-state samples (top): " + ", ".join(
            f"{s.replace('smsp__pcsamp_warps_issue_stalled_', '')} {v / tot:.0%}" for v, s in top if tot))
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        dj = sys.argv[sys.argv.index("--dram-json") + 1] if "--dram-json" in sys.argv else None
        key = sys.argv[sys.argv.index("--key") + 1] if "--key" in sys.argv else None
        pj = sys.argv[sys.argv.index("--pipe-json") + 1] if "--pipe-json" in sys.argv else None
        launches(sys.argv[2], sys.argv[3], dj, key, pj)
    else:
        full(sys.argv[2], sys.argv[3])
