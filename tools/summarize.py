"""Summarise a gpurun_out/ capture into profiles/<tag>/ (tracked):
bench JSON lines, the ncu launch list aggregated per kernel (share of step),
the --set full details page and the per-source-line hot spots of the top kernel.

    python tools/summarize.py <tag> [ncu-rep-name]
"""
import csv
import glob
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    if not rows:
        return
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        d[r[ki]][0] += 1
        d[r[ki]][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in d.values()) or 1.0
    with open(out, "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
        f.write("kernel,launches,total_ms,mean_ms,share\n")
        for k, (n, ns) in sorted(d.items(), key=lambda kv: -kv[1][1]):
            f.write(f"\"{k}\",{n},{ns/1e6:.4f},{ns/1e6/n:.4f},{ns/tot:.4f}\n")


def details(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if not rows:
        return
    h = rows[0]
    ki = h.index("Kernel Name")
    si, mi, vi, ui = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Value", "Metric Unit"))
    with open(out, "w") as f:
        for r in rows[1:]:
            if r[mi]:
                f.write(f"{r[ki][:40]} | {r[si]} | {r[mi]} | {r[vi]} {r[ui]}\n")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if rows:
        h = rows[0]
        want = [i for i, n in enumerate(h) if n in (
            "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "Kernel Name")]
        with open(out, "a") as f:
            f.write("\n# raw\n")
            for r in rows:
                f.write(",".join(r[i] for i in want) + "\n")


def main():
    tag = sys.argv[1]
    rep = sys.argv[2] if len(sys.argv) > 2 else None
    od = os.path.join(ROOT, "profiles", tag)
    os.makedirs(od, exist_ok=True)
    with open(os.path.join(od, "bench.jsonl"), "w") as f:
        for p in sorted(glob.glob(os.path.join(G, "bench*.log"))):
            for line in open(p):
                if line.startswith("{"):
                    f.write(line)
    lc = os.path.join(G, "launches.csv")
    if os.path.exists(lc):
        launches(lc, os.path.join(od, "launches_summary.csv"))
    if rep:
        rp = os.path.join(G, rep + ".ncu-rep")
        details(rp, os.path.join(od, rep + "_details.txt"))
        src = subprocess.run(["ncu", "-i", rp, "--page", "source", "--csv", "--print-source",
                              "cuda,sass"], capture_output=True, text=True).stdout
        tmp = "/tmp/_src.csv"
        open(tmp, "w").write(src)
        hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), tmp, "40"],
                             capture_output=True, text=True).stdout
        open(os.path.join(od, rep + "_hotlines.txt"), "w").write(hot)
    print("wrote", od)


if __name__ == "__main__":
    main()
