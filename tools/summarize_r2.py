"""Summarise the round-2 evidence pass (tools/gpurun_r2_final.sh; its ncu
reports were exported to CSV on the box) into profiles/r2_final/ (tracked):
bench JSON lines, the headline step's launch list per kernel (share of step),
per-capture details + selected raw metrics + per-source-line hot spots, the
sweep, the microbenchmarks and the GPU test tail; then refresh
profiles/traffic.json (dram bytes and warp instructions per launch of each
workload's dominant kernel, read by bench.py)."""
import csv
import glob
import gzip
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
OD = os.path.join(ROOT, "profiles", "r2_final")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from summarize import launches  # noqa: E402

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "smsp__inst_executed.sum",
       "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread")


def main():
    os.makedirs(OD, exist_ok=True)
    with open(os.path.join(OD, "bench.jsonl"), "w") as f:
        for name in ("r2_bench_default.jsonl", "r2_bench_all.jsonl", "r2_bench_reference.jsonl"):
            p = os.path.join(G, name)
            if os.path.exists(p):
                for line in open(p):
                    if line.startswith("{"):
                        f.write(line)
    lc = os.path.join(G, "r2_launches.csv")
    if os.path.exists(lc):
        launches(lc, os.path.join(OD, "launches_summary.csv"))
    traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    import bench
    for det in sorted(glob.glob(os.path.join(G, "r2_full_*_details.csv"))):
        tag = os.path.basename(det)[len("r2_full_"):-len("_details.csv")]
        rows = list(csv.reader(open(det)))
        if not rows:
            continue
        h = rows[0]
        ki = h.index("Kernel Name")
        si, mi, vi, ui = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Value", "Metric Unit"))
        with open(os.path.join(OD, f"full_{tag}_details.txt"), "w") as f:
            for r in rows[1:]:
                if len(r) > ui and r[mi]:
                    f.write(f"{r[ki][:40]} | {r[si]} | {r[mi]} | {r[vi]} {r[ui]}\n")
            raw = list(csv.reader(open(os.path.join(G, f"r2_full_{tag}_raw.csv"))))
            if raw:
                rh, ru, rv = raw[0], raw[1], raw[2]
                f.write("\n# raw\n")
                vals = {}
                for name in RAW:
                    if name in rh:
                        i = rh.index(name)
                        f.write(f"{name},{ru[i]},{rv[i]}\n")
                        vals[name] = (rv[i], ru[i])
                # dominant kernels' traffic / instructions for bench.py
                wl = tag.split("_k_")[0]
                try:
                    name = bench._workload(wl, 1)["name"]
                except SystemExit:
                    name = None
                if name and "dram__bytes_read.sum" in vals and "_k_split" not in tag:
                    tot = sum(float(vals[k][0].replace(",", "")) * UNIT[vals[k][1]]
                              for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
                    traffic[name] = {"bytes_per_launch": tot,
                                     "warp_inst_per_launch": float(vals["smsp__inst_executed.sum"][0].replace(",", "")),
                                     "kernel": rv[rh.index("Kernel Name")] if "Kernel Name" in rh else tag,
                                     "source": f"profiles/r2_final/full_{tag}_details.txt"}
        src = os.path.join(G, f"r2_full_{tag}_source.csv.gz")
        if os.path.exists(src):
            tmp = "/tmp/_r2src.csv"
            with gzip.open(src, "rt") as g, open(tmp, "w") as o:
                o.write(g.read())
            hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), tmp, "40"],
                                 capture_output=True, text=True).stdout
            open(os.path.join(OD, f"full_{tag}_hotlines.txt"), "w").write(hot)
    json.dump(traffic, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    for name, out in (("r2_sweep.txt", "sweep.txt"), ("r2_ubench.txt", "ubench.txt"),
                      ("r2_hgd_lat.txt", "hgd_lat.txt"), ("r2_box.txt", "box.txt"), ("r2_smoke.log", "smoke.txt"),
                      ("r2_checked.txt", "checked_suite.txt"), ("guards.log", "guards_tail.txt"),
                      ("checked.log", "checked_tail.txt")):
        p = os.path.join(G, name)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(OD, out))
    p = os.path.join(G, "r2_pytest_gpu.log")
    if os.path.exists(p):
        open(os.path.join(OD, "pytest_gpu_tail.txt"), "w").writelines(open(p).readlines()[-30:])
    print("wrote", OD)


if __name__ == "__main__":
    main()
