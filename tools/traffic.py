"""profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum (bytes per
launch) and smsp__inst_executed.sum (warp instructions per launch, for
roofline.issue) of each workload's dominant kernel, from the ncu --set full captures
gpurun_out/full_<workload>.ncu-rep (read by bench.py for roofline.traffic)."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
out = {}
try:    # entries of workloads not captured this time are kept
    out = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
except Exception:
    pass
for w in ["headline", "cfg1", "complement", "wr", "bernoulli", "gnm", "algb"]:
    rep = os.path.join(ROOT, "gpurun_out", f"full_{w}.ncu-rep")
    if not os.path.exists(rep):
        continue
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    tot = 0.0
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(name)
        tot += float(v[i].replace(",", "")) * UNIT[u[i]]
    name = bench._workload(w, 1)["name"]
    wi = float(v[h.index("smsp__inst_executed.sum")].replace(",", "")) if "smsp__inst_executed.sum" in h else None
    out[name] = {"bytes_per_launch": tot, "warp_inst_per_launch": wi, "kernel": v[h.index("Kernel Name")],
                 "source": f"full_{w}.ncu-rep"}
    print(name, out[name])
json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
