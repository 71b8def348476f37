"""Record per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and issued
warp instructions (smsp__inst_executed.sum) of the kernels in an `ncu --set full` report
into profiles/ncu_traffic.json, keyed by workload, so bench.py can put them beside the
algorithmic bytes in its roofline object (HBM fraction and issue fraction).

  python tools/ncu_traffic.py REPORT.ncu-rep WORKLOAD_KEY   (e.g. C4:N=268435456:M=64)
Several launches of one kernel are averaged.
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, key = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(io.StringIO(raw))
hdr = next(r)
units = dict(zip(hdr, next(r)))
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
acc = {}
inst = {}
for row in r:
    d = dict(zip(hdr, row))
    name = d["Kernel Name"].replace("void ", "").split("<")[0].split("(")[0].split("::")[-1]
    # bench.py keys kernels by kind: the warp-specialised and compile-time instances of a pass
    # (k_stages_ws, k_stages_wsc, k_pass1c) report under their pass's name
    for kind in ("k_stages", "k_pass1"):
        if name.startswith(kind):
            name = kind
    tot = sum(float(d[m].replace(",", "")) * scale[units[m]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    acc.setdefault(name, []).append(tot)
    if "smsp__inst_executed.sum" in d:
        inst.setdefault(name, []).append(float(d["smsp__inst_executed.sum"].replace(",", "")))
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
db = json.load(open(path)) if os.path.exists(path) else {}
ent = db.setdefault(key, {})
for k, v in acc.items():
    ent[k] = sum(v) / len(v)
    print(f"{key} {k}: {ent[k] / 1e9:.3f} GB per launch ({len(v)} launches)")
ient = db.setdefault(key + ":warp_inst", {})
for k, v in inst.items():
    ient[k] = sum(v) / len(v)
    print(f"{key} {k}: {ient[k]:.4g} warp instructions per launch")
json.dump(db, open(path, "w"), indent=1, sort_keys=True)
