"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file):
per kernel launch count, total device time and share of the profiled step(s).

  python tools/launch_shares.py gpurun_out/launches.csv [skip_kernel_regex]
"""
import csv
import io
import re
import sys
from collections import OrderedDict

path = sys.argv[1]
skip = re.compile(sys.argv[2]) if len(sys.argv) > 2 else re.compile(r"^(k_init|k_debug|k_gather)")
lines = [ln for ln in open(path) if ln.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
agg = OrderedDict()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    base = name.split("<")[0]
    if skip.search(base):
        continue
    key = f"{name} grid={r['Grid Size']} block={r['Block Size']}"
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r["Metric Unit"], 1e-6)
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += float(r["Metric Value"].replace(",", "")) * scale
tot = sum(v[1] for v in agg.values()) or 1.0
print(f"{'kernel (template, grid, block)':70s} {'launches':>8s} {'ms total':>10s} {'ms/launch':>10s} {'share':>6s}")
for k, (n, t) in agg.items():
    print(f"{k[:70]:70s} {n:8d} {t:10.3f} {t / n:10.4f} {t / tot:6.3f}")
print(f"{'total':70s} {sum(v[0] for v in agg.values()):8d} {tot:10.3f}")
