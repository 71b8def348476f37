"""Per-source-line instruction counts and stall samples from an ncu report (cuda,sass view)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
cur_file = None
hdr = None
agg = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",) or not r[0]:
        continue
    d = dict(zip(hdr[:4], r[:4]))
    try:
        samples = int(r[4]) if r[4] not in ("-", "") else 0
        inst = int(r[7]) if r[7] not in ("-", "") else 0
    except (ValueError, IndexError):
        continue
    agg.append((inst, samples, cur_file, r[0], r[1][:90]))
tot_i = sum(a[0] for a in agg) or 1
tot_s = sum(a[1] for a in agg) or 1
print(f"total warp-inst {tot_i}, samples {tot_s}")
for inst, samp, f, ln, src in sorted(agg, reverse=True)[:top]:
    print(f"{100*inst/tot_i:5.1f}% inst {100*samp/tot_s:5.1f}% stall  {f}:{ln}  {src}")
print("--- by stall samples")
for inst, samp, f, ln, src in sorted(agg, key=lambda a: -a[1])[:top // 2]:
    print(f"{100*inst/tot_i:5.1f}% inst {100*samp/tot_s:5.1f}% stall  {f}:{ln}  {src}")
