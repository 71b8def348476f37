"""Per-source-line stall breakdown from an ncu report: python tools/ncu_stalls.py rep kernel [top]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
f = None; hdr = None; out = []
for r in rows:
    if not r: continue
    if r[0] == "File Name" or r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or not r[0].isdigit(): continue
    if len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    d["Source"] = r[1]
    st = {k[6:]: int(d[k]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k and d.get(k, "0").isdigit()}
    tot = sum(st.values())
    if tot: out.append((tot, f, int(r[0]), d["Source"].strip()[:70], st, int(d.get("Instructions Executed", "0") or 0)))
T = sum(o[0] for o in out)
I = sum(o[5] for o in out)
agg = {}
for o in out:
    for k, v in o[4].items(): agg[k] = agg.get(k, 0) + v
print("total samples", T, "warp-inst", I, " ".join(f"{k}={100*v/T:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
for tot, f, ln, src, st, ni in sorted(out, reverse=True)[:top]:
    s3 = sorted(st.items(), key=lambda x: -x[1])[:3]
    print(f"{100*tot/T:5.1f}% {100*ni/max(I,1):5.1f}%i {f}:{ln} {src} | " + " ".join(f"{k}:{100*v/tot:.0f}" for k, v in s3))
