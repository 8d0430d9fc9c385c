"""Summarise an ncu --page source --csv --print-source cuda,sass dump: top source
lines by warp-stall samples and by executed warp instructions."""
import csv
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hdr = None
fname = "?"
agg = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or len(r) < 8:
        continue
    d = dict(zip(hdr, r))
    try:
        smp = int(d["Warp Stall Sampling (All Samples)"])
        ins = int(d["Instructions Executed"])
    except (ValueError, KeyError):
        continue
    stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
    top = sorted(stalls.items(), key=lambda x: -x[1])[:2]
    agg.append((smp, ins, f"{fname}:{r[0]}", r[1].strip()[:90], top))
tot_s = sum(a[0] for a in agg)
tot_i = sum(a[1] for a in agg)
print(f"total samples {tot_s}, warp instructions {tot_i}")
print("== by stall samples")
for a in sorted(agg, key=lambda x: -x[0])[:n]:
    print(f"{100*a[0]/tot_s:5.1f}% {100*a[1]/tot_i:5.1f}%i {a[2]:<22} {a[3]:<90} {a[4]}")
print("== by instructions")
for a in sorted(agg, key=lambda x: -x[1])[:n]:
    print(f"{100*a[0]/tot_s:5.1f}% {100*a[1]/tot_i:5.1f}%i {a[2]:<22} {a[3]}")
