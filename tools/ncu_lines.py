"""Per-function and per-line summary of an ncu cuda,sass source export:
  ncu -i rep --page source --csv --print-source cuda,sass > cs.csv
  python tools/ncu_lines.py cs.csv paper_2603_17456_b200/csrc/device/engine.cuh [N]
Prints executed warp instructions, stall samples and barrier-stall samples per
engine function (by the line ranges of the `MF_FN`/`MF_NOINLINE` members of the
given source) and the N hottest source lines."""
import csv
import re
import sys

path, src = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
lines = open(src).read().split("\n")
starts = []
for i, l in enumerate(lines, 1):
    m = re.match(r"\s*(?:template <[^>]*>\s*)?(MF_FN|MF_NOINLINE)\s+[\w:<>,\s\*&]+?\b(\w+)\(", l)
    if m:
        starts.append((i, m.group(2)))


def func_of(line):
    name = "?"
    for s, f in starts:
        if s <= line:
            name = f
        else:
            break
    return name


rows = csv.reader(open(path))
hdr = None
fname = ""
per_line = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or not r[0].isdigit():
        continue

    def g(k):
        try:
            return int(r[hdr[k]])
        except (KeyError, ValueError):
            return 0
    key = (fname.split("/")[-1], int(r[0]))
    a = per_line.setdefault(key, [0, 0, 0, 0, r[1].strip()[:80]])
    a[0] += g("Instructions Executed")
    a[1] += g("Warp Stall Sampling (All Samples)")
    a[2] += g("stall_barrier")
    a[3] += g("stall_no_inst")
tot_i = sum(v[0] for v in per_line.values()) or 1
tot_s = sum(v[1] for v in per_line.values()) or 1
funcs = {}
base = src.split("/")[-1]
for (f, ln), v in per_line.items():
    k = func_of(ln) if f == base else f
    a = funcs.setdefault(k, [0, 0, 0, 0])
    for j in range(4):
        a[j] += v[j]
print(f"warp instructions {tot_i}, stall samples {tot_s}")
print(f"{'function':<28} {'%instr':>7} {'%stall':>7} {'%barrier':>8} {'%noinst':>8}")
for k, a in sorted(funcs.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{k:<28} {100*a[0]/tot_i:7.2f} {100*a[1]/tot_s:7.2f} {100*a[2]/tot_s:8.2f} {100*a[3]/tot_s:8.2f}")
print("== hottest lines by instructions")
for (f, ln), v in sorted(per_line.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{100*v[0]/tot_i:5.2f}%i {100*v[1]/tot_s:5.2f}%s {f}:{ln:<5} {v[4]}")
