"""Dev probe: working-set sizes of bench sweep instances (max active, touched links, pool)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_17456_b200 import sweep
from paper_2603_17456_b200.native import DeviceBatch, product
lib = product()
n = int(sys.argv[1]); req = int(sys.argv[2])
cells = bench.cells_for(0, 1, n)
b = DeviceBatch(0, lib)
for c in cells:
    b.add_config(sweep.sweep_config(c, requests=req, lib=lib))
b.prepare(); b.run(0)
rows = []
for i, c in enumerate(cells):
    o = b.counters(i)
    rows.append((c[0], c[3], o[8], o[14], o[15], o[2]))
import collections
for pol in ["fs", "sjf", "edf", "karuna", "mfs"]:
    r = [x for x in rows if x[1] == pol]
    if not r: continue
    A = np.array([x[2] for x in r]); T = np.array([x[3] for x in r]); P = np.array([x[4] for x in r])
    print(f"{pol:7s} n={len(r):3d} maxA p50={np.median(A):.0f} p90={np.percentile(A,90):.0f} max={A.max()}  touch p50={np.median(T):.0f} max={T.max()}  pool max={P.max()}")
A = np.array([x[2] for x in rows]); print("overall maxA > 128:", (A > 128).mean(), " > 192:", (A > 192).mean(), " > 256:", (A > 256).mean())
