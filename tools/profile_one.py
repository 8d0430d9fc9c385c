"""Dev probe: one small instance per listed policy, one launch each (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_17456_b200 import sweep
from paper_2603_17456_b200.native import DeviceBatch, product
lib = product()
req = int(sys.argv[1]); pols = sys.argv[2].split(",")
b = DeviceBatch(0, lib)
for p in pols:
    b.add_config(sweep.sweep_config((0.6, 3, 1, p), requests=req, lib=lib))
b.prepare()
b.run(0)
for i in range(len(b)):
    s = b.stats(i); print(pols[i], s.events, s.steps, s.status)
b.launch(); print("kernel ms", b.sync())
