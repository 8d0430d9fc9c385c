"""Dev probe: aggregate events/s with n same-policy instances (200 requests each)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_17456_b200 import sweep
from paper_2603_17456_b200.native import DeviceBatch, product
lib = product()
n = int(sys.argv[1]); req = int(sys.argv[2])
for pol in sys.argv[3].split(","):
    cells = [c for c in sweep.sweep_cells() if c[3] == pol][:n]
    b = DeviceBatch(0, lib)
    for c in cells:
        b.add_config(sweep.sweep_config(c, requests=req, lib=lib))
    b.prepare(); b.run(0)
    ev = sum(b.stats(i).events for i in range(len(b)))
    b.launch(); ms = b.sync()
    print(f"{pol} n={n}: {ev} events in {ms:.0f} ms -> {ev/ms/1e3:.2f} M events/s; per-instance avg {ev/n:.0f} events", flush=True)
