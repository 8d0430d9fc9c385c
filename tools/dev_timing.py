"""Dev probe: per-event latency of one warp and aggregate throughput vs instance count."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_17456_b200 import sweep
from paper_2603_17456_b200.native import DeviceBatch, product

lib = product()
req = int(sys.argv[1]) if len(sys.argv) > 1 else 200
counts = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,148,592,2368").split(",")]
for pol in ["fs", "sjf", "edf", "karuna", "mfs"]:
    b = DeviceBatch(0, lib)
    b.add_config(sweep.sweep_config((0.6, 3, 1, pol), requests=req, lib=lib))
    b.prepare(); b.run(0)
    ev = b.stats(0).events
    b.launch(); ms = b.sync()
    print(f"single {pol}: events {ev} kernel {ms:.1f} ms -> {1000*ms/ev:.2f} us/event steps {b.stats(0).steps} maxA {b.stats(0).max_active}", flush=True)
for n in counts:
    cells = sweep.sweep_cells()[:n]
    b = DeviceBatch(0, lib)
    t = time.time()
    for c in cells:
        b.add_config(sweep.sweep_config(c, requests=req, lib=lib))
    b.prepare(); t1 = time.time(); b.run(0)
    ev = sum(b.stats(i).events for i in range(len(b)))
    b.launch(); ms = b.sync()
    print(f"n={n}: events {ev} kernel {ms:.1f} ms -> {ev/ms*1e3/1e6:.2f} M events/s  (prep {t1-t:.1f}s, dev bytes {b.device_bytes/1e9:.2f} GB)", flush=True)
