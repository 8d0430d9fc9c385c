"""A/B of engine builds on the bench workload: for each library (and instance
count) run W warm-up slices then K timed slices of S ms; print events/s.
  python tools/ab_variants.py N S K lib1.so[:N1] lib2.so[:N2] ..."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_17456_b200 import sweep  # noqa: E402
from paper_2603_17456_b200.native import DeviceBatch, Native  # noqa: E402

n_def, slice_ms, k = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
for spec in sys.argv[4:]:
    path, _, nn = spec.partition(":")
    n = int(nn) if nn else n_def
    lib = Native(path)
    b = DeviceBatch(0, lib)
    t0 = time.time()
    for c in bench.cells_for(0, 1, n):
        b.add_config(sweep.sweep_config(c, requests=2000, lib=lib))
    b.prepare()
    b.upload()
    setup = time.time() - t0
    for _ in range(2):
        b.launch_slice(int(slice_ms * 1e6))
    b.sync()
    b.download(0)
    e0 = sum(b.stats(i).events for i in range(n))
    ms = 0.0
    for _ in range(k):
        b.launch_slice(int(slice_ms * 1e6))
        ms += b.sync()
    b.download(0)
    e1 = sum(b.stats(i).events for i in range(n))
    print(f"{os.path.basename(path)} n={n}: {(e1 - e0) / ms * 1e3 / 1e6:.3f} M events/s "
          f"({e1 - e0} events in {ms:.0f} ms, setup {setup:.1f}s)", flush=True)
    del b
