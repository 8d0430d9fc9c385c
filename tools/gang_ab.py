"""A/B of the lock-step gang kernel (MFSIM_GANG = warps per block) on the bench
workload, plus a bit-exactness check of every golden fixture under each gang size.

  python tools/gang_ab.py N SLICE_MS K SPEC1 SPEC2 ...
SPEC = W[:noparity][:lib=PATH][:nomin] (W = 1: the one-warp kernel; noparity:
skip the fixture check; lib: an A/B build of the library instead of the
product; nomin: no forced gang for small batches -- the library sizes the gang
to the running instances itself).
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import bench  # noqa: E402
import cases  # noqa: E402
from parity import mismatches  # noqa: E402
from paper_2603_17456_b200 import sweep  # noqa: E402
from paper_2603_17456_b200.native import DeviceBatch, Native, product  # noqa: E402

n, slice_ms, k = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
for spec in sys.argv[4:]:
    parts = spec.split(":")
    lib = product()
    for p in parts:
        if p.startswith("lib="):
            lib = Native(p[4:])
    w = int(parts[0])
    os.environ["MFSIM_GANG"] = str(w)
    os.environ["MFSIM_GANG_MIN"] = "1"
    if "nomin" in parts:  # the library's own choice of kernel and gang size
        os.environ.pop("MFSIM_GANG_MIN")
    for p in parts[1:]:  # MFSIM_*=value: an environment knob for this spec only
        if p.startswith("MFSIM_") and "=" in p:
            knob, val = p.split("=", 1)
            os.environ[knob] = val
    w = spec
    if "noparity" in parts:
        man, wl = [], []
    # parity: every manual + workload fixture in one launch
    b = DeviceBatch(0, lib)
    if "noparity" not in parts:
        man = sorted(cases.manual_cases())
        wl = sorted(cases.workload_cases())
    for m in man:
        b.add_manual(cases.manual_cases()[m])
    for c in wl:
        b.add_config(cases.workload_cases()[c])
    if man or wl:
        b.prepare()
        b.run(2)
    bad = {}
    for i, m in enumerate(man):
        x = mismatches(b.result(i, 2), "manual", m)
        if x:
            bad[m] = x
    for j, c in enumerate(wl):
        x = mismatches(b.result(len(man) + j, 2), "workload", c)
        if x:
            bad[c] = x
    del b
    print(f"gang {w}: fixtures {'bit-exact' if not bad else 'MISMATCH ' + str(bad)[:400]}", flush=True)
    # throughput on the bench cells
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
    print(f"gang {w} n={n}: {(e1 - e0) / ms * 1e3 / 1e6:.3f} M events/s "
          f"({e1 - e0} events in {ms:.0f} ms, setup {setup:.1f}s)", flush=True)
    del b
    for p in parts[1:]:
        if p.startswith("MFSIM_") and "=" in p:
            os.environ.pop(p.split("=", 1)[0], None)
