"""Dev probe: throughput over the whole life of a batch of sweep instances.

Runs bench's first N cells to completion in time slices and prints, per slice,
the events simulated, the instances still running and the events/s, then the
whole-run rate (total events / makespan). Shows how representative bench's
steady-state window is. Usage: rate_curve.py N [slice_ms] [max_s]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_17456_b200 import sweep  # noqa: E402
from paper_2603_17456_b200.native import DeviceBatch, product  # noqa: E402

n = int(sys.argv[1])
slice_ms = float(sys.argv[2]) if len(sys.argv) > 2 else 2000.0
max_s = float(sys.argv[3]) if len(sys.argv) > 3 else 600.0
lib = product()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
cells = bench.cells_for(0, 1, n)
t0 = time.perf_counter()
b = DeviceBatch(0, lib, stream=stream.cuda_stream)
for c in cells:
    b.add_config(sweep.sweep_config(c, requests=2000, lib=lib))
b.prepare()
b.upload()
print(f"setup {time.perf_counter() - t0:.1f}s, {len(b)} instances, {b.device_bytes / 1e9:.1f} GB", flush=True)


def events():
    b.download(0)
    return sum(b.stats(i).events for i in range(n))


tot_ms, ev_prev = 0.0, 0
while tot_ms < max_s * 1000:
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    b.launch_slice(int(slice_ms * 1e6))
    e.record(stream)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    tot_ms += ms
    ev = events()
    rem = b.remaining()
    print(f"t={tot_ms / 1000:7.1f}s  slice {ms:7.1f}ms  events {ev - ev_prev:10d}  "
          f"rate {(ev - ev_prev) / ms * 1e3:12.0f}/s  running {rem}", flush=True)
    ev_prev = ev
    if rem == 0:
        break
by_pol = {}
for i, c in enumerate(cells):
    st = b.stats(i)
    by_pol.setdefault(c[3], []).append(st.events)
print(f"whole run: {ev_prev} events in {tot_ms / 1000:.1f}s = {ev_prev / tot_ms * 1e3:.0f} events/s")
for p, v in sorted(by_pol.items()):
    print(f"  {p:7s} {len(v):5d} instances  mean events {sum(v) / len(v):.0f}")
