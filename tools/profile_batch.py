"""Dev probe for ncu: a full-occupancy batch of sweep instances, warmed up,
then ONE profiled time-sliced launch between cudaProfilerStart/Stop.

  ncu --profile-from-start off --set full ... python tools/profile_batch.py N REQ SLICE_MS
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_17456_b200 import sweep  # noqa: E402
from paper_2603_17456_b200.native import DeviceBatch, product  # noqa: E402

n = int(sys.argv[1])
req = int(sys.argv[2])
slice_ms = float(sys.argv[3])
lib = product()
b = DeviceBatch(0, lib)
for c in bench.cells_for(0, 1, n):
    b.add_config(sweep.sweep_config(c, requests=req, lib=lib))
b.prepare()
b.upload()
for _ in range(2):
    b.launch_slice(int(slice_ms * 1e6))
b.sync()
b.download(0)
e0 = sum(b.stats(i).events for i in range(n))
torch.cuda.cudart().cudaProfilerStart()
b.launch_slice(int(slice_ms * 1e6))
ms = b.sync()
torch.cuda.cudart().cudaProfilerStop()
b.download(0)
e1 = sum(b.stats(i).events for i in range(n))
print(f"profiled launch: {ms:.1f} ms, {e1 - e0} events, {(e1 - e0) / ms * 1e3:.0f} events/s, "
      f"running {b.remaining()}")
