"""Dev probe: per-phase device cycles per event (profiling build) over the
first BUDGET events of single BASELINE configs[2] instances (one warp each).
  python tools/phase_profile_budget.py LIB POLICY BUDGET"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_17456_b200 import configs  # noqa: E402
from paper_2603_17456_b200.native import DeviceBatch, Native  # noqa: E402

lib = Native(sys.argv[1])
pol, budget = sys.argv[2], int(sys.argv[3])
b = DeviceBatch(0, lib)
b.add_config(configs.config3(seed=1, policy=pol))
b.prepare()
b.upload()
b.reset()
b.launch_budget(budget)
ms = b.sync()
b.download(0)
c = b.counters(0)
ev, st = c[2], c[3]
names = ["next", "advance", "handler", "decide", "alloc", "resched", "batchev", "promote"]
sn = ["a_prep", "a_count", "a_inc", "a_apply", "a_freeze", "a_restore", "finish", "release", "compute",
      "depart", "admit", "k_caps", "subset", "fullsort"]
print(f"{os.path.basename(sys.argv[1])} {pol}: events {ev} steps {st} kernel {ms:.0f} ms = {1e3 * ms / ev:.1f} us/event; "
      f"rounds/step {c[13] / max(st, 1):.1f}; cycles/event: "
      + " ".join(f"{n}={v / ev:.0f}" for n, v in zip(names, c[16:24])) + f" total={c[16:24].sum() / ev:.0f}")
print("    sub: " + " ".join(f"{n}={v / ev:.0f}" for n, v in zip(sn, c[24:38])), flush=True)
