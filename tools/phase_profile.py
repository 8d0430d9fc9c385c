"""Dev probe: per-phase device cycles per event (profiling build) for single instances."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_17456_b200 import sweep
from paper_2603_17456_b200.native import DeviceBatch, Native
lib = Native(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "libmfsim_b200_prof.so"))
req = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rho = float(sys.argv[3]) if len(sys.argv) > 3 else 0.6
names = ["next", "advance", "handler", "decide", "alloc", "resched", "batchev", "promote"]
for pol in (sys.argv[2] if len(sys.argv) > 2 else "fs,sjf,edf,karuna,mfs").split(","):
    b = DeviceBatch(0, lib)
    b.add_config(sweep.sweep_config((rho, 3, 1, pol), requests=req, lib=lib))
    b.prepare(); b.run(0)
    b.launch(); ms = b.sync(); b.download(0)
    c = b.counters(0); ev = c[2]; st = c[3]
    cyc = c[16:24]
    print(f"{pol}: maxA {c[8]} events {ev} steps {st} kernel {ms:.0f} ms = {1e6*ms/1e3/ev:.1f} us/ev; cycles/event: " +
          " ".join(f"{n}={v/ev:.0f}" for n, v in zip(names, cyc)) + f" total={cyc.sum()/ev:.0f}", flush=True)
    sub = c[24:38]
    sn = ["a_prep", "a_count", "a_inc", "a_apply", "a_freeze", "a_restore", "finish", "release", "compute", "depart", "admit", "k_caps", "subset", "fullsort"]
    print("    sub cycles/event: " + " ".join(f"{n}={v/ev:.0f}" for n, v in zip(sn, sub)), f"rounds/step={c[13]/st:.1f}", flush=True)
