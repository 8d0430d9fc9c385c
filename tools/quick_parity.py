"""Quick GPU-vs-reference parity sweep (dev tool; uses oracle/_ref as the checker)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import ref
from paper_2603_17456_b200.native import Native, run_manual, run_config, DeviceBatch

def same(x, y):
    x = np.asarray(x); y = np.asarray(y)
    if x.shape != y.shape: return False
    if x.dtype.kind == 'f':
        return np.array_equal(np.nan_to_num(x, nan=-7.0).view(np.int64), np.nan_to_num(y, nan=-7.0).view(np.int64))
    return np.array_equal(x, y)

KEYS = ["req_arrival","req_deadline","req_done","req_pruned","req_stall","flow_finish","flow_band",
        "flow_level","cof_release","cof_done","cof_stall","pipe_done"]
def compare(a, b, tag):
    bad = []
    for k in ["events","steps","pruned_count","n_batches"]:
        if getattr(a,k) != getattr(b,k): bad.append(f"{k} {getattr(a,k)} vs {getattr(b,k)}")
    for k in KEYS:
        if not same(getattr(a,k), getattr(b,k)):
            bad.append(k)
    if a.summary_json != b.summary_json: bad.append("summary")
    if a.requests_csv != b.requests_csv: bad.append("csv")
    print(tag, "OK" if not bad else bad, a.events, a.steps, flush=True)
    return not bad

if __name__ == "__main__":
    lib = Native(sys.argv[1]) if len(sys.argv) > 1 else None
    base = open(os.path.join(os.path.dirname(__file__), "..", "tests", "configs", "cluster8.conf")).read()
    ok = True
    trio = open(os.path.join(os.path.dirname(__file__), "..", "tests", "configs", "trio.spec")).read()
    for pol in ["mfs","fs","sjf","edf","karuna"]:
        spec = trio.replace("POLICY", pol)
        ok &= compare(ref.run_manual(spec), run_manual(spec, lib=lib), "trio-" + pol)
    for n in [100, 400]:
        for pol in ["fs","sjf","edf","karuna","mfs"]:
            cfg = base + f"\npolicy = {pol}\nworkload.request_count = {n}\n"
            t = time.time(); a = ref.run_config(cfg); t1 = time.time(); b = run_config(cfg, lib=lib); t2 = time.time()
            ok &= compare(a, b, f"cluster8-{n}-{pol}")
            print(f"   ref {t1-t:.2f}s dev {t2-t1:.2f}s", flush=True)
    print("ALL OK" if ok else "MISMATCH")
