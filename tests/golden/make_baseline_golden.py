#!/usr/bin/env python3
"""Golden digests for the five BASELINE.json configurations, produced by the
reference simulator itself (oracle/_ref/libmfsim_ref.so = the unmodified
reference sources compiled by oracle/Makefile).

One JSON file per case under tests/golden/baseline/: counters, SLO attainment,
summary.json text, sha256 of requests.csv and of every full-precision result
array (same digest rule as make_golden.py). The arrays themselves are too big
to commit at these sizes (configs[2]: ~22M flows per instance).

Cases (paper_2603_17456_b200/configs.py):
  cfg1_<pol>_s<seed>   configs[0]: cluster8, 1024 requests, mfs/fs, seeds 1-5
  cfg2_<pol>           configs[1]: cluster8 at the FS knee, 10k requests, 5 policies
  cfg3_<pol>_s<seed>   configs[2]: ft128 (1024 GPUs), 100k requests, 5 policies, seeds 1-3
  cfg5_<pol>           configs[4]: 4096-GPU fat-tree, heavy-tailed trace, mfs/fs
  cfg2_aalo            configs[1]'s coflow baseline (extension, no reference
                       counterpart): produced by the C restatement
                       (oracle/_ref/libmfsim_oracle.so), marked "oracle": "restatement"

Runs where /root/reference exists (this container), many cases in parallel,
skipping cases whose file already exists:
  python tests/golden/make_baseline_golden.py [-j N] [substring ...]
"""
import json
import os
import sys
import time
from multiprocessing import Pool

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.join(HERE, "..", "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

OUT = os.path.join(HERE, "baseline")
POLICIES = ("fs", "sjf", "edf", "karuna", "mfs")


def baseline_cases():
    from paper_2603_17456_b200 import configs
    c = {}
    for p in ("mfs", "fs"):
        for s in range(1, 6):
            c[f"cfg1_{p}_s{s}"] = configs.config1(seed=s, policy=p)
    for p in POLICIES + ("aalo",):
        c[f"cfg2_{p}"] = configs.config2(policy=p)
    for p in POLICIES:
        for s in (1, 2, 3):
            c[f"cfg3_{p}_s{s}"] = configs.config3(seed=s, policy=p)
    for p in ("mfs", "fs"):
        c[f"cfg5_{p}"] = configs.config5(policy=p)
    return c


def _cost(name):  # longest first (measured CPU ratios)
    size = {"cfg1": 1, "cfg2": 10, "cfg3": 100, "cfg5": 50}[name[:4]]
    pol = name.split("_")[1]
    return size * {"karuna": 14, "mfs": 3}.get(pol, 1)


def _one(item):
    name, text = item
    from oracle import ref
    from make_golden import record
    t0 = time.time()
    so = ref.ORACLE_SO if "policy = aalo" in text else ref.REF_SO
    res = ref.run_config(text, so=so)
    meta = record(res, {}, name, full=False)
    meta["n_requests"] = int(len(res.req_done))
    meta["n_flows"] = int(len(res.flow_finish))
    meta["ref_seconds"] = round(time.time() - t0, 1)
    meta["config"] = text
    meta["oracle"] = "restatement" if so == ref.ORACLE_SO else "reference"
    path = os.path.join(OUT, name + ".json")
    with open(path + ".tmp", "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    os.replace(path + ".tmp", path)
    return name, res.events, res.attainment, meta["ref_seconds"]


def main():
    args = sys.argv[1:]
    jobs = os.cpu_count() or 4
    if args[:1] == ["-j"]:
        jobs, args = int(args[1]), args[2:]
    os.makedirs(OUT, exist_ok=True)
    todo = [(n, t) for n, t in baseline_cases().items()
            if not os.path.exists(os.path.join(OUT, n + ".json")) and (not args or any(a in n for a in args))]
    todo.sort(key=lambda x: -_cost(x[0]))
    with Pool(jobs, maxtasksperchild=1) as pool:
        for name, ev, att, sec in pool.imap_unordered(_one, todo):
            print(f"{name}: events={ev} attainment={att} ({sec}s)", flush=True)


if __name__ == "__main__":
    main()
