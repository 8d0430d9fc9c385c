#!/usr/bin/env python3
"""Generate the golden fixtures from the reference simulator itself.

Runs oracle/_ref/libmfsim_ref.so (the unmodified reference sources compiled by
oracle/Makefile) on every case in cases.py and stores full-precision results:
  golden/manual.npz, golden/workload.npz   arrays per case (bit patterns kept)
  golden/manifest.json                    counters + sha256 of every array
Big cases (BASELINE configs[0] sizes) are stored as hashes only.

Must run where /root/reference exists (this container); the GPU box only reads
the committed fixtures.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, HERE)

from oracle import ref  # noqa: E402
import cases  # noqa: E402

ARRAYS = ("req_arrival", "req_deadline", "req_done", "req_pruned", "req_stall", "flow_finish",
          "flow_band", "flow_level", "cof_release", "cof_done", "cof_stall", "pipe_done")
SCALARS = ("events", "steps", "pruned_count", "n_batches")


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype.kind == "f":
        a = np.nan_to_num(a.astype(np.float64), nan=-7.0)
    elif a.dtype.kind in "iu":
        a = a.astype(np.int64)
    return hashlib.sha256(a.tobytes()).hexdigest()


def record(res, store, name, full=True):
    meta = {k: int(getattr(res, k)) for k in SCALARS}
    meta["attainment"] = res.attainment
    meta["sha256"] = {k: digest(getattr(res, k)) for k in ARRAYS}
    meta["summary_json"] = res.summary_json
    meta["requests_csv_sha256"] = hashlib.sha256(res.requests_csv.encode()).hexdigest()
    if full:
        for k in ARRAYS:
            store[f"{name}/{k}"] = np.asarray(getattr(res, k))
    return meta


def main():
    big = "--big" in sys.argv
    manifest = {"manual": {}, "workload": {}, "errors": {}}
    store_m, store_w = {}, {}
    for name, spec in cases.manual_cases().items():
        manifest["manual"][name] = record(ref.run_manual(spec), store_m, name)
    try:
        ref.run_manual(cases.livelock())
        manifest["errors"]["livelock"] = 0
    except ref.RefError as e:
        manifest["errors"]["livelock"] = e.code
    for name, text in cases.workload_cases(big=big).items():
        res = ref.run_config(text)
        full = not name.startswith("cluster8_1024")
        manifest["workload"][name] = record(res, store_w, name, full=full)
        print(name, res.events, res.steps, res.attainment, flush=True)
    np.savez_compressed(os.path.join(HERE, "manual.npz"), **store_m)
    np.savez_compressed(os.path.join(HERE, "workload.npz"), **store_w)
    json.dump(manifest, open(os.path.join(HERE, "manifest.json"), "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
