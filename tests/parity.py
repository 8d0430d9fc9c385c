"""Bit-exact comparison of engine results against the golden fixtures."""
import hashlib
import json
import os

import numpy as np

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ARRAYS = ("req_arrival", "req_deadline", "req_done", "req_pruned", "req_stall", "flow_finish",
          "flow_band", "flow_level", "cof_release", "cof_done", "cof_stall", "pipe_done")
SCALARS = ("events", "steps", "pruned_count", "n_batches")

_cache = {}


def manifest():
    if "m" not in _cache:
        _cache["m"] = json.load(open(os.path.join(GOLD, "manifest.json")))
    return _cache["m"]


def arrays(group):
    if group not in _cache:
        _cache[group] = np.load(os.path.join(GOLD, f"{group}.npz"))
    return _cache[group]


def digest(a):
    a = np.ascontiguousarray(a)
    if a.dtype.kind == "f":
        a = np.nan_to_num(a.astype(np.float64), nan=-7.0)
    elif a.dtype.kind in "iu":
        a = a.astype(np.int64)
    return hashlib.sha256(a.tobytes()).hexdigest()


def bits_equal(x, y):
    x, y = np.asarray(x), np.asarray(y)
    if x.shape != y.shape:
        return False
    if x.dtype.kind == "f" or y.dtype.kind == "f":
        return np.array_equal(np.nan_to_num(x.astype(np.float64), nan=-7.0).view(np.int64),
                              np.nan_to_num(y.astype(np.float64), nan=-7.0).view(np.int64))
    return np.array_equal(x.astype(np.int64), y.astype(np.int64))


def mismatches(res, group, name):
    """list of differing fields (empty = bit-exact) vs the stored fixture"""
    m = manifest()[group][name]
    bad = [f"{k}: {getattr(res, k)} != {m[k]}" for k in SCALARS if int(getattr(res, k)) != m[k]]
    store = arrays(group)
    for k in ARRAYS:
        key = f"{name}/{k}"
        if key in store.files:
            if not bits_equal(getattr(res, k), store[key]):
                bad.append(k)
        elif digest(getattr(res, k)) != m["sha256"][k]:
            bad.append(k + " (sha256)")
    if res.summary_json and res.summary_json != m["summary_json"]:
        bad.append("summary.json bytes")
    if res.requests_csv and hashlib.sha256(res.requests_csv.encode()).hexdigest() != m["requests_csv_sha256"]:
        bad.append("requests.csv bytes")
    return bad
