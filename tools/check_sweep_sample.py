"""Spot-check a configs[3] full-grid run (sweep_run --grid configs3) against
the reference simulator (oracle/_ref) on a deterministic sample of cells.

  extract ttft.npz sample.npz   on the GPU box: keep the sampled cells' TTFTs
  precompute cache.npz          here, before the GPU run ends: the reference on
                                the sampled cells of the grid (same rates)
  check sweep.csv sample.npz [cache.npz]
                                here: run the reference on each sampled cell
                                (all host cores), compare the sweep.csv row and
                                the per-request TTFTs bit for bit

Test infrastructure: the reference is the checker, never the thing measured."""
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
N_SAMPLE = 40


def sample_keys(keys):
    """every 277th cell of the grid order (varies policy, load, seed and SLO scale)"""
    return keys[::277][:N_SAMPLE]


def rows(csv_path):
    lines = open(csv_path).read().splitlines(keepends=True)
    return lines[0], lines[1:]


def key_of_row(r):
    p, rate, seed, slo = r.split(",")[:4]
    return f"{p}/rate_{rate}/seed_{seed}/slo_{slo}"


def extract(npz_in, npz_out):
    z = np.load(npz_in)
    keys = [k[:-len("/ttft")] for k in z.files if k.endswith("/ttft")]  # grid order
    keep = sample_keys(keys)
    np.savez_compressed(npz_out, **{k + "/ttft": z[k + "/ttft"] for k in keep})
    print(f"kept {len(keep)} of {len(keys)} cells")


def _ref_cell(key):
    from oracle import ref
    from paper_2603_17456_b200 import sweep, sweep_run
    p, rate, seed, slo = [x.split("_", 1)[-1] for x in key.split("/")]
    base = sweep.text(dict(sweep.FT128, **{"workload.request_count": 2000}))
    res = ref.run_config(base + f"policy = {p}\nworkload.rate_rps = {rate}\nsim.seed = {seed}\n"
                                f"workload.slo_multiplier = {slo}\n")
    row = sweep_run.csv_row((p, rate, seed, slo), res.summary_json)
    return key, row, np.asarray(res.req_done) - np.asarray(res.req_arrival), res.events


def grid_keys():
    from paper_2603_17456_b200 import sweep, sweep_run
    from paper_2603_17456_b200.native import Native
    emu = Native(os.path.join(ROOT, "build", "libmfsim_emu.so"))
    rates = [repr(sweep.rate_for_load(x, sweep.FT128, emu)) for x in sweep.LOADS]
    cells = sweep_run.sweep_cells(list(sweep.POLICIES), rates, [str(x) for x in range(1, 65)],
                                  [str(x) for x in sweep.SLO_SCALES])
    return [sweep_run.cell_key(c) for c in cells]


def precompute(cache):
    keys = sample_keys(grid_keys())
    out = {}
    with ProcessPoolExecutor(os.cpu_count()) as ex:
        for key, row, ttft, ev in ex.map(_ref_cell, keys):
            out[key + "/row"] = np.frombuffer(row.encode(), np.uint8)
            out[key + "/ttft"] = ttft
            out[key + "/events"] = np.array([ev])
            print(key, ev, flush=True)
    np.savez_compressed(cache, **out)


def _cached(cache):
    z = np.load(cache)
    keys = [k[:-len("/row")] for k in z.files if k.endswith("/row")]
    return {k: (k, z[k + "/row"].tobytes().decode(), z[k + "/ttft"], int(z[k + "/events"][0]))
            for k in keys}


def check(csv_path, npz_path, cache=None):
    _, body = rows(csv_path)
    by_key = {key_of_row(r): r for r in body}
    assert len(by_key) == 11200, len(by_key)
    z = np.load(npz_path)
    keys = [k.rsplit("/", 1)[0] for k in z.files]
    bad = 0
    have = _cached(cache) if cache else {}
    with ProcessPoolExecutor(os.cpu_count()) as ex:
        todo = [k for k in keys if k not in have]
        for key, row, ttft, ev in [have[k] for k in keys if k in have] + list(ex.map(_ref_cell, todo)):
            ok_row = by_key[key] == row
            ok_ttft = np.array_equal(z[key + "/ttft"], ttft, equal_nan=True)
            bad += not (ok_row and ok_ttft)
            att = row.split(",")[4]
            print(f"{key}: events {ev}, slo_attainment {att}, row {'==' if ok_row else '!='}, "
                  f"ttft {'bit-exact' if ok_ttft else 'DIFFERS'}", flush=True)
    print(f"{len(keys)} sampled cells, {bad} mismatches")
    return bad


if __name__ == "__main__":
    if sys.argv[1] == "extract":
        extract(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "precompute":
        precompute(sys.argv[2])
    else:
        sys.exit(1 if check(sys.argv[2], sys.argv[3], *sys.argv[4:5]) else 0)
