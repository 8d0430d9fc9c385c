"""Sharded sweep driver: the reference's `simsweep` (tools/simsweep.cpp:26-94)
on 1..8 GPUs of one node.

Cells are (policy, rate, seed) exactly as simsweep enumerates them
(simsweep.cpp:58-60: policy-major, then rate, then seed). Every rank takes a
disjoint share of the cells (longest-processing-time-first over a static cost
estimate, identical on all ranks), runs its whole share as ONE device batch
(`mfsim_dev_*`, one persistent launch), and writes each cell's
`requests.csv` / `summary.json` into `<out>/<policy>/rate_<r>/seed_<s>/` like
`mfsim_run` does (simsweep.cpp:62-66). There is no collective on the data
path. At the end, the per-request TTFT (f64) and SLO flag (u8) of every cell
are gathered to rank 0 with two all-gathers over the process group (NCCL on
GPUs), and rank 0 writes `<out>/sweep.csv` with simsweep's header and field
formatting (values are the summary's own JSON number tokens, i.e. nlohmann's
`os << j[key]`, simsweep.cpp:50-55), plus `<out>/ttft.npz` with the gathered
per-request arrays. Rank 0 re-derives every cell's `slo_attainment` from the
gathered flags (metrics.cpp:32-40) and fails loudly if it differs from the
cell's summary.

  python -m paper_2603_17456_b200.sweep_run --config C --policies fs,mfs \
      --rates 1,2 --seeds 1,2,3 --out DIR
  torchrun --nproc-per-node 8 --master-addr 127.0.0.1 -m paper_2603_17456_b200.sweep_run ...

Beyond simsweep, an SLO-multiplier axis (`--slo-multipliers 1,2,3`, sets
`workload.slo_multiplier`) and an offered-load axis (`--loads 0.3,0.5`, each
rho mapped to `workload.rate_rps` by `sweep.rate_for_load` on the base config)
give BASELINE configs[3]'s grid; `--grid configs3` is that whole grid (ft128,
2000 requests, rho 0.3..0.9 x SLO 1..5 x seeds 1..64 x 5 policies = 11,200
cells). With the SLO axis the cells are (policy, rate, seed, slo) and
sweep.csv gains a `slo_multiplier` column after `seed`; without it every
output is simsweep's, byte for byte. A rank's share runs in device batches of
at most `--batch-cap` instances (default: what free HBM holds).
"""
from __future__ import annotations

import argparse
import json
import os
import re
import sys

import numpy as np

CSV_HEADER = ("policy,rate_rps,seed,slo_attainment,ttft_mean_s,ttft_p99_s,cct_mean_s,"
              "cct_p99_s,earliness_nonneg_mean_s,stall_mean_s,pruned_count\n")
CSV_KEYS = ("slo_attainment", "ttft_mean_s", "ttft_p99_s", "cct_mean_s", "cct_p99_s",
            "earliness_nonneg_mean_s", "stall_mean_s", "pruned_count")
POLICY_COST = {"karuna": 14.0, "mfs": 3.0, "sjf": 1.2, "edf": 1.0, "fs": 1.0}


def split_list(s: str):
    """simsweep.cpp:17-24: comma-separated, empty items dropped"""
    return [x for x in s.split(",") if x]


def sweep_cells(policies, rates, seeds, slos=None):
    """simsweep order (policy-major, then rate, then seed); the SLO-multiplier
    axis, when given, is innermost"""
    if not slos:
        return [(p, r, s) for p in policies for r in rates for s in seeds]
    return [(p, r, s, m) for p in policies for r in rates for s in seeds for m in slos]


def cell_dir(out: str, cell) -> str:
    d = os.path.join(out, cell[0], "rate_" + cell[1], "seed_" + cell[2])
    return os.path.join(d, "slo_" + cell[3]) if len(cell) > 3 else d


def cell_key(cell) -> str:
    return "/".join([cell[0], "rate_" + cell[1], "seed_" + cell[2]] +
                    (["slo_" + cell[3]] if len(cell) > 3 else []))


def csv_header(slo_axis: bool) -> str:
    if not slo_axis:
        return CSV_HEADER
    return CSV_HEADER.replace("seed,", "seed,slo_multiplier,", 1)


def parse_config_text(text: str) -> dict:
    """`section.key = value` lines (config.cpp's format; '#' comments) -> dict"""
    d = {}
    for line in text.splitlines():
        line = line.split("#", 1)[0].strip()
        if "=" in line:
            k, v = line.split("=", 1)
            d[k.strip()] = v.strip()
    return d


def shard(cells, world: int, cost=None):
    """LPT assignment: cells by estimated cost descending, each to the least
    loaded rank (ties -> lowest rank). Deterministic on every rank."""
    cost = cost or (lambda c: POLICY_COST.get(c[0], 1.0) * float(c[1]))
    order = sorted(range(len(cells)), key=lambda i: (-cost(cells[i]), i))
    load = [0.0] * world
    owner = [0] * len(cells)
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        owner[i] = r
        load[r] += cost(cells[i])
    return owner


def json_token(summary: str, key: str) -> str:
    """The raw JSON text of `key`'s value ('' for null/absent) -- exactly what
    simsweep's `os << j[key]` prints for a number nlohmann itself dumped."""
    m = re.search(r'"%s":\s*([^,\n}]+)' % re.escape(key), summary)
    if not m or m.group(1).strip() == "null":
        return ""
    return m.group(1).strip()


def csv_row(cell, summary: str) -> str:
    return ",".join(list(cell) + [json_token(summary, k) for k in CSV_KEYS]) + "\n"


def ttft_and_flags(res):
    """per-request TTFT (done - arrival; NaN if never done) and SLO flag
    ((done - arrival) <= (deadline - arrival), metrics.cpp:32-40)"""
    ttft = res.req_done - res.req_arrival
    flags = np.zeros(len(ttft), np.uint8)
    ok = ~np.isnan(ttft)
    flags[ok] = (ttft[ok] <= (res.req_deadline[ok] - res.req_arrival[ok])).astype(np.uint8)
    return ttft, flags


def run_cells(texts, lib, device: int = 0, stream=None):
    """one device batch over the given config texts -> [(summary_json, ttft, flags, res)]"""
    from .native import DeviceBatch
    b = DeviceBatch(device, lib, stream=stream)
    for t in texts:
        b.add_config(t)
    b.prepare()
    b.run(1)  # detail 1: requests + coflows (the summary's CCT fields)
    out = []
    for i in range(len(texts)):
        b.raise_for_status(i)
        res = b.result(i, detail=0, reports=True)
        ttft, flags = ttft_and_flags(res)
        out.append((res.summary_json, ttft, flags, res))
    return b, out


def _gather_concat(local: np.ndarray, dtype, world: int, device):
    """all-gather variable-length 1-D arrays: sizes first, then one padded all-gather"""
    import torch
    import torch.distributed as dist
    n = torch.tensor([local.size], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(x.item()) for x in sizes]
    cap = max(max(sizes), 1)
    buf = torch.zeros(cap, dtype=dtype, device=device)
    if local.size:
        buf[:local.size] = torch.from_numpy(local).to(device)
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    return [p[:k].cpu().numpy() for p, k in zip(parts, sizes)]


def main(argv=None, lib=None, backend=None):
    ap = argparse.ArgumentParser(description="sweep (policy x rate x seed) simulation cells on B200s")
    ap.add_argument("--config", default="", help="config file (key = value lines)")
    ap.add_argument("--policies", default="fs,sjf,edf,karuna,mfs")
    ap.add_argument("--rates", default="1")
    ap.add_argument("--seeds", default="1")
    ap.add_argument("--slo-multipliers", default="", help="SLO-multiplier axis (workload.slo_multiplier)")
    ap.add_argument("--loads", default="", help="offered-load axis rho (replaces --rates)")
    ap.add_argument("--grid", default="", choices=["", "configs3"],
                    help="configs3: BASELINE configs[3]'s whole 11,200-cell grid")
    ap.add_argument("--batch-cap", type=int, default=0, help="max instances per device batch (0: all)")
    ap.add_argument("--out", default="sweep_out")
    ap.add_argument("--no-reports", action="store_true", help="skip per-cell requests.csv/summary.json")
    ap.add_argument("--no-ttft-npz", action="store_true", help="gather, check, but do not write ttft.npz")
    a = ap.parse_args(argv)

    import torch
    import torch.distributed as dist
    from .native import Config, product

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if lib is None:
        lib = product()
        torch.cuda.set_device(local)
        device = torch.device("cuda", local)
        backend = backend or "nccl"
    else:  # tests: host emulation library, gloo
        device = torch.device("cpu")
        backend = backend or "gloo"
    init_here = world > 1 and not dist.is_initialized()
    if init_here:
        dist.init_process_group(backend, rank=rank, world_size=world)

    base = open(a.config).read() if a.config else ""
    if a.grid == "configs3":
        from . import sweep
        base = sweep.text(dict(sweep.FT128, **{"workload.request_count": 2000}))
        a.policies = ",".join(sweep.POLICIES)
        a.loads = ",".join(str(x) for x in sweep.LOADS)
        a.slo_multipliers = ",".join(str(x) for x in sweep.SLO_SCALES)
        a.seeds = ",".join(str(x) for x in range(1, 65))
        a.batch_cap = a.batch_cap or 4000
    rates = split_list(a.rates)
    if a.loads:  # rho -> per-unit request rate on this base config (sweep.rate_for_load)
        from . import sweep
        cfg = parse_config_text(base)
        rates = [repr(sweep.rate_for_load(float(x), cfg, lib)) for x in split_list(a.loads)]
    slos = split_list(a.slo_multipliers)
    cells = sweep_cells(split_list(a.policies), rates, split_list(a.seeds), slos)
    owner = shard(cells, world)
    mine = [i for i in range(len(cells)) if owner[i] == rank]

    def text(cell):
        c = Config(base, lib)
        c.set("policy", cell[0]).set("workload.rate_rps", cell[1]).set("sim.seed", cell[2])
        if len(cell) > 3:
            c.set("workload.slo_multiplier", cell[3])
        return c

    import time
    results = []
    cap = a.batch_cap if a.batch_cap > 0 else max(len(mine), 1)
    t0 = time.time()
    for c0 in range(0, len(mine), cap):
        part = mine[c0:c0 + cap]
        batch, res = run_cells([text(cells[i]) for i in part], lib, device=local)
        print(f"rank {rank}: batch of {len(part)} cells, {sum(r[3].events for r in res)} events, "
              f"{time.time() - t0:.1f} s since start", flush=True)
        if not a.no_reports:
            for k, i in enumerate(part):
                d = cell_dir(a.out, cells[i])
                os.makedirs(d, exist_ok=True)
                lib.check(lib.lib.mfsim_dev_write_report(batch.h, k, d.encode()))
        del batch
        results.extend(res)

    # final gather of per-request TTFT + SLO flags (and the summaries) to rank 0
    idx = np.array(mine, np.int64)
    lens = np.array([len(r[1]) for r in results], np.int64)
    ttft = np.concatenate([r[1] for r in results]) if results else np.zeros(0)
    flags = np.concatenate([r[2] for r in results]) if results else np.zeros(0, np.uint8)
    summaries = {i: r[0] for i, r in zip(mine, results)}
    if world > 1:
        g_idx = _gather_concat(idx, torch.int64, world, device)
        g_len = _gather_concat(lens, torch.int64, world, device)
        g_ttft = _gather_concat(ttft, torch.float64, world, device)
        g_flags = _gather_concat(flags, torch.uint8, world, device)
        objs = [None] * world
        dist.all_gather_object(objs, summaries)
        for o in objs:
            summaries.update(o)
    else:
        g_idx, g_len, g_ttft, g_flags = [idx], [lens], [ttft], [flags]

    if rank == 0:
        per_cell = {}
        for ids, ls, tt, fl in zip(g_idx, g_len, g_ttft, g_flags):
            off = 0
            for i, n in zip(ids.tolist(), ls.tolist()):
                per_cell[i] = (tt[off:off + n], fl[off:off + n])
                off += n
        assert sorted(per_cell) == list(range(len(cells))), "gather lost cells"
        os.makedirs(a.out, exist_ok=True)
        rows = [csv_header(bool(slos))]
        for i, cell in enumerate(cells):
            summary = summaries[i]
            tt, fl = per_cell[i]
            js = json.loads(summary)
            if len(fl):
                att = float(fl.sum()) / float(len(fl))
                if att != js["slo_attainment"]:
                    raise RuntimeError(f"cell {cell}: gathered SLO flags give {att}, "
                                       f"summary {js['slo_attainment']}")
            done = tt[~np.isnan(tt)]
            if done.size:  # metrics.cpp:56-58: sequential sum in request order
                mean = float(np.cumsum(done)[-1]) / float(done.size)
                if mean != js["ttft_mean_s"]:
                    raise RuntimeError(f"cell {cell}: gathered TTFTs give mean {mean!r}, "
                                       f"summary {js['ttft_mean_s']!r}")
            rows.append(csv_row(cell, summary))
        with open(os.path.join(a.out, "sweep.csv"), "w", newline="") as f:
            f.write("".join(rows))
        if not a.no_ttft_npz:
            np.savez_compressed(os.path.join(a.out, "ttft.npz"),
                                **{cell_key(c) + "/ttft": per_cell[i][0] for i, c in enumerate(cells)},
                                **{cell_key(c) + "/slo_met": per_cell[i][1] for i, c in enumerate(cells)})
        if len(cells) <= 1000:
            for c in cells:
                print("done " + cell_key(c))
        print(f"sweep: {len(cells)} cells on {world} rank(s), sweep.csv written", flush=True)
    if init_here:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
