#!/usr/bin/env python3
"""Throughput benchmark: simulated flow-events/sec of the B200 engine.

Workload (BASELINE.json configs[3]): the batched sweep on the ft128 fabric
("1024 GPUs" = 128 hosts x 8 NICs, k=8 fat-tree), 2000 requests per instance,
cells = offered load x SLO multiplier x seed x policy. S full-size instances
of that grid are resident per rank (weak scaling: S fixed per GPU; ranks take
disjoint cells; no collective on the data path). A step = one device launch
in which every warp advances its instance for `--slice-ms` of device time and
then suspends it to HBM (resumed exactly by the next launch), so every step is
steady-state work over the whole mix; the warm-up launches start the
instances. Events per step are measured from the device counters. flow-events = RunResult::events
(engine.cpp:611), summed over instances.

  value : events / device time of the timed launches (inputs resident in HBM,
          CUDA events on the launch stream, max over ranks)
  e2e   : same metric through the C ABI with host buffers: H2D of the inputs,
          launch, D2H of per-request results, every step
  --impl reference : the reference CPU simulator (oracle/_ref, unmodified
          sources) on all host cores, same cells, bounded sample per step
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

PEAKS = os.path.join(HERE, "MEASURED_PEAKS.json")
HBM_FALLBACK = 6650.0
NCU_SUMMARY = os.path.join(HERE, "profiles", "r02_ncu_gang_summary.json")


def ncu_traffic(events_per_launch: float):
    """DRAM bytes per launch of the engine kernel from the committed ncu --set full
    capture (dram__bytes_read.sum + dram__bytes_write.sum), scaled from the
    captured launch to this run's launch by simulated events (bytes per event)."""
    try:
        s = json.load(open(NCU_SUMMARY))
        return s["dram_bytes_per_event"] * events_per_launch, os.path.relpath(NCU_SUMMARY, HERE)
    except Exception:
        return None, None


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--instances", type=int, default=int(os.environ.get("MFSIM_BENCH_INSTANCES", 0)),
                    help="resident instances per rank (0: WARPS_PER_SM x SMs, bounded by free HBM)")
    ap.add_argument("--slice-ms", type=float, default=1000.0,
                    help="device time per step (launch): every warp advances its instance until then")
    ap.add_argument("--requests", type=int, default=2000, help="requests per instance (configs[3]: 2000)")
    ap.add_argument("--cpu-sample-s", type=float, default=30.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index: int):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=6)

    def summary(self):
        rows = [s for s in self.samples if len(s) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no-samples"]}
        load = [r for r in rows if r[7].isdigit() and int(r[7]) > 0] or rows
        sm = sorted(float(r[0]) for r in load)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(load)}


WARPS_PER_SM = 32          # resident instances per SM (registers and the shared-memory plan allow 32)
INSTANCE_BYTES = 38.0e6    # device arena of one configs[3] instance (measured 37.3 MB)


def resident_instances(device: int) -> int:
    """one warp-resident instance per warp slot, as many as free HBM holds"""
    import torch
    props = torch.cuda.get_device_properties(device)
    free, _ = torch.cuda.mem_get_info(device)
    by_mem = int((free - 8e9) / INSTANCE_BYTES)
    return max(148, min(WARPS_PER_SM * props.multi_processor_count, by_mem))


def cells_for(rank: int, world: int, n: int, step_offset: int = 0):
    """rank's slice of the sweep: consecutive chunks of the 11,200 cells ordered
    seed-major, the 175 (load, SLO scale, policy) cells of one seed in a fixed
    shuffle. A rank's instances thus mix loads, SLO scales and policies over a
    few seeds, and share those seeds' isolated-latency probes (derive_slos
    depends on the seed's requests only, not on the load, SLO scale or policy)."""
    import random

    from paper_2603_17456_b200 import sweep

    # 64 seeds = 11,200 cells; runs that need more distinct instances (weak
    # scaling to 8 GPUs x ~4k resident instances) continue with seeds 65, 66, ...
    # instead of re-simulating cells
    need = (step_offset * world + world) * n
    per_seed = len(sweep.LOADS) * len(sweep.SLO_SCALES) * len(sweep.POLICIES)
    seeds = max(64, -(-need // per_seed))
    allc = sweep.sweep_cells(seeds=range(1, seeds + 1))
    rng = random.Random(2603)
    blocks = {}
    for c in allc:
        blocks.setdefault(c[2], []).append(c)
    allc = []
    for seed in sorted(blocks):
        b = blocks[seed]
        rng.shuffle(b)
        allc.extend(b)
    start = ((step_offset * world + rank) * n) % len(allc)
    return [allc[(start + i) % len(allc)] for i in range(n)]


def cpu_reference(cells, requests, budget_s, lib_cfg):
    """The reference simulator on all host cores (thread pool; the harness releases
    the GIL), full instances run to completion. Reported rate = events divided by
    the per-instance Engine::run times packed onto the cores (sum / cores), i.e.
    the all-cores-busy rate -- it ignores the idle tail of a finite sample, which
    favours the reference."""
    from oracle import ref

    cores = os.cpu_count() or 1
    texts = [lib_cfg(c) for c in cells]
    t0 = time.perf_counter()
    events, done, run_s = 0, 0, 0.0
    with cf.ThreadPoolExecutor(max_workers=cores) as ex:
        futs, it = set(), iter(texts)
        for _ in range(cores):
            t = next(it, None)
            if t is not None:
                futs.add(ex.submit(ref.run_config, t))
        while futs:
            fin, futs = cf.wait(futs, return_when=cf.FIRST_COMPLETED)
            for f in fin:
                r = f.result()
                events += r.events
                run_s += r.t_run_s
                done += 1
                if time.perf_counter() - t0 < budget_s:
                    t = next(it, None)
                    if t is not None:
                        futs.add(ex.submit(ref.run_config, t))
    wall = time.perf_counter() - t0
    packed = events / (run_s / cores) if run_s > 0 else 0.0
    return {"events": events, "wall_s": wall, "instances": done, "cores": cores,
            "engine_run_s": run_s, "rate_packed": packed, "rate_wall": events / wall}


def reference_arm(args, rank, world):
    if rank != 0:
        return
    if args.instances <= 0:
        args.instances = WARPS_PER_SM * 148
    from paper_2603_17456_b200 import sweep

    def cfg_text(c):
        return sweep_text(c, args.requests)

    def sweep_text(c, n):
        return sweep.sweep_config(c, requests=n, lib=_emu_or_product())

    cells = cells_for(0, 1, args.instances if args.instances > 0 else WARPS_PER_SM * 148)
    # one bounded sample of the same cells, shared by the K steps: instances are
    # submitted for ~cpu_sample_s seconds and run to completion on all cores
    r = cpu_reference(cells, args.requests, args.cpu_sample_s, cfg_text)
    value = r["rate_packed"]
    wall = r["wall_s"]
    line = {
        "impl": "reference", "metric": "simulated flow-events/sec", "value": value,
        "unit": "events/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * wall, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args),
        "cpu_baseline": {"value": value, "unit": "events/s", "cores": r["cores"], "kind": "reference",
                         "sample": f"{r['instances']} sweep instances ({args.requests} requests each, "
                                   f"run to completion) on {r['cores']} host threads; rate = events / "
                                   f"(sum of Engine::run times / cores); wall-clock rate "
                                   f"{r['rate_wall']:.0f} events/s"},
        "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


_emu = None


def _emu_or_product():
    """route computation only needs the host side of the library"""
    global _emu
    if _emu is None:
        from paper_2603_17456_b200.native import Native, PRODUCT_SO
        path = PRODUCT_SO if os.path.exists(PRODUCT_SO) else os.path.join(HERE, "build", "libmfsim_emu.so")
        _emu = Native(path)
    return _emu


def workload_config(args):
    return {
        "workload": "configs[3] sweep: ft128 fat-tree (128 hosts x 8 NICs, k=8, 768 links), "
                    "16 units x 4 hosts + 64 decode, cells = load {0.3..0.9} x SLO {1..5} x "
                    "seed {1..64} x policy {fs,sjf,edf,karuna,mfs} (seeds 65.. when ranks x resident "
                    "instances exceed the 11,200 cells: every instance distinct)",
        "instances_per_rank": args.instances,
        "step": f"one launch = {args.slice_ms:g} ms of device time per warp (time-sliced, "
                "instances suspend to HBM and resume exactly)",
        "requests_per_instance": args.requests,
        "l2": "inputs larger than L2 (per-step working set >> 126 MB)",
        "parallelism": f"instance-sharded x{args.gpus}",
    }


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return

    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2603_17456_b200 import sweep
    from paper_2603_17456_b200.native import DeviceBatch, product

    lib = product()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    if args.instances <= 0:
        args.instances = resident_instances(local)
    cells = cells_for(rank, world, args.instances)
    t0 = time.perf_counter()
    batch = DeviceBatch(local, lib, stream=stream.cuda_stream)
    for c in cells:
        batch.add_config(sweep.sweep_config(c, requests=args.requests, lib=lib))
    batch.prepare()  # workload synthesis + batched derive_slos (device)
    batch.upload()   # inputs resident in HBM; instances at their initial state
    setup_s = time.perf_counter() - t0
    n = len(batch)

    def progress():
        batch.download(0)
        return (sum(batch.stats(i).events for i in range(n)),
                sum(batch.stats(i).algo_bytes for i in range(n)))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up: the first budgeted launches start every instance
    for _ in range(args.warmup):
        batch.launch_slice(int(args.slice_ms * 1e6))
    barrier()
    ev0, by0 = progress()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    launches0 = batch.kernel_launches
    with Clocks(local) as clk:
        start.record(stream)
        for _ in range(args.steps):
            batch.launch_slice(int(args.slice_ms * 1e6))
        end.record(stream)
        barrier()
    launches = batch.kernel_launches - launches0
    dev_ms = start.elapsed_time(end)
    ev1, by1 = progress()
    events, algo_bytes = ev1 - ev0, by1 - by0
    # e2e through the C ABI: H2D of the inputs, launch, D2H of per-request results
    barrier()
    e0 = time.perf_counter()
    for _ in range(args.steps):
        batch.upload_inputs()
        batch.launch_slice(int(args.slice_ms * 1e6))
        batch.download(0)
    barrier()
    e2e_s = time.perf_counter() - e0
    ev2, _ = progress()
    e2e_events = ev2 - ev1
    h2d, d2h = batch.h2d_bytes, batch.d2h_bytes

    t = torch.tensor([dev_ms, e2e_s, float(events), float(e2e_events), float(algo_bytes)],
                     dtype=torch.float64, device="cuda")
    if world > 1:
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        dev_ms, e2e_s = mx[0].item(), mx[1].item()
        events, e2e_events = sm[2].item(), sm[3].item()
    value = events / (dev_ms / 1000.0)
    e2e = e2e_events / e2e_s
    kernel_ms = dev_ms / args.steps
    achieved = algo_bytes / (dev_ms / 1000.0) / 1e9  # rank 0's launches
    traffic, traffic_src = ncu_traffic(events / world / args.steps)
    try:
        peaks = json.load(open(PEAKS))
        peak, peak_src = float(peaks["hbm_gbs"]), "measured"
    except Exception:
        peak, peak_src = HBM_FALLBACK, "fallback"

    if rank == 0:
        line = {
            "metric": "simulated flow-events/sec", "value": value, "unit": "events/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": kernel_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args),
            "e2e": {"value": e2e, "unit": "events/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": batch.last_kernel,
                         "algo_bytes_per_launch": algo_bytes / args.steps,
                         "traffic_source": traffic_src},
            "clocks": clk.summary(),
            "events_per_step": events / args.steps,
            "setup_s_rank0": setup_s,
            "device_bytes_rank0": batch.device_bytes,
        }
        if not args.no_cpu_baseline:
            def cfg_text(c):
                return sweep.sweep_config(c, requests=args.requests, lib=lib)
            try:
                r = cpu_reference(cells, args.requests, args.cpu_sample_s, cfg_text)
                line["cpu_baseline"] = {
                    "value": r["rate_packed"], "unit": "events/s", "cores": r["cores"],
                    "kind": "reference",
                    "sample": f"{r['instances']} sweep instances ({args.requests} requests each, run to "
                              f"completion) on {r['cores']} host threads; rate = events / (sum of "
                              f"Engine::run times / cores); wall-clock rate {r['rate_wall']:.0f} events/s"}
            except Exception as e:  # the oracle library is absent: report why
                line["cpu_baseline"] = {"value": None, "unit": "events/s", "cores": 0,
                                        "kind": "reference", "sample": f"unavailable: {e}"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
