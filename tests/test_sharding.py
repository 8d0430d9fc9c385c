"""Multi-GPU layout on CPU: instance sharding across ranks (gloo, world 2).

bench.py gives every rank a disjoint slice of the sweep cells with no
collective on the data path; a final gather collects per-instance results.
Here two gloo ranks run their slices on the host emulation and the gathered
results must equal a single-rank run of the union."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, n, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2603_17456_b200 import sweep
    from paper_2603_17456_b200.native import DeviceBatch, Native
    emu = Native(os.path.join(ROOT, "build", "libmfsim_emu.so"))
    cells = bench.cells_for(rank, world, n)
    b = DeviceBatch(0, emu)
    for c in cells:
        b.add_config(sweep.sweep_config(c, requests=12, lib=emu))
    b.prepare()
    b.run(0)
    mine = [(c, b.stats(i).events, b.stats(i).slo_met) for i, c in enumerate(cells)]
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        out.put(gathered)
    dist.destroy_process_group()


def test_two_rank_sharding_matches_single_rank():
    if not os.path.exists(os.path.join(ROOT, "build", "libmfsim_emu.so")):
        pytest.skip("emulation library not built")
    import sys
    sys.path.insert(0, ROOT)
    import bench
    n = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    flat = [x for part in gathered for x in part]
    cells = [x[0] for x in flat]
    assert len(set(cells)) == 2 * n  # disjoint slices
    assert cells == bench.cells_for(0, 1, 2 * n)  # rank-major tiling of the grid
    from paper_2603_17456_b200 import sweep
    from paper_2603_17456_b200.native import DeviceBatch, Native
    emu = Native(os.path.join(ROOT, "build", "libmfsim_emu.so"))
    b = DeviceBatch(0, emu)
    for c in cells:
        b.add_config(sweep.sweep_config(c, requests=12, lib=emu))
    b.prepare()
    b.run(0)
    assert [(b.stats(i).events, b.stats(i).slo_met) for i in range(len(cells))] == \
        [(x[1], x[2]) for x in flat]


def test_cells_distinct_at_eight_ranks():
    """weak scaling never re-simulates a cell: 8 ranks x 4736 resident instances
    exceed the 11,200 cells of 64 seeds and continue with seeds 65, 66, ..."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    allr = [c for r in range(8) for c in bench.cells_for(r, 8, 4736)]
    assert len(allr) == len(set(allr)) == 8 * 4736
    assert bench.cells_for(0, 1, 4736) == bench.cells_for(0, 8, 4736)  # rank 0 is stable
    assert max(c[2] for c in allr) > 64
