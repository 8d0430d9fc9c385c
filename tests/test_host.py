"""Host side: config format, routing and workload synthesis reproduce the
reference's inputs exactly (config.cpp, topology.cpp, workload.cpp)."""
import numpy as np
import pytest

from paper_2603_17456_b200 import sweep
from paper_2603_17456_b200.native import Config, DeviceBatch, link_count, route


def test_star_routes(emu):
    # test_core.cpp:82-92: host h attaches via links 2h (up) and 2h+1 (down)
    cfg = "topology.kind = star\ntopology.hosts = 4\n"
    assert route(cfg, 0, 3, emu)[0] == [0, 7]
    assert route(cfg, 2, 1, emu)[0] == [4, 3]
    assert route(cfg, 1, 1, emu)[0] == []
    assert link_count(cfg, emu) == 8


def test_fattree_shape_and_lowest_id_routes(emu):
    # k=8 fat-tree for 128 hosts: 128*2 + 8*4*4*2 + 8*4*4*2 = 768 links
    cfg = sweep.text(sweep.FT128)
    assert link_count(cfg, emu) == 768
    links, caps = route(cfg, 0, 127, emu)
    assert len(links) == 6 and caps == [1.0] * 6
    # same edge switch: host -> edge -> host
    assert len(route(cfg, 0, 1, emu)[0]) == 2
    # k=2 fat-tree (test_core.cpp:94-121): inter-pod route traverses the core
    cfg2 = "topology.kind = fattree\ntopology.hosts = 2\n"
    assert len(route(cfg2, 0, 1, emu)[0]) == 6


def test_capacity_from_gbps_and_nics(emu):
    cfg = "topology.kind = star\ntopology.hosts = 2\ntopology.link_gbps = 100\ntopology.nics_per_host = 8\n"
    assert route(cfg, 0, 1, emu)[1] == [100e9 / 8 * 8] * 2


def test_arrivals_and_deadlines_match_reference(emu):
    """synthesis + derive_slos (batched isolated runs) reproduce the reference bit for bit"""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    for text in (open("tests/configs/cluster8.conf").read() + "workload.request_count = 150\n",
                 sweep.sweep_config((0.7, 2, 5, "mfs"), requests=60, lib=emu)):
        arr, dl = ref.derive_deadlines(text)
        b = DeviceBatch(0, emu)
        b.add_config(text)
        b.prepare()
        b.run(0)
        r = b.result(0, 0)
        assert np.array_equal(r.req_arrival.view(np.int64), arr.view(np.int64))
        assert np.array_equal(r.req_deadline.view(np.int64), dl.view(np.int64))


def test_sweep_grid():
    cells = sweep.sweep_cells()
    assert len(cells) == 7 * 5 * 64 * 5 == 11200
    assert len(set(cells)) == len(cells)


def test_load_mapping_monotone(emu):
    r = [sweep.rate_for_load(x, lib=emu) for x in sweep.LOADS]
    assert all(a < b for a, b in zip(r, r[1:]))
