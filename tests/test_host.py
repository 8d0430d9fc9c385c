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


def test_deadline_cache_buckets_reuse_fraction(emu, tmp_path):
    """derive_slos keys its cache on llround(reuse_fraction * 1e9) (workload.cpp:203-205):
    a request whose fraction differs from an earlier one only below 1e-9 reuses that
    request's isolated TTFT, so its deadline is NOT its own probe's"""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    units = 8
    rows = ["arrival_s,prompt_tokens,reuse_fraction,source_unit"]
    fr = [0.3, 0.3 + 3e-12, 0.3 - 4e-11, 0.5, 0.5 + 2e-10, 0.3 + 6e-10]
    for k, f in enumerate(fr):  # request k * units lands on unit 0 (round robin)
        for u in range(units):
            rows.append(f"{(k * units + u) * 0.05:.9f},1500,{f if u == 0 else 0.25!r},{(u + 1) % units}")
    trace = tmp_path / "near.csv"
    trace.write_text("\n".join(rows) + "\n")
    text = open("tests/configs/cluster8.conf").read() + f"workload.trace = {trace}\npolicy = mfs\n"
    arr, dl = ref.derive_deadlines(text)
    b = DeviceBatch(0, emu)
    b.add_config(text)
    b.add_config(text + "policy = fs\n")  # cross-instance probe sharing
    b.prepare()
    b.run(0)
    for i in range(2):
        r = b.result(i, 0)
        assert np.array_equal(r.req_arrival.view(np.int64), arr.view(np.int64))
        assert np.array_equal(r.req_deadline.view(np.int64), dl.view(np.int64))


def test_load_model_uses_library_defaults(emu):
    """a base config that omits keys gets the simulator's defaults (config.cpp), not a KeyError"""
    base = {k: v for k, v in sweep.FT128.items()
            if k not in ("model.coll_bytes_per_token_layer", "model.layers", "workload.reuse_skew")}
    full = dict(base, **{"model.coll_bytes_per_token_layer": 250.0, "model.layers": 4,
                         "workload.reuse_skew": 1.0})
    assert sweep.busiest_link_bytes(base, lib=emu) == sweep.busiest_link_bytes(full, lib=emu)


def test_sweep_grid():
    cells = sweep.sweep_cells()
    assert len(cells) == 7 * 5 * 64 * 5 == 11200
    assert len(set(cells)) == len(cells)


def test_load_mapping_monotone(emu):
    r = [sweep.rate_for_load(x, lib=emu) for x in sweep.LOADS]
    assert all(a < b for a, b in zip(r, r[1:]))
