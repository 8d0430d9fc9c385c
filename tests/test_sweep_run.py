"""The sharded sweep driver (paper_2603_17456_b200/sweep_run.py), the
reference's simsweep on N ranks with a final TTFT/SLO gather.

CPU tier: two gloo ranks run their LPT shares on the host emulation; rank 0's
sweep.csv must equal, byte for byte, the rows simsweep writes from the
reference's own summaries (oracle/_ref) for the same cells, and the gathered
per-request TTFTs must equal the reference's. GPU tier: the same on the
sm_100a library (single rank)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONF = os.path.join(ROOT, "tests", "configs", "cluster8.conf")
ARGS = ["--config", CONF, "--policies", "fs,mfs,karuna", "--rates", "6,12", "--seeds", "1,2"]
EXTRA = "workload.request_count = 40\n"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _conf(tmp):
    p = os.path.join(tmp, "c.conf")
    with open(p, "w") as f:
        f.write(open(CONF).read() + EXTRA)
    return p


def _rank_main(rank, world, port, argv):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_2603_17456_b200 import sweep_run
    from paper_2603_17456_b200.native import Native
    emu = Native(os.path.join(ROOT, "build", "libmfsim_emu.so"))
    sweep_run.main(argv, lib=emu, backend="gloo")


def _expected(conf):
    """simsweep's sweep.csv from the reference library's own summaries"""
    from oracle import ref
    from paper_2603_17456_b200 import sweep_run
    base = open(conf).read()
    rows, ttft = [sweep_run.CSV_HEADER], {}
    for cell in sweep_run.sweep_cells(["fs", "mfs", "karuna"], ["6", "12"], ["1", "2"]):
        p, r, s = cell
        res = ref.run_config(base + f"policy = {p}\nworkload.rate_rps = {r}\nsim.seed = {s}\n")
        rows.append(sweep_run.csv_row(cell, res.summary_json))
        ttft[f"{p}/rate_{r}/seed_{s}/ttft"] = np.asarray(res.req_done) - np.asarray(res.req_arrival)
    return "".join(rows), ttft


def _check(out, conf):
    from oracle import ref
    if not ref.available():
        pytest.skip("reference library (oracle/_ref) not built")
    want_csv, want_ttft = _expected(conf)
    assert open(os.path.join(out, "sweep.csv")).read() == want_csv
    got = np.load(os.path.join(out, "ttft.npz"))
    for k, v in want_ttft.items():
        assert np.array_equal(got[k], v, equal_nan=True), k
    # per-cell reports exist where mfsim_run would put them
    assert os.path.exists(os.path.join(out, "mfs", "rate_12", "seed_2", "requests.csv"))
    assert os.path.exists(os.path.join(out, "fs", "rate_6", "seed_1", "summary.json"))


def test_shard_is_lpt_and_disjoint():
    from paper_2603_17456_b200 import sweep_run
    cells = sweep_run.sweep_cells(["fs", "karuna", "mfs"], ["1", "2"], ["1", "2", "3"])
    own = sweep_run.shard(cells, 4)
    assert sorted(set(own)) == [0, 1, 2, 3]
    load = [0.0] * 4
    for c, r in zip(cells, own):
        load[r] += sweep_run.POLICY_COST[c[0]] * float(c[1])
    assert max(load) - min(load) <= 2 * 14.0  # within the largest cell
    assert sweep_run.shard(cells, 1) == [0] * len(cells)


def test_json_token_is_nlohmann_text():
    from paper_2603_17456_b200 import sweep_run
    s = '{\n  "slo_attainment": 0.5,\n  "ttft_p99_s": null,\n  "pruned_count": 3\n}'
    assert sweep_run.json_token(s, "slo_attainment") == "0.5"
    assert sweep_run.json_token(s, "ttft_p99_s") == ""
    assert sweep_run.json_token(s, "pruned_count") == "3"


def test_two_rank_sweep_matches_reference_simsweep(tmp_path):
    if not os.path.exists(os.path.join(ROOT, "build", "libmfsim_emu.so")):
        pytest.skip("emulation library not built")
    conf = _conf(str(tmp_path))
    out = str(tmp_path / "out")
    argv = ARGS[:]
    argv[1] = conf
    argv += ["--out", out]
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, argv)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    _check(out, conf)


@pytest.mark.gpu
def test_sweep_on_device_matches_reference_simsweep(tmp_path):
    from paper_2603_17456_b200 import sweep_run
    conf = _conf(str(tmp_path))
    out = str(tmp_path / "out")
    argv = ARGS[:]
    argv[1] = conf
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        os.environ.pop(k, None)
    sweep_run.main(argv + ["--out", out])
    _check(out, conf)


def _slo_axis_and_loads(tmp_path, lib):
    """SLO-multiplier and offered-load axes (configs[3]'s grid) with batch
    chunking: every row equals the reference run of the same cell"""
    from oracle import ref
    if not ref.available():
        pytest.skip("reference library (oracle/_ref) not built")
    from paper_2603_17456_b200 import sweep, sweep_run
    from paper_2603_17456_b200.native import product
    conf = _conf(str(tmp_path))
    out = str(tmp_path / "o")
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        os.environ.pop(k, None)
    sweep_run.main(["--config", conf, "--policies", "fs,mfs", "--loads", "0.4,0.8",
                    "--seeds", "3", "--slo-multipliers", "1,4", "--batch-cap", "3",
                    "--no-reports", "--out", out], lib=lib, backend="gloo" if lib else None)
    base = open(conf).read()
    rl = lib or product()
    rates = [repr(sweep.rate_for_load(x, sweep_run.parse_config_text(base), rl)) for x in (0.4, 0.8)]
    cells = sweep_run.sweep_cells(["fs", "mfs"], rates, ["3"], ["1", "4"])
    rows = [sweep_run.csv_header(True)]
    got = np.load(os.path.join(out, "ttft.npz"))
    for c in cells:
        res = ref.run_config(base + f"policy = {c[0]}\nworkload.rate_rps = {c[1]}\n"
                                    f"sim.seed = {c[2]}\nworkload.slo_multiplier = {c[3]}\n")
        rows.append(sweep_run.csv_row(c, res.summary_json))
        want = np.asarray(res.req_done) - np.asarray(res.req_arrival)
        assert np.array_equal(got[sweep_run.cell_key(c) + "/ttft"], want, equal_nan=True)
    assert rows[0].startswith("policy,rate_rps,seed,slo_multiplier,slo_attainment")
    assert open(os.path.join(out, "sweep.csv")).read() == "".join(rows)
    # the SLO multiplier changes attainment somewhere in the grid
    assert len({r.split(",")[4] for r in rows[1:]}) > 1


def test_slo_axis_and_loads_on_emulation(tmp_path):
    from paper_2603_17456_b200.native import Native
    emu = Native(os.path.join(ROOT, "build", "libmfsim_emu.so"))
    _slo_axis_and_loads(tmp_path, emu)


@pytest.mark.gpu
def test_slo_axis_and_loads_on_device(tmp_path):
    _slo_axis_and_loads(tmp_path, None)
