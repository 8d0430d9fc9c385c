"""GPU tier: the sm_100a engine (paper_2603_17456_b200/libmfsim_b200.so) is
bit-exact against the reference on every golden case -- RMLQ bands/levels,
completion times (flow order), per-request done/SLO flags, stalls, event and
step counts, and byte-identical summary.json / requests.csv."""
import os

import numpy as np
import pytest

import cases
from parity import manifest, mismatches

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def manual_batch(product):
    """every manual case in ONE launch (one warp each)"""
    from paper_2603_17456_b200.native import DeviceBatch
    names = sorted(cases.manual_cases())
    b = DeviceBatch(0, product)
    for n in names:
        b.add_manual(cases.manual_cases()[n])
    b.prepare()
    b.run(2)
    return names, b


def test_manual_cases_batched(manual_batch):
    names, b = manual_batch
    bad = {}
    for i, n in enumerate(names):
        r = b.result(i, 2, reports=True)
        m = mismatches(r, "manual", n)
        if m:
            bad[n] = m
    assert bad == {}


@pytest.fixture(scope="module")
def workload_batch(product):
    from paper_2603_17456_b200.native import DeviceBatch
    wc = cases.workload_cases(big=True)
    names = sorted(wc)
    b = DeviceBatch(0, product)
    for n in names:
        b.add_config(wc[n])
    b.prepare()
    b.run(2)
    return names, b


def test_workload_cases_batched(workload_batch):
    names, b = workload_batch
    bad = {}
    for i, n in enumerate(names):
        r = b.result(i, 2, reports=True)
        m = mismatches(r, "workload", n)
        if m:
            bad[n] = m
    assert bad == {}


@pytest.mark.parametrize("name", ["trio_mfs", "tick_promotion", "soft_enforcement_on", "egress_mfs"])
def test_single_instance_launch(product, name):
    from paper_2603_17456_b200.native import run_manual
    assert mismatches(run_manual(cases.manual_cases()[name], lib=product), "manual", name) == []


def test_livelock_error(product):
    from paper_2603_17456_b200.native import MfsimError, run_manual
    with pytest.raises(MfsimError) as e:
        run_manual(cases.livelock(), lib=product)
    assert e.value.code == 5


def test_mfsim_run_c_abi(product, tmp_path):
    from paper_2603_17456_b200.native import mfsim_run
    s = mfsim_run(cases.workload_cases()["c9_mfs"], out_dir=str(tmp_path), lib=product)
    assert s == manifest()["workload"]["c9_mfs"]["summary_json"]
    assert open(tmp_path / "summary.json").read() == s


def test_full_size_sweep_instances(product):
    """BASELINE configs[3] instance size (2000 requests, ft128): determinism across
    launches and batch composition, conservation, and exact agreement with the
    reference when the reference library is present on this box"""
    from paper_2603_17456_b200 import sweep
    from paper_2603_17456_b200.native import DeviceBatch
    cells = [(0.9, 3, 1, "mfs"), (0.9, 3, 1, "fs"), (0.6, 1, 2, "sjf"), (0.8, 5, 3, "edf")]
    texts = [sweep.sweep_config(c, lib=product) for c in cells]
    b = DeviceBatch(0, product)
    for t in texts:
        b.add_config(t)
    b.prepare()
    b.run(2)
    first = [b.result(i, 2) for i in range(len(texts))]
    b.launch()
    b.sync()
    b.download(2)
    for i, r in enumerate(first):
        again = b.result(i, 2)
        assert np.array_equal(r.flow_finish, again.flow_finish)
        assert r.events == again.events and r.status == 0
        assert len(r.req_done) == 2000
        fin = r.flow_finish
        assert np.all(fin[fin >= 0] <= np.nanmax(r.req_done) + 1e-9)
    from oracle import ref
    if ref.available():
        for i in (0, 1):
            rr = ref.run_config(texts[i])
            assert rr.events == first[i].events
            assert np.array_equal(np.nan_to_num(rr.req_done, nan=-7).view(np.int64),
                                  np.nan_to_num(first[i].req_done, nan=-7).view(np.int64))
            assert np.array_equal(rr.flow_finish.view(np.int64), first[i].flow_finish.view(np.int64))
            assert rr.attainment == first[i].attainment
