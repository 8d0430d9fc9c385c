"""GPU tier: suspend / resume on the device is exact.

Event-budgeted (mfsim_dev_launch_budget) and time-sliced
(mfsim_dev_launch_slice) launches stop every instance mid-run, move its event
pool from shared memory back to HBM and its scalar state to sc_blob, and the
next launch stages both on chip again (engine_kernel.cu stage_instance,
engine.cuh begin/end). Golden cases with small pools (E_cap <= 64: the pool
lives on chip) and with the link-slot state on chip must still match the
fixtures bit for bit, for the one-warp kernel and the lock-step gang kernel."""
import os

import pytest

import cases
from parity import mismatches

pytestmark = pytest.mark.gpu

MANUAL = ["trio_mfs", "tick_promotion", "soft_enforcement_on", "egress_mfs", "random_000", "random_007"]
WORKLOAD = ["cluster8_400_mfs", "cluster8_400_karuna", "cluster8_400_fs", "fattree_edf", "c9_mfs"]


def _batch(product, gang):
    from paper_2603_17456_b200.native import DeviceBatch
    os.environ["MFSIM_GANG"] = str(gang)
    os.environ["MFSIM_GANG_MIN"] = "1"  # the gang kernel even for this small batch
    try:
        b = DeviceBatch(0, product)
    finally:
        os.environ.pop("MFSIM_GANG", None)
        os.environ.pop("MFSIM_GANG_MIN", None)
    man = [n for n in MANUAL if n in cases.manual_cases()]
    wl = [n for n in WORKLOAD if n in cases.workload_cases()]
    for n in man:
        b.add_manual(cases.manual_cases()[n])
    for n in wl:
        b.add_config(cases.workload_cases()[n])
    b.prepare()
    b.upload()
    b.reset()
    return b, [("manual", n) for n in man] + [("workload", n) for n in wl]


def _check(b, names):
    b.download(2)
    bad = {}
    for i, (grp, n) in enumerate(names):
        m = mismatches(b.result(i, 2, reports=True), grp, n)
        if m:
            bad[n] = m
    assert bad == {}


@pytest.mark.parametrize("gang", [1, 32])
def test_event_budget_launches(product, gang):
    b, names = _batch(product, gang)
    launches = 0
    while b.remaining() > 0:
        b.launch_budget(97)
        launches += 1
        assert launches < 100000
    assert launches > 3
    _check(b, names)


@pytest.mark.parametrize("gang", [1, 32])
def test_time_sliced_launches(product, gang):
    b, names = _batch(product, gang)
    launches = 0
    while b.remaining() > 0:
        b.launch_slice(2_000_000)  # 2 ms of device time per launch
        launches += 1
        assert launches < 100000
    assert launches > 3
    _check(b, names)
