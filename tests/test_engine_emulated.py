"""CPU tier: the engine source (csrc/device/engine.cuh) compiled as a serial
1-lane host build (TEST ONLY, build/libmfsim_emu.so) is bit-exact against the
golden fixtures. This checks engine logic without a GPU; the GPU tier runs the
same cases on the sm_100a product library."""
import pytest

import cases
from parity import manifest, mismatches
from paper_2603_17456_b200.native import MfsimError, run_config, run_manual


@pytest.mark.parametrize("name", sorted(cases.manual_cases()))
def test_manual_case(emu, name):
    res = run_manual(cases.manual_cases()[name], lib=emu)
    assert mismatches(res, "manual", name) == []


@pytest.mark.parametrize("name", sorted(cases.workload_cases()))
def test_workload_case(emu, name):
    res = run_config(cases.workload_cases()[name], lib=emu)
    assert mismatches(res, "workload", name) == []


def test_livelock_error_code(emu):
    with pytest.raises(MfsimError) as e:
        run_manual(cases.livelock(), lib=emu)
    assert e.value.code == manifest()["errors"]["livelock"]


GLOBAL_CASES = ["trio_karuna", "egress_mfs", "tick_promotion", "soft_enforcement_on", "random_004",
                "random_013", "rli_007"]


@pytest.mark.parametrize("name", GLOBAL_CASES)
def test_global_memory_variant_manual(emu, name, monkeypatch):
    """instances beyond the shared-memory plan take the generic engine variant"""
    monkeypatch.setenv("MFSIM_FORCE_GLOBAL", "1")
    res = run_manual(cases.manual_cases()[name], lib=emu)
    assert mismatches(res, "manual", name) == []


@pytest.mark.parametrize("name", ["example_karuna", "sanity_mfs", "fattree_sjf", "cluster8_400_edf"])
def test_global_memory_variant_workload(emu, name, monkeypatch):
    monkeypatch.setenv("MFSIM_FORCE_GLOBAL", "1")
    res = run_config(cases.workload_cases()[name], lib=emu)
    assert mismatches(res, "workload", name) == []


@pytest.mark.parametrize("name", ["cluster8_400_mfs", "fattree_karuna", "sanity_sjf", "example_fs"])
def test_slot_overflow_steps_fall_back(emu, name, monkeypatch):
    """steps whose links exceed the slot capacity take the per-link filling"""
    monkeypatch.setenv("MFSIM_SLOT_CAP", "6")
    res = run_config(cases.workload_cases()[name], lib=emu)
    assert mismatches(res, "workload", name) == []


@pytest.mark.parametrize("name", ["cluster8_400_mfs", "cluster8_400_karuna", "fattree_edf", "c9_mfs"])
def test_suspend_resume_is_exact(emu, name):
    """event-budgeted launches (suspend / resume through HBM) change nothing"""
    from paper_2603_17456_b200.native import DeviceBatch
    b = DeviceBatch(0, emu)
    b.add_config(cases.workload_cases()[name])
    b.prepare()
    b.upload()
    b.reset()
    launches = 0
    while b.remaining() > 0:
        b.launch_budget(61)
        launches += 1
    b.download(2)
    assert launches > 2
    assert mismatches(b.result(0, 2, reports=True), "workload", name) == []
