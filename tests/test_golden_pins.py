"""The golden fixtures (generated from the reference itself, tests/golden/make_golden.py)
agree with every known answer the reference's own tests state for this path."""
import numpy as np
import pytest

from parity import arrays, manifest


def A(group, name, key):
    return arrays(group)[f"{name}/{key}"]


def test_trio_known_answers():
    # test_engine.cpp:14-46 / acceptance C1: flow order A, B, C
    assert A("manual", "trio_mfs", "flow_finish").tolist() == [9.0, 4.0, 7.0]
    assert A("manual", "trio_fs", "flow_finish").tolist() == [6.0, 9.0, 8.0]
    assert A("manual", "trio_sjf", "flow_finish").tolist() == [2.0, 9.0, 5.0]
    assert A("manual", "trio_edf", "flow_finish").tolist() == [9.0, 7.0, 3.0]


def test_ingress_known_answers():
    # test_engine.cpp:48-72: fair sharing finishes both at 3; mfs serves the collective first
    assert A("manual", "ingress_fs", "flow_finish").tolist() == [3.0, 3.0]
    assert A("manual", "ingress_mfs", "flow_finish")[1] == 2.0


def test_egress_known_answers():
    # test_engine.cpp:55-65: layer-2 collective done 3 (mfs) / 4 (baselines), stall 1 / 2
    assert A("manual", "egress_mfs", "cof_done").tolist() == [3.0]
    assert A("manual", "egress_mfs", "req_stall").tolist() == [1.0]
    assert A("manual", "egress_mfs", "flow_finish")[0] == 4.0
    for p in ("fs", "sjf", "edf"):
        assert A("manual", f"egress_{p}", "cof_done").tolist() == [4.0]
        assert A("manual", f"egress_{p}", "req_stall").tolist() == [2.0]


def test_single_request_and_stall():
    assert A("manual", "single_request", "req_done").tolist() == [2.0]  # test_engine.cpp:74-92
    assert A("manual", "stall_zero", "cof_stall").tolist() == [0.0]      # test_engine.cpp:105-126
    assert A("manual", "stall_zero", "req_stall").tolist() == [0.0]


def test_tick_cases():
    m = manifest()["manual"]
    assert A("manual", "ticks", "req_done").tolist() == [3.0]            # test_engine.cpp:128-151
    assert m["ticks"]["events"] < 30
    fin = A("manual", "tick_promotion", "flow_finish")                   # test_engine.cpp:212-240
    assert abs(fin[1] - 3.2) < 1e-9 and abs(fin[0] - 33.0) < 1e-9
    assert A("manual", "tick_promotion", "flow_band")[1] == 0           # Band::UrgentP2D


def test_soft_enforcement():
    m = manifest()["manual"]                                            # test_engine.cpp:242-291
    assert m["soft_enforcement_on"]["pruned_count"] == 1
    assert A("manual", "soft_enforcement_on", "req_pruned").tolist() == [0, 0, 1]
    fin = A("manual", "soft_enforcement_on", "flow_finish")
    assert fin.tolist() == [2.0, 4.0, 13.0]
    assert A("manual", "soft_enforcement_on", "req_done")[2] <= 13.5
    assert m["soft_enforcement_off"]["pruned_count"] == 0


def test_livelock_is_a_sim_error():
    assert manifest()["errors"]["livelock"] == 5  # SimError (test_engine.cpp:153-172)


def test_workload_slo_flag_definition():
    # metrics.cpp:32-40 -- attainment in the manifest equals the flag recomputed
    for name in ("example_mfs", "cluster8_400_fs"):
        done = A("workload", name, "req_done")
        arr = A("workload", name, "req_arrival")
        dl = A("workload", name, "req_deadline")
        ok = ~np.isnan(done)
        met = np.zeros(done.shape, bool)
        met[ok] = (done[ok] - arr[ok]) <= (dl[ok] - arr[ok])
        assert met.mean() == manifest()["workload"][name]["attainment"]


def test_fixtures_match_live_reference():
    """When the reference library is present, the fixtures are still what it produces."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    import cases
    from parity import mismatches
    for name in ("trio_mfs", "egress_fs", "tick_promotion", "random_003"):
        assert mismatches(ref.run_manual(cases.manual_cases()[name]), "manual", name) == []
    assert mismatches(ref.run_config(cases.workload_cases()["example_mfs"]), "workload", "example_mfs") == []
