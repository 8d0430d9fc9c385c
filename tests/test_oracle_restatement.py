"""The plain-C restatement oracle (oracle/mfsim_oracle.c, built into
oracle/_ref/libmfsim_oracle.so) is pinned against the golden fixtures the
reference itself produced: every manual scenario and every workload case,
bit for bit. It is test infrastructure and the `port` CPU baseline; the
product never calls it."""
import pytest

import cases
from parity import manifest, mismatches
from oracle import ref

pytestmark = pytest.mark.skipif(not ref.available(ref.ORACLE_SO), reason="oracle not built")


@pytest.mark.parametrize("name", sorted(cases.manual_cases()))
def test_manual(name):
    assert mismatches(ref.run_manual(cases.manual_cases()[name], so=ref.ORACLE_SO), "manual", name) == []


@pytest.mark.parametrize("name", sorted(cases.workload_cases()))
def test_workload(name):
    assert mismatches(ref.run_config(cases.workload_cases()[name], so=ref.ORACLE_SO), "workload", name) == []


def test_livelock_code():
    with pytest.raises(ref.RefError) as e:
        ref.run_manual(cases.livelock(), so=ref.ORACLE_SO)
    assert e.value.code == manifest()["errors"]["livelock"]
