"""Oracle extensions: behaviour the reference cannot
express, so parity is anchored on the plain-C restatement (oracle/mfsim_oracle.c)
extended the same way, and on the reference itself wherever the extension is
switched off.

  topology.oversubscription = o  (fat-tree): every switch-to-switch link
      (edge-agg, agg-core) carries capacity / o; host links keep capacity.
      o = 1 (or absent) is the reference's uniform fabric.
"""
import os

import numpy as np
import pytest

import cases
from parity import ARRAYS, SCALARS, bits_equal, mismatches
from oracle import ref

POLICIES = ("fs", "sjf", "edf", "karuna", "mfs")
needs_oracle = pytest.mark.skipif(not ref.available(ref.ORACLE_SO), reason="oracle not built")


def diff(a, b):
    bad = [k for k in SCALARS if int(getattr(a, k)) != int(getattr(b, k))]
    bad += [k for k in ARRAYS if not bits_equal(getattr(a, k), getattr(b, k))]
    if getattr(a, "summary_json", None) and getattr(b, "summary_json", None) \
            and a.summary_json != b.summary_json:
        bad.append("summary.json bytes")
    return bad


def oversub_fattree(policy: str, o: float) -> str:
    return cases.fattree_config(policy) + f"topology.oversubscription = {o}\n"


def oversub_ft128(policy: str, o: float, requests: int = 150) -> str:
    from paper_2603_17456_b200 import sweep
    d = dict(sweep.FT128, **{"policy": policy, "workload.request_count": requests,
                             "topology.oversubscription": o, "workload.rate_rps": 0.5})
    return sweep.text(d)


def test_oversub_link_capacities(emu):
    from paper_2603_17456_b200.native import Config, route
    cfg = Config(oversub_fattree("fs", 4), emu)
    links, caps = route(cfg, 0, 11, emu)  # crosses pods: host, edge-agg, agg-core, ..., host
    assert len(links) == 6
    assert caps[0] == 800.0 and caps[-1] == 800.0
    assert all(c == 200.0 for c in caps[1:-1])


def test_oversub_rejected_on_star(emu):
    from paper_2603_17456_b200.native import Config, DeviceBatch, MfsimError
    b = DeviceBatch(0, emu)
    with pytest.raises(MfsimError):
        b.add_config(Config(cases.sanity_config("fs") + "topology.oversubscription = 2\n", emu))
        b.prepare()


@needs_oracle
@pytest.mark.parametrize("policy", POLICIES)
def test_oversub_one_is_the_reference(policy):
    """o = 1 reproduces the reference's own fixture bit for bit"""
    r = ref.run_config(oversub_fattree(policy, 1), so=ref.ORACLE_SO)
    assert mismatches(r, "workload", f"fattree_{policy}") == []


@needs_oracle
@pytest.mark.parametrize("policy", POLICIES)
def test_oversub_host_engine_matches_oracle(emu, policy):
    from paper_2603_17456_b200.native import run_config
    text = oversub_fattree(policy, 2.5)
    want = ref.run_config(text, so=ref.ORACLE_SO)
    got = run_config(text, lib=emu)
    assert diff(got, want) == []
    # the extension changes the outcome (it is not a no-op)
    base = ref.run_config(oversub_fattree(policy, 1), so=ref.ORACLE_SO)
    assert not bits_equal(base.flow_finish, want.flow_finish)


@pytest.mark.gpu
def test_oversub_device_matches_oracle(product):
    from paper_2603_17456_b200.native import DeviceBatch
    texts = [oversub_fattree(p, 2.5) for p in POLICIES] + [oversub_ft128(p, 2.0) for p in POLICIES]
    b = DeviceBatch(0, product)
    for t in texts:
        b.add_config(t)
    b.prepare()
    b.run(2)
    bad = {}
    for i, t in enumerate(texts):
        d = diff(b.result(i, 2, reports=True), ref.run_config(t, so=ref.ORACLE_SO))
        if d:
            bad[i] = d
    assert bad == {}
