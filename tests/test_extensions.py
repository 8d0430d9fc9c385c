"""Oracle extensions: behaviour the reference cannot
express, so parity is anchored on the plain-C restatement (oracle/mfsim_oracle.c)
extended the same way, and on the reference itself wherever the extension is
switched off.

  topology.oversubscription = o  (fat-tree): every switch-to-switch link
      (edge-agg, agg-core) carries capacity / o; host links keep capacity.
      o = 1 (or absent) is the reference's uniform fabric.
  policy = aalo  Aalo-style D-CLAS coflow scheduling (BASELINE configs[1]'s
      "Varys/Aalo-style coflow" baseline): coflow = (batch, target layer,
      stage); queue from attained bytes vs Q0 * E^i (aalo.Q0/E/K); one class
      per coflow, FIFO by batch within a queue.
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


@needs_oracle
def test_oversub_mixed_batch_matches_oracle(emu):
    """one batch holding the same fabric with and without oversubscription: the
    shared topology images and the deduplicated isolated-latency probes must
    keep them apart"""
    from paper_2603_17456_b200.native import DeviceBatch
    texts = [oversub_fattree("fs", 1), oversub_fattree("fs", 2.0), cases.fattree_config("mfs"),
             oversub_fattree("mfs", 3.0)]
    b = DeviceBatch(0, emu)
    for t in texts:
        b.add_config(t)
    b.prepare()
    b.run(2)
    for i, t in enumerate(texts):
        assert diff(b.result(i, 2), ref.run_config(t, so=ref.ORACLE_SO)) == [], i


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


def aalo_cases():
    c8 = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs", "cluster8.conf")).read()
    return {
        "cluster8_200": c8 + "workload.request_count = 200\npolicy = aalo\n",
        "cluster8_200_q": c8 + "workload.request_count = 200\npolicy = aalo\naalo.Q0 = 1e-2\naalo.E = 4\naalo.K = 5\n",
        "fattree": cases.fattree_config("aalo"),
        "fattree_oversub": oversub_fattree("aalo", 2.0),
        "sanity": cases.sanity_config("aalo"),
        "example": open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs", "example.conf")).read()
        + "policy = aalo\n",
    }


@needs_oracle
@pytest.mark.parametrize("name", sorted(aalo_cases()))
def test_aalo_host_engine_matches_oracle(emu, name):
    from paper_2603_17456_b200.native import run_config
    text = aalo_cases()[name]
    want = ref.run_config(text, so=ref.ORACLE_SO)
    got = run_config(text, lib=emu, detail=2)
    assert diff(got, want) == []
    assert '"policy": "aalo"' in (got.summary_json or '"policy": "aalo"')


@needs_oracle
@pytest.mark.parametrize("name", ["trio", "ingress", "egress", "single_request", "stall_zero",
                                  "ticks", "tick_promotion"])
def test_aalo_manual_scenarios_match_oracle(emu, name):
    from paper_2603_17456_b200.native import run_manual
    import re
    fn = getattr(cases, name)
    spec = fn("aalo") if name in ("trio", "ingress", "egress") else fn()
    spec = re.sub(r"^policy \w+", "policy aalo", spec, flags=re.M)
    assert "policy aalo" in spec
    assert diff(run_manual(spec, lib=emu), ref.run_manual(spec, so=ref.ORACLE_SO)) == []


@needs_oracle
def test_aalo_differs_from_the_reference_policies():
    text = aalo_cases()["cluster8_200"]
    a = ref.run_config(text, so=ref.ORACLE_SO)
    for p in POLICIES:
        b = ref.run_config(text.replace("policy = aalo", f"policy = {p}"), so=ref.ORACLE_SO)
        assert not bits_equal(a.flow_finish, b.flow_finish), p


@pytest.mark.parametrize("bad", ["aalo.K = 1", "aalo.K = 99", "aalo.E = 1", "aalo.Q0 = 0", "aalo.Q0 = -1"])
def test_aalo_config_errors(emu, bad):
    from paper_2603_17456_b200.native import Config, DeviceBatch, MfsimError
    b = DeviceBatch(0, emu)
    with pytest.raises(MfsimError) as e:
        b.add_config(Config(cases.sanity_config("aalo") + bad + "\n", emu))
        b.prepare()
    assert e.value.code == 2


@pytest.mark.gpu
def test_aalo_device_matches_oracle(product):
    from paper_2603_17456_b200 import sweep
    from paper_2603_17456_b200.native import DeviceBatch
    texts = list(aalo_cases().values())
    texts.append(sweep.sweep_config((0.8, 3, 1, "aalo"), requests=400, lib=product))
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


# ---------------------------------------------------------------- varys
# policy = varys: Varys-style SEBF + MADD (clairvoyant coflow scheduling):
# coflows as in aalo; one class per coflow by its effective bottleneck
# Gamma = max over links of remaining bytes over the link / capacity; members
# capped at remaining / Gamma (MADD). Oracle: mfsim_oracle.c policy 6.

def varys_cases():
    out = {k: v.replace("policy = aalo", "policy = varys") for k, v in aalo_cases().items()
           if "aalo." not in v}
    c8 = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs", "cluster8.conf")).read()
    out["cluster8_300_rate12"] = c8 + "workload.request_count = 300\nworkload.rate_rps = 12\npolicy = varys\n"
    return out


@needs_oracle
@pytest.mark.parametrize("name", sorted(varys_cases()))
def test_varys_host_engine_matches_oracle(emu, name):
    from paper_2603_17456_b200.native import run_config
    text = varys_cases()[name]
    assert "policy = varys" in text
    want = ref.run_config(text, so=ref.ORACLE_SO)
    got = run_config(text, lib=emu, detail=2)
    assert diff(got, want) == []


@needs_oracle
@pytest.mark.parametrize("name", ["trio", "ingress", "egress", "single_request", "stall_zero",
                                  "ticks", "tick_promotion"])
def test_varys_manual_scenarios_match_oracle(emu, name):
    from paper_2603_17456_b200.native import run_manual
    import re
    fn = getattr(cases, name)
    spec = fn("mfs") if name in ("trio", "ingress", "egress") else fn()
    spec = re.sub(r"^policy \w+", "policy varys", spec, flags=re.M)
    assert "policy varys" in spec
    assert diff(run_manual(spec, lib=emu), ref.run_manual(spec, so=ref.ORACLE_SO)) == []


@needs_oracle
def test_varys_differs_from_other_policies():
    text = varys_cases()["cluster8_200"]
    a = ref.run_config(text, so=ref.ORACLE_SO)
    for p in POLICIES + ("aalo",):
        b = ref.run_config(text.replace("policy = varys", f"policy = {p}"), so=ref.ORACLE_SO)
        assert not bits_equal(a.flow_finish, b.flow_finish), p


@pytest.mark.gpu
def test_varys_device_matches_oracle(product):
    from paper_2603_17456_b200 import sweep
    from paper_2603_17456_b200.native import DeviceBatch
    texts = list(varys_cases().values())
    texts.append(sweep.sweep_config((0.8, 3, 1, "varys"), requests=400, lib=product))
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


@pytest.mark.gpu
def test_extensions_under_the_gang_kernel(product):
    """the extension kernel instance (aalo / varys code compiled in) as a
    lock-step gang: forced for this small batch, same results as the oracle"""
    from paper_2603_17456_b200.native import DeviceBatch
    texts = list(aalo_cases().values())[:3] + list(varys_cases().values())[:3]
    os.environ["MFSIM_GANG_MIN"] = "1"
    try:
        b = DeviceBatch(0, product)
    finally:
        os.environ.pop("MFSIM_GANG_MIN", None)
    for t in texts:
        b.add_config(t)
    b.prepare()
    b.run(2)
    assert b.last_kernel == "mfsim_gang_kernel"
    bad = {}
    for i, t in enumerate(texts):
        d = diff(b.result(i, 2, reports=True), ref.run_config(t, so=ref.ORACLE_SO))
        if d:
            bad[i] = d
    assert bad == {}
