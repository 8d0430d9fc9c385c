"""Parity cases shared by the fixture generator and the tests.

Manual scenarios restate the reference's own worked examples
(tests/support/scenarios.hpp:27-132, test_engine.cpp:74-291, the
acceptance C1-C4 instances) as manual-instance specs; workload cases are the
reference's shipped configs and the configs its tests use
(test_engine.cpp:443-590, acceptance_main.cpp:358-501).
"""
from __future__ import annotations

import os
import random

HERE = os.path.dirname(os.path.abspath(__file__))
CONF = os.path.join(HERE, "..", "configs")

POLICIES = ("fs", "sjf", "edf", "karuna", "mfs")


def _read(name):
    return open(os.path.join(CONF, name)).read()


# ---------------------------------------------------------------- manual

def trio(policy: str) -> str:
    """scenarios.hpp:27-60: effective deadlines only visible to mfs"""
    eff = policy == "mfs"
    d = (9, 6, 7) if eff else (18, 12, 7)
    s = [f"policy {policy}", "node prefill", "node decode", "link 0 1 1.0"]
    for i, (size, rd) in enumerate(zip((2, 4, 3), (18, 12, 7))):
        s += [f"request 0 {rd}", f"batch 0 {i} -", f"flow {i} {i} p2d 0 1 {size} 1 0 {d[i]}"]
    return "\n".join(s) + "\n"


def ingress(policy: str) -> str:
    """scenarios.hpp:69-96"""
    return "\n".join([
        f"policy {policy}", "node prefill", "node prefill", "node prefill", "node switch",
        "link 0 3 1.0", "link 1 3 1.0", "link 3 2 1.0",
        "request 0 inf", "batch 0 0 1,1,1",
        "flow 0 0 reuse 0 2 2 3 0 -", "flow 0 0 collective 1 2 1 1 - -"]) + "\n"


def egress(policy: str) -> str:
    """scenarios.hpp:105-132"""
    return "\n".join([
        f"policy {policy}", "node prefill", "node prefill", "node decode", "node switch",
        "link 0 3 1.0", "link 3 1 1.0", "link 3 2 1.0",
        "request 0 20", "batch 0 0 1,1",
        "flow 0 0 p2d 0 2 2 1 - 20", "flow 0 0 collective 0 1 1 2 - -"]) + "\n"


def single_request() -> str:
    """test_engine.cpp:74-92: ttft = compute [0,1] + collective [1,2]"""
    return "policy fs\nnode prefill\nnode prefill\nduplex 0 1 1.0\nrequest 0 inf\nbatch 0 0 1\n" \
           "flow 0 0 collective 0 1 1 1 - -\n"


def stall_zero() -> str:
    """test_engine.cpp:105-126"""
    return "policy fs\nnode prefill\nnode prefill\nduplex 0 1 1.0\nrequest 0 inf\nbatch 0 0 5,1\n" \
           "flow 0 0 collective 0 1 1 1 0 -\n"


def ticks() -> str:
    """test_engine.cpp:128-151: ticks after the pipeline drains"""
    return "policy mfs\nparam promotion_tick 0.25\nnode prefill\nnode decode\nduplex 0 1 1.0\n" \
           "request 0 100\nbatch 0 0 1\nflow 0 0 p2d 0 1 2 1 - 100\n"


def tick_promotion() -> str:
    """test_engine.cpp:212-240: p2d@3.2, reuse@33, band urgent"""
    return "policy mfs\nset inter.enable_pruning false\nparam promotion_tick 0.4\nnode prefill\n" \
           "node prefill\nlink 0 1 1.0\nrequest 0 20\nbatch 0 0 1\n" \
           "flow 0 0 reuse 0 1 30 99 2 -\nflow 0 0 p2d 0 1 2 1 - 20\n"


def soft_enforcement(pruning: bool) -> str:
    """test_engine.cpp:242-291"""
    s = ["policy mfs", f"set inter.enable_pruning {'true' if pruning else 'false'}",
         "node prefill", "node decode", "link 0 1 1.0"]
    specs = [(8.0, 2.0, None), (9.0, 2.0, None), (13.5, 9.0, [3.0])]
    for i, (dl, size, comp) in enumerate(specs):
        s.append(f"request 0 {dl}")
        if comp:
            s.append(f"batch 0 {i} {','.join(str(c) for c in comp)}")
            s.append(f"flow {i} {i} p2d 0 1 {size} 1 - {dl}")
        else:
            s.append(f"batch 0 {i} -")
            s.append(f"flow {i} {i} p2d 0 1 {size} 1 0 {dl}")
    return "\n".join(s) + "\n"


def livelock() -> str:
    """test_engine.cpp:153-172: eight zero-size flows at t=0 trip the guard"""
    s = ["policy fs", "param livelock_events 3", "node prefill", "node prefill", "duplex 0 1 1.0",
         "request 0 inf", "batch 0 0 -"]
    s += ["flow 0 0 reuse 0 1 0 1 0 -"] * 8
    return "\n".join(s) + "\n"


def rli_instances(n: int = 60, seed: int = 404):
    """acceptance_main.cpp:102-145 (C4): random single-link pipelines under mfs"""
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        L = 1 + rng.randrange(3)
        comp = [1.0 + rng.randrange(3) for _ in range(L)]
        nf = 1 + rng.randrange(4)
        s = ["policy mfs", "node prefill", "node prefill", "link 0 1 1.0", "request 0 inf",
             f"batch 0 0 {','.join(str(c) for c in comp)}"]
        for _ in range(nf):
            s.append(f"flow 0 0 reuse 0 1 {1.0 + rng.randrange(4)} {1 + rng.randrange(L)} 0 -")
        out.append("\n".join(s) + "\n")
    return out


def random_manual(n: int = 40, seed: int = 7):
    """randomised manual instances: star fabrics, mixed stages, all policies"""
    rng = random.Random(seed)
    out = []
    for it in range(n):
        pol = POLICIES[it % 5]
        hosts = 3 + rng.randrange(4)
        s = [f"policy {pol}", f"param promotion_tick {0.1 + 0.1 * rng.randrange(5)}"]
        s += ["node prefill"] * hosts + ["node switch"]
        for h in range(hosts):
            s.append(f"duplex {h} {hosts} {0.5 + 0.5 * rng.randrange(4)}")
        nreq = 1 + rng.randrange(4)
        for r in range(nreq):
            s.append(f"request {0.5 * rng.randrange(4)} {4 + rng.randrange(20)} {100 + 50 * rng.randrange(10)}")
        for r in range(nreq):
            L = 1 + rng.randrange(3)
            comp = ",".join(str(0.5 + 0.5 * rng.randrange(4)) for _ in range(L))
            s.append(f"batch {0.5 * rng.randrange(4)} {r} {comp}")
            for _ in range(1 + rng.randrange(5)):
                st = ("reuse", "collective", "p2d")[rng.randrange(3)]
                a = rng.randrange(hosts)
                b = (a + 1 + rng.randrange(hosts - 1)) % hosts
                size = 0.5 + rng.randrange(8)
                tl = 1 + rng.randrange(L)
                rel = f"{0.5 * rng.randrange(6)}" if rng.random() < 0.25 else "-"
                dl = f"{5 + rng.randrange(25)}" if st == "p2d" else "-"
                req = r if st != "collective" else (r if rng.random() < 0.5 else -1)
                s.append(f"flow {r} {req} {st} {a} {b} {size} {tl} {rel} {dl}")
        out.append("\n".join(s) + "\n")
    return out


def manual_cases():
    """name -> spec"""
    c = {}
    for p in POLICIES:
        c[f"trio_{p}"] = trio(p)
    for p in ("mfs", "fs", "sjf", "edf"):
        c[f"ingress_{p}"] = ingress(p)
        c[f"egress_{p}"] = egress(p)
    c["single_request"] = single_request()
    c["stall_zero"] = stall_zero()
    c["ticks"] = ticks()
    c["tick_promotion"] = tick_promotion()
    c["soft_enforcement_on"] = soft_enforcement(True)
    c["soft_enforcement_off"] = soft_enforcement(False)
    for i, s in enumerate(rli_instances()):
        c[f"rli_{i:03d}"] = s
    for i, s in enumerate(random_manual()):
        c[f"random_{i:03d}"] = s
    return c


# --------------------------------------------------------------- workload

def sanity_config(policy: str) -> str:
    """test_engine.cpp:443-504"""
    return ("topology.kind = star\ntopology.hosts = 9\ntopology.link_bytes_per_s = 500\n"
            "cluster.prefill_units = 3\ncluster.hosts_per_unit = 2\ncluster.decode_hosts = 3\n"
            "model.layers = 4\nmodel.alpha_ms = 2\nmodel.beta_us_per_token = 1\n"
            "model.kv_bytes_per_token_layer = 0.8\nmodel.coll_bytes_per_token_layer = 0.3\n"
            "workload.request_count = 60\nworkload.rate_rps = 6\nworkload.prompt_mean_tokens = 300\n"
            "workload.prompt_sigma = 0.5\nworkload.reuse_fraction_mean = 0.4\nsim.seed = 5\n"
            f"policy = {policy}\n")


def fattree_config(policy: str) -> str:
    """test_engine.cpp:525-548"""
    return ("topology.kind = fattree\ntopology.hosts = 12\ntopology.link_bytes_per_s = 800\n"
            "cluster.prefill_units = 4\ncluster.hosts_per_unit = 2\ncluster.decode_hosts = 4\n"
            "model.layers = 3\nmodel.kv_bytes_per_token_layer = 0.5\n"
            "model.coll_bytes_per_token_layer = 0.25\nworkload.request_count = 30\n"
            "workload.rate_rps = 5\nworkload.prompt_mean_tokens = 200\n"
            "workload.reuse_fraction_mean = 0.5\nsim.seed = 9\n"
            f"policy = {policy}\n")


def c9_config() -> str:
    """acceptance_main.cpp:459-501"""
    return ("topology.kind = star\ntopology.hosts = 12\ntopology.link_bytes_per_s = 1.0\n"
            "cluster.prefill_units = 4\ncluster.hosts_per_unit = 2\ncluster.decode_hosts = 4\n"
            "model.layers = 8\nmodel.kv_bytes_per_token_layer = 1.2e-6\n"
            "model.coll_bytes_per_token_layer = 4.8e-7\nworkload.request_count = 300\n"
            "workload.rate_rps = 6\nworkload.prompt_mean_tokens = 1500\n"
            "workload.prompt_sigma = 0.5\npolicy = mfs\nsim.seed = 11\n")


def workload_cases(big: bool = False):
    """name -> config text. big=True adds the BASELINE-size parity configs."""
    c = {}
    for p in POLICIES:
        c[f"example_{p}"] = _read("example.conf") + f"policy = {p}\n"
        c[f"sanity_{p}"] = sanity_config(p)
        c[f"fattree_{p}"] = fattree_config(p)
        c[f"cluster8_400_{p}"] = _read("cluster8.conf") + f"policy = {p}\nworkload.request_count = 400\n"
    c["c9_mfs"] = c9_config()
    c["cluster8_rate12_mfs"] = _read("cluster8.conf") + "policy = mfs\nworkload.request_count = 300\nworkload.rate_rps = 12\n"
    c["cluster8_rate12_karuna"] = _read("cluster8.conf") + "policy = karuna\nworkload.request_count = 200\nworkload.rate_rps = 12\n"
    if big:
        for p in POLICIES:  # BASELINE configs[0]: cluster8, 1024 requests
            c[f"cluster8_1024_{p}"] = _read("cluster8.conf") + f"policy = {p}\nworkload.request_count = 1024\n"
    return c
