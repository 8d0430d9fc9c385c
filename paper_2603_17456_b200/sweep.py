"""BASELINE.json workloads as reference config text.

configs[1]  cluster8: 8 units x 2 hosts + 8 decode, star, all five policies
configs[2]  ft128:    "1024 GPUs" = 128 hosts x 8 NICs on a k=8 fat-tree (768
            links), 16 prefill units x 4 hosts, 64 decode hosts, cluster8 sizing
configs[3]  sweep:    ft128 fabric, 2000 requests per instance, offered load
            rho in {0.3..0.9} x SLO multiplier {1..5} x 64 seeds x 5 policies
            = 11,200 independent instances

Offered load rho is the predicted utilisation of the busiest link from mean
demands: per request of unit u, P2D lead(u)->decode(u) carries L*T*kv bytes,
reuse lead(src)->lead(u) carries r*L*T*kv with src ~ Zipf(skew) over the other
units, and every ordered host pair (i, j) of the unit carries L*T*coll (the
collective all-to-all per layer, batch tokens ~= T per request). Routes come
from the library's own router (Topology::route, lowest-link-id BFS).
"""
from __future__ import annotations

import itertools

POLICIES = ("fs", "sjf", "edf", "karuna", "mfs")
LOADS = (0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9)
SLO_SCALES = (1, 2, 3, 4, 5)

SIZING = {
    "model.layers": 16,
    "model.alpha_ms": 1.0,
    "model.beta_us_per_token": 0.1,
    "model.kv_bytes_per_token_layer": 1.2e-6,
    "model.coll_bytes_per_token_layer": 4.8e-7,
    "workload.prompt_mean_tokens": 2000,
    "workload.prompt_sigma": 0.6,
    "workload.reuse_fraction_mean": 0.5,
    "workload.reuse_skew": 1.0,
    "workload.max_batch_tokens": 8192,
    "mfs.K": 8,
    "mfs.E": 4,
    "mfs.U": 0.5,
    "inter.enable_pruning": "true",
    "inter.drop_budget_frac": 0.05,
    "sim.promotion_tick_ms": 10,
}

CLUSTER8 = dict(SIZING, **{
    "topology.kind": "star",
    "topology.hosts": 24,
    "topology.link_bytes_per_s": 1.0,
    "cluster.prefill_units": 8,
    "cluster.hosts_per_unit": 2,
    "cluster.decode_hosts": 8,
    "workload.rate_rps": 8,
    "workload.slo_multiplier": 3,
})

FT128 = dict(SIZING, **{
    "topology.kind": "fattree",
    "topology.hosts": 128,
    "topology.nics_per_host": 8,
    "topology.link_bytes_per_s": 0.125,
    "cluster.prefill_units": 16,
    "cluster.hosts_per_unit": 4,
    "cluster.decode_hosts": 64,
    "workload.rate_rps": 1,
    "workload.slo_multiplier": 3,
})


def text(d: dict) -> str:
    return "".join(f"{k} = {v}\n" for k, v in d.items())


def _zipf(self_u: int, units: int, skew: float):
    w = {v: 1.0 / (v + 1) ** skew for v in range(units) if v != self_u}
    s = sum(w.values())
    return {v: x / s for v, x in w.items()}


# the simulator's defaults for the keys the load model reads (config.cpp,
# CostModel / Layout / WorkloadSpec::from; decode_hosts defaults to the unit count)
LIB_DEFAULTS = {
    "cluster.prefill_units": 1,
    "cluster.hosts_per_unit": 2,
    "model.layers": 4,
    "model.kv_bytes_per_token_layer": 1000.0,
    "model.coll_bytes_per_token_layer": 250.0,
    "workload.prompt_mean_tokens": 2000.0,
    "workload.reuse_fraction_mean": 0.5,
    "workload.reuse_skew": 1.0,
}

_util_cache: dict = {}


def busiest_link_bytes(base: dict, lib=None) -> float:
    """max over links of (bytes per second per unit of per-unit request rate)/capacity."""
    from .native import Config, link_count, route

    key = tuple(sorted((k, str(v)) for k, v in base.items() if not k.startswith(("workload.rate", "sim.seed", "policy", "workload.slo", "workload.request"))))
    if key in _util_cache:
        return _util_cache[key]
    cfg = Config(text(base), lib)
    # keys the file leaves out take the simulator's defaults (config.cpp)
    eff = dict(LIB_DEFAULTS, **base)
    U = int(eff["cluster.prefill_units"])
    H = int(eff["cluster.hosts_per_unit"])
    D = int(eff.get("cluster.decode_hosts", U))
    L = float(eff["model.layers"])
    T = float(eff["workload.prompt_mean_tokens"])
    kv = float(eff["model.kv_bytes_per_token_layer"])
    coll = float(eff["model.coll_bytes_per_token_layer"])
    r = float(eff["workload.reuse_fraction_mean"])
    skew = float(eff["workload.reuse_skew"])
    load = [0.0] * link_count(cfg, lib)
    cap = [1.0] * len(load)

    def add(src, dst, b):
        links, caps = route(cfg, src, dst, lib)
        for l, c in zip(links, caps):
            load[l] += b
            cap[l] = c

    lead = lambda u: u * H  # noqa: E731
    for u in range(U):
        add(lead(u), U * H + (u % D), L * T * kv)
        if U > 1 and r > 0:
            for src, p in _zipf(u, U, skew).items():
                add(lead(src), lead(u), p * r * L * T * kv)
        for i in range(H):
            for j in range(H):
                if i != j:
                    add(u * H + i, u * H + j, L * T * coll)
    worst = max(l / c for l, c in zip(load, cap))
    _util_cache[key] = worst
    return worst


def rate_for_load(rho: float, base: dict = FT128, lib=None) -> float:
    """per-unit Poisson rate (req/s) whose predicted busiest-link utilisation is rho"""
    return rho / busiest_link_bytes(base, lib)


def sweep_cells(loads=LOADS, slos=SLO_SCALES, seeds=range(1, 65), policies=POLICIES):
    """the 7 x 5 x 64 x 5 = 11,200 cells of configs[3], in a fixed order"""
    return list(itertools.product(loads, slos, seeds, policies))


def sweep_config(cell, requests: int = 2000, base: dict = FT128, lib=None) -> str:
    rho, slo, seed, pol = cell
    d = dict(base)
    d["workload.rate_rps"] = repr(rate_for_load(rho, base, lib))
    d["workload.slo_multiplier"] = slo
    d["sim.seed"] = seed
    d["policy"] = pol
    d["workload.request_count"] = requests
    return text(d)
