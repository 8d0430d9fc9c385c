"""The five BASELINE.json configurations as reference config texts.

  [0] cluster8 (8-server / 32-GPU testbed), ~1k requests, MFS vs FS, seeds 1-5
  [1] cluster8, all five policies at the FS knee (rate 8), 10k requests
  [2] 1024-GPU fat-tree (ft128: 128 hosts x 8 NICs, k=8), 100k requests, seeds 1-3
  [3] the sweep over [2]'s fabric (sweep.py), 11,200 instances of 2000 requests
  [4] 4096-GPU fat-tree (512 hosts x 8 NICs, k=14, 3,768 links), heavy-tailed
      trace (lognormal sigma 1.5 prompts, Beta reuse), ~4.5k requests ~ 1M flows

SURVEY.md section 8(d) restates each as concrete inputs; the keys are the
reference's (config.cpp, configs/cluster8.conf). Oversubscription and the
Varys/Aalo policy are not expressible in the reference and are not offered.
"""
from __future__ import annotations

import math
import os

from . import sweep

STRESS4096 = dict(sweep.SIZING, **{
    "topology.kind": "fattree",
    "topology.hosts": 512,
    "topology.nics_per_host": 8,
    "topology.link_bytes_per_s": 0.125,
    "cluster.prefill_units": 64,
    "cluster.hosts_per_unit": 4,
    "cluster.decode_hosts": 256,
    "workload.slo_multiplier": 3,
})

TRACE_4096 = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "tests", "configs", "stress4096_trace.csv")


def config1(seed: int = 1, policy: str = "mfs", requests: int = 1024) -> str:
    return sweep.text(dict(sweep.CLUSTER8, **{"policy": policy, "sim.seed": seed,
                                               "workload.request_count": requests}))


def config2(policy: str = "mfs", requests: int = 10000, seed: int = 1) -> str:
    return sweep.text(dict(sweep.CLUSTER8, **{"policy": policy, "sim.seed": seed,
                                               "workload.rate_rps": 8,
                                               "workload.request_count": requests}))


def config3(seed: int = 1, policy: str = "mfs", requests: int = 100000) -> str:
    return sweep.text(dict(sweep.FT128, **{"policy": policy, "sim.seed": seed,
                                            "workload.request_count": requests}))


def config5(policy: str = "mfs", trace: str = TRACE_4096) -> str:
    return sweep.text(dict(STRESS4096, **{"policy": policy, "workload.trace": trace}))


def _splitmix(seed: int):
    x = seed & 0xFFFFFFFFFFFFFFFF
    while True:
        x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        yield ((z ^ (z >> 31)) >> 11) * (1.0 / (1 << 53))


def write_stress_trace(path: str = TRACE_4096, n: int = 4500, units: int = 64,
                       rate_per_unit: float = 1.0, seed: int = 1, max_tokens: int = 8192):
    """Heavy-tailed trace for config [4] (splitmix64 stream `seed`): Poisson
    arrivals, lognormal(mean 2000, sigma 1.5) prompts clamped to the batch cap,
    Beta(0.7, 0.7) reuse via a ratio of gamma-free order statistics (Johnk),
    Zipf(1.0) reuse sources. Columns: arrival_s,prompt_tokens,reuse_fraction,source_unit."""
    u = _splitmix(seed)
    sigma, mean = 1.5, 2000.0
    mu = math.log(mean) - 0.5 * sigma * sigma
    zipf_w = [1.0 / (v + 1) for v in range(units)]
    t = 0.0
    rows = ["arrival_s,prompt_tokens,reuse_fraction,source_unit"]
    for i in range(n):
        t += -math.log1p(-next(u)) / (rate_per_unit * units)
        z = math.sqrt(-2.0 * math.log(1.0 - next(u))) * math.cos(2.0 * math.pi * next(u))
        tok = min(max(int(round(math.exp(mu + sigma * z))), 1), max_tokens)
        while True:  # Johnk's Beta(a, a) sampler
            x, y = next(u) ** (1 / 0.7), next(u) ** (1 / 0.7)
            if 0.0 < x + y <= 1.0:
                reuse = x / (x + y)
                break
        reuse = min(reuse, 0.95)
        unit = i % units  # read_trace assigns units round-robin (workload.cpp)
        w = [zipf_w[v] if v != unit else 0.0 for v in range(units)]
        r = next(u) * sum(w)
        src = units - 1
        for v in range(units):
            r -= w[v]
            if w[v] > 0.0 and r <= 0.0:
                src = v
                break
        rows.append(f"{t:.9f},{tok},{reuse:.6f},{src}")
    with open(path, "w") as f:
        f.write("\n".join(rows) + "\n")
    return path


if __name__ == "__main__":
    print(write_stress_trace())
