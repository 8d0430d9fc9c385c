"""Parity at the five BASELINE.json configurations (paper_2603_17456_b200/configs.py).

The reference itself produced tests/golden/baseline/*.json (make_baseline_golden.py):
counters, SLO attainment, the summary.json bytes, the requests.csv digest and
sha256 digests of every full-precision result array. The GPU tier runs the
same configs on the sm_100a engine, all instances of a group in one launch,
and requires every digest to match: exact TTFT SLO attainment, bit-exact
per-request done times / flags / stalls, per-flow finish times and final
RMLQ (band, level), coflow times, event and step counts.

configs[2] (ft128, 100k requests, 15 instances, ~24M events each) and
configs[4] (4096 GPUs, ~2M events each) run one warp per instance for tens of
minutes; they run only with MFSIM_FULL_PARITY=1 (results kept in profiles/).
configs[3] (the sweep) is covered by test_gpu_parity.test_full_size_sweep_instances
and the bench."""
import glob
import json
import os

import pytest

from parity import SCALARS, digest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "baseline")
ARRAYS = ("req_arrival", "req_deadline", "req_done", "req_pruned", "req_stall", "flow_finish",
          "flow_band", "flow_level", "cof_release", "cof_done", "cof_stall", "pipe_done")


def golden(prefix):
    out = {}
    for p in sorted(glob.glob(os.path.join(GOLD, prefix + "_*.json"))):
        out[os.path.basename(p)[:-5]] = json.load(open(p))
    return out


def test_golden_configs_are_current():
    """the stored config texts are what configs.py generates today"""
    from paper_2603_17456_b200 import configs
    g = {**golden("cfg1"), **golden("cfg2"), **golden("cfg3"), **golden("cfg5")}
    assert len(golden("cfg1")) == 10 and len(golden("cfg2")) >= 5
    for name, m in g.items():
        parts = name.split("_")
        kind, pol = parts[0], parts[1]
        seed = int(parts[2][1:]) if len(parts) > 2 else 1
        want = {"cfg1": lambda: configs.config1(seed=seed, policy=pol),
                "cfg2": lambda: configs.config2(policy=pol),
                "cfg3": lambda: configs.config3(seed=seed, policy=pol),
                "cfg5": lambda: configs.config5(policy=pol)}[kind]()
        if kind == "cfg5":  # trace path differs between machines
            want = want.split("workload.trace")[0]
            assert m["config"].split("workload.trace")[0] == want
        else:
            assert m["config"] == want, name
        assert 0.0 <= m["attainment"] <= 1.0
        assert m["events"] > 0


def _mismatch(res, m):
    import hashlib
    bad = [k for k in SCALARS if int(getattr(res, k)) != m[k]]
    bad += [k for k in ARRAYS if digest(getattr(res, k)) != m["sha256"][k]]
    if m.get("oracle") == "restatement":  # the C restatement writes no reports
        import json as _json
        if _json.loads(res.summary_json)["slo_attainment"] != m["attainment"]:
            bad.append("slo_attainment")
        return bad
    if res.summary_json != m["summary_json"]:
        bad.append("summary.json bytes")
    if hashlib.sha256(res.requests_csv.encode()).hexdigest() != m["requests_csv_sha256"]:
        bad.append("requests.csv bytes")
    return bad


def _run_group(product, g, verbose=False):
    from paper_2603_17456_b200 import configs
    from paper_2603_17456_b200.native import DeviceBatch
    names = sorted(g)
    b = DeviceBatch(0, product)
    for n in names:
        text = g[n]["config"]
        if n.startswith("cfg5"):  # re-point the trace at this checkout
            text = text.split("workload.trace")[0] + f"workload.trace = {configs.TRACE_4096}\n"
        b.add_config(text)
    b.prepare()
    b.run(2)
    bad = {}
    for i, n in enumerate(names):
        r = b.result(i, 2, reports=True)
        mm = _mismatch(r, g[n])
        if verbose:
            print(f"{n}: events {r.events} (reference {g[n]['events']}), SLO attainment "
                  f"{r.attainment} (reference {g[n]['attainment']}), "
                  f"{'bit-exact' if not mm else 'MISMATCH ' + str(mm)}", flush=True)
        if mm:
            bad[n] = mm
    return bad


@pytest.mark.gpu
def test_configs_1_2_bit_exact(product):
    """configs[0] (cluster8 1024 req, mfs/fs, seeds 1-5) and configs[1]
    (cluster8 10k req, five policies + the aalo coflow extension, whose golden
    comes from the C restatement), all instances in one launch"""
    g = {**golden("cfg1"), **golden("cfg2")}
    assert _run_group(product, g) == {}


FULL = pytest.mark.skipif(os.environ.get("MFSIM_FULL_PARITY") != "1", reason="set MFSIM_FULL_PARITY=1")


def _full(g, product, label):
    import time
    t0 = time.time()
    bad = _run_group(product, g, verbose=True)
    print(f"{label}: {len(g)} instances in {time.time() - t0:.0f} s, mismatches: {bad}", flush=True)
    return bad


@pytest.mark.gpu
@FULL
@pytest.mark.timeout(0)
def test_config_3_bit_exact(product):
    """configs[2]: ft128 (1024 GPUs), 100k requests, fs/sjf/edf/mfs x seeds 1-3
    (12 instances in one launch, one warp each; ~25 min)"""
    g = {k: v for k, v in golden("cfg3").items() if "karuna" not in k}
    assert len(g) == 12
    assert _full(g, product, "configs[2]") == {}


@pytest.mark.gpu
@pytest.mark.skipif(os.environ.get("MFSIM_FULL_PARITY_KARUNA") != "1", reason="set MFSIM_FULL_PARITY_KARUNA=1")
@pytest.mark.timeout(0)
def test_config_3_karuna_bit_exact(product):
    """configs[2], Karuna x seeds 1-3: ~24M events at ~240 us each on one warp
    (~1.6 h) -- longer than one 60-minute box call"""
    g = {k: v for k, v in golden("cfg3").items() if "karuna" in k}
    assert len(g) == 3
    assert _full(g, product, "configs[2] karuna") == {}


@pytest.mark.gpu
@FULL
@pytest.mark.timeout(0)
def test_config_5_bit_exact(product):
    """configs[4]: 4096-GPU fat-tree (3,768 links), heavy-tailed trace, mfs/fs"""
    g = golden("cfg5")
    assert len(g) == 2
    # ~4k active flows: start above the 1024-flow first attempt (a capacity
    # overflow re-runs the whole instance)
    os.environ["MFSIM_ACTIVE_CAP"] = "8192"
    try:
        assert _full(g, product, "configs[4]") == {}
    finally:
        os.environ.pop("MFSIM_ACTIVE_CAP", None)


@pytest.mark.skipif(os.environ.get("MFSIM_EMU_FULL") != "1", reason="set MFSIM_EMU_FULL=1 (~5 min of CPU)")
@pytest.mark.timeout(0)
def test_config_5_engine_logic_on_cpu(emu):
    """configs[4] through the serial host build of the same engine source
    (build/libmfsim_emu.so): ~2 min (fs) + ~3 min (mfs) on one core against the
    reference's 1599 s / 1071 s; profiles/r02_emu_config5.log"""
    os.environ["MFSIM_ACTIVE_CAP"] = "8192"
    try:
        assert _full(golden("cfg5"), emu, "configs[4] (emulated)") == {}
    finally:
        os.environ.pop("MFSIM_ACTIVE_CAP", None)
