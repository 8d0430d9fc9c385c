"""The C-ABI library loads and exports every symbol include/*.h declares;
handle semantics and error codes follow the reference C API (mfsim.h,
mfsim_capi.cpp:19-97, test_capi.cpp)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PRODUCT = os.path.join(ROOT, "paper_2603_17456_b200", "libmfsim_b200.so")


def declared_functions():
    names = set()
    for h in ("mfsim.h", "mfsim_dev.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(mfsim_\w+)\s*\(", text):
            names.add(m.group(1))
    return sorted(names)


def test_headers_declare_the_reference_surface():
    names = declared_functions()
    for ref_fn in ("mfsim_version", "mfsim_last_error", "mfsim_config_create", "mfsim_config_load",
                   "mfsim_config_set", "mfsim_config_get", "mfsim_config_destroy", "mfsim_run",
                   "mfsim_string_free"):
        assert ref_fn in names


@pytest.mark.parametrize("path", [PRODUCT, os.path.join(ROOT, "build", "libmfsim_emu.so")])
def test_library_exports_every_declared_symbol(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built")
    lib = C.CDLL(path)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert missing == []


def test_product_library_is_cuda_only():
    """no CPU path: without a device the product reports an error instead of computing"""
    if not os.path.exists(PRODUCT):
        pytest.skip("product library not built")
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2603_17456_b200.native import MfsimError, Native, mfsim_run
    lib = Native(PRODUCT)
    with pytest.raises(MfsimError) as e:
        mfsim_run(open(os.path.join(ROOT, "tests", "configs", "example.conf")).read(), lib=lib)
    assert e.value.code == 6 and "CUDA" in str(e.value)


def test_config_handle(emu):
    from paper_2603_17456_b200.native import Config, MfsimError
    c = Config("policy = mfs\nsim.seed = 3 # comment\n", emu)
    assert c.get("policy") == "mfs" and c.get("sim.seed") == "3" and c.get("nope") is None
    c.set("policy", "fs")
    assert c.get("policy") == "fs"
    assert emu.lib.mfsim_config_load(b"/nonexistent/x.conf") is None
    assert b"cannot open config file" in emu.lib.mfsim_last_error()
    assert emu.lib.mfsim_config_set(None, b"a", b"b") == 1


@pytest.mark.parametrize("text,code", [
    ("policy = nope\n", 2),
    ("topology.kind = ring\n", 2),
    ("model.layers = 0\n", 2),
    ("workload.rate_rps = -1\n", 2),
    ("sim.promotion_tick_ms = 0\n", 2),
    ("mfs.K = 1\npolicy = mfs\n", 2),
    ("workload.request_count = 1.5\n", 2),
    ("workload.trace = /nonexistent.csv\n", 4),
])
def test_error_codes(emu, text, code):
    from paper_2603_17456_b200.native import MfsimError, mfsim_run
    with pytest.raises(MfsimError) as e:
        mfsim_run(text, lib=emu)
    assert e.value.code == code


def test_mfsim_run_reports_are_byte_identical(emu, tmp_path):
    """mfsim_run(cfg, out_dir, &summary) writes the reference's files byte for byte"""
    import cases
    from parity import manifest
    from paper_2603_17456_b200.native import mfsim_run
    text = cases.workload_cases()["example_mfs"]
    s = mfsim_run(text, out_dir=str(tmp_path), lib=emu)
    assert s == manifest()["workload"]["example_mfs"]["summary_json"]
    assert open(tmp_path / "summary.json").read() == s
    import hashlib
    assert hashlib.sha256(open(tmp_path / "requests.csv", "rb").read()).hexdigest() == \
        manifest()["workload"]["example_mfs"]["requests_csv_sha256"]
