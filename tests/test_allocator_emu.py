"""The engine's two filling variants (per-link and link-slot) against the
reference's allocate_rates (allocator.cpp:28-126) called directly, on star
fabrics: random classes and caps, and the near-ties where the engine's
approximate-then-exact minimum (a single-precision reciprocal first) must still
pick the exact min(link share, cap gap)."""
import ctypes as C
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def emu_alloc(emu):
    fn = emu.lib.mfsim_emu_allocate_star
    ip, dp = C.POINTER(C.c_int), C.POINTER(C.c_double)
    fn.argtypes = [C.c_int, C.c_double, C.c_int, ip, ip, ip, C.c_int, dp, C.c_int, dp]
    fn.restype = C.c_int

    def run(hosts, cap, src, dst, cls_of, ncls, caps, variant):
        n = len(src)
        a = [np.ascontiguousarray(x, np.int32) for x in (src, dst, cls_of)]
        cp = None if caps is None else np.ascontiguousarray(caps, np.float64)
        out = np.zeros(n)
        rc = fn(hosts, cap, n, *[x.ctypes.data_as(ip) for x in a], ncls,
                None if cp is None else cp.ctypes.data_as(dp), variant, out.ctypes.data_as(dp))
        assert rc == 0
        return out
    return run


@pytest.fixture(scope="module")
def ref_alloc():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    return ref.allocate_star


def same_bits(a, b):
    return np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))


@pytest.mark.parametrize("variant", [0, 1])
def test_cap_one_ulp_above_link_share(emu_alloc, ref_alloc, variant):
    """three flows share host 0's up link (share 1/3); one is capped one ulp above
    the exact share: the reference takes min(share, cap gap) = the share"""
    q = 1.0 / 3.0
    for n_on_link in (3, 5, 7, 11, 13, 100):
        hosts = n_on_link + 1
        src = [0] * n_on_link
        dst = list(range(1, n_on_link + 1))
        share = 1.0 / n_on_link
        for cap_v in (np.nextafter(share, np.inf), np.nextafter(np.nextafter(share, np.inf), np.inf),
                      np.nextafter(share, -np.inf), share):
            caps = np.full(n_on_link, np.nan)
            caps[0] = cap_v
            want = ref_alloc(hosts, 1.0, src, dst, [0] * n_on_link, 1, caps)
            got = emu_alloc(hosts, 1.0, src, dst, [0] * n_on_link, 1, caps, variant)
            assert same_bits(got, want), (n_on_link, cap_v, got[:3], want[:3])
    assert q > 0


@pytest.mark.parametrize("variant", [0, 1])
def test_random_classes_and_caps(emu_alloc, ref_alloc, variant):
    rng = np.random.default_rng(7)
    for _ in range(300):
        hosts = int(rng.integers(2, 12))
        n = int(rng.integers(1, 40))
        src = rng.integers(0, hosts, n)
        dst = (src + rng.integers(1, hosts, n)) % hosts if hosts > 1 else src
        ncls = int(rng.integers(1, 5))
        cls_of = rng.integers(0, ncls, n)
        caps = np.where(rng.random(n) < 0.4, rng.random(n) * 0.5, np.nan)
        if rng.random() < 0.3:  # caps near a link share
            k = max(1, int(rng.integers(1, 8)))
            caps = np.where(np.isnan(caps), caps, np.nextafter(1.0 / k, np.inf))
        want = ref_alloc(hosts, 1.0, src, dst, cls_of, ncls, caps)
        got = emu_alloc(hosts, 1.0, src, dst, cls_of, ncls, caps, variant)
        assert same_bits(got, want)
