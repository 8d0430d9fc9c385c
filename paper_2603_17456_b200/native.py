"""ctypes binding of the mfsim-b200 C ABI (include/mfsim.h + include/mfsim_dev.h).

The product loads ``paper_2603_17456_b200/libmfsim_b200.so`` -- the sm_100a
engine. If that library is missing the import of the API fails loudly; there is
no CPU fallback. ``Native(path)`` can also bind the test-only host-emulation
build (``build/libmfsim_emu.so``) so the CPU test tier can check engine logic.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PRODUCT_SO = os.path.join(HERE, "libmfsim_b200.so")

ERR_NAMES = {1: "INVALID_ARG", 2: "CONFIG", 3: "WORKLOAD", 4: "IO", 5: "SIM", 6: "INTERNAL"}


class MfsimError(RuntimeError):
    """A failing C-ABI call; ``code`` is the mfsim.h error code."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"mfsim error {code} ({ERR_NAMES.get(code, '?')}): {msg}")
        self.code = code


class DevStats(C.Structure):
    _fields_ = [(n, C.c_longlong) for n in (
        "status", "check", "events", "steps", "flows", "batches", "coflows", "pruned",
        "max_active", "pushes", "algo_bytes", "requests", "finished", "slo_met", "classes",
        "rounds")]


@dataclass
class SimResult:
    """Full-precision results of one instance (RunResult, engine.hpp:107-113)."""

    events: int = 0
    steps: int = 0
    pruned_count: int = 0
    n_batches: int = 0
    max_active: int = 0
    pushes: int = 0
    algo_bytes: int = 0
    status: int = 0
    check: int = 0
    req_arrival: np.ndarray = field(default_factory=lambda: np.zeros(0))
    req_deadline: np.ndarray = field(default_factory=lambda: np.zeros(0))
    req_done: np.ndarray = field(default_factory=lambda: np.zeros(0))
    req_pruned: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    req_stall: np.ndarray = field(default_factory=lambda: np.zeros(0))
    req_batch: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    flow_finish: np.ndarray = field(default_factory=lambda: np.zeros(0))
    flow_band: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    flow_level: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    cof_release: np.ndarray = field(default_factory=lambda: np.zeros(0))
    cof_done: np.ndarray = field(default_factory=lambda: np.zeros(0))
    cof_stall: np.ndarray = field(default_factory=lambda: np.zeros(0))
    pipe_done: np.ndarray = field(default_factory=lambda: np.zeros(0))
    summary_json: str = ""
    requests_csv: str = ""

    @property
    def slo_met(self) -> np.ndarray:
        done = self.req_done
        ok = ~np.isnan(done)
        met = np.zeros(done.shape, bool)
        met[ok] = (done[ok] - self.req_arrival[ok]) <= (self.req_deadline[ok] - self.req_arrival[ok])
        return met

    @property
    def attainment(self):
        n = len(self.req_done)
        return None if n == 0 else float(self.slo_met.sum()) / n


class Native:
    def __init__(self, path: str = PRODUCT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the B200 engine has no CPU fallback)")
        self.path = path
        L = self.lib = C.CDLL(path)
        vp, cp, i, ll = C.c_void_p, C.c_char_p, C.c_int, C.c_longlong
        dp = C.POINTER(C.c_double)
        sig = {
            "mfsim_version": ([], cp), "mfsim_last_error": ([], cp),
            "mfsim_config_create": ([], vp), "mfsim_config_load": ([cp], vp),
            "mfsim_config_set": ([vp, cp, cp], i), "mfsim_config_get": ([vp, cp], cp),
            "mfsim_config_destroy": ([vp], None),
            "mfsim_run": ([vp, cp, C.POINTER(C.c_void_p)], i),
            "mfsim_string_free": ([vp], None),
            "mfsim_dev_create": ([i, C.POINTER(vp)], i), "mfsim_dev_destroy": ([vp], None),
            "mfsim_dev_set_stream": ([vp, vp], i),
            "mfsim_dev_add_config": ([vp, vp], i), "mfsim_dev_add_manual": ([vp, cp], i),
            "mfsim_dev_prepare": ([vp], i), "mfsim_dev_upload": ([vp], i),
            "mfsim_dev_launch": ([vp], i), "mfsim_dev_sync": ([vp, dp], i),
            "mfsim_dev_download": ([vp, i], i), "mfsim_dev_run": ([vp, i], i),
            "mfsim_dev_count": ([vp], i), "mfsim_dev_stats_get": ([vp, i, C.POINTER(DevStats)], i),
            "mfsim_dev_h2d_bytes": ([vp], ll), "mfsim_dev_d2h_bytes": ([vp], ll),
            "mfsim_dev_device_bytes": ([vp], ll), "mfsim_dev_kernel_launches": ([vp], i),
            "mfsim_dev_last_kernel": ([vp], cp),
            "mfsim_dev_requests": ([vp, i, vp, vp, vp, vp, vp, vp, C.c_long], i),
            "mfsim_dev_flows": ([vp, i, vp, vp, vp, C.c_long], i),
            "mfsim_dev_coflows": ([vp, i, vp, vp, vp, C.c_long], i),
            "mfsim_dev_batches": ([vp, i, vp, C.c_long], i),
            "mfsim_dev_summary_json": ([vp, i, C.POINTER(C.c_void_p)], i),
            "mfsim_dev_requests_csv": ([vp, i, C.POINTER(C.c_void_p)], i),
            "mfsim_dev_write_report": ([vp, i, cp], i),
            "mfsim_route": ([vp, i, i, vp, vp, i, C.POINTER(i)], i),
            "mfsim_dev_counters": ([vp, i, vp, i], i),
            "mfsim_dev_reset": ([vp], i), "mfsim_dev_upload_inputs": ([vp], i), "mfsim_dev_launch_budget": ([vp, ll], i),
            "mfsim_dev_remaining": ([vp], i), "mfsim_dev_launch_slice": ([vp, ll], i),
            "mfsim_link_count": ([vp, C.POINTER(i)], i),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res

    def check(self, rc: int):
        if rc != 0:
            raise MfsimError(rc, (self.lib.mfsim_last_error() or b"").decode())

    def take_string(self, p: C.c_void_p) -> str:
        s = C.cast(p, C.c_char_p).value.decode()
        self.lib.mfsim_string_free(p)
        return s


_product = None


def product() -> Native:
    """The sm_100a product library (raises if it was not built)."""
    global _product
    if _product is None:
        _product = Native(PRODUCT_SO)
    return _product


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Config:
    """mfsim_config handle (mfsim.h:22-42)."""

    def __init__(self, text: str | dict | None = None, lib: Native | None = None):
        self.n = lib or product()
        self.h = self.n.lib.mfsim_config_create()
        if isinstance(text, dict):
            for k, v in text.items():
                self.set(k, v)
        elif text:
            for line in text.splitlines():
                line = line.split("#", 1)[0].strip()
                if not line:
                    continue
                if "=" not in line:
                    raise MfsimError(2, f"expected key = value, got '{line}'")
                k, v = line.split("=", 1)
                self.set(k.strip(), v.strip())

    def set(self, key: str, value) -> "Config":
        self.n.check(self.n.lib.mfsim_config_set(self.h, key.encode(), str(value).encode()))
        return self

    def get(self, key: str):
        v = self.n.lib.mfsim_config_get(self.h, key.encode())
        return None if v is None else v.decode()

    def __del__(self):
        try:
            self.n.lib.mfsim_config_destroy(self.h)
        except Exception:
            pass


class DeviceBatch:
    """Many independent instances run by the device engine in one launch."""

    def __init__(self, device: int = 0, lib: Native | None = None, stream=None):
        self.n = lib or product()
        h = C.c_void_p()
        self.n.check(self.n.lib.mfsim_dev_create(device, C.byref(h)))
        self.h = h
        self._keep = []
        if stream is not None:
            self.set_stream(stream)

    def set_stream(self, stream_ptr: int):
        self.n.check(self.n.lib.mfsim_dev_set_stream(self.h, C.c_void_p(stream_ptr)))

    def add_config(self, cfg) -> "DeviceBatch":
        if not isinstance(cfg, Config):
            cfg = Config(cfg, self.n)
        self._keep.append(cfg)
        self.n.check(self.n.lib.mfsim_dev_add_config(self.h, cfg.h))
        return self

    def add_manual(self, spec: str) -> "DeviceBatch":
        self.n.check(self.n.lib.mfsim_dev_add_manual(self.h, spec.encode()))
        return self

    def prepare(self):
        self.n.check(self.n.lib.mfsim_dev_prepare(self.h))

    def upload(self):
        self.n.check(self.n.lib.mfsim_dev_upload(self.h))

    def launch(self):
        self.n.check(self.n.lib.mfsim_dev_launch(self.h))

    def upload_inputs(self):
        self.n.check(self.n.lib.mfsim_dev_upload_inputs(self.h))

    def reset(self):
        self.n.check(self.n.lib.mfsim_dev_reset(self.h))

    def launch_budget(self, budget: int):
        self.n.check(self.n.lib.mfsim_dev_launch_budget(self.h, budget))

    def launch_slice(self, slice_ns: int):
        self.n.check(self.n.lib.mfsim_dev_launch_slice(self.h, slice_ns))

    def remaining(self) -> int:
        return self.n.lib.mfsim_dev_remaining(self.h)

    def sync(self) -> float:
        ms = C.c_double(0.0)
        self.n.check(self.n.lib.mfsim_dev_sync(self.h, C.byref(ms)))
        return ms.value

    def download(self, detail: int = 0):
        self.n.check(self.n.lib.mfsim_dev_download(self.h, detail))

    def run(self, detail: int = 2):
        self.n.check(self.n.lib.mfsim_dev_run(self.h, detail))

    def __len__(self):
        return self.n.lib.mfsim_dev_count(self.h)

    @property
    def h2d_bytes(self):
        return self.n.lib.mfsim_dev_h2d_bytes(self.h)

    @property
    def d2h_bytes(self):
        return self.n.lib.mfsim_dev_d2h_bytes(self.h)

    @property
    def device_bytes(self):
        return self.n.lib.mfsim_dev_device_bytes(self.h)

    @property
    def kernel_launches(self):
        return self.n.lib.mfsim_dev_kernel_launches(self.h)

    @property
    def last_kernel(self) -> str:
        return self.n.lib.mfsim_dev_last_kernel(self.h).decode()

    def stats(self, i: int) -> DevStats:
        s = DevStats()
        self.n.check(self.n.lib.mfsim_dev_stats_get(self.h, i, C.byref(s)))
        return s

    def result(self, i: int, detail: int = 2, reports: bool = False) -> SimResult:
        st = self.stats(i)
        nr = int(st.requests)
        arr, dl, done = np.zeros(nr), np.zeros(nr), np.zeros(nr)
        pr, stall, rb = np.zeros(nr, np.uint8), np.zeros(nr), np.zeros(nr, np.int32)
        self.n.check(self.n.lib.mfsim_dev_requests(self.h, i, _ptr(arr), _ptr(dl), _ptr(done),
                                                    _ptr(pr), _ptr(stall), _ptr(rb), nr))
        done = np.where(done == -1.0, np.nan, done)
        r = SimResult(events=st.events, steps=st.steps, pruned_count=st.pruned,
                      n_batches=st.batches, max_active=st.max_active, pushes=st.pushes,
                      algo_bytes=st.algo_bytes, status=st.status, check=st.check,
                      req_arrival=arr, req_deadline=dl, req_done=done, req_pruned=pr,
                      req_stall=stall, req_batch=rb)
        if detail >= 1:
            nc = int(st.coflows)
            r.cof_release, r.cof_done, r.cof_stall = np.zeros(nc), np.zeros(nc), np.zeros(nc)
            self.n.check(self.n.lib.mfsim_dev_coflows(self.h, i, _ptr(r.cof_release),
                                                       _ptr(r.cof_done), _ptr(r.cof_stall), nc))
        if detail >= 2:
            nf = int(st.flows)
            fin, band, lev = np.zeros(nf), np.zeros(nf, np.uint8), np.zeros(nf, np.uint8)
            self.n.check(self.n.lib.mfsim_dev_flows(self.h, i, _ptr(fin), _ptr(band), _ptr(lev), nf))
            r.flow_finish, r.flow_band, r.flow_level = fin, band.astype(np.int32), lev.astype(np.int32)
            nb = int(st.batches)
            r.pipe_done = np.zeros(nb)
            self.n.check(self.n.lib.mfsim_dev_batches(self.h, i, _ptr(r.pipe_done), nb))
        if reports and st.status == 0:
            p = C.c_void_p()
            self.n.check(self.n.lib.mfsim_dev_summary_json(self.h, i, C.byref(p)))
            r.summary_json = self.n.take_string(p)
            self.n.check(self.n.lib.mfsim_dev_requests_csv(self.h, i, C.byref(p)))
            r.requests_csv = self.n.take_string(p)
        return r

    def counters(self, i: int) -> np.ndarray:
        out = np.zeros(64, np.int64)
        n = self.n.lib.mfsim_dev_counters(self.h, i, _ptr(out), 64)
        return out[:max(n, 0)]

    def raise_for_status(self, i: int):
        st = self.stats(i)
        if st.status:
            raise MfsimError(int(st.status), f"instance {i} failed device check {st.check}")

    def __del__(self):
        try:
            self.n.lib.mfsim_dev_destroy(self.h)
        except Exception:
            pass


def route(cfg, src: int, dst: int, lib: Native | None = None):
    """Link ids and capacities of the route src -> dst (Topology::route)."""
    n = lib or product()
    if not isinstance(cfg, Config):
        cfg = Config(cfg, n)
    size = 64
    while True:
        links, caps, cnt = np.zeros(size, np.int32), np.zeros(size), C.c_int(0)
        n.check(n.lib.mfsim_route(cfg.h, src, dst, _ptr(links), _ptr(caps), size, C.byref(cnt)))
        if cnt.value <= size:
            return links[:cnt.value].tolist(), caps[:cnt.value].tolist()
        size = cnt.value  # a longer route than the buffers: call again with room for it


def link_count(cfg, lib: Native | None = None) -> int:
    n = lib or product()
    if not isinstance(cfg, Config):
        cfg = Config(cfg, n)
    cnt = C.c_int(0)
    n.check(n.lib.mfsim_link_count(cfg.h, C.byref(cnt)))
    return cnt.value


def run_config(text, device: int = 0, detail: int = 2, lib: Native | None = None) -> SimResult:
    """One workload-mode simulation on the device (run_simulation, sim_api.cpp:8-35)."""
    b = DeviceBatch(device, lib)
    b.add_config(text)
    b.prepare()
    b.run(detail)
    b.raise_for_status(0)
    return b.result(0, detail, reports=detail >= 1)


def run_manual(spec: str, device: int = 0, lib: Native | None = None) -> SimResult:
    """One manual instance (engine.hpp:124-133 add_* API as a text spec)."""
    b = DeviceBatch(device, lib)
    b.add_manual(spec)
    b.prepare()
    b.run(2)
    b.raise_for_status(0)
    return b.result(0, 2, reports=True)


def mfsim_run(text, out_dir: str | None = None, lib: Native | None = None) -> str:
    """The reference C entry point mfsim_run (mfsim.h:52); returns summary.json."""
    n = lib or product()
    cfg = Config(text, n)
    p = C.c_void_p()
    n.check(n.lib.mfsim_run(cfg.h, out_dir.encode() if out_dir else None, C.byref(p)))
    return n.take_string(p)
