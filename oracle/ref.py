"""ORACLE / TEST INFRASTRUCTURE ONLY -- ctypes view of oracle/_ref/libmfsim_ref.so.

The library is the unmodified reference simulator (/root/reference/proj/src/core)
compiled in place by oracle/Makefile, plus ref_harness.cpp. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmfsim_ref.so")
ORACLE_SO = os.path.join(HERE, "_ref", "libmfsim_oracle.so")


class _RefResult(C.Structure):
    _fields_ = [
        ("events", C.c_long),
        ("steps", C.c_long),
        ("pruned_count", C.c_long),
        ("n_req", C.c_int),
        ("n_flows", C.c_int),
        ("n_coflows", C.c_int),
        ("n_batches", C.c_int),
        ("t_run_s", C.c_double),
        ("t_setup_s", C.c_double),
        ("req_arrival", C.POINTER(C.c_double)),
        ("req_deadline", C.POINTER(C.c_double)),
        ("req_done", C.POINTER(C.c_double)),
        ("req_pruned", C.POINTER(C.c_ubyte)),
        ("req_stall", C.POINTER(C.c_double)),
        ("req_batch", C.POINTER(C.c_int)),
        ("flow_finish", C.POINTER(C.c_double)),
        ("flow_band", C.POINTER(C.c_int)),
        ("flow_level", C.POINTER(C.c_int)),
        ("cof_release", C.POINTER(C.c_double)),
        ("cof_done", C.POINTER(C.c_double)),
        ("cof_stall", C.POINTER(C.c_double)),
        ("pipe_done", C.POINTER(C.c_double)),
        ("summary_json", C.c_char_p),
        ("requests_csv", C.c_char_p),
        ("err", C.c_int),
        ("errmsg", C.c_char * 512),
    ]


@dataclass
class SimResult:
    """Full-precision run result; the same shape the B200 engine returns."""

    events: int = 0
    steps: int = 0
    pruned_count: int = 0
    n_batches: int = 0
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
    t_run_s: float = 0.0
    t_setup_s: float = 0.0

    @property
    def slo_met(self) -> np.ndarray:
        # metrics.cpp:32-40: (done - arrival) <= (deadline - arrival)
        done = self.req_done
        ok = ~np.isnan(done)
        met = np.zeros(done.shape, bool)
        met[ok] = (done[ok] - self.req_arrival[ok]) <= (self.req_deadline[ok] - self.req_arrival[ok])
        return met

    @property
    def attainment(self):
        n = len(self.req_done)
        return None if n == 0 else float(self.slo_met.sum()) / n


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_libs = {}


def lib(so: str = REF_SO):
    """the reference library (default) or the C restatement (ORACLE_SO)"""
    if so not in _libs:
        if not os.path.exists(so):
            raise FileNotFoundError(f"{so} missing: run `make -C oracle`")
        L = C.CDLL(so)
        for fn in ("ref_run_config", "ref_run_manual", "ref_derive_deadlines"):
            getattr(L, fn).argtypes = [C.c_char_p, C.POINTER(C.POINTER(_RefResult))]
            getattr(L, fn).restype = C.c_int
        L.ref_free.argtypes = [C.POINTER(_RefResult)]
        if hasattr(L, "ref_allocate_star"):
            L.ref_allocate_star.restype = C.c_int
        _libs[so] = L
    return _libs[so]


def available(so: str = REF_SO) -> bool:
    return os.path.exists(so)


def _convert(p, so=REF_SO) -> SimResult:
    r = p.contents
    if r.err:
        code, msg = r.err, r.errmsg.decode()
        lib(so).ref_free(p)
        raise RefError(code, msg)
    out = SimResult(
        events=r.events,
        steps=r.steps,
        pruned_count=r.pruned_count,
        n_batches=r.n_batches,
        req_arrival=_arr(r.req_arrival, r.n_req, np.float64),
        req_deadline=_arr(r.req_deadline, r.n_req, np.float64),
        req_done=_arr(r.req_done, r.n_req, np.float64) if r.req_done else np.zeros(0),
        req_pruned=_arr(r.req_pruned, r.n_req, np.uint8) if r.req_pruned else np.zeros(0, np.uint8),
        req_stall=_arr(r.req_stall, r.n_req, np.float64) if r.req_stall else np.zeros(0),
        req_batch=_arr(r.req_batch, r.n_req, np.int32) if r.req_batch else np.zeros(0, np.int32),
        flow_finish=_arr(r.flow_finish, r.n_flows, np.float64),
        flow_band=_arr(r.flow_band, r.n_flows, np.int32),
        flow_level=_arr(r.flow_level, r.n_flows, np.int32),
        cof_release=_arr(r.cof_release, r.n_coflows, np.float64),
        cof_done=_arr(r.cof_done, r.n_coflows, np.float64),
        cof_stall=_arr(r.cof_stall, r.n_coflows, np.float64),
        pipe_done=_arr(r.pipe_done, r.n_batches, np.float64),
        summary_json=(r.summary_json or b"").decode(),
        requests_csv=(r.requests_csv or b"").decode(),
        t_run_s=r.t_run_s,
        t_setup_s=r.t_setup_s,
    )
    lib(so).ref_free(p)
    return out


def run_config(text: str, so: str = REF_SO) -> SimResult:
    p = C.POINTER(_RefResult)()
    lib(so).ref_run_config(text.encode(), C.byref(p))
    return _convert(p, so)


def run_manual(spec: str, so: str = REF_SO) -> SimResult:
    p = C.POINTER(_RefResult)()
    lib(so).ref_run_manual(spec.encode(), C.byref(p))
    return _convert(p, so)


def derive_deadlines(text: str, so: str = REF_SO):
    p = C.POINTER(_RefResult)()
    lib(so).ref_derive_deadlines(text.encode(), C.byref(p))
    r = _convert(p, so)
    return r.req_arrival, r.req_deadline


def allocate_star(hosts, cap, src, dst, cls_of, ncls, caps=None):
    n = len(src)
    src = np.ascontiguousarray(src, np.int32)
    dst = np.ascontiguousarray(dst, np.int32)
    cls_of = np.ascontiguousarray(cls_of, np.int32)
    out = np.zeros(n, np.float64)
    cp = None
    if caps is not None:
        caps = np.ascontiguousarray(caps, np.float64)
        cp = caps.ctypes.data_as(C.POINTER(C.c_double))
    rc = lib().ref_allocate_star(
        C.c_int(hosts), C.c_double(cap), C.c_int(n),
        src.ctypes.data_as(C.POINTER(C.c_int)), dst.ctypes.data_as(C.POINTER(C.c_int)),
        cls_of.ctypes.data_as(C.POINTER(C.c_int)), C.c_int(ncls), cp,
        out.ctypes.data_as(C.POINTER(C.c_double)))
    if rc:
        raise RefError(rc, "allocate_star failed")
    return out
