"""Bit-exactness of long single instances at an event cut.

BASELINE configs[2] Karuna (ft128, 100k requests, ~24.3M events) needs more
device time on one warp than one GPU box call allows. The state after exactly
B events is a deterministic function of B, so the B200 run and the serial
build of the same engine (which is bit-exact against the reference over the
WHOLE run, profiles/r02_emu_config3_karuna.log) are compared at that cut:
every per-request done time, every flow's finish time,
band and level, every coflow's release / done time and every batch's
pipeline-done time, as sha256 digests.

  python tools/karuna_cut.py gpu MINUTES OUT.json    (product library; stops at
        the largest multiple of the chunk that fits the time)
  python tools/karuna_cut.py emu IN.json             (build/libmfsim_emu.so at
        the same cut; compares)"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from parity import digest  # noqa: E402
from paper_2603_17456_b200 import configs  # noqa: E402
from paper_2603_17456_b200.native import DeviceBatch, Native, product  # noqa: E402

SEEDS = (1, 2, 3)
CHUNK = 250_000
KEYS = ("req_done", "flow_finish", "flow_band", "flow_level",
        "cof_release", "cof_done", "pipe_done")


def batch(lib):
    b = DeviceBatch(0, lib)
    for s in SEEDS:
        b.add_config(configs.config3(seed=s, policy="karuna"))
    b.prepare()
    b.upload()
    b.reset()
    return b


def digests(b):
    b.download(2)
    out = {}
    for i, s in enumerate(SEEDS):
        r = b.result(i, 2)
        st = b.stats(i)
        out[str(s)] = {"events": int(st.events), "steps": int(st.steps),
                       **{k: digest(getattr(r, k)) for k in KEYS}}
    return out


def main():
    mode = sys.argv[1]
    if mode == "gpu":
        minutes, path = float(sys.argv[2]), sys.argv[3]
        b = batch(product())
        t0 = time.time()
        cut = 0
        while b.remaining() > 0:
            b.launch_budget(CHUNK)
            b.sync()
            cut += CHUNK
            el = time.time() - t0
            per = el / cut
            print(f"cut {cut} events per instance, {el:.0f} s", flush=True)
            if el + per * CHUNK * 1.2 > minutes * 60:
                break
        res = {"cut": cut, "device_s": time.time() - t0, "digests": digests(b)}
        json.dump(res, open(path, "w"), indent=1)
        print(json.dumps(res)[:400])
    else:
        want = json.load(open(sys.argv[2]))
        b = batch(Native(os.path.join(ROOT, "build", "libmfsim_emu.so")))
        t0 = time.time()
        b.launch_budget(want["cut"])
        got = digests(b)
        bad = {s: [k for k in got[s] if got[s][k] != want["digests"][s][k]] for s in got}
        print(f"cut {want['cut']} events (device {want['device_s']:.0f} s, serial build {time.time() - t0:.0f} s):",
              "bit-exact" if not any(bad.values()) else f"MISMATCH {bad}")
        for s in got:
            print(f"  seed {s}: events {got[s]['events']}, steps {got[s]['steps']}, "
                  f"{'all digests equal' if not bad[s] else bad[s]}")


if __name__ == "__main__":
    main()
