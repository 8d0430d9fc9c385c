"""mfsim-b200: B200-native flow-level simulator hot path of MFS (arXiv 2603.17456).

The per-event scheduling step of the reference simulator (Engine::run and the
policy / allocator / RMLQ / Algorithm 1 code it drives) runs on sm_100a, one
warp per independent simulation instance, behind the reference's C ABI
(``include/mfsim.h``) and a device batch ABI (``include/mfsim_dev.h``).
"""
from .native import (  # noqa: F401
    Config,
    DeviceBatch,
    MfsimError,
    Native,
    SimResult,
    mfsim_run,
    product,
    run_config,
    run_manual,
)

POLICIES = ("fs", "sjf", "edf", "karuna", "mfs")
