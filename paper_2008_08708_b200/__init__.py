"""B200-native executor for SCCL-synthesized collective schedules.

Hot path (BASELINE.json north_star): a canonical synthesized schedule
 is verified and lowered by the C++ host library to a
per-rank, per-channel program, and executed by hand-written sm_100a kernels
that push chunks into peer memory with per-(receipt, channel) flags and fuse
the reduction into the receive.  Entry points: ``sccl`` (ctypes binding of
include/sccl_exec.h) and ``schedules`` (known-answer / constructive
schedules).
"""
from . import sccl  # noqa: F401  (fails loudly if the extension is missing)

__all__ = ["sccl", "schedules"]
