"""B200-native drop-in for the reference ``commshim`` package (MPI4Dask, arXiv 2101.08878).

Same public surface as ``pkg/src/commshim/__init__.py:1-19`` (loop primitives
re-exported, ``errors``), the same module layout (``loop``, ``errors``,
``transport``, ``channels``, ``messaging``, ``endpoints``) plus:

* ``transport.nvlink`` — ``TransportConfig(kind="nvlink")``: GPU frames move
  device-to-device between B200s (CUDA IPC over NVLink), never through host
  memory, driven by the C-ABI library ``libm4d.so``;
* ``harness`` — the paper's two operators (``transpose_sum``, ``key_merge``)
  as hand-written sm_100a kernels, plus the mini cluster (scheduler / client /
  worker roles, heartbeats with suspect marking: ``harness.cluster``);
* ``cli`` — the ``commshim-bench`` / ``commshim-launch`` entry points the
  reference declares (``pkg/pyproject.toml:14-16``), wired in ``pyproject.toml``.

``import commshim`` resolves to this package through the alias package at the
repository root.
"""

from . import errors
from .loop import Event, Future, MonotonicClock, Task, TaskLoop, VirtualClock, gather, sleep, wait_for

__all__ = [
    "Event",
    "Future",
    "MonotonicClock",
    "Task",
    "TaskLoop",
    "VirtualClock",
    "errors",
    "gather",
    "sleep",
    "wait_for",
]

__version__ = "0.1.0"
