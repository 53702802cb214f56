"""Helpers that build in-process worlds on the nvlink transport (the analogue of the
reference's sim_world / sim_nodes fixtures, pkg/tests/conftest.py:7-24)."""

import time
import uuid

from paper_2101_08878_b200.channels import build_comm_table
from paper_2101_08878_b200.endpoints import Node
from paper_2101_08878_b200.loop import MonotonicClock, TaskLoop
from paper_2101_08878_b200.transport import TransportConfig, transport_init


def new_session() -> str:
    return "t" + uuid.uuid4().hex[:12]


def nvlink_transports(n, device=-1, session=None, **cfg):
    session = session or new_session()
    ts = [transport_init(n, r, TransportConfig(kind="nvlink", session=session, device=device, **cfg))
          for r in range(n)]
    for t in ts:
        t.wait_ready(5.0)
    return ts


def nvlink_world(n, device=-1, **cfg):
    loop = TaskLoop(MonotonicClock())
    ts = nvlink_transports(n, device, **cfg)
    tables = [build_comm_table(t) for t in ts]
    return loop, ts, tables


def nvlink_nodes(n, device=-1, max_chunk=None, cache_capacity=None, **cfg):
    loop = TaskLoop(MonotonicClock())
    ts = nvlink_transports(n, device, **cfg)
    nodes = [Node(t, build_comm_table(t, cache_capacity=cache_capacity), max_chunk=max_chunk) for t in ts]
    return loop, nodes


def pump(transports, *requests, timeout=20.0):
    deadline = time.monotonic() + timeout
    while any(r.pending for r in requests):
        for t in transports:
            t.progress()
        if time.monotonic() > deadline:
            raise AssertionError(f"requests stuck: {requests}")


def close_all(transports):
    for t in transports:
        t.close()
