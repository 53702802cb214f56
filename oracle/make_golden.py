#!/usr/bin/env python3
"""Generate tests/golden/*.json from the REFERENCE implementation (TEST INFRASTRUCTURE).

Runs only in the build container, where /root/reference exists: it imports the
reference ``commshim`` package from /root/reference/pkg/src (read-only, never
copied) and records byte-level outputs of its comm path, so the parity tests
can pin this repo's drop-in against the reference on the GPU box too, where
/root/reference is absent.  Operator examples come from SPEC.md:418-430
(the reference has no operator code).

    python oracle/make_golden.py            # writes tests/golden/
"""

from __future__ import annotations

import json
import math
import os
import random
import sys

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def main() -> None:
    if not os.path.isdir(REF_SRC):
        raise SystemExit(f"{REF_SRC} not found: golden vectors can only be regenerated in the build container")
    sys.path.insert(0, REF_SRC)
    for name in [m for m in sys.modules if m == "commshim" or m.startswith("commshim.")]:
        del sys.modules[name]
    import commshim  # noqa: F401  (the reference)
    from commshim import channels, messaging
    from commshim.loop import TaskLoop
    from commshim.messaging import Message, make_frame
    from commshim.transport import SimFabric
    from commshim.transport import tcp

    assert commshim.__file__.startswith(REF_SRC), commshim.__file__
    golden: dict = {"source": "reference commshim 0.1.0 at /root/reference/pkg/src (oracle/make_golden.py)"}

    # socket frame headers (tcp.py:45-56)
    golden["frame_headers"] = [
        {"channel": c, "tag": t, "domain": d, "length": n, "hex": tcp.pack_frame_header(c, t, d, n).hex()}
        for c, t, d, n in [(0, 0, 0, 8), (3, 100, 1, 5), (65537, 2**31 - 1, 0, 2**31 - 1), (1, 16, 1, 0),
                           (0xFFFFFFFF, 17, 0, 2**40)]
    ]

    # message headers (messaging.py:325-333) and transfer headers (:47, :300)
    msgs = {
        "empty": Message([]),
        "two_host": Message([make_frame(b"abc"), make_frame(b"fghij")]),
        "mixed": Message([make_frame(b"\x00\x01", 0), make_frame("héllo", 1), make_frame([1.5, -2.25, 3.0], 2),
                          make_frame(b"dev", 0, messaging.MemoryDomain.DEVICE_SIM)]),
    }
    golden["message_headers"] = {k: messaging._pack_message_header(m).hex() for k, m in msgs.items()}
    golden["transfer_headers"] = [
        {"length": n, "ser": s, "domain": d, "hex": messaging._TRANSFER_HEADER.pack(n, s, d).hex()}
        for n, s, d in [(0, 0, 0), (10, 2, 1), (2**33 + 7, 255, 0)]
    ]
    golden["eos"] = messaging._COUNT.pack(messaging._EOS_SENTINEL).hex()
    golden["serializers"] = {
        "utf8": messaging.SERIALIZERS[1][0]("héllo wörld").hex(),
        "f64": messaging.SERIALIZERS[2][0]([1.5, -2.25, 3.0, math.pi]).hex(),
        "raw": messaging.SERIALIZERS[0][0](bytearray(b"raw\x00bytes")).hex(),
    }

    # chunk plans (messaging.py:167-186)
    rng = random.Random(20261018)
    cases = [(0, 1024), (3_500_000_000, 2**30), (2**30, 2**30), (10, 4), (10, 3), (1, 1)]
    cases += [(rng.randrange(0, 1 << 34), rng.randrange(1, 1 << 31)) for _ in range(40)]
    golden["chunk_plans"] = [{"total": t, "max_chunk": m, "slices": [list(s) for s in messaging.chunk_plan(t, m).slices]}
                             for t, m in cases]

    # channel ids (channels.py:35-47, 183-206)
    golden["base_channel_ids"] = {str(n): [[channels.base_channel_id(n, i, j) if i != j else 0 for j in range(n)]
                                           for i in range(n)] for n in range(2, 9)}
    golden["duplicate_ids"] = [[b, g, channels.duplicate_channel_id(b, g)] for b, g in
                               [(1, 1), (1, 2), (6, 65535), (28, 17), (100, 3)]]
    # allocation sequence of generations with release/reuse (deterministic, seed 7 as test_channels.py:169)
    fab = SimFabric(2)
    fab.transport(1)
    table = channels.build_comm_table(fab.transport(0), cache_capacity=3)
    rng = random.Random(7)
    live, trace = [], []
    for _ in range(200):
        if live and rng.random() < 0.5:
            ch = live.pop(rng.randrange(len(live)))
            table.release(ch)
            trace.append(["release", ch.id])
        else:
            ch = table.duplicate(1)
            live.append(ch)
            trace.append(["dup", ch.id, ch.generation])
    golden["dup_cache_trace"] = {"capacity": 3, "seed": 7, "trace": trace, "hits": table.cache_hits(1)}

    # endpoint handshake bytes (endpoints.py:44-45)
    from commshim import endpoints

    golden["handshake"] = {"proposal": endpoints._PROPOSAL.pack((2 << 20) | 5).hex(),
                           "reply": endpoints._REPLY.pack((2 << 20) | 5, 3).hex(),
                           "eos": endpoints._EOS_HEADER.hex()}

    # full per-post wire stream of one message through the reference socket transport:
    # header frame + per-frame data frames, exactly as queued (tcp.py:262-275)
    rank_map = {0: ("127.0.0.1", 0), 1: ("127.0.0.1", 0)}
    t1 = tcp.SocketTransport(2, 1, rank_map)
    try:
        t1._dead_peers.clear()
        stream = bytearray()
        msg = msgs["mixed"]
        hdr = messaging._pack_message_header(msg)
        t1.post_send(0, 0, messaging.MESSAGE_TAG, hdr)
        for i, f in enumerate(msg.frames):
            t1.post_send(0, 0, messaging.data_tag(i), f.to_bytes(), f.domain)
        for item in t1._outq[0]:
            stream += bytes(item.data)
        golden["socket_stream_mixed_message"] = stream.hex()
    finally:
        t1.close()

    # sim transcript: ping-pong on the virtual clock (closed-form stamps, sim.py:132-140)
    from commshim.transport import LinkModel

    loop = TaskLoop()
    fab = SimFabric(2, link=LinkModel(latency=1e-6, bandwidth=10**9, per_chunk_overhead=2e-9), clock=loop.clock)
    ts = [fab.transport(r) for r in range(2)]
    tables = [channels.build_comm_table(t) for t in ts]

    async def pingpong():
        stamps = []
        for size in (0, 1, 100, 4096):
            t0 = loop.clock.now()
            a = messaging.send_payload(ts[0], tables[0].lookup(1), 50, make_frame(b"x" * size))
            b = messaging.recv_payload(ts[1], tables[1].lookup(0), 50)
            from commshim.loop import gather

            _, frame = await gather(a, b)
            stamps.append([size, loop.clock.now() - t0, frame.length])
        return stamps

    golden["sim_pingpong_ticks"] = {"link": [1e-6, 10**9, 2e-9], "rows": loop.run_until_complete(pingpong())}

    # operator worked examples (no reference code exists for them)
    golden["spec_examples"] = {
        "transpose_2x2": {"x": [[0, 1], [2, 3]], "y": [[0, 3], [3, 6]], "sum": 12},
        "transpose_symmetric": {"x": [[1, 2], [2, 5]], "y": [[2, 4], [4, 10]], "sum": 20},
        "merge_small": {"left": [1, 2, 3], "right": [2, 3, 4], "rows": 2},
        "merge_fraction_zero_rows": 0,
    }

    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, "reference_comm.json")
    with open(path, "w") as fh:
        json.dump(golden, fh, indent=1, sort_keys=True)
    print(f"wrote {path}")


if __name__ == "__main__":
    main()
