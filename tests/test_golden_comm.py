"""Comm-path parity pinned to golden vectors generated from the reference itself
(oracle/make_golden.py imports /root/reference/pkg/src in the build container)."""

import json
import os

import pytest

from paper_2101_08878_b200 import channels, endpoints, messaging
from paper_2101_08878_b200.loop import TaskLoop, gather
from paper_2101_08878_b200.messaging import Message, make_frame
from paper_2101_08878_b200.transport import LinkModel, MemoryDomain, SimFabric, tcp

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_comm.json")))


def test_socket_frame_headers_match_reference_bytes():
    for case in GOLDEN["frame_headers"]:
        got = tcp.pack_frame_header(case["channel"], case["tag"], case["domain"], case["length"])
        assert got.hex() == case["hex"]


def _messages():
    return {
        "empty": Message([]),
        "two_host": Message([make_frame(b"abc"), make_frame(b"fghij")]),
        "mixed": Message([make_frame(b"\x00\x01", 0), make_frame("héllo", 1), make_frame([1.5, -2.25, 3.0], 2),
                          make_frame(b"dev", 0, MemoryDomain.DEVICE_SIM)]),
    }


def test_message_and_transfer_headers_match_reference_bytes():
    for name, msg in _messages().items():
        assert messaging._pack_message_header(msg).hex() == GOLDEN["message_headers"][name]
    for case in GOLDEN["transfer_headers"]:
        assert messaging._TRANSFER_HEADER.pack(case["length"], case["ser"], case["domain"]).hex() == case["hex"]
    assert messaging._COUNT.pack(messaging._EOS_SENTINEL).hex() == GOLDEN["eos"]


def test_serializer_encodings_match_reference():
    import math

    assert messaging.SERIALIZERS[1][0]("héllo wörld").hex() == GOLDEN["serializers"]["utf8"]
    assert messaging.SERIALIZERS[2][0]([1.5, -2.25, 3.0, math.pi]).hex() == GOLDEN["serializers"]["f64"]
    assert messaging.SERIALIZERS[0][0](bytearray(b"raw\x00bytes")).hex() == GOLDEN["serializers"]["raw"]


def test_chunk_plans_match_reference():
    for case in GOLDEN["chunk_plans"]:
        got = [list(s) for s in messaging.chunk_plan(case["total"], case["max_chunk"]).slices]
        assert got == case["slices"]


def test_channel_ids_match_reference():
    for n, grid in GOLDEN["base_channel_ids"].items():
        n = int(n)
        for i in range(n):
            for j in range(n):
                if i != j:
                    assert channels.base_channel_id(n, i, j) == grid[i][j]
    for base, gen, want in GOLDEN["duplicate_ids"]:
        assert channels.duplicate_channel_id(base, gen) == want


def test_duplicate_cache_trace_matches_reference():
    import random

    fab = SimFabric(2)
    fab.transport(1)
    table = channels.build_comm_table(fab.transport(0), cache_capacity=GOLDEN["dup_cache_trace"]["capacity"])
    rng = random.Random(GOLDEN["dup_cache_trace"]["seed"])
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
    assert trace == GOLDEN["dup_cache_trace"]["trace"]
    assert table.cache_hits(1) == GOLDEN["dup_cache_trace"]["hits"]


def test_handshake_bytes_match_reference():
    assert endpoints._PROPOSAL.pack((2 << 20) | 5).hex() == GOLDEN["handshake"]["proposal"]
    assert endpoints._REPLY.pack((2 << 20) | 5, 3).hex() == GOLDEN["handshake"]["reply"]
    assert endpoints._EOS_HEADER.hex() == GOLDEN["handshake"]["eos"]


def test_socket_wire_stream_matches_reference():
    t1 = tcp.SocketTransport(2, 1, {0: ("127.0.0.1", 0), 1: ("127.0.0.1", 0)})
    try:
        msg = _messages()["mixed"]
        t1.post_send(0, 0, messaging.MESSAGE_TAG, messaging._pack_message_header(msg))
        for i, f in enumerate(msg.frames):
            t1.post_send(0, 0, messaging.data_tag(i), f.to_bytes(), f.domain)
        stream = b"".join(bytes(item.data) for item in t1._outq[0])
        assert stream.hex() == GOLDEN["socket_stream_mixed_message"]
    finally:
        t1.close()


def test_sim_pingpong_virtual_ticks_match_reference():
    lat, bw, ovh = GOLDEN["sim_pingpong_ticks"]["link"]
    loop = TaskLoop()
    fab = SimFabric(2, link=LinkModel(latency=lat, bandwidth=bw, per_chunk_overhead=ovh), clock=loop.clock)
    ts = [fab.transport(r) for r in range(2)]
    tables = [channels.build_comm_table(t) for t in ts]

    async def pingpong():
        rows = []
        for size in (0, 1, 100, 4096):
            t0 = loop.clock.now()
            _, frame = await gather(messaging.send_payload(ts[0], tables[0].lookup(1), 50, make_frame(b"x" * size)),
                                    messaging.recv_payload(ts[1], tables[1].lookup(0), 50))
            rows.append([size, loop.clock.now() - t0, frame.length])
        return rows

    assert loop.run_until_complete(pingpong()) == GOLDEN["sim_pingpong_ticks"]["rows"]
