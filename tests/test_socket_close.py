"""Socket transport close semantics (DESIGN.md §6 D4): frames a peer sent before closing
are still delivered -- read together with the EOF, or still queued when close() ran."""

import socket
import time

from paper_2101_08878_b200.transport.tcp import SocketTransport


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def pair():
    rm = {r: ("127.0.0.1", free_port()) for r in range(2)}
    ts = [SocketTransport(2, r, rm, connect_timeout=5.0) for r in range(2)]
    deadline = time.monotonic() + 10
    while not all(t.mesh_ready for t in ts):
        for t in ts:
            t.progress()
        assert time.monotonic() < deadline, "mesh not ready"
        time.sleep(0.0005)
    return ts


def test_frames_sent_before_close_reach_the_peer():
    a, b = pair()
    payloads = [bytes([k]) * (1 + 997 * k) for k in range(40)]  # up to ~39 KB, several socket reads
    sends = [a.post_send(0, 1, 7, p) for p in payloads]
    a.close()  # flushes what is still queued, half-closes, drains
    assert all(not s.pending for s in sends)
    got = []
    deadline = time.monotonic() + 10
    # rank 1 only now looks at its socket: data and EOF arrive in the same drain
    for p in payloads:
        buf = bytearray(len(p))
        r = b.post_recv(0, 0, 7, buf)
        while r.pending:
            b.progress()
            assert time.monotonic() < deadline
        assert not r.failed, r.error
        got.append(bytes(buf))
    assert got == payloads
    # and the close itself is seen: a further receive fails
    r = b.post_recv(0, 0, 7, bytearray(1))
    while r.pending:
        b.progress()
        assert time.monotonic() < deadline
    assert r.failed
    b.close()
