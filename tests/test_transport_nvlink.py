"""Contract tests of the nvlink transport (libm4d.so through ctypes).

Every test runs twice: on a host-only context (device=-1; no GPU needed, runs
in the CPU suite) and on cuda:0 (marked gpu).  The properties are those the
reference pins for its transports (pkg/tests/test_transport_sim.py,
test_transport_socket.py): exact-key FIFO, isolation, truncation, cancel,
purge, pending counters, peer failure, startup errors."""

import os
import random

import pytest

from paper_2101_08878_b200.errors import (
    ChannelError,
    CommClosedError,
    ConfigurationError,
    CountOverflowError,
    StartupError,
    TransferError,
    TruncationError,
    UsageError,
)
from paper_2101_08878_b200.transport import TransportConfig, TransferRequest, transport_init

from nvlink_fixtures import close_all, new_session, nvlink_transports, pump

DEVICES = [pytest.param(-1, id="host"), pytest.param(0, id="cuda", marks=pytest.mark.gpu)]


@pytest.fixture(params=DEVICES)
def pair(request):
    ts = nvlink_transports(2, device=request.param)
    yield ts
    close_all(ts)


@pytest.fixture(params=DEVICES)
def trio(request):
    ts = nvlink_transports(3, device=request.param)
    yield ts
    close_all(ts)


def test_eager_send_completes_before_any_recv(pair):
    t0, t1 = pair
    send = t0.post_send(0, 1, 100, b"12345678")
    assert not send.pending and send.bytes_moved == 8
    buf = bytearray(8)
    recv = t1.post_recv(0, 0, 100, buf)
    pump(pair, recv)
    assert bytes(buf) == b"12345678" and recv.bytes_moved == 8


def test_recv_posted_first_then_send(pair):
    t0, t1 = pair
    buf = bytearray(16)
    recv = t1.post_recv(0, 0, 5, buf)
    assert recv.pending
    t0.post_send(0, 1, 5, b"abc")
    pump(pair, recv)
    assert recv.bytes_moved == 3 and bytes(buf[:3]) == b"abc"


def test_roundtrip_identity_log_uniform_lengths(pair):
    t0, t1 = pair
    rng = random.Random(0x5EED)
    for _ in range(40):
        n = int(2 ** rng.uniform(0, 21))  # up to 2 MiB: exercises fragmentation
        payload = rng.randbytes(n)
        buf = bytearray(n)
        if rng.random() < 0.5:
            recv = t1.post_recv(0, 0, 33, buf)
            send = t0.post_send(0, 1, 33, payload)
        else:
            send = t0.post_send(0, 1, 33, payload)
            recv = t1.post_recv(0, 0, 33, buf)
        pump(pair, send, recv)
        assert bytes(buf) == payload


def test_fifo_per_key_and_no_cross_talk(pair):
    t0, t1 = pair
    for t in pair:
        t.register_channel(70, 1 - t.rank)
        t.register_channel(71, 1 - t.rank)
    t0.post_send(70, 1, 4, b"A1")
    t0.post_send(71, 1, 4, b"B1")
    t0.post_send(70, 1, 4, b"A2")
    t0.post_send(70, 1, 5, b"C1")
    got = {}
    reqs = []
    for key in [(71, 4), (70, 5), (70, 4), (70, 4)]:
        buf = bytearray(2)
        reqs.append((key, buf, t1.post_recv(key[0], 0, key[1], buf)))
    pump(pair, *[r for _, _, r in reqs])
    assert [bytes(b) for _, b, _ in reqs] == [b"B1", b"C1", b"A1", b"A2"]


def test_truncation_fails_the_receive(pair):
    t0, t1 = pair
    t0.post_send(0, 1, 7, b"eightbyt")
    recv = t1.post_recv(0, 0, 7, bytearray(4))
    pump(pair, recv)
    assert recv.failed and isinstance(recv.error, TruncationError)
    # the stream stays usable
    t0.post_send(0, 1, 7, b"ok")
    buf = bytearray(2)
    again = t1.post_recv(0, 0, 7, buf)
    pump(pair, again)
    assert bytes(buf) == b"ok"


def test_truncated_fragmented_message_is_discarded(pair):
    t0, t1 = pair
    big = os.urandom(3 << 20)
    t0.post_send(0, 1, 8, big)
    recv = t1.post_recv(0, 0, 8, bytearray(1000))
    t0.post_send(0, 1, 8, b"after")
    buf = bytearray(5)
    nxt = t1.post_recv(0, 0, 8, buf)
    pump(pair, recv, nxt)
    assert recv.failed and isinstance(recv.error, TruncationError)
    assert bytes(buf) == b"after"


def test_cancel_unmatched_recv_then_fresh_match(pair):
    t0, t1 = pair
    recv = t1.post_recv(0, 0, 40, bytearray(4))
    assert t1.cancel(recv) is True
    assert recv.failed and t1.cancel(recv) is False
    t0.post_send(0, 1, 40, b"zzzz")
    fresh = bytearray(4)
    recv2 = t1.post_recv(0, 0, 40, fresh)
    pump(pair, recv2)
    assert bytes(fresh) == b"zzzz"


def test_has_pending_tracks_channel_load(pair):
    t0, t1 = pair
    assert not t1.has_pending()
    recv = t1.post_recv(0, 0, 4, bytearray(2))
    assert t1.has_pending(0) and t1.has_pending()
    t0.post_send(0, 1, 4, b"pp")
    pump(pair, recv)
    assert not t1.has_pending(0)


def test_validation_errors(pair):
    t0, _ = pair
    with pytest.raises(ChannelError):
        t0.post_send(99, 1, 4, b"data")
    with pytest.raises(UsageError):
        t0.post_send(0, 0, 4, b"self")
    with pytest.raises(UsageError):
        t0.post_send(0, 5, 4, b"far")
    with pytest.raises(UsageError):
        t0.post_send(0, 1, -1, b"tag")
    with pytest.raises(UsageError):
        t0.post_recv(0, 1, 4, b"readonly")


def test_count_overflow_raised_before_any_copy():
    ts = nvlink_transports(2, device=-1, max_count=1024)
    try:
        with pytest.raises(CountOverflowError):
            ts[0].post_send(0, 1, 3, bytes(1025))
    finally:
        close_all(ts)


def test_purge_channel_drops_unmatched_state(pair):
    t0, t1 = pair
    for t in pair:
        t.register_channel(80, 1 - t.rank)
    t0.post_send(80, 1, 9, b"stale")
    posted = t1.post_recv(80, 0, 10, bytearray(4))
    pump(pair)  # let the stale message arrive
    for _ in range(10):
        t1.progress()
    t1.purge_channel(80)
    assert posted.failed
    t0.post_send(80, 1, 9, b"fresh")
    buf = bytearray(5)
    recv = t1.post_recv(80, 0, 9, buf)
    pump(pair, recv)
    assert bytes(buf) == b"fresh"


def test_peer_close_fails_pending_and_later_recvs(pair):
    t0, t1 = pair
    recv = t1.post_recv(0, 0, 12, bytearray(4))
    t0.close()
    pump([t1], recv)
    assert recv.failed and isinstance(recv.error, (TransferError, CommClosedError))
    late = t1.post_recv(0, 0, 12, bytearray(4))
    assert late.failed and isinstance(late.error, CommClosedError)


def test_unexpected_messages_survive_peer_close(pair):
    t0, t1 = pair
    t0.post_send(0, 1, 14, b"last words")
    t0.close()
    buf = bytearray(10)
    recv = t1.post_recv(0, 0, 14, buf)
    pump([t1], recv)
    assert bytes(buf) == b"last words"


def test_three_ranks_all_pairs(trio):
    sends, recvs = [], []
    for a in trio:
        for b in trio:
            if a is not b:
                sends.append(a.post_send(0, b.rank, 16 + a.rank, bytes([a.rank, b.rank]) * 100))
    for b in trio:
        for a in trio:
            if a is not b:
                buf = bytearray(200)
                recvs.append((a.rank, b.rank, buf, b.post_recv(0, a.rank, 16 + a.rank, buf)))
    pump(trio, *sends, *[r for *_, r in recvs])
    for a, b, buf, _ in recvs:
        assert bytes(buf) == bytes([a, b]) * 100


def test_startup_error_names_missing_rank():
    t1 = transport_init(2, 1, TransportConfig(kind="nvlink", session=new_session(), device=-1))
    try:
        with pytest.raises(StartupError) as info:
            t1.wait_ready(0.2)
        assert info.value.rank == 0
    finally:
        t1.close()


def test_rank_collision_is_configuration_error():
    session = new_session()
    t0 = transport_init(2, 0, TransportConfig(kind="nvlink", session=session, device=-1))
    try:
        with pytest.raises(ConfigurationError):
            transport_init(2, 0, TransportConfig(kind="nvlink", session=session, device=-1))
    finally:
        t0.close()


def test_world_size_mismatch_is_configuration_error():
    session = new_session()
    t0 = transport_init(2, 0, TransportConfig(kind="nvlink", session=session, device=-1))
    try:
        with pytest.raises(ConfigurationError):
            t1 = transport_init(3, 1, TransportConfig(kind="nvlink", session=session, device=-1))
            t1.wait_ready(1.0)
    finally:
        t0.close()


def test_requests_transition_exactly_once(pair):
    t0, t1 = pair
    sends = [t0.post_send(0, 1, 60, bytes([i]) * 64) for i in range(50)]
    bufs = [bytearray(64) for _ in range(50)]
    recvs = [t1.post_recv(0, 0, 60, b) for b in bufs]
    pump(pair, *sends, *recvs)
    for _ in range(5):
        t0.progress()
        t1.progress()
    assert all(r.state == TransferRequest.COMPLETE for r in sends + recvs)
    assert [b[0] for b in bufs] == list(range(50))
    assert t0.metrics.sends_completed == 50 and t1.metrics.recvs_completed == 50
    assert t0.metrics.staged_bytes == 0 and t1.metrics.staged_bytes == 0


DYING_PEER = """
import sys, time
sys.path.insert(0, sys.argv[1])
from paper_2101_08878_b200.transport import TransportConfig, transport_init
t = transport_init(2, 1, TransportConfig(kind="nvlink", session=sys.argv[2], device=-1, connect_timeout=20))
t.wait_ready()
print("ready", flush=True)
time.sleep(60)  # killed by the test
"""


def test_peer_death_fails_pending_receives_and_sends():
    """A peer killed mid-run (no close): its pid probe fails the pending receive and a
    queued send with TransferError and later posts with CommClosedError (the socket
    transport's peer-death handling, tcp.py:420-438 of the reference)."""
    import signal
    import subprocess
    import sys
    import time

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    session = new_session()
    child = subprocess.Popen([sys.executable, "-c", DYING_PEER, root, session], stdout=subprocess.PIPE, text=True)
    try:
        t0 = transport_init(2, 0, TransportConfig(kind="nvlink", session=session, device=-1, connect_timeout=20))
        t0.wait_ready()
        assert child.stdout.readline().strip() == "ready"
        recv = t0.post_recv(0, 1, 5, bytearray(8))
        big = t0.post_send(0, 1, 6, bytes(32 << 20))  # larger than the ring: stays queued
        child.send_signal(signal.SIGKILL)
        child.wait(timeout=10)
        deadline = time.monotonic() + 10
        while (recv.pending or big.pending) and time.monotonic() < deadline:
            t0.progress()
        assert recv.failed and isinstance(recv.error, TransferError)
        assert big.failed and isinstance(big.error, TransferError)
        late = t0.post_recv(0, 1, 5, bytearray(8))
        assert late.failed and isinstance(late.error, (CommClosedError, TransferError))
        t0.close()
    finally:
        if child.poll() is None:
            child.kill()


@pytest.mark.gpu
@pytest.mark.parametrize("env,kernel", [
    ({}, "some"),                                                     # defaults: window on the kernel, lone on the copy engine
    ({"M4D_SMALL_PULL": str(1 << 40)}, "none"),                       # everything below 1 TiB on the copy engine
    ({"M4D_PULL_ENGINE": "ce"}, "none"),                              # copy engine only
    ({"M4D_LONE_CE_MAX": "0", "M4D_SMALL_PULL": "0"}, "all"),         # every device pull on the kernel
    ({"M4D_PULL_BATCH_BYTES": "1"}, "some"),                          # one message per launch
    ({"M4D_SMALL_PULL": "-5", "M4D_LONE_CE_MAX": "-1"}, "some"),      # negative knobs fall back to the defaults
])
def test_pull_routing_knobs_keep_the_bytes(env, kernel):
    """Each pull route (SM kernel, copy engine, lone copy-engine pull, byte-capped batches)
    moves a mixed window of 64 KiB-32 MiB device frames bit-exactly; the launch counter shows
    which route ran."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "tests", "pull_routing_worker.py")],
                         env={**os.environ, **env}, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["ok"] and res["pulls"] == 12
    if kernel == "none":
        assert res["kernel_launches"] == 0
    elif kernel == "all":
        assert res["kernel_launches"] >= 6  # every lone pull launched the kernel
    else:
        assert 0 < res["kernel_launches"] < 12
