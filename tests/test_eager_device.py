"""Eager device protocol (north_star: eager and rendezvous chosen per message size for GPU
frames): device payloads up to ``eager_device_max`` bytes are copied by
the sender into its region of the receiver's device ring and announced once the copy is
done; the receiver copies them out, or lends the ring bytes (loan) without a copy.  Two
ranks in one process on cuda:0 (the multi-process and two-GPU cases are in
test_multiprocess_gpu.py)."""

import numpy as np
import pytest

from nvlink_fixtures import close_all, nvlink_transports, pump

pytestmark = pytest.mark.gpu


def pattern(n, salt):
    return ((np.arange(n, dtype=np.uint64) * (2 * salt + 3)) % 251).astype(np.uint8)


@pytest.fixture
def pair():
    ts = nvlink_transports(2, 0)
    yield ts
    close_all(ts)


def dev(n, data=None):
    from paper_2101_08878_b200.transport.nvlink import CudaRegion

    return CudaRegion(bytes(data) if data is not None else n, 0)


def stats(t):
    return t.native_stats()


def test_transport_advertises_the_threshold(pair):
    assert pair[0].eager_device_max == 64 << 10


@pytest.mark.parametrize("n", [1, 17, 4096, 64 << 10])
@pytest.mark.parametrize("order", ["recv_first", "send_first"])
def test_eager_into_a_posted_device_buffer(pair, n, order):
    from paper_2101_08878_b200.transport import MemoryDomain

    src, dst = dev(n, pattern(n, n)), dev(n)
    before = stats(pair[0])["eager_device_sends"]
    if order == "recv_first":
        r = pair[1].post_recv(0, 0, 5, dst.window(), MemoryDomain.DEVICE)
        s = pair[0].post_send_eager(0, 1, 5, src.window())
    else:
        s = pair[0].post_send_eager(0, 1, 5, src.window())
        pump(pair, s)  # eager: completes without the receiver
        r = pair[1].post_recv(0, 0, 5, dst.window(), MemoryDomain.DEVICE)
    pump(pair, s, r)
    assert r.bytes_moved == n and np.array_equal(np.frombuffer(dst.to_bytes(), np.uint8), pattern(n, n))
    assert stats(pair[0])["eager_device_sends"] == before + 1
    assert stats(pair[0])["rendezvous_pulls"] == 0 and stats(pair[1])["rendezvous_pulls"] == 0


def test_eager_into_host_memory_and_by_loan(pair):
    from paper_2101_08878_b200.transport import MemoryDomain

    n = 3000
    src = dev(n, pattern(n, 1))
    host = bytearray(n)
    s = pair[0].post_send_eager(0, 1, 6, src.window())
    r = pair[1].post_recv(0, 0, 6, host)
    pump(pair, s, r)
    assert bytes(host) == pattern(n, 1).tobytes()
    fallback = dev(n)
    s = pair[0].post_send_eager(0, 1, 7, src.window())
    r = pair[1].post_recv_loanable(0, 0, 7, fallback.window())
    pump(pair, s, r)
    loan = pair[1].take_loan(r)
    assert loan is not None and loan.ptr != fallback.ptr and loan.nbytes == n
    assert loan.to_bytes() == pattern(n, 1).tobytes()
    assert pair[1].take_loan(r) is None  # taken once
    assert stats(pair[1])["eager_device_loans"] == 1


def test_larger_frames_take_the_rendezvous(pair):
    from paper_2101_08878_b200.transport import MemoryDomain

    n = (64 << 10) + 1
    src, dst = dev(n, pattern(n, 2)), dev(n)
    s = pair[0].post_send_eager(0, 1, 8, src.window())
    r = pair[1].post_recv_loanable(0, 0, 8, dst.window())
    pump(pair, s, r)
    assert pair[1].take_loan(r) is None  # landed in the posted buffer by a pull
    assert dst.to_bytes() == pattern(n, 2).tobytes()
    assert stats(pair[1])["rendezvous_pulls"] == 1 and stats(pair[0])["eager_device_sends"] == 0


def test_truncation_fails_the_receive_and_frees_the_slot(pair):
    from paper_2101_08878_b200.errors import TruncationError
    from paper_2101_08878_b200.transport import MemoryDomain

    src, small = dev(512, pattern(512, 3)), dev(100)
    s = pair[0].post_send_eager(0, 1, 9, src.window())
    r = pair[1].post_recv(0, 0, 9, small.window(), MemoryDomain.DEVICE)
    pump(pair, s, r)
    assert r.failed and isinstance(r.error, TruncationError) and not s.failed


def test_held_loans_fill_the_ring_then_sends_fall_back_and_resume(pair):
    """100 held 64 KiB loans exceed the 4 MiB ring region: later sends still complete (by
    rendezvous); once the loans are dropped the eager path is used again."""
    import gc

    n = 64 << 10
    src = dev(n, pattern(n, 4))
    held = []
    for k in range(100):
        fallback = dev(n)
        s = pair[0].post_send_eager(0, 1, 10, src.window())
        r = pair[1].post_recv_loanable(0, 0, 10, fallback.window())
        pump(pair, s, r)
        got = pair[1].take_loan(r) or fallback
        held.append(got)
    assert all(h.to_bytes() == pattern(n, 4).tobytes() for h in held[::9])
    st = stats(pair[0])
    assert 0 < st["eager_device_sends"] < 100 and stats(pair[1])["rendezvous_pulls"] > 0
    held.clear()
    gc.collect()
    before = stats(pair[0])["eager_device_sends"]
    for k in range(80):  # the ring wraps around several times
        dst = dev(n)
        s = pair[0].post_send_eager(0, 1, 11, src.window())
        r = pair[1].post_recv_loanable(0, 0, 11, dst.window())
        pump(pair, s, r)
        loan = pair[1].take_loan(r)
        assert (loan or dst).to_bytes()[:64] == pattern(n, 4).tobytes()[:64]
        del loan
    assert stats(pair[0])["eager_device_sends"] == before + 80


def test_comm_path_device_frames_use_eager_and_loans():
    """send_payload / recv_payload of small device frames: eager sends, loaned receives,
    bytes intact; large frames keep the rendezvous."""
    from paper_2101_08878_b200.loop import gather
    from paper_2101_08878_b200.messaging import Frame, recv_payload, send_payload
    from paper_2101_08878_b200.transport import MemoryDomain

    from nvlink_fixtures import nvlink_world

    loop, ts, tables = nvlink_world(2, 0)
    try:
        sizes = [1, 999, 64 << 10, (64 << 10) + 16, 1 << 20]

        async def main():
            out = []
            for k, n in enumerate(sizes):
                frame = Frame(dev(n, pattern(n, k)), n, MemoryDomain.DEVICE)
                _, got = await gather(send_payload(ts[0], tables[0].lookup(1), 300 + k, frame),
                                      recv_payload(ts[1], tables[1].lookup(0), 300 + k))
                out.append(got)
            return out

        got = loop.run_until_complete(main())
        for k, (n, f) in enumerate(zip(sizes, got)):
            assert f.domain == MemoryDomain.DEVICE and f.to_bytes() == pattern(n, k).tobytes()
        assert stats(ts[0])["eager_device_sends"] == 3 and stats(ts[1])["eager_device_loans"] == 3
        assert stats(ts[1])["rendezvous_pulls"] == 2
    finally:
        close_all(ts)


def test_sends_are_copied_by_the_proxy_kernel(pair):
    """With the proxy (default) every eager device send is moved by the resident proxy
    kernel: no copy-engine copy, no event per message."""
    from paper_2101_08878_b200.transport import MemoryDomain

    n = 1000
    src, dst = dev(n, pattern(n, 2)), dev(n)
    s = pair[0].post_send_eager(0, 1, 12, src.window())
    r = pair[1].post_recv(0, 0, 12, dst.window(), MemoryDomain.DEVICE)
    pump(pair, s, r)
    assert dst.to_bytes() == pattern(n, 2).tobytes()
    st = stats(pair[0])
    assert st["eager_proxy_copies"] == st["eager_device_sends"] == 1


def stream_mixed(ts, count=600):
    """`count` messages 0 -> 1 on one tag, in post order: eager device frames of ragged
    sizes and misaligned sources (more than the proxy queue's 256 slots in flight),
    rendezvous frames and host frames interleaved.  Receives posted after all sends, so
    every kind waits as an unexpected message; FIFO order and bytes must hold."""
    from paper_2101_08878_b200.transport import MemoryDomain

    big = 256 << 10
    pool = dev(big + 64, pattern(big + 64, 7))
    want, sends = [], []
    for k in range(count):
        kind = k % 10
        if kind == 9:  # rendezvous (above the eager threshold)
            n, off = big, 0
            sends.append(ts[0].post_send(0, 1, 13, pool.window(off, n), MemoryDomain.DEVICE))
            want.append(("dev", pattern(big + 64, 7)[off:off + n].tobytes()))
        elif kind == 4:  # host frame
            payload = bytes([k % 251]) * (1 + k % 300)
            sends.append(ts[0].post_send(0, 1, 13, payload))
            want.append(("host", payload))
        else:
            n = 1 + (k * 997) % (8 << 10)
            off = k % 33  # misaligned sources too
            sends.append(ts[0].post_send_eager(0, 1, 13, pool.window(off, n)))
            want.append(("dev", pattern(big + 64, 7)[off:off + n].tobytes()))
    rendezvous = sends[9::10]
    pump(ts, *[s for k, s in enumerate(sends) if k % 10 != 9], timeout=60)  # complete without the receiver
    got = []
    for kind, data in want:
        if kind == "host":
            buf = bytearray(len(data))
            r = ts[1].post_recv(0, 0, 13, buf)
            pump(ts, r)
            got.append(bytes(buf[:r.bytes_moved]))
        else:
            dst = dev(len(data))
            r = ts[1].post_recv(0, 0, 13, dst.window(), MemoryDomain.DEVICE)
            pump(ts, r)
            got.append(dst.to_bytes()[:r.bytes_moved])
    pump(ts, *rendezvous)
    assert [g == w for g, (_, w) in zip(got, want)] == [True] * count
    return stats(ts[0])


def test_proxy_keeps_fifo_order_across_protocols(pair):
    st = stream_mixed(pair)
    assert st["eager_proxy_copies"] > 256 and st["eager_proxy_copies"] == st["eager_device_sends"]


def test_copy_engine_eager_path_when_the_proxy_is_off():
    """M4D_EAGER_PROXY=0: the same stream through copy-engine copies and events."""
    import os
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, 'tests'); import test_eager_device as m, nvlink_fixtures as f\n"
            "ts = f.nvlink_transports(2, 0)\n"
            "st = m.stream_mixed(ts, 200)\n"
            "f.close_all(ts)\n"
            "assert st['eager_proxy_copies'] == 0 and st['eager_device_sends'] > 100, st\n"
            "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300,
                         env=dict(os.environ, M4D_EAGER_PROXY="0"))
    assert out.returncode == 0 and "ok" in out.stdout, out.stdout[-2000:] + out.stderr[-2000:]


def test_framed_device_frames_fall_back_to_receive_slots_when_the_ring_is_full():
    """The native composites receive a lone small device frame by a loan-only receive:
    eager frames are lent from the ring; once held frames fill the ring, later ones come by
    rendezvous into transport receive slots, which are lent the same way and recycled."""
    from paper_2101_08878_b200.loop import gather
    from paper_2101_08878_b200.messaging import Frame, Message, read_message, recv_payload, send_payload, \
        write_message
    from paper_2101_08878_b200.transport import MemoryDomain

    from nvlink_fixtures import nvlink_world

    loop, ts, tables = nvlink_world(2, 0)
    try:
        n = 60 << 10
        src = [dev(n, pattern(n, k)) for k in range(4)]

        async def one(k, held):
            frame = Frame(src[k % 4], n, MemoryDomain.DEVICE)
            if k % 2:
                _, got = await gather(send_payload(ts[0], tables[0].lookup(1), 40, frame),
                                      recv_payload(ts[1], tables[1].lookup(0), 40))
            else:
                _, msg = await gather(write_message(ts[0], tables[0].lookup(1), Message([frame])),
                                      read_message(ts[1], tables[1].lookup(0)))
                got = msg.frames[0]
            assert got.domain == MemoryDomain.DEVICE
            held.append((k, got))

        held = []

        async def run(count):
            for k in range(count):
                await one(k, held)

        loop.run_until_complete(run(100))  # 100 x 60 KiB held > the 4 MiB ring region
        assert all(f.to_bytes() == pattern(n, k % 4).tobytes() for k, f in held)
        st = stats(ts[1])
        assert st["rendezvous_pulls"] > 0 and st["eager_device_loans"] > 0
        assert st["eager_device_loans"] + st["rendezvous_pulls"] == 100
        held.clear()
        import gc

        gc.collect()
        before = stats(ts[1])["rendezvous_pulls"]
        loop.run_until_complete(run(40))  # slots and ring given back: eager again
        assert stats(ts[1])["rendezvous_pulls"] == before
        assert all(f.to_bytes() == pattern(n, k % 4).tobytes() for k, f in held)
    finally:
        close_all(ts)


def test_proxy_kernel_stays_up_under_traffic_and_exits_when_idle(pair):
    """Back-to-back eager sends are served by one proxy launch; after the idle timeout
    (M4D_EAGER_PROXY_IDLE_US, 100 us) the kernel has exited and the next send relaunches it."""
    import time

    from paper_2101_08878_b200.transport import MemoryDomain

    n = 256
    src, dst = dev(n, pattern(n, 5)), dev(n)

    def one():
        s = pair[0].post_send_eager(0, 1, 14, src.window())
        r = pair[1].post_recv(0, 0, 14, dst.window(), MemoryDomain.DEVICE)
        pump(pair, s, r)
        assert dst.to_bytes() == pattern(n, 5).tobytes()

    one()
    first = stats(pair[0])["eager_proxy_launches"]
    assert first >= 1
    for _ in range(50):  # far less than 100 us apart
        s = pair[0].post_send_eager(0, 1, 15, src.window())
        pump(pair, s)
    busy = stats(pair[0])["eager_proxy_launches"] - first
    assert busy <= 10  # the kernel stayed up (50 sends; a few relaunches only if the host stalled > 100 us)
    time.sleep(0.05)  # far beyond the idle timeout
    before = stats(pair[0])["eager_proxy_launches"]
    one()
    assert stats(pair[0])["eager_proxy_launches"] == before + 1
    for _ in range(50):  # drain tag 15
        r = pair[1].post_recv(0, 0, 15, dst.window(), MemoryDomain.DEVICE)
        pump(pair, r)


@pytest.mark.parametrize("eager", [False, True])
def test_vectored_posts_match_the_per_post_loop(pair, eager):
    """post_many: a window of device sends and receives in one call each -- bytes, FIFO
    order and completions as with one call per post; ragged sizes, receives posted
    before and after the sends."""
    from paper_2101_08878_b200.transport import MemoryDomain

    sizes = [1, 17, 4096, 65536, 300_000, 1 << 20, 4096, 3]
    total = sum(sizes)
    src = dev(total, pattern(total, 9))
    dst = dev(total)
    offs, at = [], 0
    for n in sizes:
        offs.append(at)
        at += n
    sv = [src.window(o, n) for o, n in zip(offs, sizes)]
    dv = [dst.window(o, n) for o, n in zip(offs, sizes)]
    rq = pair[1].post_many("recv", 0, 0, 16, dv[:4], MemoryDomain.DEVICE, eager=False)
    sq = pair[0].post_many("send", 0, 1, 16, sv, MemoryDomain.DEVICE, eager=eager)
    rq += pair[1].post_many("recv", 0, 0, 16, dv[4:], MemoryDomain.DEVICE, eager=False)
    pump(pair, *(rq + sq))
    assert [r.bytes_moved for r in rq] == sizes and all(not r.failed for r in rq + sq)
    assert dst.to_bytes() == pattern(total, 9).tobytes()
    with pytest.raises(Exception):
        pair[0].post_many("send", 0, 1, 16, [b"host bytes"], MemoryDomain.DEVICE)
