"""The native framed composites (csrc/pyfast.cpp) behind send_payload/recv_payload and
write_message/read_message on the nvlink transport: identical wire traffic to the
generic per-post path (either side may use either), and the generic errors."""

import pytest

from nvlink_fixtures import close_all, nvlink_world
from paper_2101_08878_b200.errors import EndOfStream, ProtocolError
from paper_2101_08878_b200.loop import gather
from paper_2101_08878_b200.messaging import (
    MESSAGE_TAG,
    Message,
    await_request,
    make_frame,
    read_message,
    recv_payload,
    send_payload,
    write_end_of_stream,
    write_message,
)

MSGS = [[35], [1, 35], [0, 18, 3], [], [4096, 17, 1]]


def _generic(t, send: bool, recv: bool):
    if not send:
        t.post_send_framed = None
    if not recv:
        t.post_recv_framed = None


@pytest.mark.parametrize("send_native,recv_native", [(True, True), (False, True), (True, False)])
@pytest.mark.parametrize("max_chunk", [17, 1 << 20])
def test_messages_cross_between_native_and_generic_paths(send_native, recv_native, max_chunk):
    loop, ts, tables = nvlink_world(2)
    _generic(ts[0], send_native, True)
    _generic(ts[1], True, recv_native)
    ch0, ch1 = tables[0].lookup(1), tables[1].lookup(0)
    msgs = [Message([make_frame(bytes([i + k]) * n) for k, n in enumerate(sizes)]) for i, sizes in enumerate(MSGS)]

    async def main():
        got = []

        async def w():
            for m in msgs:
                await write_message(ts[0], ch0, m, max_chunk=max_chunk)
            await send_payload(ts[0], ch0, 40, make_frame(b"p" * 5000), max_chunk=max_chunk)
            await write_end_of_stream(ts[0], ch0)

        async def r():
            for _ in msgs:
                got.append(await read_message(ts[1], ch1, max_chunk=max_chunk))
            got.append(await recv_payload(ts[1], ch1, 40, max_chunk=max_chunk))
            from paper_2101_08878_b200.messaging import EndOfStreamReceived

            with pytest.raises(EndOfStreamReceived):
                await read_message(ts[1], ch1, max_chunk=max_chunk)

        await gather(w(), r())
        return got

    try:
        got = loop.run_until_complete(main())
    finally:
        close_all(ts)
    for want, have in zip(msgs, got):
        assert [f.to_bytes() for f in have.frames] == [f.to_bytes() for f in want.frames]
    assert got[-1].to_bytes() == b"p" * 5000


def test_native_receive_reports_the_generic_protocol_errors():
    """Corrupt header (reference test_messaging.py:277-296) and a short payload slice."""
    loop, ts, tables = nvlink_world(2)
    t0, t1 = ts
    ch0, ch1 = tables[0].lookup(1), tables[1].lookup(0)

    async def main():
        async def bad_writer():
            header = (1).to_bytes(4, "little") + (8).to_bytes(8, "little") + bytes([0, 0])
            await await_request(t0, t0.post_send(ch0.id, 1, MESSAGE_TAG, header))
            await await_request(t0, t0.post_send(ch0.id, 1, 16, b"1234"))
            hdr = (100).to_bytes(8, "little") + bytes([0, 0])
            await await_request(t0, t0.post_send(ch0.id, 1, 44, hdr))
            await await_request(t0, t0.post_send(ch0.id, 1, 44, b"x" * 50))

        async def reader():
            with pytest.raises(ProtocolError) as info:
                await read_message(t1, ch1)
            assert (info.value.expected, info.value.actual) == (8, 4)
            with pytest.raises(ProtocolError) as info:
                await recv_payload(t1, ch1, 44, max_chunk=100)
            assert (info.value.expected, info.value.actual) == (100, 50)

        await gather(bad_writer(), reader())

    try:
        loop.run_until_complete(main())
    finally:
        close_all(ts)


def test_failed_chunk_withdraws_the_chunks_posted_ahead():
    """Chunks are posted CHUNK_WINDOW ahead; when one fails, those still unmatched are
    withdrawn, so the next transfer on the same key is not swallowed by a stale receive.
    (A sender that breaks the chunk plan corrupts the stream in either design; this pins
    the clean-up, not protocol recovery.)"""
    from paper_2101_08878_b200.errors import TruncationError
    from paper_2101_08878_b200.loop import sleep

    loop, ts, tables = nvlink_world(2)
    t0, t1 = ts
    t1.post_recv_framed = None  # the per-chunk path is the one that posts ahead
    ch0, ch1 = tables[0].lookup(1), tables[1].lookup(0)
    state = {"failed": False}

    async def main():
        async def bad_then_good_writer():
            hdr = (300).to_bytes(8, "little") + bytes([0, 0])
            await await_request(t0, t0.post_send(ch0.id, 1, 60, hdr))
            await await_request(t0, t0.post_send(ch0.id, 1, 60, b"a" * 100))
            await await_request(t0, t0.post_send(ch0.id, 1, 60, b"b" * 150))  # longer than the 100-byte slice
            while not state["failed"]:
                await sleep(0)
            await send_payload(t0, ch0, 60, make_frame(b"good" * 60), max_chunk=100)

        async def reader():
            with pytest.raises(TruncationError):
                await recv_payload(t1, ch1, 60, max_chunk=100)
            assert not t1.has_pending(ch1.id)  # the third slice's receive was withdrawn
            state["failed"] = True
            frame = await recv_payload(t1, ch1, 60, max_chunk=100)
            assert frame.to_bytes() == b"good" * 60

        await gather(bad_then_good_writer(), reader())

    try:
        loop.run_until_complete(main())
    finally:
        close_all(ts)
