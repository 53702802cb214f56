"""``kind="nvlink"``: the B200 transport, a ctypes facade over ``libm4d.so``.

Replaces the reference transports (``pkg/src/commshim/transport/sim.py``,
``tcp.py``) behind the same :class:`~.base.Transport` contract
(``base.py:199-306``); selected by ``transport_init(world, rank,
TransportConfig(kind="nvlink", ...))``.  The C side (``csrc/transport.cpp``,
ABI in ``include/m4d.h`` §3) owns matching, protocols and progress:

* host payloads (headers, control messages, host frames) travel *eagerly*
  through per-pair shared-memory rings, so small sends complete at post time;
* device payloads (:class:`CudaRegion` windows) travel by *rendezvous*: the
  receiver maps the sender's allocation through CUDA IPC and pulls the bytes
  device-to-device over NVLink with the copy engines.  Nothing is staged
  through host memory, so ``device_aware`` is True and the staging counters
  stay zero (``tests/test_messaging.py:158-180`` of the reference).

Progress is cooperative: ``test()``/``progress()`` call into the library,
which drains rings, flushes queued sends and polls copy events; no host
threads exist.  Every rank of a world must be on one node and share
``TransportConfig.session`` (default: ``$M4D_SESSION``, else derived from the
torchrun rendezvous).  Ranks may also share one process (test mode).
"""

from __future__ import annotations

import ctypes
import struct
import os
import weakref

from .. import native
from ..errors import CommClosedError, ConfigurationError, TransferError, UsageError
from ..loop import MonotonicClock
from .base import (
    DeviceRegion,
    DeviceView,
    MemoryDomain,
    Transport,
    TransportConfig,
    TransferRequest,
    as_view,
)

class _Extent:
    """Length-only stand-in for the payload view of a framed composite request."""

    __slots__ = ("n",)

    def __init__(self, n: int):
        self.n = n

    def __len__(self) -> int:
        return self.n


_Config = native.TransportConfigC
Completion = native.Completion
Stats = native.TransportStats


# -- device memory ------------------------------------------------------------------------------


class CudaRegion(DeviceRegion):
    """Real B200 memory behind the reference ``DeviceRegion`` interface.

    ``window(offset, length)`` hands out :class:`DeviceView` windows (pointer
    + length), which the nvlink transport moves device-to-device.  Backed by a
    dedicated ``cudaMalloc`` (exportable through CUDA IPC) or by an external
    device pointer whose ``owner`` keeps it alive (e.g. a torch tensor).
    """

    __slots__ = ("ptr", "_nbytes", "device", "_owner", "__weakref__")

    def __init__(self, size_or_bytes, device: int = 0, *, ptr: int | None = None, owner=None):
        if ptr is not None:
            self._owner = owner
            self.ptr = int(ptr)
            self._nbytes = int(size_or_bytes)
        else:
            data = None if isinstance(size_or_bytes, int) else bytes(size_or_bytes)
            n = size_or_bytes if data is None else len(data)
            buf = native.DeviceBuffer(device, max(1, n))
            self._owner = buf
            self.ptr = buf.ptr
            self._nbytes = n
            if data:
                host = ctypes.create_string_buffer(data, n)
                native.memcpy(self.ptr, ctypes.addressof(host), n)
                native.check(native.lib().m4d_stream_sync(None))
        self.device = device

    @classmethod
    def from_tensor(cls, tensor) -> "CudaRegion":
        """Wrap a contiguous CUDA torch tensor (plumbing only; no copy)."""
        if not tensor.is_cuda or not tensor.is_contiguous():
            raise UsageError("CudaRegion.from_tensor needs a contiguous CUDA tensor")
        return cls(tensor.numel() * tensor.element_size(), tensor.device.index or 0, ptr=tensor.data_ptr(),
                   owner=tensor)

    @property
    def nbytes(self) -> int:
        return self._nbytes

    def window(self, offset: int = 0, length: int | None = None) -> DeviceView:
        offset, length = self._bounds(offset, length)
        return DeviceView(self.ptr + offset, length, self.device, self)

    def to_bytes(self) -> bytes:
        return native.to_host(self.ptr, self._nbytes)

    def __repr__(self):
        return f"<CudaRegion cuda:{self.device} {self._nbytes} B>"


class _Loan:
    """Keeps a loaned ring slot until the region lent out dies, then hands it back."""

    __slots__ = ("transport", "token")

    def __init__(self, transport, token: int):
        self.transport, self.token = transport, token

    def __del__(self):
        t = self.transport
        try:
            if getattr(t, "_h", None):
                t._fast.unloan(t._h, self.token)
        except Exception:
            pass


class _RegionPool:
    """Size-class cache of receive regions so recv_payload does not cudaMalloc per frame.

    Classes below SLAB bytes are carved out of 2 MiB slabs (one cudaMalloc per slab,
    kept until the pool dies), so a storm of small frames whose regions are held by
    the application costs no allocation per frame -- cudaMalloc / cudaFree also
    synchronise the device, and with it wait for a running eager proxy kernel to
    idle out.  Larger classes get their own allocation, cached up to CACHE_BYTES per
    class."""

    SLAB = 2 << 20
    CACHE_BYTES = 64 << 20

    def __init__(self, device: int):
        self.device = device
        self.free: dict[int, list] = {}
        self.slabs: list = []

    def get(self, n: int) -> CudaRegion:
        size = 1 << max(12, (max(n, 1) - 1).bit_length())
        bucket = self.free.setdefault(size, [])
        if not bucket:
            if size >= self.SLAB:
                buf = native.DeviceBuffer(self.device, size)
                return CudaRegion(n, self.device, ptr=buf.ptr, owner=_Lease(self, size, buf))
            slab = native.DeviceBuffer(self.device, self.SLAB)
            self.slabs.append(slab)
            bucket.extend(slab.ptr + k * size for k in range(self.SLAB // size))
        item = bucket.pop()
        ptr = item if isinstance(item, int) else item.ptr
        return CudaRegion(n, self.device, ptr=ptr, owner=_Lease(self, size, item))

    def put(self, size: int, item) -> None:
        bucket = self.free.setdefault(size, [])
        if isinstance(item, int) or len(bucket) < max(2, self.CACHE_BYTES // size):
            bucket.append(item)


class _Lease:
    """A pooled region's slot (slab address or own DeviceBuffer), back to the pool on death."""

    __slots__ = ("pool", "size", "item")

    def __init__(self, pool, size, item):
        self.pool, self.size, self.item = pool, size, item

    def __del__(self):
        try:
            self.pool.put(self.size, self.item)
        except Exception:
            pass


def default_session() -> str:
    env = os.environ.get("M4D_SESSION")
    if env:
        return env
    run = os.environ.get("TORCHELASTIC_RUN_ID")
    port = os.environ.get("MASTER_PORT")
    if run or port:
        return f"te_{run or 'x'}_{port or 'x'}".replace("/", "_")
    return "default"


# -- the transport ------------------------------------------------------------------------------


class NvlinkTransport(Transport):
    """One rank of an NVLink world (see the module docstring)."""

    def __init__(self, world_size: int, rank: int, config: TransportConfig | None = None):
        config = config or TransportConfig(kind="nvlink")
        super().__init__(world_size, rank, config.max_count, True, MonotonicClock())
        count = native.device_count()
        if config.device is not None:
            device = config.device
            if device >= 0 and device >= count:
                raise ConfigurationError(f"CUDA device {device} not present ({count} visible)")
        else:
            device = rank % count if count else -1
        self.device = device
        self.session = config.session or default_session()
        cfg = _Config(world_size, rank, device, 0, config.ring_bytes, float(config.connect_timeout),
                      self.session.encode())
        handle = ctypes.c_void_p()
        status = native.lib().m4d_transport_open(ctypes.byref(cfg), ctypes.byref(handle))
        if status != native.OK:
            raise native.error_for(status, native.last_error(), rank=_rank_in(native.last_error()))
        self._h = handle.value
        self._lib = native.lib()
        self._fast = native.fast()
        self.pull_copy_engine = os.environ.get("M4D_PULL_ENGINE") == "ce"
        self._live: dict[int, TransferRequest] = {}
        self._pool = _RegionPool(device) if device >= 0 else None
        self.connect_timeout = config.connect_timeout
        # largest device payload sent eagerly (0: no device ring, every device frame rendezvous)
        self.eager_device_max = int(self._lib.m4d_transport_eager_device_max(self._h))
        self._loans = weakref.WeakSet()  # regions lent out of the device ring

    # -- mesh -----------------------------------------------------------------------------------

    @property
    def mesh_ready(self) -> bool:
        return bool(self._lib.m4d_transport_mesh_ready(self._h))

    def wait_ready(self, timeout: float | None = None) -> None:
        """Block until every peer rank is up (StartupError names a missing rank)."""
        status = self._lib.m4d_transport_wait_ready(self._h, self.connect_timeout if timeout is None else timeout)
        if status != native.OK:
            msg = native.last_error()
            raise native.error_for(status, msg, rank=_rank_in(msg))

    # -- posts ----------------------------------------------------------------------------------

    def _post(self, direction: str, channel: int, peer: int, tag: int, data, domain, flags: int = 0) -> TransferRequest:
        view = as_view(data)
        if direction == "recv" and view.readonly:
            raise UsageError("receive buffer must be writable")
        self._check_post(channel, peer, tag, view)
        req = TransferRequest(self, direction, channel, peer, tag, view, domain)
        if isinstance(view, DeviceView):
            obj, device_len = view.ptr, len(view)
        else:
            obj, device_len = view, -1  # host: address taken through the buffer protocol
        try:
            done = self._fast.post(self._h, direction == "send", channel, peer, tag, obj, int(domain), device_len,
                                   req.id, flags)
        except OSError as exc:
            raise native.error_for(exc.args[0], native.last_error()) from None
        if done is None:
            self._live[req.id] = req
            req._native = req.id
        else:
            self._apply(req, done[0], done[1])
        return self._track(req)

    def post_many(self, direction: str, channel: int, peer: int, tag: int, views, domain=MemoryDomain.DEVICE,
                  eager: bool = False) -> list[TransferRequest]:
        """A window of device posts to one (channel, peer, tag) in one native call
        (``m4d_transport_post_many``): the same requests, in the same order, as posting
        them one by one (per-key FIFO), for a fraction of the per-call cost.  ``eager``:
        eager sends / loanable receives (``post_send_eager`` / ``post_recv_loanable``)."""
        if direction not in ("send", "recv"):
            raise UsageError(f"direction must be 'send' or 'recv', not {direction!r}")
        reqs = []
        for v in views:
            if not isinstance(v, DeviceView):
                raise UsageError("post_many takes device windows (DeviceView)")
            self._check_post(channel, peer, tag, v)
            reqs.append(TransferRequest(self, direction, channel, peer, tag, v, domain))
        if not reqs:
            return []
        try:
            done = self._fast.post_many(self._h, direction == "send", channel, peer, tag,
                                        tuple(v.ptr for v in views), tuple(len(v) for v in views), int(domain),
                                        3 if eager else 1, tuple(r.id for r in reqs))
        except OSError as exc:
            status, posted = exc.args[0]
            for r in reqs[:posted]:  # the posts made before the failure stay live
                self._live[r.id] = r
                r._native = r.id
                self._track(r)
            raise native.error_for(status, native.last_error()) from None
        inline = {i: (st, nb) for i, st, nb in done}
        for i, r in enumerate(reqs):
            if i in inline:
                self._apply(r, *inline[i])
            else:
                self._live[r.id] = r
                r._native = r.id
            self._track(r)
        return reqs

    # -- framed composites (messaging wire protocol done natively, csrc/pyfast.cpp) -------------

    def post_send_framed(self, kind: int, channel: int, peer: int, tag: int, header: bytes, bodies: tuple,
                         max_chunk: int) -> TransferRequest:
        """One request for a whole host-frame transfer: ``header`` then every body in
        ``max_chunk`` slices (kind 0: send_payload, all on ``tag``; kind 1: write_message,
        header on ``tag``, body i on data tag 16 + i)."""
        self._check_route(channel, peer)
        total = len(header) + sum(len(b) for b in bodies)
        req = TransferRequest(self, "send", channel, peer, tag, _Extent(total), MemoryDomain.HOST)
        try:
            done = self._fast.send_framed(self._h, kind, channel, peer, tag, header, bodies, max_chunk, req.id)
        except OSError as exc:
            raise native.error_for(exc.args[0], native.last_error()) from None
        if done is None:
            self._live[req.id] = req
        else:
            self._apply(req, done[0], total if done[0] == native.OK else 0)
        return self._track(req)

    def post_recv_framed(self, kind: int, channel: int, peer: int, tag: int, max_chunk: int) -> TransferRequest:
        """One request that receives a whole framed transfer (see :meth:`take_framed`).  A
        transfer whose only frame is a device frame of at most ``eager_device_max`` bytes
        is received natively too, by loan."""
        self._check_route(channel, peer)
        req = TransferRequest(self, "recv", channel, peer, tag, _Extent(0), MemoryDomain.HOST)
        try:
            done = self._fast.recv_framed(self._h, kind, channel, peer, tag, max_chunk, req.id, self.eager_device_max)
        except OSError as exc:
            raise native.error_for(exc.args[0], native.last_error()) from None
        if done is None:
            self._live[req.id] = req
        else:
            self._apply(req, done[0], done[1])
        return self._track(req)

    def take_framed(self, req: TransferRequest):
        """(outcome, header bytes, payload, (offset, expected, actual)) of a finished receive
        composite: outcome 0 = the frames were received (payload: a bytearray of the host
        frames, or the :class:`CudaRegion` lent for a lone device frame), 1 = header only
        (the caller finishes the transfer), 2 = end of stream, 3 = a slice came short."""
        outcome, raw, payload, detail = self._fast.take_framed(req.id)
        if isinstance(payload, tuple):  # a lone device frame, lent (ring bytes or a receive slot)
            nbytes = struct.unpack_from("<Q", raw, 0 if len(raw) == 10 else 4)[0]
            payload = self._lent(payload[0], payload[1], nbytes)
        return outcome, raw, payload, detail

    def _lent(self, ptr: int, token: int, nbytes: int) -> CudaRegion:
        region = CudaRegion(nbytes, self.device, ptr=ptr, owner=_Loan(self, token))
        self._loans.add(region)
        return region

    def post_send(self, channel: int, peer: int, tag: int, data,
                  domain: MemoryDomain = MemoryDomain.HOST) -> TransferRequest:
        return self._post("send", channel, peer, tag, data, domain)

    def post_recv(self, channel: int, peer: int, tag: int, buffer,
                  domain: MemoryDomain = MemoryDomain.HOST) -> TransferRequest:
        return self._post("recv", channel, peer, tag, buffer, domain)

    # -- eager device frames (protocol chosen per size) ----------------------------------------------

    def post_send_eager(self, channel: int, peer: int, tag: int, data,
                        domain: MemoryDomain = MemoryDomain.DEVICE) -> TransferRequest:
        """``post_send`` that lets a device payload of at most ``eager_device_max`` bytes go
        eagerly: the sender copies it into its region of the receiver's device ring and the
        send completes when that copy is done, without a rendezvous round trip.  Larger
        payloads (or a full ring) take the rendezvous as usual."""
        return self._post("send", channel, peer, tag, data, domain, 1)

    def post_recv_loanable(self, channel: int, peer: int, tag: int, buffer,
                           domain: MemoryDomain = MemoryDomain.DEVICE) -> TransferRequest:
        """``post_recv`` whose message, if it arrives eagerly, stays where it landed in the
        device ring and is lent out instead of copied (:meth:`take_loan`); otherwise the
        bytes land in ``buffer`` as usual."""
        return self._post("recv", channel, peer, tag, buffer, domain, 1)

    def take_loan(self, req: TransferRequest):
        """The :class:`CudaRegion` lent to a finished loanable receive (the ring bytes, valid
        while the region is alive and the transport open), or None if the bytes are in the
        posted buffer."""
        got = self._fast.loan(self._h, req.id)
        if got is None:
            return None
        return self._lent(got[0], got[1], req.bytes_moved)

    def _evacuate_loans(self) -> None:
        """Before the ring goes away (close): move every loaned region still alive into its
        own allocation, so received frames outlive the transport as the reference's do."""
        live = list(self._loans)
        if not live:
            return
        for region in live:
            buf = native.DeviceBuffer(self.device, max(1, region.nbytes))
            native.memcpy(buf.ptr, region.ptr, region.nbytes)
            region.ptr, region._owner = buf.ptr, buf  # the _Loan is dropped: its slot is moot now
        native.check(self._lib.m4d_device_sync(self.device))
        self._loans.clear()

    # -- completions ------------------------------------------------------------------------------

    def _apply(self, req: TransferRequest, status: int, nbytes: int) -> None:
        if status == native.OK:
            m = self.metrics
            if req.direction == "send":
                m.sends_completed += 1
                m.bytes_sent += nbytes
            else:
                m.recvs_completed += 1
                m.bytes_received += nbytes
            req._finish(TransferRequest.COMPLETE, nbytes)
            return
        message = native.last_error() or f"transfer failed (status {status})"
        if status == native.ERR_CLOSED:
            error = CommClosedError(f"rank {req.peer} connection closed")
        elif status == native.ERR_TRANSFER:
            error = TransferError(f"rank {req.peer} closed the connection", bytes_moved=nbytes)
        else:
            error = native.error_for(status, message, bytes_moved=nbytes)
        req._finish(TransferRequest.FAILED, nbytes if status == native.ERR_TRANSFER else 0, error)

    def progress(self) -> int:
        done = self._fast.progress(self._h)
        if done is None:
            return 0
        finished = 0
        live = self._live
        for req_id, status, nbytes in done:
            req = live.pop(req_id, None)
            if req is not None:
                self._apply(req, status, nbytes)
                finished += 1
        return finished

    def cancel(self, request: TransferRequest) -> bool:
        if request._owner is not self:
            raise UsageError("request belongs to a different transport")
        if not request.pending:
            return False
        flag = ctypes.c_int(0)
        native.check(self._lib.m4d_transport_cancel(self._h, request.id, ctypes.byref(flag)))
        if not flag.value:
            return False
        self._live.pop(request.id, None)
        self._cancelled(request)
        return True

    def purge_channel(self, channel: int) -> None:
        native.check(self._lib.m4d_transport_purge_channel(self._h, channel))
        self.progress()

    def set_pull_engine(self, copy_engine: bool) -> None:
        """Rendezvous pulls on the copy engines only (True) or SM copy kernels (False)."""
        native.check(self._lib.m4d_transport_set_pull_engine(self._h, int(bool(copy_engine))))
        self.pull_copy_engine = bool(copy_engine)

    def set_pull_ctas(self, max_ctas: int) -> None:
        """Cap the SM pull kernel's grid (pulls sharing the GPU with compute kernels)."""
        native.check(self._lib.m4d_transport_set_pull_ctas(self._h, int(max_ctas)))

    def peer_alive(self, peer: int) -> bool:
        return bool(self._lib.m4d_transport_peer_alive(self._h, peer))

    def native_stats(self) -> dict:
        st = Stats()
        native.check(self._lib.m4d_transport_stats_get(self._h, ctypes.byref(st)))
        return {name: int(getattr(st, name)) for name, _ in Stats._fields_}

    # -- device regions ------------------------------------------------------------------------

    def allocate_region(self, length: int, domain: MemoryDomain):
        """Receive buffers: device frames land in pooled B200 memory, never in host RAM."""
        if domain == MemoryDomain.DEVICE and self._pool is not None:
            return self._pool.get(length)
        return super().allocate_region(length, domain)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._evacuate_loans()
            self._fast.forget(self._h)
            self._lib.m4d_transport_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _rank_in(message: str) -> int | None:
    import re

    m = re.search(r"rank (\d+)", message or "")
    return int(m.group(1)) if m else None
