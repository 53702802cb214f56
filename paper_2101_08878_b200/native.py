"""ctypes binding to ``libm4d.so`` (the C ABI declared in ``include/m4d.h``).

The shared object is built in-tree by ``paper_2101_08878_b200/csrc/Makefile``
(``__graft_entry__.build()``).  There is deliberately no fallback: every
device operation of this package goes through this library, and a missing or
unloadable library raises :class:`NativeLibraryMissing` at first use.

Status codes map 1:1 onto the reference exception hierarchy
(``pkg/src/commshim/errors.py:6-89``) through :func:`check`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors

LIB_PATH = os.environ.get(
    "M4D_LIBRARY", os.path.join(os.path.dirname(os.path.abspath(__file__)), "libm4d.so")
)

# status codes (include/m4d.h)
OK = 0
ERR_CONFIGURATION = 1
ERR_STARTUP = 2
ERR_USAGE = 3
ERR_CHANNEL = 4
ERR_COUNT_OVERFLOW = 5
ERR_TRANSFER = 6
ERR_TRUNCATION = 7
ERR_CANCELLED = 8
ERR_PROTOCOL = 9
ERR_CLOSED = 10
ERR_BUSY = 11
ERR_CUDA = 12
ERR_NOMEM = 13
ERR_CAPACITY = 14


class NativeLibraryMissing(ImportError):
    """libm4d.so is absent or failed to load; build it with __graft_entry__.build()."""


class CudaError(errors.TransferError):
    """A CUDA runtime call inside libm4d failed."""


_c_void_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_size = ctypes.c_size_t
_dbl_p = ctypes.POINTER(ctypes.c_double)


class TsTask(ctypes.Structure):
    """Mirror of ``m4d_ts_task`` (include/m4d.h)."""

    _fields_ = [
        ("a", _c_void_p),
        ("bt", _c_void_p),
        ("y", _c_void_p),
        ("y2", _c_void_p),
        ("slot_y", _i32),
        ("slot_y2", _i32),
        ("diag", _i32),
        ("remote", _i32),
    ]


class TransportConfigC(ctypes.Structure):
    """Mirror of ``m4d_transport_config``."""

    _fields_ = [
        ("world", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("ring_bytes", ctypes.c_uint64),
        ("connect_timeout", ctypes.c_double),
        ("session", ctypes.c_char_p),
    ]


class Completion(ctypes.Structure):
    """Mirror of ``m4d_completion``."""

    _fields_ = [
        ("req_id", ctypes.c_uint64),
        ("status", ctypes.c_int32),
        ("kind", ctypes.c_int32),
        ("bytes", ctypes.c_uint64),
    ]


class TransportStats(ctypes.Structure):
    """Mirror of ``m4d_transport_stats``."""

    _fields_ = [(name, ctypes.c_uint64) for name in (
        "sends_completed", "recvs_completed", "bytes_sent", "bytes_received", "eager_bytes",
        "nvlink_bytes", "rendezvous_pulls", "unexpected_messages", "pull_kernel_launches",
        "eager_device_sends", "eager_device_loans", "eager_proxy_copies",
        "eager_proxy_launches")]


# name -> (restype, argtypes); every symbol include/m4d.h declares.
SIGNATURES: dict[str, tuple] = {
    "m4d_last_error": (_size, [ctypes.c_char_p, _size]),
    "m4d_version": (ctypes.c_int, []),
    "m4d_device_count": (ctypes.c_int, []),
    "m4d_pointer_device": (ctypes.c_int, [_c_void_p, ctypes.POINTER(ctypes.c_int)]),
    "m4d_mem_get_info": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
    "m4d_set_device": (ctypes.c_int, [ctypes.c_int]),
    "m4d_stream_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_c_void_p)]),
    "m4d_stream_destroy": (ctypes.c_int, [_c_void_p]),
    "m4d_stream_sync": (ctypes.c_int, [_c_void_p]),
    "m4d_device_sync": (ctypes.c_int, [ctypes.c_int]),
    "m4d_event_create": (ctypes.c_int, [ctypes.POINTER(_c_void_p)]),
    "m4d_event_destroy": (ctypes.c_int, [_c_void_p]),
    "m4d_event_record": (ctypes.c_int, [_c_void_p, _c_void_p]),
    "m4d_event_sync": (ctypes.c_int, [_c_void_p]),
    "m4d_stream_wait_event": (ctypes.c_int, [_c_void_p, _c_void_p]),
    "m4d_event_elapsed_ms": (ctypes.c_int, [_c_void_p, _c_void_p, ctypes.POINTER(ctypes.c_float)]),
    "m4d_malloc": (ctypes.c_int, [ctypes.c_int, _size, ctypes.POINTER(_c_void_p)]),
    "m4d_free": (ctypes.c_int, [_c_void_p]),
    "m4d_host_alloc": (ctypes.c_int, [_size, ctypes.POINTER(_c_void_p)]),
    "m4d_host_free": (ctypes.c_int, [_c_void_p]),
    "m4d_memcpy": (ctypes.c_int, [_c_void_p, _c_void_p, _size, _c_void_p]),
    "m4d_memset": (ctypes.c_int, [_c_void_p, ctypes.c_int, _size, _c_void_p]),
    "m4d_ipc_export": (ctypes.c_int, [_c_void_p, ctypes.c_char_p, ctypes.POINTER(_u64)]),
    "m4d_ipc_import": (ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(_c_void_p)]),
    "m4d_ipc_close": (ctypes.c_int, [_c_void_p]),
    "m4d_enable_peer": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "m4d_transport_open": (ctypes.c_int, [ctypes.POINTER(TransportConfigC), ctypes.POINTER(_c_void_p)]),
    "m4d_transport_wait_ready": (ctypes.c_int, [_c_void_p, ctypes.c_double]),
    "m4d_transport_mesh_ready": (ctypes.c_int, [_c_void_p]),
    "m4d_transport_post_send": (ctypes.c_int, [_c_void_p, ctypes.c_uint32, ctypes.c_int, ctypes.c_uint32, _c_void_p,
                                               _u64, ctypes.c_int, ctypes.c_int, _u64, ctypes.POINTER(Completion)]),
    "m4d_transport_post_recv": (ctypes.c_int, [_c_void_p, ctypes.c_uint32, ctypes.c_int, ctypes.c_uint32, _c_void_p,
                                               _u64, ctypes.c_int, ctypes.c_int, _u64, ctypes.POINTER(Completion)]),
    "m4d_transport_post_many": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_int, ctypes.c_uint32,
                                                _c_void_p, _c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                _c_void_p, _c_void_p, _c_void_p]),
    "m4d_transport_progress": (ctypes.c_int, [_c_void_p, ctypes.POINTER(Completion), ctypes.c_int]),
    "m4d_transport_pending_completions": (ctypes.c_int, [_c_void_p]),
    "m4d_transport_eager_device_max": (_u64, [_c_void_p]),
    "m4d_transport_take_loan": (ctypes.c_int, [_c_void_p, _u64, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
    "m4d_transport_release_loan": (ctypes.c_int, [_c_void_p, _u64]),
    "m4d_transport_cancel": (ctypes.c_int, [_c_void_p, _u64, ctypes.POINTER(ctypes.c_int)]),
    "m4d_transport_purge_channel": (ctypes.c_int, [_c_void_p, ctypes.c_uint32]),
    "m4d_transport_peer_alive": (ctypes.c_int, [_c_void_p, ctypes.c_int]),
    "m4d_transport_set_pull_ctas": (ctypes.c_int, [_c_void_p, ctypes.c_int]),
    "m4d_transport_set_pull_engine": (ctypes.c_int, [_c_void_p, ctypes.c_int]),
    "m4d_transport_stats_get": (ctypes.c_int, [_c_void_p, ctypes.POINTER(TransportStats)]),
    "m4d_transport_close": (ctypes.c_int, [_c_void_p]),
    "m4d_merge_generate": (ctypes.c_int, [_c_void_p, _c_void_p, _i64, _i64, _u64, _u64, _u64, _c_void_p]),
    "m4d_partition_scratch_bytes": (_size, [_i64, ctypes.c_int]),
    "m4d_partition": (ctypes.c_int, [_c_void_p, _c_void_p, _i64, ctypes.c_int, ctypes.c_int, _c_void_p,
                                     _c_void_p, _c_void_p, _size, _c_void_p]),
    "m4d_partition_runs": (ctypes.c_int, [_c_void_p, _i64, _c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          _c_void_p, _c_void_p, _c_void_p, _size, _c_void_p]),
    "m4d_partition_runs_scratch_bytes": (_size, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "m4d_owner_coarse_count": (ctypes.c_int, [ctypes.c_int]),
    "m4d_partition_owner_coarse": (ctypes.c_int, [_c_void_p, _c_void_p, _i64, ctypes.c_int, ctypes.c_int, _c_void_p,
                                                  _c_void_p, _c_void_p, _size, _c_void_p]),
    "m4d_partition_owner_plan": (ctypes.c_int, [_c_void_p, _c_void_p, _i64, ctypes.c_int, ctypes.c_int, _c_void_p,
                                                _c_void_p, _size, _c_void_p]),
    "m4d_partition_owner_push": (ctypes.c_int, [_c_void_p, _c_void_p, _i64, ctypes.c_int, ctypes.c_int, _c_void_p,
                                                _c_void_p, _size, _c_void_p]),
    "m4d_push_fine_smem_limit": (_size, []),
    "m4d_partition_owner_push_fine": (ctypes.c_int, [_c_void_p, _c_void_p, _i64, ctypes.c_int, ctypes.c_int, _c_void_p,
                                                     ctypes.c_int, _c_void_p, _c_void_p, _c_void_p, _size, _c_void_p]),
    "m4d_partition_launches": (ctypes.c_int, [ctypes.c_int]),
    "m4d_fine_count_smem_limit": (_size, []),
    "m4d_partition_fine_counts": (ctypes.c_int, [_c_void_p, _c_void_p, _i64, ctypes.c_int, ctypes.c_int, _c_void_p,
                                                 _c_void_p]),
    "m4d_partition_runs_counted": (ctypes.c_int, [_c_void_p, _i64, _c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                  _c_void_p, _c_void_p, _c_void_p, _c_void_p, _size, _c_void_p]),
    "m4d_join_partition_rows": (ctypes.c_int, []),
    "m4d_hash_join": (ctypes.c_int, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, ctypes.c_int,
                                     _c_void_p, _c_void_p, _c_void_p, _i64, _c_void_p, _c_void_p]),
    "m4d_fill_block_f64": (ctypes.c_int, [_c_void_p, _i64, _i64, _i64, _i64, _u64, _c_void_p]),
    "m4d_ts_plan_create": (
        ctypes.c_int,
        [ctypes.c_int, ctypes.POINTER(TsTask), ctypes.c_int, _i64, ctypes.c_int, ctypes.POINTER(_c_void_p)],
    ),
    "m4d_ts_run": (ctypes.c_int, [_c_void_p, _c_void_p, _c_void_p, _c_void_p]),
    "m4d_ts_plan_destroy": (ctypes.c_int, [_c_void_p]),
    "m4d_ts_launches_per_run": (ctypes.c_int, [_c_void_p]),
    "m4d_ts_plan_uses_tma": (ctypes.c_int, [_c_void_p]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load (once) and return the configured ctypes handle; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                )
            try:
                handle = ctypes.CDLL(LIB_PATH)
            except OSError as exc:
                raise NativeLibraryMissing(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (restype, argtypes) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = restype
                fn.argtypes = argtypes
            _lib = handle
    return _lib


_fast = None


def fast():
    """The CPython fast path of the transport calls (csrc/pyfast.cpp), bound to
    this process's libm4d.so; raises loudly when it was not built."""
    global _fast
    if _fast is not None:
        return _fast
    handle = lib()
    try:
        from . import _m4dfast
    except ImportError as exc:
        raise NativeLibraryMissing(f"_m4dfast extension not built ({exc}): run __graft_entry__.build()") from exc
    addr = [ctypes.cast(getattr(handle, n), ctypes.c_void_p).value
            for n in ("m4d_transport_post_send", "m4d_transport_post_recv", "m4d_transport_progress",
                      "m4d_transport_take_loan", "m4d_transport_release_loan", "m4d_transport_post_many")]
    _m4dfast.bind(*addr)
    _fast = _m4dfast
    return _fast


def last_error() -> str:
    buf = ctypes.create_string_buffer(512)
    lib().m4d_last_error(buf, len(buf))
    return buf.value.decode("utf-8", "replace")


def error_for(status: int, message: str, *, rank: int | None = None, bytes_moved: int = 0):
    """Exception object for a status code (errors.py classes, 1:1)."""
    if status == ERR_CONFIGURATION:
        return errors.ConfigurationError(message)
    if status == ERR_STARTUP:
        return errors.StartupError(message, rank=rank)
    if status == ERR_USAGE:
        return errors.UsageError(message)
    if status == ERR_CHANNEL:
        return errors.ChannelError(message)
    if status == ERR_COUNT_OVERFLOW:
        return errors.UsageError(message)
    if status == ERR_TRUNCATION:
        return errors.TruncationError(message, bytes_moved=bytes_moved)
    if status == ERR_CANCELLED:
        return errors.CancelledTransferError(message, bytes_moved=bytes_moved)
    if status == ERR_PROTOCOL:
        return errors.ProtocolError(message)
    if status == ERR_CLOSED:
        return errors.CommClosedError(message)
    if status == ERR_BUSY:
        return errors.BusyError(message)
    if status == ERR_CUDA:
        return CudaError(message, bytes_moved=bytes_moved)
    if status == ERR_TRANSFER:
        return errors.TransferError(message, bytes_moved=bytes_moved)
    return errors.CommShimError(f"libm4d status {status}: {message}")


def check(status: int) -> None:
    if status != OK:
        raise error_for(status, last_error())


# -- thin RAII wrappers -------------------------------------------------------------


class Stream:
    """A non-blocking CUDA stream owned by libm4d."""

    def __init__(self, device: int):
        self.device = device
        h = _c_void_p()
        check(lib().m4d_stream_create(device, ctypes.byref(h)))
        self.handle = h.value

    def synchronize(self) -> None:
        check(lib().m4d_stream_sync(self.handle))

    def close(self) -> None:
        if self.handle is not None and _lib is not None:
            lib().m4d_stream_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Event:
    def __init__(self):
        h = _c_void_p()
        check(lib().m4d_event_create(ctypes.byref(h)))
        self.handle = h.value

    def record(self, stream: Stream | None) -> None:
        if stream is not None:
            set_device(stream.device)  # a stream belongs to its device (ranks may share a process)
        check(lib().m4d_event_record(self.handle, stream.handle if stream else None))

    def synchronize(self) -> None:
        check(lib().m4d_event_sync(self.handle))

    def wait_on(self, stream: Stream) -> None:
        """Make later work on `stream` wait for this event (no host synchronisation)."""
        check(lib().m4d_stream_wait_event(stream.handle, self.handle))

    def elapsed_ms(self, later: "Event") -> float:
        out = ctypes.c_float()
        check(lib().m4d_event_elapsed_ms(self.handle, later.handle, ctypes.byref(out)))
        return float(out.value)

    def __del__(self):
        try:
            if self.handle is not None and _lib is not None:
                lib().m4d_event_destroy(self.handle)
        except Exception:
            pass


class DeviceBuffer:
    """A dedicated cudaMalloc allocation (exportable through CUDA IPC)."""

    __slots__ = ("device", "nbytes", "ptr", "_owned")

    def __init__(self, device: int, nbytes: int, *, ptr: int | None = None):
        self.device = device
        self.nbytes = int(nbytes)
        if ptr is None:
            h = _c_void_p()
            check(lib().m4d_malloc(device, self.nbytes, ctypes.byref(h)))
            self.ptr = h.value
            self._owned = True
        else:
            self.ptr = ptr
            self._owned = False

    def free(self) -> None:
        if self._owned and self.ptr:
            lib().m4d_free(self.ptr)
        self.ptr = None
        self._owned = False

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class PinnedHostBuffer:
    """Page-locked host memory (cudaHostAlloc) for async H2D/D2H copies."""

    __slots__ = ("nbytes", "ptr")

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        h = _c_void_p()
        check(lib().m4d_host_alloc(self.nbytes, ctypes.byref(h)))
        self.ptr = h.value

    def as_numpy(self, dtype="u1"):
        import numpy as np

        raw = (ctypes.c_char * self.nbytes).from_address(self.ptr)
        return np.frombuffer(raw, dtype=dtype)

    def free(self) -> None:
        if self.ptr:
            lib().m4d_host_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def memcpy(dst: int, src: int, nbytes: int, stream: Stream | None = None) -> None:
    if stream is not None:
        set_device(stream.device)
    check(lib().m4d_memcpy(dst, src, nbytes, stream.handle if stream else None))


def memset(dst: int, value: int, nbytes: int, stream: Stream | None = None) -> None:
    check(lib().m4d_memset(dst, value, nbytes, stream.handle if stream else None))


def pointer_device(ptr: int) -> int:
    """CUDA device owning `ptr` (-1: host memory)."""
    dev = ctypes.c_int(-1)
    check(lib().m4d_pointer_device(ptr, ctypes.byref(dev)))
    return dev.value


def mem_get_info(device: int) -> tuple[int, int]:
    """(free, total) bytes of `device` (cudaMemGetInfo)."""
    free, total = _u64(), _u64()
    check(lib().m4d_mem_get_info(device, ctypes.byref(free), ctypes.byref(total)))
    return free.value, total.value


def device_count() -> int:
    return int(lib().m4d_device_count())


def set_device(device: int) -> None:
    check(lib().m4d_set_device(device))


def ipc_export(ptr: int) -> tuple[bytes, int]:
    handle = ctypes.create_string_buffer(64)
    off = _u64()
    check(lib().m4d_ipc_export(ptr, handle, ctypes.byref(off)))
    return handle.raw, int(off.value)


def ipc_import(device: int, handle: bytes) -> int:
    if len(handle) != 64:
        raise errors.UsageError("CUDA IPC handles are 64 bytes")
    out = _c_void_p()
    check(lib().m4d_ipc_import(device, handle, ctypes.byref(out)))
    return int(out.value)


def ipc_close(base: int) -> None:
    check(lib().m4d_ipc_close(base))


def to_host(ptr: int, nbytes: int, stream: Stream | None = None) -> bytes:
    """Synchronous device -> host copy (tests and result readback)."""
    buf = ctypes.create_string_buffer(max(1, nbytes))
    if nbytes:
        memcpy(ctypes.addressof(buf), ptr, nbytes, stream)
        if stream is not None:
            stream.synchronize()
        else:
            check(lib().m4d_stream_sync(None))
    return buf.raw[:nbytes]
