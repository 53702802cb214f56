"""Pull-routing check (test infrastructure): two ranks in this process on cuda:0 exchange a
window of mixed-size device frames (64 KiB - 32 MiB) under the pull knobs in the environment,
then print the bytes check and the transport's pull statistics as JSON."""

import json
import os
import sys
import uuid

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2101_08878_b200 import native  # noqa: E402
from paper_2101_08878_b200.transport import MemoryDomain, TransportConfig, transport_init  # noqa: E402
from paper_2101_08878_b200.transport.base import DeviceView  # noqa: E402

SIZES = [64 << 10, 1 << 20, (4 << 20) + 16, 32 << 20, 256 << 10, 8 << 20]


def main() -> int:
    session = "pr" + uuid.uuid4().hex[:8]
    ts = [transport_init(2, r, TransportConfig(kind="nvlink", session=session, device=0)) for r in range(2)]
    for t in ts:
        t.wait_ready(10)
    total = sum(SIZES)
    src, dst = native.DeviceBuffer(0, total), native.DeviceBuffer(0, total)
    pattern = (np.arange(total, dtype=np.uint64) * 7 % 253).astype(np.uint8)
    native.memcpy(src.ptr, pattern.ctypes.data, total)
    native.check(native.lib().m4d_device_sync(0))
    offs = np.cumsum([0] + SIZES)
    ok = True
    for lone in (False, True):  # a window of all six, then each alone (the ping-pong case)
        native.check(native.lib().m4d_memset(dst.ptr, 0, total, None))
        groups = [list(range(len(SIZES)))] if not lone else [[k] for k in range(len(SIZES))]
        for g in groups:
            rq = [ts[1].post_recv(0, 0, 40, DeviceView(dst.ptr + int(offs[k]), SIZES[k], 0), MemoryDomain.DEVICE)
                  for k in g]
            sq = [ts[0].post_send(0, 1, 40, DeviceView(src.ptr + int(offs[k]), SIZES[k], 0), MemoryDomain.DEVICE)
                  for k in g]
            while any(r.pending for r in rq + sq):
                for t in ts:
                    t.progress()
            ok = ok and not any(r.failed for r in rq + sq)
        got = np.frombuffer(native.to_host(dst.ptr, total), dtype=np.uint8)
        ok = ok and bool(np.array_equal(got, pattern))
    st = ts[1].native_stats()
    print(json.dumps({"ok": ok, "pulls": st["rendezvous_pulls"], "kernel_launches": st["pull_kernel_launches"]}))
    for t in ts:
        t.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
