"""``commshim-launch`` and ``commshim-bench``: the entry points the reference declares
(``pkg/pyproject.toml:14-16``) but never shipped.

    commshim-launch --np N [--transport nvlink|socket|sim] -- PROGRAM [ARGS...]
    commshim-bench  pingpong|app ...            (see benchcli)

or ``python -m paper_2101_08878_b200.cli launch|bench ...``.

``launch`` spawns N local processes (one per rank; rank r binds cuda:r % GPUs,
the nvlink transport's default) with ``RANK``/``WORLD_SIZE``/``LOCAL_RANK``/
``LOCAL_WORLD_SIZE`` (torchrun's names), ``MASTER_ADDR=127.0.0.1``, a fresh
``M4D_SESSION`` and ``COMMSHIM_TRANSPORT``; for ``socket`` also
``COMMSHIM_SOCKET_PORTS`` (one free 127.0.0.1 port per rank).  A program
opens its rank's transport with :func:`transport_from_env`.  The launcher
waits for every rank; when one fails it stops the others and exits with that
rank's code.  ``--transport sim`` runs N simulated ranks in THIS process
instead: PROGRAM is ``module:function``, an ``async def function(transport)``
run once per rank on one executor over a SimFabric.
"""

from __future__ import annotations

import argparse
import importlib
import os
import signal
import socket
import subprocess
import sys
import time
import uuid

from .errors import UsageError


def _free_ports(n: int) -> list[int]:
    socks, ports = [], []
    for _ in range(n):
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        socks.append(s)
        ports.append(s.getsockname()[1])
    for s in socks:
        s.close()
    return ports


def transport_from_env(connect_timeout: float = 60.0):
    """This process's transport, as ``commshim-launch`` (or torchrun) configured it."""
    from .transport import TransportConfig, transport_init

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    kind = os.environ.get("COMMSHIM_TRANSPORT", "nvlink")
    if kind == "socket":
        ports = [int(p) for p in os.environ["COMMSHIM_SOCKET_PORTS"].split(",")]
        cfg = TransportConfig(kind="socket", connect_timeout=connect_timeout,
                              rank_map={r: ("127.0.0.1", p) for r, p in enumerate(ports)})
    elif kind == "nvlink":
        cfg = TransportConfig(kind="nvlink", session=os.environ.get("M4D_SESSION"), connect_timeout=connect_timeout)
    else:
        raise UsageError(f"transport {kind!r} cannot be opened from the environment (sim runs in-process)")
    t = transport_init(world, rank, cfg)
    t.wait_ready(connect_timeout)
    return t


def _run_sim(np_: int, target: str) -> int:
    from .loop import TaskLoop, gather
    from .transport import SimFabric

    module, _, func = target.partition(":")
    if not func:
        raise UsageError("--transport sim needs PROGRAM as module:function")
    fn = getattr(importlib.import_module(module), func)
    loop = TaskLoop()
    fabric = SimFabric(np_, clock=loop.clock)
    loop.run_until_complete(gather(*(fn(fabric.transport(r)) for r in range(np_))))
    return 0


def launch_main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="commshim-launch", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--np", type=int, required=True, help="ranks to start")
    ap.add_argument("--transport", choices=["nvlink", "socket", "sim"], default="nvlink")
    ap.add_argument("--timeout", type=float, default=0.0, help="kill every rank after this many seconds (0: none)")
    ap.add_argument("program", nargs=argparse.REMAINDER, help="-- PROGRAM [ARGS...]")
    args = ap.parse_args(argv)
    prog = args.program[1:] if args.program[:1] == ["--"] else args.program
    if args.np < 1 or not prog:
        ap.print_usage(sys.stderr)
        return 2
    if args.transport == "sim":
        return _run_sim(args.np, prog[0])
    session = "launch" + uuid.uuid4().hex[:10]
    base = dict(os.environ, WORLD_SIZE=str(args.np), LOCAL_WORLD_SIZE=str(args.np), MASTER_ADDR="127.0.0.1",
                MASTER_PORT=str(_free_ports(1)[0]), M4D_SESSION=session, COMMSHIM_TRANSPORT=args.transport)
    if args.transport == "socket":
        base["COMMSHIM_SOCKET_PORTS"] = ",".join(map(str, _free_ports(args.np)))
    procs = []
    for r in range(args.np):
        env = dict(base, RANK=str(r), LOCAL_RANK=str(r))
        procs.append(subprocess.Popen(prog, env=env, start_new_session=True))
    deadline = time.monotonic() + args.timeout if args.timeout > 0 else None
    rc = 0
    live = list(procs)
    while live:
        for p in list(live):
            code = p.poll()
            if code is None:
                continue
            live.remove(p)
            if code != 0 and rc == 0:
                rc = code
                for q in live:  # one rank failed: the world cannot finish, stop the rest
                    os.killpg(q.pid, signal.SIGTERM)
        if deadline is not None and time.monotonic() > deadline and live:
            for q in live:
                os.killpg(q.pid, signal.SIGKILL)
            rc = rc or 124
        time.sleep(0.01)
    return rc


def bench_main(argv=None) -> int:
    from . import benchcli

    return benchcli.main(argv)


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    if not argv or argv[0] not in ("launch", "bench"):
        print("usage: python -m paper_2101_08878_b200.cli launch|bench ...", file=sys.stderr)
        return 2
    return launch_main(argv[1:]) if argv[0] == "launch" else bench_main(argv[1:])


if __name__ == "__main__":
    sys.exit(main())
