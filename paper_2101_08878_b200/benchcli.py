"""``commshim-bench``: the paper's evaluation driver (SPEC.md benchcli module).

Usage (``python -m paper_2101_08878_b200.benchcli`` or the ``commshim-bench``
entry point the reference's ``pkg/pyproject.toml:14-16`` declares)::

    commshim-bench pingpong --sizes 1:134217728:x2 --mode cooperative|periodic:MS \\
                            --transport sim|nvlink [--device] --csv PATH
    commshim-bench app transpose-sum --dims N --block B [--workers W]
    commshim-bench app key-merge --rows R --fraction F [--workers W]

* ``pingpong`` runs ranks 0 and 1 in this process on one executor: the
  simulated transport on the loop's virtual clock (deterministic; latency =
  roundtrip/2 in virtual time) or the nvlink transport (host frames, or B200
  device frames with ``--device``).  Warm-up 10, measured 100 by default.
* ``app`` runs the operator on the local B200s (``--workers`` ranks in this
  process, one per visible GPU round-robin) and checks the determinism oracle
  (checksum / row count identical to the single-worker run) before any timing
  is reported; a mismatch exits 1.
* CSV columns are exactly ``benchmark,transport,mode,size,iters,mean_s,
  median_s,p99_s,throughput_Bps`` with a header row; ``--table`` prints aligned
  columns.  Exit codes: 0 pass, 1 correctness failure, 2 usage error.
"""

from __future__ import annotations

import argparse
import csv
import io
import statistics
import sys
import time
from dataclasses import dataclass, fields

from .errors import UsageError

CSV_COLUMNS = ("benchmark", "transport", "mode", "size", "iters", "mean_s", "median_s", "p99_s", "throughput_Bps")


@dataclass
class BenchRecord:
    benchmark: str
    transport: str
    mode: str
    size: int
    iters: int
    mean_s: float
    median_s: float
    p99_s: float
    throughput_Bps: float
    timestamp: float = 0.0  # not part of the CSV schema


def parse_sizes(spec: str) -> list[int]:
    """``lo:hi:xF`` (geometric) or ``lo:hi:+S`` (arithmetic) or a comma list; strictly increasing."""
    if ":" in spec:
        lo, hi, step = spec.split(":")
        lo, hi = int(lo), int(hi)
        out, v = [], lo
        if step.startswith("x"):
            f = int(step[1:])
            if f < 2:
                raise UsageError("geometric size step must be >= 2")
            while v <= hi:
                out.append(v)
                v = v * f if v else 1
        elif step.startswith("+"):
            s = int(step[1:])
            if s < 1:
                raise UsageError("arithmetic size step must be >= 1")
            out = list(range(lo, hi + 1, s))
        else:
            raise UsageError(f"size step {step!r} must start with x or +")
    else:
        out = [int(x) for x in spec.split(",") if x]
    if not out or any(b <= a for a, b in zip(out, out[1:])) or out[0] < 0:
        raise UsageError("sizes must be non-empty, non-negative and strictly increasing")
    return out


def _summarise(benchmark, transport, mode, size, samples) -> BenchRecord:
    ordered = sorted(samples)
    mean = statistics.fmean(samples)
    p99 = ordered[min(len(ordered) - 1, max(0, int(round(0.99 * len(ordered))) - 1))]
    return BenchRecord(benchmark, transport, mode, size, len(samples), mean, statistics.median(samples), p99,
                       (2 * size / (2 * mean)) if mean > 0 else 0.0, time.time())


def pingpong(sizes, *, transport: str = "sim", mode: str = "cooperative", warmup: int = 10, iters: int = 100,
             device: bool = False) -> list[BenchRecord]:
    """Ranks 0 and 1 in this process: rank 0 sends with ``send_payload`` and awaits the echo."""
    from .channels import build_comm_table
    from .loop import MonotonicClock, TaskLoop, gather
    from .messaging import Frame, ProgressMode, make_frame, recv_payload, send_payload, set_progress_mode
    from .transport import LinkModel, MemoryDomain, SimFabric, TransportConfig, transport_init

    if iters < 1 or warmup < 0:
        raise UsageError("iters must be >= 1 and warmup >= 0")
    if mode == "cooperative":
        pmode = ProgressMode.cooperative()
    elif mode.startswith("periodic:"):
        pmode = ProgressMode.periodic(float(mode.split(":", 1)[1]) / 1e3)
    else:
        raise UsageError(f"mode {mode!r} is not cooperative or periodic:MS")
    if transport == "sim":
        loop = TaskLoop()
        fabric = SimFabric(2, link=LinkModel(latency=1e-6, bandwidth=10e9), clock=loop.clock)
        ts = [fabric.transport(r) for r in range(2)]
    elif transport == "nvlink":
        import uuid

        loop = TaskLoop(MonotonicClock())
        session = "bench" + uuid.uuid4().hex[:10]
        ts = [transport_init(2, r, TransportConfig(kind="nvlink", session=session, device=0 if device else -1))
              for r in range(2)]
        for t in ts:
            t.wait_ready(10.0)
    else:
        raise UsageError(f"transport {transport!r} is not sim or nvlink")
    clock = ts[0].clock
    ch0, ch1 = build_comm_table(ts[0]).lookup(1), build_comm_table(ts[1]).lookup(0)
    records = []

    def frame_of(n):
        body = bytes(b"\xa5") * n
        if device:
            from .transport.nvlink import CudaRegion

            return Frame(CudaRegion(body, ts[0].device), n, MemoryDomain.DEVICE)
        return make_frame(body)

    async def leader(n, frame, count, out):
        for _ in range(count):
            start = clock.now()
            await send_payload(ts[0], ch0, 50, frame)
            await recv_payload(ts[0], ch0, 51)
            out.append(clock.to_seconds(clock.now() - start) / 2)

    async def echo(count):
        for _ in range(count):
            got = await recv_payload(ts[1], ch1, 50)
            await send_payload(ts[1], ch1, 51, got)

    async def main():
        for t in ts:
            set_progress_mode(t, pmode)
        for n in sizes:
            frame, samples = frame_of(n), []
            await gather(leader(n, frame, warmup, []), echo(warmup))
            await gather(leader(n, frame, iters, samples), echo(iters))
            records.append(_summarise("pingpong", transport + ("-device" if device else ""), mode, n, samples))
        for t in ts:
            set_progress_mode(t, ProgressMode.cooperative())

    try:
        loop.run_until_complete(main())
    finally:
        for t in ts:
            t.close()
    return records


def run_app(name: str, *, workers: int = 1, repetitions: int = 1, dims: int = 4096, block: int = 1024,
            rows: int = 1_000_000, fraction: float = 0.3) -> tuple[list[BenchRecord], bool]:
    """One operator on the local B200s (all ranks in this process), oracle-checked first."""
    from . import native

    gpus = max(1, native.device_count())
    devices = [r % gpus for r in range(workers)]
    records, ok = [], True
    if name == "transpose-sum":
        from .harness.transpose_sum import TransposeSum

        ref = TransposeSum.local_world(dims, block, 1, devices=[0])
        want = ref[0].step().checksum
        ranks = TransposeSum.local_world(dims, block, workers, devices=devices)
        for _ in range(repetitions):
            t0 = time.perf_counter()
            for r in ranks:
                r.launch()
            sums = {}
            for r in ranks:
                sums.update(r.read_block_sums())
            got = ranks[0].combine(sums).checksum if workers == 1 else _fsum_blocks(sums)
            dt = time.perf_counter() - t0
            ok &= got == want
            size = dims * dims * 8
            records.append(BenchRecord("transpose_sum", "nvlink", f"workers={workers}", size, 1, dt, dt, dt,
                                       2 * size / dt, time.time()))
    elif name == "key-merge":
        from .harness.key_merge import KeyMerge
        from .loop import MonotonicClock, TaskLoop

        if workers != 1:
            raise UsageError("in-process key-merge runs one worker; use bench.py under torchrun for more")
        km = KeyMerge(rows, fraction, device=devices[0])
        km.generate()
        loop = TaskLoop(MonotonicClock())
        want = None
        for _ in range(repetitions):
            t0 = time.perf_counter()
            got = loop.run_until_complete(km.run())
            dt = time.perf_counter() - t0
            want = want or got
            ok &= got == want
            records.append(BenchRecord("key_merge", "nvlink", f"workers={workers}", rows, 1, dt, dt, dt,
                                       2 * rows * 16 / dt, time.time()))
    else:
        raise UsageError(f"unknown app {name!r}")
    return records, ok


def _fsum_blocks(sums: dict) -> float:
    import math

    return math.fsum(sums[g] for g in sorted(sums))


def emit(records: list[BenchRecord], fmt: str = "csv", path: str | None = None) -> str:
    """CSV (header + one row per record, floats with 17 significant digits) or an aligned table."""
    if not records:
        raise UsageError("no records to emit")
    rows = [[getattr(r, c) for c in CSV_COLUMNS] for r in records]
    if fmt == "csv":
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(CSV_COLUMNS)
        for row in rows:
            w.writerow([f"{v:.17g}" if isinstance(v, float) else v for v in row])
        text = buf.getvalue()
    elif fmt == "table":
        cells = [list(CSV_COLUMNS)] + [[f"{v:.6g}" if isinstance(v, float) else str(v) for v in row] for row in rows]
        width = [max(len(c[i]) for c in cells) for i in range(len(CSV_COLUMNS))]
        text = "\n".join("  ".join(c[i].rjust(width[i]) for i in range(len(width))) for c in cells) + "\n"
    else:
        raise UsageError(f"format {fmt!r} is not csv or table")
    if path:
        try:
            with open(path, "w") as fh:
                fh.write(text)
        except OSError as exc:
            raise OSError(f"cannot write {path}: {exc}") from exc
    return text


def parse_csv(text: str) -> list[BenchRecord]:
    reader = csv.reader(io.StringIO(text))
    header = next(reader)
    if tuple(header) != CSV_COLUMNS:
        raise UsageError(f"unexpected CSV header {header}")
    types = {f.name: f.type for f in fields(BenchRecord)}
    out = []
    for row in reader:
        vals = {}
        for name, raw in zip(CSV_COLUMNS, row):
            kind = types[name]
            vals[name] = int(raw) if kind in (int, "int") else float(raw) if kind in (float, "float") else raw
        out.append(BenchRecord(**vals))
    return out


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="commshim-bench", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="cmd", required=True)
    pp = sub.add_parser("pingpong")
    pp.add_argument("--sizes", default="1:134217728:x2")
    pp.add_argument("--mode", default="cooperative")
    pp.add_argument("--transport", default="sim")
    pp.add_argument("--device", action="store_true", help="B200 device frames (nvlink transport)")
    pp.add_argument("--warmup", type=int, default=10)
    pp.add_argument("--iters", type=int, default=100)
    pp.add_argument("--csv")
    pp.add_argument("--table", action="store_true")
    app = sub.add_parser("app")
    app.add_argument("name", choices=["transpose-sum", "key-merge"])
    app.add_argument("--dims", type=int, default=4096)
    app.add_argument("--block", type=int, default=1024)
    app.add_argument("--rows", type=int, default=1_000_000)
    app.add_argument("--fraction", type=float, default=0.3)
    app.add_argument("--workers", type=int, default=1)
    app.add_argument("--repetitions", type=int, default=1)
    app.add_argument("--csv")
    app.add_argument("--table", action="store_true")
    try:
        args = ap.parse_args(argv)
    except SystemExit as exc:
        return 2 if exc.code else 0
    try:
        if args.cmd == "pingpong":
            records, ok = pingpong(parse_sizes(args.sizes), transport=args.transport, mode=args.mode,
                                   warmup=args.warmup, iters=args.iters, device=args.device), True
        else:
            records, ok = run_app(args.name, workers=args.workers, repetitions=args.repetitions, dims=args.dims,
                                  block=args.block, rows=args.rows, fraction=args.fraction)
            if not ok:
                print("correctness failure: result differs from the single-worker oracle", file=sys.stderr)
                return 1
        text = emit(records, "table" if args.table else "csv", args.csv)
        if not args.csv:
            sys.stdout.write(text)
    except UsageError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
