#!/usr/bin/env python3
"""Benchmark driver (graft contract): one JSON line on rank 0.

Default workload (N = 1 and under torchrun for N > 1): BASELINE.json config 3,
``sum(x + x.T)`` on a 40000 x 40000 fp64 array in 2000 x 2000 chunks,
round-robin row-major block ownership over N B200s, weak in
nothing: the array is fixed, so ``scaling`` is "strong".

* ``value``  : wall time per step (ms, max over ranks, CUDA events on the
  launching stream) with x resident in HBM: fused transpose-add-reduce kernel
  (partner tiles of other GPUs read over NVLink inside the kernel), block-sum
  gather, final fsum on the host.
* ``e2e``    : the same step through the public harness API with x in pinned
  HOST memory: H2D of this rank's x blocks, kernel, D2H of the result.
* ``roofline``: the fused kernel's algorithmic bytes / its event-timed
  duration against MEASURED_PEAKS.json (HBM) or the measured 770 GB/s peer
  copy (NVLink), whichever bounds it.
* ``cpu_baseline``: the oracle (oracle/liboracle.so) over the full array with x
  resident in host memory, all host threads; its block sums are also the
  full-size parity check of every block and of the checksum.

``--impl reference`` times the CPU restatement of the path (the reference has
no operator code) on the same config; under torchrun only
rank 0 runs it.  Other workloads: ``--workload key_merge|p2p``.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from types import SimpleNamespace

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

NVLINK_PEER_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)


# -- environment ------------------------------------------------------------------------------


def load_peaks() -> dict:
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            peaks = json.load(fh)
        peaks["_source"] = "measured (MEASURED_PEAKS.json)"
        return peaks
    except OSError:
        return {"hbm_gbs": 6650.0, "_source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self._reader = None

    def start(self) -> None:
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self._reader = threading.Thread(target=self._pump, daemon=True)
        self._reader.start()

    def _pump(self) -> None:
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self._reader:
            self._reader.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


class Dist:
    """Rank/world plumbing over torch.distributed (NCCL) when launched by torchrun."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.device = self.local_rank
        self.shared = False
        self.torch = None
        self.gloo = None
        if self.world > 1:
            import torch
            import torch.distributed as dist

            # More ranks than GPUs (a functional check of an N-rank run on a smaller box,
            # never a measurement): ranks share GPUs round-robin, NCCL cannot, so the
            # default group is gloo too.
            ngpu = torch.cuda.device_count()
            local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(self.world)))
            shared = ngpu and local_world > ngpu
            self.device = self.local_rank % ngpu if shared else self.local_rank
            self.shared = bool(shared)
            torch.cuda.set_device(self.device)
            if shared:
                print(f"bench: {local_world} ranks on {ngpu} GPUs (shared; functional check only)", file=sys.stderr)
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.device))
            self.gloo = dist.new_group(backend="gloo")
            self.torch = torch
            self.dist = dist

    def barrier(self) -> None:
        if self.world > 1:
            self.dist.barrier(group=self.gloo)

    def allgather_bytes(self, blob: bytes) -> list[bytes]:
        if self.world == 1:
            return [blob]
        out = [None] * self.world
        self.dist.all_gather_object(out, blob, group=self.gloo)
        return out

    def max(self, value: float) -> float:
        if self.world == 1:
            return value
        t = self.torch.tensor([value], dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.gloo)
        return float(t.item())

    def sum(self, value: float) -> float:
        if self.world == 1:
            return value
        t = self.torch.tensor([value], dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.gloo)
        return float(t.item())

    def close(self) -> None:
        if self.world > 1:
            self.dist.destroy_process_group()


def open_transport(dist: "Dist", device: int):
    """This rank's nvlink transport (session derived from the torchrun rendezvous), opened
    once per process and shared by every workload of the run (closed by main)."""
    from paper_2101_08878_b200.transport import TransportConfig, transport_init

    if getattr(dist, "transport", None) is None:
        t = transport_init(dist.world, dist.rank, TransportConfig(kind="nvlink", device=device, connect_timeout=60))
        t.wait_ready()
        dist.transport = t
    return dist.transport


def recorded_traffic(key: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture, if any."""
    try:
        with open(os.path.join(HERE, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(key)
    except (OSError, ValueError):
        return None


def host_info() -> dict:
    """The host the CPU baseline ran on (core counts, CPU model, RAM)."""
    info = {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}
    try:
        with open("/proc/cpuinfo") as fh:
            info["cpu_model"] = next((ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")), None)
        with open("/proc/meminfo") as fh:
            kb = next((int(ln.split()[1]) for ln in fh if ln.startswith("MemTotal")), 0)
        info["mem_total_gb"] = round(kb / 2**20, 1)
    except (OSError, ValueError):
        pass
    return info


def emit(line: dict) -> None:
    cpu = line.get("cpu_baseline")
    if isinstance(cpu, dict) and "host" not in cpu:
        cpu["host"] = host_info()
    print(json.dumps(line), flush=True)


# -- transpose_sum -------------------------------------------------------------------------------


def ts_cpu_full(n: int, b: int, threads: int, min_seconds: float = 10.0) -> dict:
    """The oracle (C restatement, all host threads) over the FULL array with x resident in
    host memory (generated outside the timing, as the GPU's x is): every y block and block
    sum, repeated until `min_seconds` of compute were timed (at least one pass).  The block
    sums pin the GPU result at full size."""
    import oracle

    nb = n // b
    x = [oracle.gen_block_c(n, (g // nb) * b, (g % nb) * b, b) for g in range(nb * nb)]
    a_blocks = x
    bt_blocks = [x[(g % nb) * nb + g // nb] for g in range(nb * nb)]
    y_blocks = [np_empty(b) for _ in range(nb * nb)]
    passes, t0 = 0, time.perf_counter()
    while True:
        sums = oracle.transpose_sum_resident_c(a_blocks, bt_blocks, y_blocks, threads)
        passes += 1
        dt = time.perf_counter() - t0
        if dt >= min_seconds:
            break
    return {"seconds": dt, "passes": passes, "ms": dt / passes * 1e3, "sums": sums}


def np_empty(b: int):
    import numpy as np

    return np.empty((b, b))


def bench_transpose_sum(args, dist: Dist, peaks: dict) -> dict | None:
    from paper_2101_08878_b200 import native
    from paper_2101_08878_b200.harness.transpose_sum import TransposeSum

    n, b = args.n, args.block
    device = dist.device
    native.set_device(device)
    exchange = None
    if dist.world > 1:
        from paper_2101_08878_b200.harness.collectives import allgather_sync

        transport = open_transport(dist, device)
        tags = iter(range(920, 10**9))
        exchange = lambda blob: allgather_sync(transport, blob, next(tags))  # noqa: E731
    ts = TransposeSum(n, b, rank=dist.rank, world=dist.world, device=device, exchange=exchange).setup()
    stream = ts.stream
    e0, e1 = native.Event(), native.Event()

    def step():
        return ts.step()

    # warm-up (also the parity check against the oracle on sampled blocks)
    for _ in range(args.warmup):
        res = step()
    checksum = res.checksum

    # -- timed region: K full steps (kernel + gather + fsum) --
    sampler = ClockSampler(device)
    dist.barrier()
    stream.synchronize()
    sampler.start()
    t_wall = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        res = step()
    e1.record(stream)
    e1.synchronize()
    wall_ms = (time.perf_counter() - t_wall) * 1e3 / args.steps
    step_ms_local = max(e0.elapsed_ms(e1) / args.steps, wall_ms)
    dist.barrier()
    clocks = sampler.stop()
    step_ms = dist.max(step_ms_local)
    if res.checksum != checksum:
        raise RuntimeError("checksum changed between steps")

    # -- kernel-only timing for the roofline (same stream, K back-to-back launches) --
    dist.barrier()
    stream.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        ts.launch()
    e1.record(stream)
    e1.synchronize()
    kernel_ms = dist.max(e0.elapsed_ms(e1) / args.steps)

    alg = ts.algorithmic_bytes()
    hbm_bytes = alg["hbm"]
    nvl_bytes = alg["nvlink"]
    hbm_peak = float(peaks["hbm_gbs"])
    t_hbm = hbm_bytes / (hbm_peak * 1e9)
    t_nvl = nvl_bytes / (NVLINK_PEER_GBS * 1e9)
    if t_nvl > t_hbm:
        roof = {"bound": "nvlink", "achieved": nvl_bytes / (kernel_ms * 1e-3) / 1e9, "peak": NVLINK_PEER_GBS,
                "unit": "GB/s", "peak_source": "measured peer copy, B200_PROFILING.md"}
    else:
        roof = {"bound": "hbm", "achieved": hbm_bytes / (kernel_ms * 1e-3) / 1e9, "peak": hbm_peak,
                "unit": "GB/s", "peak_source": peaks["_source"]}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = args.traffic if args.traffic is not None else recorded_traffic(f"transpose_sum/{n}/{b}/{dist.world}")
    roof["kernel"] = "ts_kernel_tma (transpose_sum.cu; event time includes the tiny fold launch)"
    roof["kernel_ms"] = kernel_ms
    roof["algorithmic_bytes_per_launch"] = {"hbm": hbm_bytes, "nvlink": nvl_bytes}
    roof["t_roof_ms"] = max(t_hbm, t_nvl) * 1e3

    # -- e2e: x from pinned host memory through the public harness API --
    # Two different arrays (seed, seed + 1) alternate between steps, each uploaded with
    # TransposeSum.load_x (H2D + the cross-rank input-ready fence) and checked against its
    # own resident checksum, so a kernel that read a peer's pool before the upload landed
    # would fail the run.
    e2e = None
    if not args.skip_e2e:
        pool = len(ts.owned) * ts.block_bytes
        hosts, want = [], []
        for seed in (ts.seed, ts.seed + 1):
            ts.seed = seed
            ts.generate()
            h = native.PinnedHostBuffer(pool)
            native.memcpy(h.ptr, ts.x.ptr, pool, stream)  # snapshot (untimed)
            stream.synchronize()
            hosts.append(h)
            want.append(ts.step().checksum)  # resident checksum of this array (untimed)
        if want[0] != checksum:
            raise RuntimeError("regenerated x does not reproduce the timed checksum")
        e2e_steps = max(2, min(args.steps, 4))
        dist.barrier()
        t0 = time.perf_counter()
        e0.record(stream)
        for k in range(e2e_steps):
            ts.load_x(hosts[k % 2].ptr)
            r = ts.step()
            if r.checksum != want[k % 2]:
                raise RuntimeError(f"e2e step {k}: checksum {r.checksum!r} != {want[k % 2]!r} (input fence?)")
        e1.record(stream)
        e1.synchronize()
        e2e_ms = max(e0.elapsed_ms(e1), (time.perf_counter() - t0) * 1e3) / e2e_steps
        e2e_ms = dist.max(e2e_ms)
        e2e = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": int(dist.sum(pool)),
               "d2h_bytes_per_step": int(dist.sum(len(ts.owned) * 8)), "steps": e2e_steps,
               "inputs": "two arrays alternated between steps (seed, seed + 1), each checked"}
        for h in hosts:
            h.free()

    # -- parity (outside timing) and the CPU baseline --
    # With the CPU leg: the oracle computes the FULL array on the host (all y blocks and
    # block sums, every host thread), which is both the baseline and full-size parity of
    # every block sum and of the checksum.  Without it: 8 sampled blocks.
    parity = None
    cpu = None
    if dist.rank == 0:
        import math as _m

        import oracle

        if not args.skip_cpu:
            threads = len(os.sched_getaffinity(0))
            full = ts_cpu_full(n, args.block, threads, min_seconds=min(10.0, args.cpu_seconds))
            ref_sums = {g: float(v) for g, v in enumerate(full["sums"])}
            worst = max(abs(res.block_sums[g] - ref_sums[g]) / max(abs(ref_sums[g]), 1e-300) for g in ref_sums)
            want = _m.fsum(ref_sums[g] for g in sorted(ref_sums))
            parity = {"blocks": len(ref_sums), "scope": "every block of the full array", "max_rel_err": float(worst),
                      "checksum_oracle": want, "checksum_rel_err": abs(checksum - want) / abs(want),
                      "tolerance": 1e-12, "ok": bool(worst <= 1e-12 and abs(checksum - want) <= 1e-12 * abs(want))}
            cpu = {"value": full["ms"], "unit": "ms", "cores": threads, "kind": "port",
                   "sample": f"oracle C restatement over the full {n}^2 array (all {ts.nb ** 2} blocks, x resident "
                             f"in host RAM) x {full['passes']} passes in {full['seconds']:.1f} s"}
        else:
            sample = sorted(res.block_sums)[:: max(1, len(res.block_sums) // 8)][:8]
            ref = oracle.transpose_sum_blocks_c(n, b, sample, threads=os.cpu_count() or 1)
            worst = max(abs(res.block_sums[g] - r) / abs(r) for g, r in zip(sample, ref))
            parity = {"blocks": len(sample), "scope": "sampled blocks", "max_rel_err": float(worst),
                      "tolerance": 1e-12, "ok": bool(worst <= 1e-12)}
        if not parity["ok"]:
            raise RuntimeError(f"transpose_sum parity failed: {parity}")
    launches_per_step = native.lib().m4d_ts_launches_per_run(ts._plan)
    ts.close()
    ts.x.free()  # 25.6 GB of pools at N=1: give the HBM back before the next workload
    ts.y.free()
    if dist.rank != 0:
        return None
    launches = args.steps * launches_per_step
    return {
        "metric": f"x+x.T sum wall time ({n}^2 fp64, {b}^2 chunks)",
        "value": step_ms,
        "unit": "ms",
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_ms,
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (splitmix64 generator, BASELINE.md §3)",
        "config": ts_config(n, b, dist.world),
        "checksum": checksum,
        "gpu_launches": launches,
        "roofline": roof,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": parity,
        "clocks": clocks,
        "wall_ms_per_step": wall_ms,
    }


# -- key_merge ------------------------------------------------------------------------------------


def km_cpu_sample(rows: int, min_seconds: float = 10.0, fraction: float = 0.3) -> dict:
    """Oracle CPU join (C, all host threads: radix partition + per-partition hash joins) of
    the FULL global inputs (`rows` per side, generated outside the timed region, as the
    GPU's inputs are): the digest pins the GPU result at full size; the join is repeated
    to >= min_seconds for the timing (min_seconds 0: one run)."""
    import oracle

    threads = len(os.sched_getaffinity(0))
    band = oracle.merge_band(rows, fraction)
    lk, lv = oracle.gen_side_c(0, rows, rows, oracle.SEED_LEFT, 0)
    rk, rv = oracle.gen_side_c(0, rows, rows, oracle.SEED_RIGHT, band)
    done, t0 = 0, time.perf_counter()
    digest = None
    while True:
        got = oracle.join_mt_c(lk, lv, rk, rv, threads)
        if digest is not None and got != digest:
            raise RuntimeError("multithreaded CPU join is not deterministic")
        digest = got
        done += 1
        dt = time.perf_counter() - t0
        if dt >= min_seconds:
            break
    if rows <= 2_000_000 and digest != oracle.key_merge_c(rows, 1, fraction):
        raise RuntimeError("multithreaded CPU join disagrees with the scalar oracle")
    return {"seconds": dt, "runs": done, "rows": rows, "threads": threads, "digest": tuple(digest),
            "ms": dt / done * 1e3}


def digest_rows(km) -> int:
    return int(getattr(km, "rows_out", 0))


def bench_key_merge(args, dist: Dist, peaks: dict) -> dict | None:
    from paper_2101_08878_b200 import native
    from paper_2101_08878_b200.harness.key_merge import KeyMerge
    from paper_2101_08878_b200.loop import MonotonicClock, TaskLoop

    device = dist.device
    native.set_device(device)
    transport = open_transport(dist, device) if dist.world > 1 else None
    km = KeyMerge(args.rows, args.fraction, rank=dist.rank, world=dist.world, device=device, transport=transport)
    km.generate()
    loop = TaskLoop(MonotonicClock())
    stream = km.stream
    e0, e1 = native.Event(), native.Event()
    for _ in range(args.warmup):
        digest = loop.run_until_complete(km.run_global())
    sampler = ClockSampler(device)
    dist.barrier()
    stream.synchronize()
    sampler.start()
    km.launches = 0
    km.timing, km.kernel_ms = True, {"partition": 0.0, "join": 0.0}
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        got = loop.run_until_complete(km.run_global())
    e1.record(stream)
    e1.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / args.steps
    step_ms = dist.max(max(wall, e0.elapsed_ms(e1) / args.steps))
    dist.barrier()
    clocks = sampler.stop()
    if got != digest:
        raise RuntimeError("merge digest changed between steps")
    launches = km.launches
    km.timing = False
    kern = {k: v / args.steps for k, v in km.kernel_ms.items()}  # this rank's per-step event times

    # per-phase timing on this rank: one extra step with a synchronise at each phase boundary
    km.profile = True
    loop.run_until_complete(km.run_global())
    km.profile = False
    phase = {k: round(v, 3) for k, v in km.phases.items()}
    # and an event trace of one more step without any added synchronisation (overlap visible)
    km.tracing = True
    loop.run_until_complete(km.run_global())
    km.tracing = False
    trace = dict(km.trace)

    alg = km.algorithmic_bytes()
    hbm_peak = float(peaks["hbm_gbs"])
    t_hbm = alg["hbm"] / (hbm_peak * 1e9)
    t_nvl = alg["nvlink"] / (NVLINK_PEER_GBS * 1e9)
    t_meas = step_ms * 1e-3
    if t_nvl > t_hbm:
        roof = {"bound": "nvlink", "achieved": alg["nvlink"] / t_meas / 1e9, "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                "peak_source": "measured peer copy, B200_PROFILING.md"}
    else:
        roof = {"bound": "hbm", "achieved": alg["hbm"] / t_meas / 1e9, "peak": hbm_peak, "unit": "GB/s",
                "peak_source": peaks["_source"]}
    traffic = args.traffic if args.traffic is not None else recorded_traffic(f"key_merge/{args.rows}/{dist.world}")
    roof.update({"frac": roof["achieved"] / roof["peak"], "traffic": traffic,
                 "kernel": "whole merge step (partition + shuffle + join kernels)",
                 "algorithmic_bytes_per_step": alg, "t_roof_ms": max(t_hbm, t_nvl) * 1e3, "phases": phase,
                 "trace_ms": trace})
    # Per kernel group, CUDA events on the merge stream inside the timed steps (rank 0).
    # join: reads both partitioned tables once, writes the output once.  partition (N=1):
    # two passes per side, each reading and writing 16 B per row (the algorithm's own
    # bytes; the strict step roofline above counts only the inputs once).
    rows_in = km.received if dist.world > 1 else [km.n, km.n]
    join_bytes = 16 * sum(rows_in) + 24 * digest_rows(km)
    groups = {"join": {"ms": kern["join"], "bytes": join_bytes, "bound": "hbm", "peak": hbm_peak}}
    if dist.world == 1:
        groups["partition"] = {"ms": kern["partition"], "bytes": 2 * 2 * 32 * km.n + 2 * 8 * km.n, "bound": "hbm",
                               "peak": hbm_peak, "note": "per side: full-id histogram (8 B/row) + 2 passes x 32 B/row"}
    else:
        groups["partition_and_shuffle"] = {
            "ms": kern["partition"], "bytes": alg["nvlink"], "bound": "nvlink", "peak": NVLINK_PEER_GBS,
            "note": "plan + push scatter of both sides, exchange, receiver split: NVLink bytes / time"}
    for g in groups.values():
        g["GBps"] = g["bytes"] / (g["ms"] * 1e-3) / 1e9 if g["ms"] else None
        g["frac"] = g["GBps"] / g["peak"] if g["GBps"] else None
    roof["kernel_groups"] = groups

    e2e = None
    if not args.skip_e2e:
        cols = [km.inputs[0].keys, km.inputs[0].vals, km.inputs[1].keys, km.inputs[1].vals]
        nbytes = km.n * 8
        host = [native.PinnedHostBuffer(max(1, nbytes)) for _ in cols]
        for h, c in zip(host, cols):
            native.memcpy(h.ptr, c.ptr, nbytes, stream)
        stream.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(max(1, min(args.steps, 3))):
            for h, c in zip(host, cols):
                native.memcpy(c.ptr, h.ptr, nbytes, stream)
            r = loop.run_until_complete(km.run_global())
        e2e_ms = dist.max((time.perf_counter() - t0) * 1e3 / max(1, min(args.steps, 3)))
        if r != digest:
            raise RuntimeError("e2e merge digest differs")
        e2e = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": int(dist.sum(4 * nbytes)),
               "d2h_bytes_per_step": int(dist.sum(32 + 8 * (2 * dist.world + 2)))}

    km.close()
    dist.barrier()  # every rank unmapped its peers' receive buffers before any rank frees its own
    cpu, parity = None, None
    if dist.rank == 0:
        # parity at FULL size: the oracle's digest of the same global inputs
        target = args.rows * dist.world
        c = km_cpu_sample(target, 0.0 if args.skip_cpu else min(10.0, args.cpu_seconds), args.fraction)
        parity = {"rows_per_side": target, "digest_equal": tuple(digest) == c["digest"],
                  "oracle_digest": list(c["digest"]), "rows_out": digest[0], "expected_fraction": args.fraction,
                  "observed_fraction": digest[0] / max(1, target), "row_conservation": dist.world == 1 or km.conserved}
        if not parity["digest_equal"]:
            raise RuntimeError(f"key_merge digest {digest} differs from the oracle's {c['digest']}")
        if not args.skip_cpu:
            cpu = {"value": c["ms"], "unit": "ms", "cores": c["threads"], "kind": "port",
                   "sample": f"oracle C join ({c['threads']} threads, radix partition + per-partition hash joins) "
                             f"of the full {target} resident rows/side x {c['runs']} runs in {c['seconds']:.1f} s"}
    if dist.rank != 0:
        return None
    return {
        "metric": f"merge wall time ({args.rows} rows/side/GPU, int64 key, fraction {args.fraction})",
        "value": step_ms, "unit": "ms", "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "int64", "data": "synthetic (splitmix64 generator, BASELINE.md §3)",
        "config": km_config(args), "partitions": km.parts, "digest": list(digest),
        "gpu_launches": launches, "roofline": roof, "e2e": e2e, "cpu_baseline": cpu, "parity": parity,
        "clocks": clocks, "wall_ms_per_step": wall,
    }


# -- p2p ---------------------------------------------------------------------------------------------


def _l2_note(nbytes: float, what: str) -> str:
    if nbytes > 8 * 126e6:
        return f"{what} ({nbytes / 1e9:.1f} GB) far larger than the 126 MB L2; no flush needed"
    return f"{what} ({nbytes / 1e6:.0f} MB) not flushed between steps (small case)"


def ts_config(n: int, b: int, world: int) -> dict:
    """The transpose_sum workload as both arms name it (identical dicts)."""
    return {"workload": "transpose_sum", "dims": n, "block": b, "workers": world,
            "ownership": "round-robin row-major (SPEC.md:447)", "l2": _l2_note(2 * n * n * 8, "inputs x+y")}


def km_config(args) -> dict:
    """The key_merge workload as both arms name it (identical dicts)."""
    return {"workload": "key_merge", "rows_per_side_per_gpu": args.rows, "fraction": args.fraction,
            "l2": _l2_note(2 * args.rows * 16, "inputs per GPU")}


def p2p_config(args) -> dict:
    return {"workload": "p2p", "sizes": f"1 B - {args.max_size} B, x4 steps", "window": 64}


def bench_p2p_brief(args, dist: Dist) -> dict | None:
    """p2p sub-record of the default line at N >= 2 (the p2p half of BASELINE.json's
    metric, so it reaches the driver's multi-GPU records): ranks 0 and 1 over the
    transport, device frames, osu_bw at 4 / 16 MiB (window 64, distinct buffers) and
    1 B latency (the eager device protocol, rendezvous, host frames).  The full sweep
    and the reference socket stack: --workload p2p."""
    from paper_2101_08878_b200.harness import p2p

    t = open_transport(dist, dist.device)  # every rank (already open after key_merge)
    out = None
    if dist.rank < 2:
        peer = 1 - dist.rank
        bw = {}
        for n in (4 << 20, 16 << 20):
            p2p.verify_once(t, peer, n, True)
            bw[n] = p2p.osu_bw(t, peer, n, 64, 4, True)
        eager = p2p.osu_latency(t, peer, 1, 1000, True, eager=True) if getattr(t, "eager_device_max", 0) else None
        rdv = p2p.osu_latency(t, peer, 1, 1000, True)
        host = p2p.osu_latency(t, peer, 1, 2000, False)
        out = {"metric": "p2p GB/s (osu_bw, >= 4 MiB)", "value": max(bw.values()), "unit": "GB/s",
               "osu_bw_GBps": {"4MiB": bw[4 << 20], "16MiB": bw[16 << 20]},
               "latency_1B_us": {"device_eager": eager, "device_rendezvous": rdv, "host": host},
               "ranks": "0 <-> 1", "frames": "device, distinct buffers per message, verified once per size"}
    dist.barrier()
    return out if dist.rank == 0 else None


def bench_p2p(args, dist: Dist, peaks: dict) -> dict | None:
    from paper_2101_08878_b200.harness import p2p

    if dist.world != 2:
        raise SystemExit("--workload p2p needs exactly 2 ranks (torchrun --nproc-per-node 2)")
    device = dist.device
    t = open_transport(dist, device)
    rows, n = [], 1
    while n <= args.max_size:
        p2p.verify_once(t, 1 - dist.rank, n, True)
        lat = p2p.osu_latency(t, 1 - dist.rank, n, 1000 if n <= 65536 else 100, True)
        bw = p2p.osu_bw(t, 1 - dist.rank, n, 64, 10 if n <= (1 << 20) else 4, True)
        rows.append({"size": n, "osu_latency_us": lat, "osu_bw_GBps": bw})
        n *= 4
    # the same 4 MiB window posted with one vectored call (m4d_transport_post_many)
    vec_4m = p2p.osu_bw(t, 1 - dist.rank, 4 << 20, 64, 4, True, vectored=True) if args.max_size >= (4 << 20) else None
    # the public comm path (send_payload / recv_payload, Listing 2/3) with device frames
    pp = {sz: p2p.pingpong(t, 1 - dist.rank, sz, 1000 if sz < (1 << 20) else 50, True)
          for sz in sorted({1, min(4 << 20, args.max_size), args.max_size})}
    # the eager device protocol at the transport layer (eager send + loaned receive)
    eager_lat = {sz: p2p.osu_latency(t, 1 - dist.rank, sz, 1000, True, eager=True)
                 for sz in (1, 4096, 65536)} if getattr(t, "eager_device_max", 0) else {}
    # host frames (Dask control messages; the reference arm's frames): transport and comm path at 1 B
    host_lat = p2p.osu_latency(t, 1 - dist.rank, 1, 2000, False)
    host_pp = p2p.pingpong(t, 1 - dist.rank, 1, 2000, False)
    # SM pull kernels this rank launched (device frames >= 64 KiB; smaller ones ride the copy engine)
    launches = t.native_stats()["pull_kernel_launches"]
    cpu = None
    if dist.rank == 0 and not args.skip_cpu:
        sample = SimpleNamespace(**{**vars(args), "max_size": 4 << 20})
        ref = run_ref_workers("p2p", 2, sample, rounds=1, warmup=0)
        if "value" in ref:
            cpu = {"value": ref["value"], "unit": "GB/s", "cores": 2, "kind": "reference",
                   "sample": ref["sample"] + ", sizes 1 B - 4 MiB", "latency_1B_us": ref["latency_1B_us"]}
    dist.barrier()
    if dist.rank != 0:
        return None
    big = [r for r in rows if r["size"] >= (4 << 20)]  # north_star: >= 4 MB messages
    best = max(big, key=lambda r: r["osu_bw_GBps"]) if big else rows[-1]
    top = pp[args.max_size]
    return {
        "metric": "p2p GB/s (osu_bw, >= 4 MiB)", "value": best["osu_bw_GBps"], "unit": "GB/s",
        "n_gpus": 2, "steps": 1, "warmup": 1, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic byte pattern, verified once per size",
        "config": p2p_config(args), "frames": "device (cuda:0 <-> cuda:1)",
        # 1 B device frame, transport layer: the protocol the transport picks for that size
        # (eager when the ring exists), the rendezvous figure beside it
        "latency_1B_us": eager_lat.get(1, rows[0]["osu_latency_us"]),
        "latency_1B_protocol": "eager" if 1 in eager_lat else "rendezvous",
        "osu_bw_4MiB_vectored_GBps": vec_4m,
        "osu_bw_note": "windows posted message by message (the OSU loop); osu_bw_4MiB_vectored_GBps: the "
                       "same 4 MiB window posted with one m4d_transport_post_many call",
        "rendezvous_latency_1B_us": rows[0]["osu_latency_us"], "sweep": rows,
        "device_eager_latency_us": {str(k): v for k, v in eager_lat.items()},
        "host_frames_1B": {"osu_latency_us": host_lat,
                           "comm_path_latency_us": host_pp["mean_s"] * 1e6 if host_pp else None},
        "comm_path": {str(k): {"latency_us": v["mean_s"] * 1e6, "GBps": v["throughput_Bps"] / 1e9}
                      for k, v in pp.items() if v},
        "gpu_launches": launches,
        "gpu_launches_note": "rank 0's rendezvous pull kernels over the whole sweep (no separate timed region)",
        "e2e": {"value": top["throughput_Bps"] / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0,
                "note": f"send_payload/recv_payload ping-pong of {args.max_size}-byte device frames (2*size/RTT)"},
        "cpu_baseline": cpu,
        "roofline": {"bound": "nvlink", "achieved": best["osu_bw_GBps"], "peak": 770.0, "unit": "GB/s",
                     "frac": best["osu_bw_GBps"] / 770.0, "traffic": None,
                     "peak_source": "measured peer copy per direction (B200_PROFILING.md)",
                     "frac_of_nominal_900": best["osu_bw_GBps"] / 900.0,
                     "by_size_GBps": {str(r["size"]): r["osu_bw_GBps"] for r in big}},
    }


# -- small-frame storm ---------------------------------------------


def storm_line(r, args, world: int) -> dict:
    return {
        "metric": f"small-frame storm throughput ({args.frames} frames of 1 B-8 KiB, {args.conns} endpoints "
                  f"per ordered worker pair)",
        "value": r.frames_per_s, "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": r.wall_s / max(1, args.steps) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (log-uniform sizes, seed 0x5EED; payload checked)",
        "config": {"workload": "storm", "frames": args.frames, "conns": args.conns, "workers": world,
                   "max_frame": 8192},
        "latency_us": {"p50": r.p50_us, "p99": r.p99_us, "max": r.max_us}, "verified_frames": r.verified,
    }


def bench_storm(args, dist: Dist, peaks: dict) -> dict | None:
    from paper_2101_08878_b200.harness import storm

    if dist.world < 2:
        raise SystemExit("--workload storm needs >= 2 ranks (torchrun --nproc-per-node N)")
    # device frames: a round's received frames hold their device-ring slots until dropped
    os.environ.setdefault("M4D_EAGER_DEVICE_RING", str(64 << 20))
    t = open_transport(dist, dist.device)
    sampler = ClockSampler(dist.device)
    sampler.start()
    ns = storm.namespace_of("paper_2101_08878_b200")
    r = storm.run_worker(ns, t, dist.allgather_bytes, conns=args.conns, total=args.frames, rounds=args.steps,
                         warmup=args.warmup)
    # the same storm with device frames (cuda:rank -> cuda:peer by the eager device protocol)
    before = t.native_stats()
    rd = storm.run_worker(ns, t, dist.allgather_bytes, conns=args.conns, total=args.frames, rounds=args.steps,
                          warmup=args.warmup, device=dist.device)
    after = t.native_stats()
    clocks = sampler.stop()
    if dist.rank != 0:
        return None
    line = storm_line(r, args, dist.world)
    dev_line = storm_line(rd, args, dist.world)
    line.update({
        "device_frames": {
            "value": rd.frames_per_s, "unit": "frames/s", "ms_per_step": dev_line["ms_per_step"],
            "latency_us": dev_line["latency_us"], "verified_frames": rd.verified,
            "eager_device_sends_rank0": after["eager_device_sends"] - before["eager_device_sends"],
            "proxy_copies_rank0": after["eager_proxy_copies"] - before["eager_proxy_copies"],
            "note": "the same frames as device frames: sender proxy kernel copies each into the receiver's "
                    "device ring over NVLink, the receiver reads it by loan (no host staging)"},
        "gpu_launches": 0,
        "note": "host frames through the nvlink transport's shared-memory rings (eager path); no kernels",
        "roofline": None,
        "e2e": {"value": r.frames_per_s, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "note": "host frames through Endpoint.write/read: end to end by construction"},
        "clocks": clocks,
    })
    if not args.skip_cpu:
        ref = run_ref_workers("storm", dist.world, args, rounds=1, warmup=0)
        if "value" in ref:
            line["cpu_baseline"] = {"value": ref["value"], "unit": "frames/s", "cores": dist.world,
                                    "kind": "reference", "sample": ref.get("sample", "")}
    return line


# -- reference arms over the reference's own SocketTransport (baseline/_ref) --------------------

REF_DIR = os.path.join(HERE, "baseline", "_ref")


def _free_ports(n: int) -> list[int]:
    import socket

    socks, ports = [], []
    for _ in range(n):
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        socks.append(s)
        ports.append(s.getsockname()[1])
    for s in socks:
        s.close()
    return ports


def run_ref_workers(kind: str, world: int, args, rounds: int, warmup: int, timeout: float = 900.0) -> dict:
    """Spawn ``world`` reference worker processes (baseline/_ref commshim, SocketTransport on
    127.0.0.1) and return rank 0's JSON summary."""
    if not os.path.isdir(os.path.join(REF_DIR, "commshim")):
        return {"unavailable": "baseline/_ref (the installed reference package) is missing"}
    ports = ",".join(map(str, _free_ports(world)))
    cmd = [sys.executable, os.path.abspath(__file__), "--ref-worker", kind, "--ref-world", str(world),
           "--ref-ports", ports, "--frames", str(args.frames), "--conns", str(args.conns),
           "--max-size", str(args.max_size), "--steps", str(rounds), "--warmup", str(warmup)]
    procs = [subprocess.Popen(cmd + ["--ref-rank", str(r)], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True) for r in range(world)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=timeout))
        except subprocess.TimeoutExpired:
            p.kill()
            outs.append(p.communicate())
    if any(p.returncode for p in procs):
        bad = next((o[1] for p, o in zip(procs, outs) if p.returncode), "")
        return {"unavailable": "reference workers failed: " + bad.strip().splitlines()[-1][:200] if bad.strip()
                else "reference workers failed"}
    return json.loads(outs[0][0].strip().splitlines()[-1])


def ref_worker_main(args) -> int:
    """One reference worker: the UNMODIFIED reference package over its SocketTransport."""
    sys.path.insert(0, REF_DIR)
    import commshim  # noqa: F401  (must resolve to baseline/_ref, not this repo's alias)

    if not os.path.abspath(commshim.__file__).startswith(os.path.abspath(REF_DIR)):
        raise SystemExit(f"reference import resolved to {commshim.__file__}")
    from commshim.transport import TransportConfig, transport_init
    from paper_2101_08878_b200.harness import p2p, storm

    ports = [int(p) for p in args.ref_ports.split(",")]
    rank, world = args.ref_rank, args.ref_world
    t = transport_init(world, rank, TransportConfig(kind="socket", connect_timeout=60.0,
                                                    rank_map={r: ("127.0.0.1", p) for r, p in enumerate(ports)}))
    t.wait_ready(60.0)
    ns = storm.namespace_of("commshim")
    if args.ref_worker == "storm":
        r = storm.run_worker(ns, t, storm.transport_sync(t), conns=args.conns, total=args.frames,
                             rounds=args.steps, warmup=args.warmup)
        out = {"value": r.frames_per_s, "wall_s": r.wall_s, "p50_us": r.p50_us, "p99_us": r.p99_us,
               "verified": r.verified,
               "sample": f"reference SocketTransport + Endpoint, {world} processes, {args.steps} round(s) of "
                         f"{args.frames} frames"}
    else:  # p2p: the same raw-post osu tests and comm-path ping-pong, host frames over sockets
        rows, n = [], 1
        while n <= args.max_size:
            p2p.verify_once(t, 1 - rank, n, False)
            lat_iters = max(3, min(1000, (64 << 20) // max(n, 1)))
            window = max(1, min(64, (64 << 20) // n))
            lat = p2p.osu_latency(t, 1 - rank, n, lat_iters, False)
            bw = p2p.osu_bw(t, 1 - rank, n, window, 2 if n >= (1 << 20) else 10, False)
            rows.append({"size": n, "osu_latency_us": lat, "osu_bw_GBps": bw, "window": window})
            n *= 4
        pp = {sz: p2p.pingpong(t, 1 - rank, sz, 200 if sz < (1 << 20) else 10, False, ns=ns)
              for sz in sorted({1, min(4 << 20, args.max_size), args.max_size})}
        big = [r for r in rows if r["size"] >= (4 << 20)] or rows[-1:]
        out = {"value": max(r["osu_bw_GBps"] for r in big), "latency_1B_us": rows[0]["osu_latency_us"],
               "sweep": rows,
               "comm_path": {str(k): {"latency_us": v["mean_s"] * 1e6, "GBps": v["throughput_Bps"] / 1e9}
                             for k, v in pp.items() if v},
               "sample": "reference SocketTransport, 2 processes, host frames; osu_bw window <= 64 MiB in flight"}
    storm.transport_sync(t, tag=960)(b"done")  # no rank closes while a peer still drains its last frames
    t.close()
    if rank == 0:
        print(json.dumps(out), flush=True)
    return 0


def reference_storm(args) -> dict:
    world = max(2, int(os.environ.get("WORLD_SIZE", str(args.gpus))))
    ref = run_ref_workers("storm", world, args, rounds=args.steps, warmup=min(args.warmup, 1))
    if "value" not in ref:
        return {"impl": "reference", **ref}
    line = storm_line(SimpleNamespace(frames_per_s=ref["value"], wall_s=ref["wall_s"], p50_us=ref["p50_us"],
                                      p99_us=ref["p99_us"], max_us=ref["p99_us"], verified=ref["verified"]),
                      args, world)
    line.pop("latency_us")
    line.update({"impl": "reference", "latency_us": {"p50": ref["p50_us"], "p99": ref["p99_us"]},
                 "cpu_baseline": {"value": ref["value"], "unit": "frames/s", "cores": world, "kind": "reference",
                                  "sample": ref["sample"]},
                 "e2e": {"value": ref["value"], "unit": "frames/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0}})
    return line


def reference_p2p(args) -> dict:
    ref = run_ref_workers("p2p", 2, args, rounds=1, warmup=0)
    if "value" not in ref:
        return {"impl": "reference", **ref}
    return {
        "impl": "reference", "metric": "p2p GB/s (osu_bw, >= 4 MiB)", "value": ref["value"], "unit": "GB/s",
        "n_gpus": 2, "steps": 1, "warmup": 1, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic byte pattern, verified once per size",
        "config": p2p_config(args), "frames": "host (reference SocketTransport)",
        "latency_1B_us": ref["latency_1B_us"], "sweep": ref["sweep"], "comm_path": ref["comm_path"],
        "cpu_baseline": {"value": ref["value"], "unit": "GB/s", "cores": 2, "kind": "reference",
                         "sample": ref["sample"]},
        "e2e": {"value": ref["comm_path"][str(args.max_size)]["GBps"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0,
                "note": f"send_payload/recv_payload ping-pong of {args.max_size}-byte host frames (2*size/RTT)"},
    }


def reference_transpose_sum(args) -> dict:
    threads = len(os.sched_getaffinity(0))
    budget = max(2.0, args.cpu_seconds / max(1, args.steps))
    full = ts_cpu_full(args.n, args.block, threads, min_seconds=budget * args.steps)
    value = full["ms"]
    nb = args.n // args.block
    sample = (f"oracle C restatement (the reference has no operator code) over the full array (all {nb * nb} "
              f"blocks, x resident in host RAM), {full['passes']} passes in {full['seconds']:.1f} s")
    import math as _m

    return {
        "impl": "reference",
        "metric": f"x+x.T sum wall time ({args.n}^2 fp64, {args.block}^2 chunks)",
        "value": value,
        "unit": "ms",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": value,
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (splitmix64 generator, BASELINE.md §3)",
        "config": ts_config(args.n, args.block, int(os.environ.get("WORLD_SIZE", "1"))),
        "checksum": _m.fsum(float(v) for v in full["sums"]),
        "cpu_baseline": {"value": value, "unit": "ms", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def reference_key_merge(args) -> dict:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    target = args.rows * world
    per = [km_cpu_sample(target, max(2.0, args.cpu_seconds / max(1, args.steps)), args.fraction)
           for _ in range(args.steps)]
    value = statistics.mean(p["ms"] for p in per)
    threads = per[0]["threads"]
    sample = (f"oracle C join ({threads} threads, radix partition + per-partition hash joins) of the full "
              f"{target} resident rows/side per step")
    return {
        "impl": "reference",
        "metric": f"merge wall time ({args.rows} rows/side/GPU, int64 key, fraction {args.fraction})",
        "value": value, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value, "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (splitmix64 generator, BASELINE.md §3)",
        "config": km_config(args),
        "cpu_baseline": {"value": value, "unit": "ms", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "digest": list(per[0]["digest"]),
    }


# -- main -------------------------------------------------------------------------------------------


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["transpose_sum", "key_merge", "p2p", "storm"], default="transpose_sum")
    ap.add_argument("--frames", type=int, default=100_000, help="storm frames per round")
    ap.add_argument("--conns", type=int, default=8, help="storm endpoints per ordered worker pair")
    ap.add_argument("--ref-worker", choices=["p2p", "storm"], help=argparse.SUPPRESS)
    ap.add_argument("--ref-rank", type=int, default=0, help=argparse.SUPPRESS)
    ap.add_argument("--ref-world", type=int, default=2, help=argparse.SUPPRESS)
    ap.add_argument("--ref-ports", default="", help=argparse.SUPPRESS)
    ap.add_argument("--rows", type=int, default=100_000_000, help="key_merge rows per side per GPU")
    ap.add_argument("--fraction", type=float, default=0.3)
    ap.add_argument("--max-size", type=int, default=64 << 20, help="p2p largest message")
    ap.add_argument("--n", type=int, default=40000)
    ap.add_argument("--block", type=int, default=2000)
    ap.add_argument("--cpu-seconds", type=float, default=30.0, help="CPU-baseline time budget (whole run)")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--no-merge", action="store_true", help="default run without the key_merge sub-record")
    ap.add_argument("--skip-p2p", action="store_true", help="default run at N >= 2 without the p2p sub-record")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch from an ncu --set full capture (reported as roofline.traffic)")
    args = ap.parse_args(argv)
    if args.ref_worker:
        return ref_worker_main(args)
    if args.warmup < 3 and args.impl == "ours":
        print("bench: W >= 3 warm-up steps required; raising to 3", file=sys.stderr)
        args.warmup = 3

    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return 0
        if args.workload == "transpose_sum":
            line = reference_transpose_sum(args)
            if not args.no_merge:
                km = reference_key_merge(args)
                line["key_merge"] = {k: km[k] for k in ("metric", "value", "unit", "ms_per_step", "config",
                                                        "cpu_baseline", "e2e", "digest")}
            emit(line)
        elif args.workload == "key_merge":
            emit(reference_key_merge(args))
        elif args.workload == "storm":
            emit(reference_storm(args))
        else:
            emit(reference_p2p(args))
        return 0

    # Watchdog: a run that hangs (e.g. a rank waiting on a peer that died) dumps every
    # thread's Python stack to stderr and exits instead of sitting until the launcher's
    # timeout (M4D_BENCH_WATCHDOG_S, default 1500 s; 0 disables).
    watchdog = float(os.environ.get("M4D_BENCH_WATCHDOG_S", "1500"))
    if watchdog > 0:
        import faulthandler

        faulthandler.dump_traceback_later(watchdog, exit=True)
    dist = Dist()
    peaks = load_peaks()
    runner = {"transpose_sum": bench_transpose_sum, "key_merge": bench_key_merge, "p2p": bench_p2p,
              "storm": bench_storm}[args.workload]
    try:
        line = runner(args, dist, peaks)
        # The default run carries the other half of BASELINE.json's metric as a sub-record:
        # the merge (config 4) at the same N, with its own timed region, roofline, e2e,
        # CPU baseline and full-size parity.
        if args.workload == "transpose_sum" and not args.no_merge:
            km = bench_key_merge(args, dist, peaks)
            if line is not None and km is not None:
                line["key_merge"] = {k: km[k] for k in ("metric", "value", "unit", "ms_per_step", "higher_is_better",
                                                        "scaling", "dtype", "config", "gpu_launches", "roofline",
                                                        "e2e", "cpu_baseline", "parity", "clocks", "wall_ms_per_step",
                                                        "partitions", "digest")}
            if dist.world >= 2 and not args.skip_p2p:
                p2 = bench_p2p_brief(args, dist)
                if line is not None and p2 is not None:
                    line["p2p"] = p2
    finally:
        if getattr(dist, "transport", None) is not None:
            dist.barrier()
            dist.transport.close()
        dist.close()
    if line is not None:
        if dist.shared:
            line["functional_check_only"] = "more ranks than GPUs: ranks shared GPUs; not a measurement"
        emit(line)
    return 0


if __name__ == "__main__":
    sys.exit(main())
