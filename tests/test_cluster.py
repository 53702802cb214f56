"""Mini cluster roles and heartbeat accounting, on the simulated
transport's virtual clock (deterministic) and across processes on the nvlink transport
through ``commshim-launch`` (host frames: runs on CPU)."""

import json
import os
import subprocess
import sys

import pytest

from paper_2101_08878_b200.channels import build_comm_table
from paper_2101_08878_b200.endpoints import Node
from paper_2101_08878_b200.errors import ConfigurationError
from paper_2101_08878_b200.harness.cluster import CLIENT, SCHEDULER, WORKER, Cluster, role_of
from paper_2101_08878_b200.loop import TaskLoop, gather, sleep
from paper_2101_08878_b200.transport import LinkModel, SimFabric

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sim_cluster(n, interval=10):
    loop = TaskLoop()
    # a fast zero-latency link: a beat costs (almost) no virtual time, so the tick
    # arithmetic of SPEC.md:433 holds exactly
    fabric = SimFabric(n, link=LinkModel(bandwidth=1e15), clock=loop.clock)
    nodes = [Node(t, build_comm_table(t)) for t in (fabric.transport(r) for r in range(n))]
    return loop, [Cluster(node, heartbeat_interval=interval) for node in nodes]


def test_roles_follow_the_dask_mpi_convention():
    assert [role_of(r, 4) for r in range(4)] == [SCHEDULER, CLIENT, WORKER, WORKER]
    assert role_of(0, 1) == "solo"
    with pytest.raises(ConfigurationError):
        role_of(0, 2)


def run(loop, cl, run_ticks, *, silent=()):
    async def rank(c):
        role = await c.bootstrap()
        if role.kind == SCHEDULER:
            return role, await c.serve()
        if role.kind == CLIENT:
            await sleep(run_ticks)
            await c.stop_all()
            return role, None
        if c.rank in silent:  # a worker that stops beating after registering (killed)
            return role, None
        return role, await c.heartbeat_loop()

    return loop.run_until_complete(gather(*(rank(c) for c in cl)))


def test_bootstrap_registers_every_worker_and_counts_beats():
    loop, cl = sim_cluster(4, interval=10)
    out = run(loop, cl, 100)
    roles = [r for r, _ in out]
    assert [r.kind for r in roles] == [SCHEDULER, CLIENT, WORKER, WORKER]
    assert all(r.workers == [2, 3] for r in roles)
    report = out[0][1]
    assert all(report.beats[w] >= 9 for w in (2, 3)), report  # >= 9 beats in 100 ticks
    assert report.suspects == [] and report.closed == []


def test_three_ranks_have_one_worker():
    loop, cl = sim_cluster(3)
    out = run(loop, cl, 50)
    assert out[0][0].workers == [2]


def test_silent_worker_is_reported_suspect_after_three_intervals():
    loop, cl = sim_cluster(4, interval=10)

    async def main():
        async def rank(c):
            role = await c.bootstrap()
            if role.kind == SCHEDULER:
                await sleep(100)
                return c.report()
            if role.kind == WORKER and c.rank == 3:
                return None  # registered, never beats
            if role.kind == WORKER:
                for seq in range(10):  # beats for 100 ticks
                    from paper_2101_08878_b200.harness.cluster import _msg

                    await c._ep.write(_msg("beat", c.rank, seq))
                    await sleep(10)
            return None

        return await gather(*(rank(c) for c in cl))

    report = loop.run_until_complete(main())[0]
    suspects = [r for _, r in report.suspects]
    assert suspects == [3], report
    when = report.suspects[0][0]
    assert 30 < when <= 50  # flagged once more than 3 intervals passed without a beat
    assert report.beats[2] >= 9


PROGRAM = os.path.join(ROOT, "tests", "cluster_program.py")


@pytest.mark.parametrize("transport", ["nvlink", "socket"])
def test_launcher_runs_a_four_process_cluster(transport):
    """commshim-launch spawns 4 processes (scheduler, client, 2 workers); heartbeats over
    the nvlink transport's shared-memory rings (or the socket transport) for 0.5 s, no
    suspects."""
    out = subprocess.run([sys.executable, "-m", "paper_2101_08878_b200.cli", "launch", "--np", "4",
                          "--transport", transport, "--", sys.executable, PROGRAM, "0.02", "0.5"],
                         cwd=ROOT, capture_output=True, text=True, timeout=180)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    report = json.loads(next(ln for ln in out.stdout.splitlines() if ln.startswith("{")))
    assert report["workers"] == [2, 3]
    assert all(b >= 10 for b in report["beats"].values()), report
    assert report["suspects"] == []


def test_launcher_reports_a_failing_rank():
    out = subprocess.run([sys.executable, "-m", "paper_2101_08878_b200.cli", "launch", "--np", "2", "--",
                          sys.executable, "-c", "import os, sys; sys.exit(3 if os.environ['RANK'] == '1' else 0)"],
                         cwd=ROOT, capture_output=True, text=True, timeout=60)
    assert out.returncode == 3
