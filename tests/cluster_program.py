"""A program for commshim-launch (test infrastructure): one rank of the mini cluster on the
transport the launcher configured; workers heartbeat until the client (after RUN seconds)
stops them; the scheduler prints the heartbeat report as JSON.

    commshim-launch --np 4 -- python tests/cluster_program.py INTERVAL RUN
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2101_08878_b200.channels import build_comm_table  # noqa: E402
from paper_2101_08878_b200.cli import transport_from_env  # noqa: E402
from paper_2101_08878_b200.endpoints import Node  # noqa: E402
from paper_2101_08878_b200.harness.cluster import CLIENT, SCHEDULER, Cluster  # noqa: E402
from paper_2101_08878_b200.harness.collectives import barrier_sync  # noqa: E402
from paper_2101_08878_b200.loop import MonotonicClock, TaskLoop, sleep  # noqa: E402


def main() -> int:
    interval, run_s = float(sys.argv[1]), float(sys.argv[2])
    t = transport_from_env()
    c = Cluster(Node(t, build_comm_table(t)), heartbeat_interval=interval)
    loop = TaskLoop(MonotonicClock())

    async def body():
        role = await c.bootstrap()
        if role.kind == SCHEDULER:
            return role, await c.serve()
        if role.kind == CLIENT:
            await sleep(run_s)
            await c.stop_all()
            return role, None
        return role, await c.heartbeat_loop()

    role, result = loop.run_until_complete(body())
    barrier_sync(t, 970)  # nobody leaves while a peer still reads its last frames
    if role.kind == SCHEDULER:
        print(json.dumps({"workers": role.workers, "beats": result.beats, "suspects": result.suspects,
                          "closed": result.closed}), flush=True)
    t.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
