"""Small-frame storm: many endpoints per worker pair,
log-uniform 1 B - 8 KiB frames, every payload checked bit-exactly.

The same harness drives this package (nvlink transport, host frames through
the shared-memory rings) and the reference package (socket transport), so the
two frameworks deliver the identical frame multiset."""

import os
import subprocess
import sys
import textwrap

import pytest

from nvlink_fixtures import close_all, new_session, nvlink_transports
from paper_2101_08878_b200.harness import storm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def test_frame_sizes_are_log_uniform_and_seeded():
    sizes = storm.frame_sizes(20000)
    assert sizes == storm.frame_sizes(20000)
    assert min(sizes) == 1 and max(sizes) <= storm.MAX_FRAME
    small = sum(s < 91 for s in sizes) / len(sizes)  # log2(91) ~ 6.5 = half of 13 bits
    assert 0.45 < small < 0.55


def test_streams_cover_every_ordered_pair_with_distinct_generations():
    ss = storm.streams(4, 8)
    assert len(ss) == 4 * 3 * 8
    for lo in range(4):
        for hi in range(lo + 1, 4):
            gens = [storm.generation(s, d, c) for s, d, c in ss if {s, d} == {lo, hi}]
            assert len(gens) == len(set(gens)) == 16
    plan = storm.assign(1000, 4, 8)
    assert sorted(k for ids in plan.values() for k in ids) == list(range(1000))


def test_storm_in_process_nvlink_host_frames():
    ts = nvlink_transports(3)
    try:
        r = storm.run_local(storm.namespace_of("paper_2101_08878_b200"), ts, conns=4, total=3000, rounds=2)
    finally:
        close_all(ts)
    assert r.frames == 6000 and r.verified == 3000
    assert r.frames_per_s > 0 and r.p50_us <= r.p99_us <= r.max_us


@pytest.mark.gpu
def test_storm_in_process_device_frames():
    """Device frames on cuda:0 (eager device protocol: proxy copies, loaned receives)."""
    ts = nvlink_transports(3, 0)
    try:
        r = storm.run_local(storm.namespace_of("paper_2101_08878_b200"), ts, conns=4, total=3000, rounds=2,
                            device=0)
        st = [t.native_stats() for t in ts]
    finally:
        close_all(ts)
    assert r.frames == 6000 and r.verified == 3000
    assert sum(x["eager_device_sends"] for x in st) == 6000
    assert sum(x["eager_device_loans"] for x in st) == 6000


DEVICE_WORKER = textwrap.dedent('''
    import os, sys
    sys.path.insert(0, sys.argv[1])
    from paper_2101_08878_b200 import native
    from paper_2101_08878_b200.harness import storm
    from paper_2101_08878_b200.transport import TransportConfig, transport_init
    rank, world, session = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    dev = rank % native.device_count()
    t = transport_init(world, rank, TransportConfig(kind="nvlink", session=session, device=dev, connect_timeout=60))
    t.wait_ready(60)
    r = storm.run_worker(storm.namespace_of("paper_2101_08878_b200"), t, storm.transport_sync(t),
                         conns=4, total=4000, rounds=2, warmup=1, device=dev)
    st = t.native_stats()
    print("RESULT", r.frames, r.verified, st["eager_device_sends"], st["eager_proxy_copies"])
    t.close()
''')


@pytest.mark.gpu
def test_storm_processes_device_frames():
    """Three processes (one per GPU when there are enough, else sharing cuda:0): device
    frames cross processes through CUDA-IPC mapped device rings."""
    session = new_session()
    procs = [subprocess.Popen([sys.executable, "-c", DEVICE_WORKER, ROOT, str(r), "3", session],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(3)]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            p.kill()
            out, _ = p.communicate()
        outs.append((p.returncode, out))
    sent = 0
    for rc, out in outs:
        assert rc == 0, out[-3000:]
        line = [l for l in out.splitlines() if l.startswith("RESULT")][0].split()
        assert int(line[1]) == 8000 and int(line[2]) == 4000
        assert int(line[3]) == int(line[4])  # every eager device send went through the proxy
        sent += int(line[3])
    assert sent == 3 * 4000  # three rounds (one warm-up) of 4000 frames, all eager


WORKER = textwrap.dedent('''
    import sys
    sys.path.insert(0, sys.argv[1])
    from paper_2101_08878_b200.harness import storm
    from paper_2101_08878_b200.transport import TransportConfig, transport_init
    rank, world, session = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    t = transport_init(world, rank, TransportConfig(kind="nvlink", session=session, device=-1, connect_timeout=30))
    t.wait_ready()
    r = storm.run_worker(storm.namespace_of("paper_2101_08878_b200"), t, storm.transport_sync(t),
                         conns=4, total=4000, rounds=2, warmup=1)
    print("RESULT", r.frames, r.verified, r.frames_per_s)
    t.close()
''')


def test_storm_three_processes_nvlink_host_frames():
    session = new_session()
    procs = [subprocess.Popen([sys.executable, "-c", WORKER, ROOT, str(r), "3", session],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(3)]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            p.kill()
            out, _ = p.communicate()
        outs.append((p.returncode, out))
    for rc, out in outs:
        assert rc == 0, out[-3000:]
        line = [l for l in out.splitlines() if l.startswith("RESULT")][0].split()
        assert int(line[1]) == 8000 and int(line[2]) == 4000


REF_SCRIPT = textwrap.dedent('''
    import sys, time, socket
    sys.path.insert(0, sys.argv[1]); sys.path.insert(1, sys.argv[2])
    import commshim
    assert commshim.__file__.startswith(sys.argv[1]), commshim.__file__
    from commshim.transport.tcp import SocketTransport
    from paper_2101_08878_b200.harness import storm
    def free_port():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0)); return s.getsockname()[1]
    rm = {r: ("127.0.0.1", free_port()) for r in range(3)}
    ts = [SocketTransport(3, r, rm, connect_timeout=5.0) for r in range(3)]
    for _ in range(20000):
        if all(t.mesh_ready for t in ts): break
        for t in ts: t.progress()
        time.sleep(0.0005)
    r = storm.run_local(storm.namespace_of("commshim"), ts, conns=4, total=3000)
    print("RESULT", r.frames, r.verified, r.bytes)
    for t in ts: t.close()
''')


def test_reference_package_runs_the_same_storm():
    if not os.path.isdir(os.path.join(REF, "commshim")):
        import pytest
        pytest.skip("baseline/_ref not installed")
    out = subprocess.run([sys.executable, "-c", REF_SCRIPT, REF, ROOT], capture_output=True, text=True, timeout=240)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")][0].split()
    assert int(line[1]) == 3000 and int(line[2]) == 3000
    assert int(line[3]) == sum(storm.frame_sizes(3000))
