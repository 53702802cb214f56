"""Operators and device frames across PROCESSES (one process per rank, as bench.py and
torchrun run them), so the CUDA-IPC branches run: transpose_sum maps the peers' x pools
(harness/transpose_sum.py connect_peers), key_merge maps the peers' receive buffers (push)
or pulls device frames (pull), the transport maps device frames.  "same": every rank on
cuda:0 (the driver's one-GPU box); "own": rank r on cuda:r, over NVLink (skipped below
the GPUs needed).  Results must be identical to the oracle and independent of the worker
count and transport."""

import json
import os
import subprocess
import sys
import uuid

import pytest

import oracle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "mp_worker.py")


def launch(mode, world, devmode, timeout=300):
    from paper_2101_08878_b200 import native

    if devmode == "own" and native.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    session = "mp" + uuid.uuid4().hex[:10]
    procs = [subprocess.Popen([sys.executable, WORKER, mode, str(r), str(world), session, devmode],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, cwd=ROOT)
             for r in range(world)]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=timeout)
        except subprocess.TimeoutExpired:
            p.kill()
            out, _ = p.communicate()
        outs.append((p.returncode, out))
    for rc, out in outs:
        assert rc == 0, out[-4000:]
    return [json.loads(next(ln for ln in reversed(out.splitlines()) if ln.startswith('{"rank"'))) for _, out in outs]


@pytest.mark.parametrize("devmode", ["same", "own"])
def test_transpose_sum_across_processes(devmode):
    res = launch("ts", 2, devmode)
    _, want = oracle.transpose_sum_checksum(2048, 256, threads=4)
    assert all(r["ok"] and r["remote_tasks"] > 0 for r in res)
    assert res[0]["checksum"] == res[1]["checksum"]
    assert abs(res[0]["checksum"] - want) <= 1e-12 * abs(want)


@pytest.mark.parametrize("devmode", ["same", "own"])
def test_transpose_sum_reuploaded_inputs_are_fenced(devmode):
    """x changes between steps (two arrays alternated through TransposeSum.load_x): a
    kernel reading a peer's pool before that peer's upload landed would mix arrays."""
    res = launch("ts_fence", 2, devmode)
    assert all(r["fenced_steps"] == 6 for r in res)


@pytest.mark.parametrize("shuffle", ["push", "pull"])
@pytest.mark.parametrize("devmode", ["same", "own"])
def test_key_merge_across_processes(shuffle, devmode):
    res = launch(f"km_{shuffle}", 2, devmode)
    want = list(oracle.key_merge_c(200_000, 2, 0.3))
    assert all(r["digest"] == want for r in res)
    # conservation: every generated row received exactly once
    assert sum(r["received"][0] for r in res) == sum(r["received"][1] for r in res) == 2 * 200_000
    if shuffle == "push":
        assert all(r["mapped_peers"] == 2 for r in res)  # both receive buffers of the peer


def test_key_merge_four_processes_own_gpus():
    res = launch("km_push", 4, "own")
    assert all(r["digest"] == list(oracle.key_merge_c(200_000, 4, 0.3)) for r in res)


@pytest.mark.parametrize("devmode", ["same", "own"])
def test_device_frames_across_processes(devmode):
    res = launch("frames", 2, devmode)
    assert all(r["staged"] == 0 and r["pulls"] > 0 for r in res)


@pytest.mark.parametrize("devmode", ["same", "own"])
def test_freed_device_frames_are_unmapped_before_free(devmode):
    """150 fresh 8 MiB frames (1.2 GB) sent and freed: the sender's device memory stays
    flat because every importer closes its mapping before the deferred cudaFree."""
    res = launch("churn", 2, devmode)
    assert res[0]["leak_mib"] < 64, res


@pytest.mark.parametrize("devmode", ["same", "own"])
def test_torch_tensors_cross_processes_as_device_array_frames(devmode):
    """Dask-style Comm.write of torch tensors (caching-allocator memory, legacy CUDA IPC),
    decoded on the far side as zero-copy CUDA arrays (serializer tag 3)."""
    res = launch("torch", 2, devmode)
    assert res[1]["tensors"] == 5 and all(r["staged"] == 0 for r in res)
