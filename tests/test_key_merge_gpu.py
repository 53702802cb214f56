"""key_merge parity on a B200: GPU digest (row count, sum of row hashes, sum of keys)
and the row multiset vs the CPU oracle; worker-count independence."""

import ctypes

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def run_world(rows_per_rank, world, fraction, parts=None, shuffle=None, steps=1, hook=None):
    from paper_2101_08878_b200.harness.key_merge import KeyMerge
    from paper_2101_08878_b200.loop import MonotonicClock, TaskLoop, gather

    from nvlink_fixtures import close_all, nvlink_transports

    ts = nvlink_transports(world, 0) if world > 1 else [None]
    ranks = [KeyMerge(rows_per_rank, fraction, rank=r, world=world, device=0, transport=ts[r], parts=parts,
                      shuffle=shuffle) for r in range(world)]
    if hook:
        hook(ranks)
    for km in ranks:
        km.generate()
    loop = TaskLoop(MonotonicClock())

    async def main():
        return await gather(*(km.run_global() for km in ranks))

    try:
        for _ in range(steps):
            results = loop.run_until_complete(main())
            assert all(r == results[0] for r in results)
    finally:
        for km in ranks:
            km.close()
        if world > 1:
            close_all(ts)
    assert all(r == results[0] for r in results)
    return ranks, results[0]


@pytest.mark.parametrize("rows,fraction", [(100_000, 0.3), (100_000, 0.0), (100_000, 1.0), (1, 0.3), (0, 0.3),
                                           (250_000, 0.5)])
def test_single_gpu_digest_matches_oracle(rows, fraction):
    _, got = run_world(rows, 1, fraction)
    assert got == oracle.key_merge_c(rows, 1, fraction)


def test_rows_match_pandas_multiset():
    ranks, got = run_world(20_000, 1, 0.3, parts=64)
    k, l, r = ranks[0].output_rows()
    want = oracle.key_merge_pandas(20_000, 1, 0.3)
    assert oracle.join_digest_np(k, l, r) == want == got
    # and the exact multiset against the C oracle's materialised rows
    lk, lv = oracle.gen_side_c(0, 20_000, 20_000, oracle.SEED_LEFT, 0)
    rk, rv = oracle.gen_side_c(0, 20_000, 20_000, oracle.SEED_RIGHT, oracle.merge_band(20_000, 0.3))
    _, (ok, ol, orr) = oracle.hash_join_c(lk, lv, rk, rv, want_rows=True)
    assert sorted(zip(k.tolist(), l.tolist(), r.tolist())) == sorted(zip(ok.tolist(), ol.tolist(), orr.tolist()))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_worker_count_independent_and_equal_to_oracle(world):
    rows = 40_000
    _, got = run_world(rows, world, 0.3)
    assert got == oracle.key_merge_c(rows, world, 0.3)
    _, one = run_world(rows * world, 1, 0.3)
    assert one == got


def test_skewed_partitions_use_multiple_build_chunks():
    """Few partitions -> partitions far above the 12288-row table chunk: still exact."""
    _, got = run_world(300_000, 1, 0.3, parts=4)
    assert got == oracle.key_merge_c(300_000, 1, 0.3)


def test_duplicate_heavy_keys():
    """Many duplicates per key (tiny key space): multimap semantics and output regrowth."""
    from paper_2101_08878_b200 import native
    from paper_2101_08878_b200.harness.key_merge import KeyMerge
    from paper_2101_08878_b200.loop import MonotonicClock, TaskLoop

    n = 50_000
    km = KeyMerge(n, 0.3, device=0)
    rng = np.random.default_rng(9)
    lk = rng.integers(0, 50, n).astype(np.int64)
    rk = rng.integers(25, 75, n).astype(np.int64)
    lv = np.arange(n, dtype=np.int64)
    rv = np.arange(n, dtype=np.int64) + 10**9
    for cols, k, v in ((km.inputs[0], lk, lv), (km.inputs[1], rk, rv)):
        native.memcpy(cols.keys.ptr, k.ctypes.data, n * 8)
        native.memcpy(cols.vals.ptr, v.ctypes.data, n * 8)
    native.check(native.lib().m4d_device_sync(0))
    got = TaskLoop(MonotonicClock()).run_until_complete(km.run())
    want = oracle.hash_join_c(lk, lv, rk, rv)
    assert got == want and got[0] > km.n  # the output buffer had to grow


def test_large_config_properties():
    """1e7 rows/side on one GPU: count near f*n, digest equal to the oracle."""
    rows = 10_000_000
    ranks, got = run_world(rows, 1, 0.3)
    assert abs(got[0] / rows - 0.3) < 0.005
    assert got == oracle.key_merge_c(rows, 1, 0.3)
    assert ranks[0].received == [rows, rows]


def test_full_scale_digest_against_the_oracle():
    """5e7 rows/side on one GPU: the digest equals the multithreaded C oracle's at full
    size (the bench checks 1e8 the same way)."""
    import os

    rows = 50_000_000
    _, got = run_world(rows, 1, 0.3)
    band = oracle.merge_band(rows, 0.3)
    lk, lv = oracle.gen_side_c(0, rows, rows, oracle.SEED_LEFT, 0)
    rk, rv = oracle.gen_side_c(0, rows, rows, oracle.SEED_RIGHT, band)
    assert got == oracle.join_mt_c(lk, lv, rk, rv, len(os.sched_getaffinity(0)))


@pytest.mark.parametrize("buckets", [1024, 8192, 32768, 65536])
def test_partition_bounds_under_extreme_skew(buckets):
    """One key fills whole CTAs (>= 65536 equal rows each): the 16-bit shared histogram
    overflows and the CTA falls back to exact global counting (32768 / 65536), or the
    speculative pass 1 overflows its regions and takes the exact fallback while its
    16-bit full-id counters are flushed before they wrap (1024 / 8192); bounds and the
    pair permutation still match a numpy recount of the same bucket function."""
    from paper_2101_08878_b200 import native

    n = 3 * 65536
    rng = np.random.default_rng(4)
    keys = rng.integers(0, 1 << 40, n).astype(np.int64)
    keys[: 2 * 65536] = 123456789  # the first two CTAs (65536 rows each) see one key only
    vals = np.arange(n, dtype=np.int64)
    lib = native.lib()
    k_d, v_d = native.DeviceBuffer(0, n * 8), native.DeviceBuffer(0, n * 8)
    native.memcpy(k_d.ptr, keys.ctypes.data, n * 8)
    native.memcpy(v_d.ptr, vals.ctypes.data, n * 8)
    out = native.DeviceBuffer(0, n * 16)
    bounds = native.DeviceBuffer(0, (buckets + 1) * 8)
    nbytes = lib.m4d_partition_scratch_bytes(n, buckets)
    scratch = native.DeviceBuffer(0, nbytes)
    native.check(lib.m4d_partition(k_d.ptr, v_d.ptr, n, 0, buckets, out.ptr, bounds.ptr, scratch.ptr, nbytes, None))
    native.check(lib.m4d_device_sync(0))
    got_b = np.frombuffer(native.to_host(bounds.ptr, (buckets + 1) * 8), dtype=np.int64)
    pairs = np.frombuffer(native.to_host(out.ptr, n * 16), dtype=np.int64).reshape(n, 2)
    h = oracle.splitmix64_np(keys.view(np.uint64))
    bucket = ((h & np.uint64(0xFFFFFFFF)) >> np.uint64(32 - int(np.log2(buckets)))).astype(np.int64)
    want_b = np.concatenate([[0], np.cumsum(np.bincount(bucket, minlength=buckets))])
    assert np.array_equal(got_b, want_b)
    assert np.array_equal(np.sort(pairs[:, 1]), vals)  # a permutation of the rows
    pb = bucket[pairs[:, 1]]
    assert np.all(np.diff(pb) >= 0)  # grouped by bucket, in bucket order
    assert np.array_equal(pairs[:, 0], keys[pairs[:, 1]])


def _partition_local(keys, buckets):
    from paper_2101_08878_b200 import native

    n = len(keys)
    vals = np.arange(n, dtype=np.int64)
    lib = native.lib()
    k_d, v_d = native.DeviceBuffer(0, n * 8), native.DeviceBuffer(0, n * 8)
    native.memcpy(k_d.ptr, keys.ctypes.data, n * 8)
    native.memcpy(v_d.ptr, vals.ctypes.data, n * 8)
    out = native.DeviceBuffer(0, n * 16)
    bounds = native.DeviceBuffer(0, (buckets + 1) * 8)
    nbytes = lib.m4d_partition_scratch_bytes(n, buckets)
    scratch = native.DeviceBuffer(0, nbytes)
    native.check(lib.m4d_partition(k_d.ptr, v_d.ptr, n, 0, buckets, out.ptr, bounds.ptr, scratch.ptr, nbytes, None))
    native.check(lib.m4d_device_sync(0))
    got_b = np.frombuffer(native.to_host(bounds.ptr, (buckets + 1) * 8), dtype=np.int64)
    pairs = np.frombuffer(native.to_host(out.ptr, n * 16), dtype=np.int64).reshape(n, 2)
    h = oracle.splitmix64_np(keys.view(np.uint64))
    bucket = ((h & np.uint64(0xFFFFFFFF)) >> np.uint64(32 - int(np.log2(buckets)))).astype(np.int64)
    want_b = np.concatenate([[0], np.cumsum(np.bincount(bucket, minlength=buckets))])
    assert np.array_equal(got_b, want_b)
    assert np.array_equal(np.sort(pairs[:, 1]), vals)  # a permutation of the rows
    assert np.all(np.diff(bucket[pairs[:, 1]]) >= 0)  # grouped by bucket, in bucket order
    assert np.array_equal(pairs[:, 0], keys[pairs[:, 1]])


@pytest.mark.parametrize("buckets", [512, 1024, 8192])
@pytest.mark.parametrize("n", [1, 777, 3_000_000])
def test_speculative_pass1_uniform_keys(buckets, n):
    """Two-pass LOCAL partition with the speculative pass 1 (regions sized from the
    mean, no histogram pass): bounds and the row permutation match numpy, including
    inputs smaller than one tile and one-row inputs."""
    rng = np.random.default_rng(n + buckets)
    _partition_local(rng.integers(-(1 << 62), 1 << 62, n).astype(np.int64), buckets)


_SPEC_STORE_SCRIPT = """
import sys
sys.path[:0] = [{root!r}, {tests!r}]
import numpy as np
from test_key_merge_gpu import _partition_local
rng = np.random.default_rng(7)
_partition_local(rng.integers(-(1 << 62), 1 << 62, 3_000_000).astype(np.int64), 8192)
keys = rng.integers(0, 1 << 40, 2_000_000).astype(np.int64)
keys[:1_000_000] = 42
_partition_local(keys, 1024)
print("ok")
"""


@pytest.mark.parametrize("store", ["rows", "bulk"])
def test_speculative_pass1_store_modes(store):
    """The speculative pass 1 with row-by-row stores and with TMA bulk run stores
    (M4D_TILE_STORE, read once per process: one interpreter each), uniform keys and an
    overflowing hot key."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _SPEC_STORE_SCRIPT.format(root=root, tests=os.path.join(root, "tests"))
    out = subprocess.run([sys.executable, "-c", code], env={**os.environ, "M4D_TILE_STORE": store}, cwd=root,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().endswith("ok")


@pytest.mark.parametrize("buckets", [1024, 8192])
@pytest.mark.parametrize("hot", [1, 3, 40])
def test_speculative_pass1_overflow_takes_the_exact_fallback(buckets, hot):
    """Duplicate-heavy keys overflow the speculative regions (one key far above a
    region's mean + 6 sigma); the gated exact fallback must still give exact bounds and
    a permutation grouped by partition."""
    n = 2_000_000
    rng = np.random.default_rng(hot)
    keys = rng.integers(0, 1 << 40, n).astype(np.int64)
    hot_keys = rng.integers(0, 1 << 40, hot)
    keys[: n // 2] = hot_keys[rng.integers(0, hot, n // 2)]
    rng.shuffle(keys)
    _partition_local(keys, buckets)


@pytest.mark.parametrize("world,coarse", [(3, 64), (8, 32), (2, 1)])
def test_owner_coarse_partition_matches_numpy(world, coarse):
    """m4d_partition_owner_coarse: bucket = owner * C + top log2 C bits of the local id."""
    from paper_2101_08878_b200 import native

    n = 300_001
    keys = np.random.default_rng(world).integers(-(1 << 62), 1 << 62, n).astype(np.int64)
    vals = np.arange(n, dtype=np.int64)
    lib = native.lib()
    k_d, v_d = native.DeviceBuffer(0, n * 8), native.DeviceBuffer(0, n * 8)
    native.memcpy(k_d.ptr, keys.ctypes.data, n * 8)
    native.memcpy(v_d.ptr, vals.ctypes.data, n * 8)
    nb = world * coarse
    out, bounds = native.DeviceBuffer(0, n * 16), native.DeviceBuffer(0, (nb + 1) * 8)
    nbytes = lib.m4d_partition_scratch_bytes(n, nb)
    scratch = native.DeviceBuffer(0, nbytes)
    native.check(lib.m4d_partition_owner_coarse(k_d.ptr, v_d.ptr, n, world, coarse, out.ptr, bounds.ptr, scratch.ptr,
                                                nbytes, None))
    native.check(lib.m4d_device_sync(0))
    got_b = np.frombuffer(native.to_host(bounds.ptr, (nb + 1) * 8), dtype=np.int64)
    pairs = np.frombuffer(native.to_host(out.ptr, n * 16), dtype=np.int64).reshape(n, 2)
    h = oracle.splitmix64_np(keys.view(np.uint64))
    owner = ((h >> np.uint64(32)) * np.uint64(world)) >> np.uint64(32)
    cbits = int(np.log2(coarse))
    low = ((h & np.uint64(0xFFFFFFFF)) >> np.uint64(32 - cbits)) if cbits else np.zeros(n, np.uint64)
    bucket = (owner * np.uint64(coarse) + low).astype(np.int64)
    want_b = np.concatenate([[0], np.cumsum(np.bincount(bucket, minlength=nb))])
    assert np.array_equal(got_b, want_b)
    assert np.all(np.diff(bucket[pairs[:, 1]]) >= 0) and np.array_equal(np.sort(pairs[:, 1]), vals)


@pytest.mark.parametrize("shuffle", ["push", "pull"])
def test_shuffle_modes_agree_over_steps(shuffle):
    """Both shuffles (fused push scatter / rendezvous pulls) give the oracle digest, step
    after step on the same buffers."""
    _, got = run_world(30_000, 3, 0.3, shuffle=shuffle, steps=3)
    assert got == oracle.key_merge_c(30_000, 3, 0.3)


def test_push_falls_back_to_pull_when_a_receive_buffer_is_small():
    """A receive buffer too small for a step's rows: every rank takes the pull path (which
    grows it) and maps the new buffers on the next step."""
    calls = {"push": 0, "pull": 0}

    def hook(ranks):
        for km in ranks:
            orig_connect, orig_pull = km._connect_push, km._shuffle_and_partition

            async def connect(km=km, orig=orig_connect, mine=[0]):
                await orig()
                if mine[0] == 0:  # first step only: every rank believes rank 1's buffers are tiny
                    km._peer_cap = [[c if r != 1 else 10 for r, c in enumerate(side)] for side in km._peer_cap]
                mine[0] += 1
                calls["push"] += 1

            async def pull(orig=orig_pull):
                calls["pull"] += 1
                return await orig()

            km._connect_push, km._shuffle_and_partition = connect, pull

    _, got = run_world(30_000, 2, 0.3, shuffle="push", steps=2, hook=hook)
    assert got == oracle.key_merge_c(30_000, 2, 0.3)
    assert calls["pull"] == 2 and calls["push"] == 4  # step 1 fell back on both ranks; step 2 reconnected


@pytest.mark.parametrize("world,coarse", [(3, 64), (8, 32), (2, 1), (1, 256)])
def test_owner_push_matches_owner_coarse(world, coarse):
    """plan + push (the fused owner scatter + shuffle) writes owner d's rows to its own
    destination, bit-identical to segment d of m4d_partition_owner_coarse."""
    from paper_2101_08878_b200 import native

    n = 300_001
    keys = np.random.default_rng(7 + world).integers(-(1 << 62), 1 << 62, n).astype(np.int64)
    vals = np.arange(n, dtype=np.int64)
    lib = native.lib()
    k_d, v_d = native.DeviceBuffer(0, n * 8), native.DeviceBuffer(0, n * 8)
    native.memcpy(k_d.ptr, keys.ctypes.data, n * 8)
    native.memcpy(v_d.ptr, vals.ctypes.data, n * 8)
    nb = world * coarse
    nbytes = lib.m4d_partition_scratch_bytes(n, nb)
    scratch = native.DeviceBuffer(0, nbytes)
    out, bounds = native.DeviceBuffer(0, n * 16), native.DeviceBuffer(0, (nb + 1) * 8)
    native.check(lib.m4d_partition_owner_coarse(k_d.ptr, v_d.ptr, n, world, coarse, out.ptr, bounds.ptr, scratch.ptr,
                                                nbytes, None))
    native.check(lib.m4d_device_sync(0))
    want = np.frombuffer(native.to_host(out.ptr, n * 16), dtype=np.int64).reshape(n, 2)
    want_b = np.frombuffer(native.to_host(bounds.ptr, (nb + 1) * 8), dtype=np.int64)
    bounds2 = native.DeviceBuffer(0, (nb + 1) * 8)
    scratch2 = native.DeviceBuffer(0, nbytes)
    native.check(lib.m4d_partition_owner_plan(k_d.ptr, v_d.ptr, n, world, coarse, bounds2.ptr, scratch2.ptr, nbytes,
                                              None))
    native.check(lib.m4d_device_sync(0))
    got_b = np.frombuffer(native.to_host(bounds2.ptr, (nb + 1) * 8), dtype=np.int64)
    assert np.array_equal(got_b, want_b)
    seg = [int(want_b[d * coarse]) for d in range(world)] + [n]
    dests = [native.DeviceBuffer(0, max(1, seg[d + 1] - seg[d]) * 16 + 4096) for d in range(world)]
    for d in dests:
        native.memset(d.ptr, 0xAB, d.nbytes)
    addrs = (ctypes.c_uint64 * world)(*[d.ptr for d in dests])
    native.check(lib.m4d_partition_owner_push(k_d.ptr, v_d.ptr, n, world, coarse, addrs, scratch2.ptr, nbytes, None))
    native.check(lib.m4d_device_sync(0))
    for d in range(world):
        rows = seg[d + 1] - seg[d]
        got = np.frombuffer(native.to_host(dests[d].ptr, rows * 16 + 4096), dtype=np.uint8)
        assert np.array_equal(got[:rows * 16].view(np.int64).reshape(rows, 2), want[seg[d]:seg[d + 1]])
        assert np.all(got[rows * 16:] == 0xAB)  # nothing written past the segment


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("fraction", [0.0, 0.3, 1.0])
def test_spec_application_oracle(world, fraction):
    """SPEC.md acceptance (application oracles): 10^4 rows per worker, fraction in {0, 0.3, 1},
    workers in {1, 2, 4}: the global digest equals the brute-force join of the oracle."""
    rows = 10_000
    _, got = run_world(rows, world, fraction)
    assert got == oracle.key_merge_c(rows, world, fraction)
    if fraction == 0.0:
        assert got[0] == 0


_VARIANT_SCRIPT = """
import sys
sys.path[:0] = [{root!r}, {tests!r}]
from test_key_merge_gpu import run_world
_, got = run_world({rows}, {world}, 0.3)
print(list(got))
"""


@pytest.mark.parametrize("env", [
    {"M4D_JOIN_PF": "0"},
    {"M4D_JOIN_PF": "7", "M4D_JOIN_PF_AHEAD": "3"},
    {"M4D_JOIN": "small"},
    {"M4D_JOIN": "small", "M4D_JOIN_PART_ROWS": "12400"},  # two build chunks per partition
    {"M4D_JOIN_PERSIST": "1", "M4D_JOIN_PART_ROWS": "500"},  # more partitions than one wave
    {"M4D_PASS1": "hist"},  # histogram pass before pass 1 instead of the speculative regions
])
def test_tuning_knobs_keep_the_digest(env):
    """Every join knob (read once per process, so each runs in its own interpreter) gives
    the oracle's digest: the knobs change the schedule, never the result."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    rows = 400_000
    code = _VARIANT_SCRIPT.format(root=root, tests=os.path.join(root, "tests"), rows=rows, world=1)
    out = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, cwd=root, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    got = tuple(int(x) for x in out.stdout.strip().splitlines()[-1].strip("[]").split(","))
    assert got == tuple(oracle.key_merge_c(rows, 1, 0.3))


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("fine", ["0", "1", "separate"])
def test_counted_receiver_split_matches_the_oracle(world, fine):
    """M4D_MERGE_FINE: receiver splits with the senders' per-partition counts (no
    histogram pass) -- counted by the push itself for both sides (default), or by a
    separate pass for side 1 (M4D_MERGE_FINE_FUSED=0) -- and without; all equal to the
    oracle, over two steps."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _VARIANT_SCRIPT.format(root=root, tests=os.path.join(root, "tests"), rows=200_000, world=world)
    code = code.replace("run_world(200000, %d, 0.3)" % world, "run_world(200000, %d, 0.3, steps=2)" % world)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                         env=dict(os.environ, M4D_MERGE_FINE="1" if fine == "separate" else fine,
                                  M4D_MERGE_FINE_FUSED="0" if fine == "separate" else "1"))
    assert out.returncode == 0, out.stderr[-2000:]
    assert eval(out.stdout.strip().splitlines()[-1]) == list(oracle.key_merge_c(200_000, world, 0.3))


@pytest.mark.parametrize("world", [2, 4])
def test_push_fine_counts_exact_under_extreme_skew(world):
    """m4d_partition_owner_push_fine: the push scatter's own (owner, partition) counts
    spill their 16-bit shared counters exactly under one key repeated 3M times, equal a
    numpy recount, and the pushed rows equal m4d_partition_owner_push's."""
    from paper_2101_08878_b200 import native

    lib = native.lib()
    n, parts = 4_000_000, 8192
    coarse = lib.m4d_owner_coarse_count(world)
    keys = np.full(n, 987654321, dtype=np.int64)
    keys[3_000_000:] = np.arange(1_000_000, dtype=np.int64) * 104729
    vals = np.arange(n, dtype=np.int64)
    k_d, v_d = native.DeviceBuffer(0, n * 8), native.DeviceBuffer(0, n * 8)
    native.memcpy(k_d.ptr, keys.ctypes.data, n * 8)
    native.memcpy(v_d.ptr, vals.ctypes.data, n * 8)
    nb = world * coarse
    nbytes = lib.m4d_partition_scratch_bytes(n, nb)
    scratch = native.DeviceBuffer(0, nbytes)
    bounds = native.DeviceBuffer(0, (nb + 1) * 8)
    native.check(lib.m4d_partition_owner_plan(k_d.ptr, v_d.ptr, n, world, coarse, bounds.ptr, scratch.ptr, nbytes,
                                              None))
    native.check(lib.m4d_device_sync(0))
    b = np.frombuffer(native.to_host(bounds.ptr, (nb + 1) * 8), dtype=np.int64)
    seg = [int(b[d * coarse]) for d in range(world)] + [n]
    outs = []
    for fused in (False, True):
        dests = [native.DeviceBuffer(0, max(1, seg[d + 1] - seg[d]) * 16) for d in range(world)]
        addrs = (ctypes.c_uint64 * world)(*[d.ptr for d in dests])
        counts = native.DeviceBuffer(0, world * parts * 4 + 4)
        native.memset(counts.ptr, 0xFF, world * parts * 4 + 4)  # the call zeroes them
        handed = native.DeviceBuffer(0, world * parts * 4)  # where each owner takes its row
        native.memset(handed.ptr, 0xFF, world * parts * 4)
        cdst = (ctypes.c_uint64 * world)(*[handed.ptr + d * parts * 4 for d in range(world)])
        if fused:
            native.check(lib.m4d_partition_owner_push_fine(k_d.ptr, v_d.ptr, n, world, coarse, addrs, parts,
                                                           counts.ptr, cdst, scratch.ptr, nbytes, None))
        else:
            native.check(lib.m4d_partition_owner_push(k_d.ptr, v_d.ptr, n, world, coarse, addrs, scratch.ptr,
                                                      nbytes, None))
        native.check(lib.m4d_device_sync(0))
        rows = [np.frombuffer(native.to_host(dests[d].ptr, (seg[d + 1] - seg[d]) * 16), dtype=np.int64)
                .reshape(-1, 2) for d in range(world)]
        outs.append([r[np.argsort(r[:, 1], kind="stable")] for r in rows])
        if fused:
            got = np.frombuffer(native.to_host(counts.ptr, world * parts * 4), dtype=np.uint32)
            assert np.array_equal(np.frombuffer(native.to_host(handed.ptr, world * parts * 4), dtype=np.uint32), got)
    for a, c in zip(*outs):
        assert np.array_equal(a, c)
    h = oracle.splitmix64_np(keys.view(np.uint64))
    owner = ((h >> np.uint64(32)) * np.uint64(world)) >> np.uint64(32)
    p = (h & np.uint64(0xFFFFFFFF)) >> np.uint64(32 - 13)
    want = np.bincount((owner * np.uint64(parts) + p).astype(np.int64), minlength=world * parts)
    assert np.array_equal(got.astype(np.int64), want)


def test_fine_counts_exact_under_extreme_skew():
    """m4d_partition_fine_counts' 16-bit shared counters spill to the global count:
    one key repeated 6M times (every CTA of the first three quarters sees ~54K rows of
    one (owner, partition) counter, so it spills) and a spread remainder count exactly
    (numpy reference of the same hash)."""
    from paper_2101_08878_b200 import native

    n, world, parts = 8_000_000, 4, 8192
    keys = np.full(n, 123456789, dtype=np.int64)
    keys[6_000_000:] = np.arange(2_000_000, dtype=np.int64) * 7919
    vals = np.arange(n, dtype=np.int64)
    d_k, d_v = native.DeviceBuffer(0, n * 8), native.DeviceBuffer(0, n * 8)
    out = native.DeviceBuffer(0, world * parts * 4)
    native.memcpy(d_k.ptr, keys.ctypes.data, n * 8)
    native.memcpy(d_v.ptr, vals.ctypes.data, n * 8)
    native.check(native.lib().m4d_partition_fine_counts(d_k.ptr, d_v.ptr, n, world, parts, out.ptr, None))
    got = np.frombuffer(native.to_host(out.ptr, world * parts * 4), dtype=np.uint32)
    h = oracle.splitmix64_np(keys.view(np.uint64))
    owner = ((h >> np.uint64(32)) * np.uint64(world)) >> np.uint64(32)
    p = (h & np.uint64(0xFFFFFFFF)) >> np.uint64(32 - 13)
    want = np.bincount((owner * np.uint64(parts) + p).astype(np.int64), minlength=world * parts)
    assert np.array_equal(got.astype(np.int64), want)
