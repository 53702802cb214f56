"""transpose_sum parity on a B200: the fused kernel vs the CPU oracle.

Bars (north_star): y bit-exact, sum within 1e-12 relative, and the checksum
identical for every worker count.
"""

import math

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

REL_TOL = 1e-12  # fp64 sum tolerance stated by north_star


@pytest.fixture(params=["tma", "ldg"])
def kernel_path(request, monkeypatch):
    """Both kernels: the TMA-fed persistent one and the LDG fallback."""
    if request.param == "ldg":
        monkeypatch.setenv("M4D_TS_FORCE_LDG", "1")
    else:
        monkeypatch.delenv("M4D_TS_FORCE_LDG", raising=False)
    return request.param


def run_world(n, b, world, seed=oracle.SEED_X):
    from paper_2101_08878_b200.harness.transpose_sum import TransposeSum

    ranks = TransposeSum.local_world(n, b, world, seed=seed)
    import os
    from paper_2101_08878_b200 import native

    want_tma = not os.environ.get("M4D_TS_FORCE_LDG") and b % 2 == 0
    for r in ranks:
        assert native.lib().m4d_ts_plan_uses_tma(r._plan) == int(want_tma)
    merged = {}
    for r in ranks:
        r.launch()
    for r in ranks:
        merged.update(r.read_block_sums())
    return ranks, merged, math.fsum(merged[g] for g in sorted(merged))


def y_block(ranks, g):
    for r in ranks:
        if g in r.slot_of:
            b = r.b
            return np.frombuffer(r.read_y_block(g), dtype=np.float64).reshape(b, b)
    raise KeyError(g)


@pytest.mark.parametrize("n,b", [(256, 64), (300, 100), (4096, 1024), (130, 65), (2000, 2000), (96, 1)])
def test_single_gpu_matches_oracle_bit_exact(cuda, kernel_path, n, b):
    ranks, sums, total = run_world(n, b, 1)
    nb = n // b
    want_sums, want_total = oracle.transpose_sum_checksum(n, b, threads=8)
    for g in range(nb * nb):
        assert sums[g] == pytest.approx(want_sums[g], rel=REL_TOL, abs=1e-300)
    assert abs(total - want_total) <= REL_TOL * abs(want_total)
    for g in list(range(nb * nb))[:: max(1, (nb * nb) // 7)]:
        i, j = divmod(g, nb)
        a = oracle.gen_block_c(n, i * b, j * b, b)
        bt = oracle.gen_block_c(n, j * b, i * b, b)
        assert np.array_equal(y_block(ranks, g), oracle.transpose_block_c(a, bt)), f"y block {g}"


def test_numpy_restatement_agrees_at_small_size(cuda):
    n, b = 192, 64
    x = np.vstack([np.hstack([oracle.gen_block_np(n, i * b, j * b, b) for j in range(3)]) for i in range(3)])
    y, _sums, total = oracle.transpose_sum_np(x, b)
    ranks, _, got = run_world(n, b, 1)
    assert abs(got - total) <= REL_TOL * abs(total)
    for g in range(9):
        i, j = divmod(g, 3)
        assert np.array_equal(y_block(ranks, g), y[i * b:(i + 1) * b, j * b:(j + 1) * b])


@pytest.mark.parametrize("world", [2, 3, 4, 5])
def test_checksum_independent_of_worker_count(cuda, kernel_path, world):
    n, b = 1024, 128
    _, sums1, total1 = run_world(n, b, 1)
    ranks, sums_w, total_w = run_world(n, b, world)
    assert total_w == total1  # bit-identical, not just close
    assert sums_w == sums1
    assert sum(r.tasks_single for r in ranks) > 0  # the remote-partner path ran
    nb = n // b
    for g in (1, nb, nb + 3, nb * nb - 2):
        i, j = divmod(g, nb)
        a = oracle.gen_block_c(n, i * b, j * b, b)
        bt = oracle.gen_block_c(n, j * b, i * b, b)
        assert np.array_equal(y_block(ranks, g), oracle.transpose_block_c(a, bt))


def test_spec_example_two_by_two(cuda):
    """x = [[0,1],[2,3]] -> y = [[0,3],[3,6]] (block 1, 2 workers as well)."""
    from paper_2101_08878_b200 import native
    from paper_2101_08878_b200.harness.transpose_sum import TransposeSum

    for world in (1, 2):
        ranks = [TransposeSum(2, 1, rank=r, world=world, exchange=lambda _b: []) for r in range(world)]
        x = np.array([[0.0, 1.0], [2.0, 3.0]])
        for r in ranks:
            for g in r.owned:
                i, j = divmod(g, 2)
                blob = np.array([x[i, j]]).tobytes()
                import ctypes

                buf = ctypes.create_string_buffer(blob, 8)
                native.memcpy(r.x_ptr(g), ctypes.addressof(buf), 8)
        native.check(native.lib().m4d_device_sync(0))
        for r in ranks:
            for p in ranks:
                if p is not r:
                    r._peer_bases[p.rank] = p.x.ptr
            r.build_plan()
            r.launch()
        got = np.array([[y_block(ranks, 0)[0, 0], y_block(ranks, 1)[0, 0]],
                        [y_block(ranks, 2)[0, 0], y_block(ranks, 3)[0, 0]]])
        assert np.array_equal(got, np.array([[0.0, 3.0], [3.0, 6.0]]))
        sums = {}
        for r in ranks:
            sums.update(r.read_block_sums())
        assert math.fsum(sums.values()) == 12.0


def test_full_config_sampled_blocks(cuda):
    """BASELINE config 3 at one GPU: 40000^2 in 2000^2 chunks, sampled blocks vs the oracle."""
    n, b = 40000, 2000
    ranks, sums, total = run_world(n, b, 1)
    nb = n // b
    sample = [0, 1, nb, nb + 1, 7 * nb + 13, nb * nb - 1, 13 * nb + 7]
    want = oracle.transpose_sum_blocks_c(n, b, sample, threads=8)
    for g, w in zip(sample, want):
        assert abs(sums[g] - w) <= REL_TOL * abs(w)
    g = 7 * nb + 13
    a = oracle.gen_block_c(n, 7 * b, 13 * b, b)
    bt = oracle.gen_block_c(n, 13 * b, 7 * b, b)
    assert np.array_equal(y_block(ranks, g), oracle.transpose_block_c(a, bt))
    # size-independent property: y(i,j) == y(j,i)^T bit-exactly
    assert np.array_equal(y_block(ranks, 13 * nb + 7), y_block(ranks, g).T)
    # run-to-run determinism
    for r in ranks:
        r.launch()
    again = {}
    for r in ranks:
        again.update(r.read_block_sums())
    assert again == sums


def test_two_gpus_partner_tiles_read_over_nvlink(cuda):
    """Ranks on distinct B200s: the TMA producer reads peer HBM through NVLink."""
    from paper_2101_08878_b200 import native
    from paper_2101_08878_b200.harness.transpose_sum import TransposeSum

    if native.device_count() < 2:
        pytest.skip("needs two GPUs")
    n, b = 2048, 256
    ranks = TransposeSum.local_world(n, b, 2, devices=[0, 1])
    for r in ranks:
        r.launch()
    sums = {}
    for r in ranks:
        sums.update(r.read_block_sums())
    want_sums, want = oracle.transpose_sum_checksum(n, b, threads=8)
    assert abs(math.fsum(sums[g] for g in sorted(sums)) - want) <= REL_TOL * want
    assert sum(r.tasks_single for r in ranks) > 0
    for g in (1, 9, 17):
        i, j = divmod(g, n // b)
        a = oracle.gen_block_c(n, i * b, j * b, b)
        bt = oracle.gen_block_c(n, j * b, i * b, b)
        assert np.array_equal(y_block(ranks, g), oracle.transpose_block_c(a, bt))
