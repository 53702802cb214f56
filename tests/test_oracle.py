"""The CPU oracle pinned against SPEC.md's worked examples and independent numpy/pandas restatements."""

import json
import math
import os

import numpy as np
import pytest

import oracle

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_comm.json")))


def test_spec_transpose_examples():
    for name in ("transpose_2x2", "transpose_symmetric"):
        ex = GOLDEN["spec_examples"][name]
        x = np.array(ex["x"], dtype=np.float64)
        y, _sums, total = oracle.transpose_sum_np(x, 1)
        assert np.array_equal(y, np.array(ex["y"], dtype=np.float64))
        assert total == ex["sum"]
        # C restatement, block by block
        for i in range(2):
            for j in range(2):
                got = oracle.transpose_block_c(x[i:i + 1, j:j + 1], x[j:j + 1, i:i + 1])
                assert got[0, 0] == ex["y"][i][j]


def test_symmetric_input_doubles():
    """symmetric x gives y = 2x (checksum doubles)."""
    rng = np.random.default_rng(3)
    a = rng.random((64, 64))
    x = a + a.T
    y, _, total = oracle.transpose_sum_np(x, 16)
    assert np.array_equal(y, 2 * x)
    assert total == pytest.approx(2 * math.fsum(x.ravel()), rel=1e-15)


def test_generators_agree_c_vs_numpy():
    for (n, r0, c0, b) in [(256, 0, 0, 64), (40000, 38000, 2000, 16), (4096, 1024, 3072, 33)]:
        assert np.array_equal(oracle.gen_block_np(n, r0, c0, b), oracle.gen_block_c(n, r0, c0, b))
    for seed, band in [(oracle.SEED_LEFT, 0), (oracle.SEED_RIGHT, 700)]:
        kn, vn = oracle.gen_side_np(5000, 3000, 10000, seed, band)
        kc, vc = oracle.gen_side_c(5000, 3000, 10000, seed, band)
        assert np.array_equal(kn, kc) and np.array_equal(vn, vc)


def test_generator_value_range_and_resolution():
    x = oracle.gen_block_c(4096, 0, 0, 256)
    assert x.min() >= 0.0 and x.max() < 1.0
    assert np.all(np.mod(x * 2.0**53, 1.0) == 0.0)  # exact multiples of 2^-53


def test_c_transpose_sum_matches_numpy_restatement():
    n, b = 384, 128
    x = np.vstack([np.hstack([oracle.gen_block_np(n, i * b, j * b, b) for j in range(3)]) for i in range(3)])
    _y, sums_np, total_np = oracle.transpose_sum_np(x, b)
    sums_c, total_c = oracle.transpose_sum_checksum(n, b, threads=4)
    for s_np, s_c in zip(sums_np, sums_c):
        assert s_c == pytest.approx(s_np, rel=1e-14)
    assert abs(total_c - total_np) <= 1e-13 * total_np


def test_checksum_independent_of_block_partitioning_order():
    """the checksum does not depend on worker count; the oracle's fsum of
    per-block sums is the same whatever order blocks are produced in."""
    n, b = 512, 64
    sums, total = oracle.transpose_sum_checksum(n, b, threads=3)
    rng = np.random.default_rng(11)
    perm = rng.permutation(len(sums))
    assert math.fsum([sums[k] for k in perm]) == total


def test_spec_merge_examples():
    ex = GOLDEN["spec_examples"]["merge_small"]
    lk = np.array(ex["left"], dtype=np.int64)
    rk = np.array(ex["right"], dtype=np.int64)
    res = oracle.hash_join_c(lk, np.arange(3), rk, np.arange(3))
    assert res[0] == ex["rows"]
    assert oracle.key_merge_c(1000, 2, 0.0)[0] == GOLDEN["spec_examples"]["merge_fraction_zero_rows"]


@pytest.mark.parametrize("rows,fraction", [(10_000, 0.0), (10_000, 0.3), (10_000, 1.0), (3_000, 0.5)])
def test_merge_oracle_worker_count_independent_and_matches_pandas(rows, fraction):
    """1-, 2- and 4-worker results equal each other and a brute-force join."""
    total = rows * 4
    want = oracle.key_merge_pandas(total, 1, fraction)
    for workers in (1, 2, 4):
        assert oracle.key_merge_c(total // workers, workers, fraction) == want


def test_merge_expected_output_fraction():
    rows, fr = 200_000, 0.3
    count, _, _ = oracle.key_merge_c(rows, 1, fr)
    assert abs(count / rows - fr) < 0.01


def test_hash_join_rows_match_pandas_multiset():
    import pandas as pd

    rng = np.random.default_rng(5)
    lk = rng.integers(0, 500, 2000)
    rk = rng.integers(250, 800, 1500)
    lv = np.arange(2000)
    rv = np.arange(1500) + 10_000
    (count, hs, ks), (ok, ol, orr) = oracle.hash_join_c(lk, lv, rk, rv, want_rows=True)
    df = pd.merge(pd.DataFrame({"key": lk, "lval": lv}), pd.DataFrame({"key": rk, "rval": rv}), on="key")
    got = sorted(zip(ok.tolist(), ol.tolist(), orr.tolist()))
    want = sorted(zip(df["key"], df["lval"], df["rval"]))
    assert got == want and count == len(want)
    assert (count, hs, ks) == oracle.join_digest_np(df["key"].to_numpy(), df["lval"].to_numpy(), df["rval"].to_numpy())


@pytest.mark.parametrize("rows,threads", [(0, 4), (1, 1), (20_000, 1), (20_000, 7), (300_000, 8)])
def test_multithreaded_join_digest_equals_single_threaded(rows, threads):
    """orc_join_mt (the timed CPU baseline: radix partition + per-partition joins) gives the
    key_merge oracle's digest for every thread count, duplicates included."""
    band = oracle.merge_band(rows, 0.3) if rows else 0
    lk, lv = oracle.gen_side_c(0, rows, max(rows, 1), oracle.SEED_LEFT, 0)
    rk, rv = oracle.gen_side_c(0, rows, max(rows, 1), oracle.SEED_RIGHT, band)
    assert oracle.join_mt_c(lk, lv, rk, rv, threads) == oracle.key_merge_c(rows, 1, 0.3)
    m = min(rows, 20_000)
    dup = np.arange(m, dtype=np.int64) % 97  # heavy duplicates
    assert (oracle.join_mt_c(dup, lv[:m], dup[::-1].copy(), rv[:m], threads)
            == oracle.hash_join_c(dup, lv[:m], dup[::-1].copy(), rv[:m]))
