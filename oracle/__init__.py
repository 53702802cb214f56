"""CPU oracle for the commshim B200 hot path — TEST INFRASTRUCTURE ONLY.

Importable by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs, as the checker or the timed CPU
baseline; the product package ``paper_2101_08878_b200`` never imports it.

Two independent restatements live here:

* ``liboracle.so`` (``oracle/oracle.c``): the C restatement used at scale;
* the numpy/pandas functions below: a second, independent restatement used to
  pin the C one (together with the worked examples of SPEC.md:418-430 in
  ``tests/golden/spec_examples.json``).

Reference anchors: transpose_sum SPEC.md:413-421, :441-449, PAPER.md:380-383;
key_merge SPEC.md:422-430, :449.  The reference has no
operator implementation, so operator parity is pinned by the
spec's examples and by numpy/pandas, not by reference code; the comm path is
pinned by golden vectors generated from the reference itself
(``oracle/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

SEED_X = 0x210108878          # transpose_sum generator seed
SEED_LEFT = 0x4C454654        # key_merge left side ("LEFT")
SEED_RIGHT = 0x52494748       # key_merge right side ("RIGH")

_MASK64 = (1 << 64) - 1


class JoinResult(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int64), ("hash_sum", ctypes.c_uint64), ("key_sum", ctypes.c_uint64)]

    def as_tuple(self):
        return int(self.count), int(self.hash_sum), int(self.key_sum)


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        h = ctypes.CDLL(LIB_PATH)
        i64, u64, p = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
        h.orc_splitmix64.restype = u64
        h.orc_splitmix64.argtypes = [u64]
        h.orc_fill_block.restype = None
        h.orc_fill_block.argtypes = [p, i64, i64, i64, i64, u64]
        h.orc_transpose_add.restype = None
        h.orc_transpose_add.argtypes = [p, p, p, i64]
        h.orc_sum.restype = ctypes.c_double
        h.orc_sum.argtypes = [p, i64]
        h.orc_transpose_sum_blocks.restype = ctypes.c_int
        h.orc_transpose_sum_blocks.argtypes = [i64, i64, u64, p, i64, p, ctypes.c_int]
        h.orc_transpose_sum_resident.restype = ctypes.c_int
        h.orc_transpose_sum_resident.argtypes = [p, p, p, i64, i64, p, ctypes.c_int]
        h.orc_gen_side.restype = None
        h.orc_gen_side.argtypes = [p, p, i64, i64, u64, u64, u64]
        h.orc_row_hash.restype = u64
        h.orc_row_hash.argtypes = [i64, i64, i64]
        h.orc_hash_join.restype = ctypes.c_int
        h.orc_hash_join.argtypes = [p, p, i64, p, p, i64, p, p, p, i64, ctypes.POINTER(JoinResult)]
        h.orc_join_mt.restype = ctypes.c_int
        h.orc_join_mt.argtypes = [p, p, i64, p, p, i64, ctypes.c_int, ctypes.POINTER(JoinResult)]
        h.orc_key_merge.restype = ctypes.c_int
        h.orc_key_merge.argtypes = [i64, ctypes.c_int, ctypes.c_double, u64, u64, ctypes.POINTER(JoinResult)]
        _lib = h
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# -- generators ----------------------------------------------------------------------------


def splitmix64_np(z: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 over uint64 (numpy restatement; wraps mod 2^64)."""
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z += np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def gen_block_np(n: int, r0: int, c0: int, b: int, seed: int = SEED_X) -> np.ndarray:
    rows = np.arange(r0, r0 + b, dtype=np.uint64)[:, None]
    cols = np.arange(c0, c0 + b, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        g = rows * np.uint64(n) + cols
    z = splitmix64_np(np.uint64(seed) ^ g)
    return (z >> np.uint64(11)).astype(np.float64) * 2.0**-53


def gen_block_c(n: int, r0: int, c0: int, b: int, seed: int = SEED_X) -> np.ndarray:
    out = np.empty((b, b), dtype=np.float64)
    lib().orc_fill_block(_ptr(out), n, r0, c0, b, seed)
    return out


def merge_band(total: int, fraction: float) -> int:
    """floor((1 - f) * total) in IEEE double, the overlap band start."""
    return int(math.floor((1.0 - fraction) * float(total)))


def gen_side_np(row0: int, count: int, total: int, seed: int, band: int = 0):
    g = np.arange(row0, row0 + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = splitmix64_np(np.uint64(seed) + g)
    keys = (np.uint64(band) + z % np.uint64(total)).astype(np.int64)
    return keys, g.astype(np.int64)


def gen_side_c(row0: int, count: int, total: int, seed: int, band: int = 0):
    k = np.empty(count, dtype=np.int64)
    v = np.empty(count, dtype=np.int64)
    lib().orc_gen_side(_ptr(k), _ptr(v), row0, count, total, seed, band)
    return k, v


# -- transpose_sum ----------------------------------------------------------------------------


def transpose_sum_np(x: np.ndarray, b: int):
    """SPEC.md:413-417 restated with numpy: y = x + x.T blockwise, per-block
    np.sum, client-side math.fsum over blocks in row-major order."""
    n = x.shape[0]
    if x.shape != (n, n) or n % b:
        raise ValueError("dims must be square and divisible by the block")
    nb = n // b
    y = np.empty_like(x)
    sums = []
    for i in range(nb):
        for j in range(nb):
            blk = x[i * b:(i + 1) * b, j * b:(j + 1) * b] + x[j * b:(j + 1) * b, i * b:(i + 1) * b].T
            y[i * b:(i + 1) * b, j * b:(j + 1) * b] = blk
            sums.append(float(np.sum(blk)))
    return y, sums, math.fsum(sums)


def transpose_sum_blocks_c(n: int, b: int, block_ids, seed: int = SEED_X, threads: int = 1) -> np.ndarray:
    ids = np.ascontiguousarray(np.asarray(block_ids, dtype=np.int64))
    out = np.empty(len(ids), dtype=np.float64)
    rc = lib().orc_transpose_sum_blocks(n, b, seed, _ptr(ids), len(ids), _ptr(out), threads)
    if rc:
        raise RuntimeError(f"orc_transpose_sum_blocks failed ({rc})")
    return out


def transpose_sum_resident_c(a_blocks, bt_blocks, y_blocks, threads: int = 1) -> np.ndarray:
    """Time-able CPU compute of y = a + bt^T and per-block sums over resident inputs."""
    n = len(a_blocks)
    b = a_blocks[0].shape[0]
    arr = lambda blocks: (ctypes.c_void_p * n)(*[blk.ctypes.data for blk in blocks])  # noqa: E731
    sums = np.empty(n, dtype=np.float64)
    lib().orc_transpose_sum_resident(arr(a_blocks), arr(bt_blocks), arr(y_blocks), n, b, _ptr(sums), threads)
    return sums


def transpose_block_c(a: np.ndarray, bt: np.ndarray) -> np.ndarray:
    b = a.shape[0]
    a = np.ascontiguousarray(a, dtype=np.float64)
    bt = np.ascontiguousarray(bt, dtype=np.float64)
    y = np.empty_like(a)
    lib().orc_transpose_add(_ptr(a), _ptr(bt), _ptr(y), b)
    return y


def transpose_sum_checksum(n: int, b: int, seed: int = SEED_X, threads: int = 1) -> tuple[list, float]:
    nb = n // b
    sums = transpose_sum_blocks_c(n, b, range(nb * nb), seed, threads)
    return list(map(float, sums)), math.fsum(sums)


# -- key_merge ------------------------------------------------------------------------------------


def row_hash_np(k: np.ndarray, l: np.ndarray, r: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        h = splitmix64_np(k.astype(np.uint64) ^ np.uint64(0x6B65795F6D657267))
        h = splitmix64_np(h ^ l.astype(np.uint64))
        return splitmix64_np(h ^ (r.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)))


def join_digest_np(k, l, r) -> tuple[int, int, int]:
    """(row count, sum of row hashes mod 2^64, sum of keys mod 2^64): order-independent."""
    k = np.asarray(k, dtype=np.int64)
    hs = int(row_hash_np(k, np.asarray(l, np.int64), np.asarray(r, np.int64)).sum(dtype=np.uint64))
    ks = int(k.astype(np.uint64).sum(dtype=np.uint64))
    return len(k), hs & _MASK64, ks & _MASK64


def hash_join_c(lk, lv, rk, rv, want_rows: bool = False):
    lk, lv, rk, rv = (np.ascontiguousarray(a, dtype=np.int64) for a in (lk, lv, rk, rv))
    res = JoinResult()
    cap = 0
    outs = (None, None, None)
    if want_rows:
        cap = len(lk) * 4 + len(rk) * 4 + 16
        outs = tuple(np.empty(cap, dtype=np.int64) for _ in range(3))
    rc = lib().orc_hash_join(_ptr(lk), _ptr(lv), len(lk), _ptr(rk), _ptr(rv), len(rk),
                             *(None if o is None else _ptr(o) for o in outs), cap, ctypes.byref(res))
    if rc:
        raise RuntimeError(f"orc_hash_join failed ({rc})")
    if want_rows:
        n = int(res.count)
        if n > cap:
            raise RuntimeError("oracle output capacity exceeded")
        return res.as_tuple(), tuple(o[:n] for o in outs)
    return res.as_tuple()


def join_mt_c(lk, lv, rk, rv, threads: int) -> tuple[int, int, int]:
    """Digest of the inner join of resident tables with `threads` POSIX threads (radix
    partition + per-partition hash joins): the timed CPU baseline of key_merge."""
    lk, lv, rk, rv = (np.ascontiguousarray(a, dtype=np.int64) for a in (lk, lv, rk, rv))
    res = JoinResult()
    rc = lib().orc_join_mt(_ptr(lk), _ptr(lv), len(lk), _ptr(rk), _ptr(rv), len(rk), threads, ctypes.byref(res))
    if rc:
        raise RuntimeError(f"orc_join_mt failed ({rc})")
    return res.as_tuple()


def key_merge_c(rows_per_worker: int, workers: int, fraction: float,
                seed_l: int = SEED_LEFT, seed_r: int = SEED_RIGHT) -> tuple[int, int, int]:
    res = JoinResult()
    rc = lib().orc_key_merge(rows_per_worker, workers, fraction, seed_l, seed_r, ctypes.byref(res))
    if rc:
        raise RuntimeError(f"orc_key_merge failed ({rc})")
    return res.as_tuple()


def key_merge_pandas(rows_per_worker: int, workers: int, fraction: float,
                     seed_l: int = SEED_LEFT, seed_r: int = SEED_RIGHT):
    """Independent restatement with pandas.merge (no partitioning): global digest."""
    import pandas as pd

    total = rows_per_worker * workers
    band = merge_band(total, fraction)
    lk, lv = gen_side_np(0, total, total, seed_l, 0)
    rk, rv = gen_side_np(0, total, total, seed_r, band)
    out = pd.merge(pd.DataFrame({"key": lk, "lval": lv}), pd.DataFrame({"key": rk, "rval": rv}),
                   on="key", how="inner")
    return join_digest_np(out["key"].to_numpy(), out["lval"].to_numpy(), out["rval"].to_numpy())
