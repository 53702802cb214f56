"""commshim-bench (SPEC.md benchcli): CSV schema, sweeps,
virtual-clock determinism, progress-mode ordering, oracle-gated app runs."""

import pytest

from paper_2101_08878_b200 import benchcli
from paper_2101_08878_b200.errors import UsageError


def test_size_specs():
    assert benchcli.parse_sizes("1:16:x2") == [1, 2, 4, 8, 16]
    assert benchcli.parse_sizes("0:4:x2") == [0, 1, 2, 4]
    assert benchcli.parse_sizes("10:30:+10") == [10, 20, 30]
    assert benchcli.parse_sizes("3,5,9") == [3, 5, 9]
    for bad in ("5,3", "", "1:8:x1", "1:8:*2"):
        with pytest.raises(UsageError):
            benchcli.parse_sizes(bad)


def test_csv_schema_and_parse_back(tmp_path):
    recs = [benchcli.BenchRecord("pingpong", "sim", "cooperative", 1, 100, 1.0000000000000002e-06, 1e-06,
                                 1.5e-06, 999999.99999999988)]
    text = benchcli.emit(recs, "csv", str(tmp_path / "out.csv"))
    assert text.splitlines()[0] == ",".join(benchcli.CSV_COLUMNS)
    assert len(text.splitlines()) == 2
    back = benchcli.parse_csv((tmp_path / "out.csv").read_text())
    assert [(r.mean_s, r.throughput_Bps, r.size) for r in back] == [(r.mean_s, r.throughput_Bps, r.size) for r in recs]
    assert "pingpong" in benchcli.emit(recs, "table")
    with pytest.raises(UsageError):
        benchcli.emit([], "csv")
    with pytest.raises(OSError, match="nope"):
        benchcli.emit(recs, "csv", str(tmp_path / "nope" / "x.csv"))


def test_sim_pingpong_is_deterministic_on_the_virtual_clock():
    a = benchcli.pingpong([0, 1, 1024, 1 << 20], transport="sim", warmup=2, iters=5)
    b = benchcli.pingpong([0, 1, 1024, 1 << 20], transport="sim", warmup=2, iters=5)
    key = lambda rs: [(r.size, r.mean_s, r.median_s, r.p99_s, r.throughput_Bps) for r in rs]  # noqa: E731
    assert key(a) == key(b)
    assert all(r.mean_s > 0 for r in a)
    assert a[-1].throughput_Bps == pytest.approx(2 * a[-1].size / (2 * a[-1].mean_s))


def test_cooperative_beats_periodic_at_every_size():
    sizes = [1, 64, 4096, 65536]
    coop = benchcli.pingpong(sizes, transport="sim", mode="cooperative", warmup=1, iters=5)
    per = benchcli.pingpong(sizes, transport="sim", mode="periodic:1", warmup=1, iters=5)
    for c, p in zip(coop, per):
        assert c.mean_s <= p.mean_s
    assert per[0].mean_s >= 2 * coop[0].mean_s  # SPEC.md:532 progress-mode A/B at 1 B


def test_nvlink_host_pingpong_sweep():
    recs = benchcli.pingpong([1, 4096, 1 << 20], transport="nvlink", warmup=2, iters=10)
    assert [r.size for r in recs] == [1, 4096, 1 << 20] and all(r.mean_s > 0 for r in recs)


def test_cli_exit_codes(capsys):
    assert benchcli.main(["pingpong", "--sizes", "1,8", "--warmup", "1", "--iters", "3"]) == 0
    assert capsys.readouterr().out.startswith("benchmark,transport,mode,size")
    assert benchcli.main(["pingpong", "--mode", "sometimes"]) == 2
    assert benchcli.main(["frobnicate"]) == 2


@pytest.mark.gpu
def test_apps_pass_the_oracle_gate_on_b200(capsys):
    assert benchcli.main(["app", "transpose-sum", "--dims", "2048", "--block", "512", "--workers", "2"]) == 0
    assert benchcli.main(["app", "key-merge", "--rows", "200000", "--repetitions", "2"]) == 0
    assert benchcli.main(["pingpong", "--transport", "nvlink", "--device", "--sizes", "1,1048576",
                          "--iters", "10", "--table"]) == 0
    assert "transpose_sum" in capsys.readouterr().out
