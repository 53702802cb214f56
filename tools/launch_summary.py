"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: per-kernel launches, mean ms, share."""
import csv
import sys
from collections import defaultdict

SCALE = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}


def main(path: str, title: str) -> None:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = defaultdict(list)
    for r in rows[1:]:
        per[r[ki].split("(")[0].replace("<unnamed>::", "")].append(float(r[vi].replace(",", "")) * SCALE[r[ui]])
    total = sum(sum(v) for v in per.values())
    print(f"# {title}")
    print("# gpu__time_duration per launch (ncu --clock-control none): cold-cache and serialised,")
    print("# so compare each kernel's SHARE of the step with bench.py, not the absolute times.")
    print(f"{'kernel':32s} {'launches':>8s} {'mean ms':>9s} {'total ms':>9s} {'share':>7s}")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:32s} {len(v):8d} {sum(v) / len(v):9.4f} {sum(v):9.3f} {100 * sum(v) / total:6.2f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
