"""Summarise an `ncu --metrics ... --csv --log-file` launch list: one row per kernel launch."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
head = None
launches = OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        head = r
        continue
    if not head or len(r) < len(head):
        continue
    d = dict(zip(head, r))
    key = (d["ID"], d["Kernel Name"][:60], d.get("Device", ""))
    v = d["Metric Value"].replace(",", "")
    unit = d["Metric Unit"]
    try:
        val = float(v)
    except ValueError:
        continue
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1, "usecond": 1e-3,
             "msecond": 1, "nsecond": 1e-6}.get(unit, 1)
    launches.setdefault(key, {})[d["Metric Name"]] = val * scale
filt = sys.argv[2] if len(sys.argv) > 2 else ""
for (i, name, dev), m in launches.items():
    if filt and filt not in name:
        continue
    ms = m.get("gpu__time_duration.sum", 0)
    def gb(k):
        return m.get(k, 0) / 1e9
    print(f"{i:>4} dev{dev} {name:60s} {ms:8.3f} ms  dram r/w {gb('dram__bytes_read.sum'):6.3f}/{gb('dram__bytes_write.sum'):6.3f} GB"
          f"  nvl tx/rx {gb('nvltx__bytes.sum'):6.3f}/{gb('nvlrx__bytes.sum'):6.3f} GB (user {gb('nvltx__bytes_data_user.sum'):6.3f}/{gb('nvlrx__bytes_data_user.sum'):6.3f})"
          + (f"  {gb('nvlrx__bytes_data_user.sum') / (ms * 1e-3):6.1f} GB/s rx-user" if ms else ""))
