"""Profile the in-process storm (2 ranks on cuda:0) with host and device frames:
frames/s and the top functions by own time.  Diagnostics for the device-frame path.

    python tools/storm_profile.py [total] [--no-profile]
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from nvlink_fixtures import close_all, nvlink_transports  # noqa: E402
from paper_2101_08878_b200.harness import storm  # noqa: E402

total = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 20000
prof = "--no-profile" not in sys.argv
ns = storm.namespace_of("paper_2101_08878_b200")
for dev in (None, 0):
    ts = nvlink_transports(2, 0)
    storm.run_local(ns, ts, conns=8, total=total, rounds=1, device=dev)
    t0 = time.perf_counter()
    pr = cProfile.Profile()
    if prof:
        pr.enable()
    r = storm.run_local(ns, ts, conns=8, total=total, rounds=1, device=dev)
    pr.disable()
    print("device", dev, "frames/s", round(r.frames_per_s), "wall", round(time.perf_counter() - t0, 3),
          "stats", {k: v for k, v in ts[0].native_stats().items() if "eager" in k or "pull" in k})
    if prof:
        pstats.Stats(pr).sort_stats("tottime").print_stats(12)
    close_all(ts)
